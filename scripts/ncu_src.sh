# Full ncu capture (source-level) of window_kernel + copy_kernel for one sweep setting.
tag=$1; shift
ncu --set full --import-source on --cache-control none --clock-control none -k regex:"window_kernel|copy_kernel" -s 6 -c 2 \
    -o gpurun_out/src_${tag} -f python tools/sweep.py --reps 2 --only "$@" > gpurun_out/src_${tag}.log 2>&1
tail -2 gpurun_out/src_${tag}.log
