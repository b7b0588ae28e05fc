# One full ncu capture of the sampler kernel on the bench workload (1 GPU), plus the launch list
# of our kernels in the same bench command.
# usage: bash scripts/ncu_sample.sh <tag> [extra bench args]
tag=${1:-r1}; shift
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"window_kernel|copy_kernel" -s 6 -c 2 \
    -o gpurun_out/prof_${tag} -f python bench.py --steps 2 --warmup 3 --no-e2e --no-per-batch --no-cpu-baseline "$@" > gpurun_out/ncu_${tag}.log 2>&1
tail -2 gpurun_out/ncu_${tag}.log
if [ -n "$LAUNCHES" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'sample_kernel|radix|scan|validate|index_build|gather' \
    --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 4 --warmup 3 --no-e2e --no-per-batch --no-cpu-baseline "$@" > gpurun_out/launches_${tag}.log 2>&1
fi
