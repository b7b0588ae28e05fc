# One ncu --set full capture (with source) of the sampler's window + copy kernels on a config,
# through tools/ktime.py (1 GPU).  usage: bash scripts/ncu_full_ktime.sh <config> <tag> [ENV=VAL ...]
cfg=${1:-C5}; tag=${2:-full}; shift 2
mkdir -p gpurun_out/full
env "$@" ncu --set full --import-source on --clock-control none -k regex:"window_kernel|copy_kernel" -s 8 -c 2 \
  --metrics lts__t_requests_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex_op_read.sum \
  -o gpurun_out/full/${cfg}_${tag} -f python tools/ktime.py --config $cfg --reps 1 > gpurun_out/full/${cfg}_${tag}.log 2>&1
ncu -i gpurun_out/full/${cfg}_${tag}.ncu-rep --page details --csv > gpurun_out/full/${cfg}_${tag}_details.csv 2>/dev/null
ncu -i gpurun_out/full/${cfg}_${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/full/${cfg}_${tag}_source.csv 2>/dev/null
