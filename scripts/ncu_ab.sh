# Request / byte counters of the sampler kernels under two env settings (A/B), one ncu pass each
# usage: bash scripts/ncu_ab.sh <config> <tag> [ENV=VAL ...]   (run twice with different env)
cfg=${1:-C5}; tag=${2:-a}; shift 2
mkdir -p gpurun_out/ab
env "$@" ncu --clock-control none -k regex:"window_kernel|copy_kernel" -s 8 -c 2 \
  --metrics gpu__time_duration.sum,lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_read_lookup_miss.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --csv python tools/ktime.py --config $cfg --reps 1 > gpurun_out/ab/ncu_${cfg}_${tag}.csv 2> gpurun_out/ab/ncu_${cfg}_${tag}.err
