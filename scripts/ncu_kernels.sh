# Warm-cache per-kernel metrics of one sampler setting (tools/sweep.py --only ...).
# usage: bash scripts/ncu_kernels.sh <tag> <setting>
tag=$1; shift
ncu --cache-control none --clock-control none -k regex:"window_kernel|copy_kernel" -s 9 -c 3 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_wavefronts_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warps_eligible.avg.per_cycle_active,launch__registers_per_thread,launch__occupancy_limit_registers \
    --csv python tools/sweep.py --reps 3 --only "$@" > gpurun_out/ncuk_${tag}.csv 2>&1
tail -3 gpurun_out/ncuk_${tag}.csv
