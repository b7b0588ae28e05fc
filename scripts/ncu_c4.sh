# C4: counters of the four sampler launches of one call (window/copy x layer 0/1) + a full capture
mkdir -p gpurun_out/c4
ncu --clock-control none -k regex:"window_kernel|copy_kernel" -s 8 -c 4 \
  --metrics gpu__time_duration.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read_lookup_miss.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
  --csv python tools/ktime.py --config C4 --reps 1 --roots 1024000 > gpurun_out/c4/counters.csv 2> gpurun_out/c4/counters.err
ncu --set full --import-source on --clock-control none -k regex:"window_kernel|copy_kernel" -s 8 -c 4 \
  -o gpurun_out/c4/full -f python tools/ktime.py --config C4 --reps 1 --roots 1024000 > gpurun_out/c4/full.log 2>&1
ncu -i gpurun_out/c4/full.ncu-rep --page source --csv --print-source sass > gpurun_out/c4/source.csv 2>/dev/null
timeout 300 python tools/ktime.py --config C4 --roots 1024000 > gpurun_out/c4/ktime.txt 2>&1
