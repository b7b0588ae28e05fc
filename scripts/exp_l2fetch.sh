# L2 fetch granularity experiment + quick parity; one gpurun call
mkdir -p gpurun_out/l2f
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for g in none 32 64 128; do
  if [ $g = none ]; then unset TGL_L2_FETCH; else export TGL_L2_FETCH=$g; fi
  timeout 600 python bench.py --no-e2e --no-per-batch --no-cpu-baseline --steps 30 2>/dev/null > gpurun_out/l2f/bench_$g.json
  python -c "import json; d=json.load(open('gpurun_out/l2f/bench_$g.json')); print('L2F $g', round(d['value']/1e9,2), 'G/s', round(d['ms_per_step']*1000,1), 'us')"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum \
      -k regex:'window_kernel|copy_kernel' -s 6 -c 2 --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-per-batch --no-cpu-baseline 2>/dev/null \
      | grep -E "window_kernel|copy_kernel" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-200 > gpurun_out/l2f/ncu_$g.txt
  cat gpurun_out/l2f/ncu_$g.txt
done
