# L2 fetch granularity (cudaLimitMaxL2FetchGranularity) A/B with per-kernel times and DRAM bytes
mkdir -p gpurun_out/l2f2
for g in none 32 64 128; do
  if [ $g = none ]; then unset TGL_L2_FETCH; else export TGL_L2_FETCH=$g; fi
  timeout 300 python tools/ktime.py --settings "[{}]" 2>/dev/null | grep env | sed "s/^/L2F=$g /"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum \
      -k regex:'window_kernel|copy_kernel' -s 4 -c 2 --csv python tools/ktime.py --reps 1 --settings "[{}]" 2>/dev/null \
      | grep -E "window_kernel|copy_kernel" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-200 | sed "s/^/L2F=$g /"
done
