mkdir -p gpurun_out/r02h
bash scripts/ab.sh gpurun_out/r02h --reps 5 -- product tools/variants/libtgl_fill128.so
bash scripts/ab.sh gpurun_out/r02h/c4 --config C4 --roots 1024000 --reps 5 -- product tools/variants/libtgl_fill128.so
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:'window_kernel|copy_kernel' -s 4 -c 2 --csv python tools/ktime.py --reps 1 > gpurun_out/r02h/ncu_fill64.csv 2>&1
TGL_LIB_PATH=$PWD/tools/variants/libtgl_fill128.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:'window_kernel|copy_kernel' -s 4 -c 2 --csv python tools/ktime.py --reps 1 > gpurun_out/r02h/ncu_fill128.csv 2>&1
grep -h "dram__bytes\|gpu__time" gpurun_out/r02h/ncu_fill*.csv | cut -c1-300
