# Round profile bundle (1 GPU): ncu launch list of the default bench command (our kernels only,
# -k filter), one full ncu capture of the sampler kernels of one timed step (-> DRAM traffic per
# root, tools/ncu_traffic.py), the default bench line using that traffic, randbw calibration.
tag=${1:-r01}
mkdir -p gpurun_out/$tag
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:'window_kernel|copy_kernel|radix|scan_|validate|aux_build|gather' \
    --csv --log-file gpurun_out/$tag/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-per-batch --no-cpu-baseline --parity-chunks 1 > gpurun_out/$tag/launches_bench.log 2>&1
ncu --set full --metrics lts__t_requests_srcunit_tex_op_read_lookup_miss.sum --clock-control none --import-source on -k regex:'window_kernel|copy_kernel' -s 6 -c 2 \
    -o gpurun_out/$tag/prof -f python bench.py --steps 2 --warmup 3 --no-e2e --no-per-batch --no-cpu-baseline > gpurun_out/$tag/ncu_full.log 2>&1
python tools/ncu_traffic.py gpurun_out/$tag/prof.ncu-rep C5 8192000 gpurun_out/$tag/traffic.json
ncu -i gpurun_out/$tag/prof.ncu-rep --page details > gpurun_out/$tag/ncu_full_details.txt 2>&1
# random-request calibration: L2-miss (DRAM) requests per second of scattered 4-byte reads
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/granule tools/granule.cu
ncu --metrics lts__t_requests_srcunit_tex_op_read_lookup_miss.sum,dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -c 2 --csv ./tools/granule > gpurun_out/$tag/granule_ncu.csv 2>&1
python tools/granule_peak.py gpurun_out/$tag/granule_ncu.csv gpurun_out/$tag/granule_peak.json
TGL_TRAFFIC_JSON=gpurun_out/$tag/traffic.json python bench.py > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
tail -c 600 gpurun_out/$tag/bench.json
