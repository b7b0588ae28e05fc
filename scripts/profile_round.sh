# Round profile bundle (1 GPU): ncu launch list of the default bench command (our kernels only,
# -k filter), one full ncu capture of the sampler kernels of one timed step (-> DRAM traffic per
# root, tools/ncu_traffic.py), the default bench line using that traffic, randbw calibration.
tag=${1:-r01}
mkdir -p gpurun_out/$tag
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:'window_kernel|copy_kernel|radix|scan_|validate|aux_build|gather' \
    --csv --log-file gpurun_out/$tag/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-per-batch --no-cpu-baseline --parity-chunks 1 > gpurun_out/$tag/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'window_kernel|copy_kernel' -s 6 -c 2 \
    -o gpurun_out/$tag/prof -f python bench.py --steps 2 --warmup 3 --no-e2e --no-per-batch --no-cpu-baseline > gpurun_out/$tag/ncu_full.log 2>&1
python tools/ncu_traffic.py gpurun_out/$tag/prof.ncu-rep C5 8192000 gpurun_out/$tag/traffic.json
ncu -i gpurun_out/$tag/prof.ncu-rep --page details > gpurun_out/$tag/ncu_full_details.txt 2>&1
TGL_TRAFFIC_JSON=gpurun_out/$tag/traffic.json python bench.py > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
# (random-read calibration: profiles/r01/randbw.json)
tail -c 600 gpurun_out/$tag/bench.json
