# round 2: default bench (C5) + node-sharded bench lines (C5, C2) at N = 1 through the C ABI
mkdir -p gpurun_out/r02f
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f/bench.json 2> gpurun_out/r02f/bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r02f/bench.json
timeout 900 python bench.py --sharding node --steps 10 --warmup 3 > gpurun_out/r02f/node_C5.json 2> gpurun_out/r02f/node_C5.err; echo "node C5 rc=$?"
tail -c 1500 gpurun_out/r02f/node_C5.json; tail -5 gpurun_out/r02f/node_C5.err
timeout 900 python bench.py --sharding node --config C2 --steps 10 --warmup 3 > gpurun_out/r02f/node_C2.json 2> gpurun_out/r02f/node_C2.err; echo "node C2 rc=$?"
tail -c 600 gpurun_out/r02f/node_C2.json; tail -5 gpurun_out/r02f/node_C2.err
