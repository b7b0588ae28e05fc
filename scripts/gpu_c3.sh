mkdir -p gpurun_out/r02c3
python -m pytest tests/test_gpu_state.py -x -q -k fused > gpurun_out/r02c3/test.log 2>&1; tail -2 gpurun_out/r02c3/test.log
timeout 900 python bench.py --config C3 --steps 30 --warmup 5 --no-e2e > gpurun_out/r02c3/bench_C3.json 2> gpurun_out/r02c3/bench_C3.err; echo "C3 rc=$?"
timeout 900 python bench.py --config C3 --steps 30 --warmup 5 --no-e2e --fused-gather > gpurun_out/r02c3/bench_C3_fused.json 2> gpurun_out/r02c3/bench_C3_fused.err; echo "C3 fused rc=$?"
for f in bench_C3 bench_C3_fused; do python -c "
import json;d=json.loads(open('gpurun_out/r02c3/$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], json.dumps(d.get('gather_roofline')), json.dumps(d.get('state_write')), d['parity']['bit_exact'])"; done
