# final round check on one box: GPU tests, smoke, default bench (driver's command), reference arm
tag=${1:-r02}
out=gpurun_out/$tag/final; mkdir -p $out
timeout 1800 python -m pytest tests -m gpu -x -q > $out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $out/reference.json 2> $out/reference.err; echo "ref rc=$?"
python -c "
import json;d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], (d['roofline'].get('random_access') or {}).get('frac'), d['parity']['bit_exact'], d['e2e']['value'], d['clocks'])"
