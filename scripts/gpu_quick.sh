# quick GPU check: parity tests, then the default bench line without the slow legs
mkdir -p gpurun_out/quick
python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 600 python bench.py --no-e2e --no-per-batch --no-cpu-baseline "$@" 2>gpurun_out/quick/bench.err | tee gpurun_out/quick/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('VALUE', d['value']/1e9, 'G/s ms', d['ms_per_step'], 'frac', d['roofline']['frac'])"
tail -3 gpurun_out/quick/bench.err
