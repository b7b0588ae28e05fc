mkdir -p gpurun_out/r02sm
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02sm/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02sm/tests.log
for env in "" "TGL_NO_SMALL_KERNEL=1"; do
  for c in C5 C1; do
    env $env timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02sm/b_$c.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/r02sm/b_$c.json').read().strip().splitlines()[-1])
print('$c', '$env', d['per_batch']['latency_us_per_batch'], d['value']/1e9, d['parity']['bit_exact'])"
  done
done
