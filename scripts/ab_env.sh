# A/B of environment knobs on the default bench (C5): bash scripts/ab_env.sh "" "TGL_NO_SKIP=1" ...
mkdir -p gpurun_out/ab
for e in "$@"; do
  tag=$(echo "base $e" | tr -c 'A-Za-z0-9_\n' '_')
  env $e timeout 600 python bench.py --no-e2e --no-per-batch --no-cpu-baseline 2>gpurun_out/ab/$tag.err > gpurun_out/ab/$tag.json
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab/$tag.json').readline()); print('$e', 'VALUE', round(d['value']/1e9,2), 'G/s ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'parity', d.get('parity'))" || tail -3 gpurun_out/ab/$tag.err
done
