# bench.py on every config (1 GPU), JSON lines into gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
for c in ${CONFIGS:-C5 C4 C3 C2 C1 C6}; do
  timeout 900 python bench.py --config $c "$@" > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -c 300 gpurun_out/bench_$c.json
done
