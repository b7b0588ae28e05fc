# bench.py on every config (1 GPU), JSON lines into gpurun_out/bench_<cfg>.json
for c in C5 C4 C3 C2 C1; do
  timeout 900 python bench.py --config $c "$@" > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -c 300 gpurun_out/bench_$c.json
done
