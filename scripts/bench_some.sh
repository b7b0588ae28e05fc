# bench.py on the given configs (1 GPU): bash scripts/bench_some.sh C3 C2 [-- extra args]
cfgs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do cfgs+=("$1"); shift; done; [ "$1" == "--" ] && shift
for c in "${cfgs[@]}"; do
  timeout 900 python bench.py --config $c "$@" > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -c 400 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
