# bench.py on every config (1 GPU), JSON lines into gpurun_out/$tag/bench/bench_<cfg>.json
tag=${TAG:-r02}
out=gpurun_out/$tag/bench; mkdir -p $out
for c in ${CONFIGS:-C5 C4 C3 C2 C1 C6}; do
  timeout 1200 python bench.py --config $c "$@" > $out/bench_$c.json 2> $out/bench_$c.err
  echo "$c rc=$?"; tail -c 300 $out/bench_$c.json; echo
done
timeout 900 python bench.py --config C3 --separate-gather "$@" > $out/bench_C3_separate.json 2> $out/bench_C3_separate.err
echo "C3 separate rc=$?"
