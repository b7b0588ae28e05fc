# round-2 first GPU call: gpu tests (incl. the timed-configuration parity), smoke, default bench,
# window-kernel register-cap A/B (ktime, separate processes)
mkdir -p gpurun_out/r02a
python -m pytest tests -m gpu -x -q > gpurun_out/r02a/gpu_tests.log 2>&1; tail -5 gpurun_out/r02a/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1; tail -2 gpurun_out/r02a/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/r02a/bench.json
for v in "" tools/variants/libtgl_wminb6.so; do
  TGL_LIB_PATH=${v:+$PWD/$v} python tools/ktime.py --reps 5 2>&1 | tail -1 | sed "s|^|${v:-product} |" >> gpurun_out/r02a/ktime.txt
done
cat gpurun_out/r02a/ktime.txt
