# compute-sanitizer over tools/sanitize_run.py (every libtgl kernel family, small inputs), libtgl
# kernels only (namespace tgl::); one log per tool under gpurun_out/$tag/sanitizer/
tag=${1:-r02}
out=gpurun_out/$tag/sanitizer; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --kernel-name kns=3tgl --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_run.py > $out/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $out/summary.txt
  tail -3 $out/$tool.log
done
