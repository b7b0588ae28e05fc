# compute-sanitizer over tools/sanitize_run.py (every libtgl kernel family, small inputs), libtgl
# kernels only (namespace tgl::); one log per tool under gpurun_out/$tag/sanitizer/
#   bash scripts/sanitize.sh TAG [tools...]      (default: memcheck racecheck synccheck initcheck)
tag=${1:-r02}; shift
tools=${@:-memcheck racecheck synccheck initcheck}
out=gpurun_out/$tag/sanitizer; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in $tools; do
  extra=""
  # racecheck instruments every shared-memory access: the sampler kernels only (the rest use smem
  # for textbook scans / radix histograms), and a smaller run
  [ $tool = racecheck ] && extra="--kernel-name regex=window_kernel|copy_kernel|unpermute_copy --racecheck-report all"
  [ $tool = memcheck ] || [ $tool = synccheck ] && extra="--kernel-name kns=3tgl"
  # initcheck: every kernel instrumented (torch's kernels initialise our inputs: a filtered run would
  # report those writes as missing); errors are then counted for libtgl kernels only (summary line)
  # racecheck: kernels serialised (CUDA_LAUNCH_BLOCKING, no programmatic dependent launch), so that
  # shared memory of concurrently resident kernels of other streams is not reported as a race
  rc_env=$([ $tool = racecheck ] && echo "SANITIZE_SMALL=1 CUDA_LAUNCH_BLOCKING=1 TGL_NO_PDL=1" || echo "SANITIZE_SMALL=0")
  env $rc_env timeout 2400 $CS --tool $tool $extra \
      --error-exitcode 9 --print-limit 2000 python tools/sanitize_run.py > $out/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $out/summary.txt
  grep "ERROR SUMMARY\|RACECHECK SUMMARY" $out/$tool.log | tail -1
  echo "  errors in libtgl kernels: $(grep -A1 'Uninitialized\|Invalid\|Race\|Barrier' $out/$tool.log | grep -c ' at tgl::\| at void tgl::')" | tee -a $out/summary.txt
done
