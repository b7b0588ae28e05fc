# GPU test suite against a debug build with device bounds checks (-DTGL_BOUNDS: TGL_CHECK traps on a
# computed index outside its array; compute-sanitizer is not available on the test pool).
#   bash scripts/bounds_tests.sh [pytest args]     (log: gpurun_out/bounds/tests.log)
set -e
mkdir -p tools/variants gpurun_out/bounds
NCCL_INC=$(python3 -c 'import nvidia.nccl, os; print(os.path.join(list(nvidia.nccl.__path__)[0], "include"))')
[ -f tools/variants/libtgl_bounds.so ] || /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
  -std=c++17 -I$NCCL_INC -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -ftz=false -prec-div=true \
  -prec-sqrt=true -fmad=true -ldl -DTGL_BOUNDS -o tools/variants/libtgl_bounds.so paper_2203_14883_b200/csrc/*.cu
set +e
TGL_LIB_PATH=$PWD/tools/variants/libtgl_bounds.so timeout 1500 python -m pytest tests -m gpu -x -q "$@" \
  > gpurun_out/bounds/tests.log 2>&1
echo "rc $?" >> gpurun_out/bounds/tests.log
TGL_LIB_PATH=$PWD/tools/variants/libtgl_bounds.so timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e \
  --no-per-batch --no-cpu-baseline > gpurun_out/bounds/bench_C5.json 2> gpurun_out/bounds/bench_C5.err
echo "bench rc $?" >> gpurun_out/bounds/tests.log
tail -3 gpurun_out/bounds/tests.log
