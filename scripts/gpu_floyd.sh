mkdir -p gpurun_out/r02f4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/r02f4/tests.log 2>&1; tail -2 gpurun_out/r02f4/tests.log
bash scripts/ab.sh gpurun_out/r02f4/c4 --config C4 --roots 1024000 --reps 5 -- product tools/variants/libtgl_minb5.so tools/variants/libtgl_head.so
bash scripts/ab.sh gpurun_out/r02f4/c2 --config C2 --roots 1024000 --reps 5 -- product tools/variants/libtgl_minb5.so tools/variants/libtgl_head.so
