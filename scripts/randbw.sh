# Random-access HBM calibration (tools/randbw.cu): useful GB/s per access width, mode and span.
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/randbw tools/randbw.cu
./tools/randbw 32 | tee gpurun_out/randbw.json
