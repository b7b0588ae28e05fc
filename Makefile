# Builds libtgl.so (sm_100a CUDA, C ABI in include/tgl.h) and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2203_14883_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/tgl.h
NCCL_INC ?= $(shell python3 -c 'import nvidia.nccl, os; print(os.path.join(list(nvidia.nccl.__path__)[0], "include"))' 2>/dev/null || echo /usr/include)
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$(NCCL_INC) \
           -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -ftz=false -prec-div=true -prec-sqrt=true \
           -fmad=true -Xptxas -v -ldl

all: $(PKG)/libtgl.so oracle/liboracle.so

$(PKG)/libtgl.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -o $@.tmp $(SRCS) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)
	mv $@.tmp $@

oracle/liboracle.so: oracle/tgl_oracle.c
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fexcess-precision=standard -fPIC -shared -o $@ $< -lm

clean:
	rm -f $(PKG)/libtgl.so oracle/liboracle.so build_ptxas.log

.PHONY: all clean
