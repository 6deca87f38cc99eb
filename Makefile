# Builds the two native artefacts in-tree (the .so files travel to the GPU box with gpurun).
#   make lib      -> paper_2206_11357_b200/libgact.so   (product: CUDA sm_100a + C ABI)
#   make oracle   -> oracle/liboracle.so                 (test infrastructure only)
NVCC ?= /usr/local/cuda/bin/nvcc
CC ?= gcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# No fast-math, no FMA contraction, IEEE division/sqrt, no flush-to-zero: the codes must be
# bit-identical to the oracle.
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xptxas -v --fmad=false -ftz=false \
           -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-ffp-contract=off,-O2 \
           -Iinclude -shared -cudart static
ORACLE_CFLAGS := -O2 -std=gnu11 -fPIC -shared -ffp-contract=off -frounding-math \
                 -fno-fast-math -Wall -Wextra

PKG := paper_2206_11357_b200
LIB_SRCS := $(PKG)/csrc/gact_kernels.cu $(PKG)/csrc/gact_host.cu
LIB_HDRS := include/gact.h $(wildcard $(PKG)/csrc/*.cuh)

all: lib oracle

lib: $(PKG)/libgact.so
oracle: oracle/liboracle.so

$(PKG)/libgact.so: $(LIB_SRCS) $(LIB_HDRS)
	$(NVCC) $(NVFLAGS) -o $@ $(LIB_SRCS) 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; exit 1)

oracle/liboracle.so: oracle/gact_oracle.c oracle/gact_oracle.h
	$(CC) $(ORACLE_CFLAGS) -o $@ oracle/gact_oracle.c -lm

clean:
	rm -f $(PKG)/libgact.so oracle/liboracle.so $(PKG)/ptxas.log

.PHONY: all lib oracle clean
