# Builds the two native artefacts in-tree (the .so files travel to the GPU box with gpurun).
#   make lib      -> paper_2206_11357_b200/libgact.so   (product: CUDA sm_100a + C ABI)
#   make oracle   -> oracle/liboracle.so                 (test infrastructure only)
NVCC ?= /usr/local/cuda/bin/nvcc
CC ?= gcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# No fast-math, no FMA contraction, IEEE division, no flush-to-zero: the codes must be
# bit-identical to the oracle.
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo --fmad=false -ftz=false -prec-div=true \
           -prec-sqrt=true -Xcompiler -fPIC,-ffp-contract=off -Iinclude
ORACLE_CFLAGS := -O2 -std=gnu11 -fPIC -shared -ffp-contract=off -frounding-math \
                 -fno-fast-math -Wall -Wextra

PKG := paper_2206_11357_b200
CSRC := $(PKG)/csrc
OBJDIR := build/obj
LIB_SRCS := $(wildcard $(CSRC)/*.cu)
LIB_OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(LIB_SRCS))
LIB_HDRS := include/gact.h include/gact_testing.h $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h)

all: lib oracle

lib: $(PKG)/libgact.so
oracle: oracle/liboracle.so

$(OBJDIR)/%.o: $(CSRC)/%.cu $(LIB_HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(PKG)/libgact.so: $(LIB_OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(LIB_OBJS)

oracle/liboracle.so: oracle/gact_oracle.c oracle/gact_oracle.h
	$(CC) $(ORACLE_CFLAGS) -o $@ oracle/gact_oracle.c -lm

clean:
	rm -rf build $(PKG)/libgact.so oracle/liboracle.so

.PHONY: all lib oracle clean
