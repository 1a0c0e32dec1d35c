# Builds the B200 engine (sm_100a) and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_1106_4198_b200
LIB := $(PKG)/lib/libisnmf_b200.so
SRC := $(PKG)/csrc/engine.cu
DEPS := $(wildcard $(PKG)/csrc/*.cuh) include/isnmf_b200.h

all: $(LIB) oracle

$(LIB): $(SRC) $(DEPS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -lcudart 2> $(PKG)/lib/ptxas.log || (cat $(PKG)/lib/ptxas.log; exit 1)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf $(PKG)/lib oracle/_build
.PHONY: all oracle clean

# experimental build with per-phase cycle counters (K1 headline variant only)
prof: $(SRC) $(DEPS)
	@mkdir -p $(PKG)/lib_prof
	$(NVCC) $(NVFLAGS) -DISNMF_PHASE_PROF -DISNMF_MIN_VARIANTS -shared -o $(PKG)/lib_prof/libisnmf_b200.so $(SRC) -lcudart 2> $(PKG)/lib_prof/ptxas.log || (cat $(PKG)/lib_prof/ptxas.log; exit 1)
.PHONY: prof
