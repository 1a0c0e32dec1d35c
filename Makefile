# Builds the B200 engine (sm_100a) and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_1106_4198_b200
LIB := $(PKG)/lib/libisnmf_b200.so
SRC := $(PKG)/csrc/engine.cu
TABLES := $(PKG)/csrc/mma_table.cu $(PKG)/csrc/mma_multi_table.cu $(PKG)/csrc/ffma_table.cu $(PKG)/csrc/large_table.cu \
          $(PKG)/csrc/tc_table.cu
DEPS := $(wildcard $(PKG)/csrc/*.cuh) include/isnmf_b200.h $(PKG)/csrc/mma_table.cu
OBJ := $(PKG)/lib/engine.o $(PKG)/lib/mma_table.o $(PKG)/lib/mma_multi_table.o $(PKG)/lib/ffma_table.o \
       $(PKG)/lib/large_table.o $(PKG)/lib/tc_table.o

all: $(LIB) oracle

# six translation units (the engine and five kernel-instantiation tables), compiled in parallel
$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart
	@cat $(OBJ:.o=.ptxas.log) > $(PKG)/lib/ptxas.log

$(PKG)/lib/%.o: $(PKG)/csrc/%.cu $(DEPS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(PKG)/lib/$*.ptxas.log || (cat $(PKG)/lib/$*.ptxas.log; exit 1)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf $(PKG)/lib $(PKG)/lib_prof oracle/_build oracle/_ref
.PHONY: all oracle clean

# debug build: device-side index checks (ISNMF_DASSERT, kernels.cuh) that print and trap;
# select it with ISNMF_LIB=paper_1106_4198_b200/lib_debug/libisnmf_b200.so
DBG := $(PKG)/lib_debug
debug: $(DBG)/libisnmf_b200.so
$(DBG)/libisnmf_b200.so: $(OBJ:$(PKG)/lib/%.o=$(DBG)/%.o)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart
$(DBG)/%.o: $(PKG)/csrc/%.cu $(DEPS)
	@mkdir -p $(DBG)
	$(NVCC) $(NVFLAGS) -DISNMF_DEBUG -c -o $@ $< 2> $(DBG)/$*.ptxas.log || (cat $(DBG)/$*.ptxas.log; exit 1)
.PHONY: debug

# K1C progress-trace build (ISNMF_PC_TRACE: per-warp sites in mapped host memory,
# isnmf_debug_pc_trace; tools/pc_trace.py)
TRC := $(PKG)/lib_trace
trace: $(TRC)/libisnmf_b200.so
$(TRC)/libisnmf_b200.so: $(OBJ:$(PKG)/lib/%.o=$(TRC)/%.o)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart
$(TRC)/%.o: $(PKG)/csrc/%.cu $(DEPS)
	@mkdir -p $(TRC)
	$(NVCC) $(NVFLAGS) $(EXTRA) -DISNMF_PC_TRACE -c -o $@ $< 2> $(TRC)/$*.ptxas.log || (cat $(TRC)/$*.ptxas.log; exit 1)
.PHONY: trace

# experimental build with per-phase cycle counters (K1 headline variant only)
prof: $(SRC) $(TABLES) $(DEPS)
	@mkdir -p $(PKG)/lib_prof
	$(NVCC) $(NVFLAGS) $(EXTRA) -DISNMF_PHASE_PROF -DISNMF_MIN_VARIANTS -shared -o $(PKG)/lib_prof/libisnmf_b200.so $(SRC) $(TABLES) -lcudart 2> $(PKG)/lib_prof/ptxas.log || (cat $(PKG)/lib_prof/ptxas.log; exit 1)
.PHONY: prof
