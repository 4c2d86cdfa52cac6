# Builds the product library (sm_100a) and the CPU-side test infrastructure.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr $(EXTRA)
SRC_DIR := paper_2208_14935_b200/csrc
LIB := paper_2208_14935_b200/lib/libhyt.so
SRCS := $(SRC_DIR)/plan.cu $(SRC_DIR)/kernels.cu $(SRC_DIR)/load.cu $(SRC_DIR)/engine.cu $(SRC_DIR)/api.cu $(SRC_DIR)/dist.cu $(SRC_DIR)/pull.cu $(SRC_DIR)/scan.cu
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
HDRS := $(SRC_DIR)/scan.h $(SRC_DIR)/hyt_internal.h $(SRC_DIR)/block_prims.cuh $(SRC_DIR)/graph.h include/hyt.h

all: $(LIB) hytgen/libhytgen.so oracle/liboracle.so

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p paper_2208_14935_b200/lib
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -ldl -lpthread

hytgen/libhytgen.so: hytgen/hytgen.c
	gcc -O3 -march=x86-64-v2 -fPIC -shared -pthread -o $@ $<

oracle/liboracle.so: oracle/oracle.c
	gcc -O3 -march=x86-64-v3 -ffp-contract=off -fPIC -shared -pthread -o $@ $< -lm

tools: tools/pin_bench tools/zc_bench tools/scatter_bench tools/red_ceiling tools/dsmem_bench

tools/pin_bench: tools/pin_bench.cu
	$(NVCC) $(ARCH) -O2 -o $@ $< -lpthread

tools/zc_bench: tools/zc_bench.cu
	$(NVCC) $(ARCH) -O3 -std=c++17 -o $@ $<

tools/scatter_bench: tools/scatter_bench.cu
	$(NVCC) $(ARCH) -O3 -std=c++17 -o $@ $<

tools/red_ceiling: tools/red_ceiling.cu
	$(NVCC) $(ARCH) -O3 -std=c++17 -o $@ $<

tools/dsmem_bench: tools/dsmem_bench.cu
	$(NVCC) $(ARCH) -O3 -std=c++17 -o $@ $<

clean:
	rm -rf build $(LIB) hytgen/libhytgen.so oracle/liboracle.so tools/pin_bench tools/zc_bench tools/scatter_bench tools/red_ceiling tools/dsmem_bench

.PHONY: all clean tools
