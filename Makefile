# Builds libspecmesh_b200.so (sm_100a) in-tree and the oracle's C++ helpers.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 $(ARCH) -O3 -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $(EXTRA)
SRC_DIR := paper_1810_02719_b200/csrc
OBJ_DIR := build/obj
LIB := paper_1810_02719_b200/lib/libspecmesh_b200.so
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS := $(wildcard $(SRC_DIR)/*.h) $(wildcard $(SRC_DIR)/*.cuh) include/specmesh_gpu.h

all: $(LIB) oracle build/abi_chain

# compiled C++ caller of the C ABI through include/specmesh_gpu.hpp (tests/test_cpp_abi.py)
build/abi_chain: tests/cpp/abi_chain.cpp include/specmesh_gpu.hpp include/specmesh_gpu.h $(LIB)
	@mkdir -p build
	g++ -std=c++17 -O2 -Wall -Wextra -Iinclude $< -Lpaper_1810_02719_b200/lib -lspecmesh_b200 \
		-Wl,-rpath,'$$ORIGIN/../paper_1810_02719_b200/lib' -o $@

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.log || (cat $@.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static -lcuda -ldl

REF_INC ?= /root/reference/proj/include
ifneq ($(wildcard $(REF_INC)/specmesh/pipeline.hpp),)
REFHARNESS := oracle/_ref/libspecmesh_ref.so
endif
oracle: oracle/_ref/rng_ref $(REFHARNESS)

# The reference's own headers compiled where they lie (never copied) over
# oracle/eigen_shim, the stand-in for its absent Eigen dependency -- only in a
# container that has /root/reference; the GPU box uses the committed fixtures.
refharness: oracle/_ref/libspecmesh_ref.so
oracle/_ref/libspecmesh_ref.so: oracle/ref_harness.cpp oracle/eigen_shim/Eigen/mini_eigen.hpp
	@mkdir -p oracle/_ref
	g++ -std=c++20 -O3 -mavx2 -mfma -ffp-contract=off -fPIC -shared -Ioracle/eigen_shim -I$(REF_INC) $< -o $@

oracle/_ref/rng_ref: oracle/rng_ref.cpp
	@mkdir -p oracle/_ref
	g++ -O2 -std=c++17 -o $@ $<

# standalone kernel timing tools (not part of the library)
tools: build/dmma_lat build/cholx_bench build/solve_bench build/solve_bench_norhs build/solve_bench_noslab build/solve_bench_halfslab build/solve_bench_notri build/solve_bench_nomma build/solve_bench_nomma_norhs build/solve_bench_nomma_noslab build/solve_bench_f3r4 build/solve_bench_nomma_ns5

build/solve_bench: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -o $@ $<

build/solve_bench_norhs: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_NO_RHS -o $@ $<

build/solve_bench_noslab: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_SLAB_DIV=1000 -o $@ $<

build/solve_bench_notri: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_NO_TRI -o $@ $<

build/solve_bench_halfslab: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_SLAB_DIV=2 -o $@ $<

build/solve_bench_f3r4: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_NSF_FORCE=3 -DSMG_SOLVE_NS_FORCE=4 -o $@ $<

build/solve_bench_nomma_ns5: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_NSF_FORCE=3 -DSMG_SOLVE_NS_FORCE=4 -DSMG_SOLVE_NO_MMA -o $@ $<

build/solve_bench_nomma_norhs: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_NO_MMA -DSMG_SOLVE_NO_RHS -o $@ $<

build/solve_bench_nomma_noslab: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_NO_MMA -DSMG_SOLVE_NO_SLAB -o $@ $<

build/solve_bench_nomma: tools/solve_bench.cu $(SRC_DIR)/solve.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_SOLVE_NO_MMA -o $@ $<

build/chol_bench: tools/chol_bench.cu $(SRC_DIR)/cholqr.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_CHOL_TIMING -o $@ $<

clean:
	rm -rf build $(LIB) oracle/_ref

.PHONY: all clean oracle tools

build/cholx_bench: tools/cholx_bench.cu $(SRC_DIR)/cholx.cu $(HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -DSMG_CHOLX_TIMING -o $@ $<

build/dmma_lat: tools/dmma_lat.cu
	@mkdir -p build
	$(NVCC) -std=c++17 $(ARCH) -O3 -o $@ $<
