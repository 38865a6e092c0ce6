# Build of the B200 normal-bake product libraries (and the oracle checkers).
#
#   paper_2605_26137_b200/libmfbake.so      CUDA kernels + C ABI (include/mfbake.h)
#   paper_2605_26137_b200/libmeshforge_b200.so
#                                           the reference-compatible C++ API
#                                           (include/meshforge/...) over the C ABI
#   build/libmfpeaks.so                     L2-read / FP64 microbenchmarks (tools/peaks.cu)
#   build/test_bake_b200                    C++ KAT tests (tests/cpp) through the
#                                           C++ API (run on a GPU by tests/test_cpp_api.py)
#   oracle/...                              see oracle/Makefile
#
# Every CUDA TU is compiled for sm_100a only, with --fmad=false so fp64
# expressions keep the reference's operation order.
NVCC ?= nvcc
CXX ?= g++
PKG := paper_2605_26137_b200
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude -Iinclude/eigen_shim \
           -Xptxas -warn-spills --expt-relaxed-constexpr
CXXFLAGS := -std=c++20 -O2 -g -ffp-contract=off -fPIC -Iinclude -Iinclude/eigen_shim -Wall -Wextra
CU_SRCS := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJS := $(patsubst $(PKG)/csrc/%.cu,build/cu/%.o,$(CU_SRCS))
CU_HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/mfbake.h
MF_HDRS := $(shell find include/meshforge -name '*.h' 2>/dev/null) include/eigen_shim/Eigen/Core

.PHONY: all lib cpp peaks oracle clean
all: lib cpp peaks oracle

lib: $(PKG)/libmfbake.so
cpp: $(PKG)/libmeshforge_b200.so build/test_bake_b200 build/test_io_cpu build/bench_api build/sort_check
peaks: build/libmfpeaks.so

build/cu/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p build/cu
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/libmfbake.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -soname=libmfbake.so

$(PKG)/libmeshforge_b200.so: $(PKG)/cpp/meshforge_b200.cpp $(PKG)/cpp/io_b200.cpp $(PKG)/cpp/metrics_b200.cpp $(MF_HDRS) include/mfbake.h \
                             $(PKG)/libmfbake.so
	$(CXX) $(CXXFLAGS) -pthread -shared -o $@ $(PKG)/cpp/meshforge_b200.cpp $(PKG)/cpp/io_b200.cpp $(PKG)/cpp/metrics_b200.cpp -L$(PKG) -lmfbake \
	  -lz -Wl,-rpath,'$$ORIGIN'

build/test_bake_b200: tests/cpp/test_bake_b200.cpp tests/cpp/doctest.h $(PKG)/libmeshforge_b200.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -pthread -Itests/cpp -o $@ $< -L$(PKG) -lmeshforge_b200 -lmfbake -Wl,-rpath,'$$ORIGIN/../$(PKG)'

build/test_io_cpu: tests/cpp/test_io_cpu.cpp tests/cpp/doctest.h $(PKG)/libmeshforge_b200.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -pthread -Itests/cpp -o $@ $< -L$(PKG) -lmeshforge_b200 -lmfbake -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# end-to-end timing of the reference-facing C++ API (bench.py e2e_api)
build/bench_api: tools/bench_api.cpp $(PKG)/libmeshforge_b200.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(PKG) -lmeshforge_b200 -lmfbake -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# the LBVH radix sort against std::stable_sort (+ its timing); run by tests/test_gpu_sort.py
build/sort_check: tools/sort_check.cu $(PKG)/libmfbake.so $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(ARCH) -O2 -std=c++17 -Iinclude -Iinclude/eigen_shim $< -L$(PKG) -lmfbake -Xlinker -rpath,'$$ORIGIN/../$(PKG)' -o $@

# L2 / FP64 microbenchmarks (tools/peaks.cu) used by bench.py for the roofline peaks
build/libmfpeaks.so: tools/peaks.cu
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -o $@ $<

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/libmfbake.so $(PKG)/libmeshforge_b200.so
	$(MAKE) -C oracle clean
