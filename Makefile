# Build for the B200 FFTMatvec (sm_100a). `make` builds:
#   paper_2508_10202_b200/libfftmv_cuda.so  -- the product (C ABI: include/fftmv_cuda.h)
#   build/fftmv_cpp_tests                   -- C++ drop-in header tests (include/fftmv/*.hpp)
#   build/fft_matvec                        -- command-line harness (SPEC.md cli module)
#   oracle/liboracle.so, oracle/_ref/libfftmv_ref.so -- test-only checkers (oracle/Makefile)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++20 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr -Xptxas -v
PKG := paper_2508_10202_b200
# nlohmann/json.hpp (sweep.hpp includes it unconditionally, as the reference's sweep.hpp:20 does)
JSON_INC := $(shell python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")/include/cudnn_frontend/thirdparty/nlohmann

all: lib oracle cpp cli stub

lib: $(PKG)/libfftmv_cuda.so

# one object per translation unit so `make -j` compiles them in parallel
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(wildcard $(PKG)/csrc/*.cu)) $(patsubst $(PKG)/csrc/%.cpp,build/obj/%.o,$(wildcard $(PKG)/csrc/*.cpp))
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/fftmv_cuda.h

$(PKG)/libfftmv_cuda.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -Xlinker --no-undefined -o $@ $(OBJS) -ldl -lcudart -lpthread
	@cat build/obj/*.ptxas.log > build_ptxas.log

build/obj/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; false)

build/obj/%.o: $(PKG)/csrc/%.cpp include/fftmv_cuda.h
	@mkdir -p build/obj
	g++ -std=c++20 -O2 -fPIC -Wall -c -o $@ $<

oracle:
	$(MAKE) -C oracle all

cpp: build/fftmv_cpp_tests

build/fftmv_cpp_tests: tests/cpp/test_dropin.cpp $(wildcard include/fftmv/*.hpp) include/fftmv_cuda.h $(PKG)/libfftmv_cuda.so
	@mkdir -p build
	g++ -std=c++20 -O2 -Wall -Iinclude -I/usr/local/cuda/include -I$(JSON_INC) -o $@ tests/cpp/test_dropin.cpp -L$(PKG) -lfftmv_cuda -Wl,-rpath,'$$ORIGIN/../$(PKG)' -L/usr/local/cuda/lib64 -lcudart

cli: build/fft_matvec build/fftmv_dropin_bench

build/fftmv_dropin_bench: $(PKG)/cli/dropin_bench.cpp $(wildcard include/fftmv/*.hpp) include/fftmv_cuda.h $(PKG)/libfftmv_cuda.so
	@mkdir -p build
	g++ -std=c++20 -O2 -Wall -Iinclude -I/usr/local/cuda/include -o $@ $(PKG)/cli/dropin_bench.cpp -L$(PKG) -lfftmv_cuda -Wl,-rpath,'$$ORIGIN/../$(PKG)' -L/usr/local/cuda/lib64 -lcudart

# test-only NCCL API over POSIX shared memory (FMV_NCCL_LIB): several ranks on one GPU
stub: build/libfmv_nccl_stub.so

build/libfmv_nccl_stub.so: tests/stub/fmv_nccl_stub.cpp
	@mkdir -p build
	g++ -std=c++20 -O2 -Wall -fPIC -shared -I/usr/local/cuda/include -o $@ $< -L/usr/local/cuda/lib64 -lcudart -lrt

build/fft_matvec: $(PKG)/cli/fft_matvec.cpp $(wildcard include/fftmv/*.hpp) include/fftmv_cuda.h $(PKG)/libfftmv_cuda.so
	@mkdir -p build
	g++ -std=c++20 -O2 -Wall -Iinclude -I/usr/local/cuda/include -I$(JSON_INC) -o $@ $(PKG)/cli/fft_matvec.cpp -L$(PKG) -lfftmv_cuda -Wl,-rpath,'$$ORIGIN/../$(PKG)' -L/usr/local/cuda/lib64 -lcudart

clean:
	rm -f $(PKG)/libfftmv_cuda.so build/fftmv_cpp_tests build/fft_matvec build/libfmv_nccl_stub.so
	$(MAKE) -C oracle clean

.PHONY: all lib oracle cpp cli stub clean
