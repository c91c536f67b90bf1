# Build of the B200-native hybrid-batch forward.
#
#   libss_gpu.so   sm_100a kernels + the ss_gpu.h C ABI (static cudart; NCCL
#                  is dlopen'ed only for tp_size > 1)
#   libss_host.so  C++20 host engine (ss_host.h), links libss_gpu.so
#   oracle/        test-only checker (see oracle/Makefile)
PKG := paper_2403_02310_b200
NVCC ?= /usr/local/cuda/bin/nvcc
# The image exports CXX=/opt/gcc/bin/g++, a wrapper whose -shared links omit
# libstdc++; use the system compiler so every .so records its C++ runtime.
CXX := $(firstword $(wildcard /usr/bin/g++) g++)
ARCH := -gencode arch=compute_100a,code=sm_100a

HOST_SRCS := $(wildcard $(PKG)/csrc/host/*.cpp)
HOST_HDRS := $(wildcard $(PKG)/csrc/host/*.hpp) include/ss_host.h include/ss_gpu.h include/ss_status.h
GPU_SRCS := $(wildcard $(PKG)/csrc/gpu/*.cu)
GPU_HDRS := $(wildcard $(PKG)/csrc/gpu/*.cuh) include/ss_gpu.h include/ss_synth.h include/ss_status.h

NVFLAGS := $(ARCH) -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xptxas -v --expt-relaxed-constexpr -Iinclude -I$(PKG)/csrc/gpu
HOSTFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Wno-unused-parameter -Iinclude

all: $(PKG)/libss_gpu.so $(PKG)/libss_host.so oracle

$(PKG)/libss_gpu.so: $(GPU_SRCS) $(GPU_HDRS)
	$(NVCC) $(NVFLAGS) -shared -cudart static -o $@ $(GPU_SRCS) -ldl -lpthread -lrt 2> build_gpu.log || (cat build_gpu.log; false)

$(PKG)/libss_host.so: $(HOST_SRCS) $(HOST_HDRS) $(PKG)/libss_gpu.so
	$(CXX) $(HOSTFLAGS) -shared -o $@ $(HOST_SRCS) -L$(PKG) -lss_gpu -Wl,-rpath,'$$ORIGIN'

# (after both libraries: oracle/_ref/ref_engine_gpu links them)
oracle: $(PKG)/libss_gpu.so $(PKG)/libss_host.so
	$(MAKE) -C oracle

clean:
	rm -f $(PKG)/libss_gpu.so $(PKG)/libss_host.so build_gpu.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
