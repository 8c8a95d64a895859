# Top-level build. `make` builds the product library and the oracle checker;
# `make ref` additionally compiles the unmodified reference (needs
# /root/reference, i.e. only in the build container).
#
#   paper_1108_1785_b200/lib/libgnetmon.so   product: sm_100a kernels + C-ABI
#   workloads/lib/libgnm_synth.so            synthetic flow generator (bench/tests)
#   oracle/lib/liborc.so                     C restatement (test infrastructure)
#   oracle/_ref/libflowmon_ref.so            unmodified reference (test infrastructure)

NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           -Xptxas -v -cudart static -Iinclude -ldl
PKG := paper_1108_1785_b200
SRCS := $(PKG)/csrc/capi.cu $(PKG)/csrc/kernels.cu $(PKG)/csrc/netflow.cu $(PKG)/csrc/hosts.cu $(PKG)/csrc/registry.cpp \
        $(PKG)/csrc/comm.cpp
HDRS := include/gnetmon.h $(PKG)/csrc/kernels.cuh $(PKG)/csrc/netflow.cuh $(PKG)/csrc/hosts.cuh $(PKG)/csrc/registry.hpp \
        $(PKG)/csrc/comm.hpp $(PKG)/csrc/rate.cuh

.PHONY: all ref clean oracle ablation
all: $(PKG)/lib/libgnetmon.so workloads/lib/libgnm_synth.so oracle

$(PKG)/lib/libgnetmon.so: $(SRCS) $(HDRS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(PKG)/lib/ptxas.log || (cat $(PKG)/lib/ptxas.log; false)

workloads/lib/libgnm_synth.so: workloads/synth.c
	@mkdir -p workloads/lib
	gcc -std=c11 -O2 -fPIC -shared -fopenmp -Wall -Wextra -o $@ $< -lm

# Measurement build with the K2 ablation switches (tools/ablation.sh); never
# loaded by the product or the tests.
ablation: $(PKG)/lib/ablation/libgnetmon.so
$(PKG)/lib/ablation/libgnetmon.so: $(SRCS) $(HDRS)
	@mkdir -p $(PKG)/lib/ablation
	$(NVCC) $(NVFLAGS) -DGNM_K2_ABLATION $(ABLATION_FLAGS) -shared -o $@ $(SRCS) 2> /dev/null

oracle:
	$(MAKE) -C oracle all

ref:
	$(MAKE) -C oracle ref
	$(MAKE) -C integration all

clean:
	rm -rf $(PKG)/lib workloads/lib
	$(MAKE) -C oracle clean
	$(MAKE) -C integration clean
