# Build for B200 (sm_100a) only. Product: paper_1109_3524_b200/libibmgpu.so (C-ABI, include/ibmgpu.h).
# Test infrastructure (CPU checkers): oracle/liboracle.so, oracle/_ref/libibmref.so (see oracle/Makefile).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_1109_3524_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HOST := $(wildcard $(PKG)/csrc/host/*.cpp)
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/host/*.hpp) include/ibmgpu.h
OBJDIR := build/obj
# make CHECKED=1: device-side bounds checks (IBM_DCHECK traps) — the stand-in for compute-sanitizer,
# which is closed on the GPU pool; run the GPU tests against this build (tools/checked_run.sh)
ifeq ($(CHECKED),1)
CHECKFLAGS := -DIBMGPU_CHECKED=1
OBJDIR := build/obj_checked
endif
# A/B variants: make EXTRA=-D... OBJDIR=build/obj_ab (tools/ab_iter.py with IBMGPU_LIB)
ifneq ($(EXTRA),)
OBJDIR := build/obj_ab
endif
OBJ := $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(SRC)) $(patsubst $(PKG)/csrc/host/%.cpp,$(OBJDIR)/host_%.o,$(HOST))
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-fopenmp -Xptxas -v --expt-relaxed-constexpr $(CHECKFLAGS) $(EXTRA)
HOSTFLAGS := -O3 -std=c++20 -fPIC -fopenmp -ffp-contract=off

all: $(PKG)/libibmgpu.so oracle

# the stepper's explicit-term kernels must round like the reference (no FMA contraction)
$(OBJDIR)/stepper.o: NVEXTRA := --fmad=false
$(OBJDIR)/assemble.o: NVEXTRA := --fmad=false

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) $(NVEXTRA) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(OBJDIR)/host_%.o: $(PKG)/csrc/host/%.cpp $(HDR)
	@mkdir -p $(OBJDIR)
	g++ $(HOSTFLAGS) -I/usr/local/cuda/include -c $< -o $@

$(PKG)/libibmgpu.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -Xcompiler -fopenmp -lcudart_static -lrt -ldl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/libibmgpu.so

.PHONY: all oracle clean
