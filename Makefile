# Top-level build: the product library (sm_100a) and the test-only oracle.
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG     := paper_2604_19769_b200
CSRC    := $(PKG)/csrc
LIBDIR  := $(PKG)/lib
OBJDIR  := build/obj
CU_SRC  := $(wildcard $(CSRC)/*.cu)
CU_OBJ  := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRC))
HDRS    := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/ttkv_gpu.h

all: lib oracle

lib: $(LIBDIR)/libttkv_gpu.so

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(LIBDIR)/libttkv_gpu.so: $(CU_OBJ)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(CU_OBJ)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean
