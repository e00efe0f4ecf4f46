# Build every native artefact in-tree (the .so files travel to the GPU box with gpurun).
#   make            all libraries
#   make clean
NVCC    ?= nvcc
CUDA_HOME ?= /usr/local/cuda
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
CC      ?= gcc
CXX     ?= g++

PKG     := paper_2602_22103_b200
CSRC    := $(PKG)/csrc
PASTA_CU  := $(wildcard $(CSRC)/*.cu)
PASTA_CPP := $(wildcard $(CSRC)/*.cpp)
PASTA_H   := include/pasta.h $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h)

LIBS := tracegen/libtracegen_host.so oracle/liboracle.so
ifneq ($(PASTA_CU),)
LIBS += $(PKG)/libpasta.so tracegen/libtracegen_dev.so
endif

all: $(LIBS) examples/hand_worked

# the C ABI from plain C (no Python): the hand-worked trace, checked on the GPU
examples/hand_worked: examples/hand_worked.c include/pasta.h $(PKG)/libpasta.so
	$(CC) -O2 -std=c11 -Iinclude -I$(CUDA_HOME)/include -o $@ $< -L$(PKG) -lpasta \
	  -L$(CUDA_HOME)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,$(CUDA_HOME)/lib64

tracegen/libtracegen_host.so: tracegen/gen_host.c
	$(CC) -O2 -std=c11 -fPIC -shared -o $@ $<

tracegen/libtracegen_dev.so: tracegen/gen_dev.cu
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -shared -o $@ $<

oracle/liboracle.so: oracle/oracle.cpp
	$(CXX) -O2 -std=c++17 -fPIC -shared -o $@ $<

$(PKG)/libpasta.so: $(PASTA_CU) $(PASTA_CPP) $(PASTA_H)
	$(NVCC) $(NVFLAGS) -Iinclude -I$(CSRC) -shared -o $@ $(PASTA_CU) $(PASTA_CPP) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

# A/B variants of the scan (same ABI): make variants VARIANTS="name:-DFLAG=1 ..."
variants: $(PASTA_CU) $(PASTA_CPP) $(PASTA_H)
	mkdir -p build/variants
	@for v in $(VARIANTS); do n=$${v%%:*}; f=$$(echo $${v#*:} | tr ',' ' '); \
	  echo "variant $$n: $$f"; \
	  $(NVCC) $(NVFLAGS) $$f -Iinclude -I$(CSRC) -shared -o build/variants/libpasta_$$n.so $(PASTA_CU) $(PASTA_CPP) 2>/dev/null || exit 1; done

clean:
	rm -f $(LIBS) examples/hand_worked build_ptxas.log

.PHONY: all clean
