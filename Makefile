# Build both native libraries in-tree (they travel to the GPU box with the gpurun snapshot).
#   make oracle   -> oracle/liboracle.so               (plain C, test infrastructure)
#   make lib      -> paper_2603_08929_b200/libbsort.so (sm_100a CUDA + C ABI, the product)
NVCC      ?= /usr/local/cuda/bin/nvcc
CC        ?= gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Iinclude \
             --expt-relaxed-constexpr -Xptxas -warn-spills
PKG       := paper_2603_08929_b200
CSRC      := $(wildcard $(PKG)/csrc/*.cu)
CHDR      := $(wildcard $(PKG)/csrc/*.cuh) include/bsort.h
OBJS      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))

all: oracle lib

oracle: oracle/liboracle.so
oracle/liboracle.so: oracle/bsort_oracle.c oracle/bsort_oracle.h
	$(CC) -O2 -std=c11 -Wall -Wextra -fPIC -shared -o $@ oracle/bsort_oracle.c

lib: $(PKG)/libbsort.so
build/%.o: $(PKG)/csrc/%.cu $(CHDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<
$(PKG)/libbsort.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

clean:
	rm -rf build oracle/liboracle.so $(PKG)/libbsort.so

.PHONY: all oracle lib clean
