# Build every native artefact in-tree (the .so files travel to the GPU box with gpurun).
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_2605_20497_b200
CSRC    := $(PKG)/csrc
CU_SRCS := $(wildcard $(CSRC)/*.cu)
CU_HDRS := $(wildcard $(CSRC)/*.cuh) include/hgp.h

.PHONY: all gen oracle cuda clean
all: gen oracle cuda

gen: hgpgen/libhgpgen.so
hgpgen/libhgpgen.so: hgpgen/hgpgen.c hgpgen/hgpgen.h
	gcc -O2 -fPIC -shared -std=c11 -Wall -Wextra -o $@ $< -lm

oracle: oracle/libhgp_ref.so
oracle/libhgp_ref.so: oracle/hgp_ref.cpp oracle/hgp_ref_refine.cpp oracle/hgp_ref.h
	g++ -O2 -fPIC -shared -std=c++17 -Wall -Wextra -o $@ oracle/hgp_ref.cpp oracle/hgp_ref_refine.cpp

cuda: $(PKG)/libhgp.so
CU_OBJS := $(patsubst $(CSRC)/%.cu,build/obj/%.o,$(CU_SRCS))
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -warn-spills -Iinclude
build/obj/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $<
$(PKG)/libhgp.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

clean:
	rm -rf build hgpgen/libhgpgen.so oracle/libhgp_ref.so $(PKG)/libhgp.so
