# Builds the sm_100a C-ABI library and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2305_00645_b200
SRCS := $(PKG)/csrc/gt_gadget_api.cu $(PKG)/csrc/gt_train.cu $(PKG)/csrc/gt_infer.cu $(PKG)/csrc/gt_party.cu
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/gtree_b200.h
OBJS := $(SRCS:.cu=.o)
LIB := $(PKG)/libgtree_b200.so

all: $(LIB) oracle

$(PKG)/csrc/%.o: $(PKG)/csrc/%.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(OBJS) $(LIB) $(PKG)/csrc/*.ptxas.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
