# Top-level build: the sm_100a product library and the oracle (test infra).
#   make            -> paper_2603_19371_b200/libwarplm_b200.so + oracle/*.so
# nvcc cross-compiles for sm_100a without a GPU.
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xptxas -warn-spills
PKG     := paper_2603_19371_b200
CSRC    := $(PKG)/csrc
SRCS    := $(CSRC)/kernels.cu $(CSRC)/hot_kernels.cu $(CSRC)/engine.cu $(CSRC)/ops.cu $(CSRC)/synth.cu $(CSRC)/slab.cu $(CSRC)/io.cu $(CSRC)/field64.cu $(CSRC)/generic.cu
HDRS    := include/wlm.h $(CSRC)/common.cuh $(CSRC)/hot.cuh $(CSRC)/kernels.cuh $(CSRC)/internal.cuh
OBJS    := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
LIB     := $(PKG)/libwarplm_b200.so

SHIM    := tests/nccl_shim/libnccl_shim.so

all: $(LIB) oracle $(SHIM)

# test infrastructure: two-rank NCCL stand-in over CUDA IPC (tests/test_slab_ranks.py)
$(SHIM): tests/nccl_shim/nccl_shim.cu
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC -shared -o $@ $< -lrt

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(ARCH) $(NVFLAGS) -Iinclude -c $< -o $@

# the sources' hash is linked in (wlm_source_hash), so a library left stale
# by edited sources is refused at load time (_lib.load)
SRC_HASH = $(shell cat $(sort $(SRCS) $(HDRS)) | sha256sum | cut -c1-16)

$(LIB): $(OBJS)
	@mkdir -p build
	printf 'const char* wlm_source_hash(void) { return "%s"; }\n' $(SRC_HASH) > build/src_hash.c
	gcc -O2 -fPIC -c build/src_hash.c -o build/src_hash.o
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) build/src_hash.o

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB) $(SHIM)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
