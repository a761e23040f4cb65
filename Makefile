# Builds the sm_100a C-ABI library (in-tree, travels to the GPU box) and the
# C oracle helpers.  `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC      ?= nvcc
PY        ?= python
PKG       := paper_2203_08069_b200
CSRC      := $(PKG)/csrc
NCCL_ROOT ?= $(shell $(PY) -c "import nvidia.nccl,os;print(os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl,'__file__',None) else list(nvidia.nccl.__path__)[0])")
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr \
             -I$(NCCL_ROOT)/include -Iinclude
LDFLAGS   := -shared -L$(NCCL_ROOT)/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $(NCCL_ROOT)/lib -cudart static
SRCS      := $(CSRC)/capi.cu $(CSRC)/gemm.cu $(CSRC)/mttkrp.cu $(CSRC)/stream.cu $(CSRC)/interp.cu $(CSRC)/comm.cu $(CSRC)/peer.cu
OBJS      := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
LIB       := $(PKG)/libdistal_b200.so

all: $(LIB)

build/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) include/distal_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) $(LDFLAGS) $(OBJS) -o $@

clean:
	rm -rf build $(LIB)

.PHONY: all clean
