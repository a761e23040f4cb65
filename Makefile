# Builds the sm_100a C-ABI library (in-tree, travels to the GPU box) and the
# C oracle helpers.  `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC      ?= nvcc
PY        ?= python
PKG       := paper_2203_08069_b200
CSRC      := $(PKG)/csrc
NCCL_ROOT ?= $(shell $(PY) -c "import nvidia.nccl,os;print(os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl,'__file__',None) else list(nvidia.nccl.__path__)[0])")
ARCH      := -gencode arch=compute_100a,code=sm_100a
# TUNING=1 also builds the tile configurations kept only for td_dgemm_config sweeps
TUNING    ?= 0
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr \
             -I$(NCCL_ROOT)/include -Iinclude $(if $(filter 1,$(TUNING)),-DTD_TUNING)
LDFLAGS   := -shared -L$(NCCL_ROOT)/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $(NCCL_ROOT)/lib -cudart static
SRCS      := $(CSRC)/capi.cu $(CSRC)/gemm.cu $(CSRC)/mttkrp.cu $(CSRC)/stream.cu $(CSRC)/interp.cu $(CSRC)/comm.cu $(CSRC)/peer.cu $(CSRC)/plan.cu
OBJS      := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
LIB       := $(PKG)/libdistal_b200.so

# The reference (pure Python, nothing to compile) is staged into oracle/_ref as
# the checker and the reference arm's CPU implementation: oracle/_ref/tendist is
# its package, oracle/_ref/tests its own unit tests.  oracle/_ref is git-ignored
# (never committed) but travels to the GPU box with the snapshot.  Only done
# where the reference checkout exists (this container); the GPU box uses the
# staged copy.
REF_PKG   ?= /root/reference/pkg
REF_OUT   := oracle/_ref

all: $(LIB) ref examples

# a C host using only the C ABI (td_execute_plan); tests/test_abi_host.py runs it on a GPU
examples: examples/plan_demo

examples/plan_demo: examples/plan_demo.c include/distal_b200.h $(LIB)
	$(NVCC) -x cu $(ARCH) -O2 -Iinclude $< -o $@ -L$(PKG) -ldistal_b200 -Xlinker -rpath -Xlinker '$$ORIGIN/../$(PKG)'

ref:
	@if [ -d $(REF_PKG)/src/tendist ]; then \
	  rm -rf $(REF_OUT) && mkdir -p $(REF_OUT) && \
	  cp -r $(REF_PKG)/src/tendist $(REF_OUT)/tendist && cp -r $(REF_PKG)/tests $(REF_OUT)/tests && \
	  chmod -R u+w $(REF_OUT) && find $(REF_OUT) -name __pycache__ -prune -exec rm -rf {} + ; \
	  echo "staged the reference into $(REF_OUT)"; \
	else echo "no reference checkout at $(REF_PKG): keeping $(REF_OUT) as is"; fi

build/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) include/distal_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) $(LDFLAGS) $(OBJS) -o $@

clean:
	rm -rf build $(LIB) examples/plan_demo

.PHONY: all clean ref examples
