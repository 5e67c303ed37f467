# Top-level build: the CUDA library (product) and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2511_13061_b200
CSRC := $(PKG)/csrc
SRCS := $(CSRC)/capi.cu $(CSRC)/spmv.cu $(CSRC)/compress.cu $(CSRC)/generate.cu $(CSRC)/convert.cu $(CSRC)/plan.cu
HDRS := $(wildcard $(CSRC)/*.cuh) include/macko_cuda.h
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))

all: lib dropin llm oracle

lib: $(PKG)/libmacko_cuda.so

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(PKG)/libmacko_cuda.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static

oracle:
	$(MAKE) -C oracle

# libmacko_llm.so: the per-token kernels of the Llama decode benchmark (the caller of the path)
llm: $(PKG)/libmacko_llm.so
$(PKG)/libmacko_llm.so: $(CSRC)/llm.cu $(CSRC)/llm_ops.cuh include/macko_llm.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CSRC)/llm.cu -cudart static 2> build/llm.ptxas.log || (cat build/llm.ptxas.log; exit 1)

clean:
	rm -rf build $(PKG)/libmacko_cuda.so
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean llm

# opt-in trace build (per-warp %globaltimer stamps; tools/trace_spmv.py), never the product .so
trace: $(PKG)/libmacko_cuda_trace.so
build/trace/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build/trace
	$(NVCC) $(NVFLAGS) -DMACKO_TRACE -c $< -o $@ 2> /dev/null
$(PKG)/libmacko_cuda_trace.so: $(patsubst $(CSRC)/%.cu,build/trace/%.o,$(SRCS))
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static
.PHONY: trace

# libmacko.so: the reference's C++ API (namespace macko: fp16 / bitpack / convert / the SPEC
# executors) backed by libmacko_cuda.so.  Compiled against the reference's own headers, which exist
# only in the build container (/root/reference); elsewhere the prebuilt .so is kept.
REF_SRC ?= /root/reference/proj/src
dropin: lib
	@if [ -d "$(REF_SRC)" ]; then \
	  g++ -std=c++20 -O2 -fPIC -shared -Wall -I include -I $(REF_SRC) -I /usr/local/cuda/include \
	    $(CSRC)/dropin/macko_dropin.cpp -o $(PKG)/libmacko.so -L $(PKG) -lmacko_cuda -Wl,-rpath,'$$ORIGIN'; \
	else echo "dropin: $(REF_SRC) absent, keeping prebuilt $(PKG)/libmacko.so"; fi

# C++ drop-in tests (reference headers + our headers); need /root/reference at build time.
#   dropin_test     — the reference's own types / encoder feeding libmacko_cuda.so via macko_cuda.hpp
#   dropin_ref_test — a reference caller linked against libmacko.so only (no reference code)
cpptest: lib dropin oracle
	@if [ -d "$(REF_SRC)" ]; then \
	  $(NVCC) $(ARCH) -std=c++20 -O2 -I include -I $(REF_SRC) tests/cpp/dropin_test.cpp -o tests/cpp/dropin_test \
	    -L $(PKG) -L oracle/_ref -lmacko_cuda -lmacko_ref \
	    -Xlinker -rpath,'$$ORIGIN/../../$(PKG)' -Xlinker -rpath,'$$ORIGIN/../../oracle/_ref' && \
	  g++ -std=c++20 -O2 -mf16c -Wall -I include -I $(REF_SRC) tests/cpp/dropin_ref_test.cpp -o tests/cpp/dropin_ref_test \
	    -L $(PKG) -lmacko -Wl,-rpath,'$$ORIGIN/../../$(PKG)'; \
	else echo "cpptest: $(REF_SRC) absent, keeping prebuilt tests/cpp/dropin_test*"; fi

.PHONY: cpptest dropin
