# Top-level build: the sm_100a C-ABI library (the product), the C++ drop-in
# library over it, and the CPU oracle (test infrastructure, oracle/Makefile).
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX       = g++
ARCH      = -gencode arch=compute_100a,code=sm_100a
NVFLAGS   = -O3 -std=c++17 $(ARCH) -lineinfo --fmad=false -Xcompiler -fPIC -Iinclude \
            -Xptxas -warn-spills
PKG       = paper_1512_08017_b200
LIB       = $(PKG)/lib/liblsqfit_cuda.so
DROPIN    = $(PKG)/lib/liblsqfit_b200.so
DROPIN_TEST = $(PKG)/lib/test_dropin_ext
CU        = $(wildcard $(PKG)/csrc/*.cu)
HDRS      = $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.hpp) include/lsqfit_cuda.h
OBJDIR    = build/obj
OBJS      = $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(CU))

PROBES    = tools/cudart_init_probe tools/init_breakdown tools/graph_bench

all: $(LIB) $(DROPIN) $(DROPIN_TEST) oracle $(PROBES)

# host-side probes the GPU tests run (CUDA driver init latency next to the
# reference acceptance harness)
tools/cudart_init_probe: tools/cudart_init_probe.cpp
	$(CXX) -O2 -I/usr/local/cuda/include -o $@ $< -L/usr/local/cuda/lib64 -lcudart
tools/graph_bench: tools/graph_bench.cpp $(LIB)
	$(CXX) -O2 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG)/lib -llsqfit_cuda \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib'
tools/init_breakdown: tools/init_breakdown.cpp $(LIB)
	$(CXX) -O2 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG)/lib -llsqfit_cuda \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib'

# one object per translation unit (each kernel family lives in one k_*.cu), so
# `make -j` compiles them in parallel
$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

$(DROPIN): $(LIB) $(wildcard $(PKG)/cpp/*.cpp) $(wildcard include/lsqfit/*.hpp) include/lsqfit_cuda.h
	$(CXX) -std=c++20 -O3 -fPIC -shared -Iinclude -I/usr/local/cuda/include -o $@ \
	    $(wildcard $(PKG)/cpp/*.cpp) -L$(PKG)/lib -llsqfit_cuda -Wl,-rpath,'$$ORIGIN'

oracle: $(DROPIN)
	$(MAKE) -C oracle

ptxas: $(CU) $(HDRS)
	for f in $(CU); do $(NVCC) $(NVFLAGS) -Xptxas -v -c -o /dev/null $$f 2>&1 | grep -E "Function properties|registers|spill"; done

clean:
	rm -f $(LIB) $(DROPIN) $(DROPIN_TEST) $(OBJS)
	$(MAKE) -C oracle clean

.PHONY: all oracle ptxas clean

# Drop-in extension checks (tests/cpp/test_dropin_ext.cpp), run by tests/test_gpu_dropin.py.
dropin_test: $(DROPIN_TEST)
$(DROPIN_TEST): tests/cpp/test_dropin_ext.cpp tests/cpp/doctest.h $(DROPIN)
	$(CXX) -std=c++20 -O2 -Itests/cpp -Iinclude -o $@ tests/cpp/test_dropin_ext.cpp \
	    -L$(PKG)/lib -llsqfit_b200 -llsqfit_cuda -Wl,-rpath,'$$ORIGIN'
