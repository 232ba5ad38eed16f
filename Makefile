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
CSRC      = $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cuh) include/lsqfit_cuda.h

all: $(LIB) $(DROPIN) $(DROPIN_TEST) oracle

$(LIB): $(CSRC)
	mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -shared -o $@ $(PKG)/csrc/capi.cu -lcudart

$(DROPIN): $(LIB) $(wildcard $(PKG)/cpp/*.cpp) $(wildcard include/lsqfit/*.hpp) include/lsqfit_cuda.h
	$(CXX) -std=c++20 -O3 -fPIC -shared -Iinclude -I/usr/local/cuda/include -o $@ \
	    $(wildcard $(PKG)/cpp/*.cpp) -L$(PKG)/lib -llsqfit_cuda -Wl,-rpath,'$$ORIGIN'

oracle: $(DROPIN)
	$(MAKE) -C oracle

ptxas: $(CSRC)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /dev/null $(PKG)/csrc/capi.cu 2>&1 | grep -E "Function properties|registers|spill" 

clean:
	rm -f $(LIB) $(DROPIN)
	$(MAKE) -C oracle clean

.PHONY: all oracle ptxas clean

# Drop-in extension checks (tests/cpp/test_dropin_ext.cpp), run by tests/test_gpu_dropin.py.
dropin_test: $(DROPIN_TEST)
$(DROPIN_TEST): tests/cpp/test_dropin_ext.cpp tests/cpp/doctest.h $(DROPIN)
	$(CXX) -std=c++20 -O2 -Itests/cpp -Iinclude -o $@ tests/cpp/test_dropin_ext.cpp \
	    -L$(PKG)/lib -llsqfit_b200 -llsqfit_cuda -Wl,-rpath,'$$ORIGIN'
