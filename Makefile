# Builds the product library paper_2305_02522_b200/libbitgnn_b200.so (sm_100a)
# and the test-infrastructure oracle (oracle/liboracle.so, oracle/_ref).
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Iinclude -Xcompiler -fPIC \
           -Xptxas -v --expt-relaxed-constexpr
CSRC    := paper_2305_02522_b200/csrc
SRCS    := $(wildcard $(CSRC)/*.cu)
OBJS    := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDRS    := $(wildcard $(CSRC)/*.cuh) include/bitgnn_b200.h
LIB     := paper_2305_02522_b200/libbitgnn_b200.so

.PHONY: all lib oracle cpptest clean
all: lib oracle cpptest
lib: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS) $(CSRC)/exports.map
	$(NVCC) $(ARCH) -shared -cudart static -Xlinker --version-script=$(CSRC)/exports.map -o $@ $(OBJS) -ldl

oracle:
	$(MAKE) -C oracle all
oracle/liboracle.so:
	$(MAKE) -C oracle all

# C++ host-API test program (tests/cpp): the header-only shim over the C ABI,
# checked against the C oracle (test infrastructure).
CPPTEST := tests/cpp/bin/test_shim
cpptest: $(CPPTEST)
$(CPPTEST): tests/cpp/test_shim.cpp include/bitgnn_b200/bitgnn.hpp include/bitgnn_b200.h $(LIB) oracle/liboracle.so
	@mkdir -p tests/cpp/bin
	g++ -std=c++20 -O1 -Wall -Wextra -Wno-missing-field-initializers -Iinclude -Ioracle -o $@ $< \
	    -L paper_2305_02522_b200 -lbitgnn_b200 -L oracle -loracle \
	    -Wl,-rpath,'$$ORIGIN/../../../paper_2305_02522_b200' -Wl,-rpath,'$$ORIGIN/../../../oracle'

clean:
	rm -rf build $(LIB) tests/cpp/bin
	$(MAKE) -C oracle clean
