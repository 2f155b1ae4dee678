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

.PHONY: all lib oracle clean
all: lib oracle
lib: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS) $(CSRC)/exports.map
	$(NVCC) $(ARCH) -shared -cudart static -Xlinker --version-script=$(CSRC)/exports.map -o $@ $(OBJS) -ldl

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean
