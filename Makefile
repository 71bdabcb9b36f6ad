# Builds the sm_100a library (product) and the CPU oracle (test infrastructure).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xptxas -v
LIB := paper_1703_06256_b200/libhogb200.so
SRC := paper_1703_06256_b200/csrc/hog_kernels.cu

all: $(LIB) oracle

$(LIB): $(SRC) include/hogb200.h
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIB) build_ptxas.log
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
