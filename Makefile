# Builds the sm_100a library (product) and the CPU oracle (test infrastructure).
# `make -j` compiles the kernel translation units in parallel.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xptxas -v
CSRC := paper_1703_06256_b200/csrc
OBJDIR := build/obj
LIB := paper_1703_06256_b200/libhogb200.so
UNITS := hog_abi k_bin k_bin_oct k_planes_a k_planes_b k_planes_c k_planes_d k_window k_scores k_scores_i8 k_detect k_rect
OBJS := $(addprefix $(OBJDIR)/,$(addsuffix .o,$(UNITS)))
HDRS := $(CSRC)/hog_common.cuh $(CSRC)/k_planes.cuh include/hogb200.h

IOLIB := paper_1703_06256_b200/libhogio.so

all: $(LIB) $(IOLIB) oracle

# host wire formats (PNM decode, descriptor text): plain C++, no CUDA
$(IOLIB): $(CSRC)/hogio.cpp include/hogio.h
	g++ -O3 -std=c++17 -fPIC -shared -pthread -o $@ $(CSRC)/hogio.cpp

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) $(EXTRA) -c -o $@ $< 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)
	cat $(OBJDIR)/*.ptxas.log > build_ptxas.log

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf $(OBJDIR) $(LIB) $(IOLIB) build_ptxas.log
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
