# Builds the sm_100a C-ABI library (in-tree, so it travels with gpurun) and the
# C oracle used by the tests.  Each .cu compiles to its own object so a kernel
# edit does not recompile the CUB-heavy units.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v $(XFLAGS)
SRC = $(wildcard paper_2411_09809_b200/csrc/*.cu)
HDR = $(wildcard paper_2411_09809_b200/csrc/*.cuh) include/glare_b200.h
BUILD ?= build/obj
LIBDIR ?= paper_2411_09809_b200/_lib
LIB = $(LIBDIR)/libglare_b200.so
OBJ = $(patsubst paper_2411_09809_b200/csrc/%.cu,$(BUILD)/%.o,$(SRC))

all: $(LIB) oracle

$(BUILD)/%.o: paper_2411_09809_b200/csrc/%.cu $(HDR)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJ)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -ldl
	cat $(BUILD)/*.ptxas.log > $(LIBDIR)/ptxas.log

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build paper_2411_09809_b200/_lib oracle/_build

.PHONY: all oracle clean
