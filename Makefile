# Builds the sm_100a C-ABI library (in-tree, so it travels with gpurun) and the
# C oracle used by the tests.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v
SRC = $(wildcard paper_2411_09809_b200/csrc/*.cu)
HDR = $(wildcard paper_2411_09809_b200/csrc/*.cuh) include/glare_b200.h
LIB = paper_2411_09809_b200/_lib/libglare_b200.so

all: $(LIB) oracle

$(LIB): $(SRC) $(HDR)
	mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> paper_2411_09809_b200/_lib/ptxas.log || (cat paper_2411_09809_b200/_lib/ptxas.log; exit 1)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf paper_2411_09809_b200/_lib oracle/_build

.PHONY: all oracle clean
