# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2006_13387_b200/csrc/*.cu)
HDR := $(wildcard paper_2006_13387_b200/csrc/*.cuh) include/msgpu.h
LIB := paper_2006_13387_b200/libmsgpu.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(ARCH) $(NVFLAGS) -shared $(SRC) -o $@ -ldl 2> /tmp/ptxas.log || (cat /tmp/ptxas.log; false)

clean:
	rm -f $(LIB)

.PHONY: all clean
