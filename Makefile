# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with gpurun).
# One object per source so `make -j` compiles them in parallel; the ptxas
# resource report of every kernel goes to build/ptxas/*.log (and /tmp/ptxas.log).
NVCC ?= nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2006_13387_b200/csrc/*.cu)
HDR := $(wildcard paper_2006_13387_b200/csrc/*.cuh) include/msgpu.h
OBJ := $(patsubst paper_2006_13387_b200/csrc/%.cu,build/obj/%.o,$(SRC))
LIB := paper_2006_13387_b200/libmsgpu.so

all: $(LIB)

build/obj/%.o: paper_2006_13387_b200/csrc/%.cu $(HDR)
	@mkdir -p build/obj build/ptxas
	$(NVCC) $(ARCH) $(NVFLAGS) -c $< -o $@ 2> build/ptxas/$*.log || (cat build/ptxas/$*.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared $(OBJ) -o $@ -ldl
	@cat build/ptxas/*.log > /tmp/ptxas.log

# bounds-checked variant (device-side asserts, -DMS_BOUNDS_CHECK) for tests/test_gpu_bounds.py
CHK_OBJ := $(patsubst paper_2006_13387_b200/csrc/%.cu,build/check/%.o,$(SRC))
CHK_LIB := build/check/libmsgpu_check.so

build/check/%.o: paper_2006_13387_b200/csrc/%.cu $(HDR)
	@mkdir -p build/check
	$(NVCC) $(ARCH) $(NVFLAGS) -DMS_BOUNDS_CHECK -c $< -o $@ 2> build/check/$*.log || (cat build/check/$*.log; false)

$(CHK_LIB): $(CHK_OBJ)
	$(NVCC) $(ARCH) -shared $(CHK_OBJ) -o $@ -ldl

check: $(CHK_LIB)

clean:
	rm -f $(LIB) $(OBJ)

.PHONY: all check clean
