# Builds the C-ABI shared library librrg.so for sm_100a (B200) and the oracle's C helpers.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude
SRC := paper_2410_18926_b200/csrc/rrg_api.cu paper_2410_18926_b200/csrc/rrg_kernels.cu paper_2410_18926_b200/csrc/rrg_cluster_score.cu paper_2410_18926_b200/csrc/rrg_ground_truth.cu paper_2410_18926_b200/csrc/rrg_sliced_gemm.cu paper_2410_18926_b200/csrc/rrg_screen.cu paper_2410_18926_b200/csrc/rrg_route_screen.cu
HDR := include/rrg.h paper_2410_18926_b200/csrc/rrg_common.cuh paper_2410_18926_b200/csrc/rrg_kernels.h
LIB := paper_2410_18926_b200/librrg.so
OBJ := $(patsubst %.cu,build/%.o,$(SRC))

all: $(LIB)

build/%.o: %.cu $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared $(OBJ) -o $@ -lz

clean:
	rm -rf build $(LIB)

.PHONY: all clean
