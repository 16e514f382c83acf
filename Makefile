# Build the C-ABI shared library for sm_100a (in-tree, travels with gpurun).
NVCC ?= nvcc
CUDA_ARCH ?= -gencode arch=compute_100a,code=sm_100a
SRC_DIR := paper_2602_19699_b200/csrc
OUT := paper_2602_19699_b200/libcacto_b200.so
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
HDRS := $(wildcard $(SRC_DIR)/*.cuh) include/cacto_b200.h
NVFLAGS := -O3 -std=c++17 $(CUDA_ARCH) -lineinfo -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr \
           -Xptxas -warn-spills $(EXTRA_NVFLAGS)

all: $(OUT)

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OUT): $(OBJS)
	$(NVCC) -shared $(CUDA_ARCH) -o $@ $(OBJS) -lcudart

clean:
	rm -rf build $(OUT)

.PHONY: all clean
