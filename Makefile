# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with
# the gpurun snapshot).  `make` == what __graft_entry__.build() runs.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -cudart shared \
           -Xptxas -v -Iinclude
SRC_DIR := paper_2601_19489_b200/csrc
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB := paper_2601_19489_b200/libtilesplat_b200.so

all: $(LIB)

build/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/tsr_common.cuh $(SRC_DIR)/tsr_vjp_adam.cuh include/tilesplat_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart shared -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean

# instrumented K2 (per-phase timestamps) for tools/k2_trace.py only
trace: build/libtilesplat_b200_trace.so
build/libtilesplat_b200_trace.so: $(SRCS) $(SRC_DIR)/tsr_common.cuh include/tilesplat_b200.h
	@mkdir -p build
	$(NVCC) -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -cudart shared -Iinclude -DTSR_K2_TRACE -shared -o $@ $(SRCS)

# experiment variants: make variant V=name VFLAGS="-DFOO=1" -> build/libtilesplat_b200_<name>.so
variant:
	@mkdir -p build
	$(NVCC) -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -cudart shared -Iinclude $(VFLAGS) -shared -o build/libtilesplat_b200_$(V).so $(SRCS)
