# Builds the sm_100a library (in-tree, travels to the GPU box with the repo).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
SRC := $(wildcard paper_2301_03251_b200/csrc/*.cu) $(wildcard paper_2301_03251_b200/csrc/*.cpp)
HDR := $(wildcard paper_2301_03251_b200/csrc/*.h) $(wildcard paper_2301_03251_b200/csrc/*.cuh) include/hq.h
LIB := paper_2301_03251_b200/libhq.so

all: $(LIB) oracle

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)

oracle:
	$(MAKE) -C oracle

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -shared -o /tmp/hq_ptxas.so $(SRC) 2>&1 | grep -E "Function properties|registers|spill|Compiling entry"

clean:
	rm -f $(LIB)

.PHONY: all clean ptxas oracle
