# Builds the sm_100a library (in-tree; the .so travels to the GPU box with the repo).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
CSRC := paper_2301_03251_b200/csrc
SRC := $(wildcard $(CSRC)/*.cu) $(wildcard $(CSRC)/*.cpp)
HDR := $(wildcard $(CSRC)/*.h) $(wildcard $(CSRC)/*.cuh) include/hq.h
LIB := paper_2301_03251_b200/libhq.so
JITINC := $(CSRC)/hq_jit_src.inc

all: $(LIB) oracle

# hq_pod.h / hq_dev.cuh embedded as strings for the NVRTC-generated kernels
$(JITINC): $(CSRC)/hq_pod.h $(CSRC)/hq_dev.cuh
	@{ printf 'static const char kJitPod[] = R"__HQ__('; grep -v '#pragma once' $(CSRC)/hq_pod.h; \
	   printf ')__HQ__";\nstatic const char kJitDev[] = R"__HQ__('; grep -v '#pragma once' $(CSRC)/hq_dev.cuh; \
	   printf ')__HQ__";\n'; } > $@

$(LIB): $(SRC) $(HDR) $(JITINC)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -ldl

oracle:
	$(MAKE) -C oracle

ptxas: $(SRC) $(HDR) $(JITINC)
	$(NVCC) $(NVFLAGS) -Xptxas -v -shared -o /tmp/hq_ptxas.so $(SRC) -ldl 2>&1 | grep -E "Function properties|registers|spill|Compiling entry"

clean:
	rm -f $(LIB) $(JITINC)

.PHONY: all clean ptxas oracle
