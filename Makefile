# B200 VQMC library: nvcc for sm_100a, in-tree outputs (they travel to the GPU box).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v
SRC := paper_2106_13308_b200/csrc/kernels.cu paper_2106_13308_b200/csrc/head.cu paper_2106_13308_b200/csrc/gemm.cu paper_2106_13308_b200/csrc/capi.cu paper_2106_13308_b200/csrc/sr.cu paper_2106_13308_b200/csrc/energy_dense.cu paper_2106_13308_b200/csrc/spec.cu
HOSTSRC := paper_2106_13308_b200/csrc/host.cpp
HDRS := $(wildcard paper_2106_13308_b200/csrc/*.cuh) include/vqmc_b200.h Makefile
LIB := paper_2106_13308_b200/lib/libvqmc_b200.so
OBJDIR := build/obj
OBJS := $(patsubst paper_2106_13308_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC)) $(OBJDIR)/host.o

CLI := paper_2106_13308_b200/bin/vqmc

all: $(LIB) $(CLI) oracle

$(OBJDIR)/%.o: paper_2106_13308_b200/csrc/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(OBJDIR)/host.o: $(HOSTSRC) include/vqmc_b200.h Makefile
	@mkdir -p $(OBJDIR)
	g++ -O3 -march=x86-64-v3 -std=c++17 -fPIC -Iinclude -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p paper_2106_13308_b200/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl -lpthread

$(CLI): tools/vqmc_cli.cpp include/vqmc_b200/vqmc.hpp include/vqmc_b200.h $(LIB)
	@mkdir -p paper_2106_13308_b200/bin
	g++ -O2 -std=c++17 -Iinclude -o $@ tools/vqmc_cli.cpp -Lpaper_2106_13308_b200/lib -lvqmc_b200 -Wl,-rpath,'$$ORIGIN/../lib'

oracle:
	$(MAKE) -s -C oracle

# timeline-instrumented copy of the library (tools/tail_trace.py): umma2 kernels record %globaltimer
TRACE_LIB := paper_2106_13308_b200/lib/trace/libvqmc_trace.so
trace: $(TRACE_LIB)
$(TRACE_LIB): $(SRC) $(HOSTSRC) $(HDRS)
	@mkdir -p paper_2106_13308_b200/lib/trace
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -DVQMC_TAIL_TRACE -shared -o $@ $(SRC) $(HOSTSRC) -ldl -lpthread

clean:
	rm -rf build paper_2106_13308_b200/lib paper_2106_13308_b200/bin oracle/_build

.PHONY: all oracle clean trace
