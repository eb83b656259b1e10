# Builds everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> product library + oracle (+ oracle/_ref when the reference is present)
#   make lib        -> paper_2304_08662_b200/_lib/libxdrop_b200.so  (sm_100a)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v
CSRC := paper_2304_08662_b200/csrc
LIB := paper_2304_08662_b200/_lib/libxdrop_b200.so
OBJDIR := build

SRCS_CU := $(CSRC)/xb_kernels.cu $(CSRC)/xb_thread.cu $(CSRC)/xb_group.cu $(CSRC)/xb_lane.cu $(CSRC)/xb_wide.cu $(CSRC)/xb_engine.cu
SRCS_CPP := $(CSRC)/xb_synth.cpp $(CSRC)/xb_ingest.cpp
HDRS := $(CSRC)/xb_internal.h $(CSRC)/xb_kernels.cuh include/xdrop_b200.h

all: lib oracle checked

# parallel object builds: make -j lib

lib: $(LIB)

$(OBJDIR)/xb_kernels.o: $(CSRC)/xb_kernels.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> $(OBJDIR)/xb_kernels.ptxas.txt || (cat $(OBJDIR)/xb_kernels.ptxas.txt; exit 1)

$(OBJDIR)/xb_thread.o: $(CSRC)/xb_thread.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> $(OBJDIR)/xb_thread.ptxas.txt || (cat $(OBJDIR)/xb_thread.ptxas.txt; exit 1)

$(OBJDIR)/xb_group.o: $(CSRC)/xb_group.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> $(OBJDIR)/xb_group.ptxas.txt || (cat $(OBJDIR)/xb_group.ptxas.txt; exit 1)

$(OBJDIR)/xb_lane.o: $(CSRC)/xb_lane.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> $(OBJDIR)/xb_lane.ptxas.txt || (cat $(OBJDIR)/xb_lane.ptxas.txt; exit 1)

$(OBJDIR)/xb_wide.o: $(CSRC)/xb_wide.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> $(OBJDIR)/xb_wide.ptxas.txt || (cat $(OBJDIR)/xb_wide.ptxas.txt; exit 1)

$(OBJDIR)/xb_engine.o: $(CSRC)/xb_engine.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> $(OBJDIR)/xb_engine.ptxas.txt || (cat $(OBJDIR)/xb_engine.ptxas.txt; exit 1)

$(OBJDIR)/xb_synth.o: $(CSRC)/xb_synth.cpp include/xdrop_b200.h
	@mkdir -p $(OBJDIR)
	/usr/bin/g++ -O3 -std=c++17 -fPIC -c -o $@ $<

$(OBJDIR)/xb_ingest.o: $(CSRC)/xb_ingest.cpp include/xdrop_b200.h
	@mkdir -p $(OBJDIR)
	/usr/bin/g++ -O3 -std=c++17 -fPIC -Wall -c -o $@ $<

$(LIB): $(OBJDIR)/xb_kernels.o $(OBJDIR)/xb_thread.o $(OBJDIR)/xb_group.o $(OBJDIR)/xb_lane.o $(OBJDIR)/xb_wide.o $(OBJDIR)/xb_engine.o $(OBJDIR)/xb_synth.o $(OBJDIR)/xb_ingest.o
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lcudadevrt -lpthread

# the bounds-checked variant (XB_CHECKS: every pool load, result row, list
# slot, record and table lookup asserted; xb_debug_checks reads the first
# failure): the GPU test-suite runs against it with XB_LIB_PATH
CHK_LIB := paper_2304_08662_b200/_lib/libxdrop_b200_checked.so
CHKDIR := build_chk
checked: $(CHK_LIB)
$(CHKDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(CHKDIR)
	$(NVCC) $(NVFLAGS) -DXB_CHECKS=1 -dc -o $@ $< > /dev/null 2>&1 || $(NVCC) $(NVFLAGS) -DXB_CHECKS=1 -dc -o $@ $<
$(CHK_LIB): $(CHKDIR)/xb_kernels.o $(CHKDIR)/xb_thread.o $(CHKDIR)/xb_group.o $(CHKDIR)/xb_lane.o $(CHKDIR)/xb_wide.o $(CHKDIR)/xb_engine.o $(OBJDIR)/xb_synth.o $(OBJDIR)/xb_ingest.o
	@mkdir -p $(dir $(CHK_LIB))
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lcudadevrt -lpthread

oracle: lib
	$(MAKE) -s -C oracle liboracle.so
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -s -C oracle ref; fi

clean:
	rm -rf $(OBJDIR) $(LIB) $(CHKDIR) $(CHK_LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean checked
