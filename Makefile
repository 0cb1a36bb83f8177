# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> product library + synth + oracle
#   make oracle     -> CPU oracle only (gcc)
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
# the library's version = the last commit that changed its sources (doc-only commits keep it,
# so ncu captures of the same kernels stay matched to the library, bench.py traffic_source)
GIT_SHA   := $(shell git log -1 --format=%h --abbrev=12 -- paper_1805_07339_b200/csrc include Makefile 2>/dev/null | grep . || echo unknown)
# uncommitted changes to those sources mark the build (a capture of it matches no commit)
GIT_SHA   := $(GIT_SHA)$(shell git status --porcelain -- paper_1805_07339_b200/csrc include Makefile 2>/dev/null | grep -q . && echo -dirty)
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -shared -cudart static
CC        ?= gcc
CFLAGS    := -O2 -std=c11 -fPIC -Wall -Wextra -shared

PKG       := paper_1805_07339_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libscn.so
LIB_TUNE  := $(PKG)/libscn_tuning.so
LIB_SRCS  := $(wildcard $(CSRC)/*.cu) $(wildcard $(CSRC)/*.cpp)
LIB_HDRS  := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/scn.h

SYNTH_HOST := scn_synth/libscn_synth_host.so
SYNTH_CUDA := scn_synth/libscn_synth_cuda.so
ORACLE     := oracle/libscn_oracle.so
MICRO      := tools/micro/k0

DEMO       := examples/scn_demo
CUDA_HOME  ?= /usr/local/cuda

all: $(LIB) $(LIB_TUNE) $(SYNTH_HOST) $(SYNTH_CUDA) $(ORACLE) $(DEMO)

lib: $(LIB)
# measurement build: the same kernels with the SCN_* environment knobs (grid, tiles,
# ring depth, L2 prefetch) read once per process; loaded by the binding when SCN_LIB=tuning
tuning: $(LIB_TUNE)
oracle: $(ORACLE) $(SYNTH_HOST)
micro: $(MICRO)

# .git/logs/HEAD changes with every commit, so the embedded SHA (scn_version) stays current
$(LIB): $(LIB_SRCS) $(LIB_HDRS) Makefile $(wildcard .git/logs/HEAD)
	$(NVCC) $(NVFLAGS) -Iinclude -DSCN_GIT_SHA=\"$(GIT_SHA)\" -Xptxas -v $(LIB_SRCS) -o $@ 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; false)

$(LIB_TUNE): $(LIB_SRCS) $(LIB_HDRS) Makefile $(wildcard .git/logs/HEAD)
	$(NVCC) $(NVFLAGS) -Iinclude -DSCN_TUNING -DSCN_GIT_SHA=\"$(GIT_SHA)-tuning\" $(LIB_SRCS) -o $@

$(SYNTH_HOST): scn_synth/synth_host.c scn_synth/scn_synth.h
	$(CC) $(CFLAGS) $< -o $@

$(SYNTH_CUDA): scn_synth/synth_cuda.cu scn_synth/synth_host.c scn_synth/scn_synth.h
	$(NVCC) $(NVFLAGS) scn_synth/synth_cuda.cu -o $@

$(ORACLE): oracle/scn_oracle.c scn_synth/synth_host.c scn_synth/scn_synth.h
	$(CC) $(CFLAGS) oracle/scn_oracle.c scn_synth/synth_host.c -o $@

# a plain C consumer of the ABI (no Python): links libscn.so and the CUDA runtime
$(DEMO): examples/scn_demo.c include/scn.h $(LIB)
	$(CC) -O2 -std=c11 -Wall -Iinclude -I$(CUDA_HOME)/include $< -o $@ -L$(PKG) -lscn \
	  -L$(CUDA_HOME)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,$(CUDA_HOME)/lib64

$(MICRO): tools/micro/k0.cu
	$(NVCC) $(ARCH) -O3 -o $@ $<

clean:
	rm -f $(LIB) $(LIB_TUNE) $(SYNTH_HOST) $(SYNTH_CUDA) $(ORACLE) $(MICRO) $(DEMO)

.PHONY: all lib tuning oracle micro clean
