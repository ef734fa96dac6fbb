# Build the B200 (sm_100a) library and the CPU parity checkers.
#   make            -> paper_1907_11678_b200/_lib/libvelan_gpu.so + oracle
#   make lib        -> the CUDA library only
#   make oracle     -> oracle/libvelan_oracle.so and oracle/_ref (test infra)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xptxas -v \
           -Xcompiler -fPIC,-ffp-contract=off,-O3 -Iinclude
LIB := paper_1907_11678_b200/_lib/libvelan_gpu.so
SRC := paper_1907_11678_b200/csrc/velan_gpu.cu paper_1907_11678_b200/csrc/synth.cpp \
       paper_1907_11678_b200/csrc/peak.cu paper_1907_11678_b200/csrc/ssf_io.cpp \
       paper_1907_11678_b200/csrc/synth_gpu.cu
HDR := paper_1907_11678_b200/csrc/semblance_kernels.cuh include/velan_gpu.h

all: lib oracle

lib: $(LIB)

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -lpthread 2> paper_1907_11678_b200/_lib/ptxas.log || (cat paper_1907_11678_b200/_lib/ptxas.log; exit 1)

oracle: lib
	$(MAKE) -C oracle

clean:
	rm -f $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean exp

# experimental builds (not shipped): make exp NAME=s3 DEFS="-DVELAN_STAGES=3"
exp:
	@mkdir -p paper_1907_11678_b200/_lib/exp
	$(NVCC) $(NVFLAGS) $(DEFS) -shared -o paper_1907_11678_b200/_lib/exp/lib$(NAME).so $(SRC) -lpthread 2> paper_1907_11678_b200/_lib/exp/$(NAME).log || (cat paper_1907_11678_b200/_lib/exp/$(NAME).log; exit 1)
