# libdspmv (C ABI, sm_100a kernels) and the oracle's O1 library.
PY        ?= python
NCCL_HOME ?= $(shell $(PY) -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])")
CUDA_HOME ?= /usr/local/cuda
NVCC      := $(CUDA_HOME)/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
SRC       := paper_2203_02530_b200/csrc
OUT       := paper_2203_02530_b200/lib
BUILD     := build/obj

NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
CXXFLAGS  := -O2 -g -fPIC -std=c++17 -Wall -Wno-unused-function -I$(CUDA_HOME)/include -I$(NCCL_HOME)/include

OBJS := $(BUILD)/kernels.o $(BUILD)/api.o $(BUILD)/planner.o $(BUILD)/schedule.o

all: $(OUT)/libdspmv.so oracle/libo1.so gen/libgenc.so

$(BUILD):
	mkdir -p $(BUILD) $(OUT)

$(BUILD)/kernels.o: $(SRC)/kernels.cu $(SRC)/runtime.h $(SRC)/internal.h include/dspmv.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_kernels.txt || (cat $(BUILD)/ptxas_kernels.txt; false)

$(BUILD)/%.o: $(SRC)/%.cpp $(SRC)/runtime.h $(SRC)/internal.h include/dspmv.h | $(BUILD)
	g++ $(CXXFLAGS) -c $< -o $@

$(OUT)/libdspmv.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL_HOME)/lib -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_HOME)/lib

# instrumented variant (per-phase clock64 counters), only with PROFILE=1
$(BUILD)/kernels_prof.o: $(SRC)/kernels.cu $(SRC)/runtime.h $(SRC)/internal.h include/dspmv.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -DDSPMV_PROFILE -c $< -o $@ 2> $(BUILD)/ptxas_prof.txt || (cat $(BUILD)/ptxas_prof.txt; false)

$(OUT)/libdspmv_prof.so: $(BUILD)/kernels_prof.o $(BUILD)/api.o $(BUILD)/planner.o $(BUILD)/schedule.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -L$(NCCL_HOME)/lib -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_HOME)/lib

# diagnostic variants (DIAG=1: no gather, DIAG=2: row-local gather, DIAG=3: CSR-stream without
# row sums, DIAG=4: CSR-stream without gathers), never the product
$(BUILD)/kernels_diag$(DIAG).o: $(SRC)/kernels.cu $(SRC)/runtime.h $(SRC)/internal.h include/dspmv.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -DDSPMV_DIAG_GATHER=$(DIAG) -c $< -o $@ 2> /dev/null

$(OUT)/libdspmv_diag$(DIAG).so: $(BUILD)/kernels_diag$(DIAG).o $(BUILD)/api.o $(BUILD)/planner.o $(BUILD)/schedule.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -L$(NCCL_HOME)/lib -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_HOME)/lib

ifeq ($(PROFILE),1)
all: $(OUT)/libdspmv_prof.so
endif

oracle/libo1.so: oracle/o1.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o $@ $< -lm

gen/libgenc.so: gen/genc.c
	gcc -O2 -ffp-contract=off -fPIC -shared -o $@ $< -lm

clean:
	rm -rf $(BUILD) $(OUT)/libdspmv.so oracle/libo1.so gen/libgenc.so

.PHONY: all clean
