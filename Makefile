# libpe: B200 (sm_100a) parareal hot path, built in-tree so the .so travels with the repo.
NVCC ?= /usr/local/cuda/bin/nvcc
CUDA_LIB ?= /usr/local/cuda/lib64
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           -Iinclude -Ipaper_2411_09244_b200/csrc --expt-relaxed-constexpr
SRC := $(wildcard paper_2411_09244_b200/csrc/*.cu)
HDR := $(wildcard paper_2411_09244_b200/csrc/*.h) include/pe.h
OBJ := $(patsubst paper_2411_09244_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2411_09244_b200/libpe.so

all: $(LIB)

build/%.o: paper_2411_09244_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -L$(CUDA_LIB) -lcublas -lcusolver \
	    -Xlinker -rpath=$(CUDA_LIB)

ptxas: $(SRC)
	@mkdir -p build
	for f in $(SRC); do $(NVCC) $(NVFLAGS) -Xptxas -v -c $$f -o /dev/null 2>&1 | grep -E "Used|spill"; done

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) | grep -cE "DMMA" ; true

clean:
	rm -rf build $(LIB)

.PHONY: all clean ptxas sass
