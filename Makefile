# Builds the in-tree C-ABI library paper_2501_11407_b200/libsparseprop_b200.so (sm_100a only)
# and the C oracle.  `python -c "import __graft_entry__ as g; g.build()"` calls this.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2501_11407_b200/csrc/*.cu)
HDR := $(wildcard paper_2501_11407_b200/csrc/*.cuh) include/sparseprop_b200.h
OBJ := $(patsubst paper_2501_11407_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2501_11407_b200/libsparseprop_b200.so

all: $(LIB)

build/%.o: paper_2501_11407_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Iinclude -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
