# Builds the C-ABI library in-tree (travels to the GPU box with the snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := $(wildcard paper_2604_08585_b200/csrc/*.cu)
OBJ := $(patsubst paper_2604_08585_b200/csrc/%.cu,build/obj/%.o,$(SRC))
LIB := paper_2604_08585_b200/libqcfuse_b200.so

all: $(LIB)

build/obj/%.o: paper_2604_08585_b200/csrc/%.cu paper_2604_08585_b200/csrc/*.cuh include/qcfuse_b200.h
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

# measurement build (tools/attn_trace.py): per-CTA timeline stamps in the attention kernel
trace: tools/bin/libqcf_trace.so
tools/bin/libqcf_trace.so: $(SRC) paper_2604_08585_b200/csrc/*.cuh include/qcfuse_b200.h
	@mkdir -p build/trace tools/bin
	for f in $(SRC); do $(NVCC) $(NVFLAGS) -DQCF_ATTN_TRACE -c $$f -o build/trace/$$(basename $$f .cu).o || exit 1; done
	$(NVCC) $(ARCH) -shared -o $@ build/trace/*.o

clean:
	rm -rf build $(LIB) tools/bin/libqcf_trace.so

.PHONY: all clean trace
