# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with the
# snapshot) and the oracle's C helpers.  `make -j` ; `make clean`.
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             --expt-relaxed-constexpr -Iinclude
PKG       := paper_2410_19367_b200
SRC       := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cpp)
OBJ       := $(patsubst $(PKG)/csrc/%,build/%.o,$(SRC))
LIB       := $(PKG)/libbitpipe_b200.so

all: $(LIB)

build/%.cu.o: $(PKG)/csrc/%.cu $(PKG)/csrc/*.cuh include/bitpipe.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/%.cpp.o: $(PKG)/csrc/%.cpp include/bitpipe.h include/bitpipe_comm.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -cudart static -ldl

# phase-traced build for tools/attn_trace.py and tools/gemm_trace.py (not the product)
TRACE_LIB := tools/libbitpipe_trace.so
trace: $(TRACE_LIB)
$(TRACE_LIB): $(SRC) $(PKG)/csrc/*.cuh include/bitpipe.h include/bitpipe_comm.h
	@mkdir -p build_trace
	for f in $(SRC); do $(NVCC) $(NVFLAGS) -DBP_ATTN_TRACE -DBP_GEMM_TRACE -c $$f -o build_trace/$$(basename $$f).o || exit 1; done
	$(NVCC) $(ARCH) -shared -o $@ build_trace/*.o -cudart static -ldl

clean:
	rm -rf build build_trace $(LIB)

.PHONY: all clean trace
