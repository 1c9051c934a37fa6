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

clean:
	rm -rf build $(LIB)

.PHONY: all clean
