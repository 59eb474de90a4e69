# Builds the sm_100a extension in-tree (the .so travels to the GPU box).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xptxas -v -cudart static --expt-relaxed-constexpr
SRC_DIR := paper_2604_07239_b200/csrc
LIB := paper_2604_07239_b200/_lib/libfade_b200.so
SRCS := $(wildcard $(SRC_DIR)/*.cu)
HDRS := $(wildcard $(SRC_DIR)/*.cuh) include/fade_b200.h
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))

all: $(LIB) oracle

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC -o $@ $(OBJS)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all clean oracle
