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

all: $(LIB) oracle experiments

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC -o $@ $(OBJS)

oracle:
	$(MAKE) -s -C oracle

# phase-instrumented build (globaltimer stamps in the W12 and e12 GEMMs, read
# by tools/phase_probe.py through FADE_LIB_PATH); never the shipped library
PROBE_OBJS := $(patsubst $(SRC_DIR)/%.cu,build/probe/%.o,$(SRCS))
build/probe/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build/probe
	$(NVCC) $(NVFLAGS) -DFADE_PHASE_PROBE -DFADE_EXPERIMENTS -dc -o $@ $< 2> build/probe/$*.ptxas.log || (cat build/probe/$*.ptxas.log; exit 1)
build/probe/libfade_b200.so: $(PROBE_OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC -o $@ $(PROBE_OBJS)
probe: build/probe/libfade_b200.so

# experiments build: reads the FADE_* tuning / debug knobs from the
# environment (common.cuh knob()); load it with FADE_LIB_PATH for A/B timing.
# The shipped library above ignores them.
EXP_OBJS := $(patsubst $(SRC_DIR)/%.cu,build/exp/%.o,$(SRCS))
build/exp/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build/exp
	$(NVCC) $(NVFLAGS) -DFADE_EXPERIMENTS -dc -o $@ $< 2> build/exp/$*.ptxas.log || (cat build/exp/$*.ptxas.log; exit 1)
build/exp/libfade_b200.so: $(EXP_OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC -o $@ $(EXP_OBJS)
experiments: build/exp/libfade_b200.so

clean:
	rm -rf build $(LIB)

.PHONY: all clean oracle probe experiments
