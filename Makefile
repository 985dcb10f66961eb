# Build the sm_100a C-ABI library (the product), its race-exploration debug
# twin, and the CPU oracle (test infrastructure).
# `python -c "import __graft_entry__ as g; g.build()"` runs the same recipe.
NVCC ?= nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
PTXAS_V ?=

PKG := paper_2206_01784_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/onesweep_b200.h
LIB := $(PKG)/_lib/libonesweep_b200.so
DEBUG_LIB := $(PKG)/_lib/libonesweep_b200_debug.so
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/release/%.o,$(SRCS))
DEBUG_OBJS := $(patsubst $(PKG)/csrc/%.cu,build/debug/%.o,$(SRCS))
# Race/failure exploration (tests/test_gpu_race.py): pseudo-random
# __nanosleep jitter around the status publishes and the look-back (the
# reference's Jitter), a 2^16-poll look-back watchdog and failure injection
# (ONESWEEP_B200_DEBUG_STALL_TILE).
DEBUG_FLAGS := -DOS_JITTER=1 "-DOS_SPIN_LIMIT=(1u<<16)"

all: $(LIB) $(DEBUG_LIB) oracle

build/release/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) $(NVFLAGS) $(PTXAS_V) -c -o $@ $<

build/debug/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) $(NVFLAGS) $(DEBUG_FLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

$(DEBUG_LIB): $(DEBUG_OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(DEBUG_OBJS) -lcudart

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	cuobjdump -sass $(LIB) > build_sass.txt

clean:
	rm -rf build $(LIB) $(DEBUG_LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean sass
