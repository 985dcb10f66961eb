# Build the sm_100a C-ABI library (the product) and the CPU oracle (test
# infrastructure).  `python -c "import __graft_entry__ as g; g.build()"` runs
# the same recipe.
NVCC ?= nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
PTXAS_V ?=

PKG := paper_2206_01784_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/onesweep_b200.h
LIB := $(PKG)/_lib/libonesweep_b200.so

all: $(LIB) oracle

$(LIB): $(SRCS) $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) $(NVFLAGS) $(PTXAS_V) -shared -o $@ $(SRCS) -lcudart

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	cuobjdump -sass $(LIB) > build_sass.txt

clean:
	rm -f $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean sass
