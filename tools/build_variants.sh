#!/bin/bash
# Build library variants for A/B timing on the GPU box:
#   tools/build_variants.sh name "-DFLAG=1 ..." [name "flags" ...]
# Each lands in paper_2206_01784_b200/_lib/variants/<name>.so (select with
# ONESWEEP_B200_LIB=...).
cd "$(dirname "$0")/.."
mkdir -p paper_2206_01784_b200/_lib/variants
SRCS=$(ls paper_2206_01784_b200/csrc/*.cu)
pids=()
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
    --expt-relaxed-constexpr $flags -shared -o paper_2206_01784_b200/_lib/variants/$name.so $SRCS -lcudart &
  pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait $p || rc=1; done
exit $rc
