#!/bin/bash
# Build the last commit's kernels as variant "head" so A/B runs compare the
# working tree against HEAD on the same GPU box.
cd "$(dirname "$0")/.."
tmp=$(mktemp -d)
git archive HEAD paper_2206_01784_b200/csrc include | tar -x -C $tmp
mkdir -p paper_2206_01784_b200/_lib/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr "$@" -shared -o paper_2206_01784_b200/_lib/variants/head.so $tmp/paper_2206_01784_b200/csrc/*.cu -lcudart
rm -rf $tmp
