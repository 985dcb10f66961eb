#!/bin/bash
# tools/bench_configs.py for the default lib and each variant: tools/gpu_cfgs.sh TAG [variant ...]
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
echo "== default"; timeout 600 python tools/bench_configs.py --steps 5 $CFG_ARGS 2>&1 | tee gpurun_out/cfgs_${TAG}_default.jsonl
for v in "$@"; do
  echo "== $v"; ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 600 python tools/bench_configs.py --steps 5 $CFG_ARGS 2>&1 | tee gpurun_out/cfgs_${TAG}_$v.jsonl
done
