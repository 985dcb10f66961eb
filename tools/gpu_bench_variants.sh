#!/bin/bash
# Bench (no e2e/cpu) + look-back diagnostics for each library variant.
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${TAG}_$v.json 2> gpurun_out/bench_${TAG}_$v.err
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python tools/lookback_diag.py >> gpurun_out/diag_$TAG.log 2>&1
done
echo done
