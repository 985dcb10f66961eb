#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python tools/lookback_diag.py >> gpurun_out/diag.log 2>&1
done
echo done
