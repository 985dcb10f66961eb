#!/bin/bash
# ncu full capture of one binning pass + one histogram of the bench workload.
# usage: tools/gpu_prof.sh TAG [variant]
cd "$(dirname "$0")/.."
TAG=$1; V=${2:-}
mkdir -p gpurun_out
LIBENV=""
if [ -n "$V" ]; then LIBENV="ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$V.so"; fi
env $LIBENV timeout 600 ncu --set full --clock-control none --import-source on -k regex:binning -s 4 -c 1 -f -o gpurun_out/prof_binning_$TAG \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_bin_$TAG.log 2>&1
env $LIBENV timeout 300 python tools/lookback_diag.py
echo done
