#!/bin/bash
# Iteration run: fast GPU tests, bench of each lib variant, ncu of the default lib.
# usage: tools/gpu_iter.sh TAG [variant ...]
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for v in "$@"; do
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${TAG}_$v.json 2> gpurun_out/bench_${TAG}_$v.err
done
V=${NCU_VARIANT:-}
LIBENV=""
if [ -n "$V" ]; then LIBENV="ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$V.so"; fi
env $LIBENV timeout 600 ncu --set full --clock-control none --import-source on -k regex:binning -s 4 -c 1 -f -o gpurun_out/prof_binning_$TAG \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_bin_$TAG.log 2>&1
env $LIBENV timeout 600 ncu --set full --clock-control none --import-source on -k regex:histogram -s 1 -c 1 -f -o gpurun_out/prof_hist_$TAG \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_hist_$TAG.log 2>&1
echo done
