#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 240 python tools/smoke_debug.py > gpurun_out/smoke_debug.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_debug.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_distributed.py -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
for v in minb2 minb3; do
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:binning -s 4 -c 1 -f -o gpurun_out/prof_binning2 \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:histogram -s 1 -c 1 -f -o gpurun_out/prof_hist2 \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_hist2.log 2>&1
echo done
