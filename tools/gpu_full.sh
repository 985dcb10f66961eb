#!/bin/bash
# Full measurement session: smoke, all GPU tests, bench x2 (variance), ncu
# launch list and full captures of the two kernels.  TAG names the outputs.
cd "$(dirname "$0")/.."
TAG=${1:-full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${TAG}_rep.json 2>> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_$TAG.err
timeout 300 python tools/lookback_diag.py > gpurun_out/diag_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:binning -s 4 -c 1 -f -o gpurun_out/prof_binning_$TAG \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_bin_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:histogram -s 1 -c 1 -f -o gpurun_out/prof_hist_$TAG \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_hist_$TAG.log 2>&1

timeout 900 python tools/bench_configs.py --steps 5 > gpurun_out/cfgs_$TAG.jsonl 2>&1
echo done
