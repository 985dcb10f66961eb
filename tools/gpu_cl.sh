#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_cl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cl.log
bash tools/gpu_bench_variants.sh cl "$@"
