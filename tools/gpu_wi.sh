#!/bin/bash
# Timing-only A/B (no correctness check): bench per variant.  usage: tools/gpu_wi.sh TAG variant...
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then LIB=""; else LIB="ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so"; fi
  env $LIB timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v'.ljust(12), round(d['value'],2), [round(x) for x in d['kernels']['binning_pass_us']])"
done
