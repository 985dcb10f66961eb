#!/bin/bash
# the write fence for every u32-key kernel with values: value widths, C3, GPU suite
cd "$(dirname "$0")/../.."
timeout 600 python tools/value_widths.py 2>&1 | grep GKey
timeout 600 python tools/bench_configs.py --steps 5 --only "C3 u32 pairs q=1,C3 u32 pairs q=16" 2>&1 | grep config
bash tools/gpu_tests.sh kvf nosan
