#!/bin/bash
# Extended fuzz sweep at HEAD (FUZZ_CASES x 3 seeds) plus the race tests
# under the jitter build, repeated
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for seed in 4 5 6; do
  FUZZ_CASES=2000 FUZZ_SEED=$seed timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3 | sed "s/^/seed $seed: /"
done > gpurun_out/fuzz_r2k.txt
for r in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_race.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done > gpurun_out/race_r2k.txt
cat gpurun_out/fuzz_r2k.txt gpurun_out/race_r2k.txt
