#!/bin/bash
# OS_PAIR_WRITE_FENCE=3 as the product: A/B against the previous commit over
# every C3 distribution and C2/C4, then the GPU suite and smoke
cd "$(dirname "$0")/../.."
bash tools/sessions/s34.sh pwf 3 "C2,C3 u32 pairs,C4 uint64" head
bash tools/gpu_tests.sh pwf nosan
