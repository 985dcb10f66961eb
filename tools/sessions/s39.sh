#!/bin/bash
# OS_SYNCWARP=2 as the product: A/B against the previous commit over C1-C4,
# then the whole GPU suite and smoke on the new library
cd "$(dirname "$0")/../.."
bash tools/sessions/s34.sh sw2 3 "C1,C2,C3 u32 pairs q=1,C3 u32 pairs q=16,C4 uint64" head
bash tools/gpu_tests.sh sw2 nosan
