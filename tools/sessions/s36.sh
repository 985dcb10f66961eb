#!/bin/bash
# knob A/B (key prefetch depth, look-back window, keys-only uniform-warp
# shortcut) over C1/C2 plus keys-only distributions for the shortcut
cd "$(dirname "$0")/../.."
bash tools/sessions/s34.sh knobs 3 "C1,C2" pf3 lb5 lb7 nouni
for v in product nouni; do
  if [ $v = product ]; then LIB=""; else LIB="ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so"; fi
  echo "== keys_dist $v"; env $LIB TAG=$v timeout 600 python tools/keys_dist.py 2>&1 | tail -6
done
