#!/bin/bash
# value-width sweep: product vs key-value write-fence variants, interleaved x2
cd "$(dirname "$0")/../.."
for r in 1 2; do
  for v in product "$@"; do
    if [ $v = product ]; then LIB=""; else LIB="ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so"; fi
    echo "== $v run $r"; env $LIB timeout 600 python tools/value_widths.py 2>&1 | grep -v "0-byte\|4-byte" | grep "GKey"
  done
done
