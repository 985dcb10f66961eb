#!/bin/bash
# Config A/B: per variant a quick correctness check and tools/bench_configs.py
# restricted to ONLY (e.g. "C3" or "C4").  usage: tools/gpu_cfg_ab.sh TAG ONLY variant...
cd "$(dirname "$0")/.."
TAG=$1; ONLY=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then LIB=""; else LIB="ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so"; fi
  env $LIB timeout 300 python tools/quick_check.py > gpurun_out/qc_${TAG}_$v.log 2>&1
  echo "== $v $(tail -1 gpurun_out/qc_${TAG}_$v.log)"
  env $LIB timeout 600 python tools/bench_configs.py --steps 5 --only "$ONLY" 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(' ', d.get('config', d.get('name','?'))[:40].ljust(40), round(d.get('value', d.get('gkeys', 0)),2), [round(x) for x in d.get('binning_pass_us', d.get('pass_us', []))][:3])
"
done
