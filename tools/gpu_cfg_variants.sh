#!/bin/bash
# Config sweep (tools/bench_configs.py) for the product library and each
# variant in paper_2206_01784_b200/_lib/variants/.  usage: TAG ONLY variant...
cd "$(dirname "$0")/.."
TAG=$1; ONLY=$2; shift 2
mkdir -p gpurun_out
timeout 600 python tools/bench_configs.py --steps 5 --only "$ONLY" > gpurun_out/cfgv_${TAG}_product.jsonl 2>&1
for v in "$@"; do
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 600 python tools/bench_configs.py --steps 5 --only "$ONLY" > gpurun_out/cfgv_${TAG}_$v.jsonl 2>&1
done
for f in gpurun_out/cfgv_${TAG}_*.jsonl; do
  echo "== $f"; python -c "
import json,sys
for l in open('$f'):
    try: d=json.loads(l)
    except Exception: continue
    print(f\"{d['config']:40s} {d['gkeys']:7.2f} GKey/s  hist {d['hist_us']:6.1f}  pass {sum(d['pass_us'])/len(d['pass_us']):7.1f} us\")
"; done
