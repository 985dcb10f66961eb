#!/bin/bash
# A/B of library variants over C1-C4 (tools/bench_configs.py), interleaved
# REPS times: usage tools/sessions/s34.sh TAG REPS ONLY variant...
cd "$(dirname "$0")/../.."
TAG=$1; REPS=$2; ONLY=$3; shift 3
mkdir -p gpurun_out
for r in $(seq 1 $REPS); do
  for v in product "$@"; do
    if [ $v = product ]; then LIB=""; else LIB="ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so"; fi
    env $LIB timeout 600 python tools/bench_configs.py --steps 5 --only "$ONLY" >> gpurun_out/ab_${TAG}_$v.jsonl 2>&1
  done
done
for v in product "$@"; do
  echo "== $v"; python - gpurun_out/ab_${TAG}_$v.jsonl <<'PY'
import json,sys,collections
acc=collections.defaultdict(list)
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: continue
    acc[d['config']].append((d['gkeys'], sum(d['pass_us'])/len(d['pass_us']), d['hist_us']))
for k,v in acc.items():
    print(f"{k:34s} " + "  ".join(f"{g:6.2f} GK/s pass {p:7.1f} hist {h:6.1f}" for g,p,h in v))
PY
done
