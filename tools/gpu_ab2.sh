#!/bin/bash
# A/B session: per variant a quick correctness check, then bench (20 steps).
# usage: tools/gpu_ab2.sh TAG variant...   ("default" = the in-tree library)
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then LIB=""; else LIB="ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so"; fi
  env $LIB timeout 300 python tools/quick_check.py > gpurun_out/qc_${TAG}_$v.log 2>&1
  env $LIB timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${TAG}_$v.json 2> gpurun_out/bench_${TAG}_$v.err
done
python - "$TAG" "$@" <<'PY' > gpurun_out/summary_$TAG.txt
import json, sys
tag = sys.argv[1]
for v in sys.argv[2:]:
    qc = open(f"gpurun_out/qc_{tag}_{v}.log").read()
    qc = "PASS" if "QUICK_CHECK PASS" in qc else "FAIL"
    try:
        d = json.loads(open(f"gpurun_out/bench_{tag}_{v}.json").read().strip().splitlines()[-1])
        k = d.get("kernels", {})
        print(f"{v:14s} {qc} {d['value']:7.2f} GKey/s  passes {[round(x) for x in k.get('binning_pass_us', [])]}  hist {k.get('histogram_us', 0):.0f}us")
    except Exception as e:
        print(f"{v:14s} {qc} bench ERR {e}")
PY
cat gpurun_out/summary_$TAG.txt
