#!/bin/bash
# A/B session on the GPU box: for each library variant (built here with
# tools/build_variants.sh), a fast correctness check (tools/quick_check.py)
# and the C2 bench (live CUDA events), interleaved over REPS rounds so box
# drift hits every variant alike.  usage: tools/gpu_ab.sh TAG REPS variant...
cd "$(dirname "$0")/.."
TAG=$1; REPS=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python tools/quick_check.py > gpurun_out/qc_${TAG}_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/qc_${TAG}_$v.log)"
done
for r in $(seq 1 $REPS); do
  for v in "$@"; do
    ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${TAG}_${v}_$r.json 2> gpurun_out/bench_${TAG}_${v}_$r.err
  done
done
python - "$TAG" "$@" <<'PY' | tee gpurun_out/summary_$TAG.txt
import glob, json, sys, statistics
tag = sys.argv[1]
for v in sys.argv[2:]:
    vals, passes, hist = [], [], []
    for f in sorted(glob.glob(f"gpurun_out/bench_{tag}_{v}_*.json")):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            vals.append(d["value"]); passes += d["kernels"]["binning_pass_us"]; hist.append(d["kernels"]["histogram_us"])
        except Exception as e:
            print(v, f, "ERR", e)
    if vals:
        print(f"{v:14s} {statistics.median(vals):7.2f} GKey/s  pass {statistics.median(passes):6.1f} us (min {min(passes):6.1f})  hist {statistics.median(hist):5.1f} us  n={len(vals)}")
PY
