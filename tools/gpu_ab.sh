#!/bin/bash
# A/B session: fast GPU parity subset on the default lib, then bench +
# look-back diagnostics per variant.  usage: tools/gpu_ab.sh TAG variant...
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -q -x -p no:cacheprovider --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
for v in "$@"; do
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${TAG}_$v.json 2> gpurun_out/bench_${TAG}_$v.err
  ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python tools/lookback_diag.py >> gpurun_out/diag_$TAG.log 2>&1
done
python - "$TAG" <<'PY' > gpurun_out/summary_$TAG.txt
import glob, json, sys
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/bench_{tag}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d.get("kernels", {})
        print(f"{f.split('bench_'+tag+'_')[1][:-5]:12s} {d['value']:7.2f} GKey/s  passes {[round(x) for x in k.get('binning_pass_us', [])]}  hist {k.get('histogram_us', 0):.0f}us")
    except Exception as e:
        print(f, "ERR", e)
PY
cat gpurun_out/summary_$TAG.txt gpurun_out/diag_$TAG.log
# prefetch sweep on the default lib
for pf in 0 296; do
  ONESWEEP_B200_PREFETCH=$pf timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/pf_${TAG}_$pf.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('prefetch', sys.argv[2], round(d['value'],2), [round(x) for x in d['kernels']['binning_pass_us']])" gpurun_out/pf_${TAG}_$pf.json $pf
done
timeout 300 python tools/lookback_diag.py; ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/trace.so timeout 300 python tools/trace_diag.py 1
