# isolate the routing overhead: HEAD, routed, same library with routing off
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for r in 1 2 3; do
  for v in head route noskip; do
    lib=$V/$v.so; env=""
    [ $v = noskip ] && lib=$V/route.so && env="ONESWEEP_B200_NO_SKIP=1"
    env $env ONESWEEP_B200_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b24_${v}_$r.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, statistics
for v in ("head", "route", "noskip"):
    p = []
    for f in sorted(glob.glob(f"gpurun_out/b24_{v}_*.json")):
        d = json.loads(open(f).read().strip().splitlines()[-1]); p += d["kernels"]["binning_pass_us"]
    print(v, round(statistics.median(p), 1), round(min(p), 1))
PY
