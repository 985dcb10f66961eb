# L2 prefetch distance for the key-value passes (C3 q=1, C4)
cd $GRAFT_REPO_ROOT
for pf in 296 0 150 600 1200; do
  ONESWEEP_B200_PREFETCH=$pf timeout 600 python tools/bench_configs.py --steps 5 --only "C3 u32 pairs q=1,C4 uint64" > gpurun_out/pf_s8_$pf.jsonl 2>&1
done
for pf in 296 0 150 600 1200; do python -c "
import json
for l in open('gpurun_out/pf_s8_$pf.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print('pf=$pf', f\"{d['config']:32s} {d['gkeys']:6.2f} GKey/s pass {sum(d['pass_us'])/len(d['pass_us']):7.1f} us\")
"; done
