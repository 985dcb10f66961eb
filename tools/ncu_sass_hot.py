"""Summarise an `ncu --page source --csv --print-source sass` dump: top stall
instructions and per-region totals.  Usage: python tools/ncu_sass_hot.py dump.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = idx["Warp Stall Sampling (All Samples)"]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[S] or 0) for r in data)
print(f"total samples {tot:.0f}")
agg = {h: sum(float(r[idx[h]] or 0) for r in data) for h in stall_cols}
for h, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"  {h:28s} {v / tot * 100:5.1f}%")
print()
ranked = sorted(data, key=lambda r: -float(r[S] or 0))[:top]
for r in ranked:
    s = float(r[S] or 0)
    main = max(stall_cols, key=lambda h: float(r[idx[h]] or 0))
    print(f"{r[0]:>6} {s / tot * 100:5.1f}% {main[6:]:12s} ex={r[idx['Instructions Executed']]:>9} wf={r[idx['L1 Wavefronts Shared']]:>9}  {r[1][:70]}")
