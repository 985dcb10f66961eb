"""Annotated SASS listing of one kernel from an `ncu --page source --csv
--print-source sass` dump (gzip), per-instruction: share of warp-stall
samples, dominant stall reason, executions and shared wavefronts per 32-key
item.  usage: python tools/ncu_regions.py dump.csv.gz N_KEYS > listing.txt"""
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
items = int(sys.argv[2]) / 32
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = idx["Warp Stall Sampling (All Samples)"]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
tot = sum(float(r[S] or 0) for r in data)
for r in data:
    ex = float(r[idx["Instructions Executed"]] or 0)
    wf = float(r[idx["L1 Wavefronts Shared"]] or 0)
    s = float(r[S] or 0)
    main = max(stall_cols, key=lambda h: float(r[idx[h]] or 0)) if s > 0 else ""
    print(f"{int(r[0], 16) - base:5x} {s / tot * 100:5.2f}% {main[6:]:12s} ex/it={ex / items:.3f} "
          f"wf/it={wf / items:.2f} {r[1].strip()[:90]}")
