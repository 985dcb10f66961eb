"""Per-source-line totals of an `ncu --page source --csv --print-source
cuda,sass` dump (the line rows carry the sums of their SASS rows):
instructions and shared wavefronts per item, stall share.
Usage: python tools/ncu_lines.py dump.csv [items] [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
items = float(sys.argv[2]) if len(sys.argv) > 2 else 268435456 / 32
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ix = {}
for i, h in enumerate(hdr):
    ix.setdefault(h, i)
lines = [r for r in rows[hi + 1:] if len(r) >= len(hdr) - 1 and r[0] not in ("", "-")]


def f(r, k):
    try:
        return float(r[ix[k]] or 0)
    except (ValueError, KeyError):
        return 0.0


I, W, S = "Instructions Executed", "L1 Wavefronts Shared", "Warp Stall Sampling (All Samples)"
ti = sum(f(r, I) for r in lines)
tw = sum(f(r, W) for r in lines)
ts = sum(f(r, S) for r in lines)
print(f"instr/item {ti / items:.2f}  shared wf/item {tw / items:.2f}")
for r in sorted(lines, key=lambda r: -f(r, I))[:top]:
    print(f"{r[0]:>5} instr {f(r, I) / items:6.2f} wf {f(r, W) / items:5.2f} stall {f(r, S) / ts * 100:5.1f}%  {r[1].strip()[:90]}")
