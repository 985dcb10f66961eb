"""Top shared-memory instructions of an `ncu --page source --csv --print-source
sass` dump by L1 shared wavefronts, with executions and conflict ratio; and
instruction totals by opcode.  Usage: python tools/ncu_smem_top.py dump.csv [N] [items]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
items = float(sys.argv[3]) if len(sys.argv) > 3 else 268435456 / 32
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def f(r, k):
    try:
        return float(r[ix[k]] or 0)
    except ValueError:
        return 0.0


W, I, S = "L1 Wavefronts Shared", "Instructions Executed", "Warp Stall Sampling (All Samples)"
tw = sum(f(r, W) for r in data)
ti = sum(f(r, I) for r in data)
ts = sum(f(r, S) for r in data)
print(f"shared wavefronts {tw:.0f} ({tw / items:.2f}/item)   instructions {ti:.0f} ({ti / items:.2f}/item)")
ops = collections.Counter()
opw = collections.Counter()
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    ops[op] += f(r, I)
    opw[op] += f(r, W)
print("by opcode (instr/item, wf/item):")
for op, v in ops.most_common(25):
    print(f"  {op:10s} {v / items:6.2f}  {opw[op] / items:6.2f}")
print(f"top {top} shared instructions:")
for r in sorted(data, key=lambda r: -f(r, W))[:top]:
    ex = f(r, I)
    w = f(r, W)
    print(f"{r[0]:>6} wf/item={w / items:5.2f} wf/exec={w / max(ex, 1):4.2f} exec/item={ex / items:5.2f} "
          f"stall={f(r, S) / max(ts, 1) * 100:4.1f}%  {r[ix['Source']][:60]}")
