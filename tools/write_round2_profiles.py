"""Turn one tools/gpu_round2.sh session into the committed evidence:
profiles/ncu_traffic.json (read by bench.py for roofline.traffic), the
bench lines, launch list, config sweep, reference-suite and sanitizer logs,
and profiles/round2_ncu_summary.md (per-kernel counters for C2 / C3 / C4 and
the shared-memory wavefront accounting of the C2 binning pass).
Usage: python tools/write_round2_profiles.py TAG"""
import collections
import csv
import gzip
import io
import json
import os
import shutil
import sys

tag = sys.argv[1]
G = "gpurun_out"
P = "profiles"


def raw(name):
    r = list(csv.reader(open(f"{G}/ncuraw_{name}_{tag}.csv")))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def num(v, u, k, default=0.0):
    try:
        x = float(v[k].replace(",", ""))
    except (KeyError, ValueError):
        return default
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e3, "us": 1, "usecond": 1,
             "msecond": 1e3, "nsecond": 1e-3}
    return x * scale.get(u.get(k, ""), 1)


KERNELS = {  # capture -> (label, keys, algorithmic bytes per launch)
    "binning": ("C2 binning pass (u32 keys-only)", 1 << 28, 2 * (1 << 28) * 4),
    "hist": ("C2 histogram (u32, 4 places)", 1 << 28, (1 << 28) * 4),
    "binning_c3": ("C3 binning pass (u32 keys + u32 values, q=1)", 1 << 28, 2 * (1 << 28) * 8),
    "binning_c4": ("C4 binning pass (u64 keys + u32 values)", 1 << 28, 2 * (1 << 28) * 12),
    "hist_c4": ("C4 histogram (u64, 8 places)", 1 << 28, (1 << 28) * 8),
}
try:
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
except FileNotFoundError:
    # the driver writes MEASURED_PEAKS.json per pod; without it, use the
    # measured peak an earlier bench line of this round recorded from it
    peak = json.loads(open(f"{P}/round2_bench.json").read())["roofline"]["peak"]
det = {}
for name, (label, n, alg) in KERNELS.items():
    try:
        v, u = raw(name)
    except FileNotFoundError:
        continue
    rd = num(v, u, "dram__bytes_read.sum")
    wr = num(v, u, "dram__bytes_write.sum")
    dur = num(v, u, "gpu__time_duration.sum")
    items = n / 32
    det[name] = {
        "label": label, "kernel": v.get("Kernel Name", "")[:120], "duration_us": dur,
        "algorithmic_bytes": alg, "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic": rd + wr,
        "gbs_alg": alg / dur / 1e3, "frac_of_measured_hbm": alg / dur / 1e3 / peak,
        "issue_active": num(v, u, "smsp__issue_active.avg.per_cycle_active"),
        "inst_per_item": num(v, u, "smsp__inst_executed.sum") / items,
        "smem_wf_per_item": num(v, u, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / items,
        "smem_conflicts_per_item": num(v, u, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") / items,
        "lsu_data_pipe_pct": num(v, u, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "l2_hit_pct": num(v, u, "lts__t_sector_hit_rate.pct"),
        "registers": v.get("launch__registers_per_thread", ""),
    }
traffic = {"binning": det["binning"]["traffic"], "histogram": det["hist"]["traffic"],
           "source": f"ncu --set full --clock-control none, one launch each (session {tag}; "
                     "profiles/round2_ncu_summary.md)", "detail": det}
json.dump(traffic, open(f"{P}/ncu_traffic.json", "w"), indent=1)

# shared-memory wavefronts of the C2 binning pass, by SASS opcode
# (the SASS-only source page: every instruction once; on the box:
#  ncu -i prof_binning_TAG.ncu-rep --page source --csv --print-source sass)
src = list(csv.reader(io.StringIO(gzip.open(f"{G}/ncusass_binning_{tag}.csv.gz", "rt").read())))
hdr = src[1]
ix = {h: i for i, h in enumerate(hdr)}
sass = [r for r in src[2:] if len(r) >= len(hdr) - 1]
W, I = "L1 Wavefronts Shared", "Instructions Executed"
by = collections.defaultdict(lambda: [0.0, 0.0])
for r in sass:
    t = r[ix["Source"]].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    if op.startswith(("LDS", "STS", "ATOMS")):
        by[op][0] += float(r[ix[I]] or 0)
        by[op][1] += float(r[ix[W]] or 0)
items = (1 << 28) / 32

rows = []
for name, d in det.items():
    rows.append(f"| {d['label']} | {d['duration_us']:.1f} | {d['algorithmic_bytes'] / 1e9:.3f} | "
                f"{d['traffic'] / 1e9:.3f} | {d['gbs_alg']:.0f} | **{d['frac_of_measured_hbm'] * 100:.1f} %** | "
                f"{d['inst_per_item']:.1f} | {d['issue_active'] * 100:.0f} % | {d['smem_wf_per_item']:.2f} | "
                f"{d['smem_conflicts_per_item']:.2f} | {d['lsu_data_pipe_pct']:.1f} % | {d['l2_hit_pct']:.1f} % | {d['registers']} |")
ops = "\n".join(f"| `{op}` | {e / items:.2f} | {w / items:.2f} | {w / max(e, 1):.2f} |"
                for op, (e, w) in sorted(by.items(), key=lambda x: -x[1][1]) if w / items >= 0.01)
b = json.loads(open(f"{G}/bench_{tag}.json").read().strip().splitlines()[-1])
md = f"""# Round 2 — ncu evidence (B200, sm_100a, clocks not locked)

Session `{tag}` (`tools/gpu_round2.sh`, one gpurun call), summarised by
`tools/write_round2_profiles.py`.  Per-kernel counters come from
`ncu --set full --clock-control none --import-source on`, one launch each.
Captures are cold-cache and serialised; compare shares, not absolute times,
with the bench.  "Item" = 32 keys (one warp instruction's worth).

Bench line of the same session (`profiles/round2_bench.json`): **{b['value']:.2f} GKey/s**,
{b['ms_per_step']:.3f} ms per 256M-key sort, binning pass {b['roofline']['launch_us']:.0f} us live
(= {2 * (1 << 28) * 4 / (b['roofline']['launch_us'] * 1e-6) / 1e9 / peak * 100:.1f} % of the measured {peak:.0f} GB/s), histogram
{b['kernels']['histogram_us']:.0f} us, e2e {b['e2e']['value']:.2f} GKey/s (PCIe-bound),
SM clock {b['clocks']['sm_mhz']:.0f} MHz, throttle reasons {b['clocks']['reasons']}.

## Per-kernel counters

| kernel | ncu µs | algorithmic GB | DRAM GB (r+w) | GB/s (alg.) | of measured HBM | instr / item | issue active | smem wavefronts / item | of which conflicts | L1 data pipe | L2 hit | regs |
|---|---|---|---|---|---|---|---|---|---|---|---|---|
{chr(10).join(rows)}

## C2 binning pass: shared-memory wavefronts by instruction (per 32-key item)

| SASS | executions / item | wavefronts / item | wavefronts / execution |
|---|---|---|---|
{ops}
"""
open(f"{P}/round2_ncu_summary.md", "w").write(md)
for s, d in [(f"bench_{tag}.json", "round2_bench.json"), (f"bench_{tag}_ref.json", "round2_bench_reference.json"),
             (f"launches_{tag}.csv", "round2_launches.csv"), (f"cfgs_{tag}.jsonl", "round2_configs.jsonl"),
             (f"reference_suite_{tag}.log", "round2_reference_suite.txt")]:
    if d == "round2_reference_suite.txt" and "rc=0" not in open(f"{G}/{s}").read() if os.path.exists(f"{G}/{s}") else False:
        print("reference suite did not pass in this session:", s, "(kept the committed file)")
        continue
    try:
        shutil.copy(f"{G}/{s}", f"{P}/{d}")
    except FileNotFoundError:
        print("missing", s)
san = {}
for tool in ("memcheck", "racecheck", "synccheck", "initcheck"):
    try:
        lines = open(f"{G}/sanitize_{tool}_{tag}.log").read().splitlines()
    except FileNotFoundError:
        continue
    keep = [ln for ln in lines if ln.startswith("case ok") or "SUMMARY" in ln or "SANITIZE" in ln]
    if any("SUMMARY" in ln for ln in keep):  # (a refused run, e.g. the pool closed the tool, keeps the last file)
        san[tool] = keep
if san:
    with open(f"{P}/round2_sanitize.txt", "w") as out:
        for tool, keep in san.items():
            out.write(f"== compute-sanitizer --tool {tool} python tools/sanitize_cases.py  (session {tag})\n" + "\n".join(keep) + "\n\n")
else:
    print("no sanitizer summaries in this session: profiles/round2_sanitize.txt kept")
print(open(f"{P}/round2_ncu_summary.md").read())
