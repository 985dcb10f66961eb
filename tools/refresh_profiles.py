"""Refresh profiles/ncu_traffic.json (read by bench.py for roofline.traffic),
the launch list and the config sweep from one tools/gpu_full.sh session.
Usage: python tools/refresh_profiles.py TAG"""
import csv
import io
import json
import shutil
import subprocess
import sys

tag = sys.argv[1]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def nbytes(v, u):
    return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]


d = {}
for name in ("binning", "hist"):
    v, u = raw(f"gpurun_out/prof_{name}_{tag}.ncu-rep")
    rd = nbytes(v["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
    wr = nbytes(v["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    dur = float(v["gpu__time_duration.sum"]) * (1000 if u["gpu__time_duration.sum"] == "ms" else 1)
    d["histogram" if name == "hist" else name] = {
        "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic": rd + wr, "duration_us": dur,
        "issue_active": float(v["smsp__issue_active.avg.per_cycle_active"]),
        "inst_executed": float(v["smsp__inst_executed.sum"]),
        "smem_wavefronts": float(v["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]),
        "smem_bank_conflicts": float(v["l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]),
        "lsu_data_pipe_pct": float(v.get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 0) or 0),
        "l2_hit_pct": float(v["lts__t_sector_hit_rate.pct"]),
        "registers": v["launch__registers_per_thread"],
    }
out = {"binning": d["binning"]["traffic"], "histogram": d["histogram"]["traffic"],
       "source": f"ncu --set full --clock-control none, one launch each (session {tag}; "
                 "profiles/round1_ncu_summary.md)", "detail": d}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
shutil.copy(f"gpurun_out/launches_{tag}.csv", "profiles/round1_launches.csv")
shutil.copy(f"gpurun_out/cfgs_{tag}.jsonl", "profiles/round1_configs.jsonl")
shutil.copy(f"gpurun_out/bench_{tag}.json", "profiles/round1_bench.json")
print(json.dumps(d, indent=1))
