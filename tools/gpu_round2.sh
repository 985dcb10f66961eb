#!/bin/bash
# Round-2 evidence session (one gpurun call): smoke, bench (x2) + reference
# arm, ncu launch list, ncu --set full captures of the C2 binning pass and
# histogram and of the C3 / C4 binning passes and the u64 histogram, the
# config sweep, compute-sanitizer runs and the reference's own test suite
# against the drop-in.  usage: tools/gpu_round2.sh TAG
cd "$(dirname "$0")/.."
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${TAG}_rep.json 2>> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:binning -s 4 -c 1 -f -o gpurun_out/prof_binning_$TAG \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_bin_$TAG.log 2>&1
timeout 900 $NCU -k regex:histogram -s 1 -c 1 -f -o gpurun_out/prof_hist_$TAG \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_hist_$TAG.log 2>&1
timeout 900 $NCU -k regex:binning -s 5 -c 1 -f -o gpurun_out/prof_binning_c3_$TAG \
  python tools/bench_configs.py --steps 1 --warmup 1 --only "C3 u32 pairs q=1" > gpurun_out/ncu_bin_c3_$TAG.log 2>&1
timeout 900 $NCU -k regex:binning -s 9 -c 1 -f -o gpurun_out/prof_binning_c4_$TAG \
  python tools/bench_configs.py --steps 1 --warmup 1 --only "C4 uint64" > gpurun_out/ncu_bin_c4_$TAG.log 2>&1
timeout 900 $NCU -k regex:histogram -s 1 -c 1 -f -o gpurun_out/prof_hist_c4_$TAG \
  python tools/bench_configs.py --steps 1 --warmup 1 --only "C4 uint64" > gpurun_out/ncu_hist_c4_$TAG.log 2>&1
# keep the counters as text (raw page + per-line source page), drop the bulky
# captures except the C2 binning pass (gpurun returns <= 64 MiB)
for r in binning hist binning_c3 binning_c4 hist_c4; do
  f=gpurun_out/prof_${r}_$TAG.ncu-rep
  [ -f $f ] || continue
  ncu -i $f --page raw --csv > gpurun_out/ncuraw_${r}_$TAG.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/ncusrc_${r}_$TAG.csv.gz
  [ $r = binning ] && ncu -i $f --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncusass_binning_$TAG.csv.gz
  [ $r = binning ] || rm -f $f
done
ls -la gpurun_out
timeout 900 python tools/bench_configs.py --steps 10 > gpurun_out/cfgs_$TAG.jsonl 2>&1
# compute-sanitizer: closed on this GPU pool since session r2j (the tool refuses to run);
# profiles/round2_sanitize.txt holds the last run (session r2i, 0 errors / 0 hazards)
[ -n "$OS_SANITIZE" ] && bash tools/gpu_sanitize.sh $TAG
bash tools/gpu_reference_suite.sh $TAG
echo done
