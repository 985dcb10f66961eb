#!/bin/bash
# ncu --set full (source + stall samples) of one C4 (u64 keys + u32 values)
# and one C3 q=1 (u32 pairs) binning pass, for the per-phase reading of the
# latency-bound key-value kernels.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for spec in "c4:C4 uint64" "c3:C3 u32 pairs q=1"; do
  tag=${spec%%:*}; only=${spec#*:}
  timeout 900 $NCU -k regex:binning -s 3 -c 1 -f -o gpurun_out/prof_$tag \
    python tools/bench_configs.py --steps 1 --warmup 1 --only "$only" > gpurun_out/ncu_$tag.log 2>&1
  f=gpurun_out/prof_$tag.ncu-rep
  if [ -f $f ]; then
    ncu -i $f --page raw --csv > gpurun_out/ncuraw_$tag.csv 2>/dev/null
    ncu -i $f --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncusass_$tag.csv.gz
  fi
done
rm -f gpurun_out/*.ncu-rep; ls -la gpurun_out; tail -5 gpurun_out/ncu_c4.log
echo done
