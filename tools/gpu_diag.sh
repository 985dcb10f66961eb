#!/bin/bash
# Diagnostic session: smoke, bench, one ncu --set full capture of the C2
# binning pass (raw + per-SASS source page with stall samples), then an A/B
# of library variants.  usage: tools/gpu_diag.sh TAG REPS variant...
cd "$(dirname "$0")/.."
TAG=$1; REPS=$2; shift 2
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:binning -s 4 -c 1 -f -o gpurun_out/prof_binning_$TAG \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_bin_$TAG.log 2>&1
f=gpurun_out/prof_binning_$TAG.ncu-rep
if [ -f $f ]; then
  ncu -i $f --page raw --csv > gpurun_out/ncuraw_binning_$TAG.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncusass_binning_$TAG.csv.gz
  ncu -i $f --page details --csv > gpurun_out/ncudetails_binning_$TAG.csv 2>/dev/null
fi
[ $# -gt 0 ] && bash tools/gpu_ab.sh $TAG $REPS "$@"
echo done
