#!/bin/bash
# L2 hit rate of the look-back status words: they are the only accesses with an
# evict_last policy, so the evict_last hit/miss sector counters isolate them.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-st}
# needs a build with -DOS_STATUS_KEEP=1 (LIB below); usage: tools/gpu_status_l2.sh TAG
LIB=$PWD/paper_2206_01784_b200/_lib/variants/keep.so
ONESWEEP_B200_LIB=$LIB timeout 900 ncu --metrics lts__t_sectors_srcunit_tex_evict_last_lookup_hit.sum,lts__t_sectors_srcunit_tex_evict_last_lookup_miss.sum,lts__t_sectors_evict_last_lookup_hit.sum,lts__t_sectors_evict_last_lookup_miss.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:binning -s 4 -c 4 --csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/status_l2_$TAG.csv 2> gpurun_out/status_l2_$TAG.err
grep -E "evict_last|hit_rate|duration" gpurun_out/status_l2_$TAG.csv | awk -F'","' '{print $(NF-2), $(NF)}' | head -24
