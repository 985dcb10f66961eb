# C1 with persistent keys-only blocks; ncu source captures of the C3 and C4 binning passes
cd $GRAFT_REPO_ROOT
bash tools/gpu_cfg_variants.sh s3c "C1,C2" base pkeys > gpurun_out/cfgv_s3_summary.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
for c in "C3 u32 pairs q=1:5:c3" "C4 uint64:9:c4"; do
  IFS=: read name skip tag <<< "$c"
  timeout 900 $NCU -k regex:binning -s $skip -c 1 -f -o gpurun_out/prof_$tag \
    python tools/bench_configs.py --steps 1 --warmup 1 --only "$name" > gpurun_out/ncu_$tag.log 2>&1
  f=gpurun_out/prof_$tag.ncu-rep
  if [ -f $f ]; then
    ncu -i $f --page raw --csv > gpurun_out/ncuraw_$tag.csv 2>/dev/null
    ncu -i $f --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncusass_$tag.csv.gz
    rm -f $f
  fi
done
echo done
