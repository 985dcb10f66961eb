# per-instruction comparison of the C2 pass: HEAD vs ticket routing
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for v in head route; do
  ONESWEEP_B200_LIB=$V/$v.so ncu --set full --import-source on --clock-control none -k regex:binning -s 4 -c 1 -f -o gpurun_out/prof_s22_$v \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
  ncu -i gpurun_out/prof_s22_$v.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncusass_s22_$v.csv.gz
  ncu -i gpurun_out/prof_s22_$v.ncu-rep --page raw --csv > gpurun_out/ncuraw_s22_$v.csv 2>/dev/null
  rm -f gpurun_out/prof_s22_$v.ncu-rep
done
