# keys-only u32 tile size vs n (small-n wave quantisation)
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for v in head i32 i24 i48; do
  echo "$v $(ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/quick_check.py 2>&1 | tail -1)"
done
for r in 1 2; do
  for v in head i32 i24 i48; do
    ONESWEEP_B200_LIB=$V/$v.so TAG=$v timeout 300 python tools/size_sweep.py 2>&1 | tail -7
  done
done
