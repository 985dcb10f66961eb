# L2 residency between passes at small n: write-back stores, TMA without evict_first
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for r in 1 2; do for v in base wb wbn; do
  TAG=$v ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/size_sweep.py > gpurun_out/sizes_s9_${v}_$r.txt 2>&1
done; done
for v in base wb wbn; do paste gpurun_out/sizes_s9_${v}_1.txt gpurun_out/sizes_s9_${v}_2.txt | awk '{print $1, $2, $5, $10}'; done
