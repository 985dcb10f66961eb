# per-warp TMA slices in the keys-only kernel too (C2)
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
ONESWEEP_B200_LIB=$V/sall.so timeout 300 python tools/quick_check.py > gpurun_out/qc_s12.log 2>&1; tail -1 gpurun_out/qc_s12.log
bash tools/gpu_ab.sh s12 3 base sall
for v in base sall; do TAG=$v ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/size_sweep.py; done
