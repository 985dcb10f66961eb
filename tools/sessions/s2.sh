cd $GRAFT_REPO_ROOT
for v in base new; do ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python tools/lookback_diag.py > gpurun_out/lbd_s2_$v.txt 2>&1; done
bash tools/gpu_ab.sh s2 3 base new noearly nosolo
bash tools/gpu_cfg_variants.sh s2c "C1,C3 u32 pairs q=1,C3 u32 pairs q=16,C4 uint64" base new ahead > gpurun_out/cfgv_s2_summary.txt 2>&1
