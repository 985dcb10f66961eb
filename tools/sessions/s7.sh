# persistent keys-only blocks with a start stagger per SM slot; key-value stagger
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for v in pk0 pk2 pk35 st35; do
  ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/quick_check.py > gpurun_out/qc_s7_$v.log 2>&1; echo "$v $(tail -1 gpurun_out/qc_s7_$v.log)" >> gpurun_out/qc_s7.txt
done
for v in pk0t pk35t; do ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/trace_diag.py 1 > gpurun_out/trace_s7_$v.txt 2>&1; done
bash tools/gpu_ab.sh s7 3 head pk0 pk2 pk35
bash tools/gpu_cfg_variants.sh s7c "C1,C3 u32 pairs q=1,C4 uint64" head pk35 st35 > gpurun_out/cfgv_s7_summary.txt 2>&1
echo done
