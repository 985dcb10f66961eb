# per-tile traces at 2^24 / 2^28 (graph replay off); C3/C4 geometry variants
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for n in 16777216 268435456; do
  ONESWEEP_B200_LIB=$V/headtrace.so timeout 300 python tools/trace_diag.py 1 $n > gpurun_out/trace_s6_$n.txt 2>&1
done
for v in c3a c3b c4a c4b; do
  ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/quick_check.py > gpurun_out/qc_s6_$v.log 2>&1; echo "$v $(tail -1 gpurun_out/qc_s6_$v.log)" >> gpurun_out/qc_s6.txt
done
bash tools/gpu_cfg_variants.sh s6c "C3 u32 pairs q=1,C3 u32 pairs q=16,C4 uint64" head c3a c3b c4a c4b > gpurun_out/cfgv_s6_summary.txt 2>&1
echo done
