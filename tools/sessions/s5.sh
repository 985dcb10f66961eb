# look-back transient: per-tile trace at 2^24 and 2^28 (HEAD + OS_TRACE), look-back
# stats at 2^24 and 2^28, adaptive-window variants on C1/C2
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for n in 16777216 268435456; do
  ONESWEEP_B200_LIB=$V/headtrace.so timeout 300 python tools/trace_diag.py 1 $n > gpurun_out/trace_s5_$n.txt 2>&1
  for v in head w3x24; do ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/lookback_diag.py $n > gpurun_out/lbd_s5_${v}_$n.txt 2>&1; done
done
for v in head lam w3x24 w2x16 w4x32; do
  ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/quick_check.py > gpurun_out/qc_s5_$v.log 2>&1; echo "$v $(tail -1 gpurun_out/qc_s5_$v.log)" >> gpurun_out/qc_s5.txt
done
for r in 1 2; do
for v in head lam w3x24 w2x16 w4x32; do
  TAG=$v ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/size_sweep.py > gpurun_out/sizes_s5_${v}_$r.txt 2>&1
done
done
echo done
