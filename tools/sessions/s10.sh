# (key, value) pair STS.64 reorder for u32 pairs (C3)
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for v in pair; do ONESWEEP_B200_LIB=$V/$v.so timeout 300 python tools/quick_check.py > gpurun_out/qc_s10_$v.log 2>&1; tail -1 gpurun_out/qc_s10_$v.log; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide_values.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
bash tools/gpu_cfg_variants.sh s10c "C3" nopair pair > gpurun_out/cfgv_s10_summary.txt 2>&1
cat gpurun_out/cfgv_s10_summary.txt
