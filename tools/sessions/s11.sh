# per-warp TMA key slices in the looping key-value kernels (C3, C4)
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
ONESWEEP_B200_LIB=$V/slice.so timeout 300 python tools/quick_check.py > gpurun_out/qc_s11.log 2>&1; tail -1 gpurun_out/qc_s11.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide_values.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
bash tools/gpu_cfg_variants.sh s11c "C3 u32 pairs q=1,C3 u32 pairs q=16,C4" noslice slice > gpurun_out/cfgv_s11_summary.txt 2>&1
cat gpurun_out/cfgv_s11_summary.txt
