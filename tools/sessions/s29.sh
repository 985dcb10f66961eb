# count phase on digit pairs
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
ONESWEEP_B200_LIB=$V/cpairs.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_skip.py tests/test_gpu_value_widths.py tests/test_gpu_distributed.py tests/test_gpu_rts.py -x -q 2>&1 | tail -1
bash tools/gpu_ab.sh s29 4 head cpairs
bash tools/gpu_cfg_variants.sh s29c "C1,C3 u32 pairs q=1,C3 u32 pairs q=16,C4 uint64" head cpairs > gpurun_out/cfgv_s29_summary.txt 2>&1
grep -v product gpurun_out/cfgv_s29_summary.txt
cat gpurun_out/summary_s29.txt
