# count phase keeps the per-warp counts in registers
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
ONESWEEP_B200_LIB=$V/keep.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_skip.py -x -q 2>&1 | tail -1
bash tools/gpu_ab.sh s28 4 head keep
bash tools/gpu_cfg_variants.sh s28c "C1,C3 u32 pairs q=1,C4 uint64" head keep > gpurun_out/cfgv_s28_summary.txt 2>&1
grep -v product gpurun_out/cfgv_s28_summary.txt
