# digit-pair count phase for 8192 x 8-byte tiles (C4, u64 keys-only)
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
ONESWEEP_B200_LIB=$V/wp.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_value_widths.py tests/test_gpu_skip.py -x -q 2>&1 | tail -1
bash tools/gpu_cfg_variants.sh s30c "C4" head wp > gpurun_out/cfgv_s30_summary.txt 2>&1
grep -v product gpurun_out/cfgv_s30_summary.txt
for v in head wp; do echo "== $v"; ONESWEEP_B200_LIB=$V/$v.so timeout 600 python tools/value_widths.py 2>&1 | grep "u64"; done
