# route-base table: tests, C2 three-way, configs
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_skip.py tests/test_gpu_parity.py tests/test_gpu_value_widths.py -x -q 2>&1 | tail -2
bash tools/sessions/s24.sh
bash tools/gpu_cfg_variants.sh s26c "C1,C3 u32 pairs q=1,C3 u32 pairs q=16,C3 u32 pairs all-equal,C4" head route > gpurun_out/cfgv_s26_summary.txt 2>&1
grep -v product gpurun_out/cfgv_s26_summary.txt | head -20
