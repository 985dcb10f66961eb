# ticket-encoded pass routing: tests, C2 A/B, configs, structured inputs
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_skip.py tests/test_gpu_parity.py tests/test_gpu_value_widths.py -x -q 2>&1 | tail -2
bash tools/gpu_ab.sh s23 3 head route
bash tools/gpu_cfg_variants.sh s23c "C1,C3 u32 pairs q=1,C3 u32 pairs all-equal,C4" head route > gpurun_out/cfgv_s23_summary.txt 2>&1
cat gpurun_out/cfgv_s23_summary.txt
ONESWEEP_B200_NO_SKIP=1 timeout 600 python tools/skip_probe.py
timeout 600 python tools/skip_probe.py
