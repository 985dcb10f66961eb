# pass skipping with the vectorised copy: structured inputs, fixed vs routed
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_skip.py -x -q 2>&1 | tail -1
ONESWEEP_B200_NO_SKIP=1 timeout 600 python tools/skip_probe.py
timeout 600 python tools/skip_probe.py
