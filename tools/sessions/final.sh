# round-2 final evidence: the standard session plus value widths, pass skipping and the full GPU suite
cd $GRAFT_REPO_ROOT
TAG=${1:-r2g}
bash tools/gpu_round2.sh $TAG > gpurun_out/session_$TAG.log 2>&1
timeout 600 python tools/value_widths.py > gpurun_out/value_widths_$TAG.txt 2>&1
(ONESWEEP_B200_NO_SKIP=1 timeout 600 python tools/skip_probe.py; timeout 600 python tools/skip_probe.py) > gpurun_out/skip_probe_$TAG.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputests_$TAG.log 2>&1
tail -3 gpurun_out/gputests_$TAG.log; tail -12 gpurun_out/session_$TAG.log
