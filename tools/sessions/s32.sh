# e2e: pipeline probe vs the bench's e2e leg on the same box
cd $GRAFT_REPO_ROOT
timeout 300 python tools/pipe_probe.py 2>&1 | tail -7
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench e2e', d['e2e']['ms_per_step'], 'sync', d['e2e']['synchronous']['ms_per_step'])"
timeout 300 python tools/pipe_probe.py 2>&1 | tail -7
nvidia-smi -q | grep -i -A3 "copy\|async\|pcie\|Link Width\|Link Gen" | head -40
