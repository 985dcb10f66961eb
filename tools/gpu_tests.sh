#!/bin/bash
# GPU test session: smoke, the whole -m gpu suite, compute-sanitizer runs.
# usage: tools/gpu_tests.sh TAG [nosan]
cd "$(dirname "$0")/.."
TAG=$1
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -15 gpurun_out/pytest_$TAG.log
if [ "$2" != "nosan" ]; then bash tools/gpu_sanitize.sh $TAG; fi
