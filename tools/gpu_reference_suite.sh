#!/bin/bash
# Run the reference's test suite (staged by tools/stage_reference_suite.sh)
# against the drop-in on the GPU box.  usage: tools/gpu_reference_suite.sh TAG
cd "$(dirname "$0")/.."
TAG=${1:-ref}
mkdir -p gpurun_out
PYTHONPATH=$PWD/tests/reference_suite timeout 1500 python -m pytest -p onesweep_alias oracle/_ref/reference_tests \
  -q -rfxX -p no:cacheprovider --timeout 600 -o addopts="" > gpurun_out/reference_suite_$TAG.log 2>&1
echo "reference suite rc=$?" >> gpurun_out/reference_suite_$TAG.log
tail -5 gpurun_out/reference_suite_$TAG.log
