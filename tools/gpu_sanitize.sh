#!/bin/bash
# compute-sanitizer runs over tools/sanitize_cases.py (all kernels, small
# sizes).  usage: tools/gpu_sanitize.sh TAG [case...]
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  # (no --leak-check: the only leaks it reports are torch allocator blocks alive at exit)
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py "$@" \
    > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$? $(grep -c 'case ok' gpurun_out/sanitize_${tool}_$TAG.log) cases ok; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_$TAG.log | tail -1)"
done
