#!/bin/bash
# Copy the reference's own test files into oracle/_ref/reference_tests/
# (git-ignored, travels to the GPU box) so tools/gpu_reference_suite.sh can
# run them against the drop-in.  Run here, where /root/reference exists.
cd "$(dirname "$0")/.."
REF=${REF:-/root/reference/pkg/tests}
mkdir -p oracle/_ref/reference_tests
cp "$REF"/test_*.py oracle/_ref/reference_tests/
ls oracle/_ref/reference_tests
