#!/bin/bash
# Stage the reference's own unit tests for the hot-path modules into baseline/_ref_tests
# (git-ignored, like the baseline/_ref install; it travels to the GPU box with gpurun).
# Run there:  PYTHONPATH=tests/dropin python -m pytest baseline/_ref_tests -q
set -e
cd "$(dirname "$0")/.."
mkdir -p baseline/_ref_tests
for f in test_compressor test_entropy test_rank_model test_controller; do
  cp /root/reference/pkg/tests/$f.py baseline/_ref_tests/
done
ls baseline/_ref_tests
