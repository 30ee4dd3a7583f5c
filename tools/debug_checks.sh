#!/bin/bash
# Bounds-checked build of libubqp (UBQP_DEBUG_CHECKS: device-side traps on out-of-range indices)
# and the GPU parity suites against it -- the stand-in for compute-sanitizer, which is closed on
# the GPU pool.  Usage (on a GPU box): tools/debug_checks.sh [pytest -k expression]
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
UBQP_NVCC_EXTRA="-DUBQP_DEBUG_CHECKS=1" python tools/build_variant.py variants/debug_checks.so
UBQP_LIB=variants/debug_checks.so python -m pytest tests -m gpu -x -q ${1:+-k "$1"} \
    --deselect tests/test_gpu_c_abi.py
