#!/bin/bash
# K4b one-pass row writes vs zero-then-scatter; prewarm parity tests.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_prewarm_gpu.py tests/test_prewarm_wide_gpu.py -q > gpurun_out/pytest_j.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_j.txt
bash tools/need_sweep.sh "-DPDG_NEED_ONEPASS=0" "-DPDG_NEED_ONEPASS=1" "-DPDG_NEED_ONEPASS=1 -DPDG_NEED_STCS=0" \
  "-DPDG_NEED_ONEPASS=1 -DPDG_NEED_BATCH=4" "-DPDG_NEED_ONEPASS=0"
echo all-done
