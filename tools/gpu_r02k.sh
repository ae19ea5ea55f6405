#!/bin/bash
# Scan-with-predicate + lean pool pointer: engine A/B, tests, bench (pipelined e2e).
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_k.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_k.txt
AB_ROUNDS=2 bash tools/ab2.sh
timeout 900 python bench.py > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err
echo all-done
