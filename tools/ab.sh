#!/bin/bash
# A/B timing of the engine: ab_base/csrc (A) vs the working tree
# (B), interleaved twice.  Usage: bash tools/ab.sh ["-DFLAGS for B"]
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
: > gpurun_out/sweep.txt
for r in 1 2; do
  echo "-- A (base)" >> gpurun_out/sweep.txt
  SWEEP_APPEND=1 SWEEP_TAG=a$r SWEEP_SRC=ab_base/csrc bash tools/engine_sweep.sh ""
  echo "-- B (tree)" >> gpurun_out/sweep.txt
  SWEEP_APPEND=1 SWEEP_TAG=b$r bash tools/engine_sweep.sh "${1:-}"
done
