#!/bin/bash
# Fast perf/parity iteration: engine-related GPU tests, then the bench (no extras).
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --no-extra --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
