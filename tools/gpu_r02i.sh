#!/bin/bash
# careful pass = full variant: full GPU suite, smoke, LLM timing, bench.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_i.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_i.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_i.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_i.txt
timeout 300 python tools/llm_time.py > gpurun_out/llm_time_i.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
echo all-done
