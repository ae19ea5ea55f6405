#!/bin/bash
# K1b quad kernel + engine micro-optimisations: parity tests, timings, ncu.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gittins_gpu.py tests/test_engine_gpu.py \
  tests/test_workload_gpu.py tests/test_policy_gpu.py tests/test_kb_refresh_gpu.py \
  tests/test_stream_gpu.py tests/test_integration_gpu.py tests/test_order_gpu.py tests/test_attained_gpu.py -q > gpurun_out/pytest_b.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_b.txt
timeout 300 python -c "
import json, torch, bench
d = torch.device('cuda', 0)
a = bench.bench_k1_large(d)
b = bench.bench_k1_large(d, n=100_000)
print(json.dumps({'1m': a, '100k': b}))
" > gpurun_out/k1.json 2>&1
bash tools/ab2.sh
for lib in /tmp/pdg_a.so /tmp/pdg_b.so; do PDG_LIB_PATH=$lib timeout 300 python tools/order_bench.py 100000 1000000 >> gpurun_out/order.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gittins_quad" \
  -s 3 -c 1 -o gpurun_out/k1q -f python -c "
import torch, bench
bench.bench_k1_large(torch.device('cuda', 0), reps=2)" > gpurun_out/ncu_k1q.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk" \
  -s 2 -c 1 -o gpurun_out/engine_llm -f python tools/llm_engine_run.py 100000 3 \
  > gpurun_out/ncu_engine_llm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk" \
  -s 3 -c 1 -o gpurun_out/engine_b -f python bench.py --steps 1 --warmup 3 --ncu --no-extra \
  > gpurun_out/ncu_engine_b.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
echo all-done
