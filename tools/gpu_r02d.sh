#!/bin/bash
# K1b pair kernel: parity, timings (in-tree build + -D variants), ncu at 1M rows.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gittins_gpu.py tests/test_stream_gpu.py \
  tests/test_workload_gpu.py tests/test_integration_gpu.py -q > gpurun_out/pytest_d.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_d.txt
timeout 300 python -c "
import json, torch, bench
d = torch.device('cuda', 0)
a = bench.bench_k1_large(d)
b = bench.bench_k1_large(d, n=100_000)
print(json.dumps({'1m': a, '100k': b}))
" > gpurun_out/k1_d.json 2>&1
bash tools/k1_sweep.sh "-DPDG_PAIR_WARPS=4 -DPDG_PAIR_STAGES=2 -DPDG_PAIR_MINB=3" \
  "-DPDG_PAIR_WARPS=2 -DPDG_PAIR_STAGES=3 -DPDG_PAIR_MINB=4" \
  "-DPDG_PAIR_WARPS=4 -DPDG_PAIR_STAGES=1 -DPDG_PAIR_MINB=4" \
  "-DPDG_PAIR_WARPS=8 -DPDG_PAIR_STAGES=2 -DPDG_PAIR_MINB=1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gittins_pair" \
  -s 3 -c 1 -o gpurun_out/k1p -f python -c "
import torch, bench
bench.bench_k1_large(torch.device('cuda', 0), reps=2)" > gpurun_out/ncu_k1p.log 2>&1
echo all-done
