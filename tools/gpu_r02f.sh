#!/bin/bash
# One-kernel K5b, K1b defaults: full GPU suite, K1b variants, bench, ncu captures.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_f.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_f.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_f.txt
bash tools/k1_sweep.sh "-DPDG_PAIR_WARPS=8 -DPDG_PAIR_STAGES=1 -DPDG_PAIR_MINB=3" \
  "-DPDG_PAIR_WARPS=2 -DPDG_PAIR_STAGES=1 -DPDG_PAIR_MINB=12" \
  "-DPDG_PAIR_WARPS=4 -DPDG_PAIR_STAGES=1 -DPDG_PAIR_MINB=6"
timeout 300 python tools/order_bench.py 100000 1000000 > gpurun_out/order_f.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gittins_pair" \
  -s 3 -c 1 -o gpurun_out/k1 -f python -c "
import torch, bench
bench.bench_k1_large(torch.device('cuda', 0), reps=2)" > gpurun_out/ncu_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk" \
  -s 3 -c 1 -o gpurun_out/engine -f python bench.py --steps 1 --warmup 3 --ncu --no-extra \
  > gpurun_out/ncu_engine.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
echo all-done
