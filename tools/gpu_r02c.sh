#!/bin/bash
# Full GPU suite, engine A/B (duration + LLM variants), bench, sanitizer reruns.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_c.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_c.txt
AB_ROUNDS=2 bash tools/ab2.sh
for lib in /tmp/pdg_a.so /tmp/pdg_b.so; do PDG_LIB_PATH=$lib timeout 300 python tools/llm_time.py >> gpurun_out/llm_time.txt 2>&1; done
timeout 900 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk" \
  -s 3 -c 1 -o gpurun_out/engine_c -f python bench.py --steps 1 --warmup 3 --ncu --no-extra \
  > gpurun_out/ncu_engine_c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk" \
  -s 2 -c 1 -o gpurun_out/engine_llm_c -f python tools/llm_engine_run.py 100000 3 \
  > gpurun_out/ncu_engine_llm_c.log 2>&1
mkdir -p gpurun_out/sanitizer
TOOLS=racecheck SAN_TIMEOUT=600 TESTS_OVERRIDE="tests/test_engine_gpu.py::test_golden_mc_cases_bit_exact tests/test_engine_gpu.py::test_understated_bank_features_stay_exact tests/test_engine_gpu.py::test_lemire_rejection_replayed_exactly tests/test_engine_gpu.py::test_wide_graph_32_units_many_successors tests/test_engine_gpu.py::test_histogram_rows_match_set_remaining tests/test_workload_gpu.py::test_synth_sample_bit_exact tests/test_policy_gpu.py tests/test_gittins_gpu.py::test_hist_queue_quad_path_vs_oracle tests/test_order_gpu.py tests/test_engine_gpu.py::test_wide_graph_64bit_unit_sets" bash tools/sanitize.sh
mv gpurun_out/sanitizer/racecheck.log gpurun_out/sanitizer/racecheck_c.log
TOOLS=initcheck KNS= SAN_TIMEOUT=600 TESTS_OVERRIDE="tests/test_engine_gpu.py::test_golden_mc_cases_bit_exact tests/test_gittins_gpu.py::test_hist_queue_vs_oracle tests/test_prewarm_gpu.py::test_need_grid_vs_oracle tests/test_dispatch_gpu.py::test_plan_random_tables_vs_oracle" bash tools/sanitize.sh
mv gpurun_out/sanitizer/initcheck.log gpurun_out/sanitizer/initcheck_c.log
echo all-done
