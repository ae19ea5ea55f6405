#!/bin/bash
# Engine A/B under ncu (instruction count, issue activity, stall mix) of
# ab_base/csrc (a) vs the working tree (b): one mc_walk launch each.
# Development tool; the numbers are profiler numbers, not timings.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
build() {
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -shared -cudart static -I include -o $2 $1/*.cu > $2.log 2>&1
}
build ab_base/csrc /tmp/pdg_a.so & build paper_2506_14851_b200/csrc /tmp/pdg_b.so & wait
: > gpurun_out/ncu_ab.txt
for v in a b; do
  PDG_LIB_PATH=/tmp/pdg_$v.so timeout 600 ncu --clock-control none -k regex:mc_walk -s 2 -c 1 \
    --section SchedulerStats --section WarpStateStats --section Occupancy \
    --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio \
    --csv --page raw python tools/engine_bench.py --reps 3 > gpurun_out/ncu_ab_$v.csv 2>/dev/null
  echo "== $v" >> gpurun_out/ncu_ab.txt
done
python - <<'PY' >> gpurun_out/ncu_ab.txt
import csv
for v in "ab":
    rows = list(csv.reader(open(f"gpurun_out/ncu_ab_{v}.csv")))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h, d = rows[hdr], rows[hdr + 2]
    out = {}
    for k, x in zip(h, d):
        if any(t in k for t in ("inst_executed.sum", "time_duration", "issue_active", "per_inst_executed",
                                "warps_active.avg.pct", "pcsamp_warps_issue_stalled")):
            out[k] = x
    print(v, out)
PY
