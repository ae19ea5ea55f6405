"""Profiling target for the LLM engine variant (development tool): the
bench's config2-llm queue, engine launched `reps` times.  Usage under ncu:
  ncu -k regex:mc_walk -s 2 -c 1 python tools/llm_engine_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_14851_b200.estimator import DemandEngine  # noqa: E402
from paper_2506_14851_b200.graphs import graph_from_kb  # noqa: E402
from paper_2506_14851_b200.queue import HistQueue  # noqa: E402
from tools import synth  # noqa: E402

n_apps = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
docs = synth.llm_docs(256, 200, seed=2027)
eng = DemandEngine({k: graph_from_kb(v) for k, v in docs.items()})
q = synth.llm_queue(docs, n_apps, seed=9)
jobs = synth.llm_jobs(eng, q, eng.device)
hq = HistQueue(n_apps, bench.N_BINS)
for _ in range(reps):
    eng.run(*jobs, n=bench.N_SAMP, bucket_count=bench.N_BINS, visit_cap=bench.VISIT_CAP,
            queue=hq)
torch.cuda.synchronize()
print("ok")
