"""Timing of the multi-kind engine variant (development tool): the bench's
config2-llm queue (100k apps over 256 depth-8 LLM / own-input / K3
templates), engine launch time by CUDA events, median of reps."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_14851_b200.estimator import DemandEngine  # noqa: E402
from paper_2506_14851_b200.graphs import graph_from_kb  # noqa: E402
from paper_2506_14851_b200.queue import HistQueue  # noqa: E402
from tools import synth  # noqa: E402

n_apps = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
docs = synth.llm_docs(256, 200, seed=2027)
eng = DemandEngine({k: graph_from_kb(v) for k, v in docs.items()})
q = synth.llm_queue(docs, n_apps, seed=9)
jobs = synth.llm_jobs(eng, q, eng.device)
hq = HistQueue(n_apps, bench.N_BINS)
ts = []
for i in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.run(*jobs, n=bench.N_SAMP, bucket_count=bench.N_BINS, visit_cap=bench.VISIT_CAP,
            queue=hq)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
c = hq.counts[:n_apps].to(torch.int64)
chk = int((c * torch.arange(c.shape[1], device=c.device)).sum().item())
print(json.dumps({"lib": os.environ.get("PDG_LIB_PATH", "in-tree"), "apps": n_apps,
                  "engine_ms": float(np.median(ts)), "checksum": chk}))
