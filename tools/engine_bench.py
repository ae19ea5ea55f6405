"""Engine-only timing on the config-2 workload (development tool).

    python tools/engine_bench.py [--apps 100000] [--reps 10]

Prints one JSON line: average mc kernel time per launch (CUDA events) and
a checksum of the histogram rows (so variants can be compared for equality).
"""

import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.queue import HistQueue
    from tools import synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--apps", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = a.apps
    w = synth.make(n, 256, seed=1000)
    eng = DemandEngine(synth.bank(w, device=str(dev)), device=str(dev))
    jb = synth.jobs(n, seed=1001)
    q = HistQueue(n, 256)
    g = torch.arange(n, dtype=torch.int32, device=dev)
    u = torch.from_numpy(jb["unit"]).to(dev)
    s = torch.from_numpy(jb["seed"]).to(dev)
    for _ in range(2):
        eng.run(g, u, s, n=512, bucket_count=256, visit_cap=64, queue=q)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.run(g, u, s, n=512, bucket_count=256, visit_cap=64, queue=q)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    h = hashlib.sha256(q.counts[:n].cpu().numpy().tobytes() + q.lo[:n].cpu().numpy().tobytes())
    print(json.dumps({"lib": os.environ.get("PDG_LIB_PATH", "default"), "ms": sum(ts) / len(ts),
                      "min_ms": min(ts), "sha": h.hexdigest()[:16]}))


if __name__ == "__main__":
    main()
