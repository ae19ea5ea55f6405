"""Development probe: does the engine's tail shrink if the queue is handed out
longest-first?  Times DemandEngine.run on the config-2 queue in its own order
and permuted by each application's expected remaining walk length (solved
from the synthetic graphs' successor tables), descending.

    python tools/lpt_probe.py [--apps 100000] [--reps 10]
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def expected_steps(w):
    """E[u] = 1 + sum_v P(u -> v) E[v] per application (successor tables)."""
    A, U = w["succ_len"].shape
    P = np.zeros((A, U, U))
    cum = w["succ_cum"]
    prev = np.concatenate([np.zeros((A, U, 1)), cum[:, :, :-1]], axis=2)
    p = cum - prev
    for s in range(w["succ_nxt"].shape[2]):
        v = w["succ_nxt"][:, :, s]
        ok = v >= 0
        a_i, u_i = np.nonzero(ok)
        P[a_i, u_i, v[ok]] += p[a_i, u_i, s]
    M = np.eye(U)[None] - P
    return np.linalg.solve(M, np.ones((A, U, 1)))[..., 0]


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
    E = expected_steps(w)[np.arange(n), jb["unit"]]
    q = HistQueue(n, 256)
    res = {"apps": n, "E_min": float(E.min()), "E_mean": float(E.mean()), "E_max": float(E.max())}
    orders = {"queue": np.arange(n), "lpt": np.argsort(-E, kind="stable"),
              "spt": np.argsort(E, kind="stable")}
    for name, o in list(orders.items()) + [("queue2", np.arange(n)), ("lpt2", orders["lpt"])]:
        g = torch.from_numpy(o.astype(np.int32)).to(dev)
        u = torch.from_numpy(jb["unit"][o]).to(dev)
        s = torch.from_numpy(jb["seed"][o]).to(dev)
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
        res[name + "_ms"] = sum(ts) / len(ts)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
