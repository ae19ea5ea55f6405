"""Per-core speed of the unmodified reference (pdgsim from baseline/_ref, or
/root/reference/pkg/src here) against the oracle port that bench.py's CPU legs
time, on the same config-2 apps: MC(n=512) + set_remaining's bucketing (256)
+ one Gittins row each.  Prints one JSON line.

    python tools/ref_vs_port.py [apps]
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "pdgsim")):
        sys.path.insert(0, cand)
        break


def main():
    from pdgsim import distributions, estimator, pdgraph, sched

    from oracle import pdg_oracle as O
    from tools import synth
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    w = synth.make(n, 256, seed=1000)
    jb = synth.jobs(n, seed=1001)
    docs, rg, keep = [], [], []
    for a in range(n):                 # the reference rejects graphs with unreachable units
        d = synth.kb_doc(w, a)
        try:
            rg.append(pdgraph.graph_from_dict(d))
        except Exception:
            continue
        docs.append(d)
        keep.append(a)
    og = [O.graph_from_kb(d) for d in docs]
    jb = {k: v[keep] for k, v in jb.items()}
    n = len(keep)
    env = pdgraph.RateProfile() if hasattr(pdgraph, "RateProfile") else None

    t0 = time.perf_counter()
    ref_keys = []
    for a in range(n):
        r = estimator.monte_carlo_remaining_demand(rg[a], f"s{jb['unit'][a]}", [], env, 512,
                                                   int(jb["seed"][a]), 64)
        d = distributions.EmpiricalDistribution(r.samples, capacity=max(len(r.samples), 1),
                                                bucket_count=256)
        vals, probs = d.bucket_points()
        ref_keys.append(sched.gittins_rank_batch(np.asarray(vals)[None] + 10.0,
                                                 np.asarray(probs)[None], np.array([20.0]))[0])
    t_ref = time.perf_counter() - t0

    t0 = time.perf_counter()
    port_keys = []
    for a in range(n):
        r = O.mc_remaining_demand(og[a], f"s{jb['unit'][a]}", [], 512, int(jb["seed"][a]), 64)
        b = O.bucketize(r.samples.tolist(), 256)
        port_keys.append(O.gittins_rank_batch((b.midpoints() + 10.0)[None], b.probs[None],
                                              np.array([20.0]))[0])
    t_port = time.perf_counter() - t0
    same = bool(np.array_equal(np.asarray(ref_keys), np.asarray(port_keys), equal_nan=True))
    print(json.dumps({"apps": n, "reference_apps_per_s_per_core": n / t_ref,
                      "port_apps_per_s_per_core": n / t_port, "port_over_reference": t_ref / t_port,
                      "keys_identical": same,
                      "reference_from": sys.path[0]}))


if __name__ == "__main__":
    main()
