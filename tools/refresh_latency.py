"""Policy runtime of one batched refresh (the paper's "scheduling overhead",
sched.py:269-310 elapsed_ns) at config-1 sizes: our drop-in
refresh_priorities vs the reference's, same application objects."""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def apps(pdgsim, m, bins, rng):
    from pdgsim.estimator import RemainingDemand
    from pdgsim.sched import ApplicationInstance
    out = []
    for i in range(m):
        s = rng.lognormal(3, 1, 512).tolist()
        a = ApplicationInstance(f"a{i}", "g", float(i))
        a.set_remaining(RemainingDemand(samples=s, sample_count=512), bins)
        a.attained_service = float(rng.uniform(0, 1.2) * max(s))
        out.append(a)
    return out


def main():
    from tests.dispatch_hook import import_pdgsim
    pdgsim = import_pdgsim()
    from pdgsim import sched as ref
    from paper_2506_14851_b200 import sched as ours
    rng = np.random.default_rng(0)
    res = {}
    for m in (47, 1000):
        live = apps(pdgsim, m, 64 if m == 47 else 10, rng)
        for name, fn in (("reference", ref.refresh_priorities), ("ours", ours.refresh_priorities)):
            for _ in range(20):
                fn(live, 0.0, 1.0, force=True)
            ts = [fn(live, 0.0, 1.0, force=True).elapsed_ns for _ in range(500)]
            res[f"{name}_apps{m}_p50_us"] = float(np.median(ts)) / 1e3
    print(json.dumps(res))


if __name__ == "__main__":
    main()
