"""BASELINE config 1 end to end: the reference simulator's wall time with its
own hot path, and with the hot path swapped to the GPU drop-in
(integration.patch_pdgsim); also the per-call latency of the Monte Carlo
drop-in against the reference's on the simulation's own calls.  Prints one
JSON line.  Needs pdgsim in baseline/_ref (or /root/reference here)."""

import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "pdgsim")):
        sys.path.insert(0, cand)
        break


def measure() -> dict:
    import pdgsim
    from pdgsim import simcore
    from pdgsim.prewarm import CachePolicy
    from pdgsim.sched import Policy
    from pdgsim.workload import archetype, generate

    from paper_2506_14851_b200 import integration
    code_gen = archetype("code-check", {"trials": 200, "bucket_count": 64, "scale": 0.6,
                                        "app_id": "code-gen"}, seed=3)
    fact = archetype("verify-chain", {"trials": 200, "bucket_count": 64,
                                      "app_id": "fact-verify"}, seed=1)
    wl = generate({"small": 1.0}, 1000, 1000.0, seed=0,
                  class_apps={"small": ["code-gen", "fact-verify"]})
    cfg = simcore.SimConfig(bucket_count=64, mc_samples=512,
                            cache_policy=CachePolicy.HERMES_PLAN)
    graphs = {"code-gen": code_gen, "fact-verify": fact}

    calls = []
    ref_mc = simcore.monte_carlo_remaining_demand

    def rec(*a, **k):
        t0 = time.perf_counter()
        r = ref_mc(*a, **k)
        calls.append((a, k, time.perf_counter() - t0))
        return r
    simcore.monte_carlo_remaining_demand = rec
    t0 = time.perf_counter()
    ref = simcore.run_simulation(graphs, wl, Policy.GITTINS, cfg, seed=0)
    t_ref = time.perf_counter() - t0
    simcore.monte_carlo_remaining_demand = ref_mc

    integration.patch_pdgsim(pdgsim)
    try:
        ours_mc = pdgsim.simcore.monte_carlo_remaining_demand
        run = simcore.run_simulation(graphs, wl, Policy.GITTINS, cfg, seed=0)   # warm
        t0 = time.perf_counter()
        run = simcore.run_simulation(graphs, wl, Policy.GITTINS, cfg, seed=0)
        t_ours = time.perf_counter() - t0
        lat = []
        for a, k, _ in calls[:400]:
            t1 = time.perf_counter()
            ours_mc(*a, **k)
            lat.append(time.perf_counter() - t1)
    finally:
        integration.restore()
    return {
        "sim_wall_s_reference": t_ref, "sim_wall_s_dropin": t_ours,
        "event_logs_identical": run.event_log == ref.event_log,
        "mc_calls": len(calls),
        "mc_call_p50_ms_reference": statistics.median(c[2] for c in calls) * 1e3,
        "mc_call_p50_ms_dropin": statistics.median(lat) * 1e3}


if __name__ == "__main__":
    print(json.dumps(measure()))
