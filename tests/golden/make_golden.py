"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

Everything written here is produced by the reference implementation itself
(``pdgsim`` imported read-only from /root/reference/pkg/src); the fixtures
travel to the GPU box, the reference does not.  Outputs:

* ``graphs.json.gz``     knowledge-base JSON (pdgraph.graph_to_dict) of every
                        graph used below
* ``mc_cases.json``     monte_carlo_remaining_demand calls: inputs, sha256 of
                        the float64 sample bytes, mean, conditioned, capped
* ``mc_samples.npz``    full sample vectors for a subset of those calls
* ``gittins.npz``       gittins_rank_batch inputs/outputs (hand cases, random
                        batches, rows captured from the config-1 simulation)
* ``binning.json.gz``    bucketize / bucket_points / bucket_index / survival
* ``prewarm.json``      plan_prewarm calls (hand, random, config-1 captured)
* ``config1.json.gz``    config-1 simulation summary: every MC call (hashes),
                        refresh statistics, event-log sha256
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import pdgsim  # noqa: E402
from pdgsim import estimator as est  # noqa: E402
from pdgsim import sched, simcore  # noqa: E402
from pdgsim.distributions import EmpiricalDistribution  # noqa: E402
from pdgsim.estimator import Observation, build_masks  # noqa: E402
from pdgsim.pdgraph import (BackendKind, BackendSpec, FunctionalUnit, PDGraph,  # noqa: E402
                            RateProfile, UnitRecord, graph_to_dict, record_trial)
from pdgsim.prewarm import CachePolicy, plan_prewarm  # noqa: E402
from pdgsim.workload import archetype, generate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ENV = RateProfile(10000.0, 50.0)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


# --------------------------------------------------------------------------
# graphs
# --------------------------------------------------------------------------

def docker(uid, image="img", bc=10):
    return FunctionalUnit(uid, BackendSpec(BackendKind.DOCKER_EXEC, image_id=image),
                          bucket_count=bc)


def llm(uid, bc=10):
    return FunctionalUnit(uid, BackendSpec(BackendKind.LLM_INFERENCE, model_id="m"),
                          bucket_count=bc)


def duration_graph(name, edges):
    """Same construction as the reference test helper (test_estimator.py:37-56)."""
    g = PDGraph(name, "a")
    for uid in edges:
        g.add_unit(docker(uid))
    n_trials = max(len(v) for v in edges.values())
    for t in range(n_trials):
        trial = {}
        for uid, rows in edges.items():
            if t < len(rows):
                dur, nxt = rows[t]
                trial[uid] = UnitRecord(t, duration=dur, next_unit=nxt)
        path, uid = {}, "a"
        while uid in trial and uid not in path:
            path[uid] = trial[uid]
            uid = trial[uid].next_unit
        record_trial(g, path)
    return g


def bimodal_graph():
    g = PDGraph("bimodal", "up")
    g.add_unit(llm("up"))
    g.add_unit(llm("down"))
    for t in range(40):
        heavy = t % 2 == 0
        up_out = 1000.0 if heavy else 10.0
        record_trial(g, {
            "up": UnitRecord(t, input_len=400, output_len=up_out, next_unit="down"),
            "down": UnitRecord(t, input_len=up_out + 5,
                               output_len=8000.0 if heavy else 80.0),
        })
    return build_masks(g)


def cond_graph():
    g = PDGraph("cond", "up")
    g.add_unit(llm("up"))
    g.add_unit(llm("down"))
    rows = [(10.0, 3.0)] * 5 + [(90.0, 50.0)]
    for t, (up_out, down_in) in enumerate(rows):
        record_trial(g, {
            "up": UnitRecord(t, input_len=500, output_len=up_out, next_unit="down"),
            "down": UnitRecord(t, input_len=down_in, output_len=20.0),
        })
    g.units["down"].masks.input_upstream_output = True
    return g


def depth8_graph(seed: int, n_samples: int = 300, bc: int = 64):
    """Depth-8 synthetic graph (config-2 shape): non-LLM units, chain with a
    3-way branch, a self-loop and a back-edge loop; lognormal durations."""
    rnd = random.Random(seed)
    uids = [f"s{i}" for i in range(8)]
    g = PDGraph(f"depth8-{seed}", uids[0])
    for u in uids:
        g.add_unit(docker(u, image=f"img-{u}", bc=bc))
    means = {u: rnd.uniform(0.5, 60.0) for u in uids}
    sig = {u: rnd.uniform(0.2, 0.8) for u in uids}
    p_self = rnd.uniform(0.3, 0.7)
    p_back = rnd.uniform(0.2, 0.5)

    def dur(u):
        mu = np.log(means[u]) - sig[u] ** 2 / 2
        return rnd.lognormvariate(mu, sig[u])

    for t in range(n_samples):
        trial, seq = {}, []
        cur, visits = "s0", 0
        seen = set()
        while cur is not None and visits < 40:
            visits += 1
            i = int(cur[1:])
            if cur == "s2" and rnd.random() < p_self:
                nxt = "s2"
            elif cur == "s5" and rnd.random() < p_back:
                nxt = "s3"
            elif cur == "s1":
                nxt = rnd.choice(["s2", "s3", "s4"])
            elif i < 7:
                nxt = f"s{i + 1}"
            else:
                nxt = None
            if cur not in seen:   # one record per unit per trial (first visit)
                trial[cur] = UnitRecord(t, duration=dur(cur), next_unit=nxt)
                seen.add(cur)
            seq.append(cur)
            cur = nxt if nxt not in seen else None
        record_trial(g, trial)
    g.validate()
    return g


def all_graphs():
    gs = {}
    gs["fanout-reduce"] = archetype("fanout-reduce", {"trials": 120}, seed=5)
    gs["verify-chain-bimodal"] = archetype(
        "verify-chain", {"trials": 200, "bucket_count": 64, "bimodal": True}, seed=2)
    gs["react-loop"] = archetype("react-loop", {"trials": 150}, seed=4)
    gs["plan-execute"] = archetype("plan-execute", {"trials": 150}, seed=6)
    gs["code-gen"] = archetype(
        "code-check", {"trials": 200, "bucket_count": 64, "scale": 0.6,
                       "app_id": "code-gen"}, seed=3)
    gs["fact-verify"] = archetype(
        "verify-chain", {"trials": 200, "bucket_count": 64, "app_id": "fact-verify"},
        seed=1)
    gs["point"] = duration_graph("point", {"a": [(5.0, None)] * 3})
    gs["chain"] = duration_graph("chain", {"a": [(3.0, "b")] * 3, "b": [(4.0, None)] * 3})
    gs["branch"] = duration_graph("branch", {
        "a": [(1.0, "b"), (1.0, "c")] * 10, "b": [(2.0, None)] * 20,
        "c": [(10.0, None)] * 20})
    gs["selfloop"] = duration_graph("selfloop", {"a": [(1.0, "a")] * 4})
    gs["mixed"] = duration_graph("mixed", {
        "a": [(1.0, "b"), (2.0, None)] * 5, "b": [(4.0, None)] * 5})
    gs["bimodal"] = bimodal_graph()
    gs["cond"] = cond_graph()
    for s in range(3):
        g = depth8_graph(100 + s)
        gs[g.app_id] = g
    for k, g in gs.items():
        g.app_id = k
    return gs


# --------------------------------------------------------------------------
# MC cases
# --------------------------------------------------------------------------

def obs_to_json(o: Observation):
    return {"unit_id": o.unit_id, "input_len": o.input_len,
            "output_len": o.output_len, "parallelism": o.parallelism}


def mc_case(g, gid, cur, obs, n, seed, cap, keep_full, full):
    rem = est.monte_carlo_remaining_demand(g, cur, obs, ENV, n=n, seed=seed,
                                           visit_cap=cap)
    s = np.asarray(rem.samples, dtype=np.float64)
    case = {"graph": gid, "current": cur, "obs": [obs_to_json(o) for o in obs],
            "n": n, "seed": seed, "visit_cap": cap, "sha256": sha(s),
            "mean": float(s.mean()), "conditioned": bool(rem.conditioned),
            "capped": int(rem.capped_walks)}
    if keep_full:
        key = f"c{len(full)}"
        full[key] = s
        case["full"] = key
    return case


def make_mc_cases(gs):
    rnd = random.Random(2026)
    cases, full = [], {}
    for gid, g in gs.items():
        uids = sorted(g.units)
        for rep in range(6):
            cur = uids[rep % len(uids)]
            obs = []
            ups = [u for u in uids if cur in g.units[u].successors]
            if ups and rep % 2 == 1:
                up = g.units[rnd.choice(ups)]
                rec = rnd.choice(list(up.records))
                if rep % 3 == 0:   # off-distribution observation -> sparse bucket
                    obs = [Observation(up.unit_id, input_len=rec.input_len * 7.0,
                                       output_len=rec.output_len * 9.0 + 1.0,
                                       parallelism=rec.parallelism)]
                else:
                    obs = [Observation(up.unit_id, input_len=rec.input_len,
                                       output_len=rec.output_len,
                                       parallelism=rec.parallelism)]
                # an irrelevant earlier observation must be skipped over
                obs = [Observation(cur, input_len=1.0, output_len=1.0)] + obs
            n = [512, 1, 7, 100, 1000, 33][rep]
            cap = 8 if (gid == "selfloop" and rep == 0) else 64
            seed = rnd.randrange(0, 2 ** 31 - 1)
            cases.append(mc_case(g, gid, cur, obs, n, seed, cap,
                                 keep_full=(rep < 2), full=full))
    return cases, full


# --------------------------------------------------------------------------
# binning / gittins / prewarm
# --------------------------------------------------------------------------

def make_binning():
    rnd = random.Random(7)
    out = []
    lists = [[1, 1, 2, 9], [7, 7, 7], [0, 100], [0, 10], [3, 8, 1, 9], [5.0]]
    for _ in range(40):
        k = rnd.randint(1, 40)
        lists.append([rnd.lognormvariate(2.0, 1.5) for _ in range(k)])
    for _ in range(10):
        lists.append([round(rnd.uniform(0, 50), 1) for _ in range(rnd.randint(2, 300))])
    for li, xs in enumerate(lists):
        for bc in ((1, 2, 10, 64, 256) if len(xs) <= 40 else (3, 64)):
            d = EmpiricalDistribution(xs, capacity=max(len(xs), 1), bucket_count=bc)
            b = d.bucketize()
            vals, probs = d.bucket_points()
            qs = sorted(set([min(xs), max(xs), (min(xs) + max(xs)) / 2,
                             min(xs) - 1.0, max(xs) + 1.0] + list(xs[:5])
                            + [b[0][0] + i * (b[-1][1] - b[0][0]) / len(b)
                               for i in range(len(b))]))
            out.append({"samples": [float(x) for x in xs], "bucket_count": bc,
                        "buckets": [list(t) for t in b], "values": vals,
                        "probs": probs, "boundaries": d.bucket_boundaries(),
                        "queries": qs,
                        "index": [d.bucket_index(q) for q in qs],
                        "survival": [d.survival(q) for q in qs]})
    return out


def make_gittins(captured):
    out = {}
    # hand cases (test_sched.py:40-48, 80-91, 179-185)
    hv = [[10.0, 10.0], [2.0, 10.0], [2.0, 10.0], [1.0, 4.0, 9.0], [3.0, 3.0],
          [5.0, 5.0]]
    hp = [[0.5, 0.5], [0.5, 0.5], [0.5, 0.5], [0.5, 0.25, 0.25], [1.0, 0.0],
          [0.5, 0.5]]
    ha = [4.0, 0.0, 2.0, 0.5, 3.0, 8.0]
    out["hand_values"] = np.array(hv[:3] + [hv[4]] + [hv[5]])
    out["hand_probs"] = np.array(hp[:3] + [hp[4]] + [hp[5]])
    out["hand_ages"] = np.array(ha[:3] + [ha[4]] + [ha[5]])
    out["hand_ranks"] = sched.gittins_rank_batch(out["hand_values"], out["hand_probs"],
                                                 out["hand_ages"])
    out["pts_values"] = np.array(hv[3])
    out["pts_probs"] = np.array(hp[3])
    # random batch (test_sched.py:93-107)
    rng = np.random.default_rng(11)
    v = np.sort(rng.uniform(1, 100, size=(40, 10)), axis=1)
    p = rng.uniform(0.1, 1, size=(40, 10))
    p /= p.sum(axis=1, keepdims=True)
    a = rng.uniform(0, 50, size=40)
    out["r10_values"], out["r10_probs"], out["r10_ages"] = v, p, a
    out["r10_ranks"] = sched.gittins_rank_batch(v, p, a)
    # heavy-tailed 256-bin rows with zero-mass bins and large ages
    rng = np.random.default_rng(2026)
    n, b = 100, 256
    lo = rng.uniform(0, 3000, size=n)
    w = rng.uniform(0.01, 20, size=n)
    est_age = rng.uniform(0, 500, size=n)
    j = np.arange(b)
    v = ((lo[:, None] + j * w[:, None]) + (lo[:, None] + (j + 1) * w[:, None])) / 2.0
    v = v + est_age[:, None]
    p = rng.lognormal(0, 2, size=(n, b))
    p[rng.random((n, b)) < 0.3] = 0.0
    p /= np.maximum(p.sum(axis=1, keepdims=True), 1e-300)
    age = est_age + rng.uniform(0, 1.1, size=n) * (lo + b * w)
    age[:5] = v[:5, -1]          # exactly at the last support point: exhausted
    age[5:10] = v[5:10, 17]      # exactly at a support point
    out["r256_values"], out["r256_probs"], out["r256_ages"] = v, p, age
    out["r256_ranks"] = sched.gittins_rank_batch(v, p, age)
    # rows captured from the config-1 simulation
    if captured:
        V = np.concatenate([c[0] for c in captured])
        P = np.concatenate([c[1] for c in captured])
        A = np.concatenate([c[2] for c in captured])
        R = np.concatenate([c[3] for c in captured])
        out["cfg1_values"], out["cfg1_probs"], out["cfg1_ages"], out["cfg1_ranks"] = V, P, A, R
    return out


def make_prewarm(captured):
    def dist(xs, bc=10):
        return EmpiricalDistribution(xs, capacity=max(len(xs), 1), bucket_count=bc)

    cases = []

    def add(xs, bc, p_s, t_p, knob, now):
        plan = plan_prewarm(dist(xs, bc), p_s, t_p, knob, now)
        cases.append({"samples": [float(x) for x in xs], "bucket_count": bc,
                      "p_s": p_s, "t_p": t_p, "knob": knob, "now": now,
                      "plan": None if plan is None else [plan.trigger_time, plan.p_e]})

    # prewarm test cases (test_prewarm.py:24-46)
    add([60.0], 10, 0.3, 10.0, 0.5, 0.0)
    add([60.0], 10, 1.0, 10.0, 0.5, 0.0)
    add([40.0, 80.0], 1, 0.8, 10.0, 0.4, 0.0)
    add([5.0], 10, 0.6, 50.0, 0.6, 0.0)
    add([60.0], 10, 1.0, 10.0, 0.5, 55.0)
    rnd = random.Random(31)
    for _ in range(300):
        m = rnd.randint(1, 60)
        xs = [rnd.uniform(1, 500) for _ in range(m)]
        now = rnd.choice([0.0, rnd.uniform(0, 400)])
        add(xs, rnd.choice([1, 3, 10, 32, 64]), rnd.uniform(0, 1), rnd.uniform(0, 60),
            rnd.uniform(0, 1), now)
    for c in captured:
        cases.append(c)
    return cases


# --------------------------------------------------------------------------
# config-1 simulation capture
# --------------------------------------------------------------------------

def run_config1():
    code_gen = archetype("code-check", {"trials": 200, "bucket_count": 64, "scale": 0.6,
                                        "app_id": "code-gen"}, seed=3)
    fact = archetype("verify-chain", {"trials": 200, "bucket_count": 64,
                                      "app_id": "fact-verify"}, seed=1)
    graphs = {"code-gen": code_gen, "fact-verify": fact}
    wl = generate({"small": 1.0}, 1000, 1000.0, seed=0,
                  class_apps={"small": ["code-gen", "fact-verify"]})
    cfg = simcore.SimConfig(bucket_count=64, mc_samples=512,
                            cache_policy=CachePolicy.HERMES_PLAN)
    mc_calls, gcalls, pcalls = [], [], []
    orig_mc = simcore.monte_carlo_remaining_demand
    orig_g = sched.gittins_rank_batch
    orig_p = simcore.plan_prewarm

    def mc_hook(graph, current_unit, observations, env, n, seed, visit_cap=64):
        rem = orig_mc(graph, current_unit, observations, env, n=n, seed=seed,
                      visit_cap=visit_cap)
        s = np.asarray(rem.samples, dtype=np.float64)
        mc_calls.append({"graph": graph.app_id, "current": current_unit,
                         "obs": [obs_to_json(o) for o in observations], "n": n,
                         "seed": seed, "visit_cap": visit_cap, "sha256": sha(s),
                         "mean": float(s.mean()), "conditioned": bool(rem.conditioned),
                         "capped": int(rem.capped_walks)})
        return rem

    def g_hook(values, probs, ages):
        r = orig_g(values, probs, ages)
        gcalls.append((np.array(values, dtype=np.float64), np.array(probs, dtype=np.float64),
                       np.array(ages, dtype=np.float64), np.array(r)))
        return r

    def p_hook(completion_dist, p_s, t_p, knob, now, target_backend=None):
        plan = orig_p(completion_dist, p_s, t_p, knob, now, target_backend=target_backend)
        pcalls.append({"samples": completion_dist.samples,
                       "bucket_count": completion_dist.bucket_count, "p_s": p_s,
                       "t_p": t_p, "knob": knob, "now": now,
                       "plan": None if plan is None else [plan.trigger_time, plan.p_e]})
        return plan

    simcore.monte_carlo_remaining_demand = mc_hook
    sched.gittins_rank_batch = g_hook
    simcore.plan_prewarm = p_hook
    try:
        res = simcore.run_simulation(graphs, wl, sched.Policy.GITTINS, cfg, seed=0)
    finally:
        simcore.monte_carlo_remaining_demand = orig_mc
        sched.gittins_rank_batch = orig_g
        simcore.plan_prewarm = orig_p
    log_sha = hashlib.sha256("\n".join(res.event_log).encode()).hexdigest()
    rows = sum(len(c[3]) for c in gcalls)
    summary = {"n_mc_calls": len(mc_calls), "n_gittins_calls": len(gcalls),
               "n_gittins_rows": rows, "n_prewarm_calls": len(pcalls),
               "event_log_sha256": log_sha, "event_log_lines": len(res.event_log),
               "mc_calls": mc_calls}
    # keep a bounded subsample of refresh rows: one call in every 40, <= 1200 rows
    keep, total = [], 0
    for i, c in enumerate(gcalls):
        if i % 40 == 0 and total + len(c[3]) <= 600:
            keep.append(c)
            total += len(c[3])
    return graphs, summary, keep, pcalls


def main():
    gs = all_graphs()
    c1_graphs, c1_summary, c1_rows, c1_prewarm = run_config1()
    for k, g in c1_graphs.items():
        gs[k] = g      # identical construction; config-1 graphs win
    graphs_doc = {k: graph_to_dict(g) for k, g in sorted(gs.items())}
    with gzip.open(os.path.join(OUT, "graphs.json.gz"), "wt") as fh:
        json.dump(graphs_doc, fh)
    cases, full = make_mc_cases(gs)
    meta = {"numpy": np.__version__, "pdgsim": pdgsim.__version__,
            "generator": "tests/golden/make_golden.py"}
    with open(os.path.join(OUT, "mc_cases.json"), "w") as fh:
        json.dump({"meta": meta, "cases": cases}, fh)
    np.savez_compressed(os.path.join(OUT, "mc_samples.npz"), **full)
    np.savez_compressed(os.path.join(OUT, "gittins.npz"), **make_gittins(c1_rows))
    with gzip.open(os.path.join(OUT, "binning.json.gz"), "wt") as fh:
        json.dump(make_binning(), fh)
    with open(os.path.join(OUT, "prewarm.json"), "w") as fh:
        json.dump(make_prewarm(c1_prewarm), fh)
    c1_summary["meta"] = meta
    with gzip.open(os.path.join(OUT, "config1.json.gz"), "wt") as fh:
        json.dump(c1_summary, fh)
    print("mc cases", len(cases), "config1 mc calls", c1_summary["n_mc_calls"],
          "gittins rows kept", sum(len(c[3]) for c in c1_rows),
          "prewarm calls", c1_summary["n_prewarm_calls"])


if __name__ == "__main__":
    main()
