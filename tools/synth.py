"""Synthetic config-2/3 workload: app-unique depth-8 PDGraphs.

Each application owns an 8-unit graph s0..s7 of non-LLM units (duration
records) shaped as a chain with a 3-way branch, a self-loop and a back-edge
loop:

    s0 -> s1 -> {s2 | s3 | s4};  s2 -> {s2 (self-loop) | s3};  s3 -> s4 -> s5
    s5 -> {s3 (back edge) | s6};  s6 -> s7 -> end

Every unit holds `n_rec` profiling records: a lognormal duration (mean
U(0.5, 60) s, sigma U(0.2, 0.8), app-specific) and the recorded next unit;
branch probabilities are the record frequencies (pdgraph.py:182-194).  The
same arrays are emitted both as device tables for the engine (vectorised, no
per-graph Python) and, for a sample of apps, as knowledge-base documents the
CPU oracle consumes -- so both sides see identical graphs.
"""

from __future__ import annotations

import numpy as np

U = 8
SLOT = 4        # successor-table slot per unit: <= 3 successors + terminal
UNIT_IDS = [f"s{i}" for i in range(U)]


def make(n_apps: int, n_rec: int = 256, seed: int = 2026):
    rng = np.random.default_rng(seed)
    mean = rng.uniform(0.5, 60.0, (n_apps, U))
    sig = rng.uniform(0.2, 0.8, (n_apps, U))
    mu = np.log(mean) - sig * sig / 2.0
    dur = np.exp(mu[..., None] + sig[..., None] * rng.standard_normal((n_apps, U, n_rec)))
    p_self = rng.uniform(0.3, 0.7, n_apps)
    p_back = rng.uniform(0.2, 0.5, n_apps)
    split = rng.dirichlet([1.0, 1.0, 1.0], n_apps)
    # recorded next unit per (app, unit, record); -1 = end
    nxt = np.full((n_apps, U, n_rec), -1, dtype=np.int8)
    nxt[:, 0] = 1
    r = rng.random((n_apps, n_rec))
    c = np.cumsum(split, axis=1)
    nxt[:, 1] = 2 + (r[:, :] >= c[:, 0:1]) + (r[:, :] >= c[:, 1:2])
    nxt[:, 2] = np.where(rng.random((n_apps, n_rec)) < p_self[:, None], 2, 3)
    nxt[:, 3] = 4
    nxt[:, 4] = 5
    nxt[:, 5] = np.where(rng.random((n_apps, n_rec)) < p_back[:, None], 3, 6)
    nxt[:, 6] = 7
    # every branch keeps at least one record, so every unit stays reachable
    # from s0 and the graph passes the reference's PDGraph.validate
    # (pdgraph.py:208-225; a Dirichlet split can otherwise draw no record)
    if n_rec >= 3:
        nxt[:, 1, :3] = np.array([2, 3, 4], dtype=np.int8)
        nxt[:, 2, :2] = np.array([2, 3], dtype=np.int8)
        nxt[:, 5, :2] = np.array([3, 6], dtype=np.int8)
    # successor tables: sorted by unit id == ascending index; probability =
    # count / n_rec; units never recorded as next are absent
    counts = np.zeros((n_apps, U, U), dtype=np.int64)
    for v in range(U):
        counts[:, :, v] = np.count_nonzero(nxt == v, axis=2)
    succ_cum = np.zeros((n_apps, U, SLOT))
    succ_nxt = np.full((n_apps, U, SLOT), -1, dtype=np.int32)
    succ_len = np.zeros((n_apps, U), dtype=np.int32)
    for u in range(U):
        present = counts[:, u, :] > 0                      # [A, U]
        k = present.sum(axis=1)
        succ_len[:, u] = k
        order = np.argsort(~present, axis=1, kind="stable")[:, :SLOT - 1]
        prob = np.take_along_axis(counts[:, u, :], order, axis=1) / float(n_rec)
        valid = np.arange(SLOT - 1)[None, :] < k[:, None]
        prob = np.where(valid, prob, 0.0)
        cs = np.cumsum(prob, axis=1)
        succ_cum[:, u, :SLOT - 1] = np.where(valid, cs, 0.0)
        succ_nxt[:, u, :SLOT - 1] = np.where(valid, order, -1)
    return {"n_apps": n_apps, "n_rec": n_rec, "dur": dur, "nxt": nxt, "succ_cum": succ_cum,
            "succ_nxt": succ_nxt, "succ_len": succ_len}


def bank(w, device="cuda"):
    """GraphBank with one graph per app (layout of graphs.UNIT_DTYPE)."""
    from paper_2506_14851_b200.graphs import UNIT_DTYPE, GraphBank
    A, R = w["n_apps"], w["n_rec"]
    units = np.zeros(A * U, dtype=UNIT_DTYPE)
    idx = np.arange(A * U)
    units["a_off"] = idx * R
    units["a_len"] = R
    units["succ_off"] = idx * SLOT
    units["succ_len"] = w["succ_len"].reshape(-1)
    return GraphBank.from_arrays(
        units=units, vals=w["dur"].reshape(-1), graph_base=np.arange(A) * U,
        graph_n=np.full(A, U), succ_cum=w["succ_cum"].reshape(-1),
        succ_nxt=w["succ_nxt"].reshape(-1), unit_capacity=np.full(A * U, 1000),
        device=device, unit_order={})


def kb_doc(w, app: int) -> dict:
    """Knowledge-base document (pdgraph.graph_to_dict shape) of one app."""
    units = []
    for u in range(U):
        recs = [{"trial_id": t, "duration": float(w["dur"][app, u, t]),
                 "next_unit": (UNIT_IDS[int(w["nxt"][app, u, t])]
                               if w["nxt"][app, u, t] >= 0 else None)}
                for t in range(w["n_rec"])]
        units.append({"unit_id": UNIT_IDS[u],
                      "backend": {"kind": "docker-exec", "image_id": f"img-{u}"},
                      "records": recs, "capacity": 1000, "bucket_count": 10})
    return {"app_id": f"app-{app}", "entry_unit": "s0", "units": units}


def jobs(n_apps: int, seed: int = 7):
    """Queue state: current unit uniform over the 8 (all reachable) units,
    per-app numpy seeds."""
    rng = np.random.default_rng(seed)
    return {"unit": rng.integers(0, U, n_apps).astype(np.int32),
            "seed": rng.integers(0, 2**62, n_apps).astype(np.int64)}


# ---------------------------------------------------------------------------
# config 4: refinement events over a queue of template apps
# ---------------------------------------------------------------------------

def template_queue(graphs: dict, n_apps: int, seed: int = 7):
    """Queue of n_apps instances of the template graphs (name -> KBGraph),
    each at a random unit that has at least one successor."""
    rng = np.random.default_rng(seed)
    names = list(graphs)
    orders = {nm: sorted(graphs[nm].units) for nm in names}
    gi = rng.integers(0, len(names), n_apps).astype(np.int32)
    ui = np.zeros(n_apps, dtype=np.int32)
    for g, nm in enumerate(names):
        cand = [i for i, u in enumerate(orders[nm]) if graphs[nm].units[u].successors]
        sel = gi == g
        ui[sel] = rng.choice(cand, int(sel.sum()))
    return {"names": names, "orders": orders, "graph": gi, "unit": ui}


def events(graphs: dict, q: dict, n_events: int, seed: int = 7):
    """n_events unit completions on distinct apps: the app's current unit
    completes with an observation drawn from that unit's records; the next
    unit is drawn by branch probability (pdgraph.py:182-194)."""
    rng = np.random.default_rng(seed)
    apps = rng.choice(len(q["graph"]), n_events, replace=False).astype(np.int32)
    nxt = np.zeros(n_events, dtype=np.int32)
    obs = np.zeros((n_events, 3))
    for e, a in enumerate(apps):
        nm = q["names"][q["graph"][a]]
        g = graphs[nm]
        uid = q["orders"][nm][q["unit"][a]]
        unit = g.units[uid]
        succ = sorted(unit.successors.items())
        p = np.array([x for _, x in succ])
        k = rng.choice(len(succ), p=p / p.sum())
        nxt[e] = q["orders"][nm].index(succ[k][0])
        r = unit.records[rng.integers(0, len(unit.records))]
        obs[e] = (r.input_len, r.output_len, float(r.parallelism))
    return {"app": apps, "completed": q["unit"][apps].copy(), "next": nxt, "obs": obs,
            "seed": rng.integers(0, 2**62, n_events).astype(np.int64)}


# ---------------------------------------------------------------------------
# config-2 LLM variant: depth-8 templates mixing LLM, own-input and
# upstream-conditioned (K3) units, as knowledge-base documents
# ---------------------------------------------------------------------------

# s0 plan (LLM) -> s1 retrieve (docker) -> {s2 draft | s3 refine | s4 tool};
# s2 draft (LLM, output ~ own input, self-loop) -> {s2 | s3};
# s3 refine (LLM, input ~ upstream output) -> s4 tool (dnn) -> s5 verify
# (LLM, output ~ upstream output) -> {s3 back edge | s6}; s6 run (docker) ->
# s7 report (LLM, output ~ own input) -> end
LLM_KINDS = ["llm", "docker", "llm", "llm", "dnn", "llm", "docker", "llm"]
LLM_MASKS = {2: {"output_own_input": True}, 3: {"input_upstream_output": True},
             5: {"output_upstream_output": True}, 7: {"output_own_input": True}}


def llm_docs(n_templates: int, n_trials: int = 200, seed: int = 2027) -> dict:
    """n_templates KB documents with the synth topology.  Every trial writes
    one record per unit (same trial_id across units, so K3 joins records);
    LLM lengths are lognormal, the masked dependencies are real correlations
    (own input -> output, upstream output -> input / output)."""
    rng = np.random.default_rng(seed)
    docs = {}
    for t in range(n_templates):
        T = n_trials
        p_self, p_back = rng.uniform(0.3, 0.6), rng.uniform(0.2, 0.4)
        split = rng.dirichlet([1.0, 1.0, 1.0])
        ln = lambda m, s, size=T: np.exp(np.log(m) - s * s / 2 + s * rng.standard_normal(size))  # noqa: E731
        inp = np.zeros((U, T))
        out = np.zeros((U, T))
        dur = np.zeros((U, T))
        for u in range(U):
            if LLM_KINDS[u] == "llm":
                inp[u] = ln(rng.uniform(300, 3000), 0.5)
                out[u] = ln(rng.uniform(100, 900), 0.5)
            else:
                dur[u] = ln(rng.uniform(1.0, 40.0), 0.5)
        out[2] = inp[2] * rng.uniform(0.2, 0.5) * ln(1.0, 0.15)       # own input
        inp[3] = out[2] * rng.uniform(1.0, 2.0) + ln(200.0, 0.3)        # upstream output
        out[5] = out[3] * rng.uniform(0.3, 0.8) * ln(1.0, 0.2)          # upstream output
        out[7] = inp[7] * rng.uniform(0.1, 0.4) * ln(1.0, 0.15)         # own input
        nxt = np.full((U, T), -1)
        nxt[0] = 1
        r = rng.random(T)
        nxt[1] = 2 + (r >= split[0]) + (r >= split[0] + split[1])
        nxt[2] = np.where(rng.random(T) < p_self, 2, 3)
        nxt[3], nxt[4] = 4, 5
        nxt[5] = np.where(rng.random(T) < p_back, 3, 6)
        nxt[6] = 7
        nxt[1, :3], nxt[2, :2], nxt[5, :2] = [2, 3, 4], [2, 3], [3, 6]
        units = []
        for u in range(U):
            kind = LLM_KINDS[u]
            backend = ({"kind": "llm-inference", "model_id": "base-7b", "warmup_time": 0.0}
                       if kind == "llm" else
                       {"kind": "docker-exec", "image_id": f"img-{t}-{u}", "warmup_time": 15.0}
                       if kind == "docker" else
                       {"kind": "dnn-tool", "tool_id": f"tool-{t}-{u}", "warmup_time": 8.0})
            recs = [{"trial_id": k, "input_len": float(inp[u, k]), "output_len": float(out[u, k]),
                     "parallelism": 1, "duration": float(dur[u, k]),
                     "next_unit": UNIT_IDS[nxt[u, k]] if nxt[u, k] >= 0 else None}
                    for k in range(T)]
            units.append({"unit_id": UNIT_IDS[u], "backend": backend, "records": recs,
                          "masks": dict(LLM_MASKS.get(u, {})), "capacity": 1000,
                          "bucket_count": 16})
        docs[f"llm8-{t}"] = {"app_id": f"llm8-{t}", "entry_unit": "s0", "units": units}
    return docs


def llm_queue(docs: dict, n_apps: int, seed: int = 9):
    """n_apps instances: template, current unit, and (for 3 in 4 apps) an
    observation of a recorded upstream execution of the current unit."""
    rng = np.random.default_rng(seed)
    names = list(docs)
    gi = rng.integers(0, len(names), n_apps).astype(np.int32)
    ui = rng.integers(0, U, n_apps).astype(np.int32)
    obs = []
    for a in range(n_apps):
        doc = docs[names[gi[a]]]
        cur = UNIT_IDS[ui[a]]
        ups = [u for u in doc["units"]
               if any(r["next_unit"] == cur for r in u["records"])] if rng.random() < 0.75 else []
        if ups:
            up = ups[rng.integers(0, len(ups))]
            r = up["records"][rng.integers(0, len(up["records"]))]
            obs.append((up["unit_id"], r["input_len"], r["output_len"], r["parallelism"]))
        else:
            obs.append(None)
    return {"names": names, "graph": gi, "unit": ui, "obs": obs,
            "seed": rng.integers(0, 2**62, n_apps).astype(np.int64)}


def llm_jobs(eng, q: dict, device):
    """Device job arrays for DemandEngine.run from llm_queue(): graph, unit,
    seed, conditioning upstream (local index, -1 = none) and its values."""
    import torch
    names, n = q["names"], len(q["graph"])
    ou = np.full(n, -1, dtype=np.int32)
    ov = np.zeros((n, 3))
    gidx = np.array([eng.bank.index[nm] for nm in names], dtype=np.int32)
    for a, o in enumerate(q["obs"]):
        if o is not None:
            ou[a] = eng.bank.local_unit(names[q["graph"][a]], o[0])
            ov[a] = o[1:]
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(device)  # noqa: E731
    return (t(gidx[q["graph"]]), t(q["unit"]), t(q["seed"]), t(ou), t(ov))
