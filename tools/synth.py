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
