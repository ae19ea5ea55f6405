"""PDGraph -> device template tables ("graph bank") for the demand engine.

Accepts the reference's own ``pdgsim.PDGraph`` objects (duck-typed: only
``units``, ``records``, ``*_dist.samples``, ``successors``, ``masks``,
``bucket_count``, ``is_llm`` are read) or knowledge-base JSON documents in the
reference's format (pdgraph.py:304-409, parsed here by ``KBGraph``).

What is precomputed per unit is fixed by the profiled knowledge base
(SPEC: templates change only on profiling updates), so it is compiled once
and kept resident in HBM:

* sample pools (float64) the walk draws from (estimator.py:250-269):
  input/output token lengths for LLM units, durations otherwise;
* the unit's input-length bucketing and the per-bucket output pools used for
  within-unit input->output correlation (estimator.py:255-264, 275-283);
* the cumulative successor table and next-unit indices (estimator.py:336-339,
  pdgraph.py:182-194);
* for online refinement (K3, estimator.py:155-233): the records joined on
  trial_id with every upstream, with the upstream bucket of each masked
  variable precomputed.

Unit order inside a graph is ``sorted(unit_id)`` exactly as the reference
walk indexes units (estimator.py:326-327).
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

# unit descriptor flags (mirrors include/pdg_b200.h)
F_LLM = 1
F_OWN = 2            # output_own_input mask with records (estimator.py:255)
F_ANYMASK = 4        # masks.any() (estimator.py:299)
FEATURES_VALID = 0x40000000   # pdg_graph_bank.features: the kind bits are set
F_IUI = 8            # input_upstream_input
F_IUO = 16           # input_upstream_output
F_OUO = 32           # output_upstream_output
F_PUP = 64           # parallelism_upstream_parallelism

UNIT_DTYPE = np.dtype([
    ("flags", "<i4"), ("a_off", "<i4"), ("a_len", "<i4"), ("b_off", "<i4"),
    ("b_len", "<i4"), ("succ_off", "<i4"), ("succ_len", "<i4"), ("pool_off", "<i4"),
    ("ib_k", "<i4"), ("cond_off", "<i4"), ("ib_lo", "<f8"), ("ib_hi", "<f8"),
    ("cond_len", "<i4"), ("pad", "<i4")])
assert UNIT_DTYPE.itemsize == 64

# upstream-bucketing descriptor per (unit, upstream) pair for K3
COND_DTYPE = np.dtype([
    ("up_local", "<i4"), ("pair_off", "<i4"), ("pair_len", "<i4"), ("pad", "<i4"),
    ("lo", "<f8", (3,)), ("hi", "<f8", (3,)), ("k", "<i4", (3,)), ("ok", "<i4", (3,)),
    ("pad2", "<i4", (2,))])
# per joined pair: upstream buckets of (input, output, parallelism) + the
# unit record's (input, output)
PAIR_DTYPE = np.dtype([("bk", "<i4", (3,)), ("pad", "<i4"), ("in", "<f8"), ("out", "<f8")])


# ---------------------------------------------------------------------------
# knowledge-base JSON model (independent of the reference package)
# ---------------------------------------------------------------------------

@dataclass
class KBRecord:
    trial_id: int
    input_len: float
    output_len: float
    parallelism: int
    duration: float
    next_unit: Optional[str]


class _Samples:
    def __init__(self, xs):
        self.samples = list(xs)


@dataclass
class KBMasks:
    input_upstream_input: bool = False
    input_upstream_output: bool = False
    output_upstream_output: bool = False
    output_own_input: bool = False
    parallelism_upstream_parallelism: bool = False

    def any(self) -> bool:
        return (self.input_upstream_input or self.input_upstream_output
                or self.output_upstream_output or self.output_own_input
                or self.parallelism_upstream_parallelism)


@dataclass
class KBUnit:
    unit_id: str
    is_llm: bool
    capacity: int
    bucket_count: int
    records: list
    masks: KBMasks
    warmup_time: float = 0.0
    warm_content: Optional[str] = None
    successors: dict = field(default_factory=dict)

    @property
    def input_dist(self):
        return _Samples([r.input_len for r in self.records] if self.is_llm else [])

    @property
    def output_dist(self):
        return _Samples([r.output_len for r in self.records] if self.is_llm else [])

    @property
    def parallelism_dist(self):
        return _Samples([float(r.parallelism) for r in self.records] if self.is_llm else [])

    @property
    def duration_dist(self):
        return _Samples([] if self.is_llm else [r.duration for r in self.records])


@dataclass
class KBGraph:
    app_id: str
    entry_unit: str
    units: dict


def graph_from_kb(doc: dict) -> KBGraph:
    """Parse one knowledge-base document (pdgraph.graph_from_dict semantics:
    distributions and branch frequencies are rebuilt from the FIFO-capped
    records, pdgraph.py:162-194, 376-407)."""
    units = {}
    for u in doc["units"]:
        b = u["backend"]
        kind = b.get("kind")
        cap = int(u.get("capacity", 1000))
        recs = deque(maxlen=cap)
        for r in u.get("records", []):
            recs.append(KBRecord(int(r["trial_id"]), float(r.get("input_len", 0.0)),
                                 float(r.get("output_len", 0.0)), int(r.get("parallelism", 1)),
                                 float(r.get("duration", 0.0)), r.get("next_unit")))
        if kind == "llm-inference":
            warm = b.get("kv_prefix_id") or b.get("lora_id")
        elif kind == "docker-exec":
            warm = b.get("image_id")
        else:
            warm = b.get("tool_id")
        m = u.get("masks", {})
        unit = KBUnit(u["unit_id"], kind == "llm-inference", cap, int(u.get("bucket_count", 10)),
                      list(recs), KBMasks(**{k: bool(v) for k, v in m.items()}),
                      float(b.get("warmup_time", 0.0)), warm)
        counts: dict = {}
        for r in unit.records:
            if r.next_unit is not None:
                counts[r.next_unit] = counts.get(r.next_unit, 0) + 1
        n = len(unit.records)
        unit.successors = {k: c / n for k, c in sorted(counts.items())} if n else {}
        units[unit.unit_id] = unit
    return KBGraph(doc["app_id"], doc["entry_unit"], units)


class GraphError(ValueError):
    """Mirror of pdgsim.errors.GraphError for KB graphs."""


def record_trial(graph: KBGraph, trial: dict) -> KBGraph:
    """Append one profiling trial (unit id -> KBRecord) to a KB graph, as
    pdgraph.record_trial does (pdgraph.py:247-279): unknown units and
    records not connected to the entry unit are rejected; each unit keeps
    its last `capacity` records (FunctionalUnit.records is a capped deque,
    pdgraph.py:148-160) and its branch frequencies are recomputed
    (branch_probabilities, pdgraph.py:182-194).  Masks are left alone
    (build_masks recomputes them, estimator.py:108-142).  Then call
    GraphBank.update / DemandEngine.refresh."""
    for uid in trial:
        if uid not in graph.units:
            raise GraphError(f"trial references unknown unit {uid!r}")
    if graph.entry_unit not in trial:
        raise GraphError(f"trial does not include the entry unit {graph.entry_unit!r}")
    visited: set = set()
    stack = [graph.entry_unit]
    while stack:
        uid = stack.pop()
        if uid in visited or uid not in trial:
            continue
        visited.add(uid)
        nxt = trial[uid].next_unit
        if nxt is not None:
            stack.append(nxt)
    disconnected = set(trial) - visited
    if disconnected:
        raise GraphError(f"trial records disconnected from entry: {sorted(disconnected)}")
    for uid in sorted(trial):
        u = graph.units[uid]
        u.records = (list(u.records) + [trial[uid]])[-u.capacity:]
        counts: dict = {}
        for r in u.records:
            if r.next_unit is not None:
                counts[r.next_unit] = counts.get(r.next_unit, 0) + 1
        n = len(u.records)
        u.successors = {k: c / n for k, c in sorted(counts.items())} if n else {}
    return graph


MASK_NAMES = ("input_upstream_input", "input_upstream_output", "output_upstream_output",
              "output_own_input", "parallelism_upstream_parallelism")


def _mask_jobs(graph):
    """(unit, mask, xs, ys) correlated by build_masks (estimator.py:108-142):
    a unit without upstreams only gets output_own_input; otherwise the
    (upstream record, unit record) pairs joined on trial_id, upstreams in
    sorted order (_joined_pairs, estimator.py:84-95)."""
    jobs = []
    for uid in sorted(graph.units):
        u = graph.units[uid]
        ups = [v for v in sorted(graph.units)
               if any(r.next_unit == uid for r in graph.units[v].records)]
        own = ([r.output_len for r in u.records], [r.input_len for r in u.records])
        if not ups:
            jobs.append((uid, "output_own_input") + own)
            continue
        by_trial = {r.trial_id: r for r in u.records}
        pairs = [(ur, by_trial[ur.trial_id]) for v in ups for ur in graph.units[v].records
                 if ur.next_unit == uid and ur.trial_id in by_trial]
        up_in = [p[0].input_len for p in pairs]
        up_out = [p[0].output_len for p in pairs]
        my_in = [p[1].input_len for p in pairs]
        my_out = [p[1].output_len for p in pairs]
        jobs += [(uid, "input_upstream_input", my_in, up_in),
                 (uid, "input_upstream_output", my_in, up_out),
                 (uid, "output_upstream_output", my_out, up_out),
                 (uid, "output_own_input") + own,
                 (uid, "parallelism_upstream_parallelism",
                  [float(p[1].parallelism) for p in pairs],
                  [float(p[0].parallelism) for p in pairs])]
    return jobs


def build_masks(graphs, threshold: float = 0.5, device: str = "cuda", timing=None):
    """estimator.build_masks (estimator.py:108-142) for a set of graphs in one
    launch (pdg_pearson_flags): sets every unit's correlation masks in place
    and returns {name: {unit: {mask: rho or None}}}.  timing (dict, optional)
    receives the kernel time in ms (CUDA events)."""
    import ctypes as C

    import torch

    from . import _lib
    if not isinstance(graphs, dict):
        graphs = {"g": graphs}
    jobs, xs, ys, off, ln = [], [], [], [], []
    for nm, g in graphs.items():
        for uid, mask, x, y in _mask_jobs(g):
            jobs.append((nm, uid, mask))
            off.append(len(xs))
            ln.append(len(x) if len(x) == len(y) else 0)
            xs.extend(x)
            ys.extend(y)
    dev = torch.device(device)
    t = lambda a, dt: torch.tensor(a if len(a) else [0], dtype=dt, device=dev)  # noqa: E731
    X, Y, O, N = t(xs, torch.float64), t(ys, torch.float64), t(off, torch.int32), \
        t(ln, torch.int32)
    rho = torch.empty(max(len(jobs), 1), dtype=torch.float64, device=dev)
    flag = torch.empty(max(len(jobs), 1), dtype=torch.uint8, device=dev)
    if timing is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    _lib.check(_lib.lib().pdg_pearson_flags(_lib.ptr(X), _lib.ptr(Y), _lib.ptr(O), _lib.ptr(N),
                                            len(jobs), C.c_double(threshold), _lib.ptr(rho),
                                            _lib.ptr(flag), _lib.stream_ptr()),
               "pdg_pearson_flags")
    if timing is not None:
        e1.record()
        e1.synchronize()
        timing["kernel_ms"] = e0.elapsed_time(e1)
    rho_h, flag_h = rho.cpu().numpy(), flag.cpu().numpy()
    out: dict = {}
    for nm, g in graphs.items():
        for uid, u in g.units.items():
            for k in MASK_NAMES:
                setattr(u.masks, k, False)
    for i, (nm, uid, mask) in enumerate(jobs):
        setattr(graphs[nm].units[uid].masks, mask, bool(flag_h[i]))
        r = float(rho_h[i])
        out.setdefault(nm, {}).setdefault(uid, {})[mask] = None if r != r else r
    return out


# ---------------------------------------------------------------------------
# bucketing helpers (distributions.py:79-118), host side, exact float64
# ---------------------------------------------------------------------------

def binning(samples, k: int):
    """(lo, hi_edge, k_eff) of equal-width bucketing; k_eff = 1 when degenerate.
    hi_edge = lo + k*width is the last bucket's upper edge (bucket_index uses
    it, not the sample max)."""
    xs = [float(x) for x in samples]
    if not xs:
        return None
    lo, hi = min(xs), max(xs)
    if lo == hi:
        return lo, lo, 1
    w = (hi - lo) / k
    return lo, lo + k * w, int(k)


def bucket_index(bn, value: float) -> int:
    lo, hi, k = bn
    if hi == lo or value <= lo:
        return 0
    if value >= hi:
        return k - 1
    return min(int((value - lo) / ((hi - lo) / k)), k - 1)


def _masks(unit):
    m = unit.masks
    f = 0
    if m.any():
        f |= F_ANYMASK
    f |= F_IUI if m.input_upstream_input else 0
    f |= F_IUO if m.input_upstream_output else 0
    f |= F_OUO if m.output_upstream_output else 0
    f |= F_PUP if m.parallelism_upstream_parallelism else 0
    return f


# ---------------------------------------------------------------------------
# the bank
# ---------------------------------------------------------------------------

class GraphBank:
    """Compiled device tables for a set of graphs (name -> graph).

    Each graph compiles to a self-contained segment (offsets local to the
    segment); the bank is the concatenation of the segments with the
    offsets rebased.  ``update(name)`` recompiles one graph after its
    records changed (``record_trial``) and rebuilds the device tables from
    the cached segments, so a profiling trial costs one graph's compile."""

    def __init__(self, graphs: dict, device: str = "cuda"):
        self.names = list(graphs)
        self.index = {nm: i for i, nm in enumerate(self.names)}
        self.unit_order = {}        # name -> [uid sorted]
        self.empty_units = {}       # name -> [(uid, message)] (estimator.py:246-268)
        self.graphs = graphs
        self.device = device
        self._segments = {nm: self._compile(nm, graphs[nm]) for nm in self.names}
        self._place()

    def update(self, name: str, graph=None) -> None:
        """Recompile graph `name` (optionally replacing it) and rebuild the
        device tables.  Pointers held by a DemandEngine must be re-bound
        (DemandEngine.refresh does both)."""
        if name not in self.index:
            raise KeyError(name)
        if graph is not None:
            self.graphs[name] = graph
        self.empty_units.pop(name, None)
        self._segments[name] = self._compile(name, self.graphs[name])
        self._place()

    def _compile(self, nm, g) -> dict:
        vals: list = []
        kinds: list = []            # 0 duration, 1 input (/prefill), 2 output (/decode)
        units = []
        pools_off, pools_len = [], []
        succ_cum, succ_nxt = [], []
        conds, pairs = [], []

        def push(xs, kind=0) -> tuple[int, int]:
            off = len(vals)
            vals.extend(float(x) for x in xs)
            kinds.extend([kind] * len(xs))
            return off, len(xs)

        order = sorted(g.units)
        if len(order) > 64:
            raise ValueError(f"graph {nm!r}: more than 64 units")
        self.unit_order[nm] = order
        for uid in order:
            u = g.units[uid]
            if u.is_llm and (not list(u.input_dist.samples) or
                             not list(u.output_dist.samples)):
                self.empty_units.setdefault(nm, []).append(
                    (uid, f"unit {uid!r} has no token-length samples"))
            elif not u.is_llm and not list(u.duration_dist.samples):
                self.empty_units.setdefault(nm, []).append(
                    (uid, f"unit {uid!r} has no duration samples"))
        pos = {u: i for i, u in enumerate(order)}
        for uid in order:
            u = g.units[uid]
            d = np.zeros((), dtype=UNIT_DTYPE)
            flags = _masks(u)
            if u.is_llm:
                flags |= F_LLM
                a = list(u.input_dist.samples)
                b = list(u.output_dist.samples)
                d["a_off"], d["a_len"] = push(a, 1)
                d["b_off"], d["b_len"] = push(b, 2)
                d["pool_off"] = len(pools_off)
                bn = binning(a, u.bucket_count)
                if bn is not None:
                    d["ib_lo"], d["ib_hi"], d["ib_k"] = bn
                if u.masks.output_own_input and len(u.records) > 0 and bn is not None:
                    flags |= F_OWN
                    groups: dict = {}
                    for r in u.records:
                        groups.setdefault(bucket_index(bn, r.input_len), []).append(
                            r.output_len)
                    for kb in range(bn[2]):
                        xs = groups.get(kb, [])
                        o, ln = push(xs, 2) if xs else (0, 0)
                        pools_off.append(o)
                        pools_len.append(ln)
            else:
                d["a_off"], d["a_len"] = push(list(u.duration_dist.samples))
            d["flags"] = flags
            succ = sorted(u.successors.items())
            d["succ_off"] = len(succ_nxt)
            d["succ_len"] = len(succ)
            cum = np.cumsum([p for _, p in succ]) if succ else np.zeros(0)
            succ_cum.extend(cum.tolist() + [0.0])
            succ_nxt.extend([pos[s] for s, _ in succ] + [-1])
            # K3 tables: joined records with every upstream (estimator.py:168-173)
            d["cond_off"] = len(conds)
            ups = [v for v in order if uid in g.units[v].successors]
            for up_id in ups:
                up = g.units[up_id]
                c = np.zeros((), dtype=COND_DTYPE)
                c["up_local"] = pos[up_id]
                dists = [up.input_dist.samples, up.output_dist.samples,
                         up.parallelism_dist.samples]
                bns = [binning(x, up.bucket_count) for x in dists]
                for j, bnj in enumerate(bns):
                    if bnj is not None:
                        c["lo"][j], c["hi"][j], c["k"][j] = bnj
                        c["ok"][j] = 1
                mine = {}
                for r in u.records:
                    mine[r.trial_id] = r
                c["pair_off"] = len(pairs)
                for ur in up.records:
                    if ur.next_unit == uid and ur.trial_id in mine:
                        pr = np.zeros((), dtype=PAIR_DTYPE)
                        for j, (bnj, v) in enumerate(zip(bns, (ur.input_len, ur.output_len,
                                                               float(ur.parallelism)))):
                            pr["bk"][j] = bucket_index(bnj, v) if bnj is not None else -1
                        r = mine[ur.trial_id]
                        pr["in"], pr["out"] = r.input_len, r.output_len
                        pairs.append(pr)
                c["pair_len"] = len(pairs) - int(c["pair_off"])
                conds.append(c)
            d["cond_len"] = len(conds) - int(d["cond_off"])
            units.append(d)
        return {"units": np.array(units, dtype=UNIT_DTYPE) if units else
                np.zeros(0, UNIT_DTYPE),
                "vals": np.asarray(vals, dtype=np.float64),
                "kinds": np.asarray(kinds, dtype=np.int8),
                "pools_off": np.asarray(pools_off, dtype=np.int64),
                "pools_len": np.asarray(pools_len, dtype=np.int64),
                "succ_cum": np.asarray(succ_cum, dtype=np.float64),
                "succ_nxt": np.asarray(succ_nxt, dtype=np.int64),
                "conds": np.array(conds, dtype=COND_DTYPE) if conds else
                np.zeros(0, COND_DTYPE),
                "pairs": np.array(pairs, dtype=PAIR_DTYPE) if pairs else
                np.zeros(0, PAIR_DTYPE),
                "caps": [getattr(g.units[uid], "capacity", 1000) for uid in order]}

    def _place(self) -> None:
        """Concatenate the segments (rebasing their local offsets) and upload."""
        units, vals, po, pl, sc, sn, cs, ps, caps = [], [], [], [], [], [], [], [], []
        kinds = []
        gbase, gn = [], []
        nv = npool = nsucc = ncond = npair = nunit = 0
        for nm in self.names:
            sg = self._segments[nm]
            u = sg["units"].copy()
            llm = (u["flags"] & F_LLM) != 0
            u["a_off"] += nv
            u["b_off"] += np.where(llm, nv, 0).astype(u["b_off"].dtype)
            u["pool_off"] += np.where(llm, npool, 0).astype(u["pool_off"].dtype)
            u["succ_off"] += nsucc
            u["cond_off"] += ncond
            c = sg["conds"].copy()
            c["pair_off"] += npair
            units.append(u)
            vals.append(sg["vals"])
            kinds.append(sg["kinds"])
            po.append(np.where(sg["pools_len"] > 0, sg["pools_off"] + nv, 0))
            pl.append(sg["pools_len"])
            sc.append(sg["succ_cum"])
            sn.append(sg["succ_nxt"])
            cs.append(c)
            ps.append(sg["pairs"])
            caps.extend(sg["caps"])
            gbase.append(nunit)
            gn.append(len(u))
            nv += len(sg["vals"])
            npool += len(sg["pools_off"])
            nsucc += len(sg["succ_nxt"])
            ncond += len(c)
            npair += len(sg["pairs"])
            nunit += len(u)
        cat = lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt)  # noqa: E731
        self.host_kinds = cat(kinds, np.int8)
        self._finish(self.device, cat(units, UNIT_DTYPE), cat(vals, np.float64), gbase, gn,
                     caps, cat(po, np.int64), cat(pl, np.int64), cat(sc, np.float64),
                     cat(sn, np.int64), list(cat(cs, COND_DTYPE)), list(cat(ps, PAIR_DTYPE)))

    @classmethod
    def from_arrays(cls, *, units, vals, graph_base, graph_n, succ_cum, succ_nxt,
                    unit_capacity, device: str = "cuda", names=None, unit_order=None):
        """Bank from pre-built tables (vectorised synthetic workloads); same
        layout the compiler produces.  No K3 records, no own-input pools."""
        self = cls.__new__(cls)
        g = len(graph_base)
        self.empty_units = {}
        self.names = list(names) if names is not None else [str(i) for i in range(g)]
        self.index = {nm: i for i, nm in enumerate(self.names)}
        self.unit_order = unit_order or {}
        self.graphs = {}
        self.device = device
        self.host_kinds = np.zeros(len(vals), dtype=np.int8)
        self._finish(device, units, vals, graph_base, graph_n, unit_capacity, [], [],
                     succ_cum, succ_nxt, [], [])
        return self

    def _finish(self, device, units, vals, gbase, gn, caps, pools_off, pools_len, succ_cum,
                succ_nxt, conds, pairs):
        import torch
        dev = torch.device(device)

        def t(a, dt):
            a = np.asarray(a, dtype=dt)
            if a.size == 0:
                a = np.zeros(1, dtype=dt)
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        self.host_units = units
        self.n_units = len(units)
        self.units = t(units.view(np.uint8).reshape(-1), np.uint8)
        self.vals = t(vals, np.float64)
        kinds = getattr(self, "host_kinds", None)
        self.vals_kind = t(kinds if kinds is not None and len(kinds) == len(vals)
                           else np.zeros(len(vals), np.int8), np.int8)
        self.graph_base = t(gbase, np.int32)
        self.graph_n = t(gn, np.int32)
        self.unit_capacity = t(caps, np.int32)
        self.pool_off = t(pools_off, np.int32)
        self.pool_len = t(pools_len, np.int32)
        self.succ_cum = t(succ_cum, np.float64)
        # integer form of `cum <= u` for u = k * 2^-53: k >= ceil(cum * 2^53)
        # (exact: scaling by 2^53 and ceil are exact for cum in [0, 2))
        cum = np.asarray(succ_cum, dtype=np.float64)
        thr = np.ceil(cum * 2.0 ** 53).astype(np.uint64)
        # every listed successor has probability > 0, so thresholds are >= 1
        # (the engine compares raw words against thr * 2^11 - 1)
        if len(succ_nxt) and np.any(thr[np.asarray(succ_nxt)[:len(thr)] >= 0] == 0):
            raise ValueError("successor with zero branch probability")
        self.succ_thr = t(thr.view(np.int64), np.int64)
        self.succ_nxt = t(succ_nxt, np.int32)
        self.max_units = int(np.max(gn)) if len(gn) else 1
        # unit kinds present (pdg_graph_bank.features: the engine compiles out
        # the paths of absent kinds)
        kinds_present = int(np.bitwise_or.reduce(units["flags"] & (F_LLM | F_OWN | F_ANYMASK))
                            if len(units) else 0)
        self.features = FEATURES_VALID | kinds_present
        self.unit_class = t(unit_classes(units, gbase, gn, succ_cum, succ_nxt), np.uint8)
        ca = np.array(conds, dtype=COND_DTYPE) if len(conds) else np.zeros(1, COND_DTYPE)
        pa = np.array(pairs, dtype=PAIR_DTYPE) if len(pairs) else np.zeros(1, PAIR_DTYPE)
        self.host_conds = ca
        self.conds = t(ca.view(np.uint8).reshape(-1), np.uint8)
        self.pairs = t(pa.view(np.uint8).reshape(-1), np.uint8)
        self.max_unit_k = int(units["ib_k"].max()) if len(units) else 1
        self.max_pairs = int(ca["pair_len"].max())

    def local_unit(self, name: str, uid: str) -> int:
        return self.unit_order[name].index(uid)


def unit_classes(units, gbase, gn, succ_cum, succ_nxt, iters: int = 32) -> np.ndarray:
    """Scheduling hint per unit (pdg_graph_bank.unit_class): the expected
    number of walk steps left from the unit, E[u] = 1 + sum_v p(u->v) E[v]
    over the branch tables (32 value-iteration sweeps, cycles included),
    clipped to classes 0..15.  Speed only: the engine's results do not
    depend on it."""
    nu = len(units)
    if nu == 0:
        return np.zeros(1, np.uint8)
    slen = np.asarray(units["succ_len"], dtype=np.int64)
    soff = np.asarray(units["succ_off"], dtype=np.int64)
    ubase = np.repeat(np.asarray(gbase, dtype=np.int64), np.asarray(gn, dtype=np.int64))[:nu]
    src = np.repeat(np.arange(nu), slen)
    first = np.repeat(np.cumsum(slen) - slen, slen)
    slot = np.arange(len(src)) - first
    pos = soff[src] + slot
    cum = np.asarray(succ_cum, dtype=np.float64)
    nxt = np.asarray(succ_nxt, dtype=np.int64)
    ok = (nxt[pos] >= 0) if len(pos) else np.zeros(0, bool)
    p = cum[pos] - np.where(slot > 0, cum[np.maximum(pos - 1, 0)], 0.0)
    src, dst, p = src[ok], ubase[src[ok]] + nxt[pos[ok]], p[ok]
    e = np.ones(nu)
    for _ in range(iters):
        e = 1.0 + np.bincount(src, weights=p * e[dst], minlength=nu)
    return np.clip(np.floor(e), 0, 15).astype(np.uint8)


# ---------------------------------------------------------------------------
# PCG64 jump-ahead tables (constant): state after j steps = A_j*s + inc*G_j
# ---------------------------------------------------------------------------

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
_M128 = (1 << 128) - 1


def jump_tables() -> np.ndarray:
    """uint64 [3, 1024, 4]: level 0 = j in [0,1024), level 1 = j = 1024*q,
    entry = (A.lo, A.hi, G.lo, G.hi).  Level 2 drives the engine's strided
    decode (lane l reads words l, l+32, ... of a visit's stream segment):
    entry l < 32 = (A'_l, K_l) with A'_l = A_32^-1 A_{l+1} and
    K_l = A_32^-1 (G_{l+1} - G_32), so that the state one stride before word l
    is A'_l s + K_l inc; entry 32 = (A_32, G_32)."""
    out = np.zeros((3, 1024, 4), dtype=np.uint64)
    lo = lambda x: x & (2**64 - 1)  # noqa: E731
    A, G = 1, 0
    for j in range(1024):
        out[0, j] = [lo(A), A >> 64, lo(G), G >> 64]
        A, G = (A * PCG_MULT) & _M128, (G * PCG_MULT + 1) & _M128
    A1024, G1024 = A, G       # one step of level 1
    A, G = 1, 0
    for q in range(1024):
        out[1, q] = [lo(A), A >> 64, lo(G), G >> 64]
        # compose: (A,G) o (A1024,G1024): s -> A1024*(A*s + inc*G) + inc*G1024
        A, G = (A1024 * A) & _M128, (A1024 * G + G1024) & _M128
    a32 = int(out[0, 32, 0]) | (int(out[0, 32, 1]) << 64)
    g32 = int(out[0, 32, 2]) | (int(out[0, 32, 3]) << 64)
    inv = pow(a32, -1, 1 << 128)
    for lane in range(32):
        al = int(out[0, lane + 1, 0]) | (int(out[0, lane + 1, 1]) << 64)
        gl = int(out[0, lane + 1, 2]) | (int(out[0, lane + 1, 3]) << 64)
        ap = (inv * al) & _M128
        kp = (inv * (gl - g32)) & _M128
        out[2, lane] = [lo(ap), ap >> 64, lo(kp), kp >> 64]
    out[2, 32] = [lo(a32), a32 >> 64, lo(g32), g32 >> 64]
    return out
