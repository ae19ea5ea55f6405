"""CPU oracle for the PDGraph scoring hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2506_14851_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may call it, and only as the
checker (or as the timed CPU baseline), never as the product path.

It is a float64 numpy restatement of the reference algorithm
(``/root/reference/pkg/src/pdgsim``, cited as ``file.py:line``).  It consumes
graphs in the reference's own knowledge-base JSON format
(``pdgraph.graph_to_dict`` / ``graph_from_dict``, ``pdgraph.py:304-409``) so
that it runs on the GPU box, where ``/root/reference`` does not exist.

Parity pinning: ``tests/golden/make_golden.py`` runs the *reference itself*
in the build container and records its outputs; ``tests/test_oracle_cpu.py``
checks this restatement against those recordings (bit-exact for the Monte
Carlo engine, binning and prewarm; 1e-12 relative for Gittins).  The Monte
Carlo restatement reproduces the reference's numpy PCG64 call sequence
(``estimator.py:325-353``), so identical seeds give identical samples.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

WALK_VISIT_CAP = 64            # estimator.py:26
MIN_CONDITIONAL_SAMPLES = 5    # estimator.py:25
OVERRUN_PENALTY_FACTOR = 2.0   # sched.py:24


class OracleExhausted(Exception):
    """Mirror of ExhaustedDistributionError (errors.py:16-21)."""


# ---------------------------------------------------------------------------
# a4: equal-width binning over [min, max]   (distributions.py:73-133)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Binning:
    """Result of bucketize() for one sample list (distributions.py:79-105)."""
    lo: float
    hi: float          # sample max
    k: int             # number of buckets (1 when degenerate)
    width: float       # (hi - lo) / k ; 0.0 when degenerate
    counts: np.ndarray  # int64 [k]
    n: int

    @property
    def probs(self) -> np.ndarray:
        # counts[i] / n in float64, as distributions.py:103
        return np.array([c / self.n for c in self.counts.tolist()], dtype=np.float64)

    def edges(self) -> list[tuple[float, float]]:
        if self.k == 1 and self.width == 0.0:
            return [(self.lo, self.hi)]
        return [(self.lo + i * self.width, self.lo + (i + 1) * self.width)
                for i in range(self.k)]

    def midpoints(self) -> np.ndarray:
        # distributions.py:131 -- (lower + upper) / 2.0 per bucket
        return np.array([(a + b) / 2.0 for a, b in self.edges()], dtype=np.float64)

    def boundaries(self) -> list[float]:
        # distributions.py:120-126
        e = self.edges()
        out = [e[0][0]] + [b for _, b in e]
        return [out[0]] if out[0] == out[-1] else out

    def index_of(self, value: float) -> int:
        # distributions.py:107-118: note the width is recomputed from the
        # bucket edges, not from the sample max.
        e = self.edges()
        lo, hi = e[0][0], e[-1][1]
        if hi == lo or value <= lo:
            return 0
        if value >= hi:
            return len(e) - 1
        return min(int((value - lo) / ((hi - lo) / len(e))), len(e) - 1)


def bucketize(samples: Sequence[float], bucket_count: int) -> Binning:
    """distributions.py:79-105 (sample list already FIFO-capped)."""
    xs = [float(s) for s in samples]
    if not xs:
        raise ValueError("cannot bucketize: no data")
    lo, hi = min(xs), max(xs)
    n = len(xs)
    if lo == hi:
        return Binning(lo, hi, 1, 0.0, np.array([n], dtype=np.int64), n)
    k = int(bucket_count)
    w = (hi - lo) / k
    counts = np.zeros(k, dtype=np.int64)
    for s in xs:
        j = int((s - lo) / w)
        counts[min(j, k - 1)] += 1
    return Binning(lo, hi, k, w, counts, n)


def survival(samples: Sequence[float], x: float) -> float:
    """P(X >= x) over the samples (distributions.py:73-77)."""
    if len(samples) == 0:
        return 0.0
    return sum(1 for s in samples if s >= x) / len(samples)


# ---------------------------------------------------------------------------
# a1 / a3: Gittins rank (sched.py:51-129)
# ---------------------------------------------------------------------------

def gittins_rank_batch(values, probs, ages) -> np.ndarray:
    """Vectorised Gittins rank, NaN when exhausted (sched.py:102-129)."""
    v = np.asarray(values, dtype=np.float64)
    p = np.asarray(probs, dtype=np.float64)
    a = np.asarray(ages, dtype=np.float64)
    d = v - a[:, None]
    live = d > 0
    m = np.where(live, p, 0.0)
    z = m.sum(axis=1)
    dead = z <= 0
    c = m / np.where(dead, 1.0, z)[:, None]
    cp = np.cumsum(c, axis=1)
    dl = np.where(live, d, 0.0)
    cpv = np.cumsum(c * dl, axis=1)
    num = cpv + dl * (1.0 - cp)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = num / cp
    r = np.where(live & (cp > 0), r, np.inf)
    out = r.min(axis=1)
    return np.where(dead, np.nan, out)


def gittins_rank_samples(samples: Sequence[float], age: float) -> float:
    """Scalar sample-form rank over distinct support offsets (sched.py:51-85)."""
    tail = sorted(s - age for s in samples if s > age)
    if not tail:
        raise OracleExhausted(age)
    n = len(tail)
    if tail[0] == tail[-1]:
        return tail[0]
    best, acc, i = math.inf, 0.0, 0
    while i < n:
        j = i
        while j < n and tail[j] == tail[i]:
            acc += tail[j]
            j += 1
        best = min(best, (acc + tail[i] * (n - j)) / j)
        i = j
    return best


def refresh_keys(rows_values: Sequence[np.ndarray], rows_probs: Sequence[np.ndarray],
                 ages: Sequence[float],
                 penalty: float = OVERRUN_PENALTY_FACTOR) -> tuple[np.ndarray, np.ndarray]:
    """Batched refresh: ragged pad + rank + overrun penalty (sched.py:271-300).

    Returns (keys float64 [m], overrun bool [m]).
    """
    m = len(rows_values)
    widths = [len(r) for r in rows_values]
    width = max(widths)
    vals = np.zeros((m, width))
    prbs = np.zeros((m, width))
    for i, (rv, rp) in enumerate(zip(rows_values, rows_probs)):
        k = len(rv)
        vals[i, :k] = rv
        prbs[i, :k] = rp
        if k < width:
            vals[i, k:] = vals[i, k - 1]
    a = np.asarray(ages, dtype=np.float64)
    r = gittins_rank_batch(vals, prbs, a)
    bad = np.isnan(r)
    return np.where(bad, a * penalty, r), bad


# ---------------------------------------------------------------------------
# the other demand-aware keys (sched.py:132-140, 217-225)
# ---------------------------------------------------------------------------

def py_sum(xs: Sequence[float]) -> float:
    """Python's built-in ``sum`` over floats, as RemainingDemand.mean() calls
    it (estimator.py:55-56).  CPython >= 3.12 (the interpreter the reference
    runs on here) compensates with Neumaier's algorithm
    (Python/bltinmodule.c, builtin_sum_impl): the running total starts as
    0 + x0, each further x adds its rounding error to c, and c is added at
    the end when it is non-zero and finite."""
    it = iter(xs)
    try:
        f = 0 + next(it)
    except StopIteration:
        return 0
    c = 0.0
    for x in it:
        t = f + x
        if abs(f) >= abs(x):
            c += (f - t) + x
        else:
            c += (x - t) + f
        f = t
    if c and math.isfinite(c):
        f += c
    return f


def srpt_mean_key(samples: Sequence[float], attained: float, estimate_age: float) -> float:
    """compute_priority(SRPT_MEAN) (sched.py:216-218)."""
    served_since = attained - estimate_age
    return py_sum(samples) / len(samples) - served_since


def lstf_key(samples: Sequence[float], attained: float, estimate_age: float,
             deadline: float, now: float) -> float:
    """compute_priority(LSTF) (sched.py:219-224) -> lstf_slack (132-140)."""
    total = [s + estimate_age for s in samples]
    return deadline - now - (max(total) - attained)


# ---------------------------------------------------------------------------
# dispatch / preemption on one PriorityRefresh
# (simcore.py:636-644 -> _preempt 652-687, _dispatch 512-516)
# ---------------------------------------------------------------------------

def plan_dispatch(backend, active, key, app_rank, stage, request, slots, hysteresis=1.5,
                  preempt=True):
    """Events [(kind, task)] (kind 1 = preempt, 2 = start) in the order the
    simulator applies them: preemption swaps of every backend, then the
    dispatch fill of every backend.  Task order = _task_sort_key
    (simcore.py:339-344) with (arrival_time, app_instance_id) as app_rank."""
    nb = len(slots)
    tup = lambda t: (key[t], app_rank[t], stage[t], request[t])  # noqa: E731
    queue = [[t for t in range(len(backend)) if backend[t] == b and not active[t]]
             for b in range(nb)]
    act = [[t for t in range(len(backend)) if backend[t] == b and active[t]]
           for b in range(nb)]
    ev = []
    if preempt:
        for b in range(nb):
            if not queue[b]:
                continue
            changed = True
            while changed:
                changed = False
                if not queue[b] or not act[b]:
                    break
                w = min(queue[b], key=tup)
                x = max(act[b], key=tup)
                if key[x] > key[w] * hysteresis and key[x] > key[w]:
                    act[b].remove(x)
                    queue[b].append(x)
                    act[b].append(w)
                    queue[b].remove(w)
                    ev += [(1, x), (2, w)]
                    changed = True
    for b in range(nb):
        while queue[b] and len(act[b]) < slots[b]:
            w = min(queue[b], key=tup)
            queue[b].remove(w)
            act[b].append(w)
            ev.append((2, w))
    return ev


# ---------------------------------------------------------------------------
# correlation masks (estimator.py:62-142)
# ---------------------------------------------------------------------------

MASK_NAMES = ("input_upstream_input", "input_upstream_output", "output_upstream_output",
              "output_own_input", "parallelism_upstream_parallelism")


def pearson(x: Sequence[float], y: Sequence[float]) -> Optional[float]:
    """estimator.pearson (62-81) in the reference's own float operations
    (CPython sum(), ** 2, math.sqrt); None where it raises."""
    if len(x) != len(y) or len(x) < 2:
        return None
    n = len(x)
    mx = py_sum(x) / n
    my = py_sum(y) / n
    sxx = py_sum([(a - mx) ** 2 for a in x])
    syy = py_sum([(b - my) ** 2 for b in y])
    if sxx == 0 or syy == 0:
        return None
    sxy = py_sum([(a - mx) * (b - my) for a, b in zip(x, y)])
    return max(-1.0, min(1.0, sxy / math.sqrt(sxx * syy)))


def mask_jobs(g: "OGraph"):
    """The (unit, mask, xs, ys) pairs build_masks correlates (estimator.py:
    108-142): joined (upstream record, unit record) pairs on trial_id, in
    upstream order (sorted ids) then record order (_joined_pairs, 84-95)."""
    jobs = []
    for uid in sorted(g.units):
        u = g.units[uid]
        ups = [v for v in sorted(g.units) if any(r.next_unit == uid for r in g.units[v].records)]
        own = ([r.output_len for r in u.records], [r.input_len for r in u.records])
        if not ups:
            jobs.append((uid, "output_own_input") + own)
            continue
        by_trial = {r.trial_id: r for r in u.records}
        pairs = [(ur, by_trial[ur.trial_id]) for v in ups for ur in g.units[v].records
                 if ur.next_unit == uid and ur.trial_id in by_trial]
        up_in = [p[0].input_len for p in pairs]
        up_out = [p[0].output_len for p in pairs]
        up_par = [float(p[0].parallelism) for p in pairs]
        my_in = [p[1].input_len for p in pairs]
        my_out = [p[1].output_len for p in pairs]
        my_par = [float(p[1].parallelism) for p in pairs]
        jobs += [(uid, "input_upstream_input", my_in, up_in),
                 (uid, "input_upstream_output", my_in, up_out),
                 (uid, "output_upstream_output", my_out, up_out),
                 (uid, "output_own_input") + own,
                 (uid, "parallelism_upstream_parallelism", my_par, up_par)]
    return jobs


def build_masks(g: "OGraph", threshold: float = 0.5) -> dict:
    """uid -> {mask: bool} as estimator.build_masks sets them (_flag, 97-105:
    fewer than 2 points or an undefined correlation -> False)."""
    out = {uid: {k: False for k in MASK_NAMES} for uid in g.units}
    for uid, name, xs, ys in mask_jobs(g):
        r = pearson(xs, ys)
        out[uid][name] = r is not None and abs(r) > threshold
    return out


# ---------------------------------------------------------------------------
# a10: prewarm planner (prewarm.py:42-96)
# ---------------------------------------------------------------------------

def plan_prewarm(completion_samples: Sequence[float], bucket_count: int,
                 p_s: float, t_p: float, knob: float,
                 now: float) -> Optional[tuple[float, float]]:
    """Latest-safe trigger; returns (trigger_time, p_e) or None."""
    if not (0.0 <= knob <= 1.0):
        raise ValueError("knob")
    if t_p < 0:
        raise ValueError("t_p")
    if p_s < knob:
        return None
    live = [float(s) for s in completion_samples if s > now]
    if not live:
        live = [float(s) for s in completion_samples]
    grid = bucketize(live, bucket_count).boundaries()
    cands = sorted({max(b - t_p, now) for b in grid} | {now}, reverse=True)
    for t_s in cands:
        pe = p_s * survival(live, t_s + t_p)
        if pe >= knob:
            return t_s, pe
    return now, p_s * survival(live, now + t_p)


# ---------------------------------------------------------------------------
# Graph model over the knowledge-base JSON (pdgraph.py:79-244, 304-409)
# ---------------------------------------------------------------------------

@dataclass
class ORecord:
    trial_id: int
    input_len: float
    output_len: float
    parallelism: int
    duration: float
    next_unit: Optional[str]


@dataclass
class OUnit:
    uid: str
    is_llm: bool
    capacity: int
    bucket_count: int
    records: list
    masks: dict
    warmup_time: float = 0.0
    warm_content: Optional[str] = None
    succ: dict = field(default_factory=dict)

    # FIFO-capped per-variable sample lists (pdgraph.py:162-170)
    def samples(self, var: str) -> list[float]:
        if self.is_llm:
            if var == "input":
                return [r.input_len for r in self.records]
            if var == "output":
                return [r.output_len for r in self.records]
            if var == "parallelism":
                return [float(r.parallelism) for r in self.records]
            return []
        return [r.duration for r in self.records] if var == "duration" else []

    def binning(self, var: str) -> Optional[Binning]:
        xs = self.samples(var)
        return bucketize(xs, self.bucket_count) if xs else None

    def any_mask(self) -> bool:
        return any(bool(v) for v in self.masks.values())


@dataclass
class OGraph:
    app_id: str
    entry: str
    units: dict


def graph_from_kb(doc: dict) -> OGraph:
    """Rebuild a graph from knowledge-base JSON (pdgraph.py:344-409)."""
    units = {}
    for u in doc["units"]:
        b = u["backend"]
        kind = b.get("kind")
        is_llm = kind == "llm-inference"
        cap = int(u.get("capacity", 1000))
        recs = deque(maxlen=cap)
        for r in u.get("records", []):
            recs.append(ORecord(int(r["trial_id"]), float(r.get("input_len", 0.0)),
                                float(r.get("output_len", 0.0)),
                                int(r.get("parallelism", 1)),
                                float(r.get("duration", 0.0)), r.get("next_unit")))
        if is_llm:
            warm = b.get("kv_prefix_id") or b.get("lora_id")
        elif kind == "docker-exec":
            warm = b.get("image_id")
        else:
            warm = b.get("tool_id")
        unit = OUnit(u["unit_id"], is_llm, cap, int(u.get("bucket_count", 10)),
                     list(recs), dict(u.get("masks", {})),
                     float(b.get("warmup_time", 0.0)), warm)
        # pdgraph.py:182-194: frequency over all (capped) records
        cnt: dict = {}
        for r in unit.records:
            if r.next_unit is not None:
                cnt[r.next_unit] = cnt.get(r.next_unit, 0) + 1
        tot = len(unit.records)
        unit.succ = {k: c / tot for k, c in sorted(cnt.items())} if tot else {}
        units[unit.uid] = unit
    return OGraph(doc["app_id"], doc["entry_unit"], units)


@dataclass(frozen=True)
class OObs:
    unit_id: str
    input_len: float = 0.0
    output_len: float = 0.0
    parallelism: int = 1


# ---------------------------------------------------------------------------
# a7: one-hop conditioning (estimator.py:155-233, 289-302)
# ---------------------------------------------------------------------------

@dataclass
class OOverride:
    input_vals: list
    output_vals: list
    conditioned: bool


def _filtered(unit: OUnit, up: OUnit, obs: OObs, target: str,
              conds: list) -> tuple[Optional[list], bool]:
    """Kept target values, or (None, False) for the prior (estimator.py:184-206)."""
    if not conds:
        return None, False
    mine = {}
    for r in unit.records:
        mine[r.trial_id] = r
    pairs = [(ur, mine[ur.trial_id]) for ur in up.records
             if ur.next_unit == unit.uid and ur.trial_id in mine]
    if not pairs:
        return None, False
    kept = []
    for ur, r in pairs:
        ok = True
        for attr, val, bn in conds:
            if bn is None or bn.index_of(getattr(ur, attr)) != bn.index_of(val):
                ok = False
                break
        if ok:
            kept.append(getattr(r, target))
    if len(kept) < MIN_CONDITIONAL_SAMPLES:
        return None, False
    return list(deque(kept, maxlen=unit.capacity)), True


def conditioning_for(g: OGraph, current: str,
                     observations: Sequence[OObs]) -> Optional[OOverride]:
    """estimator.py:289-302 + conditional_filter 155-233."""
    unit = g.units[current]
    for obs in reversed(list(observations)):
        up = g.units.get(obs.unit_id)
        if up is None or current not in up.succ:
            continue
        if not unit.any_mask():
            return None
        m = unit.masks
        in_c, out_c, par_c = [], [], []
        if m.get("input_upstream_input"):
            in_c.append(("input_len", obs.input_len, up.binning("input")))
        if m.get("input_upstream_output"):
            in_c.append(("output_len", obs.output_len, up.binning("output")))
        if m.get("output_upstream_output"):
            out_c.append(("output_len", obs.output_len, up.binning("output")))
        if m.get("parallelism_upstream_parallelism"):
            par_c.append(("parallelism", float(obs.parallelism),
                          up.binning("parallelism")))
        iv, ic = _filtered(unit, up, obs, "input_len", in_c)
        ov, oc = _filtered(unit, up, obs, "output_len", out_c)
        _, pc = _filtered(unit, up, obs, "parallelism", par_c)
        return OOverride(iv if iv is not None else unit.samples("input"),
                         ov if ov is not None else unit.samples("output"),
                         ic or oc or pc)
    return None


# ---------------------------------------------------------------------------
# a5 / a6 / a8: Monte Carlo remaining demand (estimator.py:236-362)
# ---------------------------------------------------------------------------

class _Stage:
    """Per-unit stage-time sampler with the reference's draw order
    (estimator.py:236-286)."""

    def __init__(self, unit: OUnit, prefill: float, decode: float,
                 ov: Optional[OOverride]):
        self.llm = unit.is_llm
        self.prefill, self.decode = prefill, decode
        self.pools = None
        if self.llm:
            iv = ov.input_vals if ov is not None else unit.samples("input")
            ovl = ov.output_vals if ov is not None else unit.samples("output")
            if not iv or not ovl:
                raise ValueError(f"unit {unit.uid!r} has no token-length samples")
            self.iv = np.asarray(iv, dtype=np.float64)
            self.ov = np.asarray(ovl, dtype=np.float64)
            if unit.masks.get("output_own_input") and ov is None and unit.records:
                self.bins = unit.binning("input")
                grp: dict = {}
                for r in unit.records:
                    grp.setdefault(self.bins.index_of(r.input_len), []).append(r.output_len)
                self.pools = {b: np.asarray(x, dtype=np.float64) for b, x in grp.items()}
        else:
            dv = unit.samples("duration")
            if not dv:
                raise ValueError(f"unit {unit.uid!r} has no duration samples")
            self.dv = np.asarray(dv, dtype=np.float64)

    def draw(self, m: int, rng: np.random.Generator) -> np.ndarray:
        if not self.llm:
            return rng.choice(self.dv, size=m)
        i = rng.choice(self.iv, size=m)
        if self.pools is None:
            o = rng.choice(self.ov, size=m)
        else:
            o = np.empty(m)
            key = np.array([self.bins.index_of(x) for x in i])
            for b in np.unique(key):
                sel = key == b
                pool = self.pools.get(int(b))
                if pool is None or len(pool) == 0:
                    pool = self.ov
                o[sel] = rng.choice(pool, size=int(sel.sum()))
        return i / self.prefill + o / self.decode


@dataclass
class OMC:
    samples: np.ndarray
    conditioned: bool
    capped: int


def mc_remaining_demand(g: OGraph, current: str, observations: Sequence[OObs],
                        n: int, seed: int, visit_cap: int = WALK_VISIT_CAP,
                        prefill: float = 10000.0, decode: float = 50.0) -> OMC:
    """n random walks from ``current`` (estimator.py:305-362).

    Walk bookkeeping mirrors the reference: per outer step the set of
    occupied units is fixed first; units are then visited in ascending
    sorted-id order, each taking every walk that sits on it *at that
    moment* (so a walk that moves to a later unit in the same step is
    visited again in that step).
    """
    if n < 1:
        raise ValueError("n")
    if current not in g.units:
        raise KeyError(current)
    rng = np.random.default_rng(seed)
    order = sorted(g.units)
    pos = {u: i for i, u in enumerate(order)}
    ov = conditioning_for(g, current, observations)
    stages, tables = [], []
    for u in order:
        unit = g.units[u]
        stages.append(_Stage(unit, prefill, decode, ov if u == current else None))
        succ = sorted(unit.succ.items())
        cum = np.cumsum([p for _, p in succ])
        nxt = np.array([pos[s] for s, _ in succ] + [-1], dtype=np.int64)
        tables.append((cum, nxt))
    where = np.full(n, pos[current], dtype=np.int64)
    acc = np.zeros(n)
    for _ in range(visit_cap):
        alive = where >= 0
        if not alive.any():
            break
        for ui in np.unique(where[alive]):
            idx = np.flatnonzero(where == ui)
            acc[idx] += stages[ui].draw(len(idx), rng)
            cum, nxt = tables[ui]
            u = rng.random(len(idx))
            where[idx] = nxt[np.searchsorted(cum, u, side="right")] if len(cum) else -1
    return OMC(acc, bool(ov is not None and ov.conditioned), int((where >= 0).sum()))


def unit_service_samples(unit: OUnit, prefill: float = 10000.0,
                         decode: float = 50.0) -> list[float]:
    """Unconditioned stage times for prewarm (simcore.py:480-487, pdgraph.py:294-298)."""
    if unit.is_llm:
        return [r.input_len / prefill + r.output_len / decode for r in unit.records]
    return unit.samples("duration")


# ---------------------------------------------------------------------------
# a12: exact expected remaining demand for acyclic graphs (estimator.py:377-422)
# ---------------------------------------------------------------------------

def exact_mean(g: OGraph, current: str, prefill: float = 10000.0,
               decode: float = 50.0) -> float:
    memo: dict = {}
    busy: set = set()

    def stage_mean(u: OUnit) -> float:
        if u.is_llm:
            iv, ov = u.samples("input"), u.samples("output")
            mi = sum(iv) / len(iv)
            mo = sum(ov) / len(ov)
            return mi / prefill + mo / decode
        dv = u.samples("duration")
        return sum(dv) / len(dv)

    def rec(uid: str) -> float:
        if uid in memo:
            return memo[uid]
        if uid in busy:
            raise ValueError(f"cycle at {uid}")
        busy.add(uid)
        e = stage_mean(g.units[uid])
        for s, p in sorted(g.units[uid].succ.items()):
            if p > 0.0:
                e += p * rec(s)
        busy.discard(uid)
        memo[uid] = e
        return e

    return rec(current)


# ---------------------------------------------------------------------------
# config 5: need probability per backend type and window (derived from
# plan_prewarm's completion distribution, prewarm.py:65-67, simcore.py:450-487)
# ---------------------------------------------------------------------------

def need_grid(svc_samples: Sequence[float], successors: Sequence[tuple], now: float,
              windows: Sequence[float], n_types: int) -> np.ndarray:
    """need[t, k] = sum_{(p_s, type) in successors, type == t} p_s * P(C < now + W_k),
    C = now + s conditioned on C > now (all samples if none), P(C < x) =
    1 - survival(x)."""
    comp = [now + s for s in svc_samples]
    live = [c for c in comp if c > now] or comp
    out = np.zeros((n_types, len(windows)))
    for k, wk in enumerate(windows):
        pneed = 1.0 - survival(live, now + wk) if live else 0.0
        for p_s, t in successors:
            if t is not None and t >= 0:
                out[t, k] += p_s * pneed
    return out


# ---------------------------------------------------------------------------
# a11b: Simulator._update_attained (simcore.py:306-313)
# ---------------------------------------------------------------------------

def update_attained(completed: Sequence[float], progress: Sequence[float],
                    tasks: Sequence[tuple], now: float) -> list:
    """attained[a] = completed[a] + max(progress[a], min(service, max(0, now -
    (start + cold)))) over the active tasks (app, start, cold, service) of
    app a with start not None, in the reference's operation order."""
    prog = list(progress)
    for a, start, cold, service in tasks:
        if start is None:
            continue
        run = max(0.0, now - (start + cold))
        prog[a] = max(prog[a], min(service, run))
    return [c + p for c, p in zip(completed, prog)]
