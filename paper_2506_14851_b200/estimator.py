"""GPU demand engine: drop-in for ``pdgsim.estimator.monte_carlo_remaining_demand``
(estimator.py:305-362) and the batched, device-resident form behind it.

``DemandEngine.run`` estimates many applications in one launch (one warp per
application, kernel ``mc_engine_kernel``); each job is (graph, current unit,
relevant observation, seed).  Outputs are the raw samples (optional) and the
``set_remaining`` histogram rows (bucket grid + u16 counts) written straight
into a :class:`~paper_2506_14851_b200.queue.HistQueue`, where K1 scores them.

The drop-in ``monte_carlo_remaining_demand`` keeps the reference signature and
returns a ``RemainingDemand`` whose samples are bit-identical to the
reference's for the same inputs.
"""

from __future__ import annotations

import ctypes as C
import weakref
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import EstimationError
from .graphs import GraphBank, jump_tables

WALK_VISIT_CAP = 64


class GraphBankC(C.Structure):
    _fields_ = [("units", C.c_void_p), ("graph_base", C.c_void_p), ("graph_n", C.c_void_p),
                ("unit_capacity", C.c_void_p), ("vals", C.c_void_p),
                ("pool_off", C.c_void_p), ("pool_len", C.c_void_p),
                ("succ_cum", C.c_void_p), ("succ_nxt", C.c_void_p), ("conds", C.c_void_p),
                ("pairs", C.c_void_p), ("jump", C.c_void_p), ("prefill_rate", C.c_double),
                ("decode_rate", C.c_double), ("succ_thr", C.c_void_p), ("max_units", C.c_int32),
                ("vals_div", C.c_void_p), ("features", C.c_int32),
                ("unit_class", C.c_void_p)]


class JobsC(C.Structure):
    _fields_ = [("graph", C.c_void_p), ("unit", C.c_void_p), ("seed", C.c_void_p),
                ("obs_unit", C.c_void_p), ("obs_val", C.c_void_p)]


class OutC(C.Structure):
    _fields_ = [("samples", C.c_void_p), ("samples_stride", C.c_int64), ("lo", C.c_void_p),
                ("width", C.c_void_p), ("nbins", C.c_void_p), ("nsamp", C.c_void_p),
                ("counts", C.c_void_p), ("stride", C.c_int64), ("slot", C.c_void_p),
                ("capped", C.c_void_p), ("flags", C.c_void_p), ("mean", C.c_void_p),
                ("worst", C.c_void_p)]


_JUMP = {}


def _jump_tensor(device) -> torch.Tensor:
    key = str(device)
    if key not in _JUMP:
        _JUMP[key] = torch.from_numpy(jump_tables().view(np.int64).reshape(-1).copy()).to(device)
    return _JUMP[key]


@dataclass
class RemainingDemand:
    """Mirror of the reference result type (estimator.py:40-59), used when the
    reference package is not loaded; ``integration.patch_pdgsim`` switches
    the drop-in to the reference's own class (``RESULT_TYPE``), so helpers
    that dispatch on it (sched._samples_of, sched.py:45-48) behave unchanged."""
    samples: list
    sample_count: int
    conditioned: bool = False
    capped_walks: int = 0
    hist: Optional[tuple] = field(default=None, repr=False)   # (lo, width, k, counts) from the GPU

    def __post_init__(self):
        if self.sample_count != len(self.samples) or self.sample_count <= 0:
            raise EstimationError("sample_count must equal len(samples) and be > 0")
        if any(s < 0 for s in self.samples):
            raise EstimationError("remaining-demand samples must be >= 0")

    def __iter__(self):
        return iter(self.samples)

    def __len__(self) -> int:
        return self.sample_count

    def mean(self) -> float:
        return sum(self.samples) / self.sample_count

    def max(self) -> float:
        return max(self.samples)


RESULT_TYPE = RemainingDemand       # rebound to pdgsim.estimator.RemainingDemand by patch_pdgsim


class DemandEngine:
    """Resident graph bank + launch wrapper for K2/K3/a4."""

    def __init__(self, graphs, prefill_rate: float = 10000.0, decode_rate: float = 50.0,
                 device: str = "cuda"):
        """graphs: dict name -> graph (reference PDGraph or KBGraph), or a
        prebuilt GraphBank."""
        _lib.lib()
        self.device = torch.device(device)
        self.bank = graphs if isinstance(graphs, GraphBank) else GraphBank(graphs, device=device)
        self.jump = _jump_tensor(self.device)
        self._rates = (float(prefill_rate), float(decode_rate))
        self._bind()
        self._scratch = None
        self._one = {}                  # n -> (pinned host, device, view) for run_one

    def refresh(self, name: str, graph=None) -> None:
        """Template refresh after profiling trials were recorded into graph
        `name` (graphs.record_trial / pdgraph.record_trial): recompile that
        graph's tables and re-bind the device pointers."""
        self.bank.update(name, graph)
        self._bind()

    def _bind(self):
        b = self.bank
        prefill_rate, decode_rate = self._rates
        # pool values divided by their rate once (i/prefill, o/decode: the
        # reference's own per-draw divisions, estimator.py:286, so exact)
        # (tensor / tensor: torch turns division by a scalar into a
        # multiplication by its reciprocal, which is not the same rounding)
        k = b.vals_kind
        pre = torch.full_like(b.vals, prefill_rate)
        dec = torch.full_like(b.vals, decode_rate)
        self.vals_div = torch.where(k == 1, b.vals / pre, torch.where(k == 2, b.vals / dec,
                                                                      b.vals))
        self.c_bank = GraphBankC(
            _lib.ptr(b.units), _lib.ptr(b.graph_base), _lib.ptr(b.graph_n),
            _lib.ptr(b.unit_capacity), _lib.ptr(b.vals), _lib.ptr(b.pool_off),
            _lib.ptr(b.pool_len), _lib.ptr(b.succ_cum), _lib.ptr(b.succ_nxt),
            _lib.ptr(b.conds), _lib.ptr(b.pairs), _lib.ptr(self.jump),
            float(prefill_rate), float(decode_rate), _lib.ptr(b.succ_thr), int(b.max_units),
            _lib.ptr(self.vals_div), int(b.features), _lib.ptr(b.unit_class))
        self.max_unit_k = b.max_unit_k
        self.max_pairs = b.max_pairs

    # -- job marshalling ------------------------------------------------------
    def relevant_observation(self, name: str, current: str, observations) -> tuple[int, tuple]:
        """Latest observation whose unit lists `current` as a successor
        (estimator.py:295-298); returns (local upstream index or -1, values)."""
        g = self.bank.graphs[name]
        for obs in reversed(list(observations)):
            up = g.units.get(obs.unit_id)
            if up is None or current not in up.successors:
                continue
            return (self.bank.local_unit(name, obs.unit_id),
                    (float(obs.input_len), float(obs.output_len), float(obs.parallelism)))
        return -1, (0.0, 0.0, 0.0)

    def _scratch_for(self, n: int, n_jobs: int) -> torch.Tensor:
        L = _lib.lib()
        need = int(L.pdg_mc_scratch_bytes(n, self.max_pairs, L.pdg_mc_grid_warps())) + 8 * n_jobs
        if self._scratch is None or self._scratch.numel() < need:
            self._scratch = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
        return self._scratch

    def run(self, graph_idx, unit_idx, seeds, obs_unit=None, obs_val=None, *, n: int,
            bucket_count: int, visit_cap: int = WALK_VISIT_CAP, queue=None, slots=None,
            samples: bool = False, mean: bool = False, stream=None):
        """Launch the engine on device-resident job arrays (torch tensors).

        Writes histogram rows into `queue` (HistQueue) at `slots` (default:
        rows 0..N-1), plus each row's worst case (max sample) and, with
        mean=True, RemainingDemand.mean() for the SRPT-mean / LSTF keys.  Returns dict(samples=[N,n] f64 or None, capped, flags).
        """
        if n < 1:
            raise EstimationError(f"sample count must be >= 1, got {n}")
        if queue is not None and n > 65535:
            raise EstimationError("u16 histogram counts need n <= 65535")
        N = int(graph_idx.numel())
        dev = self.device
        if self.bank.empty_units:
            # the reference builds a sampler for every unit and raises before
            # walking (estimator.py:246-268): reject jobs on such graphs
            bad = {self.bank.index[nm] for nm in self.bank.empty_units}
            used = set(graph_idx.cpu().tolist())
            hit = sorted(bad & used)
            if hit:
                nm = self.bank.names[hit[0]]
                raise EstimationError(self.bank.empty_units[nm][0][1])
        out_samples = torch.empty((N, n), dtype=torch.float64, device=dev) if samples else None
        capped = torch.empty(N, dtype=torch.int32, device=dev)
        flags = torch.empty(N, dtype=torch.uint8, device=dev)
        if queue is None:
            from .queue import HistQueue
            queue = HistQueue(max(N, 1), max(bucket_count, 1), device=str(dev))
        if bucket_count > queue.stride:
            raise ValueError("queue rows narrower than bucket_count")
        jobs = JobsC(_lib.ptr(graph_idx), _lib.ptr(unit_idx), _lib.ptr(seeds),
                     _lib.ptr(obs_unit), _lib.ptr(obs_val))
        out = OutC(_lib.ptr(out_samples), n, _lib.ptr(queue.lo), _lib.ptr(queue.width),
                   _lib.ptr(queue.nbins), _lib.ptr(queue.nsamp), _lib.ptr(queue.counts),
                   queue.stride, _lib.ptr(slots), _lib.ptr(capped), _lib.ptr(flags),
                   _lib.ptr(queue.mean) if mean else None, _lib.ptr(queue.worst))
        scratch = self._scratch_for(n, N)
        L = _lib.lib()
        _lib.check(L.pdg_mc_remaining_demand(
            C.byref(self.c_bank), C.byref(jobs), N, n, visit_cap, bucket_count,
            self.max_unit_k, self.max_pairs, C.byref(out), _lib.ptr(scratch),
            scratch.numel(), _lib.stream_ptr(stream)), "pdg_mc_remaining_demand")
        if slots is None:
            queue.n = max(queue.n, N)
        return {"samples": out_samples, "capped": capped, "flags": flags, "queue": queue}


    def run_one(self, name: str, unit_local: int, seed: int, obs_up: int, obs_vals,
                n: int, visit_cap: int = WALK_VISIT_CAP):
        """One application, host values in and out (the drop-in's call): the
        job record goes up and the samples, capped count and flags come back
        through one reused pinned staging buffer -- one upload, one launch, one
        download, one synchronisation.  Returns (samples f64[n] numpy view of
        the staging buffer, capped, flags); copy the samples before the next
        call."""
        if n < 1:
            raise EstimationError(f"sample count must be >= 1, got {n}")
        if name in self.bank.empty_units:
            raise EstimationError(self.bank.empty_units[name][0][1])
        st = self._one.get(n)
        if st is None:
            nbytes = 64 + 8 * n + 16
            h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
            d = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)   # padding read back too
            hv = h.numpy()
            st = self._one[n] = (h, d, hv)
        h, d, hv = st
        base = _lib.ptr(d)
        job = hv[:64]
        job[0:16].view(np.int32)[:] = (self.bank.index[name], unit_local, obs_up, 0)
        job[16:24].view(np.int64)[0] = int(seed)
        job[24:48].view(np.float64)[:] = obs_vals
        stream = torch.cuda.current_stream(self.device)
        d[:64].copy_(h[:64], non_blocking=True)
        jobs = JobsC(base, base + 4, base + 16, base + 8, base + 24)
        out = OutC(base + 64, n, None, None, None, None, None, 1, None, base + 64 + 8 * n,
                   base + 68 + 8 * n, None, None)
        scratch = self._scratch_for(n, 1)
        L = _lib.lib()
        _lib.check(L.pdg_mc_remaining_demand(
            C.byref(self.c_bank), C.byref(jobs), 1, n, visit_cap, 1, self.max_unit_k,
            self.max_pairs, C.byref(out), _lib.ptr(scratch), scratch.numel(),
            _lib.stream_ptr(stream)), "pdg_mc_remaining_demand")
        d2 = d[64:]
        h[64:].copy_(d2, non_blocking=True)
        stream.synchronize()
        tail = hv[64 + 8 * n:]
        return (hv[64:64 + 8 * n].view(np.float64), int(tail[:4].view(np.int32)[0]),
                int(tail[4]))


# ---------------------------------------------------------------------------
# drop-in single-application API (estimator.py:305-362)
# ---------------------------------------------------------------------------

# One engine per live graph object.  The cache holds the graph weakly (an
# entry dies with its graph, so a recycled id() can never alias it) and is
# bounded (least recently used first out).  Each hit re-checks a fingerprint
# of everything the device tables are compiled from, so in-place mutation is
# seen: a FIFO-capped record append (pdgraph.py:162-169 -- the deque length
# stays at capacity but its first and last record objects change), a
# build_masks pass (estimator.py:108-142 -- mask flags set in place), or a
# direct append to a unit's sample distribution.
_ENGINES: "OrderedDict[int, tuple]" = OrderedDict()
MAX_ENGINES = 64


def _tail_id(seq) -> tuple:
    n = len(seq)
    return (n, id(seq[0]), id(seq[-1])) if n else (0, 0, 0)


def _dist_fp(d) -> tuple:
    raw = getattr(d, "_samples", None)
    if raw is None:
        raw = getattr(d, "samples", ())
    n = len(raw)
    return (n, raw[0], raw[-1]) if n else (0,)


def _mask_fp(m) -> tuple:
    if m is None:
        return ()
    if isinstance(m, dict):
        return tuple(sorted((k, bool(v)) for k, v in m.items()))
    return tuple(sorted((k, bool(v)) for k, v in vars(m).items()))


def _fingerprint(graph) -> tuple:
    """Cheap content fingerprint: per unit the record container and its
    first/last record identities (a record object in the deque stays alive,
    so a new last record always has a new identity), the last record's
    fields, the per-variable sample lists' length and end values, mask
    flags, successor probabilities, bucket count and capacity."""
    out = []
    for uid, u in sorted(graph.units.items()):
        recs = u.records
        last = recs[-1] if len(recs) else None
        out.append((uid, id(recs), _tail_id(recs),
                    None if last is None else (last.trial_id, last.input_len, last.output_len,
                                               last.parallelism, last.duration,
                                               last.next_unit),
                    _dist_fp(u.input_dist), _dist_fp(u.output_dist),
                    _dist_fp(u.parallelism_dist), _dist_fp(u.duration_dist),
                    _mask_fp(getattr(u, "masks", None)),
                    tuple(sorted(u.successors.items())),
                    getattr(u, "bucket_count", None), getattr(u, "capacity", None),
                    bool(u.is_llm)))
    return (getattr(graph, "entry_unit", None), tuple(out))


def _forget(key, ref):
    hit = _ENGINES.get(key)
    if hit is not None and hit[0] is ref:
        del _ENGINES[key]


def engine_for(graph, env) -> tuple[DemandEngine, str]:
    rates = (float(env.prefill_rate), float(env.decode_rate))
    fp = _fingerprint(graph)
    key = id(graph)
    hit = _ENGINES.get(key)
    if hit is not None and hit[0]() is graph and hit[1] == rates:
        eng = hit[3]
        if hit[2] != fp:                    # mutated in place: recompile its tables
            eng.refresh("g", graph)
            _ENGINES[key] = (hit[0], rates, fp, eng)
        _ENGINES.move_to_end(key)
        return eng, "g"
    eng = DemandEngine({"g": graph}, *rates)
    ref = weakref.ref(graph, lambda r, k=key: _forget(k, r))
    _ENGINES[key] = (ref, rates, fp, eng)
    while len(_ENGINES) > MAX_ENGINES:
        _ENGINES.popitem(last=False)
    return eng, "g"


def monte_carlo_remaining_demand(graph, current_unit: str, observations: Sequence, env,
                                 n: int, seed: int,
                                 visit_cap: int = WALK_VISIT_CAP) -> RemainingDemand:
    """Same contract as the reference; computed by the sm_100a engine."""
    if n < 1:
        raise EstimationError(f"sample count must be >= 1, got {n}")
    if current_unit not in graph.units:
        raise EstimationError(f"unknown unit {current_unit!r}")
    eng, name = engine_for(graph, env)
    up, vals = eng.relevant_observation(name, current_unit, observations)
    s, capped, flags = eng.run_one(name, eng.bank.local_unit(name, current_unit), int(seed), up,
                                   vals, n, visit_cap)
    if capped:
        import logging
        logging.getLogger(__name__).warning(
            "%d of %d walks hit the %d-visit cap", capped, n, visit_cap)
    return RESULT_TYPE(samples=s.tolist(), sample_count=n, conditioned=bool(flags & 1),
                       capped_walks=capped)
