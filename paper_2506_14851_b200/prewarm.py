"""GPU backend-prewarm estimator (K4): drop-in ``plan_prewarm`` and the
per-backend-type need-probability grid.

* ``plan_prewarm`` / ``plan_prewarm_batch`` -- the reference's latest-safe
  trigger rule (prewarm.py:42-96), bit-exact, one warp per (app, successor).
* ``PrewarmTables.need`` -- need[a, type, window] for a whole queue (BASELINE
  config 5), from the same completion-time samples ``_plan_prewarms`` uses
  (simcore.py:450-487).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib

DEFAULT_KNOB = 0.5          # prewarm.py:21


@dataclass
class PrewarmPlan:
    """Mirror of the reference decision record (prewarm.py:24-39)."""
    target_backend: object
    p_s: float
    t_p: float
    trigger_time: float
    p_e: float
    knob: float

    def __post_init__(self):
        if not (0.0 <= self.knob <= 1.0):
            raise ValueError(f"knob must be in [0, 1], got {self.knob}")
        if self.p_s < self.knob:
            raise ValueError("plan must not exist when p_s < K")


def plan_prewarm_batch(samples: Sequence[Sequence[float]], bucket_count, p_s, t_p, knob, now):
    """Vectorised plan_prewarm over J jobs (lists of absolute completion
    samples).  Returns (has_plan bool[J], trigger f64[J], p_e f64[J])."""
    J = len(samples)
    L = _lib.lib()
    dev = torch.device("cuda")
    lens = np.array([len(s) for s in samples], dtype=np.int32)
    offs = np.zeros(J, dtype=np.int32)
    if J > 1:
        offs[1:] = np.cumsum(lens)[:-1]
    pool = np.concatenate([np.asarray(s, dtype=np.float64) for s in samples]) if J else np.zeros(0)

    def col(x, dt):
        a = np.broadcast_to(np.asarray(x, dtype=dt), (J,)).copy()
        return torch.from_numpy(a).to(dev)

    knob_a = np.broadcast_to(np.asarray(knob, dtype=np.float64), (J,))
    tp_a = np.broadcast_to(np.asarray(t_p, dtype=np.float64), (J,))
    if ((knob_a < 0) | (knob_a > 1)).any():
        raise ValueError("knob must be in [0, 1]")
    if (tp_a < 0).any():
        raise ValueError("warm-up duration must be >= 0")
    if J == 0:
        return np.zeros(0, bool), np.zeros(0), np.zeros(0)
    if J <= 256 and pool.size <= (1 << 16):
        return _plan_staged(pool, offs, lens, bucket_count, p_s, t_p, knob, now, J)
    tpool = torch.from_numpy(pool if pool.size else np.zeros(1)).to(dev)
    has = torch.empty(J, dtype=torch.uint8, device=dev)
    trig = torch.empty(J, dtype=torch.float64, device=dev)
    pe = torch.empty(J, dtype=torch.float64, device=dev)
    args = [col(offs, np.int32), col(lens, np.int32), col(bucket_count, np.int32),
            col(p_s, np.float64), col(t_p, np.float64), col(knob, np.float64),
            col(now, np.float64)]
    _lib.check(L.pdg_plan_prewarm(_lib.ptr(tpool), *[_lib.ptr(t) for t in args], J,
                                  _lib.ptr(has), _lib.ptr(trig), _lib.ptr(pe),
                                  _lib.stream_ptr()), "pdg_plan_prewarm")
    return has.cpu().numpy().astype(bool), trig.cpu().numpy(), pe.cpu().numpy()


def _plan_staged(pool, offs, lens, bucket_count, p_s, t_p, knob, now, J):
    """Small batches (the drop-in's one job per call): every input in one
    pinned upload, the kernel, one download, one synchronisation."""
    from .sched import _stage
    P = max(int(pool.size), 1)
    o_i = 8 * P                                   # int32 columns: offs, lens, bucket_count
    o_f = (o_i + 12 * J + 15) // 16 * 16          # float64 columns: p_s, t_p, knob, now
    o_out = o_f + 32 * J                          # outputs: trigger, p_e, has_plan
    end = o_out + 17 * J
    h, d, hv = _stage(end)
    if pool.size:
        hv[:8 * pool.size] = pool.view(np.uint8)
    ic = hv[o_i:o_i + 12 * J].view(np.int32).reshape(3, J)
    ic[0], ic[1] = offs, lens
    ic[2] = np.broadcast_to(np.asarray(bucket_count, dtype=np.int32), (J,))
    fc = hv[o_f:o_out].view(np.float64).reshape(4, J)
    for i, x in enumerate((p_s, t_p, knob, now)):
        fc[i] = np.broadcast_to(np.asarray(x, dtype=np.float64), (J,))
    stream = torch.cuda.current_stream()
    d[:o_out].copy_(h[:o_out], non_blocking=True)
    b = _lib.ptr(d)
    _lib.check(_lib.lib().pdg_plan_prewarm(
        b, b + o_i, b + o_i + 4 * J, b + o_i + 8 * J, b + o_f, b + o_f + 8 * J,
        b + o_f + 16 * J, b + o_f + 24 * J, J, b + o_out + 16 * J, b + o_out, b + o_out + 8 * J,
        _lib.stream_ptr(stream)), "pdg_plan_prewarm")
    h[o_out:end].copy_(d[o_out:end], non_blocking=True)
    stream.synchronize()
    trig = hv[o_out:o_out + 8 * J].view(np.float64).copy()
    pe = hv[o_out + 8 * J:o_out + 16 * J].view(np.float64).copy()
    has = hv[o_out + 16 * J:end].astype(bool)
    return has, trig, pe


def plan_prewarm(completion_dist, p_s: float, t_p: float, knob: float, now: float,
                 target_backend=None) -> Optional[PrewarmPlan]:
    """Same contract as the reference; `completion_dist` needs `.samples` and
    `.bucket_count` (an EmpiricalDistribution)."""
    if not (0.0 <= knob <= 1.0):
        raise ValueError(f"knob must be in [0, 1], got {knob}")
    if t_p < 0:
        raise ValueError(f"warm-up duration must be >= 0, got {t_p}")
    if p_s < knob:
        return None
    has, trig, pe = plan_prewarm_batch([list(completion_dist.samples)],
                                       completion_dist.bucket_count, p_s, t_p, knob, now)
    if not has[0]:
        return None
    return PrewarmPlan(target_backend=target_backend, p_s=p_s, t_p=t_p,
                       trigger_time=float(trig[0]), p_e=float(pe[0]), knob=knob)


# ---------------------------------------------------------------------------
# need-probability grid (config 5)
# ---------------------------------------------------------------------------

def _check_index(graph_idx, unit_idx, now, device):
    """The queue columns the prewarm kernels read: int32 graph / unit indices
    and float64 `now`, contiguous, on the tables' device."""
    for nm, x, dt in (("graph_idx", graph_idx, torch.int32), ("unit_idx", unit_idx, torch.int32),
                      ("now", now, torch.float64)):
        if not isinstance(x, torch.Tensor) or x.dtype != dt or not x.is_contiguous() \
                or x.device != device:
            raise TypeError(f"{nm} must be a contiguous {dt} tensor on {device}")
    if not (graph_idx.numel() == unit_idx.numel() == now.numel()):
        raise ValueError("graph_idx, unit_idx and now must have one entry per application")


class PrewarmTablesC(C.Structure):
    _fields_ = [(nm, C.c_void_p) for nm in ("svc_sorted", "svc_off", "svc_len", "graph_base",
                                            "succ_off", "succ_len", "succ_nxt", "succ_p",
                                            "unit_type", "win_idx", "unit_rec")]


class PrewarmTables:
    """Sorted service-time pools, successor probabilities and backend types
    per unit, resident on the device."""

    def __init__(self, *, svc_sorted, svc_off, svc_len, graph_base, succ_off, succ_len,
                 succ_nxt, succ_p, unit_type, n_types, device="cuda"):
        _lib.lib()
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None and torch.cuda.is_available():
            dev = torch.device("cuda", torch.cuda.current_device())

        def t(a, dt):
            a = np.ascontiguousarray(np.asarray(a, dtype=dt))
            return torch.from_numpy(a if a.size else np.zeros(1, dtype=dt)).to(dev)

        self.device = dev
        self.n_types = int(n_types)
        self.t = dict(svc_sorted=t(svc_sorted, np.float64), svc_off=t(svc_off, np.int32),
                      svc_len=t(svc_len, np.int32), graph_base=t(graph_base, np.int32),
                      succ_off=t(succ_off, np.int32), succ_len=t(succ_len, np.int32),
                      succ_nxt=t(succ_nxt, np.int32), succ_p=t(succ_p, np.float64),
                      unit_type=t(unit_type, np.int32))
        # one 48-byte record per unit for the need kernel: (svc_off, svc_len,
        # successor backend types x4, float(p_s) bits x4, 0, 0)
        soff_a, slen_a = np.asarray(svc_off, np.int64), np.asarray(svc_len, np.int64)
        so_a, sl_a = np.asarray(succ_off, np.int64), np.asarray(succ_len, np.int64)
        nx_a, p_a = np.asarray(succ_nxt, np.int64), np.asarray(succ_p, np.float64)
        ut_a, gb_a = np.asarray(unit_type, np.int64), np.asarray(graph_base, np.int64)
        U = soff_a.size
        rec = np.zeros((max(U, 1), 12), dtype=np.int32)
        gof = np.zeros(U, dtype=np.int64)                  # graph base of each unit
        for g in range(gb_a.size):
            gof[gb_a[g]:(gb_a[g + 1] if g + 1 < gb_a.size else U)] = gb_a[g]
        rec[:U, 0], rec[:U, 1] = soff_a, slen_a
        rec[:U, 2:6] = -1
        for i in range(4):
            has = sl_a > i
            idx = np.where(has, so_a + i, 0)
            rec[:U, 2 + i] = np.where(has, ut_a[gof + nx_a[idx]] if nx_a.size else -1, -1)
            pf = np.where(has, p_a[idx] if p_a.size else 0.0, 0.0).astype(np.float32)
            rec[:U, 6 + i] = pf.view(np.int32)
        # the packed records hold four successors: wider fan-outs take the
        # table-walking need kernel
        self.max_succ = int(sl_a.max()) if sl_a.size else 0
        self.max_type = int(ut_a.max()) if ut_a.size else -1
        if self.max_succ <= 4:
            self.t["unit_rec"] = t(rec.reshape(-1), np.int32)
        self.c = PrewarmTablesC(*[_lib.ptr(self.t[nm]) if nm in self.t else None
                                  for nm, _ in PrewarmTablesC._fields_])
        self.n_units = int(np.asarray(svc_len).size)
        self._win = None            # (windows, index) cache for pdg_prewarm_window_index

    @classmethod
    def from_graphs(cls, graphs: dict, prefill_rate=10000.0, decode_rate=50.0, device="cuda"):
        """Tables for named graphs (reference PDGraph or KBGraph); graph and
        unit order match GraphBank (graph insertion order, sorted unit ids)."""
        svc, soff, slen, gbase = [], [], [], []
        s_off, s_len, s_nxt, s_p, utype = [], [], [], [], []
        types: dict = {}
        for nm, g in graphs.items():
            order = sorted(g.units)
            pos = {u: i for i, u in enumerate(order)}
            gbase.append(len(slen))
            for uid in order:
                u = g.units[uid]
                if u.is_llm:       # simcore.py:480-487 (records' joint i, o)
                    xs = [r.input_len / prefill_rate + r.output_len / decode_rate
                          for r in u.records]
                else:
                    xs = list(u.duration_dist.samples)
                soff.append(len(svc))
                slen.append(len(xs))
                svc.extend(sorted(xs))
                succ = sorted(u.successors.items())
                s_off.append(len(s_nxt))
                s_len.append(len(succ))
                s_nxt.extend(pos[v] for v, _ in succ)
                s_p.extend(p for _, p in succ)
                backend = getattr(u, "backend", None)
                wc = backend.warm_content_id() if backend is not None else getattr(
                    u, "warm_content", None)
                utype.append(types.setdefault(wc, len(types)) if wc is not None else -1)
        tb = cls(svc_sorted=svc, svc_off=soff, svc_len=slen, graph_base=gbase, succ_off=s_off,
                 succ_len=s_len, succ_nxt=s_nxt, succ_p=s_p, unit_type=utype,
                 n_types=max(len(types), 1), device=device)
        tb.type_ids = types
        return tb

    def _window_index(self, windows, stream=None):
        if self._win is None or not torch.equal(self._win[0], windows):
            idx = torch.empty(max(self.n_units, 1) * int(windows.numel()), dtype=torch.int32,
                              device=self.device)
            self.c.win_idx = None
            _lib.check(_lib.lib().pdg_prewarm_window_index(
                C.byref(self.c), self.n_units, _lib.ptr(windows), int(windows.numel()),
                _lib.ptr(idx), _lib.stream_ptr(stream)), "pdg_prewarm_window_index")
            self._win = (windows.clone(), idx)
        return self._win[1]

    def triggers(self, graph_idx, unit_idx, now, warmup_by_type, knob: float,
                 bucket_count: int, stream=None):
        """plan_prewarm for every (application, successor slot) of the queue
        (config 5's latest-safe triggers, _plan_prewarms simcore.py:450-478):
        (has_plan bool[N,S], trigger f64[N,S], p_e f64[N,S]) on the device,
        S = the bank's largest fan-out, successors in sorted order."""
        if len(warmup_by_type) <= self.max_type:
            raise ValueError(f"warmup_by_type has {len(warmup_by_type)} entries; the tables "
                             f"hold backend type {self.max_type}")
        _check_index(graph_idx, unit_idx, now, self.device)
        n = int(graph_idx.numel())
        S = max(self.max_succ, 1)
        dev = self.device
        stream = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.stream(stream):              # outputs and temp live on `stream`
            has = torch.zeros((n, S), dtype=torch.uint8, device=dev)
            trig = torch.zeros((n, S), dtype=torch.float64, device=dev)
            pe = torch.zeros((n, S), dtype=torch.float64, device=dev)
            L = _lib.lib()
            tb = int(L.pdg_prewarm_triggers_temp_bytes(n, S))
            temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
            w = torch.as_tensor(warmup_by_type, dtype=torch.float64, device=dev).contiguous()
            _lib.check(L.pdg_prewarm_triggers(
                C.byref(self.c), _lib.ptr(graph_idx), _lib.ptr(unit_idx), _lib.ptr(now), n, S,
                _lib.ptr(w), int(w.numel()), float(knob), int(bucket_count), _lib.ptr(has),
                _lib.ptr(trig), _lib.ptr(pe), _lib.ptr(temp), temp.numel(),
                _lib.stream_ptr(stream)), "pdg_prewarm_triggers")
            return has == 1, trig, pe

    def need(self, graph_idx, unit_idx, now, windows, *, dense=True, aggregate=True,
             out=None, window_index=True, unit_records=True, stream=None):
        """need[N, T, K] float32 (dense) and/or agg[T, K] float64 over the queue.
        window_index: per-(unit, window) lower bounds computed once per window
        grid instead of a binary search per application."""
        _check_index(graph_idx, unit_idx, now, self.device)
        n = int(graph_idx.numel())
        K = int(windows.numel())
        dev = self.device
        self.c.win_idx = _lib.ptr(self._window_index(windows, stream)) if window_index else None
        self.c.unit_rec = (_lib.ptr(self.t["unit_rec"])
                           if unit_records and "unit_rec" in self.t else None)
        need = out if out is not None else (
            torch.empty((n, self.n_types, K), dtype=torch.float32, device=dev) if dense else None)
        agg = torch.zeros((self.n_types, K), dtype=torch.float64, device=dev) if aggregate else None
        L = _lib.lib()
        _lib.check(L.pdg_prewarm_need(C.byref(self.c), _lib.ptr(graph_idx), _lib.ptr(unit_idx),
                                      _lib.ptr(now), n, _lib.ptr(windows), K, self.n_types,
                                      _lib.ptr(need), _lib.ptr(agg), _lib.stream_ptr(stream)),
                   "pdg_prewarm_need")
        return need, agg
