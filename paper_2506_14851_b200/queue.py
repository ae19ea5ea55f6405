"""Device-resident scoring queue: the struct-of-arrays form of the histograms
the reference caches per application (``ApplicationInstance.set_remaining``,
sched.py:170-181) plus the per-refresh attained service.

HBM layout (one row per queued application, row = queue slot):

    lo, width, est_age, age : float64 [N]      bucket grid + ages
    nbins, nsamp            : int32   [N]      bucket count k (1 = point mass), n
    counts                  : uint16  [N, S]   bucket counts, S = ceil(B/8)*8
    tiebreak                : int32   [N]      arrival-order position (sched.py:168)
    mean, worst, deadline   : float64 [N]      RemainingDemand.mean() / worst_case /
                                               deadline (SRPT-mean and LSTF keys)

p_j = counts_j / n reproduces the reference's float64 probabilities exactly
and the bucket values are rebuilt bit-exactly from (lo, width, est_age), so a
256-bucket row costs 512 + 40 bytes instead of the 4 KB of float64 rows.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib

PDG_FLAG_OVERRUN = 0x1


def round8(b: int) -> int:
    return (int(b) + 7) // 8 * 8


class HistQueue:
    def __init__(self, capacity: int, max_bins: int = 256, device: str = "cuda"):
        _lib.lib()      # loud failure without the CUDA library / device
        if capacity < 1 or max_bins < 1 or max_bins > 1024:
            raise ValueError("capacity >= 1 and 1 <= max_bins <= 1024 required")
        self.capacity = int(capacity)
        self.max_bins = int(max_bins)
        self.stride = round8(max_bins)
        dev = torch.device(device)
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.lo = torch.zeros(capacity, **f64)
        self.width = torch.zeros(capacity, **f64)
        self.est_age = torch.zeros(capacity, **f64)
        self.age = torch.zeros(capacity, **f64)
        self.nbins = torch.ones(capacity, **i32)
        self.nsamp = torch.ones(capacity, **i32)
        self.counts = torch.zeros(capacity, self.stride, dtype=torch.uint16, device=dev)
        self.tiebreak = torch.arange(capacity, **i32)
        self.mean = torch.zeros(capacity, **f64)
        self.worst = torch.zeros(capacity, **f64)
        self.deadline = torch.zeros(capacity, **f64)
        self.key_f64 = torch.zeros(capacity, **f64)
        self.key_f32 = torch.zeros(capacity, dtype=torch.float32, device=dev)
        self.flags = torch.zeros(capacity, dtype=torch.uint8, device=dev)
        self.keys = torch.zeros(capacity, dtype=torch.int64, device=dev)
        self.slots = torch.arange(capacity, **i32)
        self.sorted_keys = torch.zeros(capacity, dtype=torch.int64, device=dev)
        self.sorted_slots = torch.zeros(capacity, **i32)
        tb = _lib.load().pdg_order_temp_bytes(capacity)
        self._temp = torch.empty(max(int(tb), 16), dtype=torch.uint8, device=dev)
        self.n = 0
        self._rows = _lib.HistRows()
        self._bind()

    def _bind(self):
        r = self._rows
        r.lo, r.width, r.est_age = (_lib.ptr(self.lo), _lib.ptr(self.width),
                                    _lib.ptr(self.est_age))
        r.nbins, r.nsamp, r.counts = (_lib.ptr(self.nbins), _lib.ptr(self.nsamp),
                                      _lib.ptr(self.counts))
        r.stride = self.stride

    # -- host loading (tests / bench; the engine fills rows on device) --------
    def load_rows(self, lo, width, est_age, nbins, nsamp, counts, age=None,
                  tiebreak=None, start: int = 0) -> None:
        m = len(lo)
        if start + m > self.capacity:
            raise ValueError("queue capacity exceeded")
        sl = slice(start, start + m)
        self.lo[sl] = torch.as_tensor(np.asarray(lo, dtype=np.float64))
        self.width[sl] = torch.as_tensor(np.asarray(width, dtype=np.float64))
        self.est_age[sl] = torch.as_tensor(np.asarray(est_age, dtype=np.float64))
        self.nbins[sl] = torch.as_tensor(np.asarray(nbins, dtype=np.int32))
        self.nsamp[sl] = torch.as_tensor(np.asarray(nsamp, dtype=np.int32))
        c = np.asarray(counts)
        if c.shape[1] > self.stride:
            raise ValueError("row wider than max_bins")
        buf = np.zeros((m, self.stride), dtype=np.uint16)
        buf[:, :c.shape[1]] = c
        self.counts[sl] = torch.as_tensor(buf)
        if age is not None:
            self.age[sl] = torch.as_tensor(np.asarray(age, dtype=np.float64))
        if tiebreak is not None:
            self.tiebreak[sl] = torch.as_tensor(np.asarray(tiebreak, dtype=np.int64).astype(np.int32))
        self.n = max(self.n, start + m)

    # -- attained service (a11b) -------------------------------------------------
    def update_attained(self, completed, progress, task_app, task_active, task_start,
                        task_cold, task_service, now: float, n: Optional[int] = None,
                        stream=None) -> None:
        """Simulator._update_attained (simcore.py:306-313) for the first n rows
        on the device: age = completed + max(progress, min(service, max(0, now -
        (start + cold)))) over each row's active started tasks (task_app = the
        task's queue row, task_start NaN = not started)."""
        n = self.n if n is None else int(n)
        nt = int(task_app.numel())
        f64, i32, u8 = torch.float64, torch.int32, torch.uint8
        for nm, x, dt in (("completed", completed, f64), ("progress", progress, f64),
                          ("task_app", task_app, i32), ("task_active", task_active, u8),
                          ("task_start", task_start, f64), ("task_cold", task_cold, f64),
                          ("task_service", task_service, f64)):
            if x.dtype != dt or not x.is_contiguous() or x.device != self.age.device:
                raise TypeError(f"{nm} must be a contiguous {dt} tensor on {self.age.device}")
        if completed.numel() < n or progress.numel() < n or task_active.numel() < nt \
                or task_start.numel() < nt or task_cold.numel() < nt \
                or task_service.numel() < nt:
            raise ValueError("update_attained: column shorter than its table")
        if getattr(self, "_att_temp", None) is None or self._att_temp.numel() < 8 * n:
            self._att_temp = torch.empty(max(8 * self.capacity, 16), dtype=torch.uint8,
                                         device=self.age.device)
        _lib.check(_lib.lib().pdg_attained_service(
            _lib.ptr(completed), _lib.ptr(progress), n, _lib.ptr(task_app),
            _lib.ptr(task_active), _lib.ptr(task_start), _lib.ptr(task_cold),
            _lib.ptr(task_service), nt, float(now), _lib.ptr(self.age),
            _lib.ptr(self._att_temp), self._att_temp.numel(), _lib.stream_ptr(stream)),
            "pdg_attained_service")

    # -- scoring ---------------------------------------------------------------
    def score(self, penalty: float = 2.0, n: Optional[int] = None, stream=None,
              keys: bool = True, rows: Optional[torch.Tensor] = None) -> None:
        """K1b over the first n rows (or only `rows`, an int32 device tensor):
        key_f32, flags and packed sort keys, indexed by row."""
        n = (self.n if n is None else int(n)) if rows is None else int(rows.numel())
        L = _lib.lib()
        _lib.check(L.pdg_gittins_score_hist(
            C.byref(self._rows), _lib.ptr(self.age), n, float(penalty),
            _lib.ptr(self.key_f32), _lib.ptr(self.flags), _lib.ptr(self.tiebreak),
            _lib.ptr(self.keys) if keys else None, _lib.ptr(rows), _lib.stream_ptr(stream)),
            "pdg_gittins_score_hist")

    def score_policy(self, policy, now: float, n: Optional[int] = None, stream=None,
                     rows: Optional[torch.Tensor] = None) -> None:
        """K1c: SRPT-mean or LSTF keys (float64, bit-identical to
        compute_priority, sched.py:216-224) into key_f64 and, order-preserving,
        into keys; sort with order() (full 64-bit keys)."""
        pv = getattr(policy, "value", policy)
        code = {"srpt-mean": 1, "lstf": 2}.get(pv)
        if code is None:
            raise ValueError(f"score_policy: {pv!r} is not SRPT_MEAN or LSTF")
        n = (self.n if n is None else int(n)) if rows is None else int(rows.numel())
        L = _lib.lib()
        _lib.check(L.pdg_policy_keys(
            code, _lib.ptr(self.mean), _lib.ptr(self.worst), _lib.ptr(self.est_age),
            _lib.ptr(self.age), _lib.ptr(self.deadline), float(now), n, _lib.ptr(rows),
            _lib.ptr(self.key_f64), _lib.ptr(self.keys), _lib.stream_ptr(stream)),
            "pdg_policy_keys")

    def order(self, n: Optional[int] = None, stream=None,
              arrival_ordered: bool = False) -> torch.Tensor:
        """K5 (single GPU): queue slots sorted by (key, arrival order).

        arrival_ordered=True asserts slot order == arrival order, so a stable
        sort on the 32-bit key alone yields the same order in half the passes.
        """
        n = self.n if n is None else int(n)
        L = _lib.lib()
        _lib.check(L.pdg_order(_lib.ptr(self.keys), _lib.ptr(self.sorted_keys),
                               _lib.ptr(self.slots), _lib.ptr(self.sorted_slots), n,
                               32 if arrival_ordered else 0,
                               _lib.ptr(self._temp), self._temp.numel(),
                               _lib.stream_ptr(stream)), "pdg_order")
        return self.sorted_slots[:n]
