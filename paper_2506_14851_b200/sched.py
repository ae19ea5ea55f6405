"""Drop-in Gittins scheduling API backed by the sm_100a scorers.

Mirrors the reference module ``pdgsim.sched`` (sched.py:24-318): same names,
argument meaning, NaN/penalty conventions and error types.  Functions accept
the reference's own ``ApplicationInstance`` / ``Policy`` objects (duck-typed:
only attributes are read, policies compare by ``.value``), so they can be
patched into ``pdgsim.sched`` / ``pdgsim.simcore``.

All ranking arithmetic runs in kernel K1a (``pdg_gittins_rank_f64``); the
host side only marshals rows, exactly as the reference does around its numpy
call.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass
from enum import Enum
from itertools import repeat
from typing import Iterable, NamedTuple, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import EstimationError, ExhaustedDistributionError

OVERRUN_PENALTY_FACTOR = 2.0     # sched.py:24


class Policy(Enum):
    """Same values as the reference enum (sched.py:27-42)."""
    GITTINS = "gittins"
    LSTF = "lstf"
    FCFS_REQUEST = "fcfs-request"
    FCFS_APP = "fcfs-app"
    SRPT_MEAN = "srpt-mean"
    EDF = "edf"
    FAIR_SHARE = "fair-share"

    @property
    def needs_estimate(self) -> bool:
        return self in (Policy.GITTINS, Policy.LSTF, Policy.SRPT_MEAN)

    @property
    def needs_deadline(self) -> bool:
        return self in (Policy.LSTF, Policy.EDF)


def _pv(policy) -> str:
    return getattr(policy, "value", policy)


class Priority(NamedTuple):
    """Scheduling key; lower is served first (sched.py:184-192)."""
    policy: object
    key: float
    tiebreak: tuple

    def sort_key(self) -> tuple:
        return (self.key, *self.tiebreak)


@dataclass
class RefreshResult:
    refreshed: list
    elapsed_ns: int
    priorities: dict


# ---------------------------------------------------------------------------
# a1: batched rank (sched.py:102-129)
# ---------------------------------------------------------------------------

def gittins_rank_batch(values, probs, ages) -> np.ndarray:
    """Gittins ranks of N aligned support rows; NaN marks exhausted rows.
    Host arrays go straight to the C ABI (pdg_gittins_rank_f64_host: small
    batches are read in place by the K1a kernel from mapped pinned memory,
    large ones take one staged upload and one download)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    p = np.ascontiguousarray(probs, dtype=np.float64)
    a = np.ascontiguousarray(ages, dtype=np.float64)
    if v.ndim != 2 or p.shape != v.shape or a.shape != (v.shape[0],):
        raise ValueError(f"shape mismatch: values {v.shape}, probs {p.shape}, ages {a.shape}")
    n, b = v.shape
    if n == 0:
        return np.empty(0)
    if b == 0:       # no support at all: every row is exhausted
        return np.full(n, np.nan)
    out = np.empty(n)
    _lib.check(_lib.lib().pdg_gittins_rank_f64_host(
        v.ctypes.data, p.ctypes.data, a.ctypes.data, n, b, out.ctypes.data, None),
        "pdg_gittins_rank_f64_host")
    return out


def gittins_rank_points(values: Sequence[float], probs: Sequence[float],
                        age: float) -> float:
    """Rank of one weighted discrete distribution (sched.py:88-99)."""
    r = gittins_rank_batch(np.asarray(values, dtype=float)[None, :],
                           np.asarray(probs, dtype=float)[None, :], np.array([age]))
    if np.isnan(r[0]):
        raise ExhaustedDistributionError(
            f"no support point exceeds age {age}; distribution exhausted")
    return float(r[0])


def _samples_of(dist) -> list:
    s = getattr(dist, "samples", dist)
    return list(s)


def gittins_rank(dist, age: float) -> float:
    """Sample form (sched.py:51-85) on the device, bit-identical to the
    reference's scan: pdg_gittins_rank_samples_host sorts the tail
    {s - age : s > age} and scans it in the reference's operation order."""
    samples = _samples_of(dist)
    if not samples:
        raise EstimationError("gittins_rank: empty distribution")
    s = np.ascontiguousarray(np.asarray(samples, dtype=np.float64))
    out = C.c_double(0.0)
    _lib.check(_lib.lib().pdg_gittins_rank_samples_host(
        s.ctypes.data, int(s.size), float(age), C.byref(out), None),
        "pdg_gittins_rank_samples_host")
    if math.isnan(out.value):
        raise ExhaustedDistributionError(
            f"no sample exceeds age {age}; distribution exhausted")
    return out.value


def lstf_slack(dist, age: float, deadline: float, now: float) -> float:
    """Worst-case slack (sched.py:132-140)."""
    samples = _samples_of(dist)
    if not samples:
        raise EstimationError("lstf_slack: empty distribution")
    return deadline - now - (max(samples) - age)


# ---------------------------------------------------------------------------
# a4: set_remaining's bucket view (sched.py:170-181, distributions.py:79-133)
# ---------------------------------------------------------------------------

_STAGE: dict = {}                 # reused pinned host + device buffer per size class


def _stage(nbytes: int):
    cap = 1 << max(12, (nbytes - 1).bit_length())
    st = _STAGE.get(cap)
    if st is None:
        h = torch.empty(cap, dtype=torch.uint8).pin_memory()
        st = _STAGE[cap] = (h, torch.empty(cap, dtype=torch.uint8, device="cuda"), h.numpy())
    return st


def _bucketize_staged(x: np.ndarray, bucket_count: int, stride: int):
    """Small batches (the drop-in's one row per call): one upload, the
    kernel, one download and one synchronisation through a reused pinned
    buffer."""
    R, n = x.shape
    off_lo = (R * n * 8 + 15) // 16 * 16
    off_w, off_nb, off_c = off_lo + 8 * R, off_lo + 16 * R, off_lo + 20 * R
    off_c = (off_c + 15) // 16 * 16
    end = off_c + 2 * R * stride
    h, d, hv = _stage(end)
    hv[:8 * R * n] = x.reshape(-1).view(np.uint8)
    stream = torch.cuda.current_stream()
    d[:8 * R * n].copy_(h[:8 * R * n], non_blocking=True)
    base = _lib.ptr(d)
    _lib.check(_lib.lib().pdg_bucketize(base, R, n, int(bucket_count), base + off_lo,
                                        base + off_w, base + off_nb, base + off_c, stride,
                                        _lib.stream_ptr(stream)), "pdg_bucketize")
    h[off_lo:end].copy_(d[off_lo:end], non_blocking=True)
    stream.synchronize()
    return (hv[off_lo:off_w].view(np.float64).copy(), hv[off_w:off_nb].view(np.float64).copy(),
            hv[off_nb:off_nb + 4 * R].view(np.int32).copy(),
            hv[off_c:end].view(np.uint16).reshape(R, stride).copy())


def bucketize_rows(samples, bucket_count: int):
    """GPU bucketing of sample rows [R, n] -> (lo, width, nbins, counts u16)."""
    x = np.ascontiguousarray(np.asarray(samples, dtype=np.float64))
    if x.ndim == 1:
        x = x[None, :]
    R, n = x.shape
    stride = (int(bucket_count) + 7) // 8 * 8
    if R * n <= (1 << 17) and 1 <= n <= 65535 and 1 <= bucket_count <= 1024:
        return _bucketize_staged(x, bucket_count, stride)
    L = _lib.lib()
    dev = torch.device("cuda")
    t = torch.from_numpy(x).to(dev)
    lo = torch.empty(R, dtype=torch.float64, device=dev)
    w = torch.empty(R, dtype=torch.float64, device=dev)
    nb = torch.empty(R, dtype=torch.int32, device=dev)
    cnt = torch.empty((R, stride), dtype=torch.uint16, device=dev)
    _lib.check(L.pdg_bucketize(_lib.ptr(t), R, n, int(bucket_count), _lib.ptr(lo), _lib.ptr(w),
                               _lib.ptr(nb), _lib.ptr(cnt), stride, _lib.stream_ptr()),
               "pdg_bucketize")
    return lo.cpu().numpy(), w.cpu().numpy(), nb.cpu().numpy(), cnt.cpu().numpy()


def bucket_points_from(lo: float, width: float, k: int, counts, n: int):
    """(values, probs) exactly as EmpiricalDistribution.bucket_points builds
    them from the bucket grid (distributions.py:102-104, 128-133)."""
    if k == 1 and width == 0.0:
        return [lo], [1.0]
    vals = [((lo + i * width) + (lo + (i + 1) * width)) / 2.0 for i in range(k)]
    return vals, [int(c) / n for c in counts[:k]]


def set_remaining(app, remaining, bucket_count: int) -> None:
    """ApplicationInstance.set_remaining with the bucketing on the GPU."""
    samples = list(remaining.samples)
    app.remaining = remaining
    app.estimate_age = app.attained_service
    lo, w, nb, cnt = bucketize_rows(np.asarray(samples)[None, :], bucket_count)
    values, probs = bucket_points_from(float(lo[0]), float(w[0]), int(nb[0]), cnt[0],
                                       len(samples))
    app.bucket_values = np.asarray(values)
    app.bucket_probs = np.asarray(probs)
    app.shifted_values = app.bucket_values + app.estimate_age
    app.bucket_width = len(values)
    app.worst_case = max(samples)


# ---------------------------------------------------------------------------
# a3: single-instance priority (sched.py:195-234)
# ---------------------------------------------------------------------------

def compute_priority(policy, app, now: float,
                     tenant_service: Optional[dict] = None,
                     overrun_penalty_factor: float = OVERRUN_PENALTY_FACTOR) -> Priority:
    tiebreak = (app.arrival_time, app.app_instance_id)
    pv = _pv(policy)
    if pv in ("fcfs-app", "fcfs-request"):
        return Priority(policy, app.arrival_time, tiebreak)
    if pv == "edf":
        if app.deadline is None:
            raise EstimationError(f"{app.app_instance_id}: EDF requires a deadline")
        return Priority(policy, app.deadline, tiebreak)
    if pv == "fair-share":
        return Priority(policy, (tenant_service or {}).get(app.tenant_id, 0.0), tiebreak)
    if app.remaining is None:
        raise EstimationError(
            f"{app.app_instance_id}: policy {pv} requires a demand estimate")
    served_since = app.attained_service - app.estimate_age
    if pv == "srpt-mean":
        return Priority(policy, app.remaining.mean() - served_since, tiebreak)
    if pv == "lstf":
        if app.deadline is None:
            raise EstimationError(f"{app.app_instance_id}: LSTF requires a deadline")
        total = [s + app.estimate_age for s in app.remaining.samples]
        return Priority(policy, lstf_slack(total, app.attained_service, app.deadline, now),
                        tiebreak)
    if pv == "gittins":
        try:
            key = gittins_rank_points(app.shifted_values, app.bucket_probs,
                                      app.attained_service)
        except ExhaustedDistributionError:
            key = app.attained_service * overrun_penalty_factor
            app.overrun_flagged = True
        return Priority(policy, key, tiebreak)
    raise ValueError(f"unknown policy {policy!r}")


# ---------------------------------------------------------------------------
# a2: batched periodic refresh (sched.py:244-318)
# ---------------------------------------------------------------------------

def refresh_priorities(live: Iterable, now: float, bucket_period: float,
                       policy=Policy.GITTINS, tenant_service: Optional[dict] = None,
                       overrun_penalty_factor: float = OVERRUN_PENALTY_FACTOR,
                       force: bool = False) -> RefreshResult:
    if bucket_period <= 0:
        raise ValueError("bucket_period must be positive")
    instances = list(live)
    due = [a for a in instances
           if force or a.observation_pending or (now - a.last_refresh) >= bucket_period]
    priorities: dict = {}
    start = time.perf_counter_ns()
    rest = due
    if _pv(policy) == "gittins" and due:
        gapps, rest = [], []
        for a in due:
            (gapps if a.remaining is not None else rest).append(a)
        if gapps:
            m = len(gapps)
            width0 = gapps[0].bucket_width
            if all(a.bucket_width == width0 for a in gapps):   # sched.py:276-281
                vals = np.concatenate([a.shifted_values for a in gapps]).reshape(m, width0)
                prbs = np.concatenate([a.bucket_probs for a in gapps]).reshape(m, width0)
            else:
                width = max(a.bucket_width for a in gapps)
                vals = np.zeros((m, width))
                prbs = np.zeros((m, width))
                for i, a in enumerate(gapps):     # ragged rows: pad with last value, 0 mass
                    k = a.bucket_width
                    vals[i, :k] = a.shifted_values
                    prbs[i, :k] = a.bucket_probs
                    if k < width:
                        vals[i, k:] = vals[i, k - 1]
            ages = np.fromiter((a.attained_service for a in gapps), float, m)
            ranks = gittins_rank_batch(vals, prbs, ages)
            nan = np.isnan(ranks)
            if nan.any():
                ranks = np.where(nan, ages * overrun_penalty_factor, ranks)
                for a, flagged in zip(gapps, nan.tolist()):
                    if flagged:
                        a.overrun_flagged = True
            priorities = dict(zip([a.app_instance_id for a in gapps],
                                  map(Priority, repeat(policy, m), ranks.tolist(),
                                      [a.tiebreak for a in gapps])))
    for a in rest:
        priorities[a.app_instance_id] = compute_priority(
            policy, a, now, tenant_service, overrun_penalty_factor)
    elapsed = time.perf_counter_ns() - start
    for a in due:
        a.last_refresh = now
        a.observation_pending = False
    return RefreshResult(refreshed=[a.app_instance_id for a in due], elapsed_ns=elapsed,
                         priorities=priorities)
