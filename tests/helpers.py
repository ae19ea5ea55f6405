"""Shared test helpers: synthetic histogram rows and oracle views of them."""

import numpy as np


def hist_rows(rng, n, b, nsamp=512, degenerate_frac=0.02, exhaust_frac=0.02,
              on_support_frac=0.02, ragged=False):
    """Random queue rows in the HistQueue layout + the ages to score them at."""
    lo = rng.uniform(0, 3000, n)
    w = rng.lognormal(0, 1.5, n)
    est = rng.uniform(0, 500, n)
    nb = np.full(n, b, dtype=np.int64)
    if ragged:
        nb = rng.integers(1, b + 1, n)
    probs = rng.lognormal(0, 2, (n, b))
    probs[rng.random((n, b)) < 0.3] = 0.0
    counts = np.zeros((n, b), dtype=np.int64)
    for i in range(n):
        k = nb[i]
        pr = probs[i, :k]
        pr = pr / pr.sum() if pr.sum() > 0 else np.full(k, 1.0 / k)
        counts[i, :k] = rng.multinomial(nsamp, pr)
    deg = rng.random(n) < degenerate_frac
    nb[deg] = 1
    w[deg] = 0.0
    counts[deg] = 0
    counts[deg, 0] = nsamp
    span = nb * w
    age = est + rng.uniform(-0.1, 1.1, n) * np.maximum(span, 1.0)
    age = np.maximum(age, 0.0)
    vals = midpoints(lo, w, est, nb, b)
    ex = rng.random(n) < exhaust_frac
    age[ex] = vals[ex, 0] + (nb[ex] + 1) * np.maximum(w[ex], 1.0)
    on = rng.random(n) < on_support_frac
    idx = rng.integers(0, nb)          # exact support value: d == 0 on that bucket
    age[on] = vals[np.arange(n), idx][on]
    return dict(lo=lo, width=w, est_age=est, nbins=nb, nsamp=np.full(n, nsamp),
                counts=counts, age=age)


def midpoints(lo, w, est, nb, b):
    """Bucket values exactly as set_remaining builds them (distributions.py:103,131,
    sched.py:179); buckets past nb repeat the last value (ragged pad)."""
    j = np.arange(b, dtype=np.float64)
    a = lo[:, None] + j[None, :] * w[:, None]
    c = lo[:, None] + (j[None, :] + 1.0) * w[:, None]
    v = (a + c) / 2.0 + est[:, None]
    last = v[np.arange(len(lo)), nb - 1]
    pad = j[None, :] >= nb[:, None]
    return np.where(pad, last[:, None], v)


def oracle_keys(O, rows, penalty=2.0):
    b = rows["counts"].shape[1]
    vals = midpoints(rows["lo"], rows["width"], rows["est_age"], rows["nbins"], b)
    probs = rows["counts"] / rows["nsamp"][:, None].astype(np.float64)
    r = O.gittins_rank_batch(vals, probs, rows["age"])
    bad = np.isnan(r)
    return np.where(bad, rows["age"] * penalty, r), bad
