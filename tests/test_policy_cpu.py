"""SRPT-mean / LSTF keys: the oracle restatement is
pinned to the interpreter's own sum() and, when /root/reference is present,
to the reference's compute_priority on the golden Monte Carlo samples."""

import math
import os
import sys

import numpy as np
import pytest

from oracle import pdg_oracle as O

REF = "/root/reference/pkg/src"


def test_py_sum_is_builtin_sum():
    rng = np.random.default_rng(5)
    for t in range(3000):
        n = int(rng.integers(1, 700))
        kind = t % 4
        if kind == 0:
            a = rng.lognormal(0, 2, n)
        elif kind == 1:
            a = rng.uniform(0, 1e6, n) * (10.0 ** rng.integers(-8, 8, n))
        elif kind == 2:
            a = np.abs(rng.standard_normal(n)) * 1e16
        else:
            a = np.concatenate([[1e100], rng.uniform(0, 1, n), [1e100]])
        xs = a.tolist()
        assert O.py_sum(xs) == sum(xs)
    assert O.py_sum([]) == 0
    assert math.isinf(O.py_sum([1e308, 1e308]))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_keys_match_reference_compute_priority(mc_full):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from pdgsim.estimator import RemainingDemand
    from pdgsim.sched import ApplicationInstance, Policy, compute_priority
    rng = np.random.default_rng(9)
    for name, s in sorted(mc_full.items()):
        samples = s.tolist()
        for _ in range(4):
            est = float(rng.uniform(0, 50))
            att = est + float(rng.uniform(0, 2 * max(samples)))
            dl = float(rng.uniform(0, 5000))
            now = float(rng.uniform(0, 3000))
            app = ApplicationInstance("a", "g", 0.0, deadline=dl)
            app.remaining = RemainingDemand(samples=samples, sample_count=len(samples))
            app.estimate_age = est
            app.attained_service = att
            k1 = compute_priority(Policy.SRPT_MEAN, app, now).key
            k2 = compute_priority(Policy.LSTF, app, now).key
            assert O.srpt_mean_key(samples, att, est) == k1, name
            assert O.lstf_key(samples, att, est, dl, now) == k2, name
