"""Oracle pin for the sample-form Gittins rank: oracle.gittins_rank_samples
equals the reference's own pdgsim.sched.gittins_rank (sched.py:51-85) bit for
bit on random sample lists with repeated values, degenerate tails and ages
on sample values."""

import numpy as np
import pytest

from oracle import pdg_oracle as O
from tests.dispatch_hook import import_pdgsim


def cases(seed=0, count=60):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        n = int(rng.choice([1, 2, 5, 64, 512, 1000, 4096]))
        s = np.round(rng.gamma(2.0, 20.0, n), int(rng.integers(0, 4)))   # repeated values
        if i % 9 == 0:
            s[:] = s[0]
        age = float(rng.choice([0.0, s[rng.integers(0, n)], rng.uniform(0, s.max())]))
        out.append((s.tolist(), age))
    return out


def test_oracle_matches_reference_gittins_rank():
    try:
        import_pdgsim()
    except ImportError:
        pytest.skip("pdgsim not importable")
    from pdgsim.errors import ExhaustedDistributionError
    from pdgsim.sched import gittins_rank
    for s, age in cases():
        try:
            want = gittins_rank(s, age)
        except ExhaustedDistributionError:
            want = None
        got = O.gittins_rank_samples(s, age) if any(x > age for x in s) else None
        assert got == want, (len(s), age)
