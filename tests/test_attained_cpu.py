"""a11b oracle pin: oracle.update_attained equals the reference's own
Simulator._update_attained (simcore.py:306-313), called on stub simulator
state, bit for bit."""

import types

import numpy as np
import pytest

from oracle import pdg_oracle as O
from tests.dispatch_hook import import_pdgsim


def random_tables(seed, n_apps=50, n_tasks=400):
    rng = np.random.default_rng(seed)
    now = float(rng.uniform(50, 500))
    completed = rng.uniform(0, 300, n_apps)
    progress = rng.uniform(0, 20, n_apps)
    progress[::7] = 0.0
    app = rng.integers(0, n_apps, n_tasks)
    start = rng.uniform(0, now + 20, n_tasks)
    start[::5] = np.nan                                  # not started
    cold = np.where(rng.random(n_tasks) < 0.5, 0.0, rng.uniform(0, 30, n_tasks))
    service = rng.uniform(0, 80, n_tasks)
    service[::11] = now - (start[::11] + cold[::11])     # ties between run and service
    active = (rng.random(n_tasks) < 0.8).astype(np.uint8)
    return now, completed, progress, app, start, cold, service, active


def oracle_of(now, completed, progress, app, start, cold, service, active):
    tasks = [(int(a), None if np.isnan(s) else float(s), float(c), float(v))
             for a, s, c, v, on in zip(app, start, cold, service, active) if on]
    return O.update_attained(completed.tolist(), progress.tolist(), tasks, now)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_matches_reference_update_attained(seed):
    try:
        import_pdgsim()
    except ImportError:
        pytest.skip("pdgsim not importable")
    from pdgsim.simcore import Simulator
    now, completed, progress, app, start, cold, service, active = random_tables(seed)
    apps = [types.SimpleNamespace(unit_progress=float(p), completed_service=float(c),
                                  inst=types.SimpleNamespace(attained_service=None))
            for c, p in zip(completed, progress)]
    backends = {}
    for b in range(3):
        act = {}
        for t in np.flatnonzero((active == 1) & (np.arange(len(app)) % 3 == b)):
            act[int(t)] = types.SimpleNamespace(
                app=apps[app[t]], start_time=None if np.isnan(start[t]) else float(start[t]),
                cold_delay=float(cold[t]), service=float(service[t]))
        backends[b] = types.SimpleNamespace(active=act)
    sim = types.SimpleNamespace(backends=backends, now=now)
    for a in apps:
        Simulator._update_attained(sim, a)
    want = [a.inst.attained_service for a in apps]
    got = oracle_of(now, completed, progress, app, start, cold, service, active)
    assert np.array_equal(np.array(got), np.array(want))
