"""K6 on the GPU: the device dispatch / preemption plan equals the reference
simulator's actions on every PriorityRefresh of BASELINE config 1, and the
oracle's plan on random task tables (ties, negative keys, many backends)."""

import numpy as np
import pytest

from oracle import pdg_oracle as O

pytestmark = pytest.mark.gpu


def _dev(table):
    import torch
    d = "cuda"
    return (torch.tensor(table["backend"], dtype=torch.int32, device=d),
            torch.tensor(table["active"], dtype=torch.uint8, device=d),
            torch.tensor(table["key"], dtype=torch.float64, device=d),
            torch.tensor(table["app_rank"], dtype=torch.int32, device=d),
            torch.tensor(table["stage"], dtype=torch.int32, device=d),
            torch.tensor(table["request"], dtype=torch.int32, device=d))


def test_plan_matches_reference_config1():
    from tests.dispatch_hook import import_pdgsim, record_config1
    try:
        import_pdgsim()
    except ImportError:
        pytest.skip("pdgsim not installed in baseline/_ref")
    from paper_2506_14851_b200.dispatch import DispatchPlanner
    planner = DispatchPlanner()
    recs = record_config1()
    assert len(recs) > 100
    for table, slots, h, acts in recs:
        assert planner.plan(*_dev(table), slots, hysteresis=h) == acts


def test_plan_random_tables_vs_oracle():
    from paper_2506_14851_b200.dispatch import DispatchPlanner
    planner = DispatchPlanner()
    rng = np.random.default_rng(3)
    for trial in range(60):
        nb = int(rng.integers(1, 6))
        slots = [int(rng.integers(0, 40)) for _ in range(nb)]
        n = int(rng.integers(0, 3000))
        be = rng.integers(0, nb, n)
        act = np.zeros(n, dtype=np.int64)
        for b in range(nb):                       # at most `slots` running per backend
            idx = np.flatnonzero(be == b)
            k = min(len(idx), int(rng.integers(0, slots[b] + 1)))
            act[rng.choice(idx, k, replace=False)] = 1
        key = np.round(rng.lognormal(0, 2, n), 1)  # many exact ties
        if trial % 3 == 0:
            key = key - 20.0                       # negative keys (LSTF slack)
        rank = rng.integers(0, max(n // 3, 1), n)
        stage = rng.integers(0, 4, n)
        req = rng.integers(0, 3, n)
        table = {"backend": be.tolist(), "active": act.tolist(), "key": key.tolist(),
                 "app_rank": rank.tolist(), "stage": stage.tolist(), "request": req.tolist()}
        h = [1.0, 1.5, 3.0][trial % 3]
        for pre in (True, False):
            want = O.plan_dispatch(be.tolist(), act.tolist(), key.tolist(), rank.tolist(),
                                   stage.tolist(), req.tolist(), slots, h, preempt=pre)
            got = planner.plan(*_dev(table), slots, hysteresis=h, preempt=pre)
            assert got == want, (trial, pre)


def test_plan_rejects_overfull_backend():
    from paper_2506_14851_b200.dispatch import DispatchPlanner
    table = {"backend": [0, 0, 0], "active": [1, 1, 1], "key": [1.0, 2.0, 3.0],
             "app_rank": [0, 1, 2], "stage": [0, 0, 0], "request": [0, 0, 0]}
    with pytest.raises(ValueError):
        DispatchPlanner().plan(*_dev(table), [2])
