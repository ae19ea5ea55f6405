"""K6 oracle (dispatch / preemption plan) pinned to the reference simulator:
on every PriorityRefresh of BASELINE config 1 the restatement must predict
exactly the preemptions and starts the reference performs."""

import os

import numpy as np
import pytest

from oracle import pdg_oracle as O

HAVE_REF = any(os.path.isdir(p) for p in ("/root/reference/pkg/src",
               os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "baseline", "_ref")))


@pytest.mark.skipif(not HAVE_REF, reason="reference pdgsim not available")
def test_oracle_matches_reference_config1():
    from tests.dispatch_hook import record_config1
    recs = record_config1()
    assert len(recs) > 100
    kinds = set()
    for table, slots, h, acts in recs:
        ev = O.plan_dispatch(table["backend"], table["active"], table["key"],
                             table["app_rank"], table["stage"], table["request"], slots, h)
        assert ev == acts
        kinds |= {k for k, _ in acts}
    assert kinds == {1, 2}          # preemptions happened too


def test_oracle_small_cases():
    # one backend, 2 slots; running keys 9 and 1, waiting 2 and 5 (h = 1.5)
    be, act = [0, 0, 0, 0], [1, 1, 0, 0]
    key, rank = [9.0, 1.0, 2.0, 5.0], [0, 1, 2, 3]
    z = [0, 0, 0, 0]
    assert O.plan_dispatch(be, act, key, rank, z, z, [2], 1.5) == [(1, 0), (2, 2)]
    assert O.plan_dispatch(be, act, key, rank, z, z, [2], 1.5, preempt=False) == []
    assert O.plan_dispatch(be, act, key, rank, z, z, [4], 1.5) == [(1, 0), (2, 2), (2, 3),
                                                                   (2, 0)]
    # ties on the key fall back to arrival rank, stage, request
    assert O.plan_dispatch([0, 0, 0], [0, 0, 0], [1.0, 1.0, 1.0], [1, 0, 0], [0, 1, 0],
                           [0, 0, 0], [3], 1.5) == [(2, 2), (2, 1), (2, 0)]
    rng = np.random.default_rng(0)
    assert O.plan_dispatch([], [], [], [], [], [], [3, 1], 1.5) == []
    del rng
