"""The drop-in monte_carlo_remaining_demand caches one compiled engine per
graph object.  Graphs are mutated in place by the reference's own profiling
path -- record_trial on a unit already at FIFO capacity (pdgraph.py:162-169,
the record count does not change) and build_masks (estimator.py:108-142,
mask flags set in place) -- and the drop-in must see both: its samples stay
bit-identical to the reference's monte_carlo_remaining_demand on the mutated
graph."""

import numpy as np
import pytest

from tests.dispatch_hook import import_pdgsim

pytestmark = pytest.mark.gpu


def _setup():
    try:
        import_pdgsim()
    except ImportError:
        pytest.skip("pdgsim not installed in baseline/_ref")
    from pdgsim.workload import archetype
    cap = 150
    g = archetype("verify-chain", {"trials": cap, "capacity": cap, "bucket_count": 16,
                                   "app_id": "vc"}, seed=3)
    src = archetype("verify-chain", {"trials": 40, "capacity": cap, "bucket_count": 16,
                                     "app_id": "vc"}, seed=11)
    assert all(len(u.records) == cap for u in g.units.values())
    by_trial: dict = {}
    for uid, u in src.units.items():
        for r in u.records:
            by_trial.setdefault(r.trial_id, {})[uid] = r
    return g, [by_trial[t] for t in sorted(by_trial)]


def _same(g, unit, obs, seed):
    from pdgsim.estimator import monte_carlo_remaining_demand as ref_mc
    from pdgsim.pdgraph import RateProfile
    from paper_2506_14851_b200.estimator import monte_carlo_remaining_demand as ours
    env = RateProfile()
    want = ref_mc(g, unit, obs, env, 512, seed)
    got = ours(g, unit, obs, env, 512, seed)
    assert np.array_equal(np.asarray(got.samples), np.asarray(want.samples)), (unit, seed)
    assert got.conditioned == want.conditioned
    assert got.capped_walks == want.capped_walks
    return want


def test_dropin_sees_record_trial_at_capacity():
    g, trials = _setup()
    from pdgsim.pdgraph import UnitRecord, record_trial
    for k, uid in enumerate(sorted(g.units)):
        _same(g, uid, [], 100 + k)                      # engine compiled and cached
    for i, tr in enumerate(trials[:12]):
        rec = {uid: UnitRecord(5000 + i, r.input_len, r.output_len, r.parallelism, r.duration,
                               r.next_unit) for uid, r in tr.items()}
        lens = {uid: len(u.records) for uid, u in g.units.items()}
        record_trial(g, rec)
        assert {uid: len(u.records) for uid, u in g.units.items()} == lens   # FIFO at cap
        for k, uid in enumerate(sorted(g.units)):
            _same(g, uid, [], 200 + 10 * i + k)


def test_dropin_sees_build_masks_and_in_place_flags():
    g, _ = _setup()
    from pdgsim.estimator import Observation, build_masks
    ex = g.units["extract"].records[7]
    obs = [Observation("extract", ex.input_len, ex.output_len, 1)]
    base = _same(g, "verify", obs, 7)
    masks0 = {uid: u.masks.to_dict() for uid, u in g.units.items()}
    build_masks(g, threshold=0.999)                     # flags drop in place
    assert {uid: u.masks.to_dict() for uid, u in g.units.items()} != masks0
    _same(g, "verify", obs, 7)
    build_masks(g, threshold=0.5)                       # and come back
    again = _same(g, "verify", obs, 7)
    assert np.array_equal(np.asarray(again.samples), np.asarray(base.samples))
    g.units["verify"].masks.output_own_input = not g.units["verify"].masks.output_own_input
    _same(g, "verify", [], 8)
    _same(g, "verify", obs, 9)
    assert base.conditioned


def test_dropin_returns_reference_type_when_patched():
    g, _ = _setup()
    import pdgsim
    from pdgsim.estimator import RemainingDemand
    from pdgsim.pdgraph import RateProfile
    from pdgsim.sched import gittins_rank
    from paper_2506_14851_b200 import integration
    from paper_2506_14851_b200.estimator import monte_carlo_remaining_demand as ours
    integration.patch_pdgsim(pdgsim)
    try:
        r = ours(g, "extract", [], RateProfile(), 256, 5)
        assert isinstance(r, RemainingDemand)
        assert gittins_rank(r, 0.0) > 0          # sched._samples_of path
    finally:
        integration.restore()
    r = ours(g, "extract", [], RateProfile(), 256, 5)
    assert list(r) == r.samples and len(r) == 256
