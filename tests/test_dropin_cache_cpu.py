"""Host side of the drop-in engine cache: the fingerprint that decides when
the cached device tables are recompiled changes on every in-place mutation
the reference performs (FIFO-capped record_trial, build_masks), and only
then."""

import pytest

from tests.dispatch_hook import import_pdgsim


def test_fingerprint_tracks_in_place_mutation():
    try:
        import_pdgsim()
    except ImportError:
        pytest.skip("pdgsim not importable")
    from pdgsim.estimator import build_masks
    from pdgsim.pdgraph import UnitRecord, record_trial
    from pdgsim.workload import archetype
    from paper_2506_14851_b200.estimator import _fingerprint
    g = archetype("verify-chain", {"trials": 60, "capacity": 60, "bucket_count": 8}, seed=2)
    f0 = _fingerprint(g)
    assert _fingerprint(g) == f0                          # stable without mutation
    recs = {uid: u.records[3] for uid, u in g.units.items()}
    record_trial(g, {uid: UnitRecord(999, r.input_len, r.output_len, r.parallelism,
                                     r.duration, r.next_unit) for uid, r in recs.items()})
    assert all(len(u.records) == 60 for u in g.units.values())
    f1 = _fingerprint(g)
    assert f1 != f0                                       # same length, new content
    build_masks(g, threshold=0.999)
    f2 = _fingerprint(g)
    assert f2 != f1
    g.units["verify"].masks.output_own_input = not g.units["verify"].masks.output_own_input
    assert _fingerprint(g) != f2
