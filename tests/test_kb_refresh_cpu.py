"""Template refresh: graphs.record_trial follows
pdgraph.record_trial (records, FIFO cap, branch frequencies), and an
incremental GraphBank.update equals a bank compiled from scratch."""

import os

import pytest

from tests.dispatch_hook import ROOT

HAVE_REF = any(os.path.isdir(p) for p in ("/root/reference/pkg/src",
                                          os.path.join(ROOT, "baseline", "_ref")))
pytestmark = pytest.mark.skipif(not HAVE_REF, reason="reference pdgsim not available")


def test_record_trial_matches_reference():
    from tests.dispatch_hook import import_pdgsim
    import_pdgsim()
    from pdgsim.pdgraph import record_trial as ref_record
    from paper_2506_14851_b200.graphs import record_trial
    from tests.kb_trials import setup
    base, kb, ref_trials, kb_trials = setup()
    for rt, kt in zip(ref_trials, kb_trials):
        ref_record(base, rt)
        record_trial(kb, kt)
    for uid, u in base.units.items():
        ku = kb.units[uid]
        assert [(r.trial_id, r.input_len, r.output_len, r.duration, r.next_unit)
                for r in u.records] == [(r.trial_id, r.input_len, r.output_len, r.duration,
                                         r.next_unit) for r in ku.records]
        assert len(ku.records) <= u.capacity
        assert u.successors == ku.successors


def test_record_trial_rejects_bad_trials():
    from paper_2506_14851_b200.graphs import GraphError, KBRecord, record_trial
    from tests.kb_trials import setup
    _, kb, _, kb_trials = setup(n_trials=1)
    with pytest.raises(GraphError):
        record_trial(kb, {"ghost": KBRecord(1, 1.0, 1.0, 1, 0.0, None)})
    t = dict(kb_trials[0])
    t.pop(kb.entry_unit)
    with pytest.raises(GraphError):
        record_trial(kb, t)


def test_bank_update_equals_fresh_compile():
    import gzip
    import json

    import torch

    from paper_2506_14851_b200.graphs import GraphBank, graph_from_kb, record_trial
    from tests.kb_trials import setup
    with gzip.open(os.path.join(ROOT, "tests", "golden", "graphs.json.gz"), "rt") as fh:
        docs = json.load(fh)
    _, kb, _, kb_trials = setup()
    graphs = {k: graph_from_kb(v) for k, v in list(docs.items())[:5]}
    graphs["vc"] = kb
    bank = GraphBank(graphs, device="cpu")
    for kt in kb_trials:
        record_trial(kb, kt)
    bank.update("vc")
    fresh = GraphBank(graphs, device="cpu")
    for f in ("units", "vals", "graph_base", "graph_n", "unit_capacity", "pool_off",
              "pool_len", "succ_cum", "succ_thr", "succ_nxt", "conds", "pairs"):
        assert torch.equal(getattr(bank, f), getattr(fresh, f)), f
    assert (bank.max_pairs, bank.max_unit_k) == (fresh.max_pairs, fresh.max_unit_k)
