"""Correlation masks: the oracle's build_masks is the
reference's build_masks (flags and the Pearson values, bit for bit)."""

import gzip
import json
import os

import pytest

from oracle import pdg_oracle as O
from tests.dispatch_hook import ROOT

HAVE_REF = any(os.path.isdir(p) for p in ("/root/reference/pkg/src",
                                          os.path.join(ROOT, "baseline", "_ref")))


@pytest.mark.skipif(not HAVE_REF, reason="reference pdgsim not available")
def test_oracle_masks_match_reference():
    from tests.dispatch_hook import import_pdgsim
    import_pdgsim()
    from pdgsim.estimator import build_masks, pearson
    from pdgsim.errors import EstimationError
    from pdgsim.pdgraph import graph_from_dict
    with gzip.open(os.path.join(ROOT, "tests", "golden", "graphs.json.gz"), "rt") as fh:
        docs = json.load(fh)
    seen = 0
    for name, doc in docs.items():
        ref = graph_from_dict(doc)
        og = O.graph_from_kb(doc)
        build_masks(ref)
        got = O.build_masks(og)
        for uid, u in ref.units.items():
            assert u.masks.to_dict() == got[uid], (name, uid)
        for uid, mask, xs, ys in O.mask_jobs(og):
            try:
                want = pearson(xs, ys) if len(xs) >= 2 else None
            except EstimationError:
                want = None
            assert O.pearson(xs, ys) == want, (name, uid, mask)
            seen += want is not None
    assert seen > 20
