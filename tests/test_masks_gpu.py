"""Correlation masks on the GPU: every flag equals the oracle's (= the
reference's build_masks, tests/test_masks_cpu.py) and rho agrees to 1e-13
on all golden graphs and on freshly generated archetype graphs."""

import copy

import numpy as np
import pytest

from oracle import pdg_oracle as O

pytestmark = pytest.mark.gpu


def _check(docs):
    from paper_2506_14851_b200.graphs import build_masks, graph_from_kb
    graphs = {k: graph_from_kb(copy.deepcopy(v)) for k, v in docs.items()}
    got = build_masks(graphs)
    n_rho = 0
    for nm, doc in docs.items():
        og = O.graph_from_kb(doc)
        want = O.build_masks(og)
        for uid, u in graphs[nm].units.items():
            for k in O.MASK_NAMES:
                assert getattr(u.masks, k) == want[uid][k], (nm, uid, k)
        for uid, mask, xs, ys in O.mask_jobs(og):
            r = O.pearson(xs, ys)
            g = got[nm][uid][mask]
            assert (r is None) == (g is None), (nm, uid, mask)
            if r is not None:
                assert abs(g - r) <= 1e-13 * max(1.0, abs(r)), (nm, uid, mask, g, r)
                n_rho += 1
    return n_rho


def test_masks_golden_graphs(kb_graphs):
    assert _check(kb_graphs) > 20


def test_masks_generated_archetypes():
    from tests.dispatch_hook import import_pdgsim
    try:
        import_pdgsim()
    except ImportError:
        pytest.skip("pdgsim not installed in baseline/_ref")
    from pdgsim.pdgraph import graph_to_dict
    from pdgsim.workload import archetype
    docs = {}
    rng = np.random.default_rng(4)
    for kind in ("code-check", "verify-chain", "plan-execute", "react-loop", "fanout-reduce"):
        for i in range(4):
            docs[f"{kind}-{i}"] = graph_to_dict(archetype(
                kind, {"trials": int(rng.integers(20, 300)), "app_id": f"{kind}-{i}"},
                seed=int(rng.integers(0, 10**6))))
    assert _check(docs) > 40
