"""Graph-bank limits (host side, no GPU): graphs of up to 64 units compile
(64-bit unit sets in the engine), wider ones are rejected up front."""
import numpy as np
import pytest

from tests.test_engine_gpu import _wide_graph_doc


@pytest.mark.parametrize("n_units", [32, 33, 64])
def test_bank_accepts_up_to_64_units(n_units):
    from paper_2506_14851_b200.graphs import GraphBank, graph_from_kb
    doc = _wide_graph_doc(np.random.default_rng(n_units), n_units=n_units)
    bank = GraphBank({"wide": graph_from_kb(doc)}, device="cpu")
    assert bank.max_units == n_units


def test_bank_rejects_65_units():
    from paper_2506_14851_b200.graphs import GraphBank, graph_from_kb
    doc = _wide_graph_doc(np.random.default_rng(65), n_units=65)
    with pytest.raises(ValueError, match="more than 64 units"):
        GraphBank({"wide": graph_from_kb(doc)}, device="cpu")
