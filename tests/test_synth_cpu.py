"""The benchmark's synthetic PDGraphs (tools/synth.py) are graphs the
reference itself accepts: every app's knowledge-base document loads through
pdgsim.pdgraph.graph_from_dict and passes PDGraph.validate (pdgraph.py:208-236,
344-409), including every branch successor being reachable."""
import pytest

from tests.dispatch_hook import import_pdgsim
from tools import synth


def test_synth_graphs_load_in_reference():
    try:
        import_pdgsim()
    except ImportError:
        pytest.skip("reference pdgsim not importable")
    from pdgsim.pdgraph import graph_from_dict
    w = synth.make(300, 256, seed=1000)
    for app in range(300):
        g = graph_from_dict(synth.kb_doc(w, app))
        g.validate()
