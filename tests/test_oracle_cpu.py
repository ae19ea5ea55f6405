"""Pin the CPU oracle (oracle/pdg_oracle.py) to the reference's own outputs.

The golden fixtures were produced by running the reference itself
(tests/golden/make_golden.py); these tests need no GPU and no /root/reference.
"""

import hashlib

import numpy as np
import pytest

from oracle import pdg_oracle as O


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _obs(lst):
    return [O.OObs(o["unit_id"], o["input_len"], o["output_len"], o["parallelism"])
            for o in lst]


@pytest.fixture(scope="module")
def ograph(kb_graphs):
    return {k: O.graph_from_kb(v) for k, v in kb_graphs.items()}


def test_mc_cases_bit_exact(ograph, mc_cases, mc_full):
    for c in mc_cases["cases"]:
        r = O.mc_remaining_demand(ograph[c["graph"]], c["current"], _obs(c["obs"]),
                                  c["n"], c["seed"], c["visit_cap"])
        assert _sha(r.samples) == c["sha256"], c
        assert r.conditioned == c["conditioned"]
        assert r.capped == c["capped"]
        if "full" in c:
            np.testing.assert_array_equal(r.samples, mc_full[c["full"]])


def test_config1_mc_calls_bit_exact(ograph, config1_golden):
    calls = config1_golden["mc_calls"]
    assert len(calls) == config1_golden["n_mc_calls"] > 3000
    for c in calls[::3]:
        r = O.mc_remaining_demand(ograph[c["graph"]], c["current"], _obs(c["obs"]),
                                  c["n"], c["seed"], c["visit_cap"])
        assert _sha(r.samples) == c["sha256"]
        assert r.conditioned == c["conditioned"]
    assert any(c["conditioned"] for c in calls)


def test_binning(binning_golden):
    for c in binning_golden:
        b = O.bucketize(c["samples"], c["bucket_count"])
        assert [list(e) + [p] for e, p in zip(b.edges(), b.probs.tolist())] == c["buckets"]
        assert b.midpoints().tolist() == c["values"]
        assert b.probs.tolist() == c["probs"]
        assert b.boundaries() == c["boundaries"]
        assert [b.index_of(q) for q in c["queries"]] == c["index"]
        assert [O.survival(c["samples"], q) for q in c["queries"]] == c["survival"]


@pytest.mark.parametrize("tag", ["hand", "r10", "r256", "cfg1"])
def test_gittins(gittins_golden, tag):
    g = gittins_golden
    r = O.gittins_rank_batch(g[f"{tag}_values"], g[f"{tag}_probs"], g[f"{tag}_ages"])
    np.testing.assert_array_equal(np.isnan(r), np.isnan(g[f"{tag}_ranks"]))
    ok = ~np.isnan(r)
    np.testing.assert_allclose(r[ok], g[f"{tag}_ranks"][ok], rtol=1e-12)


def test_gittins_hand_values(gittins_golden):
    # test_sched.py:40-48 / 179-185 known answers
    r = gittins_golden["hand_ranks"]
    assert r[0] == pytest.approx(6.0) and r[1] == pytest.approx(4.0)
    assert r[2] == pytest.approx(8.0) and np.isnan(r[3]) and np.isnan(r[4])
    assert O.gittins_rank_samples([1.0, 1.0, 4.0, 9.0], 0.5) == pytest.approx(
        O.gittins_rank_batch(gittins_golden["pts_values"][None],
                             gittins_golden["pts_probs"][None], np.array([0.5]))[0])


def test_prewarm(prewarm_golden):
    for c in prewarm_golden:
        got = O.plan_prewarm(c["samples"], c["bucket_count"], c["p_s"], c["t_p"],
                             c["knob"], c["now"])
        if c["plan"] is None:
            assert got is None
        else:
            assert list(got) == c["plan"], c


def test_exact_mean_matches_reference_fixtures(ograph):
    # test_estimator.py:242-253 known answers
    assert O.exact_mean(ograph["point"], "a") == pytest.approx(5.0)
    assert O.exact_mean(ograph["chain"], "a") == pytest.approx(7.0)
    assert O.exact_mean(ograph["branch"], "a") == pytest.approx(7.0)
    with pytest.raises(ValueError):
        O.exact_mean(ograph["selfloop"], "a")
