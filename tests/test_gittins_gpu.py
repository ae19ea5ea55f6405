"""K1 parity on the GPU: the sm_100a scorers against the CPU oracle and the
reference's golden outputs (tests/golden/gittins.npz)."""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle import pdg_oracle as O
from tests.helpers import hist_rows, oracle_keys

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2506_14851_b200 import sched
    return sched


@pytest.mark.parametrize("tag", ["hand", "r10", "r256", "cfg1"])
def test_rank_batch_matches_reference_golden(S, gittins_golden, tag):
    g = gittins_golden
    got = S.gittins_rank_batch(g[f"{tag}_values"], g[f"{tag}_probs"], g[f"{tag}_ages"])
    want = g[f"{tag}_ranks"]
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    np.testing.assert_allclose(got[ok], want[ok], rtol=1e-12)


def test_rank_batch_known_answers(S):
    # test_sched.py:40-52, 80-91
    assert S.gittins_rank_points([10.0], [1.0], 4.0) == pytest.approx(6.0)
    assert S.gittins_rank_points([2.0, 10.0], [0.5, 0.5], 0.0) == pytest.approx(4.0)
    assert S.gittins_rank_points([2.0, 10.0], [0.5, 0.5], 2.0) == pytest.approx(8.0)
    with pytest.raises(S.ExhaustedDistributionError):
        S.gittins_rank_points([3.0], [1.0], 3.0)
    for age in (0.0, 0.5, 2.0, 5.0):
        assert S.gittins_rank([1.0, 1.0, 4.0, 9.0], age) == pytest.approx(
            O.gittins_rank_samples([1.0, 1.0, 4.0, 9.0], age), rel=1e-12)


def test_rank_batch_random_vs_oracle(S):
    rng = np.random.default_rng(5)
    for n, b in [(1, 1), (7, 3), (1000, 10), (3000, 64), (500, 256), (50, 1000), (3, 2049)]:
        v = np.sort(rng.lognormal(3, 1.5, (n, b)), axis=1)
        p = rng.lognormal(0, 2, (n, b))
        p[rng.random((n, b)) < 0.25] = 0.0
        p /= np.maximum(p.sum(axis=1, keepdims=True), 1e-300)
        a = rng.uniform(0, 1.2, n) * v[:, -1]
        got = S.gittins_rank_batch(v, p, a)
        want = O.gittins_rank_batch(v, p, a)
        np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
        ok = ~np.isnan(want)
        np.testing.assert_allclose(got[ok], want[ok], rtol=1e-11)


def test_rank_batch_empty_and_zero_width(S):
    assert S.gittins_rank_batch(np.zeros((0, 4)), np.zeros((0, 4)), np.zeros(0)).shape == (0,)
    assert np.isnan(S.gittins_rank_batch(np.zeros((2, 0)), np.zeros((2, 0)), np.zeros(2))).all()


def _inst(i, vals, probs, age, arrival):
    return SimpleNamespace(app_instance_id=f"app-{i:05d}", arrival_time=arrival,
                           tiebreak=(arrival, f"app-{i:05d}"), remaining=object(),
                           shifted_values=np.asarray(vals), bucket_probs=np.asarray(probs),
                           bucket_width=len(vals), attained_service=age, estimate_age=0.0,
                           last_refresh=-np.inf, observation_pending=False,
                           overrun_flagged=False, tenant_id="t", deadline=None)


def test_refresh_priorities_ragged_and_overrun(S):
    rng = np.random.default_rng(9)
    insts, rv, rp, ages = [], [], [], []
    for i in range(200):
        k = int(rng.integers(1, 12))
        vals = np.sort(rng.uniform(1, 100, k))
        probs = rng.uniform(0, 1, k)
        probs /= probs.sum()
        age = float(rng.uniform(0, 110))
        insts.append(_inst(i, vals, probs, age, float(i)))
        rv.append(vals)
        rp.append(probs)
        ages.append(age)
    res = S.refresh_priorities(insts, now=10.0, bucket_period=5.0)
    keys, bad = O.refresh_keys(rv, rp, ages)
    assert res.refreshed == [a.app_instance_id for a in insts]
    for inst, k, b in zip(insts, keys, bad):
        assert res.priorities[inst.app_instance_id].key == pytest.approx(k, rel=1e-12)
        assert inst.overrun_flagged == bool(b)
        assert inst.last_refresh == 10.0
    assert bad.any()
    # not due -> no-op (test_sched.py:198-203)
    res2 = S.refresh_priorities(insts, now=11.0, bucket_period=5.0)
    assert res2.refreshed == [] and res2.priorities == {}
    with pytest.raises(ValueError):
        S.refresh_priorities([], now=0.0, bucket_period=0.0)


@pytest.mark.parametrize("b,ragged", [(1, False), (10, False), (64, False), (64, True),
                                      (256, False), (256, True), (300, False),
                                      (1000, True)])
def test_hist_queue_vs_oracle(b, ragged):
    from paper_2506_14851_b200.queue import HistQueue
    rng = np.random.default_rng(b + 7 * ragged)
    n = 4000 if b <= 256 else 800
    rows = hist_rows(rng, n, b, ragged=ragged)
    q = HistQueue(n, b)
    q.load_rows(rows["lo"], rows["width"], rows["est_age"], rows["nbins"], rows["nsamp"],
                rows["counts"], age=rows["age"])
    q.score(penalty=2.0)
    got = q.key_f32[:n].cpu().numpy().astype(np.float64)
    flags = q.flags[:n].cpu().numpy()
    want, bad = oracle_keys(O, rows)
    np.testing.assert_array_equal(flags == 1, bad)
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() < 1e-5, (rel.max(), np.argmax(rel))


def test_hist_queue_full_size_and_order():
    """BASELINE config-2 shape (100k x 256): every key within 1e-5 of the
    float64 oracle; the global order equals the oracle's except inside ties
    whose keys agree to 1e-5."""
    import torch
    from paper_2506_14851_b200.queue import HistQueue
    rng = np.random.default_rng(2026)
    n, b = 100_000, 256
    rows = hist_rows(rng, n, b, degenerate_frac=0.01, exhaust_frac=0.01)
    tb = rng.permutation(n)
    q = HistQueue(n, b)
    q.load_rows(rows["lo"], rows["width"], rows["est_age"], rows["nbins"], rows["nsamp"],
                rows["counts"], age=rows["age"], tiebreak=tb)
    q.score()
    order = q.order().cpu().numpy()
    torch.cuda.synchronize()
    got = q.key_f32[:n].cpu().numpy().astype(np.float64)
    want, _ = oracle_keys(O, rows)
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() < 1e-5, rel.max()
    assert sorted(order.tolist()) == list(range(n))
    ref_order = np.lexsort((tb, want))            # (key, arrival order)
    # positions may differ only between keys equal within tolerance
    wk = want[order]
    assert np.all(wk[1:] >= wk[:-1] * (1 - 2e-5) - 1e-12)
    mism = order != ref_order
    if mism.any():
        a, bb = want[order[mism]], want[ref_order[mism]]
        assert np.all(np.abs(a - bb) <= 2e-5 * np.maximum(a, bb))


def test_rank_samples_bit_exact_vs_oracle(S):
    """Sample form on the device (pdg_gittins_rank_samples_host) equals the
    reference-pinned oracle bit for bit (tests/test_gittins_samples_cpu.py)."""
    from tests.test_gittins_samples_cpu import cases
    for s, age in cases(1, 80) + [([3.0] * 16384, 1.0), (list(np.arange(16384.0)), 100.5)]:
        if any(x > age for x in s):
            assert S.gittins_rank(s, age) == O.gittins_rank_samples(s, age), (len(s), age)
        else:
            with pytest.raises(S.ExhaustedDistributionError):
                S.gittins_rank(s, age)
    with pytest.raises(S.EstimationError):
        S.gittins_rank([], 0.0)


@pytest.mark.parametrize("b,ragged,nsamp", [(8, False, 512), (64, True, 512), (200, False, 512),
                                            (256, False, 512), (256, True, 512),
                                            (256, False, 60000)])
def test_hist_queue_quad_path_vs_oracle(b, ragged, nsamp):
    """Queues large enough for the 4-lanes-per-row kernel (gittins_quad_kernel):
    narrow strides, ragged rows, dead prefixes at every offset, exhausted and
    degenerate rows, exact-support ages, sample counts up to the u16 limit;
    then a scattered subset re-scored through row_idx."""
    import torch
    from paper_2506_14851_b200.queue import HistQueue
    rng = np.random.default_rng(1000 + b + 7 * ragged)
    n = 20_000
    rows = hist_rows(rng, n, b, nsamp=nsamp, ragged=ragged, degenerate_frac=0.03,
                     exhaust_frac=0.03, on_support_frac=0.05)
    q = HistQueue(n, b)
    q.load_rows(rows["lo"], rows["width"], rows["est_age"], rows["nbins"], rows["nsamp"],
                rows["counts"], age=rows["age"])
    q.score(penalty=2.0)
    got = q.key_f32[:n].cpu().numpy().astype(np.float64)
    flags = q.flags[:n].cpu().numpy()
    want, bad = oracle_keys(O, rows)
    np.testing.assert_array_equal(flags == 1, bad)
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() < 1e-5, (rel.max(), np.argmax(rel))
    # subset through row_idx: the other rows keep their keys
    sub = np.sort(rng.choice(n, 6000, replace=False)).astype(np.int32)
    q.key_f32.zero_()
    q.score(penalty=2.0, rows=torch.tensor(sub, device=q.key_f32.device))
    got2 = q.key_f32[:n].cpu().numpy().astype(np.float64)
    assert np.all(got2[np.setdiff1d(np.arange(n), sub)] == 0.0)
    np.testing.assert_array_equal(got2[sub], got[sub])


@pytest.mark.parametrize("n", [4736, 4741, 33_333])
def test_hist_queue_pair_path_partial_tiles(n):
    """Queue sizes at and just past the pair kernel's threshold and with a
    partial last 16-row tile: every row scored, none written twice."""
    from paper_2506_14851_b200.queue import HistQueue
    rng = np.random.default_rng(n)
    rows = hist_rows(rng, n, 256, degenerate_frac=0.02, exhaust_frac=0.02)
    q = HistQueue(n + 37, 256)                     # capacity above n: rows past n untouched
    q.load_rows(rows["lo"], rows["width"], rows["est_age"], rows["nbins"], rows["nsamp"],
                rows["counts"], age=rows["age"])
    q.key_f32.fill_(-1.0)
    q.score(penalty=2.0, n=n)
    got = q.key_f32.cpu().numpy().astype(np.float64)
    want, bad = oracle_keys(O, rows)
    rel = np.abs(got[:n] - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() < 1e-5, (rel.max(), np.argmax(rel))
    assert np.all(got[n:] == -1.0)
    np.testing.assert_array_equal(q.flags[:n].cpu().numpy() == 1, bad)
