"""K2/K3/a4 parity on the GPU: demand-engine samples bit-identical to the
reference Monte Carlo (golden hashes recorded from the reference itself),
histogram rows identical to set_remaining's bucketing."""

import hashlib

import numpy as np
import pytest

from oracle import pdg_oracle as O

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


class Obs:
    def __init__(self, d):
        self.unit_id = d["unit_id"]
        self.input_len = d["input_len"]
        self.output_len = d["output_len"]
        self.parallelism = d["parallelism"]


@pytest.fixture(scope="module")
def engine(kb_graphs):
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    graphs = {k: graph_from_kb(v) for k, v in kb_graphs.items()}
    return DemandEngine(graphs)


def run_cases(engine, cases, bucket_count=64):
    """One launch per (n, visit_cap) group; returns samples, capped, flags, queue."""
    import torch
    dev = engine.device
    out = {}
    groups = {}
    for i, c in enumerate(cases):
        groups.setdefault((c["n"], c["visit_cap"]), []).append(i)
    for (n, cap), idx in groups.items():
        gi, ui, sd, ou, ov = [], [], [], [], []
        for i in idx:
            c = cases[i]
            gi.append(engine.bank.index[c["graph"]])
            ui.append(engine.bank.local_unit(c["graph"], c["current"]))
            sd.append(c["seed"])
            up, vals = engine.relevant_observation(c["graph"], c["current"],
                                                   [Obs(o) for o in c["obs"]])
            ou.append(up)
            ov.append(list(vals))
        t = lambda a, dt: torch.tensor(a, dtype=dt, device=dev)  # noqa: E731
        res = engine.run(t(gi, torch.int32), t(ui, torch.int32), t(sd, torch.int64),
                         t(ou, torch.int32), t(ov, torch.float64), n=n,
                         bucket_count=bucket_count, visit_cap=cap, samples=True)
        S = res["samples"].cpu().numpy()
        cp = res["capped"].cpu().numpy()
        fl = res["flags"].cpu().numpy()
        q = res["queue"]
        lo, w = q.lo.cpu().numpy(), q.width.cpu().numpy()
        nb, cnt = q.nbins.cpu().numpy(), q.counts.cpu().numpy()
        for r, i in enumerate(idx):
            out[i] = (S[r], int(cp[r]), int(fl[r]), (lo[r], w[r], int(nb[r]), cnt[r]))
    return out


def test_golden_mc_cases_bit_exact(engine, mc_cases, mc_full):
    cases = mc_cases["cases"]
    got = run_cases(engine, cases)
    for i, c in enumerate(cases):
        s, capped, flags, _ = got[i]
        assert _sha(s) == c["sha256"], (i, c["graph"], c["current"], c["n"])
        assert capped == c["capped"], i
        assert bool(flags & 1) == c["conditioned"], i
        if "full" in c:
            np.testing.assert_array_equal(s, mc_full[c["full"]])


@pytest.mark.parametrize("kinds", [0, 1, 4, 5])
def test_understated_bank_features_stay_exact(engine, mc_cases, kinds):
    """pdg_graph_bank.features is a speed hint: a walk kernel compiled
    without the LLM / own-input / K3 paths hands the jobs that need them to
    the serial kernel, so the golden cases stay bit-exact."""
    from paper_2506_14851_b200.graphs import FEATURES_VALID
    saved = engine.c_bank.features
    engine.c_bank.features = FEATURES_VALID | kinds
    try:
        cases = mc_cases["cases"]
        got = run_cases(engine, cases)
    finally:
        engine.c_bank.features = saved
    for i, c in enumerate(cases):
        s, capped, flags, _ = got[i]
        assert _sha(s) == c["sha256"], (kinds, i, c["graph"], c["current"], c["n"])
        assert capped == c["capped"], i
        assert bool(flags & 1) == c["conditioned"], i


def test_config1_all_mc_calls_bit_exact(engine, config1_golden):
    """Every Monte Carlo call of the config-1 simulation (3.5k calls, with
    online-refinement observations) reproduced in one batched launch."""
    calls = config1_golden["mc_calls"]
    got = run_cases(engine, calls)
    bad = [i for i, c in enumerate(calls) if _sha(got[i][0]) != c["sha256"]]
    assert not bad, (len(bad), bad[:5])
    assert all(bool(got[i][2] & 1) == c["conditioned"] for i, c in enumerate(calls))
    assert sum(c["conditioned"] for c in calls) > 0


def test_histogram_rows_match_set_remaining(engine, mc_cases):
    cases = [c for c in mc_cases["cases"] if c["n"] > 1]
    for bc in (1, 10, 64, 256):
        got = run_cases(engine, cases, bucket_count=bc)
        for i, c in enumerate(cases):
            s, _, _, (lo, w, nb, cnt) = got[i]
            b = O.bucketize(s.tolist(), bc)
            assert lo == b.lo and nb == b.k and w == b.width, (i, bc)
            np.testing.assert_array_equal(cnt[:b.k], b.counts)
            assert cnt[b.k:].sum() == 0


def test_drop_in_single_call(kb_graphs):
    from paper_2506_14851_b200 import estimator as E
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.errors import EstimationError

    class Env:
        prefill_rate, decode_rate = 10000.0, 50.0

    g = graph_from_kb(kb_graphs["bimodal"])
    og = O.graph_from_kb(kb_graphs["bimodal"])
    obs = [O.OObs("up", 400.0, 10.0, 1)]
    r = E.monte_carlo_remaining_demand(g, "down", obs, Env, n=4000, seed=3)
    want = O.mc_remaining_demand(og, "down", obs, 4000, 3)
    np.testing.assert_array_equal(np.asarray(r.samples), want.samples)
    assert r.conditioned is True and r.sample_count == 4000
    with pytest.raises(EstimationError):
        E.monte_carlo_remaining_demand(g, "down", [], Env, n=0, seed=1)
    with pytest.raises(EstimationError):
        E.monte_carlo_remaining_demand(g, "ghost", [], Env, n=5, seed=1)


def test_random_graphs_vs_oracle(engine, kb_graphs):
    """Depth-8 graphs, every unit as the current unit, large n (global
    scratch path) and tiny n."""
    rng = np.random.default_rng(77)
    cases = []
    for gid in ("depth8-100", "depth8-101", "depth8-102", "plan-execute", "react-loop",
                "fanout-reduce", "verify-chain-bimodal", "code-gen"):
        og = O.graph_from_kb(kb_graphs[gid])
        for uid in sorted(og.units):
            for n in (1, 37, 700):
                cases.append({"graph": gid, "current": uid, "obs": [], "n": n,
                              "seed": int(rng.integers(0, 2**62)), "visit_cap": 64})
    got = run_cases(engine, cases)
    ogs = {}
    for i, c in enumerate(cases):
        og = ogs.setdefault(c["graph"], O.graph_from_kb(kb_graphs[c["graph"]]))
        want = O.mc_remaining_demand(og, c["current"], [], c["n"], c["seed"], c["visit_cap"])
        np.testing.assert_array_equal(got[i][0], want.samples, err_msg=str(c))
        assert got[i][1] == want.capped


def _rejecting_seed(P, n, steps, window=200):
    """A seed whose stream hits a Lemire rejection inside the u32 halves the
    single-unit self-loop walk consumes (n walks, `steps` visits each)."""
    thr = (2**32 - P) % P
    per_step = n // 2 + (n % 2) + n       # words per step (halves region first)
    for seed in range(window):
        raw = np.random.default_rng(seed).bit_generator.random_raw(per_step * steps)
        for t in range(steps):
            base = t * per_step
            hw = raw[base: base + (n + 1) // 2]
            halves = np.concatenate([hw & 0xFFFFFFFF, hw >> 32]).astype(np.uint64)
            left = (halves * np.uint64(P)) & np.uint64(0xFFFFFFFF)
            if (left < thr).any():
                return seed
    return None


@pytest.mark.parametrize("n", [4000, 512, 96])      # mc_engine_kernel / mc_walk_kernel
def test_lemire_rejection_replayed_exactly(n):
    """numpy rejects a bounded draw with probability < P/2^32; the engine's
    warp vote must detect it and redraw the visit's bounded values with the
    sequential generator (mc_walk_kernel) or replay the application
    (mc_engine_kernel -> mc_serial_kernel)."""
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    P = max(range(900, 1001), key=lambda p: (2**32 - p) % p)
    steps = 64
    rng = np.random.default_rng(5)
    durs = rng.uniform(1.0, 2.0, P)
    doc = {"app_id": "rej", "entry_unit": "a", "units": [{
        "unit_id": "a", "backend": {"kind": "docker-exec", "image_id": "i"},
        "capacity": 1000, "bucket_count": 10,
        "records": [{"trial_id": t, "duration": float(durs[t]), "next_unit": "a"}
                    for t in range(P)]}]}
    seed = _rejecting_seed(P, n, steps, window=200 if n >= 4000 else 6000)
    if seed is None:
        pytest.skip("no rejecting seed found in the scan window")
    # the scan assumes a pure halves/doubles layout without earlier rejections;
    # the oracle is the judge either way
    eng = DemandEngine({"rej": graph_from_kb(doc)})
    og = O.graph_from_kb(doc)
    case = [{"graph": "rej", "current": "a", "obs": [], "n": n, "seed": seed,
             "visit_cap": steps}]
    got = run_cases(eng, case)
    want = O.mc_remaining_demand(og, "a", [], n, seed, steps)
    np.testing.assert_array_equal(got[0][0], want.samples)
    # n <= 512: redrawn inside the visit (flags bit 3); above: the sequential
    # replay kernel (bit 2)
    bit = 8 if n <= 512 else 4
    assert got[0][2] & bit, "the rejection path was not exercised"


def test_visit_cap_zero_and_empty_units(kb_graphs):
    """visit_cap=0: no step runs, every walk is capped at 0 (estimator.py:343);
    a graph with a sample-less unit raises like the reference sampler."""
    import torch
    from paper_2506_14851_b200 import estimator as E
    from paper_2506_14851_b200.errors import EstimationError
    from paper_2506_14851_b200.graphs import graph_from_kb

    class Env:
        prefill_rate, decode_rate = 10000.0, 50.0

    g = graph_from_kb(kb_graphs["chain"])
    r = E.monte_carlo_remaining_demand(g, "a", [], Env, n=64, seed=3, visit_cap=0)
    og = O.graph_from_kb(kb_graphs["chain"])
    want = O.mc_remaining_demand(og, "a", [], 64, 3, visit_cap=0)
    np.testing.assert_array_equal(np.asarray(r.samples), want.samples)
    assert r.capped_walks == want.capped == 64
    doc = dict(kb_graphs["chain"])
    doc["units"] = [dict(u) for u in doc["units"]]
    doc["units"][1]["records"] = []             # unit "b" loses its samples
    g2 = graph_from_kb(doc)
    with pytest.raises(EstimationError, match="no duration samples"):
        E.monte_carlo_remaining_demand(g2, "a", [], Env, n=8, seed=1)


def _wide_graph_doc(rng, n_units=32):
    """n_units units (32: the widest graph on 32-bit unit sets), up to 6
    successors per unit (the > 3 successor path), single-sample pools, LLM
    and duration units."""
    ids = [f"u{i:02d}" for i in range(n_units)]
    units = []
    for i, uid in enumerate(ids):
        llm = i % 3 == 0
        n_rec = 1 if i % 7 == 5 else int(rng.integers(20, 60))
        succ = rng.choice(n_units, size=int(rng.integers(1, 7)), replace=False)
        recs = []
        for t in range(n_rec):
            nxt = None if rng.random() < 0.25 else ids[int(rng.choice(succ))]
            r = {"trial_id": t, "next_unit": nxt}
            if llm:
                r.update(input_len=float(rng.integers(10, 3000)),
                         output_len=float(rng.integers(5, 900)), parallelism=1)
            else:
                r["duration"] = float(rng.lognormal(1, 1))
            recs.append(r)
        kind = {"kind": "llm-inference", "model_id": "m"} if llm else \
            {"kind": "docker-exec", "image_id": f"i{i}"}
        units.append({"unit_id": uid, "backend": kind, "capacity": 1000, "bucket_count": 10,
                      "records": recs})
    return {"app_id": "wide", "entry_unit": ids[0], "units": units}


def test_wide_graph_32_units_many_successors():
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    rng = np.random.default_rng(31)
    doc = _wide_graph_doc(rng)
    eng = DemandEngine({"wide": graph_from_kb(doc)})
    og = O.graph_from_kb(doc)
    assert max(len(u.succ) for u in og.units.values()) > 3
    cases = []
    for uid in sorted(og.units)[::3]:
        for n in (1, 37, 300, 512):
            cases.append({"graph": "wide", "current": uid, "obs": [], "n": n,
                          "seed": int(rng.integers(0, 2**62)), "visit_cap": 64})
    got = run_cases(eng, cases)
    for i, c in enumerate(cases):
        want = O.mc_remaining_demand(og, c["current"], [], c["n"], c["seed"], c["visit_cap"])
        np.testing.assert_array_equal(got[i][0], want.samples, err_msg=str(c))
        assert got[i][1] == want.capped


@pytest.mark.parametrize("n_units", [33, 48, 64])
def test_wide_graph_64bit_unit_sets(n_units):
    """Graphs past 32 units run on 64-bit unit sets (mc_walk_kernel<7, u64>
    for n <= 512, the compaction kernel above): samples bit-identical to the
    reference walk (estimator.py:326-353 has no unit cap)."""
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    rng = np.random.default_rng(n_units)
    doc = _wide_graph_doc(rng, n_units=n_units)
    eng = DemandEngine({"wide": graph_from_kb(doc)})
    og = O.graph_from_kb(doc)
    cases = []
    ids = sorted(og.units)
    for uid in ids[::5] + [ids[-1]]:
        for n in (1, 300, 512, 700):
            cases.append({"graph": "wide", "current": uid, "obs": [], "n": n,
                          "seed": int(rng.integers(0, 2**62)), "visit_cap": 64})
    got = run_cases(eng, cases)
    for i, c in enumerate(cases):
        want = O.mc_remaining_demand(og, c["current"], [], c["n"], c["seed"], c["visit_cap"])
        np.testing.assert_array_equal(got[i][0], want.samples, err_msg=str(c))
        assert got[i][1] == want.capped


@pytest.mark.parametrize("k", [2, 7, 64, 256, 1000])
def test_bucketize_boundary_samples_exact(k):
    """Bucketing divides by one reciprocal multiply and falls back to the exact
    division near bucket boundaries (common.cuh trunc_div): samples placed on
    and one or a few ulps around every boundary lo + j*w must land in the
    bucket Python's int((s - lo) / w) picks (distributions.py:98-101)."""
    from paper_2506_14851_b200.sched import bucketize_rows
    rng = np.random.default_rng(k)
    rows = []
    for r in range(24):
        lo = float(rng.uniform(-50, 500)) if r % 3 else 0.0
        wt = float(rng.lognormal(0, 2))
        j = np.arange(k + 1, dtype=np.float64)
        base = lo + j * wt
        s = np.concatenate([base, np.nextafter(base, np.inf), np.nextafter(base, -np.inf),
                            base + 4 * np.spacing(base), base - 4 * np.spacing(base)])
        s = s[(s >= lo) & (s <= base[-1])]
        s = rng.permutation(s)[:1024]
        s[0], s[1] = lo, base[-1]                     # pin min / max
        rows.append(s)
    n = min(len(x) for x in rows)
    X = np.stack([x[:n] for x in rows])
    lo, w, nb, cnt = bucketize_rows(X, k)
    for i in range(len(X)):
        want = O.bucketize(X[i], k)
        assert lo[i] == want.lo and nb[i] == want.k
        np.testing.assert_array_equal(cnt[i, :want.k], want.counts, err_msg=f"row {i}")
