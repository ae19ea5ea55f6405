"""K6 (config 4): micro-batched refinement events over a resident queue --
each event's re-estimate is bit-identical to the reference Monte Carlo with
the observation (K3 conditioning), its key is rescored in place, and the
global order stays a sorted permutation."""

import numpy as np
import pytest

from oracle import pdg_oracle as O
from tools import synth

pytestmark = pytest.mark.gpu

TEMPLATES = ["code-gen", "fact-verify", "verify-chain-bimodal", "bimodal", "plan-execute",
             "react-loop", "fanout-reduce", "cond"]


def test_event_stream_parity(kb_graphs):
    import torch
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.queue import HistQueue
    from paper_2506_14851_b200.stream import RefinementStream
    graphs = {k: graph_from_kb(kb_graphs[k]) for k in TEMPLATES}
    ogs = {k: O.graph_from_kb(kb_graphs[k]) for k in TEMPLATES}
    n = 20000
    q = synth.template_queue(graphs, n, seed=3)
    eng = DemandEngine(graphs)
    dev = eng.device
    hq = HistQueue(n, 64)
    gi = torch.from_numpy(q["graph"]).to(dev)
    ui = torch.from_numpy(q["unit"].copy()).to(dev)
    seeds = torch.arange(n, dtype=torch.int64, device=dev) * 7919
    eng.run(gi, ui, seeds, n=512, bucket_count=64, queue=hq)
    hq.est_age[:n] = 0.0
    hq.age[:n] = 0.0
    hq.n = n
    hq.score()
    st = RefinementStream(eng, hq, gi, ui, bucket_count=64)
    ev = synth.events(graphs, q, 3000, seed=5)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    obs_unit = t(ev["completed"], torch.int32)
    for lo in range(0, 3000, 500):                       # micro-batches of 500 events
        sl = slice(lo, lo + 500)
        st.process(t(ev["app"][sl], torch.int32), t(ev["next"][sl], torch.int32),
                   t(ev["seed"][sl], torch.int64), obs_unit[sl],
                   t(ev["obs"][sl], torch.float64), t(np.full(500, 3.0), torch.float64))
    inc = st.order_slots.clone()                         # K5b: merged batch by batch
    order = st.order().cpu().numpy()                     # K5: full re-sort
    torch.cuda.synchronize()
    np.testing.assert_array_equal(inc.cpu().numpy(), order)
    keys = hq.key_f32[:n].cpu().numpy()
    assert sorted(order.tolist()) == list(range(n))
    assert np.all(np.diff(keys[order]) >= 0)
    assert (ui.cpu().numpy()[ev["app"]] == ev["next"]).all()
    # bit-exact re-estimates for a sample of events
    lo_ = hq.lo.cpu().numpy()
    cnt = hq.counts.cpu().numpy()
    rng = np.random.default_rng(0)
    conditioned = 0
    for e in rng.choice(3000, 150, replace=False):
        a = ev["app"][e]
        nm = q["names"][q["graph"][a]]
        og = ogs[nm]
        order_u = sorted(og.units)
        obs = [O.OObs(order_u[ev["completed"][e]], *ev["obs"][e][:2], int(ev["obs"][e][2]))]
        want = O.mc_remaining_demand(og, order_u[ev["next"][e]], obs, 512, int(ev["seed"][e]))
        conditioned += want.conditioned
        b = O.bucketize(want.samples.tolist(), 64)
        assert lo_[a] == b.lo
        np.testing.assert_array_equal(cnt[a, :b.k], b.counts)
        v = b.midpoints() + 3.0
        r = O.gittins_rank_batch(v[None], b.probs[None], np.array([3.0]))[0]
        assert abs(keys[a] - r) <= 1e-5 * r
    assert conditioned > 0


def test_sharded_stream_single_rank_matches(kb_graphs):
    """ShardedRefinementStream (routing + gathered updates + merged global
    order) on one rank equals the plain stream batch by batch."""
    import torch
    from paper_2506_14851_b200.distributed import ShardedRefinementStream
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.queue import HistQueue
    from paper_2506_14851_b200.stream import RefinementStream
    graphs = {k: graph_from_kb(kb_graphs[k]) for k in TEMPLATES}
    n = 8000
    q = synth.template_queue(graphs, n, seed=13)
    eng = DemandEngine(graphs)
    dev = eng.device
    streams = []
    for _ in range(2):
        hq = HistQueue(n, 64)
        gi = torch.from_numpy(q["graph"]).to(dev)
        ui = torch.from_numpy(q["unit"].copy()).to(dev)
        eng.run(gi, ui, torch.arange(n, dtype=torch.int64, device=dev) * 17, n=512,
                bucket_count=64, queue=hq)
        hq.est_age[:n] = 0.0
        hq.age[:n] = 0.0
        hq.n = n
        hq.score()
        streams.append(RefinementStream(eng, hq, gi, ui, bucket_count=64))
    plain = streams[0]
    plain.order()
    sharded = ShardedRefinementStream(streams[1], n)
    ev = synth.events(graphs, q, 1200, seed=15)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    for lo in range(0, 1200, 300):
        sl = slice(lo, lo + 300)
        args = (t(ev["next"][sl], torch.int32), t(ev["seed"][sl], torch.int64),
                t(ev["completed"][sl], torch.int32), t(ev["obs"][sl], torch.float64),
                t(np.full(300, 2.0), torch.float64))
        plain.process(t(ev["app"][sl], torch.int32), *args)
        got = sharded.process(t(ev["app"][sl], torch.int64), *args)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), plain.order_slots.cpu().numpy())


def test_event_stream_full_size_order(kb_graphs):
    """Config 4 at full size: a 1M-app queue, 5 micro-batches of 1000 events;
    the incrementally merged order equals a full re-sort, is a permutation and
    is sorted by (key, arrival)."""
    import torch
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.queue import HistQueue
    from paper_2506_14851_b200.stream import RefinementStream
    graphs = {k: graph_from_kb(kb_graphs[k]) for k in TEMPLATES}
    n = 1_000_000
    q = synth.template_queue(graphs, n, seed=23)
    eng = DemandEngine(graphs)
    dev = eng.device
    hq = HistQueue(n, 256)
    gi = torch.from_numpy(q["graph"]).to(dev)
    ui = torch.from_numpy(q["unit"].copy()).to(dev)
    eng.run(gi, ui, torch.arange(n, dtype=torch.int64, device=dev) * 13, n=512,
            bucket_count=256, queue=hq)
    hq.est_age[:n] = 0.0
    hq.age[:n] = 0.0
    hq.n = n
    hq.score()
    st = RefinementStream(eng, hq, gi, ui, bucket_count=256)
    st.order()
    ev = synth.events(graphs, q, 5000, seed=29)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    for lo in range(0, 5000, 1000):
        sl = slice(lo, lo + 1000)
        st.process(t(ev["app"][sl], torch.int32), t(ev["next"][sl], torch.int32),
                   t(ev["seed"][sl], torch.int64), t(ev["completed"][sl], torch.int32),
                   t(ev["obs"][sl], torch.float64), t(np.full(1000, 4.0), torch.float64))
    inc = st.order_slots.clone()
    full = st.order()
    assert torch.equal(inc, full)
    o = full.long()
    assert torch.equal(torch.sort(o).values, torch.arange(n, device=dev))
    k = hq.keys[:n][o]
    assert bool((k[1:] > k[:-1]).all())          # packed (key, arrival): strictly increasing
