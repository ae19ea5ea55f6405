"""K4 parity on the GPU: plan_prewarm bit-exact against the reference's own
outputs (tests/golden/prewarm.json, including the config-1 simulation's plan)
and the need-probability grid against the oracle."""

import numpy as np
import pytest

from oracle import pdg_oracle as O

pytestmark = pytest.mark.gpu


def test_plan_prewarm_batch_matches_reference(prewarm_golden):
    from paper_2506_14851_b200.prewarm import plan_prewarm_batch
    cases = prewarm_golden
    has, trig, pe = plan_prewarm_batch([c["samples"] for c in cases],
                                       [c["bucket_count"] for c in cases],
                                       [c["p_s"] for c in cases], [c["t_p"] for c in cases],
                                       [c["knob"] for c in cases], [c["now"] for c in cases])
    for i, c in enumerate(cases):
        if c["plan"] is None:
            assert not has[i], c
        else:
            assert has[i], c
            assert [trig[i], pe[i]] == c["plan"], (i, c, trig[i], pe[i])


def test_plan_prewarm_drop_in():
    from paper_2506_14851_b200.prewarm import PrewarmPlan, plan_prewarm

    class D:
        def __init__(self, xs, bc=10):
            self.samples, self.bucket_count = list(xs), bc

    assert plan_prewarm(D([60.0]), p_s=0.3, t_p=10.0, knob=0.5, now=0.0) is None
    p = plan_prewarm(D([60.0]), p_s=1.0, t_p=10.0, knob=0.5, now=0.0)
    assert p.trigger_time == pytest.approx(50.0) and p.p_e == pytest.approx(1.0)
    p = plan_prewarm(D([40.0, 80.0], 1), p_s=0.8, t_p=10.0, knob=0.4, now=0.0)
    assert p.trigger_time == pytest.approx(70.0) and p.p_e == pytest.approx(0.4)
    p = plan_prewarm(D([5.0]), p_s=0.6, t_p=50.0, knob=0.6, now=0.0)
    assert p.trigger_time == 0.0 and p.p_e < 0.6
    assert plan_prewarm(D([60.0]), 1.0, 10.0, 0.5, now=55.0).trigger_time == pytest.approx(55.0)
    with pytest.raises(ValueError):
        plan_prewarm(D([60.0]), 1.0, 10.0, 1.5, 0.0)
    with pytest.raises(ValueError):
        plan_prewarm(D([60.0]), 1.0, -1.0, 0.5, 0.0)
    with pytest.raises(ValueError):
        PrewarmPlan(None, 0.3, 1.0, 0.0, 0.3, 0.5)


def test_plan_prewarm_random_vs_oracle():
    from paper_2506_14851_b200.prewarm import plan_prewarm_batch
    rng = np.random.default_rng(4)
    J = 2000
    samples = [rng.uniform(0, 300, rng.integers(1, 400)).tolist() for _ in range(J)]
    bc = rng.choice([1, 5, 10, 64, 256], J)
    ps, tp, kn = rng.uniform(0, 1, J), rng.uniform(0, 80, J), rng.uniform(0, 1, J)
    now = np.where(rng.random(J) < 0.5, 0.0, rng.uniform(0, 250, J))
    has, trig, pe = plan_prewarm_batch(samples, bc, ps, tp, kn, now)
    for i in range(J):
        want = O.plan_prewarm(samples[i], int(bc[i]), ps[i], tp[i], kn[i], now[i])
        if want is None:
            assert not has[i]
        else:
            assert has[i] and (trig[i], pe[i]) == want, (i, want, trig[i], pe[i])


def test_need_grid_vs_oracle(kb_graphs):
    import torch
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.prewarm import PrewarmTables
    names = ["plan-execute", "code-gen", "fact-verify", "fanout-reduce", "react-loop",
             "depth8-100"]
    graphs = {k: graph_from_kb(kb_graphs[k]) for k in names}
    tb = PrewarmTables.from_graphs(graphs)
    rng = np.random.default_rng(8)
    jobs = [(gi, ui) for gi, k in enumerate(names) for ui in range(len(graphs[k].units))]
    jobs = jobs * 20
    g = torch.tensor([j[0] for j in jobs], dtype=torch.int32, device="cuda")
    u = torch.tensor([j[1] for j in jobs], dtype=torch.int32, device="cuda")
    nowv = rng.uniform(0, 50, len(jobs))
    nowv[::3] = rng.uniform(1e6, 1e9, len(nowv[::3]))   # completion times that round
    now = torch.tensor(nowv, dtype=torch.float64, device="cuda")
    win = np.sort(rng.uniform(0, 400, 32))
    win[:8] = np.sort(np.concatenate([graphs["code-gen"].units[x].duration_dist.samples[:2]
                                      for x in sorted(graphs["code-gen"].units)
                                      if not graphs["code-gen"].units[x].is_llm] +
                                     [np.array(win[:8])]))[:8]   # windows on sample values
    win = np.sort(win)
    wt = torch.tensor(win, dtype=torch.float64, device="cuda")
    need, agg = tb.need(g, u, now, wt)                          # window-index path
    need2, agg2 = tb.need(g, u, now, wt, window_index=False,    # per-app search path
                          unit_records=False)
    np.testing.assert_array_equal(need.cpu().numpy(), need2.cpu().numpy())
    need = need.cpu().numpy()
    T = tb.n_types
    tot = np.zeros((T, 32))
    for i, (gi, ui) in enumerate(jobs):
        gr = graphs[names[gi]]
        uid = sorted(gr.units)[ui]
        unit = gr.units[uid]
        if unit.is_llm:
            svc = [r.input_len / 1e4 + r.output_len / 50.0 for r in unit.records]
        else:
            svc = unit.duration_dist.samples
        succ = [(p, tb.type_ids.get(gr.units[v].warm_content, -1)
                 if gr.units[v].warm_content is not None else -1)
                for v, p in sorted(unit.successors.items())]
        want = O.need_grid(svc, succ, nowv[i], win, T)
        tot += want
        np.testing.assert_allclose(need[i], want, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(agg.cpu().numpy(), tot, rtol=1e-6, atol=1e-6)


def test_need_full_size_properties():
    """Config 5 at full size (1M apps x 16 types x 32 windows): need rows are
    probabilities, nondecreasing in the window, their per-window sum over
    types is at most the successors' total probability, the aggregate is the
    column sum, and a sample of apps equals the oracle."""
    import torch
    from paper_2506_14851_b200.prewarm import PrewarmTables
    from tools import synth
    A, U, R, T, N = 64, synth.U, 64, 16, 1_000_000
    w = synth.make(A, R, seed=31)
    rng = np.random.default_rng(32)
    svc = np.sort(w["dur"], axis=2)
    counts = np.zeros((A, U, U))
    for v in range(U):
        counts[:, :, v] = (w["nxt"] == v).sum(axis=2)
    s_len = w["succ_len"].reshape(-1)
    s_nxt = w["succ_nxt"].reshape(-1)
    s_p = np.zeros(A * U * synth.SLOT)
    for a_u in range(A * U):
        a, u = divmod(a_u, U)
        for q in range(s_len[a_u]):
            s_p[a_u * synth.SLOT + q] = counts[a, u, s_nxt[a_u * synth.SLOT + q]] / R
    utype = rng.integers(0, T, A * U)
    tb = PrewarmTables(svc_sorted=svc.reshape(-1), svc_off=np.arange(A * U) * R,
                       svc_len=np.full(A * U, R), graph_base=np.arange(A) * U,
                       succ_off=np.arange(A * U) * synth.SLOT, succ_len=s_len, succ_nxt=s_nxt,
                       succ_p=s_p, unit_type=utype, n_types=T)
    gi = rng.integers(0, A, N).astype(np.int32)
    ui = rng.integers(0, U, N).astype(np.int32)
    nowv = rng.uniform(0, 100, N)
    win = np.linspace(2.0, 64.0, 32)
    dev = "cuda"
    need, agg = tb.need(torch.from_numpy(gi).to(dev), torch.from_numpy(ui).to(dev),
                        torch.from_numpy(nowv).to(dev), torch.tensor(win, device=dev))
    assert need.shape == (N, T, 32)
    assert bool((need >= 0).all()) and bool((need <= 1.0 + 1e-6).all())
    assert bool((need[:, :, 1:] >= need[:, :, :-1]).all())        # CDF in the window
    psum = torch.from_numpy(s_p.reshape(A * U, synth.SLOT).sum(1)).to(dev)
    colsum = need.sum(1)                                           # [N, 32]
    bound = psum[torch.from_numpy(gi.astype(np.int64) * U + ui).to(dev)]
    assert bool((colsum <= bound[:, None] + 1e-5).all())
    torch.testing.assert_close(agg, need.double().sum(0), rtol=1e-9, atol=1e-6)
    sel = rng.choice(N, 300, replace=False)
    got = need[torch.from_numpy(sel).to(dev)].cpu().numpy()
    for i, a in enumerate(sel):
        g_, u_ = int(gi[a]), int(ui[a])
        base = (g_ * U + u_) * synth.SLOT
        succ = [(s_p[base + q], int(utype[g_ * U + s_nxt[base + q]]))
                for q in range(s_len[g_ * U + u_])]
        want = O.need_grid(svc[g_, u_], succ, nowv[a], win, T)
        np.testing.assert_allclose(got[i], want, rtol=1e-6, atol=1e-6)


def test_triggers_vs_oracle(kb_graphs):
    """Config 5's per-successor plans from the prewarm tables equal
    plan_prewarm on the completion distribution _plan_prewarms builds."""
    import torch
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.prewarm import PrewarmTables
    names = ["plan-execute", "code-gen", "fact-verify", "fanout-reduce", "react-loop",
             "depth8-100"]
    graphs = {k: graph_from_kb(kb_graphs[k]) for k in names}
    tb = PrewarmTables.from_graphs(graphs)
    rng = np.random.default_rng(18)
    jobs = [(gi, ui) for gi, k in enumerate(names) for ui in range(len(graphs[k].units))] * 10
    nowv = rng.uniform(0, 50, len(jobs))
    nowv[::4] = rng.uniform(1e6, 1e9, len(nowv[::4]))
    T = tb.n_types
    warm = rng.uniform(0.0, 30.0, T)
    g = torch.tensor([j[0] for j in jobs], dtype=torch.int32, device="cuda")
    u = torch.tensor([j[1] for j in jobs], dtype=torch.int32, device="cuda")
    now = torch.tensor(nowv, dtype=torch.float64, device="cuda")
    for knob, bc in ((0.3, 64), (0.05, 10)):
        has, trig, pe = tb.triggers(g, u, now, warm, knob, bc)
        has, trig, pe = has.cpu().numpy(), trig.cpu().numpy(), pe.cpu().numpy()
        planned = 0
        for i, (gi, ui) in enumerate(jobs):
            gr = graphs[names[gi]]
            unit = gr.units[sorted(gr.units)[ui]]
            if unit.is_llm:
                svc = [r.input_len / 1e4 + r.output_len / 50.0 for r in unit.records]
            else:
                svc = unit.duration_dist.samples
            comp = [nowv[i] + s for s in svc]
            for slot, (v, p) in enumerate(sorted(unit.successors.items())):
                wc = gr.units[v].warm_content
                ty = tb.type_ids.get(wc, -1) if wc is not None else -1
                want = (O.plan_prewarm(comp, bc, p, warm[ty], knob, nowv[i])
                        if ty >= 0 and svc else None)
                assert bool(has[i, slot]) == (want is not None), (i, slot)
                if want is not None:
                    planned += 1
                    assert trig[i, slot] == want[0] and pe[i, slot] == want[1], (i, slot)
            assert not has[i, len(unit.successors):].any()
        assert planned > 0
