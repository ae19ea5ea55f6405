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
