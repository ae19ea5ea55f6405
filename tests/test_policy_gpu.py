"""K1c on the GPU: the engine's per-row mean (Python sum() semantics) and
worst case, and the SRPT-mean / LSTF keys and order over the device queue,
bit-identical to the oracle (which tests/test_policy_cpu.py pins to the
reference's compute_priority)."""

import numpy as np
import pytest

from oracle import pdg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine(kb_graphs):
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    return DemandEngine({k: graph_from_kb(v) for k, v in kb_graphs.items()})


def _run(engine, cases):
    import torch
    from paper_2506_14851_b200.queue import HistQueue
    dev = engine.device
    groups = {}
    for i, c in enumerate(cases):
        groups.setdefault((c["n"], c["visit_cap"]), []).append(i)
    q = HistQueue(len(cases), 64)
    samples = {}
    for (n, cap), idx in groups.items():
        t = lambda a, dt: torch.tensor(a, dtype=dt, device=dev)  # noqa: E731
        gi = [engine.bank.index[cases[i]["graph"]] for i in idx]
        ui = [engine.bank.local_unit(cases[i]["graph"], cases[i]["current"]) for i in idx]
        sd = [cases[i]["seed"] for i in idx]
        res = engine.run(t(gi, torch.int32), t(ui, torch.int32), t(sd, torch.int64), n=n,
                         bucket_count=64, visit_cap=cap, queue=q, slots=t(idx, torch.int32),
                         samples=True, mean=True)
        S = res["samples"].cpu().numpy()
        for r, i in enumerate(idx):
            samples[i] = S[r]
    q.n = len(cases)
    return q, samples


def test_engine_mean_and_worst_bit_exact(engine, mc_cases):
    cases = [dict(c, obs=[]) for c in mc_cases["cases"]]
    q, samples = _run(engine, cases)
    mean = q.mean[:len(cases)].cpu().numpy()
    worst = q.worst[:len(cases)].cpu().numpy()
    for i in range(len(cases)):
        s = samples[i].tolist()
        assert mean[i] == O.py_sum(s) / len(s), i
        assert worst[i] == max(s), i


def test_srpt_and_lstf_keys_and_order(engine, kb_graphs):
    import torch
    from paper_2506_14851_b200.sched import Policy
    rng = np.random.default_rng(21)
    names = ["depth8-100", "plan-execute", "react-loop", "code-gen", "fanout-reduce"]
    cases = []
    for k in range(600):
        nm = names[k % len(names)]
        og = O.graph_from_kb(kb_graphs[nm])
        uid = sorted(og.units)[int(rng.integers(0, len(og.units)))]
        cases.append({"graph": nm, "current": uid, "n": 512, "visit_cap": 64,
                      "seed": int(rng.integers(0, 2**62))})
    q, samples = _run(engine, cases)
    m = len(cases)
    est = rng.uniform(0, 30, m)
    att = est + rng.uniform(0, 1, m) * np.array([max(samples[i]) for i in range(m)]) * 1.2
    dl = rng.uniform(0, 4000, m)
    now = 1234.5
    q.est_age[:m] = torch.from_numpy(est).to(q.est_age.device)
    q.age[:m] = torch.from_numpy(att).to(q.age.device)
    q.deadline[:m] = torch.from_numpy(dl).to(q.deadline.device)
    for pol in (Policy.SRPT_MEAN, Policy.LSTF):
        q.score_policy(pol, now)
        got = q.key_f64[:m].cpu().numpy()
        if pol is Policy.SRPT_MEAN:
            want = [O.srpt_mean_key(samples[i].tolist(), att[i], est[i]) for i in range(m)]
        else:
            want = [O.lstf_key(samples[i].tolist(), att[i], est[i], dl[i], now)
                    for i in range(m)]
        np.testing.assert_array_equal(got, np.asarray(want))
        assert (np.asarray(want) < 0).any() or pol is Policy.SRPT_MEAN
        order = q.order().cpu().numpy()
        ref = sorted(range(m), key=lambda i: (want[i], i))
        np.testing.assert_array_equal(order, ref)


def test_policy_keys_reject_bad_policy():
    from paper_2506_14851_b200.queue import HistQueue
    q = HistQueue(4, 8)
    q.n = 4
    with pytest.raises(ValueError):
        q.score_policy("gittins", 0.0)
