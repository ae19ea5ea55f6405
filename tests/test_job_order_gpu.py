"""Longest-first job order (pdg_graph_bank.unit_class) is a scheduling hint
only: the engine's rows are bit-identical with and without it, and the hint
classes follow the expected remaining walk length (E[u] = 1 + sum p E[v])."""

import numpy as np
import pytest
import torch

from paper_2506_14851_b200.graphs import UNIT_DTYPE, unit_classes
from tools import synth


def _expected_steps(w):
    A, U = w["succ_len"].shape
    P = np.zeros((A, U, U))
    cum = w["succ_cum"]
    p = cum - np.concatenate([np.zeros((A, U, 1)), cum[:, :, :-1]], axis=2)
    for s in range(w["succ_nxt"].shape[2]):
        v = w["succ_nxt"][:, :, s]
        a_i, u_i = np.nonzero(v >= 0)
        P[a_i, u_i, v[v >= 0]] += p[a_i, u_i, s]
    return np.linalg.solve(np.eye(U)[None] - P, np.ones((A, U, 1)))[..., 0]


def test_unit_classes_follow_expected_walk_length():
    w = synth.make(500, 64, seed=1000)
    A, U = w["succ_len"].shape
    units = np.zeros(A * U, dtype=UNIT_DTYPE)
    units["succ_off"] = np.arange(A * U) * w["succ_nxt"].shape[2]
    units["succ_len"] = w["succ_len"].reshape(-1)
    c = unit_classes(units, np.arange(A) * U, np.full(A, U), w["succ_cum"].reshape(-1),
                     w["succ_nxt"].reshape(-1))
    want = np.clip(np.floor(_expected_steps(w).reshape(-1)), 0, 15)
    assert np.abs(c.astype(int) - want).max() <= 1       # 32 sweeps vs the solve
    assert (c == want).mean() > 0.95


@pytest.mark.gpu
@pytest.mark.parametrize("n_apps", [1, 777, 20000])
def test_engine_rows_identical_with_and_without_job_order(n_apps):
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.queue import HistQueue

    dev = torch.device("cuda", 0)
    w = synth.make(n_apps, 256, seed=1000)
    eng = DemandEngine(synth.bank(w, device=str(dev)), device=str(dev))
    assert eng.c_bank.unit_class                            # the hint is on by default
    jb = synth.jobs(n_apps, seed=1001)
    g = torch.arange(n_apps, dtype=torch.int32, device=dev)
    u = torch.from_numpy(jb["unit"]).to(dev)
    s = torch.from_numpy(jb["seed"]).to(dev)
    rows = []
    for hint in (True, False):
        if not hint:
            eng.c_bank.unit_class = None
        q = HistQueue(n_apps, 256)
        eng.run(g, u, s, n=512, bucket_count=256, visit_cap=64, queue=q)
        torch.cuda.synchronize()
        rows.append([t[:n_apps].cpu().numpy().tobytes() for t in (q.counts, q.lo, q.width)])
    assert rows[0] == rows[1]
