"""K4 on units with more than four successors and on malformed type tables:
_plan_prewarms plans every successor in sorted order (simcore.py:459-478), so
the trigger outputs are sized by the bank's largest fan-out and the need grid
sums every successor's p_s by backend type.  A C caller that passes fewer
slots than a unit's fan-out, or a type without a warmup entry, gets the
PDG_PLAN_OVERFLOW / PDG_PLAN_BAD_TYPE flags instead of a silently dropped plan."""

import ctypes as C

import numpy as np
import pytest

from oracle import pdg_oracle as O

pytestmark = pytest.mark.gpu

A, U, R = 5, 9, 64        # graphs, units per graph, service samples per unit


def _tables(seed=3):
    """Unit 0 of every graph fans out to units 1..8 (8 successors, repeated
    and missing types); the others have 0-2 successors."""
    import torch
    from paper_2506_14851_b200.prewarm import PrewarmTables
    rng = np.random.default_rng(seed)
    svc = np.sort(rng.uniform(0.5, 80.0, (A * U, R)), axis=1)
    s_off, s_len, s_nxt, s_p = [], [], [], []
    for a in range(A):
        for u in range(U):
            succ = list(range(1, U)) if u == 0 else ([u + 1] if u + 1 < U else [])
            if u == 3:
                succ = [4, 6]
            p = rng.dirichlet(np.ones(len(succ))) if succ else []
            s_off.append(len(s_nxt))
            s_len.append(len(succ))
            s_nxt.extend(succ)
            s_p.extend(p)
    utype = rng.integers(-1, 5, A * U)          # -1: no warm content
    utype[1:U:2] = 2                            # repeated types inside the fan-out
    tb = PrewarmTables(svc_sorted=svc.ravel(), svc_off=np.arange(A * U) * R,
                       svc_len=np.full(A * U, R), graph_base=np.arange(A) * U,
                       succ_off=s_off, succ_len=s_len, succ_nxt=s_nxt, succ_p=s_p,
                       unit_type=utype, n_types=5, device="cuda")
    jobs = [(a, u) for a in range(A) for u in range(U)] * 3
    g = torch.tensor([j[0] for j in jobs], dtype=torch.int32, device="cuda")
    u = torch.tensor([j[1] for j in jobs], dtype=torch.int32, device="cuda")
    nowv = rng.uniform(0, 40, len(jobs))
    now = torch.tensor(nowv, dtype=torch.float64, device="cuda")
    return tb, svc, s_off, s_len, s_nxt, s_p, utype, jobs, g, u, nowv, now


def test_wide_fanout_need_and_triggers():
    import torch
    tb, svc, s_off, s_len, s_nxt, s_p, utype, jobs, g, u, nowv, now = _tables()
    assert tb.max_succ == U - 1 and "unit_rec" not in tb.t
    win = np.sort(np.random.default_rng(5).uniform(0, 120, 32))
    need, agg = tb.need(g, u, now, torch.tensor(win, dtype=torch.float64, device="cuda"))
    need = need.cpu().numpy()
    warm = np.random.default_rng(6).uniform(0.0, 30.0, 5)
    has, trig, pe = tb.triggers(g, u, now, warm, 0.05, 16)
    assert has.shape == (len(jobs), U - 1)
    has, trig, pe = has.cpu().numpy(), trig.cpu().numpy(), pe.cpu().numpy()
    tot = np.zeros((5, 32))
    wide_plans = 0
    for i, (a, uu) in enumerate(jobs):
        k = a * U + uu
        succ = [(s_p[s_off[k] + q], int(utype[a * U + s_nxt[s_off[k] + q]]))
                for q in range(s_len[k])]
        want = O.need_grid(svc[k], succ, nowv[i], win, 5)
        tot += want
        np.testing.assert_allclose(need[i], want, rtol=1e-6, atol=1e-6)
        comp = [nowv[i] + s for s in svc[k]]
        for q, (p, ty) in enumerate(succ):
            w = O.plan_prewarm(comp, 16, p, warm[ty], 0.05, nowv[i]) if ty >= 0 else None
            assert bool(has[i, q]) == (w is not None), (i, q)
            if w is not None:
                assert (trig[i, q], pe[i, q]) == w
                wide_plans += q >= 4
        assert not has[i, len(succ):].any()
    assert wide_plans > 0
    np.testing.assert_allclose(agg.cpu().numpy(), tot, rtol=1e-6, atol=1e-6)


def test_c_abi_flags_overflow_and_bad_type():
    import torch
    from paper_2506_14851_b200 import _lib
    tb, svc, s_off, s_len, s_nxt, s_p, utype, jobs, g, u, nowv, now = _tables()
    L = _lib.lib()
    n, S = len(jobs), 4                              # fewer slots than unit 0's fan-out
    warm = torch.zeros(2, dtype=torch.float64, device="cuda")     # types 2.. have no entry
    has = torch.full((n, S), 7, dtype=torch.uint8, device="cuda")
    trig = torch.zeros((n, S), dtype=torch.float64, device="cuda")
    pe = torch.zeros((n, S), dtype=torch.float64, device="cuda")
    temp = torch.empty(int(L.pdg_prewarm_triggers_temp_bytes(n, S)), dtype=torch.uint8,
                       device="cuda")
    rc = L.pdg_prewarm_triggers(C.byref(tb.c), _lib.ptr(g), _lib.ptr(u), _lib.ptr(now), n, S,
                                _lib.ptr(warm), 2, 0.0, 16, _lib.ptr(has), _lib.ptr(trig),
                                _lib.ptr(pe), _lib.ptr(temp), temp.numel(), None)
    assert rc == 0
    h = has.cpu().numpy()
    for i, (a, uu) in enumerate(jobs):
        k = a * U + uu
        if s_len[k] > S:
            assert (h[i] == 2).all(), i                          # PDG_PLAN_OVERFLOW
            continue
        for q in range(S):
            if q >= s_len[k]:
                assert h[i, q] == 0
                continue
            ty = int(utype[a * U + s_nxt[s_off[k] + q]])
            assert h[i, q] == (3 if ty >= 2 else (0 if ty < 0 else 1)), (i, q, ty)
    assert L.pdg_prewarm_triggers(C.byref(tb.c), _lib.ptr(g), _lib.ptr(u), _lib.ptr(now), n, 0,
                                  _lib.ptr(warm), 2, 0.0, 16, _lib.ptr(has), _lib.ptr(trig),
                                  _lib.ptr(pe), _lib.ptr(temp), temp.numel(), None) != 0
    with pytest.raises(ValueError):
        tb.triggers(g, u, now, [1.0, 2.0], 0.1, 16)            # warmup shorter than types
    with pytest.raises(TypeError):
        tb.triggers(g.long(), u, now, np.ones(5), 0.1, 16)      # int64 indices
