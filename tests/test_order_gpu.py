"""K5 pdg_order (csrc/sort.cu, one cooperative kernel): a stable radix sort of
packed (key << 32 | tiebreak) words with a u32 payload, equal to numpy's
stable argsort on the sorted bits (the reference's (key, arrival) order,
sched.py:191-192, simcore.py:339-344)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _order(keys_np, slots_np, begin_bit):
    import torch
    from paper_2506_14851_b200 import _lib
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    n = keys_np.size
    k = torch.from_numpy(keys_np.view(np.int64)).to(dev)
    s = torch.from_numpy(slots_np.view(np.int32)).to(dev)
    ko, so = torch.empty_like(k), torch.empty_like(s)
    tb = int(L.pdg_order_temp_bytes(n))
    temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
    _lib.check(L.pdg_order(_lib.ptr(k), _lib.ptr(ko), _lib.ptr(s), _lib.ptr(so), n, begin_bit,
                           _lib.ptr(temp), temp.numel(), _lib.stream_ptr()), "pdg_order")
    torch.cuda.synchronize()
    return ko.cpu().numpy().view(np.uint64), so.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("n", [1, 2, 1023, 1024, 1025, 4097, 100_000, 1_000_000])
@pytest.mark.parametrize("begin_bit", [32, 0])
def test_order_matches_stable_argsort(n, begin_bit):
    rng = np.random.default_rng(n + begin_bit)
    # few distinct float keys (heavy ties) and arbitrary tiebreak words
    fk = rng.choice(rng.uniform(0, 100, max(2, n // 50)).astype(np.float32), n)
    hi = fk.view(np.uint32).astype(np.uint64) << np.uint64(32)
    lo = rng.integers(0, 2**32, n, dtype=np.uint64)
    keys = hi | lo
    slots = rng.permutation(n).astype(np.uint32)
    got_k, got_s = _order(keys, slots, begin_bit)
    sort_on = keys >> np.uint64(32) if begin_bit == 32 else keys
    ref = np.argsort(sort_on, kind="stable")
    np.testing.assert_array_equal(got_k, keys[ref])
    np.testing.assert_array_equal(got_s, slots[ref])


def test_order_zero_length():
    got_k, got_s = _order(np.zeros(0, np.uint64), np.zeros(0, np.uint32), 32)
    assert got_k.size == 0 and got_s.size == 0


@pytest.mark.parametrize("n,m", [(1, 1), (1000, 0), (1000, 1), (5000, 1000), (100_000, 1000),
                                 (100_000, 4096), (200_000, 6000), (3000, 3000)])
def test_order_update_equals_full_sort(n, m):
    """K5b pdg_order_update (one cooperative kernel): the previous order minus
    m re-scored rows merged with their new keys equals a full sort of the
    updated keys; the mark buffer is left zeroed.  m > 4096 takes the
    pre-sorted batch path."""
    import torch
    from paper_2506_14851_b200 import _lib
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(n * 7 + m)
    fk = rng.choice(rng.uniform(0, 10, max(2, n // 20)).astype(np.float32), n)
    keys = (fk.view(np.uint32).astype(np.uint64) << np.uint64(32)) | np.arange(n, dtype=np.uint64)
    order = np.argsort(keys, kind="stable")
    rows = rng.choice(n, m, replace=False).astype(np.int32)
    new = keys.copy()
    nf = rng.uniform(0, 10, m).astype(np.float32)
    new[rows] = (nf.view(np.uint32).astype(np.uint64) << np.uint64(32)) | rows.astype(np.uint64)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)  # noqa: E731
    k_all = t(new, np.int64)
    ski, ssi = t(keys[order], np.int64), t(order.astype(np.uint32), np.int32)
    rw = t(rows, np.int32) if m else torch.zeros(1, dtype=torch.int32, device=dev)
    mark = torch.zeros(n, dtype=torch.uint8, device=dev)
    sko, sso = torch.empty_like(ski), torch.empty_like(ssi)
    tb = int(L.pdg_order_update_temp_bytes(n, m))
    temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
    _lib.check(L.pdg_order_update(_lib.ptr(k_all), _lib.ptr(ski), _lib.ptr(ssi), n, _lib.ptr(rw),
                                  m, _lib.ptr(mark), _lib.ptr(sko), _lib.ptr(sso),
                                  _lib.ptr(temp), temp.numel(), _lib.stream_ptr()),
               "pdg_order_update")
    torch.cuda.synchronize()
    want = np.argsort(new, kind="stable")
    np.testing.assert_array_equal(sso.cpu().numpy().view(np.uint32), want.astype(np.uint32))
    np.testing.assert_array_equal(sko.cpu().numpy().view(np.uint64), new[want])
    assert int(mark.sum().item()) == 0
