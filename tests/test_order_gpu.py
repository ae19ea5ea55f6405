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
