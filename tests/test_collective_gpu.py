"""K5 across ranks as one C call (pdg_rank_allgather_sort):
ncclAllGather + radix sort through the C ABI on a one-rank communicator made
with libnccl directly (the multi-rank exchange logic is covered on gloo by
tests/test_distributed_cpu.py)."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _UniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


def _nccl_comm():
    import torch  # noqa: F401  (loads the libnccl torch ships)
    nccl = C.CDLL("libnccl.so.2")
    uid = _UniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    return nccl, comm


@pytest.mark.parametrize("n", [1, 1000, 100_003])
def test_rank_allgather_sort_one_rank(n):
    import torch

    from paper_2506_14851_b200 import _lib
    from paper_2506_14851_b200.distributed import pack_keys, unpack_positions
    torch.cuda.set_device(0)
    nccl, comm = _nccl_comm()
    try:
        rng = np.random.default_rng(n)
        k = rng.lognormal(1, 1, n).astype(np.float32)
        k[rng.random(n) < 0.3] = 2.5                   # ties broken by arrival
        keys = pack_keys(torch.from_numpy(k), torch.arange(n)).cuda()
        gathered = torch.empty_like(keys)
        out = torch.empty_like(keys)
        L = _lib.lib()
        tb = int(L.pdg_rank_allgather_sort_temp_bytes(n, 1))
        temp = torch.empty(tb, dtype=torch.uint8, device="cuda")
        for bit in (0, 32):
            _lib.check(L.pdg_rank_allgather_sort(comm, _lib.ptr(keys), n, 1, _lib.ptr(gathered),
                                                 _lib.ptr(out), bit, _lib.ptr(temp), tb,
                                                 _lib.stream_ptr()), "pdg_rank_allgather_sort")
            torch.cuda.synchronize()
            assert torch.equal(gathered, keys)
            want = np.lexsort((np.arange(n), k.astype(np.float64)))
            np.testing.assert_array_equal(unpack_positions(out).cpu().numpy(), want)
    finally:
        nccl.ncclCommDestroy(comm)


def test_rank_allgather_sort_rejects_bad_args():
    from paper_2506_14851_b200 import _lib
    L = _lib.lib()
    assert L.pdg_rank_allgather_sort(None, None, 4, 1, None, None, 0, None, 0, None) != 0
