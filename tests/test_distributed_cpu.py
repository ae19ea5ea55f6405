"""K5 exchange on CPU: world_size-2 gloo processes shard a queue by arrival
order, pack their keys, all-gather them and obtain the reference global
order (key, arrival) -- the host-side logic of the multi-GPU path.  The sort
is injected (torch stable sort) because the product sort is the CUDA radix
sort; the kernels themselves are covered by the -m gpu tests."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_14851_b200.distributed import (SENTINEL, global_order, pack_keys,
                                               shard_range, unpack_positions)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stable_sort_high(keys):
    # stable sort on the high 32 bits only: relies on arrival-ordered input
    hi = keys >> 32
    idx = torch.sort(hi, stable=True).indices
    return keys[idx]


def _keys_for(n_total, seed):
    rng = np.random.default_rng(seed)
    k = rng.lognormal(2, 1, n_total).astype(np.float32)
    k[rng.random(n_total) < 0.2] = 7.0          # many exact ties
    k[:5] = 0.0
    return k


def _worker(rank, world, port, n_total, seed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = _keys_for(n_total, seed)
        lo, hi = shard_range(n_total, world, rank)
        local = pack_keys(torch.from_numpy(keys[lo:hi]), torch.arange(lo, hi))
        order = global_order(local, n_total, sort_fn=_stable_sort_high)
        full = global_order(local, n_total,
                            sort_fn=lambda k: torch.sort(k).values)   # full 64-bit sort
        out[rank] = (unpack_positions(order).numpy(), unpack_positions(full).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [10, 1001, 4096])
def test_two_rank_global_order(n_total):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, 3, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    keys = _keys_for(n_total, 3)
    want = np.lexsort((np.arange(n_total), keys.astype(np.float64)))
    for r in range(2):
        stable, full = out[r]
        np.testing.assert_array_equal(stable, want)
        np.testing.assert_array_equal(full, want)


def test_shard_ranges_cover():
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_pack_keys_orders_like_reference_tiebreak():
    k = torch.tensor([3.0, 1.0, 3.0, 0.0, float("inf")], dtype=torch.float32)
    pos = torch.tensor([4, 1, 2, 3, 0])
    keys = pack_keys(k, pos)
    assert int(keys.max()) < SENTINEL
    order = unpack_positions(torch.sort(keys).values).tolist()
    assert order == [3, 1, 2, 4, 0]


def test_global_order_refuses_cpu_without_sort():
    from paper_2506_14851_b200._lib import PdgDeviceError
    with pytest.raises(PdgDeviceError):
        global_order(pack_keys(torch.ones(3), torch.arange(3)), 3)
