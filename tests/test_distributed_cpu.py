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


# ---- config 4 over N ranks: event routing + gathered key updates ----------
class _FakeQueue:
    def __init__(self, keys):
        self.keys = keys


class _FakeLocal:
    """Stands in for this rank's RefinementStream: an event's new key is a
    deterministic function of its seed (the engine is covered by -m gpu)."""

    def __init__(self, lo, hi, keys_f32):
        self.lo = lo
        self.q = _FakeQueue(pack_keys(torch.from_numpy(keys_f32[lo:hi]), torch.arange(lo, hi)))
        self.seen = []

    def process(self, rows, next_unit, seed, obs_unit, obs_val, attained, resort=True):
        assert not resort
        self.seen.append((rows.clone(), next_unit.clone(), obs_val.clone()))
        self.q.keys[rows.long()] = pack_keys(_event_key(seed), rows.long() + self.lo)


def _event_key(seed):
    return ((seed % 997).to(torch.float64) / 8.0).to(torch.float32)


def _event_batches(n_total, world, batches, per_rank, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(batches):
        apps = rng.permutation(n_total)[: world * per_rank]
        out.append([apps[r * per_rank:(r + 1) * per_rank] for r in range(world)])
    return out


def _full_sort(keys, sorted_keys, sorted_pos, pos):
    s = torch.sort(keys).values
    return s, unpack_positions(s).to(torch.int32)


def _stream_worker(rank, world, port, n_total, out):
    from paper_2506_14851_b200.distributed import ShardedRefinementStream, route_events
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = _keys_for(n_total, 5)
        lo, hi = shard_range(n_total, world, rank)
        local = _FakeLocal(lo, hi, keys)
        st = ShardedRefinementStream(local, n_total, order_fn=_full_sort)
        orders = []
        for b, per in enumerate(_event_batches(n_total, world, 4, 37, 9)):
            apps = torch.from_numpy(per[rank]).to(torch.int64)
            m = apps.numel()
            seed = apps * 31 + b
            nu = (apps % 5).to(torch.int32)
            ov = torch.stack([apps.double(), apps.double() * 2, apps.double() * 3], 1)
            orders.append(st.process(apps, nu, seed, None, ov, None).numpy().copy())
        # routed events landed on their owner with their own fields
        for rows, nu, ov in local.seen:
            g = rows.long() + lo
            assert bool(((g >= lo) & (g < hi)).all())
            assert torch.equal(nu, (g % 5).to(torch.int32))
            assert torch.equal(ov[:, 0], g.double())
        # config 5: the need aggregate summed over ranks
        from paper_2506_14851_b200.distributed import reduce_need_aggregate
        agg = torch.full((16, 32), float(rank + 1), dtype=torch.float64)
        reduce_need_aggregate(agg)
        assert bool((agg == 3.0).all())
        # route_events alone: every event reaches exactly its owner
        apps = torch.arange(rank, n_total, world, dtype=torch.int64)
        rows, (tag,) = route_events(apps, [apps * 10], n_total)
        got = rows + lo
        out[rank] = (orders, got.numpy(), tag.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [301, 1000])
def test_two_rank_event_stream(n_total):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_stream_worker, args=(r, 2, port, n_total, out))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    # single-process reference: apply the same events in order, full sort
    keys = torch.from_numpy(_keys_for(n_total, 5))
    packed = pack_keys(keys, torch.arange(n_total))
    want = []
    for b, per in enumerate(_event_batches(n_total, 2, 4, 37, 9)):
        apps = torch.from_numpy(np.concatenate(per)).to(torch.int64)
        packed[apps] = pack_keys(_event_key(apps * 31 + b), apps)
        want.append(unpack_positions(torch.sort(packed).values).numpy())
    for r in range(2):
        orders, got, tag = out[r]
        for o, w in zip(orders, want):
            np.testing.assert_array_equal(o, w)
        lo, hi = shard_range(n_total, 2, r)
        np.testing.assert_array_equal(np.sort(got), np.arange(lo, hi))
        np.testing.assert_array_equal(tag, got * 10)


def test_owner_of_inverts_shard_range():
    from paper_2506_14851_b200.distributed import owner_of
    for n in (1, 2, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            own = owner_of(torch.arange(n), n, w)
            for r in range(w):
                lo, hi = shard_range(n, w, r)
                assert bool((own[lo:hi] == r).all())
