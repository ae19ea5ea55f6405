"""K5: multi-GPU global ranking (one process per GPU, torch.distributed).

Applications are independent (sched.py:111-129, estimator.py:305-362), so a
queue shards by contiguous ranges of the global arrival order: each rank runs
the demand engine and the scorer on its own shard with no data-path
collective.  The only exchange is the global order: every rank packs its
keys as 8 bytes (float32 key bits << 32 | global arrival position, so the
reference tie-break (key, arrival_time, app_instance_id), sched.py:191-192,
is one integer compare), one all-gather over NCCL/NVLink collects them, and a
radix sort (pdg_order) orders them.  Shards of unequal size are padded with
a sentinel that sorts last.

Because the gathered array is rank-major and every shard is in arrival order,
it is already in global arrival order: a stable sort on the 32-bit key alone
(pdg_order begin_bit=32, half the radix passes) yields the exact order.
"""

from __future__ import annotations

from typing import Callable, Optional

import torch

from . import _lib

SENTINEL = 0x7FFFFFFFFFFFFFFF       # > every packed key, signed or unsigned


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of the global arrival order, balanced by count."""
    base, extra = divmod(int(n_total), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_keys(key_f32: torch.Tensor, global_pos: torch.Tensor) -> torch.Tensor:
    """int64 sort keys (float32 bits << 32 | position); keys must be >= +0."""
    bits = key_f32.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    return (bits << 32) | (global_pos.to(torch.int64) & 0xFFFFFFFF)


def unpack_positions(keys: torch.Tensor) -> torch.Tensor:
    return (keys & 0xFFFFFFFF).to(torch.int64)


def _cuda_sort(keys: torch.Tensor) -> torch.Tensor:
    """Stable radix sort on the key bits (pdg_order, begin_bit = 32)."""
    L = _lib.lib()
    n = keys.numel()
    out = torch.empty_like(keys)
    slots = torch.arange(n, dtype=torch.int32, device=keys.device)
    oslots = torch.empty_like(slots)
    tb = int(L.pdg_order_temp_bytes(n))
    temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=keys.device)
    _lib.check(L.pdg_order(_lib.ptr(keys), _lib.ptr(out), _lib.ptr(slots), _lib.ptr(oslots),
                           n, 32, _lib.ptr(temp), temp.numel(), _lib.stream_ptr()),
               "pdg_order")
    return out


def global_order(local_keys: torch.Tensor, n_total: int, group=None,
                 sort_fn: Optional[Callable[[torch.Tensor], torch.Tensor]] = None
                 ) -> torch.Tensor:
    """All-gather the packed keys of every shard and return the n_total keys
    in global (key, arrival) order on every rank.

    local_keys: this rank's packed keys (shard_range order).  sort_fn: the
    sort to apply to the gathered array; the default is the CUDA radix sort
    (tests inject a reference sort to exercise the exchange on gloo/CPU).
    """
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(n_total, world, rank)
    if local_keys.numel() != hi - lo:
        raise ValueError(f"rank {rank}: {local_keys.numel()} keys for shard [{lo}, {hi})")
    width = -(-n_total // world)
    buf = torch.full((width,), SENTINEL, dtype=torch.int64, device=local_keys.device)
    buf[: local_keys.numel()] = local_keys
    if world > 1:
        gathered = torch.empty(world * width, dtype=torch.int64, device=local_keys.device)
        dist.all_gather_into_tensor(gathered, buf, group=group)
    else:
        gathered = buf
    if sort_fn is None:
        if not gathered.is_cuda:
            raise _lib.PdgDeviceError("global_order needs CUDA tensors (no CPU fallback)")
        sort_fn = _cuda_sort
    return sort_fn(gathered)[:n_total]


# ---------------------------------------------------------------------------
# Config 4 over N GPUs: refinement events are routed to the
# rank that owns the application, applied there (K3 + K2 + K1 on the owned
# rows), and the re-scored (global position, key) pairs are all-gathered so
# every rank's copy of the global order is updated per micro-batch.
# ---------------------------------------------------------------------------
def _world(group):
    import torch.distributed as dist
    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def owner_of(app_global: torch.Tensor, n_total: int, world: int) -> torch.Tensor:
    """Rank owning each global arrival position (inverse of shard_range)."""
    base, extra = divmod(int(n_total), int(world))
    a = app_global.to(torch.int64)
    big = extra * (base + 1)                 # the first `extra` ranks hold base + 1
    if base == 0:
        return a
    return torch.where(a < big, a // (base + 1), extra + (a - big) // base)


def route_events(app_global: torch.Tensor, fields: list, n_total: int, group=None):
    """Send every event to the rank owning its application (one all_to_all
    per field).  app_global: int64[m] global arrival positions of this rank's
    events; fields: tensors with a leading dimension m (None entries pass
    through as None).  Returns (local rows int64, routed fields), received
    events in (source rank, source order) order -- the same app never
    appears twice in a micro-batch, so per-app order is preserved."""
    import torch.distributed as dist
    world, rank = _world(group)
    lo, _ = shard_range(n_total, world, rank)
    if world == 1:
        return app_global.to(torch.int64) - lo, list(fields)
    owner = owner_of(app_global, n_total, world)
    perm = torch.sort(owner, stable=True).indices
    send = torch.bincount(owner, minlength=world).to(torch.int64)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    sc, rc = send.tolist(), recv.tolist()
    m_in = int(sum(rc))

    def a2a(t):
        t = t.index_select(0, perm.to(t.device)).contiguous()
        out = torch.empty((m_in,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_to_all_single(out, t, rc, sc, group=group)
        return out

    apps = a2a(app_global.to(torch.int64))
    return apps - lo, [None if f is None else a2a(f) for f in fields]


def gather_updates(packed_keys: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's re-scored packed keys (variable counts; the
    position is in the low 32 bits)."""
    import torch.distributed as dist
    world, _ = _world(group)
    if world == 1:
        return packed_keys
    cnt = torch.tensor([packed_keys.numel()], dtype=torch.int64, device=packed_keys.device)
    cnts = torch.empty(world, dtype=torch.int64, device=packed_keys.device)
    dist.all_gather_into_tensor(cnts, cnt, group=group)
    width = int(cnts.max().item())
    buf = torch.full((width,), SENTINEL, dtype=torch.int64, device=packed_keys.device)
    buf[: packed_keys.numel()] = packed_keys
    allb = torch.empty(world * width, dtype=torch.int64, device=packed_keys.device)
    dist.all_gather_into_tensor(allb, buf, group=group)
    keep = torch.cat([torch.arange(r * width, r * width + int(c), device=allb.device)
                      for r, c in enumerate(cnts.tolist())])
    return allb.index_select(0, keep)


class ShardedRefinementStream:
    """RefinementStream over a queue sharded by arrival range.

    local: this rank's RefinementStream (its queue's packed keys must carry
    the global arrival position as tiebreak).  Every rank keeps the global
    packed keys and their order; process() routes a micro-batch, applies the
    owned events, gathers the re-scored keys and merges them into the order
    (pdg_order_update).  order_fn(keys, sorted_keys, sorted_pos, pos) may
    replace the merge (tests on gloo/CPU); the default is the CUDA one."""

    def __init__(self, local, n_total: int, group=None, order_fn=None):
        self.local = local
        self.n_total = int(n_total)
        self.group = group
        world, rank = _world(group)
        self.lo, self.hi = shard_range(self.n_total, world, rank)
        self.order_fn = order_fn
        dev = local.q.keys.device
        sorted_keys = global_order(local.q.keys[: self.hi - self.lo].contiguous(), self.n_total,
                                   group, sort_fn=None if order_fn is None else
                                   (lambda k: torch.sort(k).values))
        self.sorted_keys = sorted_keys
        self.sorted_pos = unpack_positions(sorted_keys).to(torch.int32)
        self.keys = torch.empty(self.n_total, dtype=torch.int64, device=dev)
        self.keys.index_copy_(0, self.sorted_pos.long(), sorted_keys)
        self._mark = torch.zeros(self.n_total, dtype=torch.uint8, device=dev)
        self._k2 = torch.empty_like(self.sorted_keys)
        self._p2 = torch.empty_like(self.sorted_pos)
        self._temp = None

    def process(self, app_global, next_unit, seed, obs_unit=None, obs_val=None, attained=None):
        """One micro-batch of events (any rank may hold any events; an app
        appears at most once per batch across all ranks).  Returns the global
        order (positions) after the batch."""
        rows, (nu, sd, ou, ov, at) = route_events(
            app_global, [next_unit, seed, obs_unit, obs_val, attained], self.n_total, self.group)
        if rows.numel():
            self.local.process(rows.to(torch.int32), nu, sd, ou, ov, at, resort=False)
        upd = gather_updates(self.local.q.keys.index_select(0, rows.to(self.local.q.keys.device)),
                             self.group)
        pos = unpack_positions(upd)
        self.keys.index_copy_(0, pos, upd)
        if self.order_fn is not None:
            self.sorted_keys, self.sorted_pos = self.order_fn(self.keys, self.sorted_keys,
                                                              self.sorted_pos, pos)
        elif pos.numel():
            self._merge(pos.to(torch.int32))
        return self.sorted_pos

    def _merge(self, pos: torch.Tensor) -> None:
        L = _lib.lib()
        m = int(pos.numel())
        need = int(L.pdg_order_update_temp_bytes(self.n_total, m))
        if self._temp is None or self._temp.numel() < need:
            self._temp = torch.empty(max(need, 16), dtype=torch.uint8, device=self.keys.device)
        _lib.check(L.pdg_order_update(
            _lib.ptr(self.keys), _lib.ptr(self.sorted_keys), _lib.ptr(self.sorted_pos),
            self.n_total, _lib.ptr(pos), m, _lib.ptr(self._mark), _lib.ptr(self._k2),
            _lib.ptr(self._p2), _lib.ptr(self._temp), self._temp.numel(), _lib.stream_ptr()),
            "pdg_order_update")
        self.sorted_keys, self._k2 = self._k2, self.sorted_keys
        self.sorted_pos, self._p2 = self._p2, self.sorted_pos


def reduce_need_aggregate(agg: torch.Tensor, group=None) -> torch.Tensor:
    """Config 5 on N GPUs: the [types, windows] need aggregate of every shard
    (PrewarmTables.need(..., agg=...)) summed over ranks in place (one
    all-reduce of T*K float64)."""
    import torch.distributed as dist
    world, _ = _world(group)
    if world > 1:
        dist.all_reduce(agg, op=dist.ReduceOp.SUM, group=group)
    return agg
