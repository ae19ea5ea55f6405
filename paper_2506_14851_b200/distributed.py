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
