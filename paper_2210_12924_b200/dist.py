"""Multi-GPU host logic: candidate / row sharding and the single allreduce-argmin.

One process per GPU (torch.distributed; NCCL on B200, gloo in CPU tests).

* Candidate scoring shards by contiguous candidate ranges. Every rank's fused
  kernel leaves the first-minimum key ``peak << 20 | global_index`` of its
  shard; ONE ``allreduce(MIN)`` on that 8-byte key yields the global
  first-minimum, identical to a serial first-minimum scan (lowest index wins
  ties, oracle.cpp:78-81). Keys that cannot be packed fall back to an
  allgather of (peak, index).
* Pair generation / validation shard by row ranges balanced on per-row work
  (the count pass); concatenating the shards in rank order reproduces the
  reference's lexicographic pair order.
"""
from __future__ import annotations

import numpy as np

KEY_INDEX_BITS = 20
KEY_MAX_PEAK = 1 << 43          # keeps the key a non-negative int64 for NCCL MIN
NO_KEY = (1 << 63) - 1          # "no valid candidate" as int64
OVERFLOW_KEY = (1 << 63) - 2    # kernel marker (MP_KEY_OVERFLOW): key does not fit


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of `total` items for `rank`."""
    return total * rank // world, total * (rank + 1) // world


def pack_key(peak: int, index: int) -> int:
    if index < 0:
        return NO_KEY
    if peak >= KEY_MAX_PEAK or index >= (1 << KEY_INDEX_BITS):
        raise OverflowError("argmin key does not fit; use allgather_argmin")
    return (peak << KEY_INDEX_BITS) | index


def unpack_key(key: int) -> tuple[int, int]:
    """(peak, global index), or (0, -1) when no candidate was valid."""
    if key == NO_KEY:
        return 0, -1
    return key >> KEY_INDEX_BITS, key & ((1 << KEY_INDEX_BITS) - 1)


def check_device_key(key: int) -> int:
    """Validate a key read back from the device (MP_KEY_OVERFLOW -> fallback)."""
    if key == OVERFLOW_KEY:
        raise OverflowError("device argmin key overflowed; use allgather_argmin")
    return key


def allreduce_argmin(key_tensor, group=None):
    """In-place allreduce(MIN) of a 1-element int64 tensor holding a packed key."""
    import torch.distributed as dist
    dist.all_reduce(key_tensor, op=dist.ReduceOp.MIN, group=group)
    return key_tensor


def allgather_argmin(peak: int, index: int, group=None) -> tuple[int, int]:
    """Fallback when keys cannot be packed: gather (peak, index) and pick the first minimum."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    mine = torch.tensor([peak if index >= 0 else -1, index], dtype=torch.int64)
    out = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, mine, group=group)
    best = (0, -1)
    for t in out:
        p, i = int(t[0]), int(t[1])
        if i < 0:
            continue
        if best[1] < 0 or p < best[0] or (p == best[0] and i < best[1]):
            best = (p, i)
    return best


def balanced_row_ranges(row_work, world: int) -> list[tuple[int, int]]:
    """Split rows [0, len) into `world` contiguous ranges of ~equal summed work."""
    w = np.asarray(row_work, dtype=np.float64)
    n = w.size
    if n == 0:
        return [(0, 0)] * world
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def triangular_row_work(num_edges: int):
    """Per-row compare work of the pairwise sweep (row i scans j > i)."""
    return np.arange(num_edges, 0, -1, dtype=np.float64)
