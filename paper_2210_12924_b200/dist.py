"""Multi-GPU host logic: candidate / row sharding and the single allreduce-argmin.

One process per GPU (torch.distributed; NCCL on B200, gloo in CPU tests).

* Candidate scoring shards by contiguous candidate ranges. Every rank's fused
  kernel leaves {first-minimum key ``peak << 20 | global_index``, overflow
  flag} of its shard; ONE ``allreduce(MIN)`` on those 16 bytes yields the
  global first-minimum, identical to a serial first-minimum scan (lowest index
  wins ties, oracle.cpp:78-81), and tells every rank whether any shard had a
  key that cannot be packed - then all ranks fall back to an allgather of
  (peak, index).
* Pair generation / validation shard by row ranges balanced on per-row work
  (the count pass); concatenating the shards in rank order reproduces the
  reference's lexicographic pair order.
"""
from __future__ import annotations

import numpy as np

KEY_INDEX_BITS = 20
KEY_MAX_PEAK = 1 << 42          # MP_KEY_MAX_PEAK: keys stay below NO_KEY as int64
NO_KEY = 0x7F7F7F7F7F7F7F7F     # MP_KEY_NONE: byte-memset identity of the MIN
OVERFLOW_KEY = 0x7F7F7F7F7F7F7F7E  # MP_KEY_OVERFLOW: mp_argmin_key_d out[2] only


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of `total` items for `rank`."""
    return total * rank // world, total * (rank + 1) // world


def pack_key(peak: int, index: int) -> int:
    if index < 0:
        return NO_KEY
    if peak >= KEY_MAX_PEAK or index >= (1 << KEY_INDEX_BITS):
        raise OverflowError("argmin key does not fit; use allgather_argmin")
    return (peak << KEY_INDEX_BITS) | index


def key_pair(peak: int, index: int) -> list[int]:
    """The 2-word fused key {key, overflow} one shard contributes (host side)."""
    if index >= 0 and (peak >= KEY_MAX_PEAK or index >= (1 << KEY_INDEX_BITS)):
        return [NO_KEY, 0]
    return [pack_key(peak, index), NO_KEY]


def unpack_key(key: int) -> tuple[int, int]:
    """(peak, global index), or (0, -1) when no candidate was valid."""
    if key == NO_KEY:
        return 0, -1
    return key >> KEY_INDEX_BITS, key & ((1 << KEY_INDEX_BITS) - 1)


def key_overflowed(pair) -> bool:
    """True when any candidate behind a (reduced) {key, overflow} pair did not fit."""
    return int(pair[1]) == 0


def check_device_key(pair) -> int:
    """The key of a (reduced) {key, overflow} pair read back from the device;
    OverflowError when some shard overflowed (-> allgather_argmin fallback)."""
    if isinstance(pair, int):
        pair = [pair, NO_KEY]
    if key_overflowed(pair) or int(pair[0]) == OVERFLOW_KEY:
        raise OverflowError("device argmin key overflowed; use allgather_argmin")
    return int(pair[0])


def allreduce_argmin(key_pair_tensor, group=None):
    """In-place allreduce(MIN) of the 2-element int64 {key, overflow} tensor: the
    reduced key is the global first minimum, and overflow == 0 iff ANY rank had a
    candidate whose key did not fit (that rank's key would otherwise be hidden
    by the MIN), in which case every rank takes allgather_argmin."""
    import torch.distributed as dist
    dist.all_reduce(key_pair_tensor, op=dist.ReduceOp.MIN, group=group)
    return key_pair_tensor


def global_argmin(key_pair_tensor, peak: int, index: int, group=None) -> tuple[int, int]:
    """One allreduce on the fused pair; the allgather fallback only if it reports
    an overflow anywhere. (peak, index) is this rank's own first minimum (global
    index, -1 if none), needed only by the fallback."""
    allreduce_argmin(key_pair_tensor, group)
    pair = [int(x) for x in key_pair_tensor.tolist()]
    if key_overflowed(pair):
        return allgather_argmin(peak, index, group)
    return unpack_key(pair[0])


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


def _world_rank(group=None) -> tuple[int, int]:
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def exchange_counts(local: int, device=None, group=None) -> tuple[int, int, list[int]]:
    """The one exchange of the row-sharded pair sweep: allgather
    of the per-rank pair counts. Returns (this rank's global offset, total,
    per-rank counts); rank r's pairs occupy [offset, offset + counts[r]) of the
    reference's lexicographic list."""
    import torch
    import torch.distributed as dist
    world, rank = _world_rank(group)
    if world == 1:
        return 0, int(local), [int(local)]
    mine = torch.tensor([int(local)], dtype=torch.int64, device=device)
    out = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(out, mine, group=group)
    counts = [int(t.item()) for t in out]
    return sum(counts[:rank]), sum(counts), counts


def sharded_overlap_pairs(shard_fn, num_edges: int, device=None, group=None):
    """encode_addresses' pair loop (encode.cpp:347-367) sharded by rows over the
    ranks: rank r sweeps rows ``balanced_row_ranges(triangular_row_work(E))[r]``
    with ``shard_fn(row_begin, row_end) -> int32 [k, 2]`` (the K2 kernel on its
    GPU), then ONE allgather of the counts gives every rank its global offset.
    Pairs stay rank-local; concatenated in rank order they are the reference's
    list. Returns (local pairs, offset, total)."""
    world, rank = _world_rank(group)
    r0, r1 = balanced_row_ranges(triangular_row_work(num_edges), world)[rank]
    pairs = shard_fn(r0, r1)
    off, total, _ = exchange_counts(len(pairs), device, group)
    return pairs, off, total


def sharded_conflicts(shard_fn, num_edges: int, device=None, group=None, gather: bool = True):
    """validate_plan's pairwise check (plan.cpp:390-404) sharded by rows: ONE
    allreduce(sum) of the violation count; only when it is non-zero are the
    violating pairs gathered (padded allgather), in rank order = (i, j) order.
    ``shard_fn(row_begin, row_end) -> int32 [k, 2]``. Returns (total count,
    all violating pairs as an int32 numpy [total, 2], or None with gather=False)."""
    import torch
    import torch.distributed as dist
    world, rank = _world_rank(group)
    r0, r1 = balanced_row_ranges(triangular_row_work(num_edges), world)[rank]
    viol = shard_fn(r0, r1)
    k = len(viol)
    if world == 1:
        total = k
        allv = np.asarray(viol.cpu() if hasattr(viol, "cpu") else viol, np.int32).reshape(-1, 2)
        return total, (allv if gather else None)
    t = torch.tensor([k], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    total = int(t.item())
    if not gather or total == 0:
        return total, (np.zeros((0, 2), np.int32) if gather else None)
    _, _, counts = exchange_counts(k, device, group)
    width = max(counts)
    buf = torch.full((width, 2), -1, dtype=torch.int32, device=device)
    if k:
        v = viol if isinstance(viol, torch.Tensor) else torch.from_numpy(np.asarray(viol))
        buf[:k] = v.to(device=buf.device, dtype=torch.int32)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    parts = [o[:c].cpu().numpy() for o, c in zip(out, counts)]
    return total, np.concatenate(parts).astype(np.int32).reshape(-1, 2)
