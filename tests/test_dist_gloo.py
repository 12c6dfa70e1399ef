"""CPU, world size 2 over gloo: the multi-GPU host logic (candidate sharding +
one allreduce-argmin, row sharding of the pair sweep) reproduces the serial
reference semantics. The per-shard device work is replaced here by the C
restatement of the same functions (this runs without a GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp_

from paper_2210_12924_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, peaks, valid, lo, hi, size, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import oracle as O
    # --- candidate sharding + single allreduce(min) on the packed key
    b, e = D.shard_range(len(peaks), world, rank)
    best = -1
    for c in range(b, e):
        if valid[c] and (best < 0 or peaks[c] < peaks[best]):
            best = c
    key = torch.tensor(D.key_pair(int(peaks[best]), best) if best >= 0 else [D.NO_KEY, D.NO_KEY],
                       dtype=torch.int64)
    D.allreduce_argmin(key)
    fallback = D.allgather_argmin(int(peaks[best]) if best >= 0 else 0, best)
    # --- row-sharded pair generation, concatenated in rank order
    ranges = D.balanced_row_ranges(D.triangular_row_work(len(lo)), world)
    r0, r1 = ranges[rank]
    pairs = O.overlap_pairs(lo, hi, size)
    mine = pairs[(pairs[:, 0] >= r0) & (pairs[:, 0] < r1)] if len(pairs) else pairs
    gathered = [None] * world
    dist.all_gather_object(gathered, mine.tolist())
    if rank == 0:
        out_q.put((D.check_device_key(key.tolist()), fallback, gathered, ranges))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_argmin_and_row_shards(world):
    rng = np.random.default_rng(0)
    C = 1000
    peaks = rng.integers(1000, 1100, C).astype(np.int64)
    valid = (rng.random(C) > 0.1).astype(np.uint8)
    peaks[[17, 640]] = 999          # tie across the two shards: lowest index must win
    valid[[17, 640]] = 1
    E = 300
    lo = rng.integers(1, 200, E).astype(np.int32)
    hi = (lo + rng.integers(-3, 40, E)).astype(np.int32)
    size = rng.integers(0, 3, E).astype(np.uint64)
    ctx = mp_.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, peaks, valid, lo, hi, size, q))
             for r in range(world)]
    for p in procs:
        p.start()
    key, fallback, gathered, ranges = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert D.unpack_key(key) == (999, 17)
    assert fallback == (999, 17)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import oracle as O
    full = O.overlap_pairs(lo, hi, size).tolist()
    assert sum(gathered, []) == full
    assert ranges[0][0] == 0 and ranges[-1][1] == E and ranges[0][1] == ranges[1][0]


def test_key_packing_edges():
    assert D.unpack_key(D.pack_key(5, 3)) == (5, 3)
    assert D.unpack_key(D.NO_KEY) == (0, -1)
    assert D.pack_key(0, -1) == D.NO_KEY
    with pytest.raises(OverflowError):
        D.pack_key(1 << 42, 0)
    with pytest.raises(OverflowError):
        D.check_device_key(D.OVERFLOW_KEY)
    with pytest.raises(OverflowError):
        D.check_device_key([D.pack_key(5, 3), 0])     # some shard overflowed
    assert D.check_device_key([D.NO_KEY, D.NO_KEY]) == D.NO_KEY
    assert D.key_pair(1 << 42, 7) == [D.NO_KEY, 0]
    # every packable key sorts below the memset identity, as int64
    assert D.pack_key(D.KEY_MAX_PEAK - 1, (1 << 20) - 1) < D.NO_KEY < (1 << 63)
    assert int.from_bytes(b"\x7f" * 8, "little") == D.NO_KEY
    assert [D.shard_range(10, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]
    assert D.balanced_row_ranges([], 2) == [(0, 0), (0, 0)]


def _worker_sharded(rank, world, port, lo, hi, size, has, addr, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import oracle as O
    full = O.overlap_pairs(lo, hi, size)
    viol_full = O.validate_pairs(lo, hi, size, has, addr)

    def rows(p, r0, r1):   # the per-GPU kernel's output for rows [r0, r1), from the C restatement
        return p[(p[:, 0] >= r0) & (p[:, 0] < r1)] if len(p) else p.reshape(0, 2)

    pairs, off, total = D.sharded_overlap_pairs(lambda a, b: rows(full, a, b), len(lo))
    nv, viol = D.sharded_conflicts(lambda a, b: rows(viol_full, a, b), len(lo))
    nv0, none = D.sharded_conflicts(lambda a, b: rows(viol_full[:0], a, b), len(lo))
    out_q.put((rank, pairs.tolist(), off, total, nv, viol.tolist(), nv0, none.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_pairs_and_conflicts():
    """Row-sharded pair sweep (one allgather of counts) and validation (one
    allreduce(sum), violators gathered only when non-zero) reproduce the
    serial lists in the reference's (i, j) order."""
    rng = np.random.default_rng(3)
    E = 400
    lo = rng.integers(1, 300, E).astype(np.int32)
    hi = (lo + rng.integers(-3, 60, E)).astype(np.int32)
    size = rng.integers(0, 4, E).astype(np.uint64)
    has = (rng.random(E) > 0.2).astype(np.uint8)
    addr = rng.integers(0, 64, E).astype(np.uint64)
    ctx = mp_.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sharded,
                         args=(r, 2, port, lo, hi, size, has, addr, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import oracle as O
    full = O.overlap_pairs(lo, hi, size).tolist()
    viol = O.validate_pairs(lo, hi, size, has, addr).tolist()
    assert len(full) > 1000 and len(viol) > 10
    (_, p0, off0, tot0, nv, v0, nv0, z0), (_, p1, off1, tot1, _, v1, _, _) = res
    assert off0 == 0 and off1 == len(p0) and tot0 == tot1 == len(full)
    assert p0 + p1 == full
    assert nv == len(viol) and v0 == v1 == viol
    assert nv0 == 0 and z0 == []


def _worker_overflow(rank, world, port, out_q):
    """Rank 1's only candidate has a peak too large to pack; rank 0's smaller
    peak still wins, but only after every rank learned of the overflow."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = (1000, 3) if rank == 0 else (D.KEY_MAX_PEAK + 5, 10)
    key = torch.tensor(D.key_pair(*mine), dtype=torch.int64)
    peak, idx = D.global_argmin(key, *mine)
    if rank == 0:
        out_q.put((peak, idx, key.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def _worker_overflow_wins(rank, world, port, out_q):
    """The overflowing rank holds the index-order first minimum among equal huge
    peaks: only the fallback can find it."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    big = D.KEY_MAX_PEAK + 1
    mine = (big, 1 << 21) if rank == 0 else (big, 5)   # rank 0's index does not fit either
    key = torch.tensor(D.key_pair(*mine), dtype=torch.int64)
    peak, idx = D.global_argmin(key, *mine)
    if rank == 0:
        out_q.put((peak, idx, key.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("worker,expect", [("_worker_overflow", (1000, 3)),
                                           ("_worker_overflow_wins", (D.KEY_MAX_PEAK + 1, 5))])
def test_overflow_on_one_rank_reaches_every_rank(worker, expect):
    """an overflowing rank must not be silently discarded by the MIN -
    the 2-word {key, overflow} reduction makes every rank take the allgather."""
    ctx = mp_.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=globals()[worker], args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    peak, idx, reduced = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert reduced[1] == 0                  # the overflow flag survived the MIN
    assert (peak, idx) == expect
