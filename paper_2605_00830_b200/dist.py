"""Multi-GPU plumbing (torch.distributed only; every search step runs in libfastged's kernels).

Two modes:

* Batches of independent pairs: pair k goes to rank k mod world (``shard_pairs``); each rank runs
  ``fastged_solve_batch`` on its own GPU with no data-path collective; ``gather_results`` brings
  the per-rank results back to rank 0 in global pair order (``solve_batch_sharded`` = both).
* One large pair: ``sharded_handle`` creates a handle whose frontier is split into equal slices over
  all ranks (one GPU each, peer access over NVLink); rank 0 creates the 128-byte ncclUniqueId
  (``binding.nccl_unique_id``) and torch.distributed broadcasts it; every rank then calls ``solve_pair``
  collectively.  NCCL only bootstraps (CUDA IPC handles, two stream barriers per call): the per-level
  exchange runs inside the sharded kernel over peer memory.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def shard_pairs(npairs: int, rank: int, world: int) -> np.ndarray:
    """Strided assignment: pair k -> rank k mod world (deterministic, balanced by construction)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return np.arange(rank, npairs, world, dtype=np.int64)


def broadcast_bytes(payload: Optional[bytes], src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string from `src` (uses the process group's default device)."""
    import torch
    import torch.distributed as dist
    obj = [payload]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def nccl_id_for_group(group=None) -> bytes:
    """Rank 0 creates the ncclUniqueId; all ranks receive the same 128 bytes."""
    import torch.distributed as dist
    from . import binding
    payload = binding.nccl_unique_id() if dist.get_rank(group) == 0 else None
    uid = broadcast_bytes(payload, src=0, group=group)
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128
    return bytes(uid)


def sharded_handle(device: int, group=None, flags: int = 0):
    """A handle for the sharded single-pair mode over all ranks of `group`."""
    import torch.distributed as dist
    from . import binding
    uid = nccl_id_for_group(group)
    return binding.Handle(device, world_size=dist.get_world_size(group), rank=dist.get_rank(group),
                          nccl_id=uid, flags=flags)


def gather_results(npairs: int, idx: np.ndarray, costs: np.ndarray, maps: np.ndarray, offs: np.ndarray,
                   n1_all: Sequence[int], group=None) -> Optional[Tuple[np.ndarray, np.ndarray, np.ndarray]]:
    """Collect (cost, mapping) of every pair on rank 0 in global pair order (None on other ranks).

    idx: the global pair indices this rank solved; costs/maps/offs: its solve_batch outputs (flat
    mappings, offsets per local pair).  Returns (costs int64[npairs], mappings int32 flat in global
    pair order, offsets int64[npairs + 1]).  Mappings travel as int16 (g2 indices < 2^15).
    """
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mp = np.asarray(maps)
    wire = mp.astype(np.int16) if (mp.size == 0 or int(mp.max(initial=-1)) < 2 ** 15) else mp.astype(np.int32)
    mine = (np.asarray(idx, np.int64), np.asarray(costs, np.int64), wire, np.asarray(offs, np.int64))
    parts = [None] * world if rank == 0 else None
    dist.gather_object(mine, parts, dst=0, group=group)
    if rank != 0:
        return None
    n1 = np.asarray(n1_all, np.int64)
    goffs = np.zeros(npairs + 1, np.int64)
    goffs[1:] = np.cumsum(n1)
    out_c = np.full(npairs, -1, np.int64)
    out_m = np.full(int(goffs[-1]), -2, np.int32)
    for pidx, pc, pm, po in parts:
        out_c[pidx] = pc
        lens = np.diff(po)
        assert np.array_equal(lens, n1[pidx]), "a rank returned a mapping of the wrong length"
        # destination of local entry t of local pair x: goffs[pidx[x]] + t
        starts = np.repeat(goffs[pidx] - po[:-1], lens)
        out_m[starts + np.arange(int(po[-1]))] = pm[: int(po[-1])]
    assert (out_c >= 0).all(), "a pair was not solved by any rank"
    assert not (out_m == -2).any(), "a mapping entry was not filled"
    return out_c, out_m, goffs


def solve_batch_sharded(solver, packed, pair_a, pair_b, costs, K: int, group=None):
    """§8(e) batch mode: every rank passes the same canonical batch; pair r is solved by rank
    r mod world (``shard_pairs``) with ``solver.solve_batch`` (a ``binding.Handle`` on this rank's GPU),
    and the costs and mappings are gathered to rank 0 in global order.  Returns
    (costs, flat mappings, offsets) on rank 0 and None elsewhere; no data-path collective runs
    before the final gather (pairs are independent)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pair_a, pair_b = np.asarray(pair_a, np.int64), np.asarray(pair_b, np.int64)
    idx = shard_pairs(pair_a.shape[0], rank, world)
    c, m, offs, _ = solver.solve_batch(packed, pair_a[idx], pair_b[idx], costs, K)
    return gather_results(pair_a.shape[0], idx, c, m, offs, np.asarray(packed.n)[pair_a], group=group)
