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

    idx: the global pair indices this rank solved (``shard_pairs``); costs/maps/offs: its solve_batch outputs
    (flat mappings, offsets per local pair); n1_all: n1 of every global pair.  Every rank knows every rank's
    pairs (pair r -> rank r mod world) and their mapping lengths, so one fixed-size tensor gather suffices:
    each rank sends [costs as (lo, hi) int32 words | mappings int32] padded to the largest rank's length (on
    the process group's device: NCCL ranks gather on their GPU).  Returns (costs int64[npairs], mappings int32
    flat in global pair order, offsets int64[npairs + 1]).
    """
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n1 = np.asarray(n1_all, np.int64)
    parts = [shard_pairs(npairs, r, world) for r in range(world)]
    if not np.array_equal(np.asarray(idx, np.int64), parts[rank]):
        raise ValueError("gather_results: this rank's pairs are not shard_pairs(npairs, rank, world)")
    lens = [2 * p.shape[0] + int(n1[p].sum()) for p in parts]
    L = max(lens) if lens else 0
    c = np.asarray(costs, np.int64)
    mp = np.asarray(maps, np.int32)[: int(np.asarray(offs)[-1])] if len(offs) else np.zeros(0, np.int32)
    if mp.shape[0] != int(n1[parts[rank]].sum()):
        raise ValueError("gather_results: mapping length does not match the pairs' n1")
    buf = np.zeros(max(L, 1), np.int32)
    buf[: 2 * c.shape[0]] = c.view(np.int32)  # (little endian: lo, hi per cost)
    buf[2 * c.shape[0]: 2 * c.shape[0] + mp.shape[0]] = mp
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.from_numpy(buf).to(dev)
    recv = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, recv, dst=0, group=group)
    if rank != 0:
        return None
    goffs = np.zeros(npairs + 1, np.int64)
    goffs[1:] = np.cumsum(n1)
    out_c = np.empty(npairs, np.int64)
    out_m = np.empty(int(goffs[-1]), np.int32)
    for r, (p, tr) in enumerate(zip(parts, recv)):
        a = tr.cpu().numpy()
        k = p.shape[0]
        out_c[p] = a[: 2 * k].view(np.int64)
        lens_r = n1[p]
        # destination of local entry t of local pair x: goffs[p[x]] + t
        starts = np.repeat(goffs[p] - np.concatenate([[0], np.cumsum(lens_r)[:-1]]), lens_r)
        out_m[starts + np.arange(int(lens_r.sum()))] = a[2 * k: 2 * k + int(lens_r.sum())]
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
