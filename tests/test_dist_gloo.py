"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host logic: pair sharding, result
gathering in global order, and the ncclUniqueId broadcast for the sharded single-pair mode.
The per-rank search itself needs a GPU; here each rank's "solve" is the CPU oracle, which is
exactly what the GPU parity tests compare the kernels against."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2605_00830_b200 import dist as fdist
        from paper_2605_00830_b200 import synth
        from paper_2605_00830_b200 import binding
        w = synth.config_workload(3, npairs=11, K=40)
        packed = binding.PackedGraphs(w.graphs)
        seen = []

        class OracleSolver:  # stands in for binding.Handle (the per-rank GPU search) on a CPU box
            def solve_batch(self, pk, a, b, costs, K):
                seen.extend(int(x) // 2 for x in a)
                pairs = [(w.graphs[int(x)], w.graphs[int(y)]) for x, y in zip(a, b)]
                c, maps, ch = oracle.kbest_batch(pairs, costs, K, nthreads=1)
                offs = np.concatenate([[0], np.cumsum([m.shape[0] for m in maps])]).astype(np.int64)
                flat = np.concatenate(maps + [np.zeros(0, np.int32)]).astype(np.int32)
                return c, flat, offs, ch

        res = fdist.solve_batch_sharded(OracleSolver(), packed, w.pair_a, w.pair_b, w.costs, w.K)
        assert seen == list(range(rank, w.npairs, world))  # pair r -> rank r mod world
        uid = fdist.nccl_id_for_group()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        q.put((rank, None if res is None else
               (res[0].tolist(), [res[1][res[2][k]:res[2][k + 1]].tolist() for k in range(w.npairs)]),
               len(uid), all(x == ids[0] for x in ids)))
    finally:
        dist.destroy_process_group()


def test_shard_pairs_partition():
    from paper_2605_00830_b200 import dist as fdist
    for n in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            parts = [fdist.shard_pairs(n, r, world) for r in range(world)]
            allk = np.sort(np.concatenate(parts))
            assert np.array_equal(allk, np.arange(n))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


@pytest.mark.timeout(300)
def test_two_rank_gather_and_nccl_id():
    from oracle import oracle
    from paper_2605_00830_b200 import binding, build, synth
    oracle.build()
    build.build()
    binding.lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = dict((g[0], g[1:]) for g in got)
    res, idlen, same = got[0]
    assert idlen == 128 and same and got[1][1] == 128 and got[1][2]
    w = synth.config_workload(3, npairs=11, K=40)
    ref_c, ref_m, _ = oracle.kbest_batch([w.pair(k) for k in range(w.npairs)], w.costs, w.K, nthreads=2)
    assert res[0] == ref_c.tolist()
    assert res[1] == [m.tolist() for m in ref_m]
    assert got[1][0] is None


def _gather_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_00830_b200 import dist as fdist
        npairs = 13
        n1 = [(k * 7) % 5 for k in range(npairs)]  # unequal mapping lengths, some empty
        idx = fdist.shard_pairs(npairs, rank, world)
        costs = np.array([(1 << 40) + 3 * int(k) for k in idx], np.int64)  # costs beyond 2^31
        maps = [np.arange(n1[int(k)], dtype=np.int32) + 100 * int(k) for k in idx]
        offs = np.concatenate([[0], np.cumsum([m.shape[0] for m in maps])]).astype(np.int64)
        flat = np.concatenate(maps + [np.zeros(0, np.int32)]).astype(np.int32)
        res = fdist.gather_results(npairs, idx, costs, flat, offs, n1)
        q.put((rank, None if res is None else (res[0].tolist(), res[1].tolist(), res[2].tolist())))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_three_rank_gather_unequal_lengths():
    """gather_results with 3 ranks: unequal per-rank lengths (padding), empty mappings, int64 costs > 2^31."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[1] is None and got[2] is None
    c, m, o = got[0]
    n1 = [(k * 7) % 5 for k in range(13)]
    assert c == [(1 << 40) + 3 * k for k in range(13)]
    assert o == [0] + list(np.cumsum(n1))
    assert m == [100 * k + t for k in range(13) for t in range(n1[k])]
