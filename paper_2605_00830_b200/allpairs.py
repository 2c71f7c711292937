"""All-pairs GED with checkpoint / resume (SURVEY §5 auxiliary subsystems; BASELINE configs[4]: the
1,999,000 unordered pairs of 2,000 graphs).

The pairs (a < b, graph a = source g1, graph b = target g2) are solved in chunks through
``fastged_solve_batch``; every finished chunk is written atomically (temporary file + rename) to
``out_dir/chunk_NNNNN.npz`` together with a manifest that fixes what the run computes (K, costs, chunk
size, number of graphs and a digest of their arrays).  A rerun with the same manifest skips the chunks
already on disk, so a job killed at any point loses at most one chunk.  A rerun with a different
manifest refuses to mix results.  Only host I/O lives here; every GED is computed by the GPU path.
"""
from __future__ import annotations

import hashlib
import json
import os
from typing import Sequence

import numpy as np


def _digest(graphs) -> str:
    h = hashlib.sha256()
    for g in graphs:
        h.update(np.int64(g.n).tobytes())
        h.update(np.ascontiguousarray(g.vlabels, np.int32).tobytes())
        h.update(np.ascontiguousarray(g.edges, np.int32).tobytes())
        if g.elabels is not None:
            h.update(np.ascontiguousarray(g.elabels, np.int32).tobytes())
    return h.hexdigest()[:32]


def all_pairs(solver, graphs: Sequence, costs, K: int, out_dir: str, chunk: int = 100_000,
              keep_mappings: bool = False, max_chunks: int = None):
    """Solve every unordered pair (a < b) of ``graphs`` with checkpointing.

    solver: an object with ``solve_batch(packed, pair_a, pair_b, costs, K)`` (``binding.Handle``).
    Returns (pair_a, pair_b, costs int64, children int64[, mappings int16 flat, offsets]) over all pairs
    in (a, b) lexicographic order; with ``max_chunks`` only that many new chunks are computed (the
    function then returns None), which is how a job is split or how a crash is simulated in the tests.
    """
    from .binding import PackedGraphs
    os.makedirs(out_dir, exist_ok=True)
    ng = len(graphs)
    ia, ib = np.triu_indices(ng, 1)
    ia, ib = ia.astype(np.int64), ib.astype(np.int64)
    npairs = ia.shape[0]
    manifest = {"npairs": int(npairs), "ngraphs": ng, "K": int(K), "costs": [int(x) for x in costs],
                "chunk": int(chunk), "graphs_sha256_32": _digest(graphs), "keep_mappings": bool(keep_mappings)}
    mpath = os.path.join(out_dir, "manifest.json")
    if os.path.exists(mpath):
        old = json.load(open(mpath))
        if old != manifest:
            raise ValueError(f"{out_dir} holds results of a different run: {old} != {manifest}")
    else:
        tmp = mpath + ".tmp"
        json.dump(manifest, open(tmp, "w"))
        os.replace(tmp, mpath)
    nchunks = (npairs + chunk - 1) // chunk
    packed = None
    done_now = 0
    for c in range(nchunks):
        path = os.path.join(out_dir, f"chunk_{c:05d}.npz")
        if os.path.exists(path):
            continue
        if max_chunks is not None and done_now >= max_chunks:
            return None
        if packed is None:
            packed = PackedGraphs(graphs)
        s0, s1 = c * chunk, min(npairs, (c + 1) * chunk)
        cost, maps, offs, ch = solver.solve_batch(packed, ia[s0:s1], ib[s0:s1], costs, K)
        arrays = {"cost": np.asarray(cost, np.int64), "children": np.asarray(ch, np.int64)}
        if keep_mappings:
            arrays["map"] = np.asarray(maps, np.int16)
            arrays["offs"] = np.asarray(offs, np.int64)
        tmp = path + ".tmp.npz"
        np.savez(tmp, **arrays)
        os.replace(tmp, path)  # atomic: a chunk file exists only when complete
        done_now += 1
    cost = np.empty(npairs, np.int64)
    children = np.empty(npairs, np.int64)
    maps, moffs = [], [0]
    for c in range(nchunks):
        z = np.load(os.path.join(out_dir, f"chunk_{c:05d}.npz"))
        s0, s1 = c * chunk, min(npairs, (c + 1) * chunk)
        cost[s0:s1] = z["cost"]
        children[s0:s1] = z["children"]
        if keep_mappings:
            maps.append(z["map"])
            moffs.extend((moffs[-1] + z["offs"][1:]).tolist())
    if keep_mappings:
        return ia, ib, cost, children, np.concatenate(maps) if maps else np.zeros(0, np.int16), np.array(moffs, np.int64)
    return ia, ib, cost, children
