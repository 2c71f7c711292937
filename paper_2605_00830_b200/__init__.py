"""FAST-GED K-Best hot path on B200 (arXiv 2605.00830).

The search runs in hand-written sm_100a CUDA kernels inside ``libfastged.so``
behind the C ABI declared in ``include/fastged.h``; ``binding`` is the thin
ctypes layer (argument marshalling only).  ``synth`` holds the seeded input
generators.  Importing the package does not load the library; the first call
into ``binding`` does, and fails loudly if it is missing.

Convenience entry points (each a thin wrapper over the C ABI on one GPU):

    from paper_2605_00830_b200 import Graph, COSTS, ged, ged_batch
    r = ged(g1, g2, COSTS["setting1"], K=1000)            # dict(cost, mapping, children, ...)
    costs, mappings = ged_batch(pairs, COSTS["setting1"], K=1000)
"""
from .synth import COSTS, Graph  # noqa: F401  (plain data types, no arithmetic)

__all__ = ["binding", "synth", "dist", "knn", "allpairs", "Graph", "COSTS", "ged", "ged_batch"]

_handles = {}


def _handle(device: int, flags: int):
    from . import binding
    key = (device, flags)
    if key not in _handles:
        _handles[key] = binding.Handle(device, flags=flags)
    return _handles[key]


def ged(g1, g2, costs, K: int = 1000, device: int = 0, flags: int = 0) -> dict:
    """GED upper bound of the K-Best search (g1 = source, g2 = target) and its vertex mapping
    (mapping[i] = g2 vertex or -1 = deleted)."""
    return _handle(device, flags).solve_pair(g1, g2, costs, K)


def ged_batch(pairs, costs, K: int = 1000, device: int = 0, flags: int = 0):
    """Many pairs in one batched call: returns (costs int64[P], list of mappings)."""
    import numpy as np
    from . import binding
    graphs = [g for ab in pairs for g in ab]
    a = np.arange(0, 2 * len(pairs), 2)
    c, m, offs, _ = _handle(device, flags).solve_batch(binding.PackedGraphs(graphs), a, a + 1, costs, K)
    return c, [m[offs[k]:offs[k + 1]] for k in range(len(pairs))]
