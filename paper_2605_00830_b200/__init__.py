"""FAST-GED K-Best hot path on B200 (arXiv 2605.00830).

The search runs in hand-written sm_100a CUDA kernels inside ``libfastged.so``
behind the C ABI declared in ``include/fastged.h``; ``binding`` is the thin
ctypes layer (argument marshalling only).  ``synth`` holds the seeded input
generators.  Importing the package does not load the library; the first call
into ``binding`` does, and fails loudly if it is missing.
"""
__all__ = ["binding", "synth"]
