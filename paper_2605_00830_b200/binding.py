"""Thin ctypes binding of libfastged.so (include/fastged.h).

Argument marshalling only: every step of the K-Best search runs in the library's
CUDA kernels.  There is no fallback — if the library or a CUDA device is missing,
calls raise ``FastGedError``.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfastged.so")

OK, ERR_ARG, ERR_INPUT, ERR_CAPACITY, ERR_OVERFLOW, ERR_CUDA, ERR_NCCL = range(7)
FLAG_TIMING = 1
FLAG_DEBUG_WINDOW = 2
FLAG_FORCE_LARGE = 4
FLAG_VIRTUAL_SHARDS = 8
FLAG_LAST_BY_TOTAL = 16  # method variant: last level ranked by PED + completion (every path)


def FLAG_APPROX(shift: int) -> int:
    """Method variant: approximate top-K with PED bins of 2**shift (include/fastged.h FASTGED_FLAG_APPROX)."""
    return (int(shift) & 15) << 8

# The symbols include/fastged.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "fastged_create", "fastged_destroy", "fastged_last_error", "fastged_solve_pair", "fastged_solve_pair_ex",
    "fastged_solve_batch", "fastged_batch_upload", "fastged_batch_run", "fastged_batch_download",
    "fastged_batch_free", "fastged_get_stats", "fastged_version", "fastged_nccl_unique_id",
    "fastged_edit_path", "fastged_apply_edit_path", "fastged_graphs_equal_under_mapping",
)
OP_NAMES = {1: "vsub", 2: "vdel", 3: "vins", 4: "esub", 5: "edel", 6: "eins"}


class FastGedError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fastged error {code}: {msg}")
        self.code = code


class GraphT(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("vlabels", C.c_void_p), ("edges", C.c_void_p),
                ("elabels", C.c_void_p)]


# numpy twin of fastged_graph_t for vectorised batch marshalling
GRAPH_DTYPE = np.dtype([("n", "<i4"), ("m", "<i4"), ("vlabels", "<u8"), ("edges", "<u8"), ("elabels", "<u8")])
assert GRAPH_DTYPE.itemsize == C.sizeof(GraphT)


class CostsT(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("vsub", "vdel", "vins", "esub", "edel", "eins")]


class ConfigT(C.Structure):
    _fields_ = [("device", C.c_int32), ("stream", C.c_void_p), ("world_size", C.c_int32), ("rank", C.c_int32),
                ("nccl_id", C.c_void_p), ("flags", C.c_uint32)]


class ResultT(C.Structure):
    _fields_ = [("cost", C.c_int64), ("mapping", C.c_void_p), ("children_evaluated", C.c_int64),
                ("parents_expanded", C.c_int64), ("device_ms", C.c_float)]


class EditOpT(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("kind", "a", "b", "c", "d", "cost")]


class StatsT(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("device_ms", C.c_float), ("branch_ms", C.c_float),
                ("branch_launches", C.c_int64), ("children_evaluated", C.c_int64),
                ("parents_expanded", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("alg_bytes", C.c_int64), ("alg_ops", C.c_int64), ("phase_ms", C.c_float * 5),
                ("hist_children", C.c_int64)]


_lib = None


def lib(path: Optional[str] = None):
    """Load libfastged.so (built by ``__graft_entry__.build()``); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("FASTGED_LIB") or LIB_PATH  # FASTGED_LIB: A/B builds (scripts/ab_build.py)
    if not os.path.exists(path):
        raise FastGedError(ERR_CUDA, f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(path)
    P = C.c_void_p
    L.fastged_create.argtypes = [C.POINTER(ConfigT), C.POINTER(P)]
    L.fastged_destroy.argtypes = [P]
    L.fastged_destroy.restype = None
    L.fastged_last_error.argtypes = [P]
    L.fastged_last_error.restype = C.c_char_p
    L.fastged_solve_pair.argtypes = [P, C.POINTER(GraphT), C.POINTER(GraphT), C.POINTER(CostsT), C.c_int64,
                                     C.POINTER(ResultT)]
    L.fastged_solve_pair_ex.argtypes = [P, C.POINTER(GraphT), C.POINTER(GraphT), C.POINTER(CostsT), C.c_int64,
                                        C.POINTER(ResultT), P]
    L.fastged_solve_batch.argtypes = [P, C.c_int32, P, P, C.POINTER(CostsT), C.c_int64, P, P, P]
    L.fastged_batch_upload.argtypes = [P, C.c_int32, P, P, C.POINTER(P)]
    L.fastged_batch_run.argtypes = [P, P, C.POINTER(CostsT), C.c_int64]
    L.fastged_batch_download.argtypes = [P, P, P, P, P]
    L.fastged_batch_free.argtypes = [P, P]
    L.fastged_batch_free.restype = None
    L.fastged_get_stats.argtypes = [P, C.POINTER(StatsT)]
    L.fastged_version.restype = C.c_char_p
    L.fastged_nccl_unique_id.argtypes = [P]
    L.fastged_nccl_unique_id.restype = C.c_int
    L.fastged_edit_path.argtypes = [C.POINTER(GraphT), C.POINTER(GraphT), C.POINTER(CostsT), P, P, C.c_int32,
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
    L.fastged_apply_edit_path.argtypes = [C.POINTER(GraphT), C.POINTER(GraphT), P, C.c_int32, C.POINTER(C.c_int32),
                                          P, P, C.POINTER(C.c_int32), P, P]
    L.fastged_graphs_equal_under_mapping.argtypes = [C.POINTER(GraphT), C.POINTER(GraphT), P]
    for name in ("fastged_edit_path", "fastged_apply_edit_path", "fastged_graphs_equal_under_mapping"):
        getattr(L, name).restype = C.c_int
    for name in ("fastged_create", "fastged_solve_pair", "fastged_solve_pair_ex", "fastged_solve_batch",
                 "fastged_batch_upload", "fastged_batch_run", "fastged_batch_download", "fastged_get_stats"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


# ------------------------------------------------------------------ marshalling
def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int32)


def _graph_struct(g, keep: list) -> GraphT:
    vl, e = _i32(g.vlabels).reshape(-1), _i32(g.edges).reshape(-1)
    el = None if g.elabels is None else _i32(g.elabels).reshape(-1)
    keep += [vl, e, el]
    return GraphT(int(g.n), int(e.size // 2), vl.ctypes.data if vl.size else None,
                  e.ctypes.data if e.size else None, el.ctypes.data if el is not None and el.size else None)


class PackedGraphs:
    """All distinct graphs of a workload in three flat int32 arrays plus a fastged_graph_t table."""

    def __init__(self, graphs: Sequence):
        G = len(graphs)
        ns = np.fromiter((g.n for g in graphs), np.int64, G)
        ms = np.fromiter((g.edges.shape[0] for g in graphs), np.int64, G)
        self.vl = np.concatenate([_i32(g.vlabels).reshape(-1) for g in graphs] + [np.zeros(1, np.int32)])
        self.e = np.concatenate([_i32(g.edges).reshape(-1) for g in graphs] + [np.zeros(2, np.int32)])
        haslab = np.fromiter((g.elabels is not None for g in graphs), bool, G)
        self.el = np.concatenate([(_i32(g.elabels) if g.elabels is not None else np.zeros(g.edges.shape[0], np.int32))
                                  for g in graphs] + [np.zeros(1, np.int32)])
        voff = np.concatenate([[0], np.cumsum(ns)[:-1]]) if G else np.zeros(0, np.int64)
        eoff = np.concatenate([[0], np.cumsum(ms)[:-1]]) if G else np.zeros(0, np.int64)
        t = np.zeros(G, GRAPH_DTYPE)
        t["n"], t["m"] = ns, ms
        t["vlabels"] = self.vl.ctypes.data + 4 * voff
        t["edges"] = self.e.ctypes.data + 8 * eoff
        t["elabels"] = np.where(haslab, self.el.ctypes.data + 4 * eoff, 0)
        self.table = t
        self.n = ns

    def select(self, idx: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(self.table[np.asarray(idx, np.int64)])


def _costs(c) -> CostsT:
    return CostsT(*[int(x) for x in c])


# ------------------------------------------------------------------ handle
class Handle:
    """fastged_handle_t: one CUDA device (+ optional stream).  Synchronous calls unless noted."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, flags: int = 0,
                 world_size: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None):
        L = lib()
        self._L = L
        self._h = C.c_void_p()
        self._id = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
        cfg = ConfigT(int(device), C.c_void_p(stream) if stream else None, int(world_size), int(rank),
                      C.cast(self._id, C.c_void_p) if self._id is not None else None, int(flags))
        rc = L.fastged_create(C.byref(cfg), C.byref(self._h))
        if rc != OK:
            raise FastGedError(rc, L.fastged_last_error(None).decode())

    def close(self):
        if self._h:
            self._L.fastged_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc: int):
        if rc != OK:
            raise FastGedError(rc, self._L.fastged_last_error(self._h).decode())

    # -------------------------------------------------------------- calls
    def solve_pair(self, g1, g2, costs, K: int, levels: bool = False) -> dict:
        keep: list = []
        G1, G2 = _graph_struct(g1, keep), _graph_struct(g2, keep)
        mp = np.zeros(max(int(g1.n), 1), np.int32)
        res = ResultT(0, mp.ctypes.data, 0, 0, 0.0)
        lv = np.zeros(3 * max(int(g1.n), 1), np.int64) if levels else None
        self._check(self._L.fastged_solve_pair_ex(self._h, C.byref(G1), C.byref(G2), C.byref(_costs(costs)),
                                                  int(K), C.byref(res), lv.ctypes.data if levels else None))
        out = dict(cost=int(res.cost), mapping=mp[: int(g1.n)].copy(), children=int(res.children_evaluated),
                   parents=int(res.parents_expanded), device_ms=float(res.device_ms))
        if levels:
            out["levels"] = [tuple(int(x) for x in lv[3 * i:3 * i + 3]) for i in range(int(g1.n))]
        return out

    def solve_batch(self, packed: PackedGraphs, pair_a, pair_b, costs, K: int):
        """One call: H2D of the packed pairs, search, D2H.  Returns (costs, mappings_flat, map_offsets, children)."""
        g1s, g2s = packed.select(pair_a), packed.select(pair_b)
        P = g1s.shape[0]
        offs = np.concatenate([[0], np.cumsum(g1s["n"].astype(np.int64))])
        out_c = np.zeros(max(P, 1), np.int64)
        out_ch = np.zeros(max(P, 1), np.int64)
        out_m = np.zeros(max(int(offs[-1]), 1), np.int32)
        self._check(self._L.fastged_solve_batch(self._h, P, g1s.ctypes.data, g2s.ctypes.data, C.byref(_costs(costs)),
                                                int(K), out_c.ctypes.data, out_m.ctypes.data, out_ch.ctypes.data))
        return out_c[:P], out_m[: int(offs[-1])], offs, out_ch[:P]

    def stats(self) -> dict:
        s = StatsT()
        self._check(self._L.fastged_get_stats(self._h, C.byref(s)))
        return {k: (list(getattr(s, k)) if k == "phase_ms" else getattr(s, k)) for k, _ in StatsT._fields_}

    def upload(self, packed: PackedGraphs, pair_a, pair_b) -> "DeviceBatch":
        return DeviceBatch(self, packed, pair_a, pair_b)


class DeviceBatch:
    """fastged_batch_t: pairs validated, packed and resident in HBM."""

    def __init__(self, h: Handle, packed: PackedGraphs, pair_a, pair_b):
        self.h = h
        g1s, g2s = packed.select(pair_a), packed.select(pair_b)
        self.npairs = int(g1s.shape[0])
        self.offs = np.concatenate([[0], np.cumsum(g1s["n"].astype(np.int64))])
        self._b = C.c_void_p()
        h._check(h._L.fastged_batch_upload(h._h, self.npairs, g1s.ctypes.data, g2s.ctypes.data, C.byref(self._b)))

    def run(self, costs, K: int):
        """Enqueue the search on the handle's stream (asynchronous)."""
        self.h._check(self.h._L.fastged_batch_run(self.h._h, self._b, C.byref(_costs(costs)), int(K)))

    def download(self):
        P = self.npairs
        out_c = np.zeros(max(P, 1), np.int64)
        out_ch = np.zeros(max(P, 1), np.int64)
        out_m = np.zeros(max(int(self.offs[-1]), 1), np.int32)
        self.h._check(self.h._L.fastged_batch_download(self.h._h, self._b, out_c.ctypes.data, out_m.ctypes.data,
                                                       out_ch.ctypes.data))
        return out_c[:P], out_m[: int(self.offs[-1])], self.offs, out_ch[:P]

    def free(self):
        if self._b:
            self.h._L.fastged_batch_free(self.h._h, self._b)
            self._b = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for the sharded single-pair mode (rank 0 creates, torch.distributed broadcasts)."""
    buf = C.create_string_buffer(128)
    rc = lib().fastged_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc != OK:
        raise FastGedError(rc, "ncclGetUniqueId failed")
    return buf.raw


def _global_error(rc: int):
    if rc != 0:
        raise FastGedError(rc, (lib().fastged_last_error(None) or b"").decode())


def edit_path(g1, g2, costs, mapping):
    """Explicit edit path of a complete mapping (fastged_edit_path): (list of (op, a, b, c, d, cost), cost)."""
    keep = []
    G1, G2 = _graph_struct(g1, keep), _graph_struct(g2, keep)
    mp = _i32(mapping).reshape(-1)
    n, cost = C.c_int32(0), C.c_int64(0)
    _global_error(lib().fastged_edit_path(C.byref(G1), C.byref(G2), C.byref(_costs(costs)),
                                          mp.ctypes.data if mp.size else None, None, 0, C.byref(n), C.byref(cost)))
    ops = (EditOpT * max(n.value, 1))()
    _global_error(lib().fastged_edit_path(C.byref(G1), C.byref(G2), C.byref(_costs(costs)),
                                          mp.ctypes.data if mp.size else None, C.cast(ops, C.c_void_p), n.value,
                                          C.byref(n), C.byref(cost)))
    return [(OP_NAMES[o.kind], o.a, o.b, o.c, o.d, o.cost) for o in ops[: n.value]], int(cost.value)


def apply_edit_path(g1, g2, mapping, prefix_len: int):
    """The graph after the first prefix_len vertex operations (fastged_apply_edit_path).
    Returns (Graph, origin) with origin[v] = g2 vertex or -1 - g1 index (unresolved)."""
    from .synth import Graph
    keep = []
    G1, G2 = _graph_struct(g1, keep), _graph_struct(g2, keep)
    mp = _i32(mapping).reshape(-1)
    cap_n, cap_m = int(g1.n) + int(g2.n) + 1, int(g1.edges.shape[0]) + int(g2.edges.shape[0]) + 1
    vl, org = np.zeros(cap_n, np.int32), np.zeros(cap_n, np.int32)
    e, el = np.zeros(2 * cap_m, np.int32), np.zeros(cap_m, np.int32)
    n, m = C.c_int32(0), C.c_int32(0)
    _global_error(lib().fastged_apply_edit_path(C.byref(G1), C.byref(G2), mp.ctypes.data if mp.size else None,
                                                int(prefix_len), C.byref(n), vl.ctypes.data, org.ctypes.data, C.byref(m),
                                                e.ctypes.data, el.ctypes.data))
    return Graph(n.value, vl[: n.value], e[: 2 * m.value].reshape(-1, 2), el[: m.value]), org[: n.value]


def graphs_equal_under_mapping(a, b, mapping) -> bool:
    keep = []
    A, B = _graph_struct(a, keep), _graph_struct(b, keep)
    mp = _i32(mapping).reshape(-1)
    r = lib().fastged_graphs_equal_under_mapping(C.byref(A), C.byref(B), mp.ctypes.data if mp.size else None)
    if r < 0:
        _global_error(-r)
    return bool(r)


def version() -> str:
    return lib().fastged_version().decode()
