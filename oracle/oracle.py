"""ctypes binding of oracle/fastged_oracle.c — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Graphs are duck-typed: any object with ``n``, ``vlabels`` (int32[n]),
``edges`` (int32[m,2]) and ``elabels`` (int32[m] or None).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FASTGED_ORACLE_LIB: a mutated build for scripts/oracle_mutations.py (never set otherwise)
LIB_PATH = os.environ.get("FASTGED_ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "fastged_oracle.c")


class OgGraph(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("vlabels", C.c_void_p),
                ("edges", C.c_void_p), ("elabels", C.c_void_p)]


class OgCosts(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("vsub", "vdel", "vins", "esub", "edel", "eins")]


class OgLevel(C.Structure):
    _fields_ = [("frontier", C.c_int64), ("candidates", C.c_int64), ("threshold", C.c_int64),
                ("min_ped", C.c_int64)]


ERRORS = {0: "ok", 1: "bad argument", 2: "invalid graph", 3: "out of memory", 7: "witness self-check failed"}


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle error {code}: {ERRORS.get(code, '?')}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp).  Building the checker is not using it."""
    if os.environ.get("FASTGED_ORACLE_LIB"):
        return LIB_PATH
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-Wall",
                               "-o", tmp, SRC_PATH])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.og_kbest.argtypes = [C.POINTER(OgGraph), C.POINTER(OgGraph), C.POINTER(OgCosts), C.c_int64,
                               C.POINTER(C.c_int64), C.c_void_p, C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64), C.c_void_p]
        L.og_kbest.restype = C.c_int
        L.og_kbest_batch.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(OgCosts), C.c_int64,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
        L.og_kbest_batch.restype = C.c_int
        L.og_exact.argtypes = [C.POINTER(OgGraph), C.POINTER(OgGraph), C.POINTER(OgCosts), C.c_int64, C.c_int64,
                               C.POINTER(C.c_int64), C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.og_exact.restype = C.c_int
        L.og_exact_batch.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(OgCosts), C.c_int64, C.c_int64,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
        L.og_exact_batch.restype = C.c_int
        L.og_kbest_ex.argtypes = L.og_kbest.argtypes + [C.c_int32]
        L.og_kbest_ex.restype = C.c_int
        L.og_kbest_batch_ex.argtypes = L.og_kbest_batch.argtypes + [C.c_int32]
        L.og_kbest_batch_ex.restype = C.c_int
        L.og_mapping_cost.argtypes = [C.POINTER(OgGraph), C.POINTER(OgGraph), C.POINTER(OgCosts),
                                      C.c_void_p, C.POINTER(C.c_int64)]
        L.og_mapping_cost.restype = C.c_int
        L.og_max_threads.restype = C.c_int
        L.og_select.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        L.og_select.restype = C.c_int
        _lib = L
    return _lib


def _arr(x, dtype=np.int32):
    return np.ascontiguousarray(x, dtype=dtype)


def _graph(g, keep):
    vl = _arr(g.vlabels).reshape(-1)
    e = _arr(g.edges).reshape(-1)
    el = None if g.elabels is None else _arr(g.elabels).reshape(-1)
    keep += [vl, e, el]
    return OgGraph(int(g.n), int(e.shape[0] // 2), vl.ctypes.data if vl.size else None,
                   e.ctypes.data if e.size else None, None if el is None or el.size == 0 else el.ctypes.data)


def _costs(c):
    return OgCosts(*[int(x) for x in c])


LAST_BY_TOTAL = 1  # method variant: last level ranked by PED + completion


def APPROX(shift: int) -> int:
    """flags of the approximate top-K variant: bins of 2**shift PED units."""
    return (int(shift) & 15) << 8


def kbest(g1, g2, costs, K, levels: bool = False, flags: int = 0):
    """Returns dict(cost, mapping, children, parents[, levels])."""
    keep = []
    G1, G2 = _graph(g1, keep), _graph(g2, keep)
    cost, ch, pa = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    mp = np.zeros(max(int(g1.n), 1), np.int32)
    lv = (OgLevel * max(int(g1.n), 1))() if levels else None
    rc = lib().og_kbest_ex(C.byref(G1), C.byref(G2), C.byref(_costs(costs)), int(K), C.byref(cost),
                           mp.ctypes.data, C.byref(ch), C.byref(pa), C.cast(lv, C.c_void_p) if levels else None,
                           int(flags))
    if rc != 0:
        raise OracleError(rc)
    out = dict(cost=int(cost.value), mapping=mp[: int(g1.n)].copy(), children=int(ch.value), parents=int(pa.value))
    if levels:
        out["levels"] = [(lv[i].frontier, lv[i].candidates, lv[i].threshold) for i in range(int(g1.n))]
        out["min_ped"] = [lv[i].min_ped for i in range(int(g1.n))]
    return out


def kbest_batch(pairs, costs, K, nthreads: int = 0, flags: int = 0):
    """pairs: sequence of (g1, g2).  Returns (costs int64[P], mappings list, children int64[P])."""
    keep = []
    P = len(pairs)
    G1 = (OgGraph * max(P, 1))()
    G2 = (OgGraph * max(P, 1))()
    offs = np.zeros(P + 1, np.int64)
    for k, (a, b) in enumerate(pairs):
        G1[k] = _graph(a, keep)
        G2[k] = _graph(b, keep)
        offs[k + 1] = offs[k] + int(a.n)
    out_c = np.zeros(max(P, 1), np.int64)
    out_ch = np.zeros(max(P, 1), np.int64)
    out_m = np.zeros(max(int(offs[-1]), 1), np.int32)
    st = np.zeros(max(P, 1), np.int32)
    rc = lib().og_kbest_batch_ex(P, C.cast(G1, C.c_void_p), C.cast(G2, C.c_void_p), C.byref(_costs(costs)), int(K),
                                 out_c.ctypes.data, out_m.ctypes.data, offs.ctypes.data, out_ch.ctypes.data,
                                 int(nthreads), st.ctypes.data, int(flags))
    if rc != 0:
        raise OracleError(rc)
    maps = [out_m[offs[k]:offs[k + 1]].copy() for k in range(P)]
    return out_c[:P].copy(), maps, out_ch[:P].copy()


def exact(g1, g2, costs, K0: int = 1, node_limit: int = 10 ** 9):
    """Exact GED by DFS branch and bound.  Returns dict(cost, mapping, nodes, optimal);
    optimal is False when node_limit expansions ran out (cost is then the best path found)."""
    keep = []
    G1, G2 = _graph(g1, keep), _graph(g2, keep)
    cost, nodes, opt = C.c_int64(0), C.c_int64(0), C.c_int32(0)
    mp = np.zeros(max(int(g1.n), 1), np.int32)
    rc = lib().og_exact(C.byref(G1), C.byref(G2), C.byref(_costs(costs)), int(K0), int(node_limit), C.byref(cost),
                        mp.ctypes.data, C.byref(nodes), C.byref(opt))
    if rc != 0:
        raise OracleError(rc)
    return dict(cost=int(cost.value), mapping=mp[: int(g1.n)].copy(), nodes=int(nodes.value), optimal=bool(opt.value))


def exact_batch(pairs, costs, K0: int = 1, node_limit: int = 10 ** 9, nthreads: int = 0):
    """Exact GED of every pair (OpenMP over pairs).  Returns (costs, mappings, nodes, optimal)."""
    keep = []
    P = len(pairs)
    G1 = (OgGraph * max(P, 1))()
    G2 = (OgGraph * max(P, 1))()
    offs = np.zeros(P + 1, np.int64)
    for k, (a, b) in enumerate(pairs):
        G1[k] = _graph(a, keep)
        G2[k] = _graph(b, keep)
        offs[k + 1] = offs[k] + int(a.n)
    out_c = np.zeros(max(P, 1), np.int64)
    out_n = np.zeros(max(P, 1), np.int64)
    out_o = np.zeros(max(P, 1), np.int32)
    out_m = np.zeros(max(int(offs[-1]), 1), np.int32)
    st = np.zeros(max(P, 1), np.int32)
    rc = lib().og_exact_batch(P, C.cast(G1, C.c_void_p), C.cast(G2, C.c_void_p), C.byref(_costs(costs)), int(K0),
                              int(node_limit), out_c.ctypes.data, out_m.ctypes.data, offs.ctypes.data,
                              out_n.ctypes.data, out_o.ctypes.data, int(nthreads), st.ctypes.data)
    if rc != 0:
        raise OracleError(rc)
    maps = [out_m[offs[k]:offs[k + 1]].copy() for k in range(P)]
    return out_c[:P].copy(), maps, out_n[:P].copy(), out_o[:P].astype(bool)


def mapping_cost(g1, g2, costs, mapping) -> int:
    keep = []
    G1, G2 = _graph(g1, keep), _graph(g2, keep)
    f = _arr(mapping)
    out = C.c_int64(0)
    rc = lib().og_mapping_cost(C.byref(G1), C.byref(G2), C.byref(_costs(costs)),
                               f.ctypes.data if f.size else None, C.byref(out))
    if rc != 0:
        raise OracleError(rc)
    return int(out.value)


def select(ped, p, j, k) -> np.ndarray:
    """Indices (ascending) of the k smallest keys (ped, p, j) as the oracle's selection step picks them."""
    ped, p, j = _arr(ped, np.int64), _arr(p, np.int64), _arr(j, np.int32)
    n = int(ped.shape[0])
    out = np.zeros(max(min(int(k), n), 1), np.int64)
    rc = lib().og_select(ped.ctypes.data, p.ctypes.data, j.ctypes.data, n, int(k), out.ctypes.data)
    if rc != 0:
        raise OracleError(rc)
    return out[:min(int(k), n)].copy()


def max_threads() -> int:
    return int(lib().og_max_threads())
