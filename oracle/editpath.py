"""Edit-path oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain Python restatement of SPEC S:78-96 / PAPER.md:89-116 for checking libfastged's host functions
fastged_edit_path / fastged_apply_edit_path / fastged_graphs_equal_under_mapping.  Shares no code with them.

Path order (the one include/fastged.h documents): for v_0..v_{n1-1} its vertex operation, then the implied
operations on the edges between v_i and each earlier v_q (q ascending; second-endpoint rule, reading C7);
then vertex insertions (ascending g2 index), then insertions of the g2 edges with an unused endpoint.
"""
from __future__ import annotations


def _adj(g):
    lab = {}
    el = g.elabels if g.elabels is not None else [0] * g.edges.shape[0]
    for (a, b), l in zip(g.edges.tolist(), list(el)):
        lab[(a, b)] = lab[(b, a)] = int(l)
    return lab


def edit_path(g1, g2, costs, mapping):
    vsub, vdel, vins, esub, edel, eins = costs
    A, B = _adj(g1), _adj(g2)
    ops, used = [], set()
    for i in range(g1.n):
        t = int(mapping[i])
        if t < 0:
            ops.append(("vdel", i, -1, -1, -1, vdel))
        else:
            ops.append(("vsub", i, t, -1, -1, 0 if g1.vlabels[i] == g2.vlabels[t] else vsub))
            used.add(t)
        for q in range(i):
            s = int(mapping[q])
            e1 = A.get((i, q))
            e2 = B.get((t, s)) if (t >= 0 and s >= 0) else None
            if e1 is not None and e2 is not None:
                ops.append(("esub", q, s, i, t, 0 if e1 == e2 else esub))
            elif e1 is not None:
                ops.append(("edel", q, -1, i, -1, edel))
            elif e2 is not None:
                ops.append(("eins", -1, s, -1, t, eins))
    for u in range(g2.n):
        if u not in used:
            ops.append(("vins", -1, u, -1, -1, vins))
    for x, y in sorted((min(a, b), max(a, b)) for a, b in g2.edges.tolist()):
        if x not in used or y not in used:
            ops.append(("eins", -1, x, -1, y, eins))
    return ops, sum(o[5] for o in ops)


def apply_edit_path(g1, g2, mapping, prefix_len):
    """Returns (n, vlabels, sorted edge list [(a, b, label)], origin) after the first prefix_len vertex ops."""
    used = {int(t) for t in mapping if t >= 0}
    ins = [u for u in range(g2.n) if u not in used]
    assert 0 <= prefix_len <= g1.n + len(ins)
    res, nins = min(prefix_len, g1.n), max(0, prefix_len - g1.n)
    A, B = _adj(g1), _adj(g2)
    verts = []  # (label, origin, g1 index or None)
    for i in range(g1.n):
        if i < res and mapping[i] < 0:
            continue  # deleted with its incident edges
        if i < res:
            verts.append((int(g2.vlabels[mapping[i]]), int(mapping[i]), i))
        else:
            verts.append((int(g1.vlabels[i]), -1 - i, i))
    for u in ins[:nins]:
        verts.append((int(g2.vlabels[u]), u, None))
    edges = []
    for a in range(len(verts)):
        for b in range(a + 1, len(verts)):
            oa, ob = verts[a][1], verts[b][1]
            if oa >= 0 and ob >= 0:
                l = B.get((oa, ob))
            else:
                l = A.get((verts[a][2], verts[b][2])) if verts[a][2] is not None and verts[b][2] is not None else None
            if l is not None:
                edges.append((a, b, l))
    return len(verts), [v[0] for v in verts], edges, [v[1] for v in verts]


def graphs_equal_under_mapping(a, b, mapping):
    if a.n != b.n or sorted(int(x) for x in mapping) != list(range(b.n)):
        raise ValueError("mapping is not a bijection")
    if any(int(a.vlabels[v]) != int(b.vlabels[mapping[v]]) for v in range(a.n)):
        return False
    A, B = _adj(a), _adj(b)
    if len(A) != len(B):
        return False
    return all(B.get((int(mapping[x]), int(mapping[y]))) == l for (x, y), l in A.items())
