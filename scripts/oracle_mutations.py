#!/usr/bin/env python3
"""Mutation sweep of the CPU oracle against its pins (VERDICT r1 'Next round' #1).

Each mutant is one plausible mistake in oracle/fastged_oracle.c (a dropped term, a swapped cost,
a wrong tie key, a wrong reading of C10/C13, ...).  The mutated source is compiled to a temporary
library and tests/test_oracle_pins.py is run against it (FASTGED_ORACLE_LIB).  A pin set is only
trusted if every mutant is killed (at least one pin fails).

    python scripts/oracle_mutations.py [--out profiles/r2_oracle_mutations.txt]
"""
import argparse
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "fastged_oracle.c")

C10_ALT = """        if (i == n1 - 1) /* MUTANT: rank the last level by PED + completion (C10 alternative) */
            for (int64_t s = 0; s < cnt; s++) {
                char *u = used + pool[s].p * (int64_t)n2;
                if (pool[s].j < n2) u[pool[s].j] = 1;
                pool[s].key = pool[s].ped + completion_cost(g2, c, u);
                if (pool[s].j < n2) u[pool[s].j] = 0;
            }
        select_k(pool, cnt, keep);
"""

# (name, exact text in the source, replacement)
MUTANTS = [
    ("C13: survivors not re-sorted by (p, j)", "        qsort(pool, (size_t)keep, sizeof(cand), cmp_pos);\n", "\n"),
    ("C10: last level ranked by PED + completion", "        select_k(pool, cnt, keep);\n", C10_ALT),
    ("C12: parent tie key reversed", "    if (a->p != b->p) return a->p < b->p ? -1 : 1;\n    return (a->j > b->j) - (a->j < b->j);\n}\nstatic int cmp_pos",
     "    if (a->p != b->p) return a->p > b->p ? -1 : 1;\n    return (a->j > b->j) - (a->j < b->j);\n}\nstatic int cmp_pos"),
    ("C12: child tie key reversed", "    return (a->j > b->j) - (a->j < b->j);\n}\nstatic int cmp_pos",
     "    return (a->j < b->j) - (a->j > b->j);\n}\nstatic int cmp_pos"),
    ("C12: PED order reversed", "    if (a->key != b->key) return a->key < b->key ? -1 : 1;", "    if (a->key != b->key) return a->key > b->key ? -1 : 1;"),
    ("keep K + 1 survivors", "        int64_t keep = cnt < K ? cnt : K;\n", "        int64_t keep = cnt < K + 1 ? cnt : K + 1;\n"),
    ("keep K - 1 survivors", "        int64_t keep = cnt < K ? cnt : K;\n", "        int64_t keep = cnt < K - 1 || K == 1 ? (cnt < K ? cnt : K) : K - 1;\n"),
    ("edel <-> eins in the implied-edge charge", "    if (e1) return c->edel;\n    if (e2) return c->eins;",
     "    if (e1) return c->eins;\n    if (e2) return c->edel;"),
    ("esub dropped (labelled edges substitute for free)", "? 0 : c->esub;\n    if (e1)", "? 0 : 0;\n    if (e1)"),
    ("edge-label test inverted", "lab1[i * n1 + q] == lab2[j * n2 + t] ? 0 : c->esub", "lab1[i * n1 + q] == lab2[j * n2 + t] ? c->esub : 0"),
    ("implied edges: last earlier level skipped", "for (int q = 0; q < i; q++) /* implied", "for (int q = 0; q + 1 < i; q++) /* implied"),
    ("implied edges: first level skipped", "for (int q = 0; q < i; q++) /* implied", "for (int q = 1; q < i; q++) /* implied"),
    ("vdel <-> vins (vertex deletion charged vins)", "    if (j == DEL) return c->vdel;", "    if (j == DEL) return c->vins;"),
    ("vertex substitution free on different labels", "g1->vlabels[i] == g2->vlabels[j] ? 0 : c->vsub;", "g1->vlabels[i] != g2->vlabels[j] ? 0 : c->vsub;"),
    ("completion: g2 edge needs both endpoints unused", "        if (!used[x] || !used[y]) s += c->eins;", "        if (!used[x] && !used[y]) s += c->eins;"),
    ("completion: unused vertex charged vdel", "        if (!used[u]) s += c->vins;", "        if (!used[u]) s += c->vdel;"),
    ("completion dropped", "            int64_t total = ped[k] + completion_cost(g2, c, used + k * (n2 > 0 ? n2 : 0));",
     "            int64_t total = ped[k];"),
    ("deletion child never generated", "                valid[slot] = (op == DEL) || !used[p * n2 + op];", "                valid[slot] = (op != DEL) && !used[p * n2 + op];"),
    ("deletion child first (j = 0 deletes)", "                int op = (j == n2) ? DEL : j;", "                int op = (j == 0) ? DEL : j - 1;"),
    ("used target not marked in the child", "            if (op != DEL) nused[k * n2 + op] = 1;", "            (void)0;"),
    ("argmin takes the last of equal totals", "if (best < 0 || total < best_total)", "if (best < 0 || total <= best_total)"),
    ("g1 vertices branched in reverse order", "        int64_t e = ped[p] + vertex_cost(g1, g2, c, i, op);", "        int64_t e = ped[p] + vertex_cost(g1, g2, c, n1 - 1 - i, op);"),
    # exact branch and bound (og_exact, NEXT-1)
    ("B&B: lower bound doubled (not admissible)", "    return (r1 > r2 ? (r1 - r2) * c->vdel : (r2 - r1) * c->vins) +",
     "    return 2 * (r1 > r2 ? (r1 - r2) * c->vdel : (r2 - r1) * c->vins) +"),
    ("B&B: leaf completion drops the edge insertions", "        const int64_t total = ped + (int64_t)S->c->vins * (n2 - nused) + (int64_t)S->c->eins * (g2->m - e2u);",
     "        const int64_t total = ped + (int64_t)S->c->vins * (n2 - nused);"),
    ("B&B: used target not released after the subtree", "        if (op != DEL) S->used[op] = 0;\n        if (S->over) return;", "        if (S->over) return;"),
    ("B&B: g2 edges among unused vertices not decremented", "        const int64_t nrem2 = rem2 - cf;", "        const int64_t nrem2 = rem2;"),
]


def build(src_text: str, out: str) -> bool:
    cpath = out[:-3] + ".c"
    with open(cpath, "w") as f:
        f.write(src_text)
    r = subprocess.run(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", out, cpath],
                       capture_output=True, text=True)
    return r.returncode == 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    base = open(SRC).read()
    lines = []
    killed = 0
    with tempfile.TemporaryDirectory() as td:
        for k, (name, old, new) in enumerate(MUTANTS):
            if base.count(old) != 1:
                lines.append(f"SKIP  {name}: pattern found {base.count(old)} times")
                continue
            lib = os.path.join(td, f"m{k}.so")
            if not build(base.replace(old, new), lib):
                lines.append(f"SKIP  {name}: mutant does not compile")
                continue
            env = dict(os.environ, FASTGED_ORACLE_LIB=lib)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                                os.path.join(ROOT, "tests", "test_oracle_pins.py"),
                                os.path.join(ROOT, "tests", "test_exact_oracle.py")],
                               capture_output=True, text=True, env=env, cwd=ROOT, timeout=1200)
            failed = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            if r.returncode != 0:
                killed += 1
                lines.append(f"KILLED {name}: {failed[0][7:] if failed else 'error'}")
            else:
                lines.append(f"SURVIVED {name}")
            print(lines[-1], flush=True)
    lines.append(f"{killed} of {len(MUTANTS)} mutants killed by tests/test_oracle_pins.py + tests/test_exact_oracle.py")
    print(lines[-1])
    if args.out:
        with open(args.out, "w") as f:
            f.write("# python scripts/oracle_mutations.py (oracle/fastged_oracle.c vs tests/test_oracle_pins.py + test_exact_oracle.py)\n")
            f.write("\n".join(lines) + "\n")
    return 0 if killed == len(MUTANTS) else 1


if __name__ == "__main__":
    sys.exit(main())
