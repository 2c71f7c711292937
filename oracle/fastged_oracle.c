/*
 * fastged_oracle.c -- CPU ORACLE for the FAST-GED K-Best search (arXiv 2605.00830).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the plain, slow, obviously-correct
 * statement of what the CUDA hot path must compute.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load it.  It shares no code, header, table or helper with
 * paper_2605_00830_b200/ (the product), and the product never calls it.
 *
 * Citations: P:<line> = /root/reference/PAPER.md, S:<line> = SPEC.md, and the
 * readings C1..C27 of SURVEY.md §8(c) O.2 (restated in DESIGN.md §3).
 *
 *   Graph  G = (V, E, alpha, beta), simple undirected labelled  (C17)
 *   Vertex-centric edit operations: substitution, deletion, insertion
 *   Implied edge operations, three cases
 *   Cost function: six integer constants, 0 for equal labels      (C1, C2)
 *   Algorithm 1: level loop, branch, evaluate, keep best K
 *   Branching: |R_V2| substitutions + one deletion child           (C5)
 *   Evaluation: PED = E(parent) + c(v<-u) + Imp_cost               (Alg. 2)
 *   Insertions only after the last level                          (C6)
 *   best_path <- lambda of the best node in the final List         (C10)
 *
 * Readings: g1 vertices are branched in index order v_0..v_{n1-1} (C4);
 * the deletion child has index j = n2 (C5); every successor of a level competes
 * in one pool (C27) and exactly min(K, |pool|) are kept, the smallest under the
 * lexicographic key (PED, p, j) where p is the parent's position in the
 * canonical frontier order (C12); survivors form the next frontier in ascending
 * (p, j) order (C13); at the last level the K survivors (selected by PED, C10)
 * get the completion cost and the argmin by (total, position) is returned.
 * Selection is Hoare's FIND (quickselect) on the unique keys, then a sort of only the K
 * survivors by (p, j) -- the same set a full sort would give (P5 pin).
 *
 * Parity pins: see tests/test_oracle_pins.py (worked examples S:64-76,
 * S:191-213, closed forms, brute force over all partial injections).
 *
 * Arithmetic is int64 throughout; nothing is rounded.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t n, m;
    const int32_t *vlabels; /* [n] */
    const int32_t *edges;   /* [2m] (u, v) pairs */
    const int32_t *elabels; /* [m] or NULL = every edge has label 0 */
} og_graph;

typedef struct {
    int32_t vsub, vdel, vins, esub, edel, eins;
} og_costs;

/* Per-level record (optional output): frontier size entering the level,
 * candidates generated, PED of the last kept candidate (-1 when all kept). */
typedef struct {
    int64_t frontier;
    int64_t candidates;
    int64_t threshold;
    int64_t min_ped;    /* smallest candidate PED of the level */
} og_level;

enum { OG_OK = 0, OG_ERR_ARG = 1, OG_ERR_INPUT = 2, OG_ERR_MEM = 3, OG_ERR_SELFCHECK = 7 };

#define DEL (-1)

/* ---- validation: simple undirected graph, no loops, endpoints in range (C17) ---- */
static int validate_graph(const og_graph *g) {
    if (!g || g->n < 0 || g->m < 0) return OG_ERR_ARG;
    if (g->n > 0 && !g->vlabels) return OG_ERR_ARG;
    if (g->m > 0 && !g->edges) return OG_ERR_ARG;
    for (int e = 0; e < g->m; e++) {
        int a = g->edges[2 * e], b = g->edges[2 * e + 1];
        if (a < 0 || b < 0 || a >= g->n || b >= g->n || a == b) return OG_ERR_INPUT;
    }
    return OG_OK;
}

/* Dense adjacency: has[i*n+j] = 1 if edge, lab[i*n+j] = its label.
 * Returns OG_ERR_INPUT on a duplicate edge (at most one edge per pair). */
static int dense_adjacency(const og_graph *g, char *has, int32_t *lab) {
    int n = g->n;
    memset(has, 0, (size_t)n * n);
    for (int e = 0; e < g->m; e++) {
        int a = g->edges[2 * e], b = g->edges[2 * e + 1];
        int32_t l = g->elabels ? g->elabels[e] : 0;
        if (has[a * n + b]) return OG_ERR_INPUT;
        has[a * n + b] = has[b * n + a] = 1;
        lab[a * n + b] = lab[b * n + a] = l;
    }
    return OG_OK;
}

/* Vertex operation cost: substitution is 0 on equal labels else vsub; deletion vdel. */
static int64_t vertex_cost(const og_graph *g1, const og_graph *g2, const og_costs *c, int i, int j) {
    if (j == DEL) return c->vdel;
    return g1->vlabels[i] == g2->vlabels[j] ? 0 : c->vsub;
}

/* Implied edge charge between the new operation v_i -> j and an earlier operation
 * v_q -> t.  Edge in both graphs: substituted, esub unless
 * labels are equal (C2).  Only in g1: deleted (edel).  Only in g2: inserted (eins).
 * A deleted endpoint has no g2 image, so its g1 edges are deleted. */
static int64_t edge_charge(const char *has1, const int32_t *lab1, int n1,
                           const char *has2, const int32_t *lab2, int n2,
                           const og_costs *c, int i, int j, int q, int t) {
    int e1 = has1[i * n1 + q];
    int e2 = (j != DEL && t != DEL) ? has2[j * n2 + t] : 0;
    if (e1 && e2) return lab1[i * n1 + q] == lab2[j * n2 + t] ? 0 : c->esub;
    if (e1) return c->edel;
    if (e2) return c->eins;
    return 0;
}

typedef struct {
    int64_t ped;
    int64_t p; /* parent position in the frontier */
    int32_t j; /* g2 vertex index, or n2 for deletion */
    int64_t key; /* ranking value: the PED, or (variant, last level) PED + completion */
} cand;

static int cmp_key(const void *x, const void *y) { /* (PED, p, j) ascending (C12) */
    const cand *a = (const cand *)x, *b = (const cand *)y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->p != b->p) return a->p < b->p ? -1 : 1;
    return (a->j > b->j) - (a->j < b->j);
}
static int cmp_pos(const void *x, const void *y) { /* (p, j) ascending (C13) */
    const cand *a = (const cand *)x, *b = (const cand *)y;
    if (a->p != b->p) return a->p < b->p ? -1 : 1;
    return (a->j > b->j) - (a->j < b->j);
}

/* "List <- best K nodes of list_tmp" without a full sort: Hoare's FIND
 * (quickselect).  Rearranges a[0..n) so that a[0..k) holds the k smallest keys under
 * (PED, p, j) (C12), in no particular order.  Keys are unique, so the set is unique (SURVEY
 * §8(c) O.3 P5) and does not depend on the pivots, which come from a fixed xorshift sequence. */
static void select_k(cand *a, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n - 1; /* invariant: the k-th smallest lies in a[lo..hi] */
    uint64_t rnd = 0x9E3779B97F4A7C15ull;
    if (k <= 0 || k >= n) return;
    while (lo < hi) {
        rnd ^= rnd << 13; rnd ^= rnd >> 7; rnd ^= rnd << 17;
        cand pivot = a[lo + (int64_t)(rnd % (uint64_t)(hi - lo + 1))];
        int64_t i = lo, j = hi;
        while (i <= j) { /* Hoare partition around the pivot key */
            while (cmp_key(&a[i], &pivot) < 0) i++;
            while (cmp_key(&a[j], &pivot) > 0) j--;
            if (i <= j) { cand t = a[i]; a[i] = a[j]; a[j] = t; i++; j--; }
        }
        /* now a[lo..j] <= pivot <= a[i..hi], and j < i */
        if (k - 1 <= j) hi = j;
        else if (k - 1 >= i) lo = i;
        else return; /* a[j+1..i-1] equal the pivot: position k-1 is settled */
    }
}

/* Completion (C6): insert every unused g2 vertex (vins each) and
 * every g2 edge with at least one unused endpoint (eins each, second-endpoint rule C7). */
static int64_t completion_cost(const og_graph *g2, const og_costs *c, const char *used) {
    int64_t s = 0;
    for (int u = 0; u < g2->n; u++)
        if (!used[u]) s += c->vins;
    for (int e = 0; e < g2->m; e++) {
        int x = g2->edges[2 * e], y = g2->edges[2 * e + 1];
        if (!used[x] || !used[y]) s += c->eins;
    }
    return s;
}

/* Order-free cost of a complete vertex mapping f: V1 -> V2 u {DEL} (
 * SURVEY §8(c) O.4).  Used only to re-verify the returned witness. */
static int64_t mapping_cost(const og_graph *g1, const og_graph *g2, const og_costs *c,
                            const char *has1, const char *has2, const int32_t *lab2, const int32_t *f) {
    int n1 = g1->n, n2 = g2->n;
    int64_t s = 0;
    char *img = (char *)calloc((size_t)(n2 > 0 ? n2 : 1), 1);
    int32_t *inv = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n2 > 0 ? n2 : 1));
    for (int u = 0; u < n2; u++) inv[u] = -1;
    for (int i = 0; i < n1; i++) {
        if (f[i] == DEL) s += c->vdel;
        else {
            s += (g1->vlabels[i] == g2->vlabels[f[i]]) ? 0 : c->vsub;
            img[f[i]] = 1;
            inv[f[i]] = i;
        }
    }
    for (int u = 0; u < n2; u++)
        if (!img[u]) s += c->vins;
    for (int e = 0; e < g1->m; e++) {
        int a = g1->edges[2 * e], b = g1->edges[2 * e + 1];
        int32_t l1 = g1->elabels ? g1->elabels[e] : 0;
        if (f[a] != DEL && f[b] != DEL && has2[f[a] * n2 + f[b]])
            s += (l1 == lab2[f[a] * n2 + f[b]]) ? 0 : c->esub;
        else
            s += c->edel;
    }
    for (int e = 0; e < g2->m; e++) {
        int x = g2->edges[2 * e], y = g2->edges[2 * e + 1];
        int matched = 0;
        if (img[x] && img[y]) matched = has1[inv[x] * n1 + inv[y]];
        if (!matched) s += c->eins;
    }
    free(img);
    free(inv);
    return s;
}

#define OG_LAST_BY_TOTAL 1 /* method variant: last level ranked by PED + completion */
/* method variant ("approximate top-k selection"): flags bits 8..11 = s > 0 --
 * each level keeps the min(K, c_i) smallest children under the coarse key (floor((PED - lo_i) / 2^s), p, j),
 * lo_i = the smallest PED of the level's parents: children whose PEDs share a bin of width 2^s are
 * ranked by position only (s = 0: the exact selection) */
#define OG_APPROX_SHIFT(flags) (((flags) >> 8) & 15)

/*
 * og_kbest: Algorithm 1 with the readings listed at the top.
 *   cost_out      : GED upper bound (the cost of the returned edit path)
 *   mapping_out   : [g1->n] g2 index or -1 (deleted); insertions are implied
 *   children_out  : total candidates generated over all levels (sum c_i), may be NULL
 *   parents_out   : total frontier nodes expanded (sum N_i), may be NULL
 *   levels_out    : [g1->n] per-level record, may be NULL
 */
int og_kbest_ex(const og_graph *g1, const og_graph *g2, const og_costs *c, int64_t K,
                int64_t *cost_out, int32_t *mapping_out, int64_t *children_out,
                int64_t *parents_out, og_level *levels_out, int32_t flags) {
    int rc;
    if (!c || !cost_out || K < 1) return OG_ERR_ARG;
    if (c->vsub < 0 || c->vdel < 0 || c->vins < 0 || c->esub < 0 || c->edel < 0 || c->eins < 0)
        return OG_ERR_ARG;
    if ((rc = validate_graph(g1)) != OG_OK) return rc;
    if ((rc = validate_graph(g2)) != OG_OK) return rc;
    if (g1->n > 0 && !mapping_out) return OG_ERR_ARG;

    const int n1 = g1->n, n2 = g2->n;
    const size_t a1 = (size_t)(n1 > 0 ? n1 * n1 : 1), a2 = (size_t)(n2 > 0 ? n2 * n2 : 1);
    char *has1 = (char *)malloc(a1), *has2 = (char *)malloc(a2);
    int32_t *lab1 = (int32_t *)malloc(a1 * sizeof(int32_t)), *lab2 = (int32_t *)malloc(a2 * sizeof(int32_t));
    if (dense_adjacency(g1, has1, lab1) != OG_OK || dense_adjacency(g2, has2, lab2) != OG_OK) {
        free(has1); free(has2); free(lab1); free(lab2);
        return OG_ERR_INPUT;
    }

    /* Frontier F_i: node k has ped[k], map[k*n1 + q] for q < i, used[k*n2 + u]. */
    int64_t N = 1; /* root: lambda empty, all of V2 remaining */
    int64_t *ped = (int64_t *)calloc(1, sizeof(int64_t));
    int32_t *map = (int32_t *)calloc((size_t)(n1 > 0 ? n1 : 1), sizeof(int32_t));
    char *used = (char *)calloc((size_t)(n2 > 0 ? n2 : 1), 1);
    int64_t children = 0, parents = 0;
    rc = OG_OK;

    for (int i = 0; i < n1 && rc == OG_OK; i++) { /* ForEach v in V1, order C4 */
        /* Branch + evaluate every node of List. */
        int64_t C = N * (int64_t)(n2 + 1);
        const int shift = OG_APPROX_SHIFT(flags);
        int64_t lo = ped[0]; /* smallest parent PED (the bins' origin) */
        for (int64_t p = 1; p < N; p++)
            if (ped[p] < lo) lo = ped[p];
        cand *pool = (cand *)malloc(sizeof(cand) * (size_t)C);
        char *valid = (char *)malloc((size_t)C);
        if (!pool || !valid) { free(pool); free(valid); rc = OG_ERR_MEM; break; }
#pragma omp parallel for schedule(dynamic, 64) if (N * (int64_t)(n2 + 1) * (i + 1) > (1 << 20))
        for (int64_t p = 0; p < N; p++) {
            for (int j = 0; j <= n2; j++) { /* j = n2 is the deletion child (C5) */
                int64_t slot = p * (n2 + 1) + j;
                int op = (j == n2) ? DEL : j;
                valid[slot] = (op == DEL) || !used[p * n2 + op];
                if (!valid[slot]) continue;
                int64_t e = ped[p] + vertex_cost(g1, g2, c, i, op);
                for (int q = 0; q < i; q++) /* implied edges vs all earlier operations */
                    e += edge_charge(has1, lab1, n1, has2, lab2, n2, c, i, op, q, map[p * n1 + q]);
                pool[slot].ped = e;
                pool[slot].p = p;
                pool[slot].j = j;
                pool[slot].key = shift ? (e - lo) >> shift : e; /* (e >= ped[p] >= lo) */
            }
        }
        int64_t cnt = 0;
        for (int64_t s = 0; s < C; s++)
            if (valid[s]) pool[cnt++] = pool[s];
        free(valid);
        children += cnt;
        parents += N;

        /* List <- best K nodes of list_tmp: the min(K, cnt) smallest keys (C12). */
        int64_t keep = cnt < K ? cnt : K;
        if ((flags & OG_LAST_BY_TOTAL) && i == n1 - 1) {
            /* variant: rank the last level by the total PED + completion of each child (the
             * alternative to reading C10 of P:185-187) */
            char *u2 = (char *)malloc((size_t)(n2 > 0 ? n2 : 1));
            if (!u2) { free(pool); rc = OG_ERR_MEM; break; }
            for (int64_t s = 0; s < cnt; s++) {
                if (n2 > 0) memcpy(u2, used + pool[s].p * n2, (size_t)n2);
                if (pool[s].j < n2) u2[pool[s].j] = 1;
                pool[s].key = pool[s].ped + completion_cost(g2, c, u2);
            }
            free(u2);
        }
        select_k(pool, cnt, keep);
        if (levels_out) {
            int64_t mn = -1, mx = -1;
            for (int64_t s = 0; s < cnt; s++)
                if (mn < 0 || pool[s].key < mn) mn = pool[s].key;
            for (int64_t s = 0; s < keep; s++)
                if (pool[s].key > mx) mx = pool[s].key;
            levels_out[i].frontier = N;
            levels_out[i].candidates = cnt;
            levels_out[i].threshold = (cnt > K) ? mx : -1; /* ranking value of the K-th smallest key */
            levels_out[i].min_ped = mn;
        }
        /* Next frontier in canonical (p, j) order (C13). */
        qsort(pool, (size_t)keep, sizeof(cand), cmp_pos);
        int64_t *nped = (int64_t *)malloc(sizeof(int64_t) * (size_t)keep);
        int32_t *nmap = (int32_t *)malloc(sizeof(int32_t) * (size_t)keep * (size_t)n1);
        char *nused = (char *)malloc((size_t)keep * (size_t)(n2 > 0 ? n2 : 1));
        if (!nped || !nmap || !nused) { free(pool); free(nped); free(nmap); free(nused); rc = OG_ERR_MEM; break; }
        for (int64_t k = 0; k < keep; k++) {
            int64_t p = pool[k].p;
            int op = pool[k].j == n2 ? DEL : pool[k].j;
            nped[k] = pool[k].ped;
            memcpy(nmap + k * n1, map + p * n1, sizeof(int32_t) * (size_t)n1);
            nmap[k * n1 + i] = op;
            if (n2 > 0) memcpy(nused + k * n2, used + p * n2, (size_t)n2);
            if (op != DEL) nused[k * n2 + op] = 1;
        }
        free(pool);
        free(ped); free(map); free(used);
        ped = nped; map = nmap; used = nused;
        N = keep;
    }

    if (rc == OG_OK) {
        /* Insertions at the end and best_path <- best node (C10). */
        int64_t best = -1, best_total = 0;
        for (int64_t k = 0; k < N; k++) {
            int64_t total = ped[k] + completion_cost(g2, c, used + k * (n2 > 0 ? n2 : 0));
            if (best < 0 || total < best_total) { best = k; best_total = total; }
        }
        for (int q = 0; q < n1; q++) mapping_out[q] = map[best * n1 + q];
        *cost_out = best_total;
        if (children_out) *children_out = children;
        if (parents_out) *parents_out = parents;
        /* Self-check: the witness re-verifies with the order-free formula. */
        if (mapping_cost(g1, g2, c, has1, has2, lab2, mapping_out) != best_total) rc = OG_ERR_SELFCHECK;
    }
    free(ped); free(map); free(used);
    free(has1); free(has2); free(lab1); free(lab2);
    return rc;
}

int og_kbest(const og_graph *g1, const og_graph *g2, const og_costs *c, int64_t K,
             int64_t *cost_out, int32_t *mapping_out, int64_t *children_out,
             int64_t *parents_out, og_level *levels_out) {
    return og_kbest_ex(g1, g2, c, K, cost_out, mapping_out, children_out, parents_out, levels_out, 0);
}

/* Independent pairs in parallel (no change to any pair's arithmetic). */
int og_kbest_batch_ex(int32_t npairs, const og_graph *g1s, const og_graph *g2s, const og_costs *c,
                      int64_t K, int64_t *costs_out, int32_t *mappings_out, const int64_t *map_offsets,
                      int64_t *children_out, int32_t nthreads, int32_t *status_out, int32_t flags) {
    if (npairs < 0 || (npairs > 0 && (!g1s || !g2s || !costs_out || !map_offsets || !status_out)))
        return OG_ERR_ARG;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    int rc = OG_OK;
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t k = 0; k < npairs; k++) {
        int64_t ch = 0;
        status_out[k] = og_kbest_ex(&g1s[k], &g2s[k], c, K, &costs_out[k],
                                    mappings_out ? mappings_out + map_offsets[k] : NULL, &ch, NULL, NULL, flags);
        if (children_out) children_out[k] = ch;
    }
    for (int32_t k = 0; k < npairs; k++)
        if (status_out[k] != OG_OK) { rc = status_out[k]; break; }
    return rc;
}

int og_kbest_batch(int32_t npairs, const og_graph *g1s, const og_graph *g2s, const og_costs *c,
                   int64_t K, int64_t *costs_out, int32_t *mappings_out, const int64_t *map_offsets,
                   int64_t *children_out, int32_t nthreads, int32_t *status_out) {
    return og_kbest_batch_ex(npairs, g1s, g2s, c, K, costs_out, mappings_out, map_offsets, children_out, nthreads,
                             status_out, 0);
}

int og_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------------------------------
 * Exact GED by depth-first branch and bound: the same
 * vertex-branching tree as og_kbest (v_0..v_{n1-1}; children = substitutions by ascending g2 index,
 * then the deletion), the same incremental PED (Alg. 2 P:247 with the implied edges of P:103-116) and
 * the same completion at the leaves.  A subtree is pruned when PED + lower_bound >= the
 * incumbent, with the admissible bound of S:275:
 *   max(0, |R1| - |R2|) vdel + max(0, |R2| - |R1|) vins + max(0, e1 - e2) edel + max(0, e2 - e1) eins,
 * R1 / R2 = unresolved g1 / unused g2 vertices, e1 / e2 = edges with both endpoints in R1 / R2.
 * The incumbent starts from og_kbest at K = K0 (a pruning aid only; the optimum does not depend on it).
 * node_limit bounds the expansions: beyond it the incumbent is returned with *optimal_out = 0.
 * ------------------------------------------------------------------------------------------------ */
typedef struct {
    const og_graph *g1, *g2;
    const og_costs *c;
    const char *has1, *has2;
    const int32_t *lab1, *lab2;
    int64_t *rem1;       /* rem1[i] = g1 edges with both endpoints >= i */
    int32_t *map;        /* current path: map[q], q < depth */
    char *used;          /* used g2 vertices */
    int64_t best;        /* incumbent cost */
    int32_t *best_map;
    int64_t nodes, limit;
    int over;
} bnb_state;

static int64_t bnb_lower_bound(const bnb_state *S, int i, int nused, int64_t rem2) {
    const og_costs *c = S->c;
    const int64_t r1 = S->g1->n - i, r2 = S->g2->n - nused, e1 = S->rem1[i];
    return (r1 > r2 ? (r1 - r2) * c->vdel : (r2 - r1) * c->vins) +
           (e1 > rem2 ? (e1 - rem2) * c->edel : (rem2 - e1) * c->eins);
}

/* depth i: v_i is branched; ped = PED of the node; nused / e2u / rem2 = used g2 vertices, g2 edges with
 * both endpoints used, g2 edges with both endpoints unused */
static void bnb_dfs(bnb_state *S, int i, int64_t ped, int nused, int64_t e2u, int64_t rem2) {
    const og_graph *g1 = S->g1, *g2 = S->g2;
    const int n1 = g1->n, n2 = g2->n;
    if (S->over) return;
    if (i == n1) { /* leaf: insertion completion */
        const int64_t total = ped + (int64_t)S->c->vins * (n2 - nused) + (int64_t)S->c->eins * (g2->m - e2u);
        if (total < S->best) {
            S->best = total;
            memcpy(S->best_map, S->map, sizeof(int32_t) * (size_t)n1);
        }
        return;
    }
    if (++S->nodes > S->limit) { S->over = 1; return; }
    for (int j = 0; j <= n2; j++) { /* substitutions ascending, then the deletion */
        const int op = (j == n2) ? DEL : j;
        if (op != DEL && S->used[op]) continue;
        int64_t e = ped + vertex_cost(g1, g2, S->c, i, op);
        for (int q = 0; q < i; q++)
            e += edge_charge(S->has1, S->lab1, n1, S->has2, S->lab2, n2, S->c, i, op, q, S->map[q]);
        int cu = 0, cf = 0; /* used / unused g2 neighbours of op */
        if (op != DEL)
            for (int u = 0; u < n2; u++)
                if (u != op && S->has2[op * n2 + u]) { if (S->used[u]) cu++; else cf++; }
        const int nu = nused + (op != DEL), ne2u = (int)e2u + cu;
        const int64_t nrem2 = rem2 - cf;
        if (e + bnb_lower_bound(S, i + 1, nu, nrem2) >= S->best) continue; /* prune */
        S->map[i] = op;
        if (op != DEL) S->used[op] = 1;
        bnb_dfs(S, i + 1, e, nu, ne2u, nrem2);
        if (op != DEL) S->used[op] = 0;
        if (S->over) return;
    }
}

int og_exact(const og_graph *g1, const og_graph *g2, const og_costs *c, int64_t K0, int64_t node_limit,
             int64_t *cost_out, int32_t *mapping_out, int64_t *nodes_out, int32_t *optimal_out) {
    int rc;
    if (!c || !cost_out || node_limit < 1 || K0 < 1) return OG_ERR_ARG;
    if ((rc = validate_graph(g1)) != OG_OK) return rc;
    if ((rc = validate_graph(g2)) != OG_OK) return rc;
    if (g1->n > 0 && !mapping_out) return OG_ERR_ARG;
    const int n1 = g1->n, n2 = g2->n;
    bnb_state S;
    memset(&S, 0, sizeof S);
    S.g1 = g1; S.g2 = g2; S.c = c; S.limit = node_limit;
    const size_t a1 = (size_t)(n1 > 0 ? n1 * n1 : 1), a2 = (size_t)(n2 > 0 ? n2 * n2 : 1);
    char *has1 = (char *)malloc(a1), *has2 = (char *)malloc(a2);
    int32_t *lab1 = (int32_t *)malloc(a1 * sizeof(int32_t)), *lab2 = (int32_t *)malloc(a2 * sizeof(int32_t));
    S.rem1 = (int64_t *)calloc((size_t)n1 + 1, sizeof(int64_t));
    S.map = (int32_t *)calloc((size_t)(n1 > 0 ? n1 : 1), sizeof(int32_t));
    S.best_map = (int32_t *)calloc((size_t)(n1 > 0 ? n1 : 1), sizeof(int32_t));
    S.used = (char *)calloc((size_t)(n2 > 0 ? n2 : 1), 1);
    rc = OG_OK;
    if (!has1 || !has2 || !lab1 || !lab2 || !S.rem1 || !S.map || !S.best_map || !S.used) rc = OG_ERR_MEM;
    else if (dense_adjacency(g1, has1, lab1) != OG_OK || dense_adjacency(g2, has2, lab2) != OG_OK) rc = OG_ERR_INPUT;
    if (rc == OG_OK) {
        S.has1 = has1; S.has2 = has2; S.lab1 = lab1; S.lab2 = lab2;
        for (int e = 0; e < g1->m; e++) { /* rem1[i] = edges with both endpoints >= i */
            int lo = g1->edges[2 * e] < g1->edges[2 * e + 1] ? g1->edges[2 * e] : g1->edges[2 * e + 1];
            for (int i = 0; i <= lo; i++) S.rem1[i]++;
        }
        /* incumbent: the K-Best result at K0 (S: "incumbent initialized by the K=1 greedy result") */
        int64_t kc = 0;
        rc = og_kbest(g1, g2, c, K0, &kc, S.best_map, NULL, NULL, NULL);
        if (rc == OG_OK) {
            if (n1 > 0) memcpy(mapping_out, S.best_map, sizeof(int32_t) * (size_t)n1);
            /* best = kc + 1 so that the strict prune (PED + LB >= best) keeps every path of cost <= kc:
             * the K-Best path itself is never pruned (its prefixes satisfy PED + LB <= kc) */
            S.best = kc + 1;
            bnb_dfs(&S, 0, 0, 0, 0, g2->m);
            if (S.best <= kc) { /* a leaf of cost <= kc was reached */
                *cost_out = S.best;
                if (n1 > 0) memcpy(mapping_out, S.best_map, sizeof(int32_t) * (size_t)n1);
            } else
                *cost_out = kc; /* (only when the budget ran out before any leaf) */
            if (nodes_out) *nodes_out = S.nodes;
            if (optimal_out) *optimal_out = !S.over;
            if (mapping_cost(g1, g2, c, has1, has2, lab2, mapping_out) != *cost_out) rc = OG_ERR_SELFCHECK;
        }
    }
    free(has1); free(has2); free(lab1); free(lab2); free(S.rem1); free(S.map); free(S.best_map); free(S.used);
    return rc;
}

/* Pairs in parallel (independent searches). */
int og_exact_batch(int32_t npairs, const og_graph *g1s, const og_graph *g2s, const og_costs *c, int64_t K0,
                   int64_t node_limit, int64_t *costs_out, int32_t *mappings_out, const int64_t *map_offsets,
                   int64_t *nodes_out, int32_t *optimal_out, int32_t nthreads, int32_t *status_out) {
    if (npairs < 0 || (npairs > 0 && (!g1s || !g2s || !costs_out || !map_offsets || !status_out || !optimal_out)))
        return OG_ERR_ARG;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t k = 0; k < npairs; k++)
        status_out[k] = og_exact(&g1s[k], &g2s[k], c, K0, node_limit, &costs_out[k],
                                 mappings_out ? mappings_out + map_offsets[k] : NULL, nodes_out ? &nodes_out[k] : NULL,
                                 &optimal_out[k]);
    for (int32_t k = 0; k < npairs; k++)
        if (status_out[k] != OG_OK) return status_out[k];
    return OG_OK;
}

/* Exposed for the selection pin: indices of the k smallest keys
 * (ped[x], p[x], j[x]) as chosen by select_k, ascending by index. */
int og_select(const int64_t *ped, const int64_t *p, const int32_t *j, int64_t n, int64_t k, int64_t *idx_out) {
    if (n < 0 || k < 0 || (n > 0 && (!ped || !p || !j || !idx_out))) return OG_ERR_ARG;
    cand *a = (cand *)malloc(sizeof(cand) * (size_t)(n > 0 ? n : 1));
    char *take = (char *)calloc((size_t)(n > 0 ? n : 1), 1);
    if (!a || !take) { free(a); free(take); return OG_ERR_MEM; }
    for (int64_t x = 0; x < n; x++) { a[x].ped = ped[x]; a[x].key = ped[x]; a[x].p = p[x]; a[x].j = j[x]; }
    int64_t keep = k < n ? k : n;
    select_k(a, n, keep);
    /* map each selected key back to its input index (keys are unique) */
    for (int64_t s = 0; s < keep; s++)
        for (int64_t x = 0; x < n; x++)
            if (!take[x] && a[s].ped == ped[x] && a[s].p == p[x] && a[s].j == j[x]) { take[x] = 1; break; }
    int64_t c = 0;
    for (int64_t x = 0; x < n; x++)
        if (take[x]) idx_out[c++] = x;
    free(a); free(take);
    return c == keep ? OG_OK : OG_ERR_ARG;
}

/* Exposed for the witness tests: order-free cost of a given complete mapping. */
int og_mapping_cost(const og_graph *g1, const og_graph *g2, const og_costs *c, const int32_t *f,
                    int64_t *cost_out) {
    int rc;
    if ((rc = validate_graph(g1)) != OG_OK) return rc;
    if ((rc = validate_graph(g2)) != OG_OK) return rc;
    size_t a1 = (size_t)(g1->n > 0 ? g1->n * g1->n : 1), a2 = (size_t)(g2->n > 0 ? g2->n * g2->n : 1);
    char *has1 = (char *)malloc(a1), *has2 = (char *)malloc(a2);
    int32_t *lab1 = (int32_t *)malloc(a1 * sizeof(int32_t)), *lab2 = (int32_t *)malloc(a2 * sizeof(int32_t));
    if (dense_adjacency(g1, has1, lab1) != OG_OK || dense_adjacency(g2, has2, lab2) != OG_OK) rc = OG_ERR_INPUT;
    else *cost_out = mapping_cost(g1, g2, c, has1, has2, lab2, f);
    free(has1); free(has2); free(lab1); free(lab2);
    return rc;
}
