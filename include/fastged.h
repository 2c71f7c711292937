/*
 * fastged.h -- C ABI of the B200 FAST-GED K-Best hot path (arXiv 2605.00830).
 *
 * The library (paper_2605_00830_b200/libfastged.so) runs the level-synchronous
 * K-Best search over the vertex-branching edit-path tree entirely in sm_100a
 * CUDA kernels:
 *   Branch  -- expand every kept node by mapping the level's g1 vertex to each
 *              unused g2 vertex or deleting it, PED computed incrementally
 *              (Alg. 2, implied edges PAPER.md:103-116);
 *   Rank    -- keep exactly min(K, #children) children, the smallest under the
 *              key (PED, parent position, child index), without a sort
 *              (SURVEY.md §8(c) C12);
 *   Update  -- write the next frontier on the device in canonical order
 *              (C13);
 *   Finalize-- add the insertion completion at the last level and return the
 *              best node's cost and mapping (C10).
 * There is no CPU fallback: without a usable CUDA device every solve call
 * returns FASTGED_ERR_CUDA.
 *
 * Conventions shared by every entry point
 *   - All integers are little-endian host integers.  Vertex ids are 0-based.
 *   - Labels are caller-interned int32 ids; equality of ids is label equality
 *     (reading C3).
 *   - g1 is the source, g2 the target; graphs are never swapped (C18).
 *   - The g1 vertices are branched in index order v_0 .. v_{n1-1} (C4).
 *   - Every input array is caller-owned and only read during the call.
 *   - Every output array is caller-allocated; sizes follow from the inputs.
 *   - Calls are synchronous unless stated: results are in the output arrays on return.
 *   - No C++ exception crosses the ABI.  On error the outputs are unspecified and
 *     fastged_last_error(h) describes the failure (naming the pair index in a batch).
 *   - A handle is not thread-safe; separate handles are independent.
 */
#ifndef FASTGED_H
#define FASTGED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes. */
#define FASTGED_OK 0
#define FASTGED_ERR_ARG 1      /* NULL pointer, k < 1, negative cost, npairs < 0, bad device/rank   */
#define FASTGED_ERR_INPUT 2    /* self-loop, duplicate edge, endpoint out of range, n < 0, m < 0     */
#define FASTGED_ERR_CAPACITY 3 /* buffers exceed device memory, or a size limit below; K is never shrunk */
#define FASTGED_ERR_OVERFLOW 4 /* worst-case PED n1*max(vsub,vdel)+n2*vins+(m1+m2)*max(esub,edel,eins) >= 2^31 */
#define FASTGED_ERR_CUDA 5     /* CUDA runtime failure (including: no device)                        */
#define FASTGED_ERR_NCCL 6     /* NCCL failure (sharded single-pair mode)                            */

/* fastged_config_t.flags */
#define FASTGED_FLAG_TIMING 1u      /* record CUDA events around every kernel launch (fastged_get_stats) */
#define FASTGED_FLAG_DEBUG_WINDOW 2u /* test only: 2-wide rank window, forces the multi-pass rank path   */
#define FASTGED_FLAG_FORCE_LARGE 4u  /* test only: solve_pair uses the whole-GPU path even for small pairs */
#define FASTGED_FLAG_VIRTUAL_SHARDS 8u /* test only: world_size (<= 8) ranks of one pair as equal CTA groups
                                         of one grid on this handle's GPU, the same in-kernel exchange as
                                         real ranks (rank, nccl_id ignored)                              */
#define FASTGED_FLAG_LAST_BY_TOTAL 16u /* method variant: rank the last level by
                                         PED + insertion completion instead of PED (the alternative to reading
                                         C10 of Alg. 1); never a higher cost than the
                                         paper-literal rule.  Every path (batched, whole-GPU, sharded); not
                                         combined with FASTGED_FLAG_APPROX (FASTGED_ERR_ARG). */
/* method variant ("approximate top-k selection may become an option"
 * for extreme K): each level keeps the min(K, c_i) smallest children under the coarse key
 * (floor((PED - lo_i) / 2^shift), parent, child), lo_i = the smallest PED of the level's parents --
 * children in one PED bin are ranked by position only.  shift = 1..15 (0 = the exact selection).  Runs on
 * the whole-GPU kernel (every pair of a batch is routed there); levels_out[3i+2] then reports the K-th
 * smallest key's bin. */
#define FASTGED_FLAG_APPROX(shift) ((uint32_t)((shift) & 15) << 8)
#define FASTGED_FLAG_APPROX_MASK (15u << 8)

/* Limits of this build (exceeding one returns FASTGED_ERR_CAPACITY, never a silent change). */
#define FASTGED_MAX_N 65534        /* vertices of a source graph g1                               */
#define FASTGED_MAX_N2 1024        /* vertices of a target graph g2                               */
#define FASTGED_MAX_EDGE_LABELS 253 /* distinct edge labels in one target graph g2 (batched path)   */

typedef struct fastged_handle fastged_handle_t; /* opaque: device, stream, arena, NCCL comm */
typedef struct fastged_batch fastged_batch_t;   /* opaque: a validated batch resident in HBM */

/* A simple undirected labelled graph G = (V, E, alpha, beta).
 *   n        : |V| >= 0
 *   m        : |E| >= 0
 *   vlabels  : [n]  vertex label ids (may be NULL when n == 0)
 *   edges    : [2m] endpoint pairs (u, v), 0 <= u, v < n, u != v, each unordered pair at most once
 *   elabels  : [m]  edge label ids, or NULL = every edge has label 0                         */
typedef struct {
    int32_t n, m;
    const int32_t *vlabels;
    const int32_t *edges;
    const int32_t *elabels;
} fastged_graph_t;

/* Cost model (reading C1): six integer constants >= 0; substituting equal
 * labels costs 0.  Presets: Setting 1 = {2,4,4,1,2,2}, Setting 2 = {4,12,12,1,10,10}
 * (PAPER.md:579).                                                                            */
typedef struct {
    int32_t vsub, vdel, vins, esub, edel, eins;
} fastged_costs_t;

/* Handle configuration.
 *   device     : CUDA ordinal
 *   stream     : cudaStream_t to launch on, or NULL = the handle creates and owns one.  Batched
 *                runs fork onto up to three side streams the handle owns (one per word-width group,
 *                running concurrently) and join back onto this stream before a call returns or a
 *                fastged_batch_run's work is complete on it: callers only ever order against `stream`.
 *   world_size : 1 = single GPU.  > 1 = sharded single-pair mode (every rank calls
 *                fastged_solve_pair collectively with identical inputs)
 *   rank       : 0 <= rank < world_size
 *   nccl_id    : 128-byte ncclUniqueId (broadcast by the caller) when world_size > 1, else NULL
 *   flags      : FASTGED_FLAG_*                                                           */
typedef struct {
    int32_t device;
    void *stream;
    int32_t world_size, rank;
    const uint8_t *nccl_id;
    uint32_t flags;
} fastged_config_t;

/* Single-pair result.
 *   cost               : GED upper bound = cost of the returned edit path (exact when K covers every level)
 *   mapping            : caller-allocated [g1.n]; g2 index, or -1 = deleted.  Unmapped g2 vertices are
 *                        inserted (in ascending order; the order does not change the cost, C6)
 *   children_evaluated : sum over levels of the candidates generated (tree nodes whose PED was computed)
 *   parents_expanded   : sum over levels of the frontier size
 *   device_ms          : device time of the search kernels (CUDA events)                  */
typedef struct {
    int64_t cost;
    int32_t *mapping;
    int64_t children_evaluated, parents_expanded;
    float device_ms;
} fastged_result_t;

/* Counters of the last solve/run call on a handle. */
typedef struct {
    int64_t kernel_launches;    /* kernels of this library launched by the last call            */
    float device_ms;            /* device time of the last call's search kernels (CUDA events)   */
    float branch_ms;            /* FASTGED_FLAG_TIMING: time in the dominant (branch/search) kernels */
    int64_t branch_launches;    /* number of launches timed in branch_ms                        */
    int64_t children_evaluated; /* sum over all pairs of the last call                          */
    int64_t parents_expanded;
    int64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved by the last call                 */
    int64_t alg_bytes;            /* algorithmic frontier bytes of the search: sum over pairs and levels of
                                     N_i (4 + b d_i) + N_{i+1} (b i + 4) + N_{i+1} (b (i+1) + 4), b = bytes per
                                     lambda entry                                    */
    int64_t alg_ops;              /* algorithmic integer lane-ops of the branch step: sum over children of
                                     4 W + 8, W = ceil(n2 / 32) words per bit row     */
    float phase_ms[5];            /* whole-GPU (large-pair) kernel only: time in its phases A+T (branch,
                                     rank), B (count), C1 (compact), C2 (update), finalize; 0 otherwise */
    int64_t hist_children;        /* whole-GPU kernel: children whose rank code entered the histogram
                                     (PED <= U_i bound); 0 otherwise           */
} fastged_stats_t;

/* Create a handle.  Returns FASTGED_ERR_CUDA if the device cannot be used, FASTGED_ERR_NCCL if the
 * communicator cannot be created (world_size > 1).  *out is NULL on failure.                    */
int fastged_create(const fastged_config_t *cfg, fastged_handle_t **out);

/* Release the handle, its device memory, its own stream and its communicator.  NULL is a no-op. */
void fastged_destroy(fastged_handle_t *h);

/* Message of the last failure on h (never NULL; "" after success).  h == NULL: the last failure of
 * fastged_create on this thread.  The string is owned by the library and valid until the next call. */
const char *fastged_last_error(const fastged_handle_t *h);

/* K-Best GED of one pair (Alg. 1).  out->mapping must hold g1->n entries (may be
 * NULL when g1->n == 0).  Sharded mode (world_size > 1, at most 8 ranks on one node, one GPU each,
 * peer access over NVLink): a collective call; all ranks pass identical inputs and receive the
 * identical result.  Each level's frontier is split into equal contiguous slices, one per rank; the
 * per-level exchange (histogram, counts, the next level's node descriptors, the final argmin) runs
 * inside the kernel over peer memory (CUDA IPC mappings set up over the NCCL communicator), with an
 * in-kernel barrier across ranks.  A rank that fails, or a peer that misses a barrier for
 * FASTGED_NCCL_TIMEOUT_S seconds (default 600), returns FASTGED_ERR_NCCL and aborts the communicator. */
int fastged_solve_pair(fastged_handle_t *h, const fastged_graph_t *g1, const fastged_graph_t *g2,
                       const fastged_costs_t *c, int64_t k, fastged_result_t *out);

/* As fastged_solve_pair; levels_out (NULL or [3 * g1->n]) receives per level i:
 * levels_out[3i] = frontier size N_i, [3i+1] = candidates c_i, [3i+2] = PED of the last kept
 * candidate when c_i > k, else -1.                                                              */
int fastged_solve_pair_ex(fastged_handle_t *h, const fastged_graph_t *g1, const fastged_graph_t *g2,
                          const fastged_costs_t *c, int64_t k, fastged_result_t *out, int64_t *levels_out);

/* K-Best GED of npairs independent pairs (g1s[p], g2s[p]) with one cost model and one K, on one GPU,
 * host buffers in and out (one H2D and one D2H per call).
 *   costs_out    : [npairs]
 *   mappings_out : [sum_p g1s[p].n], the pairs' mappings concatenated in pair order (NULL allowed
 *                  when every g1s[p].n == 0)
 *   children_out : [npairs] children evaluated per pair, or NULL                              */
int fastged_solve_batch(fastged_handle_t *h, int32_t npairs, const fastged_graph_t *g1s,
                        const fastged_graph_t *g2s, const fastged_costs_t *c, int64_t k,
                        int64_t *costs_out, int32_t *mappings_out, int64_t *children_out);

/* Device-resident split of fastged_solve_batch (the same computation):
 *   fastged_batch_upload   validates and packs the pairs and copies them to HBM (synchronous);
 *   fastged_batch_run      runs the search on the handle's stream; results stay in HBM.  It returns
 *                          after enqueueing (asynchronous; errors of the launch are reported);
 *   fastged_batch_download synchronises and copies results to the caller's arrays;
 *   fastged_batch_free     releases the batch (NULL is a no-op).                               */
int fastged_batch_upload(fastged_handle_t *h, int32_t npairs, const fastged_graph_t *g1s,
                         const fastged_graph_t *g2s, fastged_batch_t **out);
int fastged_batch_run(fastged_handle_t *h, fastged_batch_t *b, const fastged_costs_t *c, int64_t k);
int fastged_batch_download(fastged_handle_t *h, fastged_batch_t *b, int64_t *costs_out,
                           int32_t *mappings_out, int64_t *children_out);
void fastged_batch_free(fastged_handle_t *h, fastged_batch_t *b);

/* Counters of the last solve/run call. */
int fastged_get_stats(const fastged_handle_t *h, fastged_stats_t *out);

/* Writes a new 128-byte ncclUniqueId to out (call on rank 0, broadcast the bytes to every rank, pass
 * them as fastged_config_t.nccl_id).  FASTGED_ERR_NCCL on failure. */
int fastged_nccl_unique_id(uint8_t *out);

/* Library version string, e.g. "fastged-b200 0.1 sm_100a". */
const char *fastged_version(void);

/* ---------------------------------------------------------------------------------------------
 * Edit paths: the step after the search.  Host functions of the library (no
 * device needed); the mapping is any complete vertex mapping, e.g. the one fastged_solve_* returned.
 * ------------------------------------------------------------------------------------------------- */
#define FASTGED_OP_VSUB 1 /* a = g1 vertex, b = its g2 image */
#define FASTGED_OP_VDEL 2 /* a = deleted g1 vertex                                                        */
#define FASTGED_OP_VINS 3 /* b = inserted g2 vertex                                                       */
#define FASTGED_OP_ESUB 4 /* g1 edge (a, c) -> g2 edge (b, d) */
#define FASTGED_OP_EDEL 5 /* g1 edge (a, c) deleted                                                       */
#define FASTGED_OP_EINS 6 /* g2 edge (b, d) inserted                                                      */

typedef struct {
    int32_t kind;       /* FASTGED_OP_*                                   */
    int32_t a, b, c, d; /* vertex ids as above; -1 where not applicable */
    int32_t cost;       /* cost of the operation under the cost model (0 for an equal-label substitution) */
} fastged_edit_op_t;

/* The explicit edit path of a complete vertex mapping (mapping[i] = g2 vertex or -1 = deleted): for
 * v_0..v_{n1-1} its vertex operation followed by the implied operations on the edges to the earlier
 * vertices (second-endpoint rule), then the vertex insertions (ascending) and the insertions of the g2
 * edges with an unused endpoint.  The costs sum to the path cost (*cost_out), which equals
 * the GED a solve returned with that mapping.  ops may be NULL to query the count; max_ops = capacity.
 * Errors: FASTGED_ERR_ARG (NULL, capacity too small: *n_ops_out still holds the count),
 * FASTGED_ERR_INPUT (invalid graph, mapping out of range or not injective). */
int fastged_edit_path(const fastged_graph_t *g1, const fastged_graph_t *g2, const fastged_costs_t *c,
                      const int32_t *mapping, fastged_edit_op_t *ops, int32_t max_ops, int32_t *n_ops_out,
                      int64_t *cost_out);

/* Applies the first prefix_len VERTEX operations of the path (the n1 operations on v_0..v_{n1-1}, then the
 * insertions) with their implied edge effects (the NAS crossover of PAPER.md:714):
 * substituted vertices take the g2 label, deleted vertices vanish with their edges, edges between two
 * resolved (or inserted) vertices take their g2 state, unresolved g1 vertices and the edges among them or
 * to resolved vertices stay as in g1.  prefix_len = 0 gives g1; prefix_len = n1 + #insertions gives a
 * graph equal to g2 under origin_out.  Output vertices: the surviving g1 vertices in index order, then the
 * inserted g2 vertices ascending.  origin_out[v] = g2 vertex of output vertex v, or -1 - (g1 index) for an
 * unresolved g1 vertex.  Capacities: vlabels_out/origin_out [n1 + n2], edges_out [2 (m1 + m2)],
 * elabels_out [m1 + m2].  Errors as fastged_edit_path; prefix_len out of range -> FASTGED_ERR_ARG. */
int fastged_apply_edit_path(const fastged_graph_t *g1, const fastged_graph_t *g2, const int32_t *mapping,
                            int32_t prefix_len, int32_t *n_out, int32_t *vlabels_out, int32_t *origin_out,
                            int32_t *m_out, int32_t *edges_out, int32_t *elabels_out);

/* 1 if a and b are equal under the bijection mapping (a vertex v -> b vertex mapping[v]): same vertex
 * labels and the same edges with the same labels; 0 if not; negative FASTGED_ERR_* (negated) on a mapping
 * that is not a bijection or a NULL argument. */
int fastged_graphs_equal_under_mapping(const fastged_graph_t *a, const fastged_graph_t *b, const int32_t *mapping);

#ifdef __cplusplus
}
#endif
#endif /* FASTGED_H */
