// fastged.cu -- host engine and C ABI of the B200 FAST-GED K-Best hot path (include/fastged.h).
//
// Host work per call: validate the graphs (reading C17), intern edge labels, pack
// every pair into one device blob (g2 bit-packed adjacency rows, the P_i lists of earlier g1
// neighbours, labels), copy it to HBM once ("transferred once"), launch the search
// kernels, copy results back once.  Nothing of the search runs on the host.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h> // header-only NVTX v3: named host ranges for Nsight timelines

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "../../include/fastged.h"
#include "batch_kernel.cuh"
#include "large_kernel.cuh"

namespace {

thread_local std::string g_create_error;

// Device allocation owned by its holder (freed on destruction, so an error thrown mid-call
// cannot leak it); not copyable.
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), cap(o.cap) { o.p = nullptr; o.cap = 0; }
    ~DevBuf() { release(); }
    cudaError_t reserve(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max(n, (size_t)4096);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct HostPinned {
    void *p = nullptr;
    size_t cap = 0;
    HostPinned() = default;
    HostPinned(const HostPinned &) = delete;
    HostPinned &operator=(const HostPinned &) = delete;
    ~HostPinned() { release(); }
    cudaError_t reserve(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max(n, (size_t)4096);
        cudaError_t e = cudaMallocHost(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

struct FgError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw FgError{code, buf};
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            fail(e_ == cudaErrorMemoryAllocation ? FASTGED_ERR_CAPACITY : FASTGED_ERR_CUDA,        \
                 "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);       \
    } while (0)

inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// NVTX range for the lifetime of a scope (pack / plan+launch / large pair / download / sharded level)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
inline int words_for(int n2) { return std::max(1, (n2 + 31) / 32); }

// ---------------------------------------------------------------- packed pair (host side)
struct PackedPair {
    fg::PairDesc d;
    int W;
    size_t bytes; // blob bytes of this pair
};

struct GroupLaunch { fg::BatchArgs a; void *kern; int grid, nt; size_t smem, per_cta; int64_t cost; };

struct GroupKey {
    int W;
    bool lab;
    bool operator<(const GroupKey &o) const { return W != o.W ? W < o.W : lab < o.lab; }
};

} // namespace

// ---------------------------------------------------------------- handle / batch
struct fastged_batch {
    int32_t npairs = 0;
    std::vector<fg::PairDesc> descs;      // host copy (offsets)
    std::vector<int> W;                   // per pair
    std::vector<int64_t> map_off;         // per pair mapping offset
    int64_t total_map = 0;
    int n1max = 0, n2max = 0;
    DevBuf blob, ddesc, dorder, dcost, dmap, dchild, dpar, dalg, dwork;
    HostPinned stage; // this batch's pinned staging (inputs, order, results): batches can be in flight together
    cudaEvent_t ev_h2d = nullptr; // the inputs' H2D copies (on the handle's copy stream) are complete
    size_t ord_at = 0, res_at = 0; // byte offsets of the order and result areas in `stage`
    int32_t pair_base = 0;         // index of pair 0 in the caller's arrays (error messages)
    std::map<GroupKey, std::vector<int32_t>> groups; // pair indices per kernel variant
    std::vector<int32_t> large;                      // pairs beyond the batched limits
    bool ran = false;
    // cached launch plan (run_batch): valid for (plan_k, plan_c, plan_flags) and the scratch at plan_scratch
    bool plan_valid = false;
    int64_t plan_k = 0;
    fastged_costs_t plan_c{};
    uint32_t plan_flags = 0;
    void *plan_scratch = nullptr;
    std::vector<GroupLaunch> plans;
    std::vector<int32_t> order_all;
};

struct fastged_handle {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sms = 148;
    size_t smem_optin = 227 * 1024;
    uint32_t flags = 0;
    int world = 1, rank = 0;
    std::string err;
    DevBuf scratch, levels;
    HostPinned stage;
    fastged_stats_t stats{};
    std::vector<cudaEvent_t> evpool;
    int evused = 0;
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
    DevBuf lblob, lbuf; // large single-pair mode
    fastged_batch *tmp = nullptr;        // reused by solve_batch (first chunk) / solve_pair
    std::vector<fastged_batch *> tmpv;  // reused by solve_batch (later pipelined chunks)
    ncclComm_t comm = nullptr;    // sharded single-pair mode (world_size > 1): bootstrap and barriers
    DevBuf xbuf;                  // NCCL staging (IPC handles, barrier word)
    std::vector<std::vector<uint8_t>> peer_handle; // [world] CUDA IPC handle of each peer's lbuf
    std::vector<void *> peer_base;                 // [world] its mapping here (NULL: not mapped)
    // batched launches of the word-width groups run concurrently (fork/join on side streams), so the
    // tail of one group's persistent launch overlaps the next group's start
    std::vector<cudaStream_t> gstreams;
    cudaStream_t cstream = nullptr; // batch inputs' H2D copies: a chunk's upload overlaps the previous chunk's search
    std::vector<cudaEvent_t> gevents; // [0] fork, [1..] joins
};

namespace {

int set_err(fastged_handle_t *h, const FgError &e) {
    if (h) h->err = e.msg;
    return e.code;
}

// ---------------------------------------------------------------- validation
void validate_graph(const fastged_graph_t *g, int pair, const char *which) {
    if (!g) fail(FASTGED_ERR_ARG, "pair %d: %s is NULL", pair, which);
    if (g->n < 0 || g->m < 0) fail(FASTGED_ERR_INPUT, "pair %d: %s has n=%d m=%d", pair, which, g->n, g->m);
    if (g->n > FASTGED_MAX_N) fail(FASTGED_ERR_CAPACITY, "pair %d: %s has n=%d > %d", pair, which, g->n, FASTGED_MAX_N);
    if (g->n > 0 && !g->vlabels) fail(FASTGED_ERR_ARG, "pair %d: %s vlabels is NULL", pair, which);
    if (g->m > 0 && !g->edges) fail(FASTGED_ERR_ARG, "pair %d: %s edges is NULL", pair, which);
    if ((int64_t)g->m > (int64_t)g->n * (g->n - 1) / 2)
        fail(FASTGED_ERR_INPUT, "pair %d: %s has more edges than a simple graph allows", pair, which);
    for (int e = 0; e < g->m; ++e) {
        int a = g->edges[2 * e], b = g->edges[2 * e + 1];
        if (a < 0 || b < 0 || a >= g->n || b >= g->n)
            fail(FASTGED_ERR_INPUT, "pair %d: %s edge %d endpoint out of range", pair, which, e);
        if (a == b) fail(FASTGED_ERR_INPUT, "pair %d: %s edge %d is a self-loop", pair, which, e);
    }
    if (g->n <= 4096) { // duplicate edges: a per-thread adjacency bitmap, O(m) (host packing is on the e2e path)
        thread_local std::vector<uint64_t> bits;
        const size_t nw = ((size_t)g->n * g->n + 63) / 64;
        if (bits.size() < nw) bits.assign(nw, 0);
        bool dup = false;
        int e = 0;
        for (; e < g->m; ++e) {
            const int a = std::min(g->edges[2 * e], g->edges[2 * e + 1]), b = std::max(g->edges[2 * e], g->edges[2 * e + 1]);
            const size_t x = (size_t)a * g->n + b;
            if ((bits[x >> 6] >> (x & 63)) & 1u) { dup = true; break; }
            bits[x >> 6] |= 1ull << (x & 63);
        }
        for (int f = 0; f < e + (dup ? 1 : 0) && f < g->m; ++f) { // clear exactly the bits set above
            const int a = std::min(g->edges[2 * f], g->edges[2 * f + 1]), b = std::max(g->edges[2 * f], g->edges[2 * f + 1]);
            const size_t x = (size_t)a * g->n + b;
            bits[x >> 6] &= ~(1ull << (x & 63));
        }
        if (dup) fail(FASTGED_ERR_INPUT, "pair %d: %s has a duplicate edge", pair, which);
        return;
    }
    std::vector<uint64_t> keys((size_t)g->m);
    for (int e = 0; e < g->m; ++e) {
        const int a = g->edges[2 * e], b = g->edges[2 * e + 1];
        keys[e] = ((uint64_t)std::min(a, b) << 32) | (uint32_t)std::max(a, b);
    }
    std::sort(keys.begin(), keys.end());
    for (size_t e = 1; e < keys.size(); ++e)
        if (keys[e] == keys[e - 1]) fail(FASTGED_ERR_INPUT, "pair %d: %s has a duplicate edge", pair, which);
}

void validate_costs(const fastged_costs_t *c) {
    if (!c) fail(FASTGED_ERR_ARG, "costs is NULL");
    if (c->vsub < 0 || c->vdel < 0 || c->vins < 0 || c->esub < 0 || c->edel < 0 || c->eins < 0)
        fail(FASTGED_ERR_ARG, "negative cost");
}

void check_overflow(const fastged_graph_t *g1, const fastged_graph_t *g2, const fastged_costs_t *c, int pair) {
    int64_t bound = (int64_t)g1->n * std::max(c->vsub, c->vdel) + (int64_t)g2->n * c->vins +
                    ((int64_t)g1->m + g2->m) * std::max(c->esub, std::max(c->edel, c->eins)) + 512;
    if (bound >= ((int64_t)1 << 31))
        fail(FASTGED_ERR_OVERFLOW, "pair %d: worst-case PED %lld does not fit int32", pair, (long long)bound);
}

// Largest frontier any level can hold: N_{i+1} <= min(K, N_i (n2 + 1)), N_0 = 1.  When K exceeds
// the returned cap, no level has more than cap candidates, so K and the cap select identically.
int64_t frontier_cap(int n1, int n2, int64_t k) {
    int64_t N = 1, mx = 1;
    for (int i = 0; i < n1 && N < k; ++i) {
        N = std::min<int64_t>(k, N * (int64_t)(n2 + 1));
        mx = std::max(mx, N);
    }
    return std::min(mx, k);
}

// Per-CTA bytes of the batched kernel's per-level work arrays (the layout run_batch plans), in 64 bits.
size_t batched_work_bytes(int64_t Kc, int W, int csmax) {
    auto a16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
    return a16(4 * (size_t)Kc * W) + a16(4 * (size_t)(Kc + 1)) + a16((size_t)Kc * csmax) + a16(4 * (size_t)Kc) +
           a16(2 * ((size_t)Kc * csmax / 16 + 2));
}

// Batched-path limits: n2 <= 128 (lane-owned rows, W <= 4), n1 <= 1024, at most fg::LMAX distinct g2
// edge labels (label planes), and every 32-bit offset of the plan fits: the codes of one level
// (Kc * csmax bytes, indexed with int32 in the kernel), the work arrays and the frontier rows stay
// below 2^31 with room to spare.  csmax is taken at the top of the pair's word-width bucket (the
// group's plan uses the bucket maximum).  Pairs beyond the limits are solved by the whole-GPU kernel
// (solve_large), inside a batch as well.
bool fits_batched(int n1, int n2, int64_t k, int nlab) {
    if (n2 > 128 || n1 > 1024 || nlab > fg::LMAX) return false;
    const int W = words_for(n2);
    const int64_t Kc = (frontier_cap(n1, n2, k) + 3) & ~3ll;
    const int csmax = (32 * W + 1 + 3) & ~3;
    const int64_t lim = ((int64_t)1 << 31) - ((int64_t)1 << 24);
    const int64_t n1s = std::max(4, (n1 + 3) & ~3);
    return Kc * csmax < lim && (int64_t)batched_work_bytes(Kc, W, csmax) < lim && Kc * n1s < lim;
}

// Work routing: the batched kernel gives a pair one CTA, the whole-GPU kernel the whole GPU for one pair at a
// time.  A pair with wide levels (frontier cap x (n2 + 1) candidates) gains up to ~32x from the whole GPU
// (scripts/paper_points.py: one 20-vertex pair at K = 7e5 takes 399 ms on one CTA and 12.6 ms on the whole
// GPU; n = 50 at K = 5000: 9.1 vs 1.9 ms), but a batch of such pairs keeps every SM busy on the batched
// kernel.  Estimated gain g = min(32, candidates / 2^16); the whole GPU is chosen while npairs <= g / 2 (a
// single pair: above 131,072 candidates per level; at K = 1000 and n = 20 the one CTA wins, 0.35 vs 0.61 ms).
bool prefers_whole_gpu(int n1, int n2, int64_t k, int64_t npairs) {
    const int64_t cand = frontier_cap(n1, n2, k) * (int64_t)(n2 + 1);
    return 2 * npairs * ((int64_t)1 << 16) <= std::min<int64_t>(32ll << 16, cand);
}

// Number of distinct g2 edge labels (the label planes of a labelled pair).
int g2_label_count(const fastged_graph_t *g2) {
    std::vector<int32_t> l(g2->elabels ? g2->elabels : nullptr, g2->elabels ? g2->elabels + g2->m : nullptr);
    if (!g2->elabels) return g2->m > 0 ? 1 : 0;
    std::sort(l.begin(), l.end());
    return (int)(std::unique(l.begin(), l.end()) - l.begin());
}

// ---------------------------------------------------------------- packing
// Sizes a pair's blob segment.
size_t pair_blob_bytes(const fastged_graph_t *g1, const fastged_graph_t *g2, bool lab, int n2p) {
    int W = words_for(g2->n);
    size_t b = 0;
    b += align16(4 * (size_t)g1->n);       // vl1
    b += align16(4 * (size_t)g2->n);       // vl2
    b += align16(4 * (size_t)(g1->n + 1)); // pptr
    b += align16(4 * (size_t)g1->m) * 2;   // pq, pl
    b += align16(4 * (size_t)g2->n * W);   // adj2
    if (lab) b += align16((size_t)n2p * n2p);
    return b;
}

// Edge-label interning: returns true if edge labels can change a cost (more than one distinct label
// among the edges of both graphs).
bool labelled_pair(const fastged_graph_t *g1, const fastged_graph_t *g2) {
    bool have = false;
    int32_t first = 0;
    for (const fastged_graph_t *g : {g1, g2})
        for (int e = 0; e < g->m; ++e) {
            int32_t l = g->elabels ? g->elabels[e] : 0;
            if (!have) { have = true; first = l; }
            else if (l != first) return true;
        }
    return false;
}

void pack_pair(const fastged_graph_t *g1, const fastged_graph_t *g2, bool lab, int n2p, uint8_t *blob,
               int64_t off, fg::PairDesc &d, int pair) {
    const int n1 = g1->n, n2 = g2->n, W = words_for(n2);
    int64_t cur = off;
    auto seg = [&](size_t bytes, int64_t &field) {
        field = cur;
        uint8_t *q = blob + cur;
        cur += (int64_t)align16(bytes);
        return q;
    };
    d.n1 = n1; d.n2 = n2; d.m1 = g1->m; d.m2 = g2->m; d.labelled = lab ? 1 : 0; d.n2p = n2p;
    d.nlab = 0; d.pad0 = 0;
    int32_t *vl1 = (int32_t *)seg(4 * (size_t)n1, d.vl1);
    int32_t *vl2 = (int32_t *)seg(4 * (size_t)n2, d.vl2);
    int32_t *pptr = (int32_t *)seg(4 * (size_t)(n1 + 1), d.pptr);
    int32_t *pq = (int32_t *)seg(4 * (size_t)g1->m, d.pq);
    int32_t *pl = (int32_t *)seg(4 * (size_t)g1->m, d.pl);
    uint32_t *adj2 = (uint32_t *)seg(4 * (size_t)n2 * W, d.adj2);
    uint8_t *e2 = nullptr;
    if (lab) e2 = seg((size_t)n2p * n2p, d.e2lab);
    else d.e2lab = 0;
    if (n1) memcpy(vl1, g1->vlabels, 4 * (size_t)n1);
    if (n2) memcpy(vl2, g2->vlabels, 4 * (size_t)n2);
    // g2 label ids: 1..L (0 = no edge); g1 labels absent from g2 -> 255 (never equal).  A small linear table
    // (molecules have a handful of bond labels); per-thread scratch, no allocation per pair.
    thread_local std::vector<std::pair<int32_t, int>> ids;
    ids.clear();
    auto label_id = [&](int32_t l) -> int {
        for (const auto &x : ids)
            if (x.first == l) return x.second;
        return -1;
    };
    if (lab) {
        for (int e = 0; e < g2->m; ++e) {
            int32_t l = g2->elabels ? g2->elabels[e] : 0;
            if (label_id(l) < 0) {
                int id = (int)ids.size() + 1;
                if (id > FASTGED_MAX_EDGE_LABELS)
                    fail(FASTGED_ERR_CAPACITY, "pair %d: g2 has more than %d distinct edge labels", pair,
                         FASTGED_MAX_EDGE_LABELS);
                ids.push_back({l, id});
            }
        }
        memset(e2, 0, (size_t)n2p * n2p);
        d.nlab = (int)ids.size();
    }
    // P_i = {q < i : (v_q, v_i) in E1}, each g1 edge listed at its later endpoint (second-endpoint rule, C7)
    thread_local std::vector<int> cnt, fillp;
    cnt.assign((size_t)n1 + 1, 0);
    for (int e = 0; e < g1->m; ++e) cnt[std::max(g1->edges[2 * e], g1->edges[2 * e + 1])]++;
    pptr[0] = 0;
    for (int i = 0; i < n1; ++i) pptr[i + 1] = pptr[i] + cnt[i];
    fillp.assign(pptr, pptr + n1 + 1);
    for (int e = 0; e < g1->m; ++e) {
        int a = g1->edges[2 * e], b = g1->edges[2 * e + 1];
        int q = std::min(a, b), i = std::max(a, b);
        int at = fillp[i]++;
        pq[at] = q;
        int32_t l = g1->elabels ? g1->elabels[e] : 0;
        if (lab) {
            const int id = label_id(l);
            pl[at] = id < 0 ? 255 : id;
        } else pl[at] = 0;
    }
    memset(adj2, 0, 4 * (size_t)n2 * W);
    for (int e = 0; e < g2->m; ++e) {
        int x = g2->edges[2 * e], y = g2->edges[2 * e + 1];
        adj2[x * W + (y >> 5)] |= 1u << (y & 31);
        adj2[y * W + (x >> 5)] |= 1u << (x & 31);
        if (lab) {
            int32_t l = g2->elabels ? g2->elabels[e] : 0;
            uint8_t id = (uint8_t)label_id(l);
            e2[x * n2p + y] = id;
            e2[y * n2p + x] = id;
        }
    }
}

cudaEvent_t next_event(fastged_handle_t *h) {
    if (h->evused == (int)h->evpool.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        h->evpool.push_back(e);
    }
    return h->evpool[h->evused++];
}

// ---------------------------------------------------------------- batch build
void free_batch(fastged_batch *b) {
    if (!b) return;
    b->blob.release(); b->ddesc.release(); b->dorder.release(); b->dcost.release();
    b->dchild.release(); b->dpar.release(); b->dalg.release(); b->dmap.release(); b->dwork.release();
    b->stage.release();
    if (b->ev_h2d) cudaEventDestroy(b->ev_h2d);
    delete b;
}

// Validates, packs and uploads a batch.  `reuse` (optional) is a batch whose device buffers are
// recycled (solve_batch keeps one per handle, so repeated calls do no cudaMalloc/cudaFree).
fastged_batch *build_batch(fastged_handle_t *h, int32_t npairs, const fastged_graph_t *g1s,
                           const fastged_graph_t *g2s, fastged_batch *reuse = nullptr, int32_t pair_base = 0) {
    if (npairs < 0) fail(FASTGED_ERR_ARG, "npairs < 0");
    if (npairs > 0 && (!g1s || !g2s)) fail(FASTGED_ERR_ARG, "graph arrays are NULL");
    NvtxRange nv("fastged: validate + pack + H2D");
    fastged_batch *b = reuse ? reuse : new fastged_batch();
    b->ran = false;
    b->plan_valid = false; // (its device buffers may be reallocated below)
    b->n1max = b->n2max = 0;
    b->pair_base = pair_base;
    try {
        b->npairs = npairs;
        b->descs.resize(npairs);
        b->W.resize(npairs);
        b->map_off.resize(npairs + 1);
        std::vector<char> lab(npairs);
        std::vector<int> n2p(npairs);
        std::vector<int64_t> off(npairs + 1);
        off[0] = 0;
        b->map_off[0] = 0;
        // validation and sizing run in parallel over pairs (host cores); the first bad pair is reported
        std::vector<int64_t> sz(npairs);
        std::vector<FgError> perr(npairs > 0 ? 1 : 0);
        int bad = npairs;
#pragma omp parallel for schedule(dynamic, 64)
        for (int p = 0; p < npairs; ++p) {
            try {
                validate_graph(&g1s[p], pair_base + p, "g1");
                validate_graph(&g2s[p], pair_base + p, "g2");
                lab[p] = labelled_pair(&g1s[p], &g2s[p]);
                n2p[p] = (g2s[p].n + 3) & ~3;
                sz[p] = (int64_t)pair_blob_bytes(&g1s[p], &g2s[p], lab[p], n2p[p]);
            } catch (const FgError &e) {
#pragma omp critical(fg_err)
                if (p < bad) { bad = p; perr[0] = e; }
            } catch (...) { // (std::bad_alloc) no exception may leave the parallel region
#pragma omp critical(fg_err)
                if (p < bad) { bad = p; perr[0] = FgError{FASTGED_ERR_CAPACITY, "pair " + std::to_string(pair_base + p) + ": host allocation failed"}; }
            }
        }
        if (bad < npairs) throw perr[0];
        for (int p = 0; p < npairs; ++p) {
            off[p + 1] = off[p] + sz[p];
            b->map_off[p + 1] = b->map_off[p] + g1s[p].n;
            b->n1max = std::max(b->n1max, g1s[p].n);
            b->n2max = std::max(b->n2max, g2s[p].n);
        }
        b->total_map = b->map_off[npairs];
        size_t blob_bytes = (size_t)off[npairs];
        size_t desc_bytes = sizeof(fg::PairDesc) * (size_t)std::max(npairs, 1);
        b->ord_at = align16(blob_bytes + desc_bytes);
        b->res_at = align16(b->ord_at + 4 * (size_t)npairs);
        CK(b->stage.reserve(b->res_at + 32 * (size_t)npairs + 4 * (size_t)b->total_map + 64));
        uint8_t *stage = (uint8_t *)b->stage.p;
#pragma omp parallel for schedule(dynamic, 64)
        for (int p = 0; p < npairs; ++p) {
            try {
                pack_pair(&g1s[p], &g2s[p], lab[p], n2p[p], stage, off[p], b->descs[p], pair_base + p);
            } catch (const FgError &e) {
#pragma omp critical(fg_err)
                if (p < bad) { bad = p; perr[0] = e; }
            } catch (...) {
#pragma omp critical(fg_err)
                if (p < bad) { bad = p; perr[0] = FgError{FASTGED_ERR_CAPACITY, "pair " + std::to_string(pair_base + p) + ": host allocation failed"}; }
            }
            b->descs[p].map_out = b->map_off[p];
            b->W[p] = words_for(g2s[p].n);
        }
        if (bad < npairs) throw perr[0];
        memcpy(stage + blob_bytes, b->descs.data(), sizeof(fg::PairDesc) * (size_t)npairs);
        CK(b->blob.reserve(blob_bytes + 16));
        CK(b->ddesc.reserve(desc_bytes));
        CK(b->dorder.reserve(4 * (size_t)std::max(npairs, 1)));
        CK(b->dcost.reserve(8 * (size_t)std::max(npairs, 1)));
        CK(b->dchild.reserve(8 * (size_t)std::max(npairs, 1)));
        CK(b->dpar.reserve(8 * (size_t)std::max(npairs, 1)));
        CK(b->dalg.reserve(8 * (size_t)std::max(npairs, 1)));
        CK(b->dmap.reserve(4 * (size_t)std::max<int64_t>(b->total_map, 1)));
        CK(b->dwork.reserve(64 * sizeof(int)));
        // the copies go on the copy stream (run_batch orders the batch's kernels after them), so a pipelined
        // chunk's upload overlaps the search of the chunk before it
        if (!h->cstream) CK(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
        if (!b->ev_h2d) CK(cudaEventCreateWithFlags(&b->ev_h2d, cudaEventDisableTiming));
        if (blob_bytes) CK(cudaMemcpyAsync(b->blob.p, stage, blob_bytes, cudaMemcpyHostToDevice, h->cstream));
        if (npairs) CK(cudaMemcpyAsync(b->ddesc.p, stage + blob_bytes, sizeof(fg::PairDesc) * npairs,
                                       cudaMemcpyHostToDevice, h->cstream));
        CK(cudaEventRecord(b->ev_h2d, h->cstream));
        h->stats.h2d_bytes += (int64_t)(blob_bytes + sizeof(fg::PairDesc) * npairs);
        return b; // b->stage stays in use until the stream passes the copies (the next sync on it)
    } catch (...) {
        if (!reuse) {
            cudaStreamSynchronize(h->stream);
            if (h->cstream) cudaStreamSynchronize(h->cstream);
            free_batch(b);
        }
        throw;
    }
}

#ifndef FG_BATCH_NT
#define FG_BATCH_NT 256
#endif
constexpr int BATCH_NT = FG_BATCH_NT; // threads per CTA of the batched kernel (A/B: -DFG_BATCH_NT=...)
#ifndef FG_BATCH_NT_W1
#define FG_BATCH_NT_W1 128
#endif
#ifndef FG_BATCH_NT_W1_LAB
#define FG_BATCH_NT_W1_LAB 256
#endif
// one-word pairs (n2 <= 32) have small work arrays: a narrower CTA puts more pairs on an SM (unlabelled:
// 128 threads measured best); labelled one-word pairs, whose update builds the label planes, run faster at
// 256 threads (cfg5 slice 103.0 -> 100.1 ms; unlabelled cfg3 49.5 -> 50.1 ms, so not for those)
constexpr int BATCH_NT_W1 = FG_BATCH_NT_W1;
constexpr int BATCH_NT_W1_LAB = FG_BATCH_NT_W1_LAB;

constexpr int32_t PIPELINE_MIN_PAIRS = 4096; // solve_batch splits larger batches into two pipelined chunks

// Threads per CTA of a word-width group: one warp per pair when every level of every pair in the group
// has at most SMALL_CHILDREN candidates (e.g. AIDS-like pairs at K = 100: up to 16 pairs in flight per SM
// instead of 2, no cross-warp barriers), 128 for the other one-word groups, 256 otherwise.
constexpr int64_t SMALL_CHILDREN = 4096;
int batch_nt(int W, bool lab, int64_t kcap, int n2max) {
    if (W == 1 && kcap * (n2max + 1) <= SMALL_CHILDREN) return 32;
    return W == 1 ? (lab ? BATCH_NT_W1_LAB : BATCH_NT_W1) : BATCH_NT;
}

void *batch_kernel_for(int W, bool lab, bool smem, int nt) {
#define KV(WW, LL, SS, NN) \
    if (W == WW && lab == LL && smem == SS && nt == NN) return (void *)fg::kbest_batch_kernel<WW, LL, NN, SS>;
    KV(1, false, true, 32) KV(1, true, true, 32)
    KV(1, false, true, BATCH_NT_W1) KV(1, false, false, BATCH_NT_W1) KV(1, true, true, BATCH_NT_W1_LAB) KV(1, true, false, BATCH_NT_W1_LAB)
    KV(2, false, true, BATCH_NT) KV(2, true, true, BATCH_NT) KV(3, false, true, BATCH_NT) KV(3, true, true, BATCH_NT)
    KV(4, false, true, BATCH_NT) KV(4, true, true, BATCH_NT)
    KV(2, false, false, BATCH_NT) KV(2, true, false, BATCH_NT)
    KV(3, false, false, BATCH_NT) KV(3, true, false, BATCH_NT) KV(4, false, false, BATCH_NT) KV(4, true, false, BATCH_NT)
#undef KV
    return nullptr;
}

// Device destinations of one pair's results inside a batch (solve_large writes there instead of
// returning to the host).
struct LargeDst {
    int64_t *cost, *children, *parents, *algb;
    int32_t *map;
};
void solve_large(fastged_handle_t *h, const fastged_graph_t *g1, const fastged_graph_t *g2,
                 const fastged_costs_t *c, int64_t k, fastged_result_t *out, int64_t *levels_out,
                 const LargeDst *dst = nullptr, bool sharded = false);

// A pair rebuilt from its packed form in the batch's staging (vertex labels as given, edge labels
// as the interned ids of pack_pair -- equal ids exactly where the original labels are equal, which is
// all the costs depend on).  Used to hand a pair beyond the batched limits to solve_large.
struct HostGraph {
    std::vector<int32_t> vl, e, el;
    fastged_graph_t view() const {
        return fastged_graph_t{(int32_t)vl.size(), (int32_t)(e.size() / 2), vl.data(), e.data(), el.data()};
    }
};
void unpack_pair(const uint8_t *stage, const fg::PairDesc &d, HostGraph &g1, HostGraph &g2) {
    const int32_t *vl1 = (const int32_t *)(stage + d.vl1), *vl2 = (const int32_t *)(stage + d.vl2);
    const int32_t *pptr = (const int32_t *)(stage + d.pptr), *pq = (const int32_t *)(stage + d.pq);
    const int32_t *pl = (const int32_t *)(stage + d.pl);
    const uint32_t *adj2 = (const uint32_t *)(stage + d.adj2);
    const uint8_t *e2 = d.labelled ? stage + d.e2lab : nullptr;
    const int W = words_for(d.n2);
    g1.vl.assign(vl1, vl1 + d.n1);
    g2.vl.assign(vl2, vl2 + d.n2);
    g1.e.clear(); g1.el.clear(); g2.e.clear(); g2.el.clear();
    for (int i = 0; i < d.n1; ++i)
        for (int x = pptr[i]; x < pptr[i + 1]; ++x) {
            g1.e.push_back(pq[x]);
            g1.e.push_back(i);
            g1.el.push_back(pl[x]);
        }
    for (int u = 0; u < d.n2; ++u)
        for (int v = u + 1; v < d.n2; ++v)
            if ((adj2[(size_t)u * W + (v >> 5)] >> (v & 31)) & 1u) {
                g2.e.push_back(u);
                g2.e.push_back(v);
                g2.el.push_back(e2 ? (int32_t)e2[(size_t)u * d.n2p + v] : 0);
            }
    g1.el.push_back(0); // (non-empty: .data() is a valid pointer for m = 0)
    g2.el.push_back(0);
}

// first = false appends to the timing/launch stats of a preceding run_batch on the same stream
// (pipelined chunks of one solve_batch call).
void run_batch(fastged_handle_t *h, fastged_batch *b, const fastged_costs_t *c, int64_t k,
               int64_t *levels_dev, bool first = true) {
    validate_costs(c);
    if (k < 1) fail(FASTGED_ERR_ARG, "k < 1");
    NvtxRange nv("fastged: plan + launch batch");
    // The launch plan of a batch (groups, scheduling order, kernel variants, grids, scratch slices) depends
    // only on (K, costs, flags) and the handle's scratch: repeated runs of a resident batch reuse it, so a
    // small batch is not dominated by host-side planning (the device sits idle while the host plans).
    const bool reuse = b->plan_valid && b->plan_k == k && memcmp(&b->plan_c, c, sizeof *c) == 0 &&
                       b->plan_flags == h->flags && levels_dev == nullptr && b->plan_scratch == h->scratch.p;
    bool upload_order = false;
    std::vector<int32_t> order_all;
    if (!reuse) {
    b->plan_valid = false;
    // group pairs by kernel variant; schedule the largest pairs first (dynamic counter)
    b->groups.clear();
    b->large.clear();
    for (int p = 0; p < b->npairs; ++p) {
        const fg::PairDesc &d = b->descs[p];
        int64_t bound = (int64_t)d.n1 * std::max(c->vsub, c->vdel) + (int64_t)d.n2 * c->vins +
                        ((int64_t)d.m1 + d.m2) * std::max(c->esub, std::max(c->edel, c->eins)) + 512;
        if (bound >= ((int64_t)1 << 31))
            fail(FASTGED_ERR_OVERFLOW, "pair %d: worst-case PED %lld does not fit int32", b->pair_base + p, (long long)bound);
        if (fits_batched(d.n1, d.n2, k, d.labelled ? d.nlab : 0) && !(h->flags & FASTGED_FLAG_FORCE_LARGE) &&
            !(h->flags & FASTGED_FLAG_APPROX_MASK) &&
            !prefers_whole_gpu(d.n1, d.n2, k, b->npairs))
            b->groups[GroupKey{b->W[p], d.labelled != 0}].push_back(p);
        else
            b->large.push_back(p); // solved by the whole-GPU kernel after the batched launches
    }
    std::vector<std::pair<GroupKey, std::pair<size_t, size_t>>> spans;
    for (auto &kv : b->groups) {
        auto &v = kv.second;
        std::stable_sort(v.begin(), v.end(), [&](int x, int y) {
            const fg::PairDesc &a = b->descs[x], &bb = b->descs[y];
            return (int64_t)a.n1 * (a.n2 + 1) > (int64_t)bb.n1 * (bb.n2 + 1);
        });
        spans.push_back({kv.first, {order_all.size(), v.size()}});
        order_all.insert(order_all.end(), v.begin(), v.end());
    }
    int gi = 0;
    std::vector<GroupLaunch> &plans = b->plans;
    plans.clear();
    for (auto &sp : spans) {
        const GroupKey key = sp.first;
        const size_t start = sp.second.first, cnt = sp.second.second;
        int n1max = 0, n2max = 0;
        int64_t kcap = 1;
        for (size_t x = start; x < start + cnt; ++x) {
            const fg::PairDesc &d = b->descs[order_all[x]];
            n1max = std::max(n1max, d.n1);
            n2max = std::max(n2max, d.n2);
            kcap = std::max(kcap, frontier_cap(d.n1, d.n2, k));
        }
        const int W = key.W;
        fg::BatchArgs a{};
        a.descs = (const fg::PairDesc *)b->ddesc.p;
        a.order = (const int32_t *)b->dorder.p + start;
        a.ngroup = (int)cnt;
        a.blob = (const uint8_t *)b->blob.p;
        a.work = (int32_t *)b->dwork.p + gi;
        a.c = fg::Costs{c->vsub, c->vdel, c->vins, c->esub, c->edel, c->eins};
        // k beyond every level's candidate count selects like the cap (frontier_cap), so the kernel's
        // int32 K is min(k, cap)
        a.K = (int)std::min<int64_t>(k, kcap);
        a.Kc = (int)((kcap + 3) & ~3ll);
        a.win = (h->flags & FASTGED_FLAG_DEBUG_WINDOW) ? 2 : 127; // codes 0..128 (SWAR compares need <= 128)
        a.n1max = std::max(4, (n1max + 3) & ~3);
        a.csmax = (n2max + 1 + 3) & ~3;
        const size_t Kc = (size_t)a.Kc;
        const int NB = key.lab ? 1 + fg::LMAX : 1;
        // always-shared small arrays
        size_t sm = 0;
        auto sput = [&](int32_t &field, size_t bytes) { field = (int)sm; sm += align16(bytes); };
        sput(a.sm.pq, 4 * (size_t)a.n1max);
        sput(a.sm.pl, 4 * (size_t)a.n1max);
        sput(a.sm.pnl, (size_t)a.n1max);
        sput(a.sm.pnq, 4 * (size_t)a.n1max);
        sput(a.sm.adj, 4 * (size_t)std::max(n2max, 1) * W);
        sput(a.sm.adjl, key.lab ? 4 * (size_t)std::max(n2max, 1) * fg::LMAX * W : 0);
        sput(a.sm.adjh, 4 * (size_t)32 * W * fg::hrow_stride(W, key.lab));
        // per-level work arrays
        size_t wk = 0;
        auto put = [&](int32_t &field, size_t bytes) { field = (int)wk; wk += align16(bytes); };
        put(a.sm.u, 4 * Kc * W);           // parent used masks
        put(a.sm.b, 4 * (Kc + 1));         // compact code offsets
        put(a.sm.codes, Kc * a.csmax);     // rank codes of the level
        put(a.sm.sel, 4 * Kc);             // survivors
        put(a.sm.pidx, 2 * (Kc * a.csmax / 16 + 2)); // code position -> parent index
        const bool in_smem = sm + wk + 8192 <= h->smem_optin;
        size_t smem = sm;
        if (in_smem) {
            for (int32_t *f : {&a.sm.u, &a.sm.b, &a.sm.codes, &a.sm.sel, &a.sm.pidx}) *f += (int)sm;
            smem += wk;
        }
        a.sm.bytes = (int)smem;
        size_t per_cta = 2 * Kc * (4 + 4 * (size_t)W + 4 * (size_t)W * NB + (size_t)a.n1max) + (in_smem ? 0 : wk);
        per_cta = (per_cta + 255) & ~(size_t)255;
        const int nt = in_smem ? batch_nt(W, key.lab, kcap, n2max) : batch_nt(W, key.lab, 1 << 30, n2max);
        void *kern = batch_kernel_for(W, key.lab, in_smem, nt);
        if (!kern) fail(FASTGED_ERR_ARG, "no kernel variant for W=%d", W);
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem));
        occ = std::max(occ, 1);
        int grid = (int)std::min<int64_t>((int64_t)cnt, (int64_t)occ * h->sms);
        a.scratch = nullptr; // set below: this group's slice of the handle's scratch
        a.scratch_stride = (int64_t)per_cta;
        a.cost_out = (int64_t *)b->dcost.p;
        a.map_out = (int32_t *)b->dmap.p;
        a.children_out = (int64_t *)b->dchild.p;
        a.parents_out = (int64_t *)b->dpar.p;
        a.algbytes_out = (int64_t *)b->dalg.p;
        a.levels_out = levels_dev;
        a.last_by_total = (h->flags & FASTGED_FLAG_LAST_BY_TOTAL) ? 1 : 0;
        const fg::PairDesc &d0 = b->descs[order_all[start]]; // (the group's largest pair: sorted above)
        plans.push_back(GroupLaunch{a, kern, grid, nt, smem, per_cta, (int64_t)d0.n1 * (d0.n2 + 1)});
        gi++;
    }
    // longest pairs first across the groups too: the group holding the largest pair is launched first
    std::stable_sort(plans.begin(), plans.end(), [](const GroupLaunch &x, const GroupLaunch &y) { return x.cost > y.cost; });
    // scratch: one slice per group (the groups run concurrently); shrink grids, never K
    {
        size_t need = 0;
        for (auto &g : plans) need += g.per_cta * (size_t)g.grid;
        if (need > h->scratch.cap) {
            size_t free_b = 0, total_b = 0;
            CK(cudaMemGetInfo(&free_b, &total_b));
            const size_t avail = free_b + h->scratch.cap;
            for (auto &g : plans)
                if (g.per_cta > avail / 2) fail(FASTGED_ERR_CAPACITY, "frontier scratch %zu B per CTA exceeds device memory", g.per_cta);
            while (need > avail * 3 / 4) { // shrink the largest grid
                GroupLaunch *m = nullptr;
                for (auto &g : plans) if (g.grid > 1 && (!m || g.per_cta * g.grid > m->per_cta * m->grid)) m = &g;
                if (!m) break;
                m->grid--;
                need -= m->per_cta;
            }
            CK(cudaStreamSynchronize(h->stream)); // the previous slices may still be in use
            for (cudaStream_t gs : h->gstreams) CK(cudaStreamSynchronize(gs));
            h->scratch.release();
            CK(h->scratch.reserve(need));
        }
        size_t off = 0;
        for (auto &g : plans) {
            g.a.scratch = (uint8_t *)h->scratch.p + off;
            off += g.per_cta * (size_t)g.grid;
        }
    }
    b->order_all.swap(order_all);
    b->plan_valid = levels_dev == nullptr;
    b->plan_k = k;
    b->plan_c = *c;
    b->plan_flags = h->flags;
    b->plan_scratch = h->scratch.p;
    upload_order = true;
    }
    if (first) {
        h->evused = 0;
        h->stats.kernel_launches = 0;
        h->stats.branch_launches = 0;
        h->stats.branch_ms = 0.f;
    }
    if (first) CK(cudaEventRecord(h->ev_begin, h->stream));
    if (b->ev_h2d) CK(cudaStreamWaitEvent(h->stream, b->ev_h2d, 0)); // the batch's inputs are on the device
    if (upload_order && !b->order_all.empty()) {
        // the order goes behind the blob in this batch's staging (the blob's bytes may still be in flight)
        uint8_t *ord = (uint8_t *)b->stage.p + b->ord_at;
        memcpy(ord, b->order_all.data(), 4 * b->order_all.size());
        CK(cudaMemcpyAsync(b->dorder.p, ord, 4 * b->order_all.size(), cudaMemcpyHostToDevice, h->stream));
        h->stats.h2d_bytes += (int64_t)(4 * b->order_all.size());
    }
    CK(cudaMemsetAsync(b->dwork.p, 0, 64 * sizeof(int), h->stream));
    std::vector<GroupLaunch> &plans = b->plans;
    // fork: group 0 on the handle's stream, the others on side streams; join back before ev_end
    const size_t ng = plans.size();
    while (h->gstreams.size() + 1 < ng) {
        cudaStream_t gs;
        CK(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
        h->gstreams.push_back(gs);
    }
    while (h->gevents.size() < ng + 1) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->gevents.push_back(e);
    }
    if (ng > 1) CK(cudaEventRecord(h->gevents[0], h->stream));
    for (size_t g = 0; g < ng; ++g) {
        cudaStream_t st = g == 0 ? h->stream : h->gstreams[g - 1];
        if (g > 0) CK(cudaStreamWaitEvent(st, h->gevents[0], 0));
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (h->flags & FASTGED_FLAG_TIMING) {
            e0 = next_event(h);
            e1 = next_event(h);
            CK(cudaEventRecord(e0, st));
        }
        void *params[] = {(void *)&plans[g].a};
        CK(cudaLaunchKernel(plans[g].kern, dim3(plans[g].grid), dim3(plans[g].nt), params, plans[g].smem, st));
        if (e1) CK(cudaEventRecord(e1, st));
        h->stats.kernel_launches++;
        if (g > 0) {
            CK(cudaEventRecord(h->gevents[g], st));
            CK(cudaStreamWaitEvent(h->stream, h->gevents[g], 0));
        }
    }
    // pairs beyond the batched limits: the whole-GPU kernel, one pair after the other on the handle's
    // stream, results written into this batch's device outputs (SURVEY §3.3 size classes)
    for (size_t x = 0; x < b->large.size(); ++x) {
        const int p = b->large[x];
        const fg::PairDesc &d = b->descs[p];
        HostGraph G1, G2;
        unpack_pair((const uint8_t *)b->stage.p, d, G1, G2);
        const fastged_graph_t v1 = G1.view(), v2 = G2.view();
        if (x > 0) CK(cudaStreamSynchronize(h->stream)); // solve_large restages through h->stage
        LargeDst dst{(int64_t *)b->dcost.p + p, (int64_t *)b->dchild.p + p, (int64_t *)b->dpar.p + p,
                     (int64_t *)b->dalg.p + p, (int32_t *)b->dmap.p + b->map_off[p]};
        try {
            solve_large(h, &v1, &v2, c, k, nullptr, nullptr, &dst);
        } catch (FgError &e) {
            e.msg = "pair " + std::to_string(b->pair_base + p) + " (whole-GPU path): " + e.msg;
            throw;
        }
    }
    CK(cudaEventRecord(h->ev_end, h->stream));
    b->ran = true;
}

void finish_timing(fastged_handle_t *h) {
    float ms = 0.f;
    CK(cudaEventSynchronize(h->ev_end));
    CK(cudaEventElapsedTime(&ms, h->ev_begin, h->ev_end));
    h->stats.device_ms = ms;
    if (h->flags & FASTGED_FLAG_TIMING) {
        float tot = 0.f;
        for (int x = 0; x + 1 < h->evused; x += 2) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, h->evpool[x], h->evpool[x + 1]));
            tot += t;
        }
        h->stats.branch_ms = tot;
        h->stats.branch_launches = h->evused / 2;
    }
}

// Enqueue the D2H copies of a batch's results into its staging (no sync).
void download_enqueue(fastged_handle_t *h, fastged_batch *b) {
    if (!b->ran) fail(FASTGED_ERR_ARG, "batch was not run");
    NvtxRange nv("fastged: D2H results");
    const size_t P = (size_t)b->npairs, M = (size_t)b->total_map;
    uint8_t *st = (uint8_t *)b->stage.p + b->res_at;
    int64_t *hc = (int64_t *)st, *hch = hc + P, *hpa = hch + P, *hal = hpa + P;
    int32_t *hm = (int32_t *)(hal + P);
    if (P) {
        CK(cudaMemcpyAsync(hc, b->dcost.p, 8 * P, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(hch, b->dchild.p, 8 * P, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(hpa, b->dpar.p, 8 * P, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(hal, b->dalg.p, 8 * P, cudaMemcpyDeviceToHost, h->stream));
    }
    if (M) CK(cudaMemcpyAsync(hm, b->dmap.p, 4 * M, cudaMemcpyDeviceToHost, h->stream));
    h->stats.d2h_bytes += (int64_t)(32 * P + 4 * M);
}

// After the stream sync: copy a batch's results out and add its counters to the stats.
void download_collect(fastged_handle_t *h, fastged_batch *b, int64_t *costs_out, int32_t *mappings_out,
                      int64_t *children_out) {
    const size_t P = (size_t)b->npairs, M = (size_t)b->total_map;
    uint8_t *st = (uint8_t *)b->stage.p + b->res_at;
    int64_t *hc = (int64_t *)st, *hch = hc + P, *hpa = hch + P, *hal = hpa + P;
    int32_t *hm = (int32_t *)(hal + P);
    if (P) memcpy(costs_out, hc, 8 * P);
    if (M) memcpy(mappings_out, hm, 4 * M);
    if (children_out && P) memcpy(children_out, hch, 8 * P);
    int64_t ch = 0, pa = 0, al = 0, ops = 0;
    for (size_t p = 0; p < P; ++p) {
        ch += hch[p]; pa += hpa[p]; al += hal[p];
        // popcount-form lane-ops per child = 2W AND + 2W POPC + 3 cost + 2 clamp + 1
        // histogram index (the op mix scripts/micro/int_peak.cu measures as the 'alu' peak)
        ops += hch[p] * (4 * (int64_t)b->W[p] + 6);
    }
    h->stats.children_evaluated += ch;
    h->stats.parents_expanded += pa;
    h->stats.alg_bytes += al;
    h->stats.alg_ops += ops;
}

void check_outputs(const fastged_batch *b, int64_t *costs_out, int32_t *mappings_out) {
    if (b->npairs > 0 && !costs_out) fail(FASTGED_ERR_ARG, "costs_out is NULL");
    if (b->total_map > 0 && !mappings_out) fail(FASTGED_ERR_ARG, "mappings_out is NULL");
}

void download(fastged_handle_t *h, fastged_batch *b, int64_t *costs_out, int32_t *mappings_out,
              int64_t *children_out) {
    check_outputs(b, costs_out, mappings_out);
    download_enqueue(h, b);
    CK(cudaStreamSynchronize(h->stream));
    finish_timing(h);
    h->stats.children_evaluated = h->stats.parents_expanded = h->stats.alg_bytes = h->stats.alg_ops = 0;
    download_collect(h, b, costs_out, mappings_out, children_out);
}

void begin_call(fastged_handle_t *h) {
    h->err.clear();
    h->stats = fastged_stats_t{};
    CK(cudaSetDevice(h->device));
}


#include "shard_host.inc"

void solve_large(fastged_handle_t *h, const fastged_graph_t *g1, const fastged_graph_t *g2,
                 const fastged_costs_t *c, int64_t k, fastged_result_t *out, int64_t *levels_out,
                 const LargeDst *dst, bool sharded) {
    NvtxRange nv(sharded ? "fastged: sharded pair" : "fastged: whole-GPU pair");
    // sharded single pair: G ranks, each a cooperative grid on its own GPU (peer
    // memory over NVLink), or -- FASTGED_FLAG_VIRTUAL_SHARDS -- G CTA groups of one grid on this GPU
    const int G = sharded ? h->world : 1;
    const bool virt = sharded && (h->flags & FASTGED_FLAG_VIRTUAL_SHARDS);
    const bool real = G > 1 && !virt;
    const int myrank = real ? h->rank : 0;
    if (G > FG_MAXG) fail(FASTGED_ERR_ARG, "sharded mode supports at most %d ranks", FG_MAXG);
    if (real && !h->comm) fail(FASTGED_ERR_NCCL, "the handle's NCCL communicator was aborted by an earlier failure");
    if (dst && G > 1) fail(FASTGED_ERR_ARG, "internal: a batch pair is never sharded");
    const int n1 = g1->n, n2 = g2->n;
    if ((h->flags & FASTGED_FLAG_LAST_BY_TOTAL) && (h->flags & FASTGED_FLAG_APPROX_MASK))
        fail(FASTGED_ERR_ARG, "FASTGED_FLAG_LAST_BY_TOTAL and FASTGED_FLAG_APPROX are exclusive");
    if (n2 > FASTGED_MAX_N2) fail(FASTGED_ERR_CAPACITY, "target graph has n2=%d > %d (limit of this build)", n2, FASTGED_MAX_N2);
    const int64_t Kc64 = frontier_cap(n1, n2, k);
    if (Kc64 > (int64_t)1 << 30) fail(FASTGED_ERR_CAPACITY, "frontier cap %lld too large", (long long)Kc64);
    const int Kc = (int)Kc64;
    const bool lab = labelled_pair(g1, g2);
    const int n2p = (n2 + 3) & ~3;
    const int W = words_for(n2);
    const int cs = (n2 + 1 + 127) & ~127; // code / counter row stride: lane l owns u = 128 s + 4 l + b
    // g2 extras behind the packed pair: CSR neighbour lists (label id in the high half) and the
    // transposed bit rows adjT[W][cs] (bit u' of adjT[w][u] = edge (u, 32 w + u'))
    const size_t base_bytes = pair_blob_bytes(g1, g2, lab, n2p);
    const size_t o_nptr = base_bytes, o_nbr = o_nptr + align16(4 * (size_t)(n2 + 1));
    const size_t o_adjT = o_nbr + align16(8 * (size_t)g2->m + 4);
    const size_t blob_bytes = o_adjT + 4 * (size_t)W * cs;
    CK(h->stage.reserve(blob_bytes + 64));
    uint8_t *st = (uint8_t *)h->stage.p;
    fg::PairDesc pd{};
    pack_pair(g1, g2, lab, n2p, st, 0, pd, 0);
    pd.map_out = 0;
    int maxdeg = 0;
    {
        int32_t *nptr = (int32_t *)(st + o_nptr);
        uint32_t *nbr = (uint32_t *)(st + o_nbr);
        uint32_t *adjT = (uint32_t *)(st + o_adjT);
        const uint32_t *adj2 = (const uint32_t *)(st + pd.adj2);
        const uint8_t *e2 = lab ? st + pd.e2lab : nullptr;
        std::vector<int> deg(n2 + 1, 0);
        for (int e = 0; e < g2->m; ++e) { deg[g2->edges[2 * e]]++; deg[g2->edges[2 * e + 1]]++; }
        nptr[0] = 0;
        for (int u = 0; u < n2; ++u) { nptr[u + 1] = nptr[u] + deg[u]; maxdeg = std::max(maxdeg, deg[u]); }
        std::vector<int> fill(nptr, nptr + n2);
        for (int e = 0; e < g2->m; ++e) {
            const int x = g2->edges[2 * e], y = g2->edges[2 * e + 1];
            const uint32_t l = lab ? (uint32_t)e2[(size_t)x * n2p + y] : 0u;
            nbr[fill[x]++] = (uint32_t)y | (l << 16);
            nbr[fill[y]++] = (uint32_t)x | (l << 16);
        }
        memset(adjT, 0, 4 * (size_t)W * cs);
        for (int u = 0; u < n2; ++u)
            for (int w = 0; w < W; ++w) adjT[(size_t)w * cs + u] = adj2[(size_t)u * W + w];
    }
    CK(h->lblob.reserve(blob_bytes + 16));
    CK(cudaMemcpyAsync(h->lblob.p, h->stage.p, blob_bytes, cudaMemcpyHostToDevice, h->stream));
    h->stats.h2d_bytes += (int64_t)blob_bytes;

    const bool wide = n2 > 254;          // lambda entries: uint16 (255 would collide with "deleted")
    const bool c16 = maxdeg > 255;       // counters: uint16 when a degree does not fit a byte
    const int esz = wide ? 2 : 1, csz = c16 ? 2 : 1;
    // lambda row stride: a 16-byte multiple (the kernel moves rows in 16-byte chunks)
    const int n1s = wide ? std::max(8, (n1 + 7) & ~7) : std::max(16, (n1 + 15) & ~15);
    int dmax = 0;
    {
        std::vector<int> dd(n1 + 1, 0);
        for (int e = 0; e < g1->m; ++e) dd[std::max(g1->edges[2 * e], g1->edges[2 * e + 1])]++;
        for (int x : dd) dmax = std::max(dmax, x);
    }
    const int n1r = std::max(4, (dmax + 3) & ~3);
    // shared-memory staging: the CSR when the scatter form is likely (sparse g2), the transposed
    // rows otherwise; both when they fit; fewer branching warps per CTA only as a last resort
    const int nnbr = 2 * g2->m;
    const bool sparse = (n2 ? 2 * g2->m / n2 : 0) <= 32;
    bool csr_in_smem = false, adjT_in_smem = false;
    int nwa = fg::LNT / 32;
    // the kernel's static shared memory (block-wide scratch) counts against the same per-CTA limit
    size_t static_smem = 0;
    {
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, (const void *)fg::kbest_large_kernel<uint16_t, uint16_t, true, 2>));
        static_smem = fa.sharedSizeBytes;
    }
    const size_t smem_cap = (size_t)h->smem_optin - static_smem;
    auto fits = [&](bool at, bool cr, int nw) {
        return fg::large_smem_bytes(cs, csz, n1s, esz, nw, n1r, W, n2, nnbr, at, cr) <= smem_cap;
    };
    if (fits(true, true, nwa)) adjT_in_smem = csr_in_smem = true;
    else if (sparse && fits(false, true, nwa)) csr_in_smem = true;
    else if (fits(true, false, nwa)) adjT_in_smem = true;
    else if (fits(false, true, nwa)) csr_in_smem = true;
    while (nwa > 1 && !fits(adjT_in_smem, csr_in_smem, nwa)) nwa--;
    const size_t smem = fg::large_smem_bytes(cs, csz, n1s, esz, nwa, n1r, W, n2, nnbr, adjT_in_smem, csr_in_smem);
    if (smem > smem_cap) fail(FASTGED_ERR_CAPACITY, "large-mode kernel needs %zu B of shared memory", smem);
    void *kfn = nullptr;
#define LK(M, C, L) (virt ? (void *)fg::kbest_large_kernel<M, C, L, 2> \
                         : real ? (void *)fg::kbest_large_kernel<M, C, L, 1> : (void *)fg::kbest_large_kernel<M, C, L, 0>)
    if (wide) kfn = c16 ? (lab ? LK(uint16_t, uint16_t, true) : LK(uint16_t, uint16_t, false))
                        : (lab ? LK(uint16_t, uint8_t, true) : LK(uint16_t, uint8_t, false));
    else kfn = c16 ? (lab ? LK(uint8_t, uint16_t, true) : LK(uint8_t, uint16_t, false))
                   : (lab ? LK(uint8_t, uint8_t, true) : LK(uint8_t, uint8_t, false));
#undef LK
    int occ = 0;
    CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, fg::LNT, smem));
    if (occ < 1) fail(FASTGED_ERR_CAPACITY, "large-mode kernel does not fit on an SM (smem %zu)", smem);
    occ = 1; // one CTA per SM (the grid barrier cost grows with the CTA count)
    const int nb = virt ? h->sms / G : occ * h->sms; // CTAs per rank
    if (nb < 1) fail(FASTGED_ERR_ARG, "%d virtual shards on %d SMs", G, h->sms);
    const int grid = virt ? G * nb : nb;
    const int GW = nb * (fg::LNT / 32); // warps per rank
    if (nb > fg::LMAXGRID) fail(FASTGED_ERR_ARG, "large-mode grid %d exceeds %d CTAs", nb, fg::LMAXGRID);
    // device buffers: the home arrays (used on rank 0 only), then one rank-local block per rank held
    // here (G blocks in virtual mode); a rank's slice of a level holds at most ceil(Kc / G) nodes
    const size_t Kl = (size_t)((Kc + G - 1) / G);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
    const size_t o_hist = take(4 * 3 * 256), o_ci = take(8 * (size_t)(n1 + 1)), o_drop = take(4 * (size_t)(n1 + 1));
    const size_t o_lo = take(4 * (size_t)(n1 + 2)), o_hi = take(4 * (size_t)(n1 + 2));
    const size_t o_ctl = take(4 * (size_t)G * nb), o_cte = take(4 * (size_t)G * nb);
    const size_t o_best = take(8), o_bar = take(4), o_out = take(80);
    const size_t o_mapout = take(4 * (size_t)(n1 + 1)), o_lev = take(24 * (size_t)(n1 + 1));
    const size_t o_rk = take(sizeof(fg::LargeArgs::Rank) * FG_MAXG), o_xerr = take(4);
    const size_t home_bytes = off;
    off = 0;
    const size_t l_ped0 = take(4 * Kl), l_ped1 = take(4 * Kl);
    const size_t l_used0 = take(4 * Kl * W), l_used1 = take(4 * Kl * W);
    const size_t l_cnt0 = take((size_t)csz * cs * Kl), l_cnt1 = take((size_t)csz * cs * Kl);
    const size_t l_map0 = take((size_t)esz * n1s * Kl), l_map1 = take((size_t)esz * n1s * Kl);
    const size_t l_ccode = take(Kl * cs), l_ctgt = take(2 * Kl * cs), l_rown = take(4 * Kl);
    const size_t l_selp = take(4 * Kl), l_selj = take(4 * Kl), l_selped = take(4 * Kl);
    const size_t l_rowc = take(4 * Kl), l_rowpl = take(4 * Kl), l_rowpe = take(4 * Kl), l_rowmin = take(4 * Kl);
    const size_t l_wlt = take(4 * (size_t)GW), l_weq = take(4 * (size_t)GW);
    const size_t local_bytes = off;
    const int nloc = virt ? G : 1; // rank-local blocks in this process
    CK(h->lbuf.reserve(home_bytes + (size_t)nloc * local_bytes));
    uint8_t *B = (uint8_t *)h->lbuf.p;
    // base address of every rank's buffer (real mode: peers' buffers mapped over NVLink)
    std::vector<uint8_t *> rbase(G, nullptr);
    if (real) {
        const int64_t key[2] = {(int64_t)nb, (int64_t)(home_bytes + local_bytes)};
        ipc_map_peers(h, B, rbase, key);
    } else {
        rbase[0] = B;
    }
    uint8_t *H = rbase[0]; // home arrays (rank 0)
    std::vector<fg::LargeArgs::Rank> rk(FG_MAXG);
    for (int r = 0; r < G; ++r) {
        uint8_t *L = virt ? B + home_bytes + (size_t)r * local_bytes : rbase[real ? r : 0] + home_bytes;
        fg::LargeArgs::Rank &x = rk[r];
        x.ped[0] = (int32_t *)(L + l_ped0); x.ped[1] = (int32_t *)(L + l_ped1);
        x.used[0] = (uint32_t *)(L + l_used0); x.used[1] = (uint32_t *)(L + l_used1);
        x.cnt[0] = L + l_cnt0; x.cnt[1] = L + l_cnt1;
        x.map[0] = L + l_map0; x.map[1] = L + l_map1;
        x.ccode = L + l_ccode;
        x.ctgt = (uint16_t *)(L + l_ctgt);
        x.rown = (int32_t *)(L + l_rown);
        x.sel_p = (int32_t *)(L + l_selp); x.sel_j = (int32_t *)(L + l_selj); x.sel_ped = (int32_t *)(L + l_selped);
        x.rowc = (int32_t *)(L + l_rowc); x.rowpl = (int32_t *)(L + l_rowpl); x.rowpe = (int32_t *)(L + l_rowpe);
        x.rowmin = (int32_t *)(L + l_rowmin);
        x.wlt = (int32_t *)(L + l_wlt); x.weq = (int32_t *)(L + l_weq);
    }
    CK(cudaMemcpyAsync(B + o_rk, rk.data(), sizeof(fg::LargeArgs::Rank) * FG_MAXG, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemsetAsync(B + o_xerr, 0, 4, h->stream));
    if (myrank == 0) { // the home arrays (only rank 0's are read)
        CK(cudaMemsetAsync(B + o_hist, 0, 4 * 3 * 256, h->stream));
        CK(cudaMemsetAsync(B + o_ci, 0, 8 * (size_t)(n1 + 1), h->stream));
        CK(cudaMemsetAsync(B + o_drop, 0, 4 * (size_t)(n1 + 1), h->stream));
        CK(cudaMemsetAsync(B + o_lo, 0x7f, 4 * (size_t)(n1 + 2), h->stream));
        CK(cudaMemsetAsync(B + o_hi, 0x80, 4 * (size_t)(n1 + 2), h->stream));
        CK(cudaMemsetAsync(B + o_best, 0xff, 8, h->stream));
        CK(cudaMemsetAsync(B + o_bar, 0, 4, h->stream));
    }
    const uint8_t *dblob = (const uint8_t *)h->lblob.p;
    fg::LargeArgs a{};
    a.blob = dblob;
    a.pd = pd;
    a.c = fg::Costs{c->vsub, c->vdel, c->vins, c->esub, c->edel, c->eins};
    a.K = Kc;
    a.win = (h->flags & FASTGED_FLAG_DEBUG_WINDOW) ? 2 : 253;
    a.ashift = (int32_t)((h->flags & FASTGED_FLAG_APPROX_MASK) >> 8);
    a.last_by_total = (h->flags & FASTGED_FLAG_LAST_BY_TOTAL) ? 1 : 0;
    a.W = W;
    a.cs = cs;
    a.S = cs / 128;
    a.n1s = n1s;
    a.n1r = n1r;
    a.adjT_in_smem = adjT_in_smem ? 1 : 0;
    a.csr_in_smem = csr_in_smem ? 1 : 0;
    a.csz = csz;
    a.nwa = nwa;
    a.degw = std::max(1, (n2 ? (2 * g2->m + n2 - 1) / n2 : 0) + 31) / 32;
    a.nptr = (const int32_t *)(dblob + o_nptr);
    a.nbr = (const uint32_t *)(dblob + o_nbr);
    a.adjT = (const uint32_t *)(dblob + o_adjT);
    a.G = G;
    a.nb = nb;
    a.kl = (int32_t)Kl;
    a.rank = myrank;
    a.virt = virt ? 1 : 0;
    a.rk = (const fg::LargeArgs::Rank *)(B + o_rk);
    a.self = rk[myrank];
    a.vstride = virt ? (int64_t)local_bytes : 0;
    a.hist = (int32_t *)(H + o_hist);
    a.ci = (int64_t *)(H + o_ci);
    a.drop = (int32_t *)(H + o_drop);
    a.lo = (int32_t *)(H + o_lo);
    a.hi = (int32_t *)(H + o_hi);
    a.ctl = (int32_t *)(H + o_ctl); a.cte = (int32_t *)(H + o_cte);
    a.best = (unsigned long long *)(H + o_best);
    a.bar = (unsigned int *)(H + o_bar);
    a.xerr = (int32_t *)(B + o_xerr);
    a.xtimeout_ns = (int64_t)(nccl_timeout_s() * 1e9);
    a.out = (int64_t *)(H + o_out);
    a.map_out = (int32_t *)(H + o_mapout);
    a.levels_out = levels_out ? (int64_t *)(H + o_lev) : nullptr;
    void *params[] = {(void *)&a};
    if (dst) { // inside a batch: enqueue only, results stay on the device (stream-ordered copies)
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (h->flags & FASTGED_FLAG_TIMING) {
            e0 = next_event(h);
            e1 = next_event(h);
            CK(cudaEventRecord(e0, h->stream));
        }
        CK(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(fg::LNT), params, smem, h->stream));
        if (e1) CK(cudaEventRecord(e1, h->stream));
        h->stats.kernel_launches++;
        int64_t *res = a.out; // [cost, children, parents, alg_bytes, ...]
        CK(cudaMemcpyAsync(dst->cost, res + 0, 8, cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaMemcpyAsync(dst->children, res + 1, 8, cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaMemcpyAsync(dst->parents, res + 2, 8, cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaMemcpyAsync(dst->algb, res + 3, 8, cudaMemcpyDeviceToDevice, h->stream));
        if (n1) CK(cudaMemcpyAsync(dst->map, a.map_out, 4 * (size_t)n1, cudaMemcpyDeviceToDevice, h->stream));
        return;
    }
    h->evused = 0;
    cudaEvent_t e0 = next_event(h), e1 = next_event(h);
    // real mode: every rank's home/local initialisation is done before any rank's kernel starts (and,
    // below, every kernel is done before any rank reuses its buffers): an NCCL barrier on the stream
    if (real) nccl_stream_barrier(h);
    CK(cudaEventRecord(h->ev_begin, h->stream));
    CK(cudaEventRecord(e0, h->stream));
    CK(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(fg::LNT), params, smem, h->stream));
    CK(cudaEventRecord(e1, h->stream));
    CK(cudaEventRecord(h->ev_end, h->stream));
    if (real) nccl_stream_barrier(h);
    h->stats.kernel_launches = 1;
    int64_t res[10];
    int32_t xerr = 0;
    CK(cudaMemcpyAsync(res, a.out, 80, cudaMemcpyDefault, h->stream));
    CK(cudaMemcpyAsync(&xerr, a.xerr, 4, cudaMemcpyDeviceToHost, h->stream));
    if (n1) CK(cudaMemcpyAsync(out->mapping, a.map_out, 4 * (size_t)n1, cudaMemcpyDefault, h->stream));
    if (levels_out && n1) CK(cudaMemcpyAsync(levels_out, a.levels_out, 24 * (size_t)n1, cudaMemcpyDefault, h->stream));
    if (real) nccl_stream_wait(h);
    else CK(cudaStreamSynchronize(h->stream));
    if (xerr) fail(FASTGED_ERR_NCCL, "a peer rank did not reach the in-kernel exchange barrier within %.0f s", nccl_timeout_s());
    float ms = 0.f, kms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev_begin, h->ev_end));
    CK(cudaEventElapsedTime(&kms, e0, e1));
    h->stats.device_ms = ms;
    h->stats.branch_ms = kms;
    h->stats.branch_launches = 1;
    h->stats.children_evaluated = res[1];
    h->stats.parents_expanded = res[2];
    h->stats.alg_bytes = res[3];
    h->stats.alg_ops = res[1] * 12; // counters-form lane-ops per child
    for (int x = 0; x < 5; ++x) h->stats.phase_ms[x] = (float)(res[4 + x] * 1e-6);
    h->stats.hist_children = res[9];
    h->stats.d2h_bytes += 32 + 4 * (int64_t)n1;
    out->cost = res[0];
    out->children_evaluated = res[1];
    out->parents_expanded = res[2];
    out->device_ms = ms;
}

#include "editpath.inc"

} // namespace

// ================================================================ C ABI
extern "C" {

const char *fastged_version(void) { return "fastged-b200 0.1 sm_100a"; }

int fastged_nccl_unique_id(uint8_t *out) {
    if (!out) return FASTGED_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return FASTGED_ERR_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out, &id, sizeof id);
    return FASTGED_OK;
}

int fastged_create(const fastged_config_t *cfg, fastged_handle_t **out) {
    g_create_error.clear();
    if (!out) { g_create_error = "out is NULL"; return FASTGED_ERR_ARG; }
    *out = nullptr;
    fastged_handle_t *h = nullptr;
    try {
        if (!cfg) fail(FASTGED_ERR_ARG, "cfg is NULL");
        if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size)
            fail(FASTGED_ERR_ARG, "bad world_size/rank");
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0)
            fail(FASTGED_ERR_CUDA, "no CUDA device available (%s); this library has no CPU path",
                 e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
        if (cfg->device < 0 || cfg->device >= ndev) fail(FASTGED_ERR_ARG, "device %d out of range", cfg->device);
        h = new fastged_handle_t();
        h->device = cfg->device;
        h->flags = cfg->flags;
        h->world = cfg->world_size;
        h->rank = cfg->rank;
        CK(cudaSetDevice(h->device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, h->device));
        if (prop.major < 10) fail(FASTGED_ERR_CUDA, "device %d is sm_%d%d; this build targets sm_100a", h->device, prop.major, prop.minor);
        h->sms = prop.multiProcessorCount;
        h->smem_optin = prop.sharedMemPerBlockOptin;
        if (cfg->stream) h->stream = (cudaStream_t)cfg->stream;
        else {
            CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            h->own_stream = true;
        }
        CK(cudaEventCreate(&h->ev_begin));
        CK(cudaEventCreate(&h->ev_end));
        if (h->world > 1 && !(h->flags & FASTGED_FLAG_VIRTUAL_SHARDS)) {
            if (!cfg->nccl_id) fail(FASTGED_ERR_ARG, "world_size > 1 needs nccl_id (from fastged_nccl_unique_id on rank 0)");
            ncclUniqueId id;
            memcpy(&id, cfg->nccl_id, sizeof id);
            ncclResult_t nr = ncclCommInitRank(&h->comm, h->world, id, h->rank);
            if (nr != ncclSuccess) fail(FASTGED_ERR_NCCL, "ncclCommInitRank failed: %s", ncclGetErrorString(nr));
        }
        *out = h;
        return FASTGED_OK;
    } catch (const FgError &e) {
        g_create_error = e.msg;
        if (h) fastged_destroy(h);
        return e.code;
    } catch (const std::bad_alloc &) {
        g_create_error = "host allocation failed";
        if (h) fastged_destroy(h);
        return FASTGED_ERR_CAPACITY;
    }
}

void fastged_destroy(fastged_handle_t *h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->cstream) cudaStreamSynchronize(h->cstream);
    for (void *p : h->peer_base)
        if (p) cudaIpcCloseMemHandle(p);
    h->peer_base.clear();
    if (h->comm) ncclCommDestroy(h->comm);
    h->xbuf.release();
    h->lblob.release();
    h->lbuf.release();
    free_batch(h->tmp);
    for (fastged_batch *b : h->tmpv) free_batch(b);
    h->tmpv.clear();
    h->scratch.release();
    h->levels.release();
    h->stage.release();
    for (auto e : h->evpool) cudaEventDestroy(e);
    if (h->ev_begin) cudaEventDestroy(h->ev_begin);
    if (h->ev_end) cudaEventDestroy(h->ev_end);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    for (cudaStream_t gs : h->gstreams) cudaStreamDestroy(gs);
    if (h->cstream) {
        cudaStreamSynchronize(h->cstream);
        cudaStreamDestroy(h->cstream);
    }
    for (cudaEvent_t e : h->gevents) cudaEventDestroy(e);
    delete h;
}

const char *fastged_last_error(const fastged_handle_t *h) {
    return h ? h->err.c_str() : g_create_error.c_str();
}

int fastged_get_stats(const fastged_handle_t *h, fastged_stats_t *out) {
    if (!h || !out) return FASTGED_ERR_ARG;
    *out = h->stats;
    return FASTGED_OK;
}

int fastged_batch_upload(fastged_handle_t *h, int32_t npairs, const fastged_graph_t *g1s,
                         const fastged_graph_t *g2s, fastged_batch_t **out) {
    if (!h) return FASTGED_ERR_ARG;
    try {
        if (!out) fail(FASTGED_ERR_ARG, "out is NULL");
        *out = nullptr;
        begin_call(h);
        *out = build_batch(h, npairs, g1s, g2s);
        return FASTGED_OK;
    } catch (const FgError &e) {
        return set_err(h, e);
    } catch (const std::bad_alloc &) {
        return set_err(h, FgError{FASTGED_ERR_CAPACITY, "host allocation failed"});
    }
}

int fastged_batch_run(fastged_handle_t *h, fastged_batch_t *b, const fastged_costs_t *c, int64_t k) {
    if (!h) return FASTGED_ERR_ARG;
    try {
        if (!b) fail(FASTGED_ERR_ARG, "batch is NULL");
        begin_call(h);
        run_batch(h, b, c, k, nullptr);
        return FASTGED_OK;
    } catch (const FgError &e) {
        return set_err(h, e);
    } catch (const std::bad_alloc &) {
        return set_err(h, FgError{FASTGED_ERR_CAPACITY, "host allocation failed"});
    }
}

int fastged_batch_download(fastged_handle_t *h, fastged_batch_t *b, int64_t *costs_out, int32_t *mappings_out,
                           int64_t *children_out) {
    if (!h) return FASTGED_ERR_ARG;
    try {
        if (!b) fail(FASTGED_ERR_ARG, "batch is NULL");
        CK(cudaSetDevice(h->device));
        download(h, b, costs_out, mappings_out, children_out);
        return FASTGED_OK;
    } catch (const FgError &e) {
        return set_err(h, e);
    }
}

void fastged_batch_free(fastged_handle_t *h, fastged_batch_t *b) {
    if (h) {
        cudaSetDevice(h->device);
        if (h->stream) cudaStreamSynchronize(h->stream);
        if (h->cstream) cudaStreamSynchronize(h->cstream);
    }
    free_batch(b);
}

int fastged_solve_batch(fastged_handle_t *h, int32_t npairs, const fastged_graph_t *g1s,
                        const fastged_graph_t *g2s, const fastged_costs_t *c, int64_t k, int64_t *costs_out,
                        int32_t *mappings_out, int64_t *children_out) {
    if (!h) return FASTGED_ERR_ARG;
    try {
        begin_call(h);
        validate_costs(c);
        if (k < 1) fail(FASTGED_ERR_ARG, "k < 1");
        if (!h->tmp) h->tmp = new fastged_batch();
        // Pipelined chunks of doubling size: the GPU starts on a small first chunk while the host
        // validates and packs the next one (host packing is about twice as fast as the search, so the
        // GPU is not starved after the first chunk).  Same stream: every chunk's copies and kernels
        // queue behind the previous one's.  Pairs are independent: chunking changes no result.
        std::vector<std::pair<int32_t, int32_t>> cuts; // (first pair, count)
        {
            // first chunk npairs / div, then growth x g (tuning knobs FASTGED_PIPE_DIV / FASTGED_PIPE_GROWTH)
            static const int div = [] { const char *e = getenv("FASTGED_PIPE_DIV"); return e ? std::max(1, atoi(e)) : 16; }();
            static const double grow = [] { const char *e = getenv("FASTGED_PIPE_GROWTH"); return e ? std::max(1.1, atof(e)) : 2.0; }();
            int32_t start = 0;
            double szd = npairs >= PIPELINE_MIN_PAIRS ? std::max<double>(npairs / div, 256) : npairs;
            while (start < npairs) {
                const int32_t sz = (int32_t)std::max(1.0, szd);
                int32_t n = std::min<int32_t>(sz, npairs - start);
                if (npairs - start - n < sz / 2) n = npairs - start; // no small tail chunk
                cuts.push_back({start, n});
                start += n;
                szd *= grow;
            }
            if (cuts.empty()) cuts.push_back({0, 0});
        }
        std::vector<fastged_batch *> bs;
        for (size_t ci = 0; ci < cuts.size(); ++ci) {
            fastged_batch *reuse;
            if (ci == 0) reuse = h->tmp;
            else {
                while (h->tmpv.size() < ci) h->tmpv.push_back(new fastged_batch());
                reuse = h->tmpv[ci - 1];
            }
            fastged_batch *b = build_batch(h, cuts[ci].second, g1s + cuts[ci].first, g2s + cuts[ci].first, reuse,
                                           cuts[ci].first);
            run_batch(h, b, c, k, nullptr, ci == 0);
            bs.push_back(b);
        }
        int64_t map_total = 0;
        for (fastged_batch *b : bs) map_total += b->total_map;
        if (npairs > 0 && !costs_out) fail(FASTGED_ERR_ARG, "costs_out is NULL");
        if (map_total > 0 && !mappings_out) fail(FASTGED_ERR_ARG, "mappings_out is NULL");
        for (fastged_batch *b : bs) download_enqueue(h, b);
        CK(cudaStreamSynchronize(h->stream));
        finish_timing(h);
        int64_t moff = 0;
        for (size_t ci = 0; ci < bs.size(); ++ci) {
            const int32_t st0 = cuts[ci].first;
            download_collect(h, bs[ci], costs_out ? costs_out + st0 : nullptr, mappings_out ? mappings_out + moff : nullptr,
                             children_out ? children_out + st0 : nullptr);
            moff += bs[ci]->total_map;
        }
        return FASTGED_OK;
    } catch (const FgError &e) {
        cudaStreamSynchronize(h->stream);
        return set_err(h, e);
    } catch (const std::bad_alloc &) {
        cudaStreamSynchronize(h->stream);
        return set_err(h, FgError{FASTGED_ERR_CAPACITY, "host allocation failed"});
    }
}

int fastged_solve_pair_ex(fastged_handle_t *h, const fastged_graph_t *g1, const fastged_graph_t *g2,
                          const fastged_costs_t *c, int64_t k, fastged_result_t *out, int64_t *levels_out) {
    if (!h) return FASTGED_ERR_ARG;
    fastged_batch *b = nullptr;
    try {
        begin_call(h);
        if (!out) fail(FASTGED_ERR_ARG, "out is NULL");
        validate_costs(c);
        if (k < 1) fail(FASTGED_ERR_ARG, "k < 1");
        validate_graph(g1, 0, "g1");
        validate_graph(g2, 0, "g2");
        check_overflow(g1, g2, c, 0);
        if (g1->n > 0 && !out->mapping) fail(FASTGED_ERR_ARG, "out->mapping is NULL");
        if (h->world > 1) {
            solve_sharded(h, g1, g2, c, k, out, levels_out);
            return FASTGED_OK;
        }
        if (!fits_batched(g1->n, g2->n, k, labelled_pair(g1, g2) ? g2_label_count(g2) : 0) ||
            (h->flags & (FASTGED_FLAG_FORCE_LARGE | FASTGED_FLAG_APPROX_MASK)) ||
            prefers_whole_gpu(g1->n, g2->n, k, 1)) {
            solve_large(h, g1, g2, c, k, out, levels_out);
            return FASTGED_OK;
        }
        if (!h->tmp) h->tmp = new fastged_batch();
        b = build_batch(h, 1, g1, g2, h->tmp);
        int64_t *lev = nullptr;
        if (levels_out && g1->n > 0) {
            CK(h->levels.reserve(24 * (size_t)g1->n));
            lev = (int64_t *)h->levels.p;
        }
        run_batch(h, b, c, k, lev);
        int64_t cost = 0, ch = 0;
        download(h, b, &cost, out->mapping, &ch);
        if (lev) CK(cudaMemcpy(levels_out, lev, 24 * (size_t)g1->n, cudaMemcpyDeviceToHost));
        out->cost = cost;
        out->children_evaluated = h->stats.children_evaluated;
        out->parents_expanded = h->stats.parents_expanded;
        out->device_ms = h->stats.device_ms;
        return FASTGED_OK;
    } catch (const FgError &e) {
        if (b) cudaStreamSynchronize(h->stream);
        return set_err(h, e);
    } catch (const std::bad_alloc &) {
        if (b) cudaStreamSynchronize(h->stream);
        return set_err(h, FgError{FASTGED_ERR_CAPACITY, "host allocation failed"});
    }
}

int fastged_edit_path(const fastged_graph_t *g1, const fastged_graph_t *g2, const fastged_costs_t *c,
                      const int32_t *mapping, fastged_edit_op_t *ops, int32_t max_ops, int32_t *n_ops_out,
                      int64_t *cost_out) {
    g_create_error.clear();
    try {
        if (!n_ops_out || !cost_out) fail(FASTGED_ERR_ARG, "n_ops_out / cost_out is NULL");
        validate_costs(c);
        validate_graph(g1, 0, "g1");
        validate_graph(g2, 0, "g2");
        check_mapping(g1, g2, mapping);
        const std::vector<fastged_edit_op_t> v = edit_ops(g1, g2, c, mapping);
        int64_t tot = 0;
        for (const auto &o : v) tot += o.cost;
        *n_ops_out = (int32_t)v.size();
        *cost_out = tot;
        if (ops) {
            if ((int64_t)v.size() > max_ops) fail(FASTGED_ERR_ARG, "ops capacity %d < %zu operations", max_ops, v.size());
            std::copy(v.begin(), v.end(), ops);
        }
        return FASTGED_OK;
    } catch (const FgError &e) {
        g_create_error = e.msg;
        return e.code;
    } catch (...) {
        g_create_error = "host allocation failed";
        return FASTGED_ERR_CAPACITY;
    }
}

int fastged_apply_edit_path(const fastged_graph_t *g1, const fastged_graph_t *g2, const int32_t *mapping,
                            int32_t prefix_len, int32_t *n_out, int32_t *vlabels_out, int32_t *origin_out,
                            int32_t *m_out, int32_t *edges_out, int32_t *elabels_out) {
    g_create_error.clear();
    try {
        if (!n_out || !m_out || !vlabels_out || !origin_out || !edges_out || !elabels_out)
            fail(FASTGED_ERR_ARG, "an output is NULL");
        validate_graph(g1, 0, "g1");
        validate_graph(g2, 0, "g2");
        check_mapping(g1, g2, mapping);
        const int n1 = g1->n, n2 = g2->n;
        std::vector<char> used((size_t)std::max(n2, 1), 0);
        for (int i = 0; i < n1; ++i)
            if (mapping[i] >= 0) used[mapping[i]] = 1;
        std::vector<int> ins;
        for (int u = 0; u < n2; ++u)
            if (!used[u]) ins.push_back(u);
        if (prefix_len < 0 || prefix_len > n1 + (int)ins.size())
            fail(FASTGED_ERR_ARG, "prefix_len %d outside 0..%d", prefix_len, n1 + (int)ins.size());
        const int res = std::min(prefix_len, n1);                // v_0 .. v_{res-1} are resolved
        const int nins = std::max(0, prefix_len - n1);           // the first nins insertions are applied
        DenseGraph A, B;
        A.build(g1);
        B.build(g2);
        std::vector<int> id1((size_t)std::max(n1, 1), -1);       // output id of g1 vertex i (or -1: deleted)
        int n = 0;
        for (int i = 0; i < n1; ++i) {
            if (i < res && mapping[i] < 0) continue;
            id1[i] = n;
            vlabels_out[n] = i < res ? g2->vlabels[mapping[i]] : g1->vlabels[i];
            origin_out[n] = i < res ? mapping[i] : -1 - i;
            ++n;
        }
        std::vector<int> g1of((size_t)n, -1); // g1 index of output vertex v (surviving g1 vertices)
        for (int i = 0; i < n1; ++i)
            if (id1[i] >= 0) g1of[id1[i]] = i;
        std::vector<int> idi(ins.size(), -1);
        for (int x = 0; x < nins; ++x) {
            idi[x] = n;
            vlabels_out[n] = g2->vlabels[ins[x]];
            origin_out[n] = ins[x];
            ++n;
        }
        int m = 0;
        auto add = [&](int a, int b, int32_t l) {
            edges_out[2 * m] = std::min(a, b);
            edges_out[2 * m + 1] = std::max(a, b);
            elabels_out[m] = l;
            ++m;
        };
        for (int a = 0; a < n; ++a)
            for (int b = a + 1; b < n; ++b) {
                const bool ra = origin_out[a] >= 0, rb = origin_out[b] >= 0;
                if (ra && rb) { // both resolved or inserted: the g2 state
                    const int32_t l = B.at(origin_out[a], origin_out[b]);
                    if (l >= 0) add(a, b, l);
                } else { // at least one unresolved g1 vertex: the g1 edge (resolved later)
                    // g1 indices (a resolved endpoint is a g1 vertex here: insertions only follow v_{n1-1})
                    const int qa = a < (int)g1of.size() ? g1of[a] : -1, qb = b < (int)g1of.size() ? g1of[b] : -1;
                    if (qa >= 0 && qb >= 0) {
                        const int32_t l = A.at(qa, qb);
                        if (l >= 0) add(a, b, l);
                    }
                }
            }
        *n_out = n;
        *m_out = m;
        return FASTGED_OK;
    } catch (const FgError &e) {
        g_create_error = e.msg;
        return e.code;
    } catch (...) {
        g_create_error = "host allocation failed";
        return FASTGED_ERR_CAPACITY;
    }
}

int fastged_graphs_equal_under_mapping(const fastged_graph_t *a, const fastged_graph_t *b, const int32_t *mapping) {
    g_create_error.clear();
    try {
        validate_graph(a, 0, "a");
        validate_graph(b, 0, "b");
        if (a->n != b->n) fail(FASTGED_ERR_INPUT, "not a bijection: %d vs %d vertices", a->n, b->n);
        if (a->n > 0 && !mapping) fail(FASTGED_ERR_ARG, "mapping is NULL");
        std::vector<char> seen((size_t)std::max(b->n, 1), 0);
        for (int v = 0; v < a->n; ++v) {
            if (mapping[v] < 0 || mapping[v] >= b->n || seen[mapping[v]]) fail(FASTGED_ERR_INPUT, "mapping is not a bijection");
            seen[mapping[v]] = 1;
        }
        for (int v = 0; v < a->n; ++v)
            if (a->vlabels[v] != b->vlabels[mapping[v]]) return 0;
        if (a->m != b->m) return 0;
        DenseGraph B;
        B.build(b);
        for (int e = 0; e < a->m; ++e) {
            const int x = mapping[a->edges[2 * e]], y = mapping[a->edges[2 * e + 1]];
            const int32_t la = a->elabels ? a->elabels[e] : 0;
            if (B.at(x, y) != la) return 0;
        }
        return 1;
    } catch (const FgError &e) {
        g_create_error = e.msg;
        return -e.code;
    }
}

int fastged_solve_pair(fastged_handle_t *h, const fastged_graph_t *g1, const fastged_graph_t *g2,
                       const fastged_costs_t *c, int64_t k, fastged_result_t *out) {
    return fastged_solve_pair_ex(h, g1, g2, c, k, out, nullptr);
}

} // extern "C"
