// large_kernel.cuh -- one large (g1, g2) pair on the whole GPU: a persistent cooperative kernel
// runs every level of Alg. 1 with grid-wide phases and no host round trip
// ("avoiding any host-device communication").  Used for n2 > 128 or very large K
// (BASELINE configs[3]: n = 200-500, K = 1e4-1e5).
//
// Node state in HBM (row-major, double-buffered by level parity): used[k][W] uint32 (bit u: g2
//   vertex u is used), lambda map[k][n1s] (uint8, or uint16 when n2 > 254; all-ones = deleted), and
//   the counters cnt[k][cs] (uint8, or uint16 when a g2 degree exceeds 255): cnt[k][u] = number of
//   used g2 neighbours of u (the "counters" formulation of SURVEY.md §8(a) a1).  A child's counters
//   are its parent's plus the adjacency row of its target, so the per-child O(W) popcount for
//   cnt_p(u) becomes one byte load.  The survivors of a level are kept as descriptors
//   sel[k] = (parent position p, target j, PED); their rows are materialised by the next level's
//   branch step, which reads the parent's row once and both writes the child's row and expands it
//   (the paper's update/copy_kernel, fused into the following branch).
//
// Per level i (g1 vertex v_i):
//   A  materialise + branch (Alg. 2): a warp per parent (taken
//      dynamically inside the CTA's range, rows prefetched with cp.async), lane l owns the targets
//      u = 128 s + 4 l + b.  Child PED of the paper's incremental evaluation with the three
//      implied-edge cases of P:103-116 regrouped as
//          Delta(u)   = cv(i,u) + edel*d_i + eins*cnt_p(u) - (edel+eins)*cB_p(u) + esub*mis_p(u)
//          Delta(DEL) = vdel + edel*d_i
//      cB_p(u) = number of earlier g1 neighbours v_q of v_i whose image lambda_p(q) is adjacent to u
//      (the paper's VFrom/VTo, reading C8).  Two ways to get it, chosen per level by cost:
//        scatter: walk the neighbour lists of the images (CSR) and add into a per-warp array D[u]
//                 (also yields mis_p for labelled edges);
//        popcount: B_p as a bitmask, popc(adj2[u] & B_p) over the nonzero words of B_p.
//      Each child becomes a one-byte rank code (PED - base + 1, saturated) in HBM; codes that can be
//      selected (PED <= U_i, the bound of SURVEY.md §8(a) a2) go into a per-lane-column shared
//      histogram (no intra-warp address conflicts), merged with one global atomic per nonzero bin.
//   T  every CTA reads the global histogram and derives the same threshold t and tie quota r
//      (replaces the paper's local/global ranking with atomics; exact, reading C12).
//   B  per-warp counts of codes < t / == t (SWAR over 16-byte vectors).
//   C1 survivors compacted in (parent, child) order (reading C13) into sel with their PEDs; 16-byte
//      code vectors without a survivor are skipped.
// After the last level: insertion completion (reading C6) and argmin by (total, position)
// (reading C10).
#pragma once
#include <cooperative_groups.h>

#include <cstdint>
#include <type_traits>

#include "batch_kernel.cuh"

namespace fg {
namespace cg = cooperative_groups;

#ifndef FG_LNT
#define FG_LNT 736
#endif
constexpr int LNT = FG_LNT; // threads per CTA of the large kernel (one CTA per SM)
#ifndef FG_LARGE_ALIGNED_BARRIER
#define FG_LARGE_ALIGNED_BARRIER 1
#endif
__device__ __forceinline__ void lsync() {
#if FG_LARGE_ALIGNED_BARRIER
    block_sync_aligned();
#else
    block_sync();
#endif
}
#ifndef FG_C1_LIGHT
#define FG_C1_LIGHT 8 // C1: rows with at most this many survivors are emitted lane per row
#endif
#ifndef FG_LPF
#define FG_LPF 2
#endif
constexpr int LPF = FG_LPF;   // per-warp prefetch ring: the next parent's rows in flight while one is expanded
constexpr int LMAXGRID = 256; // CTAs of the large kernel per rank (one per SM)
#ifndef FG_MAXG
#define FG_MAXG 8 // ranks of the sharded single-pair mode (one 8-GPU node)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cpa4(void *sdst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa16(void *sdst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename MapT>
struct MapDel { static constexpr int value = (int)(MapT)(~(MapT)0); };

// Four consecutive counters (targets u..u+3) as one vector.
template <typename CntT>
struct Cnt4;
template <>
struct Cnt4<uint8_t> {
    using V = uint32_t;
    static __device__ __forceinline__ V load(const uint8_t *row, int u) { return *reinterpret_cast<const uint32_t *>(row + u); }
    static __device__ __forceinline__ void store(uint8_t *row, int u, V v) { *reinterpret_cast<uint32_t *>(row + u) = v; }
    static __device__ __forceinline__ int get(V v, int b) { return (int)((v >> (8 * b)) & 0xffu); }
    // add bit b of nib to counter b (bits spread to bytes 0..3; no carries between the partial products)
    static __device__ __forceinline__ V add_bits(V v, uint32_t nib) { return v + ((nib * 0x204081u) & 0x01010101u); }
};
template <>
struct Cnt4<uint16_t> {
    using V = uint2;
    static __device__ __forceinline__ V load(const uint16_t *row, int u) { return *reinterpret_cast<const uint2 *>(row + u); }
    static __device__ __forceinline__ void store(uint16_t *row, int u, V v) { *reinterpret_cast<uint2 *>(row + u) = v; }
    static __device__ __forceinline__ int get(V v, int b) {
        const uint32_t w = b < 2 ? v.x : v.y;
        return (int)((w >> (16 * (b & 1))) & 0xffffu);
    }
    static __device__ __forceinline__ V add_bits(V v, uint32_t nib) {
        v.x += (nib & 1u) | ((nib & 2u) << 15);
        v.y += ((nib >> 2) & 1u) | ((nib & 8u) << 13);
        return v;
    }
};

// SWAR byte compares (unsigned, any byte values): bit 7 of each byte set where the predicate holds.
__device__ __forceinline__ uint32_t bytes_lt(uint32_t x, uint32_t y) {
    const uint32_t z = (x | 0x80808080u) - (y & 0x7f7f7f7fu); // bit 7: low 7 bits of x >= those of y
    return ((~x & y) | (~(x ^ y) & ~z)) & 0x80808080u;
}
__device__ __forceinline__ uint32_t bytes_eq(uint32_t x, uint32_t y) {
    const uint32_t z = x ^ y;
    return ~((((z & 0x7f7f7f7fu) + 0x7f7f7f7fu) | z)) & 0x80808080u;
}

struct LargeArgs {
    const uint8_t *blob;
    PairDesc pd;
    Costs c;
    int32_t K, win, W;
    int32_t ashift;         // method variant (NEXT-4): approximate top-K with PED bins of 2^ashift (0 = exact)
    int32_t last_by_total;  // method variant (NEXT-4, reading C10 alternative): the last level ranked by PED + completion
    int32_t cs, S;          // row stride of codes / counters (multiple of 128 >= n2 + 1); S = cs / 128
    int32_t n1s;            // lambda row stride in elements (4-byte multiple)
    int32_t n1r;            // staged P_i list capacity in shared memory (>= max d, multiple of 4)
    int32_t nwa;            // warps per CTA with a branch region (shared-memory bound, <= LNT / 32)
    int32_t adjT_in_smem;   // transposed adjacency adjT[W][cs] staged in shared memory
    int32_t csr_in_smem;    // CSR (nptr, nbr) staged in shared memory
    int32_t csz;            // bytes per counter (1 or 2)
    int32_t degw;           // ceil(mean g2 degree / 32): scatter-cost estimate
    const int32_t *nptr;    // CSR of g2: [n2 + 1]
    const uint32_t *nbr;    // [2 m2]: neighbour | (edge label id << 16)
    const uint32_t *adjT;   // [W][cs]: bit (u' & 31) of adjT[w][u] = edge (u, 32 w + u')
    // Frontier sharding.  The G ranks hold contiguous, equal
    // slices of every level's frontier: rank r owns the global positions [N r / G, N (r+1) / G).
    // A node's rows live on its owner; a child whose parent lives on another rank reads the parent's
    // rows through a peer pointer (NVLink), and the descriptors of the next level are written straight
    // into the owner's arrays.  Histogram, counts, PED range and argmin go to the home arrays (rank 0's
    // memory).  G = 1 is the single-GPU kernel.  virt: the G ranks are equal CTA groups of this one
    // grid (one GPU; the exchange protocol is the same, only the barrier differs).
    int32_t G, rank, virt;
    int32_t nb;                 // CTAs per rank
    int32_t kl;                 // rows per rank buffer (debug bound checks)
    struct Rank {
        int32_t *ped[2];        // [Kl]      PED of the nodes of a level
        uint32_t *used[2];      // [Kl][W]   rows of the nodes of level L live in buffer L & 1
        void *cnt[2];           // [Kl][cs] CntT
        void *map[2];           // [Kl][n1s] MapT
        uint8_t *ccode;         // [Kl][cs] candidate list of the row, in target order: rank codes
        uint16_t *ctgt;         // [Kl][cs]                                          and targets
        int32_t *rown;          // [Kl] entries in the row's candidate list
        int32_t *sel_p, *sel_j, *sel_ped; // nodes of the next level: parent row on its rank; target
                                          // (n2 = deletion, -1 = root; int16) | parent's rank << 16; PED
        int32_t *rowc;          // [Kl] per parent row: (codes < t) | (codes == t) << 16
        int32_t *rowpl, *rowpe; // [Kl] codes < t / == t in the rows of the same B range before this row
        int32_t *rowmin;        // [Kl] smallest rank code of the row (A): B reads only rows that can hold survivors
        int32_t *wlt, *weq;     // [warps of the rank] codes < t / == t in the CTA's B ranges before this warp's
    };
    const Rank *rk;             // [G] (device memory), indexed by rank; other ranks' arrays are peer-mapped
    Rank self;                  // this rank's arrays (virtual mode: rank 0's; rank r's are at + r vstride bytes)
    int64_t vstride;
    // home arrays (rank 0)
    int32_t *hist;          // [3][256] rotating global histograms
    int64_t *ci;            // [n1] candidates per level
    int32_t *drop;          // [n1] nonzero: a valid child was left out of the candidate lists
    int32_t *lo, *hi;       // [n1 + 1] min / max survivor PED per level (init INT_MAX / INT_MIN)
    int32_t *ctl, *cte;     // [G * CTAs per rank] codes < t / == t per CTA
    unsigned long long *best;
    unsigned int *bar;      // cross-rank barrier counter (real multi-GPU mode)
    int32_t *xerr;          // this rank's own flag: a peer missed a barrier for xtimeout_ns (the kernel returns)
    int64_t xtimeout_ns;
    int64_t *out;           // [0] cost, [1] children, [2] parents, [3] algorithmic bytes,
                            // [4..8] ns in phases A+T, B, C1, -, finalize (CTA 0's clock),
                            // [9] children that entered the rank histogram
    int32_t *map_out;       // [n1]
    int64_t *levels_out;    // NULL or [3 n1]
};

// Per-warp shared region (32-bit words): sB[32], D[cs], then LPF prefetch buffers of
// counters[cs * csz / 4], used[32], lambda row [n1s * esz / 4], descriptor (k, p, j, ped)[4].
__host__ __device__ inline int large_pf_words(int cs, int csz, int n1s, int esz) { // multiple of 4 (16-byte copies)
    return ((cs * csz / 4 + 32 + n1s * esz / 4 + 4) + 3) & ~3;
}
__host__ __device__ inline int large_warp_words(int cs, int csz, int n1s, int esz) {
    return 32 + cs + LPF * large_pf_words(cs, csz, n1s, esz);
}
// Shared-memory bytes of the large kernel (must match the carve-up in the kernel).
__host__ __device__ inline size_t large_smem_bytes(int cs, int csz, int n1s, int esz, int nwa, int n1r, int W, int n2,
                                                   int nnbr, bool adjT_in_smem, bool csr_in_smem) {
    return (size_t)256 * 32 * 4 + (size_t)2 * n1r * 4 + (size_t)nwa * large_warp_words(cs, csz, n1s, esz) * 4 +
           (adjT_in_smem ? (size_t)W * cs * 4 : 0) + (csr_in_smem ? (size_t)4 * (((n2 + 4) & ~3) + nnbr) : 0);
}

// PED of child (parent row k, target j) from scratch over P_i (rare: saturated rank codes).
template <typename MapT, typename CntT, bool LAB>
__device__ int large_child_scalar(const LargeArgs &a, int d, const int32_t *pq, const int32_t *pl, int pedp,
                                  const CntT *crow, const MapT *mrow, int j, const uint32_t *adj2,
                                  const uint8_t *e2, int vl1i, const int32_t *vl2) {
    const Costs &c = a.c;
    const int n2 = a.pd.n2, W = a.W;
    if (j == n2) return pedp + c.vdel + c.edel * d;
    const int cv = (vl2[j] == vl1i) ? 0 : c.vsub;
    const int cnt = (int)crow[j];
    int cb = 0, mis = 0;
    for (int k = 0; k < d; ++k) {
        const int t = mrow[pq[k]];
        if (t == MapDel<MapT>::value) continue;
        if (!LAB) cb += (adj2[(int64_t)j * W + (t >> 5)] >> (t & 31)) & 1u;
        else {
            const int e = e2[(int64_t)t * a.pd.n2p + j];
            cb += (e != 0);
            mis += (e != 0) & (e != pl[k]);
        }
    }
    return pedp + cv + c.edel * d + c.eins * cnt - (c.edel + c.eins) * cb + c.esub * mis;
}

template <typename T>
__device__ __forceinline__ T *fg_loc(T *p, int64_t off) { return reinterpret_cast<T *>(reinterpret_cast<char *>(p) + off); }

#ifdef FG_DEBUG_CHECKS
// debug builds only: a violated bound is reported once and counted (tests then see wrong results)
__device__ unsigned int fg_dbg_bad;
#define FG_CHECK(cond, ...) do { if (!(cond)) { if (atomicAdd(&fg_dbg_bad, 1u) == 0) printf(__VA_ARGS__); } } while (0)
#else
#define FG_CHECK(cond, ...) do { } while (0)
#endif
#ifdef FG_LSTAT
__device__ unsigned long long fg_lstat[2];
#endif
// SHARD = 0: one GPU (G = 1); every sharding quantity folds to a constant, so the single-GPU kernel carries
// no register cost for the sharded mode.  SHARD = 1: one rank per GPU (the rank from the parameters, the own
// arrays at fixed addresses).  SHARD = 2: virtual ranks = CTA groups of this grid (rank, CTA index and the
// own arrays' offset from shared memory).
template <typename MapT, typename CntT, bool LAB, int SHARD>
__global__ void __launch_bounds__(LNT, 1) kbest_large_kernel(const LargeArgs a) {
    extern __shared__ __align__(16) uint8_t dsmem[];
    constexpr int NWB = LNT / 32;
    constexpr int ESZ = (int)sizeof(MapT);
    __shared__ int s_pre[2];
    __shared__ int s_red[2][NWB];
    __shared__ int s_cpre[2][LMAXGRID]; // exclusive prefix of the per-CTA counts
    __shared__ long long s_cnt;
    __shared__ int s_next; // A: next parent of this CTA's range (warps take parents dynamically)
    __shared__ int s_drop; // A: a child of this CTA was left out of the candidate lists
    __shared__ LargeArgs::Rank s_rk[FG_MAXG]; // the ranks' array pointers (a.rk), dynamically indexed
    cg::grid_group grid = cg::this_grid();
    using C4 = Cnt4<CntT>;

    // rank of this CTA and its index among the rank's CTAs (virtual mode: equal CTA groups).  Kept in
    // shared memory and re-read where used (volatile): the branch loop's registers are all taken.
    __shared__ int s_rank, s_lb;
    __shared__ long long s_roff;
    __shared__ unsigned int s_xepoch;
    const int G = SHARD ? a.G : 1, nb = SHARD ? a.nb : (int)gridDim.x;
    if (threadIdx.x == 0) {
        const int r = a.virt ? (int)blockIdx.x / nb : a.rank;
        s_rank = r;
        s_lb = a.virt ? (int)blockIdx.x % nb : (int)blockIdx.x;
        // this rank's own arrays: kernel parameters, offset by the rank's block in virtual mode
        s_roff = a.virt ? (long long)r * a.vstride : 0;
        s_xepoch = 0;
    }
    if (SHARD)
        for (int x = threadIdx.x; x < G * (int)(sizeof(LargeArgs::Rank) / 8); x += LNT)
            reinterpret_cast<unsigned long long *>(s_rk)[x] = reinterpret_cast<const unsigned long long *>(a.rk)[x];
    lsync();
#define RANK (SHARD == 2 ? s_rank : (SHARD == 1 ? a.rank : 0))
#define LB (SHARD == 2 ? s_lb : (int)blockIdx.x)
#define ML(f) (SHARD == 2 ? fg_loc(a.self.f, s_roff) : a.self.f)
    // field f of rank r's arrays (a peer's memory when sharded)
#define RK(r, f) (SHARD ? s_rk[r].f : a.self.f)
    // the one CTA that writes the home-only outputs
    auto home0 = [&]() { return RANK == 0 && LB == 0; };
    // slice of a level of n nodes owned by rank r: [rstart(n, r), rstart(n, r + 1)); owner of position k
    auto rstart = [&](int n, int r) -> int { return (int)(((int64_t)n * r) / G); };
    auto rowner = [&](int k, int n) -> int { return G == 1 ? 0 : (int)((((int64_t)k + 1) * G - 1) / n); };
    // a descriptor's target and the rank holding its parent's row
    auto dtarget = [](int32_t v) -> int { return (int)(int16_t)(v & 0xffff); };
    auto drank = [](int32_t v) -> int { return (int)((uint32_t)v >> 16); };
    // barrier over every CTA of every rank.  Virtual ranks share the grid; real ranks (one GPU each)
    // meet at a counter in rank 0's memory after their own grid barrier (system-scope release/acquire:
    // the remote descriptor writes and home atomics of every CTA are visible past it)
    // Returns false (on every CTA of the rank) when a peer did not arrive within xtimeout_ns.
    auto xsync = [&]() -> bool {
        if (SHARD == 1 && G > 1) __threadfence_system();
        lsync();
        grid.sync();
        if (SHARD == 1 && G > 1) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                const unsigned xepoch = (s_xepoch += (unsigned)G);
                atomicAdd_system(a.bar, 1u);
                uint64_t t0, t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                for (;;) {
                    unsigned v;
                    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
                    if ((int)(v - xepoch) >= 0) break;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if ((int64_t)(t - t0) > a.xtimeout_ns) { *(volatile int32_t *)a.xerr = 1; break; }
                    __nanosleep(256);
                }
            }
            lsync();
            grid.sync();
            return *(volatile int32_t *)a.xerr == 0;
        }
        return true;
    };

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gw = LB * NWB + wib, GW = nb * NWB; // warps of this rank
    const Costs c = a.c;
    const PairDesc pd = a.pd;
    const int n1 = pd.n1, n2 = pd.n2, W = a.W, K = a.K, win = a.win, cs = a.cs, S = a.S;
    constexpr int DELV = MapDel<MapT>::value;
    const int32_t *vl1 = reinterpret_cast<const int32_t *>(a.blob + pd.vl1);
    const int32_t *vl2 = reinterpret_cast<const int32_t *>(a.blob + pd.vl2);
    const int32_t *pptr = reinterpret_cast<const int32_t *>(a.blob + pd.pptr);
    const int32_t *pqg = reinterpret_cast<const int32_t *>(a.blob + pd.pq);
    const int32_t *plg = reinterpret_cast<const int32_t *>(a.blob + pd.pl);
    const uint32_t *adj2 = reinterpret_cast<const uint32_t *>(a.blob + pd.adj2);
    const uint8_t *e2 = LAB ? (a.blob + pd.e2lab) : nullptr;
    const int rowwords = a.n1s * ESZ / 4;

    // shared: per-lane-column histogram [256][32], the P_i list, per-warp regions, adjT, CSR
    int *s_hist = reinterpret_cast<int *>(dsmem);
    int32_t *s_pq = s_hist + 256 * 32;
    int32_t *s_pl = s_pq + a.n1r;
    uint32_t *wbase = reinterpret_cast<uint32_t *>(s_pl + a.n1r);
    const int WWORDS = large_warp_words(cs, a.csz, a.n1s, ESZ), PFW = large_pf_words(cs, a.csz, a.n1s, ESZ);
    const int CNTW = cs * a.csz / 4;
    const bool brancher = wib < a.nwa;
    uint32_t *sB = wbase + wib * WWORDS;
    int *D = reinterpret_cast<int *>(sB + 32);
    uint32_t *pfb = sB + 32 + cs;
    uint32_t *after = wbase + a.nwa * WWORDS;
    const uint32_t *adjT = a.adjT;
    if (a.adjT_in_smem) {
        for (int x = threadIdx.x; x < W * cs; x += LNT) after[x] = __ldg(a.adjT + x);
        adjT = after;
        after += W * cs;
    }
    const int32_t *nptr = a.nptr;
    const uint32_t *nbr = a.nbr;
    if (a.csr_in_smem) {
        const int np = (n2 + 4) & ~3, nn = 2 * pd.m2;
        int32_t *sp = reinterpret_cast<int32_t *>(after);
        for (int x = threadIdx.x; x <= n2; x += LNT) sp[x] = __ldg(a.nptr + x);
        for (int x = threadIdx.x; x < nn; x += LNT) after[np + x] = __ldg(a.nbr + x);
        nptr = sp;
        nbr = after + np;
    }
    if (brancher)
        for (int x = lane; x < cs; x += 32) D[x] = 0;
    auto adjw = [&](int j, int w) -> uint32_t { // word w of g2's bit row j
        return a.adjT_in_smem ? adjT[w * cs + j] : __ldg(adj2 + (int64_t)j * W + w);
    };
    // root: lambda empty, nothing used, PED 0 -- row 0 of level -1 (buffer 1), and the
    // descriptor of the level-0 node; both live on the owner of position 0 of a one-node level
    if (RANK == rowner(0, 1) && LB == 0) {
        if (threadIdx.x == 0) { ML(sel_p)[0] = 0; ML(sel_j)[0] = 0xffff | (RANK << 16); ML(sel_ped)[0] = 0; }
        for (int w = threadIdx.x; w < W; w += LNT) ML(used[1])[w] = 0u;
        for (int u = threadIdx.x; u < cs; u += LNT) reinterpret_cast<CntT *>(ML(cnt[1]))[u] = 0;
    }
    if (!xsync()) return;

    int N = 1, lo = 0, hi = 0, ps = 0;
    int64_t children = 0, parents = 0, algb = 0;
    int64_t tph[5] = {0, 0, 0, 0, 0}, nhist = 0;
    uint64_t tlast = 0;
    auto tick = [&](int ph) { // phase clock (thread 0 of CTA 0, after a grid barrier)
        if (home0() && threadIdx.x == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (ph >= 0) tph[ph] += (int64_t)(t - tlast);
            tlast = t;
        }
    };
    tick(-1);
    for (int i = 0; i < n1; ++i) {
        const int pv = (i + 1) & 1, cu = i & 1; // buffers of level i-1 (the parents' parents) and level i
        // this rank's nodes of level i: global positions [s0, s0 + Nl), local rows 0..Nl-1
        const int s0 = rstart(N, RANK), Nl = rstart(N, RANK + 1) - s0;
        uint32_t *Qused = ML(used[cu]);
        CntT *Qcnt = reinterpret_cast<CntT *>(ML(cnt[cu]));
        MapT *Qmap = reinterpret_cast<MapT *>(ML(map[cu]));
        const int pbeg = __ldg(pptr + i), d = __ldg(pptr + i + 1) - pbeg;
        for (int k = threadIdx.x; k < d; k += LNT) {
            s_pq[k] = __ldg(pqg + pbeg + k);
            s_pl[k] = __ldg(plg + pbeg + k);
        }
        const int vl1i = __ldg(vl1 + i);
        uint64_t mm = 0; // vertex-label mismatch of the lane's targets: bit 4 s + b for u = 128 s + 4 lane + b
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int u = 128 * s + 4 * lane + b;
                if (u < n2 && __ldg(vl2 + u) != vl1i) mm |= 1ull << (4 * s + b);
            }
        const int edd = c.edel * d, ee = c.edel + c.eins, pedDel = c.vdel + edd;
        // cB by scatter over neighbour lists, or by popcount over the nonzero words of B_p (uniform choice)
#ifndef FG_SCATTER_RATIO
#define FG_SCATTER_RATIO 13 // scatter when d * ceil(deg / 32) * 8 < S * min(W, d) * FG_SCATTER_RATIO
#endif
        const bool scatter = LAB || (d * a.degw * 8 < S * min(W, d) * FG_SCATTER_RATIO);
        const int chunk = (Nl + GW - 1) / GW; // B / C1: static contiguous code ranges per warp (local rows)
        const int p0 = min(Nl, gw * chunk), p1 = min(Nl, p0 + chunk);
        const int cchunk = (Nl + nb - 1) / nb; // A: this CTA's parents, taken dynamically
        const int cb0 = min(Nl, LB * cchunk), cb1 = min(Nl, cb0 + cchunk);
        constexpr int EPW = 4 / ESZ;                            // lambda entries per 32-bit word
        const int wprev = i > 0 ? (i - 1 + EPW - 1) / EPW : 0; // lambda words of a level-(i-1) row (entries 0..i-2)
        const int wcur = (i + EPW - 1) / EPW;                   // ... of a level-i row (entries 0..i-1)
        int base = lo, below = 0;
        bool first = true, keepall = false;
        // candidate lists hold every valid child while the frontier is below K (all may survive), else only
        // the children whose code can be selected (<= capc); a level that keeps everything although
        // children were left out is redone with complete lists (rare: N == K and one child per parent)
        bool listall = N < K;
        // method variant: the last level ranked by total = PED + insertion completion; a child's
        // completion is its parent's minus vins and eins per used neighbour of its target, so the eins cnt
        // term of its PED cancels: total = PED_p + comp_p - vins + cv + edel d - (edel + eins) cB (+ mis)
        const bool lastTot = a.last_by_total && i == n1 - 1;
        int tcode = 0, rq = 0;
        lsync(); // P_i staged

        for (;;) { // ---------------- A + T ----------------
            // Children with PED > U_i = max parent PED + vdel + edel d_i are never selected when N >= K
            // (each of the N parents has a deletion child <= U_i): their codes skip the histogram.
            const int capc = (N >= K && !lastTot) ? max(0, min(win, ((hi + pedDel - base) >> a.ashift) + 1)) : win;
            const uint32_t capc1 = (uint32_t)(capc + 1) * 0x01010101u; // (capc + 1 <= win + 1 <= 254)
            for (int k = threadIdx.x; k < 256 * 32; k += LNT) s_hist[k] = 0;
            if (threadIdx.x == 0) { s_cnt = 0; s_next = cb0; s_drop = 0; }
            if (home0())
                for (int k = threadIdx.x; k < 256; k += LNT) a.hist[((ps + 1) % 3) * 256 + k] = 0;
            lsync();
            int wcount = 0;
            if (brancher) {
                // 3-stage pipeline per warp: descriptor loads (registers) -> row prefetch (cp.async into the
                // ring) -> materialise + expand.  Buffer slot: [cnt | used | lambda | k, p, j, ped].
                auto grab = [&]() -> int {
                    int v = 0;
                    if (lane == 0) v = atomicAdd(&s_next, 1);
                    return __shfl_sync(FULL, v, 0);
                };
                auto load_desc = [&](int k) -> int { // lanes 0..2: p, j, ped of (local) node k
                    if (k >= cb1 || lane > 2) return 0;
                    return lane == 0 ? ML(sel_p)[k] : (lane == 1 ? ML(sel_j)[k] : ML(sel_ped)[k]);
                };
                auto issue = [&](int k, int dv, uint32_t *pf) {
                    const int64_t pl = __shfl_sync(FULL, dv, 0); // the parent's row on its rank
                    const int po = drank(__shfl_sync(FULL, dv, 1));
                    FG_CHECK(k >= cb1 || (po >= 0 && po < G && pl >= 0 && pl < a.kl), "DBG parent i=%d k=%d po=%d pl=%lld\n", i, k, po,
                             (long long)pl);
                    if (lane < 3) pf[PFW - 4 + 1 + lane] = (uint32_t)dv;
                    if (lane == 0) pf[PFW - 4] = (uint32_t)k;
                    if (k < cb1) {
                        // the parent's rows, on its rank (a peer's memory when sharded)
                        const uint8_t *crow8 = reinterpret_cast<const uint8_t *>(reinterpret_cast<const CntT *>(RK(po, cnt[pv])) + pl * cs);
                        for (int x = lane; x < CNTW / 4; x += 32) cpa16(pf + 4 * x, crow8 + 16 * x);
                        for (int w = lane; w < W; w += 32) cpa4(pf + CNTW + w, RK(po, used[pv]) + pl * W + w);
                        const uint32_t *mr = reinterpret_cast<const uint32_t *>(RK(po, map[pv])) + pl * rowwords;
                        // lambda row in 16-byte chunks (rows are 16-byte multiples; the words past wprev are
                        // never read as entries)
                        for (int w = 4 * lane; w < wprev; w += 128) cpa16(pf + CNTW + 32 + w, mr + w);
                    }
                    cpa_commit(); // (possibly empty group: keeps the ring's group count uniform)
                };
                int kn = grab(), dn = load_desc(kn);
                issue(kn, dn, pfb);
                kn = grab();
                dn = load_desc(kn);
                static_assert(LPF == 2, "the prefetch ring alternates two slots");
                uint32_t *pf = pfb, *pfn = pfb + PFW; // slot being expanded / slot being filled
                for (int r = 0;; ++r) {
                    if (r > 0) { uint32_t *t = pf; pf = pfn; pfn = t; } // (the slot expanded last is refilled)
                    const int kx = kn, dx = dn;
                    kn = grab();
                    dn = load_desc(kn);                               // descriptor of the parent after next
                    issue(kx, dx, pfn);                               // rows of the next parent
                    cpa_wait<1>();
                    __syncwarp();
                    const int k = (int)pf[PFW - 4];
                    if (k >= cb1) break; // (parents are taken in increasing order: the rest is empty)
                    const int j = dtarget((int32_t)pf[PFW - 2]), pedp = (int)pf[PFW - 1];
                    const int jn = (j >= 0 && j < n2) ? j : -1; // target used by this node's last step
                    uint32_t *sU = pf + CNTW;
                    uint32_t *mrow = pf + CNTW + 32;
                    if (lane == 0) ML(ped[cu])[k] = pedp;
                    // materialise row k of level i: used | j, lambda + entry i-1, counters + adj2 row j
                    int nused = 0;
                    for (int w = lane; w < W; w += 32) {
                        uint32_t uw = sU[w];
                        if (jn >= 0 && (jn >> 5) == w) uw |= 1u << (jn & 31);
                        sU[w] = uw;
                        Qused[(int64_t)k * W + w] = uw;
                        nused += __popc(uw);
                        if (!scatter) sB[w] = 0u;
                    }
                    nused = __reduce_add_sync(FULL, nused);
                    if (i > 0) {
                        const int hw = (i - 1) / EPW, sh = ((i - 1) % EPW) * 8 * ESZ;
                        const uint32_t e = (j == n2) ? (uint32_t)DELV : (uint32_t)j;
                        uint32_t *dst = reinterpret_cast<uint32_t *>(Qmap) + (int64_t)k * rowwords;
                        for (int w = 4 * lane; w < wcur; w += 128) { // 16-byte chunks
                            uint4 v = w < wprev ? *reinterpret_cast<const uint4 *>(mrow + w) : make_uint4(0u, 0u, 0u, 0u);
                            if ((unsigned)(hw - w) < 4u) {
                                uint32_t *vw = reinterpret_cast<uint32_t *>(&v);
                                uint32_t word = vw[0];
                                if (hw - w == 1) word = vw[1];
                                if (hw - w == 2) word = vw[2];
                                if (hw - w == 3) word = vw[3];
                                word = (word & ~((uint32_t)DELV << sh)) | (e << sh);
                                mrow[hw] = word;
                                if (hw - w == 0) v.x = word;
                                if (hw - w == 1) v.y = word;
                                if (hw - w == 2) v.z = word;
                                if (hw - w == 3) v.w = word;
                            }
                            *reinterpret_cast<uint4 *>(dst + w) = v;
                        }
                    }
                    __syncwarp();
                    auto tmap = [&](int q) -> int {
                        return (int)((mrow[(q * ESZ) >> 2] >> (8 * ((q * ESZ) & 3))) & (uint32_t)DELV);
                    };
                    uint32_t nzb = 0;
                    if (scatter) {
                        // D[u] += 1 (+ 1 << 16 on a label mismatch) for every neighbour u of every image t_k
                        for (int k0 = 0; k0 < d; k0 += 32) {
                            const int kk = k0 + lane;
                            const int tk = kk < d ? tmap(s_pq[kk]) : DELV;
                            const int lk = (LAB && kk < d) ? s_pl[kk] : 0;
                            // the neighbour-list range of this lane's image, loaded for all images at once
                            // (a deleted image has an empty range)
                            const int bk = tk != DELV ? nptr[tk] : 0, ek = tk != DELV ? nptr[tk + 1] : 0;
                            const int kn2 = min(32, d - k0);
                            for (int z = 0; z < kn2; ++z) {
                                const int e0 = __shfl_sync(FULL, bk, z), e1 = __shfl_sync(FULL, ek, z);
                                const int lz = LAB ? __shfl_sync(FULL, lk, z) : 0;
                                // the neighbours of one t are distinct: plain read-modify-write, no atomics
                                for (int e = e0 + lane; e < e1; e += 32) {
                                    const uint32_t v = nbr[e];
                                    D[v & 0xffffu] += (LAB && (int)(v >> 16) != lz) ? 0x10001 : 1;
                                }
                                __syncwarp();
                            }
                        }
                    } else {
                        for (int q = lane; q < d; q += 32) {
                            const int t = tmap(s_pq[q]);
                            if (t != DELV) atomicOr(&sB[t >> 5], 1u << (t & 31));
                        }
                        __syncwarp();
                        nzb = __ballot_sync(FULL, lane < W && sB[lane] != 0u);
                    }
                    __syncwarp();
                    int comp = 0; // (variant, last level) this node's insertion completion
                    if (lastTot) {
                        int e2u2 = 0; // used-neighbour counters summed over the used targets: 2 x edges among them
                        for (int s = 0; s < S; ++s) {
                            const int u0 = 128 * s + 4 * lane, wu = u0 >> 5;
                            typename C4::V cv = C4::load(reinterpret_cast<const CntT *>(pf), u0);
                            if (jn >= 0 && wu < W) cv = C4::add_bits(cv, (adjw(jn, wu) >> (u0 & 31)) & 0xfu);
                            const uint32_t ub = wu < W ? (sU[wu] >> (u0 & 31)) & 0xfu : 0u;
#pragma unroll
                            for (int b = 0; b < 4; ++b)
                                if ((ub >> b) & 1u) e2u2 += C4::get(cv, b);
                        }
                        e2u2 = __reduce_add_sync(FULL, e2u2);
                        comp = c.vins * (n2 - nused) + c.eins * (pd.m2 - e2u2 / 2);
                    }
                    const int pb = pedp - base + 1 + edd + (lastTot ? comp - c.vins : 0);
                    const int einsT = lastTot ? 0 : c.eins;
                    const int xdel = pedp + pedDel + comp - base + 1;
                    const int cdel = a.ashift ? (xdel <= 0 ? 0 : min(((xdel - 1) >> a.ashift) + 1, win + 1)) : rank_code(pedp + pedDel + comp, base, win);
                    uint8_t *crow = ML(ccode) + (int64_t)k * cs;
                    uint16_t *trow = ML(ctgt) + (int64_t)k * cs;
                    const CntT *cr = reinterpret_cast<const CntT *>(pf);
                    CntT *qc = Qcnt + (int64_t)k * cs;
                    uint32_t rmin2 = 0x00ff00ffu; // smallest code of the row, two 16-bit lanes
                    int nsel = 0;              // entries of the row's list so far (warp-uniform)
                    const unsigned lml = lanemask_lt();
                    bool dropped = false;
                    // the row's slots, 4 per lane per step (two instantiations: exact / approximate codes)
                    auto slots = [&](auto apx) {
                        constexpr bool APX = decltype(apx)::value;
                        for (int s = 0; s < S; ++s) {
                            const int u0 = 128 * s + 4 * lane, wu = u0 >> 5;
                            typename C4::V cv = C4::load(cr, u0);
                            if (jn >= 0 && wu < W) cv = C4::add_bits(cv, (adjw(jn, wu) >> (u0 & 31)) & 0xfu);
                            if (first) C4::store(qc, u0, cv);
                            const uint32_t ub = (sU[min(wu, 31)] >> (u0 & 31)) & 0xfu;
                            const uint32_t mnib = (uint32_t)(mm >> (4 * s)) & 0xfu;
                            int cb[4] = {0, 0, 0, 0}, ms[4] = {0, 0, 0, 0};
                            if (scatter) {
                                int4 *dp = reinterpret_cast<int4 *>(D + u0);
                                const int4 dv = *dp;
                                *dp = make_int4(0, 0, 0, 0);
                                if (LAB) { cb[0] = dv.x & 0xffff; cb[1] = dv.y & 0xffff; cb[2] = dv.z & 0xffff; cb[3] = dv.w & 0xffff; }
                                else { cb[0] = dv.x; cb[1] = dv.y; cb[2] = dv.z; cb[3] = dv.w; } // (no mismatch half)
                                if (LAB) { ms[0] = dv.x >> 16; ms[1] = dv.y >> 16; ms[2] = dv.z >> 16; ms[3] = dv.w >> 16; }
                            } else {
                                uint32_t m = nzb;
                                while (m) {
                                    const int w = __ffs(m) - 1;
                                    m &= m - 1;
                                    const uint4 av = *reinterpret_cast<const uint4 *>(adjT + (int64_t)w * cs + u0);
                                    const uint32_t bw = sB[w];
                                    cb[0] += __popc(av.x & bw); cb[1] += __popc(av.y & bw);
                                    cb[2] += __popc(av.z & bw); cb[3] += __popc(av.w & bw);
                                }
                            }
                            // the four slots' rank codes as bytes of one word (CODE_INVALID: used / past n2)
                            uint32_t word = 0;
    #pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                // every slot's value is computed branch-free; the deletion slot and the used /
                                // out-of-range slots are set below, once per word
                                const int x = pb + (int)((mnib >> b) & 1u) * c.vsub + einsT * C4::get(cv, b) - ee * cb[b] +
                                              (LAB ? c.esub * ms[b] : 0);
                                // rank code: x = PED - base + 1; approximate variant: PED bins of 2^ashift
                                const int cd = APX ? (x <= 0 ? 0 : min(((x - 1) >> a.ashift) + 1, win + 1)) : min(max(x, 0), win + 1);
                                word |= (uint32_t)cd << (8 * b);
                            }
                            // slot n2 - u0 (if 0..3) is the deletion child (reading C5); slots of used
                            // targets and past n2 are CODE_INVALID (bytes 0xff)
                            const int rel = n2 - u0;
                            uint32_t inv4 = ub;
                            if (rel < 4) {
                                inv4 = (ub & (rel <= 0 ? 0u : (1u << rel) - 1u)) | (rel < 0 ? 0xfu : ((0xeu << rel) & 0xfu));
                                if (rel >= 0) word = (word & ~(0xffu << (8 * rel))) | ((uint32_t)cdel << (8 * rel));
                            }
                            word |= ((inv4 * 0x00204081u) & 0x01010101u) * 0xffu;
                            // histogram of the codes that can be selected (1..capc), per lane column
                            uint32_t hmk = bytes_lt(word, capc1) & ~bytes_eq(word, 0u);
                            while (hmk) {
                                const int by = (__ffs(hmk) - 1) >> 3;
                                hmk &= hmk - 1;
                                atomicAdd(&s_hist[((word >> (8 * by)) & 0xffu) * 32 + lane], 1);
                            }
                            rmin2 = __vminu2(rmin2, __vminu2(word & 0x00ff00ffu, (word >> 8) & 0x00ff00ffu));
                            const uint32_t validb = ~bytes_eq(word, 0xffffffffu) & 0x80808080u;
                            const uint32_t listedb = listall ? validb : bytes_lt(word, capc1); // (255 > capc: never listed)
                            dropped |= (validb & ~listedb) != 0u;
                            // list entries in target order (u = 128 s + 4 lane + b: lanes first, then b): the
                            // lane's listed count (0..4) as three ballot bit planes gives its offset in the warp
                            uint32_t m4 = ((((listedb >> 7) & 0x01010101u) * 0x01020408u) >> 24) & 0xfu; // bit b: byte b listed
                            const int cnt = __popc(m4);
                            const unsigned B0 = __ballot_sync(FULL, cnt & 1), B1 = __ballot_sync(FULL, cnt & 2),
                                           B2 = __ballot_sync(FULL, cnt & 4);
                            int pos = nsel + __popc(B0 & lml) + 2 * __popc(B1 & lml) + 4 * __popc(B2 & lml);
                            while (m4) {
                                const int b = __ffs(m4) - 1;
                                m4 &= m4 - 1;
                                FG_CHECK(pos >= 0 && pos < cs, "DBG list i=%d k=%d pos=%d\n", i, k, pos);
                                crow[pos] = (uint8_t)(word >> (8 * b));
                                trow[pos++] = (uint16_t)(u0 + b);
                            }
                            nsel += __popc(B0) + 2 * __popc(B1) + 4 * __popc(B2);
                        }
                    };
                    if (a.ashift) slots(std::true_type{});
                    else slots(std::false_type{});
                    const uint32_t rmin = __reduce_min_sync(FULL, min(rmin2 & 0xffffu, rmin2 >> 16));
                    if (lane == 0) {
                        ML(rowmin)[k] = (int)rmin;
                        ML(rown)[k] = nsel;
                    }
                    if (dropped) s_drop = 1; // (benign race: every writer stores 1)
                    wcount += n2 - nused + 1;
                    __syncwarp();
                }
                cpa_wait<0>();
            }
            if (first && lane == 0) atomicAdd((unsigned long long *)&s_cnt, (unsigned long long)wcount);
            lsync();
            int *gh = a.hist + (ps % 3) * 256;
            for (int bin = threadIdx.x; bin < 256; bin += LNT) {
                int v = 0;
#pragma unroll 8
                for (int l = 0; l < 32; ++l) v += s_hist[bin * 32 + ((l + bin) & 31)];
                if (v) atomicAdd(&gh[bin], v);
            }
            if (first && threadIdx.x == 0) atomicAdd((unsigned long long *)&a.ci[i], (unsigned long long)s_cnt);
            if (threadIdx.x == 0 && s_drop) a.drop[i] = 1;
            if (!xsync()) return;
            tick(0);
            // T: every CTA derives the same threshold from the global histogram
            const int64_t ci = a.ci[i];
            keepall = (ci <= K);
            bool retry = false, slide = false;
            if (keepall && !listall && a.drop[i]) { listall = true; retry = true; }
            if (!keepall) {
                if (wib == 0) {
                    int hv[8], sum = 0;
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        const int bb = 8 * lane + x + 1; // codes 1..256
                        hv[x] = (bb <= capc) ? gh[bb] : 0;
                        sum += hv[x];
                    }
                    int incl = sum;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += y;
                    }
                    if (home0() && lane == 31) nhist += incl;
                    const unsigned hm = __ballot_sync(FULL, below + incl >= K);
                    if (hm) {
                        const int L = __ffs(hm) - 1;
                        if (lane == L) {
                            int c2 = below + incl - sum, tc = 0, rr = 0;
#pragma unroll
                            for (int x = 0; x < 8; ++x) {
                                if (tc == 0 && c2 + hv[x] >= K) { tc = 8 * lane + x + 1; rr = K - c2; }
                                c2 += hv[x];
                            }
                            s_pre[0] = tc;
                            s_pre[1] = rr;
                        }
                    } else if (lane == 31) {
                        s_pre[0] = 0;
                        s_pre[1] = incl; // every code of the window lies below the K-th smallest
                    }
                }
                lsync();
                tcode = s_pre[0];
                if (tcode) rq = s_pre[1];
                else { retry = slide = true; below += s_pre[1]; }
                lsync();
            }
            if (first) children += ci;
            ps++;
            first = false;
            if (!retry) break;
            if (slide) base += win << a.ashift; // the K-th smallest lies beyond the window: slide it (codes 0 = kept)
        }

        // ---------------- B: per-row counts of list codes < t and == t (lane per row, static ranges) ----------------
        const uint32_t t4 = (uint32_t)tcode * 0x01010101u;
        {
            int wl = 0, we = 0;
            // 32 rows per step, one per lane; only rows whose smallest code can be selected are read (SWAR
            // byte compares over 16-byte vectors of the list's codes, bytes past the list masked off)
            for (int k0 = p0; k0 < p1; k0 += 32) {
                const int kl = k0 + lane;
                int myl = 0, mye = 0; // counts of row kl
                if (kl < p1 && (keepall || ML(rowmin)[kl] <= tcode)) {
                    const int n = ML(rown)[kl];
                    const uint4 *cv = reinterpret_cast<const uint4 *>(ML(ccode) + (int64_t)kl * cs);
                    for (int x = 0; 16 * x < n; ++x) {
                        const uint4 v = cv[x];
                        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const int nbv = min(max(n - 16 * x - 4 * w, 0), 4); // list bytes in this word
                            const uint32_t vm = nbv == 4 ? 0x80808080u : (0x80808080u & ((1u << (8 * nbv)) - 1u));
                            if (keepall) myl += __popc(vm);
                            else {
                                myl += __popc(bytes_lt(wv[w], t4) & vm);
                                mye += __popc(bytes_eq(wv[w], t4) & vm);
                            }
                        }
                    }
                }
                int il = myl, ie = mye;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int yl = __shfl_up_sync(FULL, il, o), ye = __shfl_up_sync(FULL, ie, o);
                    if (lane >= o) { il += yl; ie += ye; }
                }
                if (kl < p1) {
                    ML(rowc)[kl] = myl | (mye << 16);
                    ML(rowpl)[kl] = wl + il - myl;
                    ML(rowpe)[kl] = we + ie - mye;
                }
                wl += __shfl_sync(FULL, il, 31);
                we += __shfl_sync(FULL, ie, 31);
            }
            if (lane == 0) { s_red[0][wib] = wl; s_red[1][wib] = we; }
            lsync();
            if (lane == 0) { // this warp's prefix inside the CTA
                int cl = 0, ce = 0;
                for (int w = 0; w < wib; ++w) { cl += s_red[0][w]; ce += s_red[1][w]; }
                ML(wlt)[gw] = cl;
                ML(weq)[gw] = ce;
                if (wib == NWB - 1) { a.ctl[RANK * nb + LB] = cl + wl; a.cte[RANK * nb + LB] = ce + we; }
            }
        }
        if (!xsync()) return;
        tick(1);

        // ---------------- prefix of the per-CTA counts (every CTA, redundantly) ----------------
        // CTAs in (rank, CTA) order = the global (parent, child) order; this rank's CTAs' prefixes kept
        if (wib == 0) {
            const int gend = (RANK + 1) * nb, gme = RANK * nb;
            int rl = 0, re = 0;
            for (int g0 = 0; g0 < gend; g0 += 32) {
                const int g = g0 + lane;
                const int l = g < gend ? a.ctl[g] : 0, e = g < gend ? a.cte[g] : 0;
                int il = l, ie = e;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int yl = __shfl_up_sync(FULL, il, o), ye = __shfl_up_sync(FULL, ie, o);
                    if (lane >= o) { il += yl; ie += ye; }
                }
                if (g >= gme && g < gend) { s_cpre[0][g - gme] = rl + il - l; s_cpre[1][g - gme] = re + ie - e; }
                rl += __shfl_sync(FULL, il, 31);
                re += __shfl_sync(FULL, ie, 31);
            }
        }
        lsync();
        const int Nn = keepall ? (int)a.ci[i] : K;

        // ---------------- C1: compact survivors in (parent, child) order, with their PEDs ----------------
        // Rows are dealt round-robin over all warps (survivors cluster in the rows of a few good parents,
        // so the static B ranges would leave a handful of warps with all of them); rows without a survivor
        // are skipped without reading their codes.  A row's output offset = prefix of the CTAs before its
        // B owner + the owner CTA's warps before the owner warp + the owner's rows before it.
        {
            int mylo = 0x7fffffff, myhi = (int)0x80000000;
            const unsigned lml = lanemask_lt();
            auto is_lt = [&](uint32_t e, bool in) { return keepall ? in : (int)(e & 0xffu) < tcode; };
            // survivor (row k, target u, rank code) at global position pos of the next level
            auto emit = [&](int k, int u, int code, int pos) {
                int ped;
                if (a.ashift == 0 && code >= 1 && code <= win) ped = base + code - 1;
                else { // below the window, saturated or a PED bin: recompute from the parent's materialised row
                    ped = large_child_scalar<MapT, CntT, LAB>(a, d, s_pq, s_pl, ML(ped[cu])[k], Qcnt + (int64_t)k * cs,
                                                              Qmap + (int64_t)k * a.n1s, u, adj2, e2, vl1i, vl2);
                    if (lastTot) { // (variant) + the child's completion, from the node's used row and counters
                        const uint32_t *ur = Qused + (int64_t)k * W;
                        const CntT *cr2 = Qcnt + (int64_t)k * cs;
                        int usedc = (u < n2) ? 1 : 0, e2u2 = 0;
                        for (int w = 0; w < W; ++w) {
                            uint32_t bits = ur[w];
                            usedc += __popc(bits);
                            while (bits) {
                                const int t = 32 * w + __ffs(bits) - 1;
                                bits &= bits - 1;
                                e2u2 += (int)cr2[t];
                            }
                        }
                        if (u < n2) e2u2 += 2 * (int)cr2[u];
                        ped += c.vins * (n2 - usedc) + c.eins * (pd.m2 - e2u2 / 2);
                    }
                }
                // its descriptor goes to its owner (a peer when sharded); the parent is row k of this rank
                const int no = rowner(pos, Nn);
                const int np = pos - rstart(Nn, no);
                FG_CHECK(no >= 0 && no < G && np >= 0 && np < a.kl && pos < Nn, "DBG emit i=%d pos=%d Nn=%d no=%d np=%d\n", i, pos, Nn, no, np);
                RK(no, sel_p)[np] = k;
                RK(no, sel_j)[np] = u | (RANK << 16);
                RK(no, sel_ped)[np] = ped;
                mylo = min(mylo, ped);
                myhi = max(myhi, ped);
            };
            auto is_eq = [&](uint32_t e) { return !keepall && (int)(e & 0xffu) == tcode; };
            // 32 rows per batch (row kb + l GW for lane l): their counts and prefixes are loaded in parallel,
            // then the rows holding survivors are expanded one after the other (lane x: entry x of the list)
            for (int kb = gw; kb < Nl; kb += 32 * GW) {
                const int kl = kb + lane * GW;
                int rc = 0, lp = 0, ep = 0;
                bool has = false;
                if (kl < Nl) {
                    rc = ML(rowc)[kl];
                    has = keepall ? rc != 0 : ((rc & 0xffff) != 0 || (rc >> 16) > 0);
                    if (has) {
                        const int ow = kl / chunk, oc = ow / NWB;
                        lp = s_cpre[0][oc] + ML(wlt)[ow] + ML(rowpl)[kl];
                        ep = s_cpre[1][oc] + ML(weq)[ow] + ML(rowpe)[kl];
                        if (!keepall && (rc & 0xffff) == 0 && ep >= rq) has = false; // its ties are all past the quota
                    }
                }
                unsigned hm = __ballot_sync(FULL, has);
#ifdef FG_LSTAT
                {
                    const unsigned rows = __ballot_sync(FULL, kl < Nl);
                    if (lane == 0) {
                        atomicAdd(&fg_lstat[0], (unsigned long long)__popc(hm));
                        atomicAdd(&fg_lstat[1], (unsigned long long)__popc(rows));
                    }
                }
#endif
                const int rn = has ? ML(rown)[kl] : 0;
                // rows with few survivors: lane per row (32 rows in flight); the rest: warp per row below
                const int nkeep = keepall ? (rc & 0xffff) : (rc & 0xffff) + min(rc >> 16, max(0, rq - ep));
                const bool light = has && nkeep <= FG_C1_LIGHT;
                hm &= ~__ballot_sync(FULL, light);
                if (light) {
                    int out = lp + (keepall ? 0 : min(rq, ep)), eq_seen = ep, left = nkeep;
                    const uint4 *cv = reinterpret_cast<const uint4 *>(ML(ccode) + (int64_t)kl * cs);
                    for (int x = 0; left > 0 && 16 * x < rn; ++x) {
                        const uint4 v = cv[x];
                        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const int nbv = min(max(rn - 16 * x - 4 * w, 0), 4);
                            const uint32_t vm = nbv == 4 ? 0x80808080u : (0x80808080u & ((1u << (8 * nbv)) - 1u));
                            uint32_t ml = keepall ? vm : (bytes_lt(wv[w], t4) & vm);
                            uint32_t mq = keepall ? 0u : (bytes_eq(wv[w], t4) & vm);
                            // ties at t are admitted in list (= target) order up to the quota rq
                            const int nq = __popc(mq);
                            for (int z = min(nq, max(0, rq - eq_seen)); z > 0; --z) { const uint32_t low = mq & (0u - mq); ml |= low; mq ^= low; }
                            eq_seen += nq;
                            while (ml) {
                                const int by = (__ffs(ml) - 1) >> 3;
                                ml &= ml - 1;
                                const int idx = 16 * x + 4 * w + by;
                                emit(kl, (int)ML(ctgt)[(int64_t)kl * cs + idx], (int)((wv[w] >> (8 * by)) & 0xffu), out++);
                                --left;
                            }
                        }
                    }
                }
                while (hm) {
                    const int z = __ffs(hm) - 1;
                    hm &= hm - 1;
                    const int k = kb + z * GW;
                    const int n = __shfl_sync(FULL, rn, z);
                    const int ltpre = __shfl_sync(FULL, lp, z), eqpre = __shfl_sync(FULL, ep, z);
                    int eq_seen = eqpre, out = ltpre + (keepall ? 0 : min(rq, eqpre));
                    auto ent = [&](int x) -> uint32_t { // code | target << 8 of list entry x; padding: code 255
                        return x < n ? (uint32_t)ML(ccode)[(int64_t)k * cs + x] | ((uint32_t)ML(ctgt)[(int64_t)k * cs + x] << 8)
                                     : 0xffffffffu;
                    };
                    uint32_t en = ent(lane);
                    for (int xb = 0; xb < n; xb += 32) {
                        const int x = xb + lane;
                        const uint32_t e = en;
                        if (xb + 32 < n) en = ent(x + 32);
                        const bool lt = is_lt(e, x < n), eq = is_eq(e);
                        // ties at t are admitted in list (= target) order up to the quota rq
                        const unsigned eb = __ballot_sync(FULL, eq);
                        const bool keep = lt || (eq && eq_seen + __popc(eb & lml) < rq);
                        const unsigned kbm = __ballot_sync(FULL, keep);
                        if (keep) {
                            const int pos = out + __popc(kbm & lml);
                            const int u = (int)(e >> 8), code = (int)(e & 0xffu);
                            emit(k, u, code, pos);
                        }
                        out += __popc(kbm);
                        eq_seen += __popc(eb);
                    }
                }
            }
            mylo = __reduce_min_sync(FULL, mylo);
            myhi = __reduce_max_sync(FULL, myhi);
            if (lane == 0 && mylo != 0x7fffffff) {
                atomicMin(&a.lo[i + 1], mylo);
                atomicMax(&a.hi[i + 1], myhi);
            }
        }
        if (home0() && threadIdx.x == 0 && a.levels_out) {
            a.levels_out[3 * i] = N;
            a.levels_out[3 * i + 1] = a.ci[i];
            // the K-th smallest key: its PED (exact) or its bin above the level's smallest parent PED (approximate)
            a.levels_out[3 * i + 2] = keepall ? -1 : (a.ashift ? (int64_t)(((base - lo) >> a.ashift) + tcode - 1) : (int64_t)(base + tcode - 1));
        }
        parents += N;
        algb += (int64_t)N * (4 + ESZ * d) + (int64_t)Nn * (ESZ * (2 * i + 1) + 8);
        if (!xsync()) return;
        tick(2);
        N = Nn;
        lo = a.lo[i + 1];
        hi = a.hi[i + 1];
    }

    // ---------------- finalize: completion + argmin ----------------
    {
        const int pv = (n1 + 1) & 1; // rows of level n1 - 1 (the final nodes' parents)
        const int s0 = rstart(N, RANK), Nl = rstart(N, RANK + 1) - s0;
        for (int k = gw; k < Nl; k += GW) { // warp per final node (p, j) of this rank
            const int64_t pl = ML(sel_p)[k];
            const int po = drank(ML(sel_j)[k]), j = dtarget(ML(sel_j)[k]), ped = ML(sel_ped)[k];
            const uint32_t *Pused = RK(po, used[pv]) + pl * W;
            const CntT *Pcnt = reinterpret_cast<const CntT *>(RK(po, cnt[pv])) + pl * cs;
            const int jn = (j >= 0 && j < n2) ? j : -1;
            int usedc = 0, e2u2 = 0;
            for (int w = lane; w < W; w += 32) {
                uint32_t uw = Pused[w];
                if (jn >= 0 && (jn >> 5) == w) uw |= 1u << (jn & 31);
                usedc += __popc(uw);
            }
            for (int u = lane; u < n2; u += 32) {
                uint32_t uw = Pused[u >> 5];
                if (jn >= 0 && (jn >> 5) == (u >> 5)) uw |= 1u << (jn & 31);
                if ((uw >> (u & 31)) & 1u) {
                    int cu = (int)Pcnt[u];
                    if (jn >= 0) cu += (int)((adjw(jn, u >> 5) >> (u & 31)) & 1u);
                    e2u2 += cu;
                }
            }
            usedc = __reduce_add_sync(FULL, usedc);
            e2u2 = __reduce_add_sync(FULL, e2u2); // every edge among used vertices counted from both ends
            if (lane == 0) {
                // (variant: the last level already ranked and stored PED + completion; n1 = 0 has no last level)
                const int64_t total = (a.last_by_total && n1 > 0)
                                          ? (int64_t)ped
                                          : (int64_t)ped + (int64_t)c.vins * (n2 - usedc) + (int64_t)c.eins * (pd.m2 - e2u2 / 2);
                atomicMin(a.best, ((unsigned long long)total << 32) | (unsigned)(s0 + k));
            }
        }
        if (!xsync()) return;
        if (home0() && threadIdx.x == 31) a.out[9] = nhist;
#ifdef FG_DEBUG_CHECKS
        if (home0() && threadIdx.x == 0 && fg_dbg_bad) printf("DBG violations %u\n", fg_dbg_bad);
#endif
#ifdef FG_LSTAT
        if (home0() && threadIdx.x == 0)
            printf("LSTAT parents with a survivor %llu of %llu (%.3f); A passes %d over %d levels\n", fg_lstat[0], fg_lstat[1],
                   (double)fg_lstat[0] / fg_lstat[1], ps, n1);
#endif
        if (home0()) {
            const unsigned long long best = *a.best;
            const int kb = (int)(best & 0xffffffffull);
            const int ko = rowner(kb, N), kl = kb - rstart(N, ko);
            const int64_t pl = RK(ko, sel_p)[kl];
            const int po = drank(RK(ko, sel_j)[kl]), j = dtarget(RK(ko, sel_j)[kl]);
            const MapT *row = reinterpret_cast<const MapT *>(RK(po, map[pv])) + pl * a.n1s;
            for (int q = threadIdx.x; q < n1; q += LNT) {
                const int t = (q == n1 - 1) ? ((j == n2) ? DELV : j) : (int)row[q];
                a.map_out[q] = (t == DELV) ? -1 : t;
            }
            if (threadIdx.x == 0) {
                a.out[0] = (int64_t)(best >> 32);
                a.out[1] = children;
                a.out[2] = parents;
                a.out[3] = algb;
                tick(4);
                for (int x = 0; x < 5; ++x) a.out[4 + x] = tph[x];
            }
        }
    }
}
#undef ML
#undef RK
#undef RANK
#undef LB

} // namespace fg
