// batch_kernel.cuh -- the batched K-Best search: one CTA runs one (g1, g2) pair through all
// levels of Alg. 1 and then takes the next pair from a work counter.
//
// Frontier (per CTA, global scratch, structure of arrays so every per-level pass is coalesced):
//   ped[K] int32, usedT[W][K] uint32 (bit u = g2 vertex u used), BT[W][K] uint32 (B_p of the next
//   level, see U), mapT[n1][K] uint8 (lambda, 255 = deleted).  Column k is frontier node k.
//
// Per level i (g1 vertex v_i, reading C4):
//   P  Parents' used masks to shared memory; parent p owns the compact code range
//      [off_p, off_p + f_p + 1): its f_p free targets in ascending order, then its deletion child
//      (= the (parent, child) lin order of reading C12/C13); off_p from a block scan.
//   A  Branch (Alg. 2).  The child PED is the paper's incremental
//      evaluation PED = E(parent) + c(v<-u) + Imp_cost with the three implied-edge cases of
//      PAPER.md:103-116 regrouped into popcounts:
//          Delta(u)   = cv(i,u) + edel*d_i + eins*cnt_p(u) - (edel+eins)*cB_p(u) + esub*mis_p(u)
//          Delta(DEL) = vdel + edel*d_i
//      cnt_p(u) = popc(adj2[u] & used_p), cB_p(u) = popc(adj2[u] & B_p), B_p = images of the earlier
//      g1 neighbours of v_i (replaces the paper's VFrom/VTo vectors); labelled edges:
//      mis_p(u) = cB_p(u) - sum_l popc(adj2_l[u] & B_{p,l}), one g2 label plane adj2_l per edge label and
//      B_{p,l} = the images whose g1 edge to v_i has label l (kept per node like B_p).  Wide frontiers: a thread
//      per parent iterates only that parent's free targets; narrow ones: a warp per parent with
//      lane-owned targets.  Each child becomes a one-byte rank code (PED - base + 1, saturated) in
//      shared memory and one atomic in its warp's private 128-bin histogram.  Children never reach HBM.
//   T  Threshold (replaces the paper's local/global ranking): every warp scans the
//      histograms and derives the same threshold PED t and quota r of ties at t; exactly
//      min(K, c_i) children are kept, the smallest under (PED, parent, child) (reading C12).  No sort.
//      If the K-th smallest lies beyond the window the window slides and A is repeated.
//   S  Selection: every thread owns a contiguous run of code words; SWAR byte compares count codes
//      < t / == t, a block scan gives each thread its output offset and tie admissions, survivors
//      are written as (parent, rank within parent) in (parent, child) order (C13), then decoded to
//      (p, j) and their PED (from the rank code) in a balanced pass.
//   U  Update: next frontier columns with coalesced stores; while copying the
//      lambda columns, B_p (and the label planes B_{p,l}) of the next level are accumulated.
// After the last level each survivor gets the insertion completion (C6) and the
// argmin by (total, position) is written out (C10).
#pragma once
#include <cstdint>
#include <cstdio>

namespace fg {

#ifndef FG_CZ
#define FG_CZ 2 // children evaluated per iteration of the wide branch loop (independent chains; 2 measured best: 49.6 vs 50.8 ms at 4)
#endif
#ifndef FG_MINBLOCKS
#define FG_MINBLOCKS 2 // resident CTAs per SM requested from ptxas (A/B experiments)
#endif
#ifndef FG_MINBLOCKS_128
#define FG_MINBLOCKS_128 4 // the same for the 128-thread (one-word) variants
#endif

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAP_DEL = 255;      // lambda entry of a deleted g1 vertex
constexpr int CODE_INVALID = 255; // no child in this slot (used target / padding)
constexpr int LMAX = 3;           // edge-label planes of the batched path (more labels: whole-GPU path)

struct Costs {
    int vsub, vdel, vins, esub, edel, eins;
};

// One pair inside the device blob (byte offsets into the blob).
struct PairDesc {
    int32_t n1, n2, m1, m2;
    int32_t labelled, n2p;       // n2p: row stride of the e2lab byte matrix (multiple of 4)
    int32_t nlab, pad0;          // nlab: distinct g2 edge labels (label ids 1..nlab), labelled pairs
    int64_t vl1, vl2;            // int32[n1], int32[n2]
    int64_t pptr, pq, pl;        // int32[n1+1], int32[m1], int32[m1]  (P_i lists)
    int64_t adj2;                // uint32[n2 * W]
    int64_t e2lab;               // uint8[n2p * n2p] (labelled only): g2 edge label id + 1, 0 = no edge
    int64_t map_out;             // element offset of this pair's mapping in the output array
};

// Work-array plan of a batched launch.  pq/pl/pnl/adj/adjl/adjh: byte offsets into dynamic shared
// memory.  u/b/codes/sel/pidx: byte offsets into shared memory (SMEM launches) or into the CTA's
// global scratch after its two frontier buffers (large-K launches).
struct SmemPlan {
    int32_t pq, pl, pnl, pnq, adj, adjl, adjh, u, b, codes, sel, pidx, bytes;
};

struct BatchArgs {
    const PairDesc *descs;
    const int32_t *order;   // pair indices of this launch, in scheduling order
    int32_t ngroup;
    const uint8_t *blob;
    int32_t *work;          // dynamic scheduler counter (zeroed before launch)
    Costs c;
    int32_t K;              // the K of Alg. 1 (children kept per level)
    int32_t Kc;             // frontier capacity / array stride (>= min(K, widest level), multiple of 4)
    int32_t win;            // exact rank window: codes 1..win; win+1 = saturated
    int32_t csmax;          // max code row stride of the launch
    SmemPlan sm;
    uint8_t *scratch;       // per-CTA frontier scratch
    int64_t scratch_stride;
    int32_t n1max;
    int64_t *cost_out;
    int32_t *map_out;
    int64_t *children_out;
    int64_t *parents_out;
    int64_t *algbytes_out;  // per pair: algorithmic frontier bytes of the search
    int64_t *levels_out;    // NULL, or [3 * n1] for a single-pair launch
    int32_t last_by_total;  // method variant (reading C10 alternative): the last level is
                            // ranked by PED + completion instead of PED
};

#ifdef FG_PROF
// profiling builds only: per-phase SM cycles of CTA thread 0, summed over CTAs, printed by the last CTA
__device__ unsigned long long fg_prof_cyc[8];
__device__ unsigned int fg_prof_done;
#define FG_PH(k) do { if (threadIdx.x == 0) { const long long now_ = clock64(); ph_[k] += now_ - ph_last_; ph_last_ = now_; } } while (0)
#else
#define FG_PH(k) do { } while (0)
#endif

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Block barrier that is safe after lane-divergent code.  __syncthreads() compiles to bar.sync, an
// .aligned barrier that requires every warp to arrive converged; ptxas may drop a preceding
// __syncwarp(), and a warp leaving a strided loop with unequal trip counts then reaches the
// barrier diverged (undefined behaviour, seen as out-of-phase warps under compute-sanitizer
// synccheck).  The non-aligned barrier.sync is defined for divergent arrival; the explicit
// bar.warp.sync (volatile asm, cannot be elided) reconverges the warp for the code that follows.
__device__ __forceinline__ void block_sync() {
    asm volatile("bar.warp.sync -1;" ::: "memory");
#ifdef FG_ALIGNED_BARRIER
    asm volatile("bar.sync 0;" ::: "memory");
#else
    asm volatile("barrier.sync 0;" ::: "memory");
    asm volatile("bar.warp.sync -1;" ::: "memory");
#endif
}

// The same barrier as the aligned bar.sync: the volatile bar.warp.sync reconverges the warp first, so
// every warp arrives converged with no instruction between the two.  The whole-GPU kernel uses it
// (FG_LARGE_ALIGNED_BARRIER, default on: n = 500 K = 1e5 136 -> 127 ms, its B / C1 phases -35 %);
// the batched kernel measured no difference and keeps block_sync.
__device__ __forceinline__ void block_sync_aligned() {
    asm volatile("bar.warp.sync -1;" ::: "memory");
    asm volatile("bar.sync 0;" ::: "memory");
}

// Position of the (r+1)-th set bit of x (0 <= r < popc(x)): popcount bisection, no data-dependent loop.
__device__ __forceinline__ int select_bit(uint32_t x, int r) {
    int pos = 0, c;
    c = __popc(x & 0xffffu); if (r >= c) { r -= c; x >>= 16; pos += 16; }
    c = __popc(x & 0xffu);   if (r >= c) { r -= c; x >>= 8;  pos += 8; }
    c = __popc(x & 0xfu);    if (r >= c) { r -= c; x >>= 4;  pos += 4; }
    c = __popc(x & 0x3u);    if (r >= c) { r -= c; x >>= 2;  pos += 2; }
    c = (int)(x & 1u);       if (r >= c) { pos += 1; }
    return pos;
}

// Slot of a single-bit word b = 1 << bt under the de Bruijn hash (b * 0x077CB531) >> 27, a bijection of
// 0..31: the wide branch loop addresses the g2 row of target 32 w + bt through this slot, so it needs
// neither the bit index nor the BREV/FLO pair of __ffs (both on the quarter-rate XU pipe, like POPC).
__host__ __device__ __forceinline__ uint32_t db_slot(uint32_t b) { return (b * 0x077CB531u) >> 27; }

// Row stride (words) of the slot-addressed g2 rows: W adjacency words, (labelled) LMAX label planes of
// W words, then the level's vertex cost cv(i, u); padded so a row is whole 8- or 16-byte shared loads.
__host__ __device__ constexpr int hrow_stride(int W, bool lab) {
    return lab ? (((W * (1 + LMAX) + 1) + 3) & ~3) : (W + 1 <= 2 ? 2 : (W + 1 <= 4 ? 4 : 8));
}

__device__ __forceinline__ int rank_code(int ped, int base, int win) {
    const int x = ped - base + 1;
    return x < 0 ? 0 : (x > win ? win + 1 : x);
}

// Block-wide exclusive scan of two ints (NT threads).  Returns totals.  One barrier: every warp
// publishes its total and then reads all NT/32 of them.  s_tmp must not be rewritten before every
// warp has read it: consecutive calls are separated by other block barriers in the kernel.
template <int NT>
__device__ __forceinline__ void block_scan2(int a, int b, int &apre, int &bpre, int &atot, int &btot, int *s_tmp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int xa = __shfl_up_sync(FULL, ia, o), xb = __shfl_up_sync(FULL, ib, o);
        if (lane >= o) { ia += xa; ib += xb; }
    }
    if (lane == 31) { s_tmp[warp] = ia; s_tmp[32 + warp] = ib; }
    block_sync();
    int wa = 0, wb = 0, ta = 0, tb = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const int x = s_tmp[w], y = s_tmp[32 + w];
        if (w < warp) { wa += x; wb += y; }
        ta += x;
        tb += y;
    }
    apre = wa + ia - a;
    bpre = wb + ib - b;
    atot = ta;
    btot = tb;
}

// Insertion completion (C6) of a node whose used set is U: vins per unused g2 vertex +
// eins per g2 edge with an unused endpoint.  Rows from shared memory.
template <int W>
__device__ __forceinline__ int completion_of(const uint32_t (&U)[W], const uint32_t *sAdj, int n2, int m2, const Costs &c) {
    int usedc = 0, e2u2 = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        usedc += __popc(U[w]);
        uint32_t bits = U[w];
        while (bits) {
            const int u = 32 * w + __ffs(bits) - 1;
            bits &= bits - 1;
#pragma unroll
            for (int x = 0; x < W; ++x) e2u2 += __popc(sAdj[u * W + x] & U[x]);
        }
    }
    return c.vins * (n2 - usedc) + c.eins * (m2 - e2u2 / 2);
}

template <int W, bool LAB, int NT, bool SMEM>
__global__ void __launch_bounds__(NT, NT == 128 ? FG_MINBLOCKS_128 : FG_MINBLOCKS * 256 / NT) kbest_batch_kernel(const BatchArgs a) {
    extern __shared__ __align__(16) uint8_t dsmem[];
    // per-warp rank-code histograms, row stride 132: code c at [c + 3], codes 1..128 16-byte aligned
    __shared__ __align__(16) int s_hist[(NT / 32) * 132];
    __shared__ int s_tmp[144 + 32];
    __shared__ int s_item, s_lo;
    // bit q: v_q is an earlier neighbour of v_{i+1} (n1 <= 1024); double-buffered by level parity so
    // the buffer of level i is zeroed during level i - 1 (no barrier between zeroing and filling)
    __shared__ uint32_t s_pnext2[2][32];
    __shared__ unsigned long long s_best;
    constexpr int NW = NT / 32;
    constexpr int NB = LAB ? 1 + LMAX : 1;        // B planes per node
    constexpr int HRS = hrow_stride(W, LAB);      // slot-addressed row stride (words)
    constexpr int CVW = LAB ? W * (1 + LMAX) : W; // word of the row holding cv(i, u)

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Costs c = a.c;
    const int K = a.K, Kc = a.Kc, win = a.win;

    // per-CTA frontier (two buffers): ped[K], usedT[W][K], BT[NB][W][K], mapT[n1max][K]
    uint8_t *scr = a.scratch + (int64_t)blockIdx.x * a.scratch_stride;
    const int64_t fb = (int64_t)Kc * (4 + 4 * W + 4 * W * NB + a.n1max); // bytes per frontier buffer
    // per-level work arrays: shared memory (SMEM) or, for large K, this CTA's global scratch
    uint8_t *wk = SMEM ? dsmem : scr + 2 * fb;
    int32_t *s_pq = reinterpret_cast<int32_t *>(dsmem + a.sm.pq);
    int32_t *s_pl = reinterpret_cast<int32_t *>(dsmem + a.sm.pl);
    uint8_t *s_pnl = dsmem + a.sm.pnl; // label plane of the g1 edge (v_q, v_{i+1}) for q in P_{i+1} (LAB)
    int32_t *s_pnq = reinterpret_cast<int32_t *>(dsmem + a.sm.pnq); // P_{i+1} as a list (LAB)
    uint32_t *sAdj = reinterpret_cast<uint32_t *>(dsmem + a.sm.adj);   // g2 bit rows [n2][W]
    uint32_t *sAdjL = reinterpret_cast<uint32_t *>(dsmem + a.sm.adjl); // label planes [n2][LMAX][W] (LAB)
    // the same rows at [32 w + db_slot(bit)][HRS]: W adjacency words, label planes, cv(i, u)
    uint32_t *sAdjH = reinterpret_cast<uint32_t *>(dsmem + a.sm.adjh);
    uint32_t *sU = reinterpret_cast<uint32_t *>(wk + a.sm.u);      // used mask of parent p [W][K]
    int32_t *sOff = reinterpret_cast<int32_t *>(wk + a.sm.b);      // first code of parent p [K+1]
    uint8_t *codes = wk + a.sm.codes;
    uint32_t *sel = reinterpret_cast<uint32_t *>(wk + a.sm.sel);
    // coarse code position -> parent index: pidx[g] = the parent owning code position 16 g
    uint16_t *sPidx = reinterpret_cast<uint16_t *>(wk + a.sm.pidx);

    auto fped = [&](int b) { return reinterpret_cast<int32_t *>(scr + b * fb); };
    auto fused = [&](int b) { return reinterpret_cast<uint32_t *>(scr + b * fb + 4 * (int64_t)Kc); };
    // BT[NB][W][K]: B_p (plane 0) and B_{p,l} (planes 1..LMAX) of the level about to be expanded, built
    // by the previous level's update
    auto fbt = [&](int b) { return reinterpret_cast<uint32_t *>(scr + b * fb + (int64_t)Kc * (4 + 4 * W)); };
    auto fmap = [&](int b) { return scr + b * fb + (int64_t)Kc * (4 + 4 * W + 4 * W * NB); };

#ifdef FG_PROF
    long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ph_last_ = clock64();
#endif
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(a.work, 1);
        block_sync();
        const int item = s_item;
        if (item >= a.ngroup) {
#ifdef FG_PROF
            if (threadIdx.x == 0) {
                for (int k = 0; k < 8; ++k) atomicAdd(&fg_prof_cyc[k], (unsigned long long)ph_[k]);
                __threadfence();
                if (atomicAdd(&fg_prof_done, 1u) == gridDim.x - 1) {
                    printf("FGPROF W=%d setup %llu P %llu A+T %llu S2 %llu decode %llu U %llu final %llu S1 %llu\n", W, fg_prof_cyc[0],
                           fg_prof_cyc[1], fg_prof_cyc[2], fg_prof_cyc[3], fg_prof_cyc[4], fg_prof_cyc[5], fg_prof_cyc[6], fg_prof_cyc[7]);
                    for (int k = 0; k < 8; ++k) fg_prof_cyc[k] = 0;
                    fg_prof_done = 0;
                }
            }
#endif
            return;
        }
        const PairDesc pd = a.descs[a.order[item]];
        const int n1 = pd.n1, n2 = pd.n2, n2p = pd.n2p;
        const int32_t *vl1 = reinterpret_cast<const int32_t *>(a.blob + pd.vl1);
        const int32_t *vl2 = reinterpret_cast<const int32_t *>(a.blob + pd.vl2);
        const int32_t *pptr = reinterpret_cast<const int32_t *>(a.blob + pd.pptr);
        const int32_t *pq = reinterpret_cast<const int32_t *>(a.blob + pd.pq);
        const int32_t *pl = reinterpret_cast<const int32_t *>(a.blob + pd.pl);
        const uint32_t *adj2 = reinterpret_cast<const uint32_t *>(a.blob + pd.adj2);

        for (int x = threadIdx.x; x < n2 * W; x += NT) {
            const uint32_t v = __ldg(adj2 + x);
            const int u = x / W, y = x - u * W;
            sAdj[x] = v;
            sAdjH[(32 * (u >> 5) + (int)db_slot(1u << (u & 31))) * HRS + y] = v;
        }
        if (LAB) { // label planes: bit v of plane l of row u = edge (u, v) with label id l + 1
            const uint8_t *e2 = a.blob + pd.e2lab;
            for (int x = threadIdx.x; x < n2 * LMAX * W; x += NT) {
                const int u = x / (LMAX * W), r = x - u * (LMAX * W), l = r / W, w = r - l * W;
                uint32_t v = 0;
                for (int b = 0; b < 32 && 32 * w + b < n2; ++b) v |= (uint32_t)(__ldg(e2 + u * n2p + 32 * w + b) == l + 1) << b;
                sAdjL[x] = v;
                sAdjH[(32 * (u >> 5) + (int)db_slot(1u << (u & 31))) * HRS + W + r] = v;
            }
        }
        // root node: lambda empty, all of V2 remaining, PED 0
        if (threadIdx.x == 0) fped(0)[0] = 0;
        if (threadIdx.x < W * NB) {
            if (threadIdx.x < W) fused(0)[(int64_t)threadIdx.x * Kc] = 0u;
            fbt(0)[(int64_t)threadIdx.x * Kc] = 0u; // P_0 is empty
        }
        int N = 1, lo = 0, cur = 0;
        int64_t children = 0, parents = 0, algb = 0;
        for (int x = threadIdx.x; x < 64; x += NT) (&s_pnext2[0][0])[x] = 0u;
        block_sync(); // (previous pair's last reads of s_pnext2 / the scratch rows are done)

        for (int i = 0; i < n1; ++i) {
            const int32_t *Pped = fped(cur);
            const uint32_t *PusedT = fused(cur);
            const uint8_t *PmapT = fmap(cur);
            int32_t *Qped = fped(cur ^ 1);
            uint32_t *QusedT = fused(cur ^ 1);
            uint8_t *QmapT = fmap(cur ^ 1);
            const uint32_t *PBT = fbt(cur);
            uint32_t *QBT = fbt(cur ^ 1);
            const int pbeg = __ldg(pptr + i), d = __ldg(pptr + i + 1) - pbeg;
            const int dn = (LAB && i + 1 < n1) ? __ldg(pptr + i + 2) - __ldg(pptr + i + 1) : 0; // |P_{i+1}|
            // membership of P_{i+1} over q (for the next level's B, built during the update)
            uint32_t *s_pnext = s_pnext2[i & 1];
            for (int x = threadIdx.x; x < 32; x += NT) s_pnext2[(i + 1) & 1][x] = 0u; // used last in level i - 1
            if (i + 1 < n1) {
                const int nb = __ldg(pptr + i + 1), ne = __ldg(pptr + i + 2);
                for (int k = nb + threadIdx.x; k < ne; k += NT) {
                    const int q = __ldg(pq + k);
                    atomicOr(&s_pnext[q >> 5], 1u << (q & 31));
                    if (LAB) {
                        s_pnl[q] = (uint8_t)__ldg(pl + k); // (read only for q in P_{i+1})
                        s_pnq[k - nb] = q;
                    }
                }
            }
            for (int k = threadIdx.x; k < d; k += NT) {
                s_pq[k] = __ldg(pq + pbeg + k);
                s_pl[k] = __ldg(pl + pbeg + k);
            }
            // label planes with a non-empty B_{p,l} at this level (uniform)
            unsigned lmask = 0;
            if (LAB)
                for (int k = 0; k < d; ++k) {
                    const int l = __ldg(pl + pbeg + k);
                    if (l >= 1 && l <= LMAX) lmask |= 1u << (l - 1);
                }
            for (int k = threadIdx.x; k < NW * 132; k += NT) s_hist[k] = 0;
            const int vl1i = __ldg(vl1 + i);
            uint32_t Vm[W], Mm[W]; // existing targets / label mismatches, bit u of word u >> 5
#pragma unroll
            for (int s = 0; s < W; ++s) {
                const int u = lane + 32 * s;
                const int l2 = (u < n2) ? __ldg(vl2 + u) : 0;
                Vm[s] = __ballot_sync(FULL, u < n2);
                Mm[s] = __ballot_sync(FULL, u < n2 && l2 != vl1i);
                if (u < n2) sAdjH[(32 * s + (int)db_slot(1u << lane)) * HRS + CVW] = (l2 != vl1i) ? (uint32_t)c.vsub : 0u;
            }
            const int edd = c.edel * d, ee = c.edel + c.eins, dDel = c.vdel + edd;
            // method variant: the last level ranked by total = PED + completion (children's completions
            // differ from the parent's by vins for the used target and eins per edge to a used vertex)
            const bool lastTot = a.last_by_total && i == n1 - 1;
            // labelled: PED = ... - (ee - esub) cB - esub * (label matches); unlabelled: - ee cB
            const int eeB = LAB ? ee - c.esub : ee;
            // P_i list, zeroed histograms, P_{i+1} membership and cv words: visible to A through the
            // barriers of P's block scan
            FG_PH(0);

            // ---------------- P: parents -> used masks in shared memory, compact code offsets ----------------
            // Parent p has f_p = n2 - |used_p| substitution children + 1 deletion child; its rank codes
            // occupy codes[off_p, off_p + f_p + 1) in (target ascending, deletion last) = lin order.
            // odd run length: lane t touches parent t*ppt + x, conflict-free across the banks
            const int ppt = ((N + NT - 1) / NT) | 1;
            const int pb = min(N, threadIdx.x * ppt), pe = min(N, pb + ppt);
            // parent p's codes occupy [off_p, off_p + f_p + 1): its free targets ascending, then the deletion
            auto row_bytes = [&](int p) {
                int nc = 1;
#pragma unroll
                for (int w = 0; w < W; ++w) nc += __popc(Vm[w] & ~sU[w * Kc + p]);
                return nc;
            };
            int nloc = 0;
            for (int p = pb; p < pe; ++p) {
#pragma unroll
                for (int w = 0; w < W; ++w) sU[w * Kc + p] = PusedT[(int64_t)w * Kc + p];
                nloc += row_bytes(p);
            }
            int obase, dummy, ci, dummy2;
            block_scan2<NT>(nloc, 0, obase, dummy, ci, dummy2, s_tmp); // ci = candidates of the level
            for (int p = pb; p < pe; ++p) {
                sOff[p] = obase;
                const int nb = row_bytes(p);
                if (Kc <= 65535)
                    for (int g = (obase + 15) >> 4; 16 * g < obase + nb; ++g) sPidx[g] = (uint16_t)p;
                obase += nb;
            }
            if (threadIdx.x == 0) {
                sOff[N] = ci;
                for (int x = ci; x < ((ci + 3) & ~3); ++x) codes[x] = (uint8_t)CODE_INVALID;
            }
            block_sync();
            FG_PH(1);

            // ---------------- A + T: branch, rank codes, histogram, threshold ----------------
            const int chunk = (N + NW - 1) / NW;
            const int p0 = min(N, warp * chunk), p1 = min(N, p0 + chunk);
            int base = lo, below = 0, tcode = 256, rq = 0, below_add = 0;
            bool keepall = ci <= K, retry = false;
            // exact histogram of rank codes 1..win (win <= 127): one private row per warp, shared atomics
            int *whist = s_hist + warp * 132 + 3;
            auto hist_add = [&](int code) {
                if ((unsigned)(code - 1) < (unsigned)win) atomicAdd(&whist[code], 1);
            };
            for (;;) {
                if (N >= NT / 2) {
                    // wide frontier: thread per parent, iterating only the parent's free targets (no idle lanes)
                    for (int p = threadIdx.x; p < N; p += NT) {
                        const int pedp = Pped[p];
                        uint32_t U[W], B[NB][W];
                        // B_p: images of the earlier g1 neighbours of v_i (replaces VFrom/VTo)
#pragma unroll
                        for (int w = 0; w < W; ++w) U[w] = sU[w * Kc + p];
#pragma unroll
                        for (int b = 0; b < NB; ++b)
#pragma unroll
                            for (int w = 0; w < W; ++w)
                                B[b][w] = (b == 0 || ((lmask >> (b - 1)) & 1u)) ? PBT[((int64_t)b * W + w) * Kc + p] : 0u;
                        uint8_t *crow = codes + sOff[p];
                        const int comp = lastTot ? completion_of<W>(U, sAdj, n2, pd.m2, c) : 0; // parent's completion
                        const int pb = pedp - base + 1 + edd + (lastTot ? comp - c.vins : 0);
                        const int einsT = lastTot ? 0 : c.eins; // (total: the eins cnt of the child cancels)
                        int r = 0;
#pragma unroll
                        for (int w = 0; w < W; ++w) {
                            // child for the free target whose bit is lb (lowest set bit of F, no bit index)
                            auto child_code = [&](uint32_t lb) -> int {
                                const uint32_t *row = sAdjH + (32 * w + (int)db_slot(lb)) * HRS;
                                uint32_t rv[HRS]; // W row words (+ label planes) + cv(i, u), vector loads
                                if constexpr (HRS == 2) {
                                    const uint2 q = *reinterpret_cast<const uint2 *>(row);
                                    rv[0] = q.x; rv[1] = q.y;
                                } else {
#pragma unroll
                                    for (int h = 0; h < HRS; h += 4) {
                                        const uint4 q = *reinterpret_cast<const uint4 *>(row + h);
                                        rv[h] = q.x; rv[h + 1] = q.y; rv[h + 2] = q.z; rv[h + 3] = q.w;
                                    }
                                }
                                int cnt = 0, cb = 0, mt = 0;
#pragma unroll
                                for (int x = 0; x < W; ++x) {
                                    cnt += __popc(rv[x] & U[x]);
                                    cb += __popc(rv[x] & B[0][x]);
                                }
                                if (LAB) { // edges (u, t) whose g2 label equals the g1 label of (v_i, v_q)
                                    // (the per-label sets are disjoint -- t is the image of one q, the edge (u, t)
                                    // has one label -- so one POPC of their union counts them all)
#pragma unroll
                                    for (int x = 0; x < W; ++x) {
                                        uint32_t mw = 0u;
#pragma unroll
                                        for (int l = 0; l < LMAX; ++l)
                                            if ((lmask >> l) & 1u) mw |= rv[W + l * W + x] & B[1 + l][x];
                                        mt += __popc(mw);
                                    }
                                }
                                // rank code = clamp(PED - base + 1, 0, win + 1), with pb = PED_p - base + 1 + edel d_i
                                const int x = pb + (int)rv[CVW] + einsT * cnt - eeB * cb - (LAB ? c.esub * mt : 0);
                                return min(max(x, 0), win + 1);
                            };
                            uint32_t F = Vm[w] & ~U[w];
                            while (F) { // FG_CZ free targets per iteration (independent chains); lb = 0: no child
                                uint32_t lz[FG_CZ];
#pragma unroll
                                for (int z = 0; z < FG_CZ; ++z) { lz[z] = F & (0u - F); F ^= lz[z]; }
                                int cz[FG_CZ];
#pragma unroll
                                for (int z = 0; z < FG_CZ; ++z) cz[z] = child_code(lz[z]);
#pragma unroll
                                for (int z = 0; z < FG_CZ; ++z)
                                    if (z == 0 || lz[z]) {
                                        crow[r + z] = (uint8_t)cz[z];
                                        atomicAdd(&whist[cz[z]], 1); // codes 0 and win+1 land in unused bins
                                    }
                                r += 1;
#pragma unroll
                                for (int z = 1; z < FG_CZ; ++z) r += (lz[z] != 0u);
                            }
                        }
                        const int cdel = rank_code(pedp + dDel + comp, base, win); // deletion child (C5)
                        crow[r] = (uint8_t)cdel;
                        hist_add(cdel);
                    }
                } else {
                    // narrow frontier (or labelled edges): warp per parent, lane l owns targets l + 32 s
                    for (int p = p0; p < p1; ++p) {
                        const int pedp = Pped[p];
                        uint32_t U[W];
#pragma unroll
                        for (int w = 0; w < W; ++w) U[w] = sU[w * Kc + p];
                        uint32_t B[NB][W];
#pragma unroll
                        for (int b = 0; b < NB; ++b)
#pragma unroll
                            for (int w = 0; w < W; ++w)
                                B[b][w] = (b == 0 || ((lmask >> (b - 1)) & 1u)) ? PBT[((int64_t)b * W + w) * Kc + p] : 0u;
                        int ped_s[W];
                        int comp = 0; // (variant) the parent's completion
                        if (lastTot) {
                            int e2u2 = 0, usedc = 0;
#pragma unroll
                            for (int s = 0; s < W; ++s) {
                                const int u = lane + 32 * s;
                                usedc += __popc(U[s]);
                                if (u < n2 && ((U[s] >> lane) & 1u))
#pragma unroll
                                    for (int w = 0; w < W; ++w) e2u2 += __popc(sAdj[u * W + w] & U[w]);
                            }
                            e2u2 = __reduce_add_sync(FULL, e2u2);
                            comp = c.vins * (n2 - usedc) + c.eins * (pd.m2 - e2u2 / 2);
                        }
#pragma unroll
                        for (int s = 0; s < W; ++s) {
                            const int u = lane + 32 * s;
                            int cnt = 0, cb = 0, mt = 0;
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                const uint32_t rw = (u < n2) ? sAdj[u * W + w] : 0u;
                                cnt += __popc(rw & U[w]);
                                cb += __popc(rw & B[0][w]);
                            }
                            if (LAB) { // (disjoint per-label sets: one POPC of their union)
#pragma unroll
                                for (int w = 0; w < W; ++w) {
                                    uint32_t mw = 0u;
#pragma unroll
                                    for (int l = 0; l < LMAX; ++l)
                                        if ((lmask >> l) & 1u) mw |= ((u < n2) ? sAdjL[(u * LMAX + l) * W + w] : 0u) & B[1 + l][w];
                                    mt += __popc(mw);
                                }
                            }
                            ped_s[s] = pedp + (int)((Mm[s] >> lane) & 1u) * c.vsub + edd + (lastTot ? 0 : c.eins * cnt) - eeB * cb -
                                       (LAB ? c.esub * mt : 0) + (lastTot ? comp - c.vins : 0);
                        }
                        uint8_t *crow = codes + sOff[p];
                        int r = 0;
                        const unsigned lmk = lanemask_lt();
#pragma unroll
                        for (int s = 0; s < W; ++s) {
                            const int u = lane + 32 * s;
                            const bool sub = (u < n2) && !((U[s] >> lane) & 1u);
                            const unsigned bal = __ballot_sync(FULL, sub);
                            const int code = sub ? rank_code(ped_s[s], base, win) : CODE_INVALID;
                            if (sub) crow[r + __popc(bal & lmk)] = (uint8_t)code;
                            hist_add(code);
                            r += __popc(bal);
                        }
                        if (lane == 0) {
                            const int cdel = rank_code(pedp + dDel + comp, base, win);
                            crow[r] = (uint8_t)cdel;
                            hist_add(cdel);
                        }
                        __syncwarp();
                    }
                }
                block_sync();
                { // T: every warp derives the same threshold from the per-warp histograms (4 codes per lane)
                    int hv[4] = {0, 0, 0, 0}; // codes 4 lane + 1 .. 4 lane + 4 (one 16-byte read per warp row)
                    for (int w = 0; w < NW; ++w) {
                        const int4 h4 = *reinterpret_cast<const int4 *>(s_hist + w * 132 + 4 + 4 * lane);
                        hv[0] += h4.x; hv[1] += h4.y; hv[2] += h4.z; hv[3] += h4.w;
                    }
                    int sum = 0;
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        if (4 * lane + 1 + x > win) hv[x] = 0;
                        sum += hv[x];
                    }
                    int incl = sum;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const unsigned hm = __ballot_sync(FULL, !keepall && (below + incl >= K));
                    below_add = __shfl_sync(FULL, incl, 31);
                    retry = !keepall && hm == 0u;
                    if (hm) {
                        const int L = __ffs(hm) - 1;
                        int c2 = below + incl - sum, tc = 0, rr = 0;
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            if (tc == 0 && c2 + hv[x] >= K) { tc = 4 * lane + 1 + x; rr = K - c2; }
                            c2 += hv[x];
                        }
                        tcode = __shfl_sync(FULL, tc, L);
                        rq = __shfl_sync(FULL, rr, L);
                    }
                }
                if (!retry) break; // (uniform: every warp computed the same value)
                // the K-th smallest PED lies beyond the window: slide it (all codes < base are kept)
                block_sync(); // all warps have read the histograms
                below += below_add;
                base += win;
                for (int k = threadIdx.x; k < NW * 132; k += NT) s_hist[k] = 0;
                block_sync();
            }

            FG_PH(2);
            // ---------------- S: selection by segment scan over the compact code words ----------------
            int Nn;
            {
                const uint32_t *cw = reinterpret_cast<const uint32_t *>(codes);
                const int nwords = (ci + 3) >> 2;
                // odd segment length: lane t reads word t*seg + x, conflict-free across the 32 banks
                const int seg = ((nwords + NT - 1) / NT) | 1;
                const int w0 = min(nwords, threadIdx.x * seg), w1 = min(nwords, w0 + seg);
                if (keepall) { tcode = 256; rq = 0; }
                // SWAR byte masks (codes are 0..win+1 <= 128 or 255): bit 7 of each byte set where
                //   ge(t): byte >= t (t <= 128),  valid: byte != 255
                const uint32_t t4 = (uint32_t)tcode * 0x01010101u, t41 = t4 + 0x01010101u;
                auto ge = [](uint32_t x, uint32_t tt) { return (((x | 0x80808080u) - tt) | x) & 0x80808080u; };
                auto valid = [](uint32_t x) { const uint32_t y = ~x; return (((y & 0x7f7f7f7fu) + 0x7f7f7f7fu) | y) & 0x80808080u; };
                int lt = 0, eq = 0;
                unsigned long long cmask = 0ull; // words of the run holding a code <= t (runs of <= 64 words)
#pragma unroll 4
                for (int x = w0; x < w1; ++x) {
                    const uint32_t v = cw[x];
                    if (keepall) lt += __popc(valid(v));
                    else {
                        const int g0 = __popc(ge(v, t4));
                        const int g1 = __popc(ge(v, t41));
                        lt += 4 - g0;
                        eq += g0 - g1;
                        if (g1 != 4) cmask |= 1ull << ((x - w0) & 63);
                    }
                }
                int ltpre, eqpre, lttot, eqtot;
                block_scan2<NT>(lt, eq, ltpre, eqpre, lttot, eqtot, s_tmp);
                FG_PH(7);
                Nn = keepall ? lttot : K;
                int out = ltpre + min(rq, eqpre), eq_seen = eqpre;
                if (lt + (eqpre < rq ? eq : 0) > 0) {
                    // survivors are written as flat code positions; the parent is found in the balanced decode.
                    // Runs of <= 64 words revisit only the words pass 1 marked.
                    const bool sparse = !keepall && seg <= 64;
                    for (int x = w0; x < w1; ++x) {
                        if (sparse) {
                            if (!cmask) break;
                            x = w0 + __ffsll((long long)cmask) - 1;
                            cmask &= cmask - 1;
                        }
                        const uint32_t v = cw[x];
                        uint32_t m;
                        if (keepall) m = valid(v);
                        else {
                            const uint32_t g0 = ge(v, t4);
                            m = ~g0 & 0x80808080u;
                            uint32_t meq = g0 & ~ge(v, t41);
                            if (meq) { // ties at t are admitted in code order up to the quota rq
                                const int ne = __popc(meq);
                                if (eq_seen + ne <= rq) m |= meq;
                                else
                                    for (int z = rq - eq_seen; z > 0; --z) { const uint32_t low = meq & (0u - meq); m |= low; meq ^= low; }
                                eq_seen += ne;
                            }
                        }
                        // up to four survivors of the word, written without a bit loop (no chain between them)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            if ((m >> (8 * b + 7)) & 1u) sel[out + __popc(m & ((1u << (8 * b)) - 1u))] = (uint32_t)(4 * x + b);
                        out += __popc(m);
                    }
                }
                if (threadIdx.x == 0) {
                    s_lo = 0x7fffffff;
                    if (a.levels_out) {
                        a.levels_out[3 * i] = N;
                        a.levels_out[3 * i + 1] = ci;
                        a.levels_out[3 * i + 2] = keepall ? -1 : (int64_t)(base + tcode - 1);
                    }
                }
            }
            block_sync();
            FG_PH(3);

            // ---------------- decode survivors + U part 1 (balanced: thread per survivor) ----------------
            // flat code position -> (p, child j); PED from the code (recomputed for a saturated code);
            // the survivor's PED and used mask go straight to the next frontier (coalesced over k)
            int pmin = 0x7fffffff;
            for (int kb = threadIdx.x; kb < Nn; kb += 4 * NT) {
            // the positions of up to four survivors are read first, so their decode chains overlap
            // (the in-place sel[] writes below would otherwise order every load after the previous store)
            int idxv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) idxv[u] = (kb + u * NT < Nn) ? (int)sel[kb + u * NT] : 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = kb + u * NT;
                if (k >= Nn) break;
                const int idx = idxv[u];
                int p;
                if (Kc <= 65535) { // owner of position 16 (idx / 16), advanced to the owner of idx
                    p = sPidx[idx >> 4];
                    while (sOff[p + 1] <= idx) ++p;
                } else { // last parent with off_p <= idx
                    p = 0;
                    int phi = N - 1;
                    while (p < phi) {
                        const int mid = (p + phi + 1) >> 1;
                        if (sOff[mid] <= idx) p = mid; else phi = mid - 1;
                    }
                }
                const int rnk = idx - sOff[p];
                const int code = codes[idx];
                uint32_t Up[W];
                int j = n2; // past every target: the deletion child
                int rr = rnk;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    Up[w] = sU[w * Kc + p];
                    const uint32_t F = Vm[w] & ~Up[w];
                    const int cnt = __popc(F);
                    if (rr >= 0 && rr < cnt) j = 32 * w + select_bit(F, rr);
                    rr -= cnt;
                }
                sel[k] = ((uint32_t)p << 8) | (uint32_t)j;
                int ped;
                if (code >= 1 && code <= win) ped = base + code - 1;
                else { // saturated rank code: recompute the child's PED (rare)
                    const int pedp = Pped[p];
                    if (j == n2) ped = pedp + dDel;
                    else {
                        int cnt = 0, cb = 0, mt = 0;
#pragma unroll
                        for (int w = 0; w < W; ++w) {
                            cnt += __popc(sAdj[j * W + w] & Up[w]);
                            cb += __popc(sAdj[j * W + w] & PBT[(int64_t)w * Kc + p]);
                        }
                        if (LAB)
#pragma unroll
                            for (int l = 0; l < LMAX; ++l)
                                if ((lmask >> l) & 1u)
#pragma unroll
                                    for (int w = 0; w < W; ++w)
                                        mt += __popc(sAdjL[(j * LMAX + l) * W + w] & PBT[((int64_t)(1 + l) * W + w) * Kc + p]);
                        ped = pedp + ((vl2[j] == vl1i) ? 0 : c.vsub) + edd + c.eins * cnt - eeB * cb - (LAB ? c.esub * mt : 0);
                    }
                    if (lastTot) { // variant: the code stands for the total; recompute the child's completion
                        uint32_t Uc[W];
#pragma unroll
                        for (int w = 0; w < W; ++w) Uc[w] = Up[w] | ((j < n2 && (j >> 5) == w) ? (1u << (j & 31)) : 0u);
                        ped += completion_of<W>(Uc, sAdj, n2, pd.m2, c);
                    }
                }
                Qped[k] = ped; // (variant, last level: the total)
#pragma unroll
                for (int w = 0; w < W; ++w)
                    QusedT[(int64_t)w * Kc + k] = Up[w] | ((j < n2 && (j >> 5) == w) ? (1u << (j & 31)) : 0u);
                pmin = min(pmin, ped);
            }
            }
            pmin = __reduce_min_sync(FULL, (unsigned)pmin); // PEDs are >= 0: unsigned min = signed min
            if (lane == 0 && pmin != 0x7fffffff) atomicMin(&s_lo, pmin);
            block_sync(); // the (p, j) of every survivor is in sel
            FG_PH(4);

            // ---------------- U part 2: lambda columns (and B of the next level), coalesced over k ----------------
            {
                const int nk4 = (Nn + 3) >> 2;
                const bool inext = (i + 1 < n1) && ((s_pnext[i >> 5] >> (i & 31)) & 1u);
                for (int x = threadIdx.x; x < nk4; x += NT) {
                    const int k0 = 4 * x;
                    int pp[4];
                    uint32_t last = 0, Bn[4][W]; // (unlabelled: B of the next level, built during the copy)
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int k = min(k0 + b, Nn - 1);
                        const uint32_t v = sel[k];
                        pp[b] = (int)(v >> 8);
                        const int j = (int)(v & 255u);
                        last |= ((j == n2) ? (uint32_t)MAP_DEL : (uint32_t)j) << (8 * b);
#pragma unroll
                        for (int w = 0; w < W; ++w)
                            Bn[b][w] = (!LAB && inext && j < n2 && (j >> 5) == w) ? (1u << (j & 31)) : 0u;
                    }
                    // lambda columns 0..i-1: gather 8 columns x 4 survivors into registers, then store
                    // (loads of a chunk are issued together; QmapT/PmapT are distinct buffers)
                    // (software-pipelined: the gathers of chunk c + 1 are issued before the stores of chunk c)
                    auto gather8 = [&](int q0, uint32_t (&wd)[8]) {
#pragma unroll
                        for (int z = 0; z < 8; ++z) {
                            const int q = min(q0 + z, i - 1);
                            const uint8_t *row = PmapT + (int64_t)q * Kc;
                            // plain loads: this CTA wrote the column in the previous level (visible after the
                            // barrier); the read-only (.nc) path is not coherent with such writes
                            wd[z] = (uint32_t)row[pp[0]] | ((uint32_t)row[pp[1]] << 8) |
                                    ((uint32_t)row[pp[2]] << 16) | ((uint32_t)row[pp[3]] << 24);
                        }
                    };
                    uint32_t wnext[8];
                    if (i > 0) gather8(0, wnext);
                    for (int q0 = 0; q0 < i; q0 += 8) {
                        uint32_t wd[8];
#pragma unroll
                        for (int z = 0; z < 8; ++z) wd[z] = wnext[z];
                        if (q0 + 8 < i) gather8(q0 + 8, wnext);
#pragma unroll
                        for (int z = 0; z < 8; ++z) {
                            const int q = q0 + z;
                            if (q >= i) break;
                            *reinterpret_cast<uint32_t *>(QmapT + (int64_t)q * Kc + k0) = wd[z];
                            if (!LAB && ((s_pnext[q >> 5] >> (q & 31)) & 1u)) { // v_q is an earlier neighbour of v_{i+1}
#pragma unroll
                                for (int b = 0; b < 4; ++b) {
                                    const uint32_t t = (wd[z] >> (8 * b)) & 0xffu;
#pragma unroll
                                    for (int w = 0; w < W; ++w)
                                        Bn[b][w] |= (t != (uint32_t)MAP_DEL && (int)(t >> 5) == w) ? (1u << (t & 31)) : 0u;
                                }
                            }
                        }
                    }
                    *reinterpret_cast<uint32_t *>(QmapT + (int64_t)i * Kc + k0) = last;
                    if (i + 1 < n1) {
                        if (!LAB) {
#pragma unroll
                            for (int w = 0; w < W; ++w)
#pragma unroll
                                for (int b = 0; b < 4; ++b) QBT[(int64_t)w * Kc + k0 + b] = Bn[b][w];
                        } else {
                            // labelled: B and its label planes from the (few) columns of P_{i+1}, after the copy
                            uint32_t Bl[4][NB][W];
#pragma unroll
                            for (int b = 0; b < 4; ++b)
#pragma unroll
                                for (int pl2 = 0; pl2 < NB; ++pl2)
#pragma unroll
                                    for (int w = 0; w < W; ++w) Bl[b][pl2][w] = 0u;
                            for (int e = 0; e < dn; ++e) {
                                const int q = s_pnq[e], ql = s_pnl[q];
                                uint32_t wv = last; // column i: the survivors' own targets
                                if (q < i) {
                                    const uint8_t *row = QmapT + (int64_t)q * Kc; // (this thread wrote it above)
                                    wv = *reinterpret_cast<const uint32_t *>(row + k0);
                                }
#pragma unroll
                                for (int b = 0; b < 4; ++b) {
                                    const uint32_t t = (wv >> (8 * b)) & 0xffu;
#pragma unroll
                                    for (int w = 0; w < W; ++w) {
                                        const uint32_t bt = (t != (uint32_t)MAP_DEL && (int)(t >> 5) == w) ? (1u << (t & 31)) : 0u;
                                        Bl[b][0][w] |= bt;
#pragma unroll
                                        for (int pl2 = 1; pl2 < NB; ++pl2) Bl[b][pl2][w] |= (ql == pl2) ? bt : 0u;
                                    }
                                }
                            }
#pragma unroll
                            for (int pl2 = 0; pl2 < NB; ++pl2)
#pragma unroll
                                for (int w = 0; w < W; ++w)
#pragma unroll
                                    for (int b = 0; b < 4; ++b) QBT[((int64_t)pl2 * W + w) * Kc + k0 + b] = Bl[b][pl2][w];
                        }
                    }
                }
            }
            children += ci;
            parents += N;
            // B_alg(i) = N_i (4 + b d_i) + N_{i+1} (b i + 4) + N_{i+1} (b (i+1) + 4), b = 1
            algb += (int64_t)N * (4 + d) + (int64_t)Nn * (2 * i + 9);
            block_sync();
            FG_PH(5);
            N = Nn;
            lo = s_lo;
            cur ^= 1;
        }

        // ---------------- Finalize: insertion completion + argmin ----------------
        if (threadIdx.x == 0) s_best = ~0ull;
        block_sync();
        {
            const int32_t *Pped = fped(cur);
            const uint32_t *PusedT = fused(cur);
            unsigned long long mykey = ~0ull;
            for (int k = threadIdx.x; k < N; k += NT) {
                uint32_t U[W];
                int usedc = 0, e2u2 = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) { U[w] = PusedT[(int64_t)w * Kc + k]; usedc += __popc(U[w]); }
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    uint32_t bits = U[w];
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        const int u = 32 * w + b;
#pragma unroll
                        for (int x = 0; x < W; ++x) e2u2 += __popc(sAdj[u * W + x] & U[x]);
                    }
                }
                // (variant: the last level already stored PED + completion; n1 = 0 has no last level)
                const int64_t total = (a.last_by_total && n1 > 0)
                                          ? (int64_t)Pped[k]
                                          : (int64_t)Pped[k] + (int64_t)c.vins * (n2 - usedc) + (int64_t)c.eins * (pd.m2 - e2u2 / 2);
                mykey = min(mykey, ((unsigned long long)total << 32) | (unsigned)k);
            }
            // argmin by (total, position): warp minimum, then one shared atomic per warp
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mykey = min(mykey, __shfl_xor_sync(FULL, mykey, o));
            if (lane == 0 && mykey != ~0ull) atomicMin(&s_best, mykey);
            block_sync();
            const unsigned long long best = s_best;
            const int kb = (int)(best & 0xffffffffull);
            const uint8_t *PmapT = fmap(cur);
            for (int q = threadIdx.x; q < n1; q += NT) {
                const int t = PmapT[(int64_t)q * Kc + kb];
                a.map_out[pd.map_out + q] = (t == MAP_DEL) ? -1 : t;
            }
            FG_PH(6);
            if (threadIdx.x == 0) {
                const int pidx = a.order[item];
                a.cost_out[pidx] = (int64_t)(best >> 32);
                a.children_out[pidx] = children;
                a.parents_out[pidx] = parents;
                a.algbytes_out[pidx] = algb;
            }
        }
        block_sync();
    }
}

} // namespace fg
