// batch_kernel.cuh -- the batched K-Best search: one CTA runs one (g1, g2) pair through all
// levels of Alg. 1 and then takes the next pair from a work counter.
//
// Per level i (g1 vertex v_i, reading C4) the CTA runs:
//   A  Branch (Alg. 2).  A warp takes one parent at a time;
//      lane l owns the g2 vertices u = l + 32 s (s < W), whose bit-packed adjacency rows stay in
//      registers for the whole pair.  The child PED is the paper's incremental evaluation
//      PED = E(parent) + c(v<-u) + Imp_cost with the three implied-edge cases of PAPER.md:103-116
//      regrouped into popcounts:
//          Delta(u)   = cv(i,u) + edel*d_i + eins*cnt_p(u) - (edel+eins)*cB_p(u) + esub*mis_p(u)
//          Delta(DEL) = vdel + edel*d_i
//      cnt_p(u) = popc(adj2[u] & used_p), cB_p(u) = popc(adj2[u] & B_p), B_p = images of the
//      earlier g1 neighbours of v_i (replaces the paper's VFrom/VTo vectors).
//      Each child is written as a one-byte rank code (PED - base + 1, saturated) and counted in
//      a shared-memory histogram.  Children never reach HBM.
//   T  Threshold (PAPER.md:261-265 local/global ranking, replaced): the histogram prefix gives
//      the threshold PED t and the quota r of ties at t; exactly min(K, c_i) children are kept,
//      the smallest under (PED, parent, child) (reading C12).  No sort.
//   B  Per-warp counts of codes < t and == t (SIMD byte compares), then a warp-level prefix gives
//      each warp its tie admissions and output offset.
//   C  Update: survivors are compacted in (parent, child) order (C13) and
//      the next frontier (PED, used bitmask, lambda row) is written with coalesced word copies.
// After the last level, each survivor gets the insertion completion (C6) and the
// argmin by (total, position) is written out (C10).
#pragma once
#include <cstdint>

namespace fg {

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAP_DEL = 255;     // lambda entry of a deleted g1 vertex
constexpr int CODE_INVALID = 255; // no child in this slot (used target / padding)

struct Costs {
    int vsub, vdel, vins, esub, edel, eins;
};

// One pair inside the device blob (byte offsets into the blob).
struct PairDesc {
    int32_t n1, n2, m1, m2;
    int32_t labelled, n2p;       // n2p: row stride of the e2lab byte matrix (multiple of 4)
    int64_t vl1, vl2;            // int32[n1], int32[n2]
    int64_t pptr, pq, pl;        // int32[n1+1], int32[m1], int32[m1]  (P_i lists)
    int64_t adj2;                // uint32[n2 * W]
    int64_t e2lab;               // uint8[n2p * n2p] (labelled only): g2 edge label id + 1, 0 = no edge
    int64_t map_out;             // element offset of this pair's mapping in the output array
};

struct BatchArgs {
    const PairDesc *descs;
    const int32_t *order;   // pair indices of this launch, in scheduling order
    int32_t ngroup;
    const uint8_t *blob;
    int32_t *work;          // dynamic scheduler counter (zeroed before launch)
    Costs c;
    int32_t K;
    int32_t win;            // exact rank window: codes 1..win; win+1 = saturated
    int32_t n1s;            // lambda row stride in bytes (multiple of 4, >= max n1)
    int32_t n1max;          // max n1 in this launch (P-list smem size)
    int32_t csmax;          // max code row stride
    int32_t e2bytes;        // smem bytes for e2lab (labelled launches)
    int32_t codes_in_smem, sel_in_smem;
    uint8_t *scratch;       // per-CTA frontier / code / selection scratch
    int64_t scratch_stride;
    int64_t *cost_out;
    int32_t *map_out;
    int64_t *children_out;
    int64_t *parents_out;
    int64_t *algbytes_out;  // per pair: algorithmic frontier bytes of the search
    int64_t *levels_out;    // NULL, or [3 * n1] for a single-pair launch
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int W>
struct FrontierView {
    int32_t *ped;
    uint32_t *used;
    uint8_t *map;
};

// Scalar recomputation of one child's PED (used when its rank code was saturated; rare).
template <int W, bool LAB>
__device__ int child_ped_scalar(const Costs &c, int pedp, const uint32_t *Up, const uint8_t *mrow, int j,
                                int n2, int n2p, int d, const int32_t *s_pq, const int32_t *s_pl,
                                int vl1i, const int32_t *vl2, const uint32_t *adj2, const uint8_t *s_e2) {
    if (j == n2) return pedp + c.vdel + c.edel * d;
    int cv = (vl2[j] == vl1i) ? 0 : c.vsub;
    int cnt = 0, cb = 0, mis = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) cnt += __popc(adj2[j * W + w] & Up[w]);
    for (int k = 0; k < d; ++k) {
        int t = mrow[s_pq[k]];
        if (t == MAP_DEL) continue;
        if (!LAB) {
            cb += (adj2[j * W + (t >> 5)] >> (t & 31)) & 1u;
        } else {
            int e = s_e2[t * n2p + j];
            cb += (e != 0);
            mis += (e != 0) & (e != s_pl[k]);
        }
    }
    return pedp + cv + c.edel * d + c.eins * cnt - (c.edel + c.eins) * cb + c.esub * mis;
}

template <int W, bool LAB>
__global__ void __launch_bounds__(256) kbest_batch_kernel(const BatchArgs a) {
    extern __shared__ __align__(16) uint8_t dsmem[];
    __shared__ int s_hist[256];
    __shared__ int s_wcnt[32], s_wlt[32], s_weq[32], s_weqpre[32], s_wout[32];
    __shared__ int s_item, s_keepall, s_tcode, s_r, s_retry, s_nnext, s_lo, s_below_add;
    __shared__ int64_t s_ci;
    __shared__ unsigned long long s_best;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const Costs c = a.c;
    const int K = a.K, win = a.win, n1s = a.n1s;

    // dynamic smem carve: P list, e2lab, codes (optional), sel (optional)
    int32_t *s_pq = reinterpret_cast<int32_t *>(dsmem);
    int32_t *s_pl = s_pq + a.n1max;
    uint8_t *s_e2 = reinterpret_cast<uint8_t *>(s_pl + a.n1max);
    uint8_t *sm_next = s_e2 + a.e2bytes;

    // per-CTA scratch carve (global)
    uint8_t *scr = a.scratch + (int64_t)blockIdx.x * a.scratch_stride;
    FrontierView<W> F[2];
    F[0].ped = reinterpret_cast<int32_t *>(scr);
    F[1].ped = F[0].ped + K;
    F[0].used = reinterpret_cast<uint32_t *>(F[1].ped + K);
    F[1].used = F[0].used + (int64_t)K * W;
    F[0].map = reinterpret_cast<uint8_t *>(F[1].used + (int64_t)K * W);
    F[1].map = F[0].map + (int64_t)K * n1s;
    uint8_t *gnext = F[1].map + (int64_t)K * n1s;
    uint8_t *codes;
    uint32_t *sel;
    if (a.codes_in_smem) { codes = sm_next; sm_next += ((int64_t)K * a.csmax + 15) & ~15ll; }
    else { codes = gnext; gnext += ((int64_t)K * a.csmax + 15) & ~15ll; }
    if (a.sel_in_smem) sel = reinterpret_cast<uint32_t *>(sm_next);
    else sel = reinterpret_cast<uint32_t *>(gnext);

    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(a.work, 1);
        __syncthreads();
        const int item = s_item;
        if (item >= a.ngroup) return;
        const PairDesc pd = a.descs[a.order[item]];
        const int n1 = pd.n1, n2 = pd.n2, n2p = pd.n2p;
        const int cs = (n2 + 1 + 3) & ~3;
        const int32_t *vl1 = reinterpret_cast<const int32_t *>(a.blob + pd.vl1);
        const int32_t *vl2 = reinterpret_cast<const int32_t *>(a.blob + pd.vl2);
        const int32_t *pptr = reinterpret_cast<const int32_t *>(a.blob + pd.pptr);
        const int32_t *pq = reinterpret_cast<const int32_t *>(a.blob + pd.pq);
        const int32_t *pl = reinterpret_cast<const int32_t *>(a.blob + pd.pl);
        const uint32_t *adj2 = reinterpret_cast<const uint32_t *>(a.blob + pd.adj2);

        // lane-owned adjacency rows and labels of u = lane + 32 s
        uint32_t A[W][W];
        int vl2r[W];
#pragma unroll
        for (int s = 0; s < W; ++s) {
            int u = lane + 32 * s;
#pragma unroll
            for (int w = 0; w < W; ++w) A[s][w] = (u < n2) ? __ldg(adj2 + u * W + w) : 0u;
            vl2r[s] = (u < n2) ? __ldg(vl2 + u) : 0;
        }
        if (LAB) {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(a.blob + pd.e2lab);
            uint32_t *dst = reinterpret_cast<uint32_t *>(s_e2);
            for (int x = threadIdx.x; x < n2p * n2p / 4; x += blockDim.x) dst[x] = __ldg(src + x);
        }
        // root node: lambda empty, all of V2 remaining, PED 0
        if (threadIdx.x == 0) F[0].ped[0] = 0;
        if (threadIdx.x < W) F[0].used[threadIdx.x] = 0u;
        int N = 1, lo = 0, cur = 0;
        int64_t children = 0, parents = 0, algb = 0;

        for (int i = 0; i < n1; ++i) {
            const FrontierView<W> P = F[cur], Q = F[cur ^ 1];
            const int pbeg = __ldg(pptr + i), d = __ldg(pptr + i + 1) - pbeg;
            for (int k = threadIdx.x; k < d; k += blockDim.x) {
                s_pq[k] = __ldg(pq + pbeg + k);
                s_pl[k] = __ldg(pl + pbeg + k);
            }
            for (int k = threadIdx.x; k < 256; k += blockDim.x) s_hist[k] = 0;
            const int vl1i = __ldg(vl1 + i);
            int cv[W];
#pragma unroll
            for (int s = 0; s < W; ++s) cv[s] = (vl2r[s] == vl1i) ? 0 : c.vsub;
            const int edd = c.edel * d, ee = c.edel + c.eins, dDel = c.vdel + edd;
            const int chunk = (N + NW - 1) / NW;
            const int p0 = min(N, warp * chunk), p1 = min(N, p0 + chunk);
            int base = lo, below = 0;
            bool first = true;
            __syncthreads();

            // ---------------- A + T: branch, rank codes, histogram, threshold ----------------
            for (;;) {
                int wcount = 0;
                for (int p = p0; p < p1; ++p) {
                    const int pedp = P.ped[p];
                    uint32_t U[W];
#pragma unroll
                    for (int w = 0; w < W; ++w) U[w] = P.used[(int64_t)p * W + w];
                    const uint8_t *mrow = P.map + (int64_t)p * n1s;
                    int ped_s[W];
                    if (!LAB) {
                        uint32_t B[W];
#pragma unroll
                        for (int w = 0; w < W; ++w) B[w] = 0u;
                        for (int k0 = 0; k0 < d; k0 += 32) {
                            const int k = k0 + lane;
                            const int t = (k < d) ? mrow[s_pq[k]] : MAP_DEL;
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                const unsigned bit = (t != MAP_DEL && (t >> 5) == w) ? (1u << (t & 31)) : 0u;
                                B[w] |= __reduce_or_sync(FULL, bit);
                            }
                        }
#pragma unroll
                        for (int s = 0; s < W; ++s) {
                            int cnt = 0, cb = 0;
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                cnt += __popc(A[s][w] & U[w]);
                                cb += __popc(A[s][w] & B[w]);
                            }
                            ped_s[s] = pedp + cv[s] + edd + c.eins * cnt - ee * cb;
                        }
                    } else {
                        int cb[W], mis[W];
#pragma unroll
                        for (int s = 0; s < W; ++s) { cb[s] = 0; mis[s] = 0; }
                        for (int k0 = 0; k0 < d; k0 += 32) {
                            const int k = k0 + lane;
                            int t = MAP_DEL, l = 0;
                            if (k < d) { t = mrow[s_pq[k]]; l = s_pl[k]; }
                            const int kn = min(32, d - k0);
                            for (int kk = 0; kk < kn; ++kk) {
                                const int tt = __shfl_sync(FULL, t, kk), ll = __shfl_sync(FULL, l, kk);
                                if (tt == MAP_DEL) continue;
                                const uint8_t *row = s_e2 + tt * n2p;
#pragma unroll
                                for (int s = 0; s < W; ++s) {
                                    const int u = lane + 32 * s;
                                    const int e = (u < n2p) ? row[u] : 0;
                                    cb[s] += (e != 0);
                                    mis[s] += (e != 0) & (e != ll);
                                }
                            }
                        }
#pragma unroll
                        for (int s = 0; s < W; ++s) {
                            int cnt = 0;
#pragma unroll
                            for (int w = 0; w < W; ++w) cnt += __popc(A[s][w] & U[w]);
                            ped_s[s] = pedp + cv[s] + edd + c.eins * cnt - ee * cb[s] + c.esub * mis[s];
                        }
                    }
                    const int pedD = pedp + dDel;
                    uint8_t *crow = codes + (int64_t)p * cs;
                    int nvalid = 1; // the deletion child always exists (C5)
#pragma unroll
                    for (int s = 0; s < W; ++s) {
                        const int u = lane + 32 * s;
                        const bool sub = (u < n2) && !((U[s] >> lane) & 1u);
                        const bool del = (u == n2);
                        int code = CODE_INVALID;
                        if (sub || del) {
                            const int x = (sub ? ped_s[s] : pedD) - base + 1;
                            code = x < 0 ? 0 : (x > win ? win + 1 : x);
                            if (code >= 1 && code <= win) atomicAdd(&s_hist[code], 1);
                        }
                        if (u < cs) crow[u] = (uint8_t)code;
                        nvalid += __popc(__ballot_sync(FULL, sub));
                    }
                    if (32 * W < cs) { // n2 == 32 W: the deletion slot lies past the lane slots
                        const int u = 32 * W + lane;
                        if (u < cs) {
                            int code = CODE_INVALID;
                            if (u == n2) {
                                const int x = pedD - base + 1;
                                code = x < 0 ? 0 : (x > win ? win + 1 : x);
                                if (code >= 1 && code <= win) atomicAdd(&s_hist[code], 1);
                            }
                            crow[u] = (uint8_t)code;
                        }
                    }
                    wcount += nvalid;
                }
                if (first && lane == 0) s_wcnt[warp] = wcount;
                __syncthreads();
                if (threadIdx.x == 0) {
                    if (first) {
                        int64_t ci = 0;
                        for (int w = 0; w < NW; ++w) ci += s_wcnt[w];
                        s_ci = ci;
                        s_keepall = (ci <= K);
                    }
                    s_retry = 0;
                    if (!s_keepall) {
                        int cum = below, t = 0;
                        for (int b = 1; b <= win; ++b) {
                            if (cum + s_hist[b] >= K) { t = b; break; }
                            cum += s_hist[b];
                        }
                        if (t) { s_tcode = t; s_r = K - cum; }
                        else { s_retry = 1; s_below_add = cum - below; }
                    }
                }
                __syncthreads();
                if (!s_retry) break;
                // the K-th smallest PED lies beyond the window: slide it (all codes < base are kept)
                below += s_below_add;
                base += win;
                first = false;
                for (int k = threadIdx.x; k < 256; k += blockDim.x) s_hist[k] = 0;
                __syncthreads();
            }
            const bool keepall = s_keepall;
            const int tcode = s_tcode, rq = s_r;

            // ---------------- B: per-warp counts below / at the threshold ----------------
            {
                int lt = 0, eq = 0;
                const uint32_t *cw = reinterpret_cast<const uint32_t *>(codes + (int64_t)p0 * cs);
                const int nwords = (p1 - p0) * cs / 4;
                const uint32_t t4 = (uint32_t)tcode * 0x01010101u;
                for (int x = lane; x < nwords; x += 32) {
                    const uint32_t v = cw[x];
                    if (keepall) lt += __popc(__vcmpne4(v, 0xffffffffu)) >> 3;
                    else {
                        lt += __popc(__vcmpltu4(v, t4)) >> 3;
                        eq += __popc(__vcmpeq4(v, t4)) >> 3;
                    }
                }
                lt = __reduce_add_sync(FULL, lt);
                eq = __reduce_add_sync(FULL, eq);
                if (lane == 0) { s_wlt[warp] = lt; s_weq[warp] = eq; }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int eqpre = 0, out = 0;
                for (int w = 0; w < NW; ++w) {
                    int adm = keepall ? 0 : max(0, min(rq - eqpre, s_weq[w]));
                    s_weqpre[w] = eqpre;
                    s_wout[w] = out;
                    out += s_wlt[w] + adm;
                    eqpre += s_weq[w];
                }
                s_nnext = out;
                s_lo = 0x7fffffff;
                if (a.levels_out) {
                    a.levels_out[3 * i] = N;
                    a.levels_out[3 * i + 1] = s_ci;
                    a.levels_out[3 * i + 2] = keepall ? -1 : (int64_t)(base + tcode - 1);
                }
            }
            __syncthreads();

            // ---------------- C1: compact survivors in (parent, child) order ----------------
            {
                int eq_seen = s_weqpre[warp], out = s_wout[warp];
                const unsigned lmask = lanemask_lt();
                for (int p = p0; p < p1; ++p) {
                    const uint8_t *crow = codes + (int64_t)p * cs;
                    for (int u0 = 0; u0 < cs; u0 += 32) {
                        const int u = u0 + lane;
                        const int code = (u < cs) ? crow[u] : CODE_INVALID;
                        const bool lt = keepall ? (code != CODE_INVALID) : (code < tcode);
                        const bool eq = !keepall && (code == tcode);
                        const unsigned eqm = __ballot_sync(FULL, eq);
                        const bool keep = lt || (eq && (eq_seen + __popc(eqm & lmask)) < rq);
                        const unsigned km = __ballot_sync(FULL, keep);
                        if (keep) sel[out + __popc(km & lmask)] = ((uint32_t)p << 8) | (uint32_t)u;
                        out += __popc(km);
                        eq_seen += __popc(eqm);
                    }
                }
            }
            __syncthreads();
            const int Nn = s_nnext;

            // ---------------- C2: write the next frontier ----------------
            for (int k = threadIdx.x; k < Nn; k += blockDim.x) {
                const uint32_t v = sel[k];
                const int p = (int)(v >> 8), j = (int)(v & 255u);
                const int code = codes[(int64_t)p * cs + j];
                uint32_t Up[W];
#pragma unroll
                for (int w = 0; w < W; ++w) Up[w] = P.used[(int64_t)p * W + w];
                int ped;
                if (code >= 1 && code <= win) ped = base + code - 1;
                else
                    ped = child_ped_scalar<W, LAB>(c, P.ped[p], Up, P.map + (int64_t)p * n1s, j, n2, n2p, d,
                                                   s_pq, s_pl, vl1i, vl2, adj2, s_e2);
                Q.ped[k] = ped;
#pragma unroll
                for (int w = 0; w < W; ++w)
                    Q.used[(int64_t)k * W + w] = Up[w] | ((j < n2 && (j >> 5) == w) ? (1u << (j & 31)) : 0u);
                atomicMin(&s_lo, ped);
            }
            {
                const int wpr = (i + 4) >> 2, hw = i >> 2, sh = (i & 3) * 8;
                const int total = Nn * wpr;
                for (int x = threadIdx.x; x < total; x += blockDim.x) {
                    const int k = x / wpr, w = x - k * wpr;
                    const uint32_t v = sel[k];
                    const int p = (int)(v >> 8), j = (int)(v & 255u);
                    uint32_t word = reinterpret_cast<const uint32_t *>(P.map + (int64_t)p * n1s)[w];
                    if (w == hw) {
                        const uint32_t e = (j == n2) ? (uint32_t)MAP_DEL : (uint32_t)j;
                        word = (word & ~(0xffu << sh)) | (e << sh);
                    }
                    reinterpret_cast<uint32_t *>(Q.map + (int64_t)k * n1s)[w] = word;
                }
            }
            children += s_ci;
            parents += N;
            // B_alg(i) = N_i (4 + b d_i) + N_{i+1} (b i + 4) + N_{i+1} (b (i+1) + 4), b = 1
            algb += (int64_t)N * (4 + d) + (int64_t)Nn * (2 * i + 9);
            __syncthreads();
            N = Nn;
            lo = s_lo;
            cur ^= 1;
        }

        // ---------------- Finalize: insertion completion + argmin ----------------
        if (threadIdx.x == 0) s_best = ~0ull;
        __syncthreads();
        {
            const FrontierView<W> P = F[cur];
            for (int k = threadIdx.x; k < N; k += blockDim.x) {
                uint32_t U[W];
                int usedc = 0, e2u2 = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) { U[w] = P.used[(int64_t)k * W + w]; usedc += __popc(U[w]); }
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    uint32_t bits = U[w];
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        const int u = 32 * w + b;
#pragma unroll
                        for (int x = 0; x < W; ++x) e2u2 += __popc(__ldg(adj2 + u * W + x) & U[x]);
                    }
                }
                const int64_t total = (int64_t)P.ped[k] + (int64_t)c.vins * (n2 - usedc) +
                                      (int64_t)c.eins * (pd.m2 - e2u2 / 2);
                atomicMin(&s_best, ((unsigned long long)total << 32) | (unsigned)k);
            }
            __syncthreads();
            const unsigned long long best = s_best;
            const int kb = (int)(best & 0xffffffffull);
            const uint8_t *row = P.map + (int64_t)kb * n1s;
            for (int q = threadIdx.x; q < n1; q += blockDim.x) {
                const int t = row[q];
                a.map_out[pd.map_out + q] = (t == MAP_DEL) ? -1 : t;
            }
            if (threadIdx.x == 0) {
                const int pidx = a.order[item];
                a.cost_out[pidx] = (int64_t)(best >> 32);
                a.children_out[pidx] = children;
                a.parents_out[pidx] = parents;
                a.algbytes_out[pidx] = algb;
            }
        }
        __syncthreads();
    }
}

} // namespace fg
