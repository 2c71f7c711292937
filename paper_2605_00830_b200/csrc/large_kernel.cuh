// large_kernel.cuh -- one large (g1, g2) pair on the whole GPU: a persistent cooperative kernel
// runs every level of Alg. 1 with grid-wide phases and no host round trip
// ("avoiding any host-device communication").  Used for n2 > 128 or very large K
// (BASELINE configs[3]: n = 200-500, K = 1e4-1e5).
//
// Per level: the same Branch / Threshold / Count / Compact / Update steps as batch_kernel.cuh,
// with the CTA replaced by the grid:
//   A  every warp takes a contiguous range of parents; lanes take the g2 vertices u = lane + 32 s;
//      the bit-packed g2 adjacency is held transposed in shared memory (word-major: lanes read
//      consecutive banks); only the nonzero words of the parent's used mask are visited.  Rank
//      codes go to HBM (1 byte per child), per-CTA histograms are merged with one global atomic per
//      nonzero bin (the paper's local -> global ranking, made exact).
//   T  every CTA reads the 256-bin global histogram and derives the same threshold (no extra sync).
//   B  per-warp counts < t / == t; every CTA derives its warps' prefixes from the per-warp array.
//   C  survivors are compacted in (parent, child) order; the next frontier rows are written with
//      coalesced word copies; grid barriers separate the phases.
#pragma once
#include <cooperative_groups.h>

#include <cstdint>

#include "batch_kernel.cuh"

namespace fg {
namespace cg = cooperative_groups;

struct LargeArgs {
    const uint8_t *blob;
    PairDesc pd;
    Costs c;
    int32_t K, win, W, Wp; // Wp: words per transposed plane stride (n2 rounded up to 32)
    int32_t n1s;           // lambda row stride in elements (multiple of 4 bytes)
    int32_t adj_in_smem;
    int32_t *ped[2];
    uint32_t *used[2];
    void *map[2];
    uint8_t *codes; // [K * cs]
    int32_t *sel_p, *sel_j;
    int32_t *hist;          // [3][256]
    int64_t *ci;            // [n1] candidates per level
    int32_t *lo;            // [n1 + 1] min survivor PED per level (init INT_MAX)
    int32_t *wlt, *weq;     // [total warps]
    unsigned long long *best;
    int64_t *out;           // [0] cost, [1] children, [2] parents, [3] algorithmic bytes
    int32_t *map_out;       // [n1]
    int64_t *levels_out;    // NULL or [3 n1]
};

template <typename MapT>
struct MapDel { static constexpr int value = (int)(MapT)(~(MapT)0); };

template <typename MapT, bool LAB>
__device__ int large_child_scalar(const LargeArgs &a, int i, int d, const int32_t *pq, const int32_t *pl,
                                  int pedp, const uint32_t *Up, const MapT *mrow, int j,
                                  const uint32_t *adj2, const uint8_t *e2, int vl1i, const int32_t *vl2) {
    const Costs &c = a.c;
    const int n2 = a.pd.n2, W = a.W;
    if (j == n2) return pedp + c.vdel + c.edel * d;
    int cv = (vl2[j] == vl1i) ? 0 : c.vsub;
    int cnt = 0, cb = 0, mis = 0;
    for (int w = 0; w < W; ++w) cnt += __popc(adj2[(int64_t)j * W + w] & Up[w]);
    for (int k = 0; k < d; ++k) {
        int t = mrow[pq[k]];
        if (t == MapDel<MapT>::value) continue;
        if (!LAB) cb += (adj2[(int64_t)j * W + (t >> 5)] >> (t & 31)) & 1u;
        else {
            int e = e2[(int64_t)t * a.pd.n2p + j];
            cb += (e != 0);
            mis += (e != 0) & (e != pl[k]);
        }
    }
    return pedp + cv + c.edel * d + c.eins * cnt - (c.edel + c.eins) * cb + c.esub * mis;
}

template <typename MapT, bool LAB>
__global__ void __launch_bounds__(256) kbest_large_kernel(const LargeArgs a) {
    extern __shared__ __align__(16) uint8_t dsmem[];
    __shared__ int s_hist[256];
    __shared__ int s_pre[2];
    __shared__ int s_red[2][8];
    __shared__ long long s_cnt;
    cg::grid_group grid = cg::this_grid();

    constexpr int NWB = 8; // warps per block (blockDim 256)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * NWB + wib, GW = gridDim.x * NWB;
    const Costs c = a.c;
    const PairDesc pd = a.pd;
    const int n1 = pd.n1, n2 = pd.n2, W = a.W, Wp = a.Wp, K = a.K, win = a.win;
    const int cs = (n2 + 1 + 3) & ~3;
    constexpr int DELV = MapDel<MapT>::value;
    const int32_t *vl1 = reinterpret_cast<const int32_t *>(a.blob + pd.vl1);
    const int32_t *vl2 = reinterpret_cast<const int32_t *>(a.blob + pd.vl2);
    const int32_t *pptr = reinterpret_cast<const int32_t *>(a.blob + pd.pptr);
    const int32_t *pqg = reinterpret_cast<const int32_t *>(a.blob + pd.pq);
    const int32_t *plg = reinterpret_cast<const int32_t *>(a.blob + pd.pl);
    const uint32_t *adj2 = reinterpret_cast<const uint32_t *>(a.blob + pd.adj2);
    const uint8_t *e2 = LAB ? (a.blob + pd.e2lab) : nullptr;

    // shared: per-warp parent masks (U, B, nonzero word list) then the transposed adjacency
    uint32_t *sU = reinterpret_cast<uint32_t *>(dsmem) + wib * 3 * W;
    uint32_t *sB = sU + W;
    int32_t *sNZ = reinterpret_cast<int32_t *>(sB + W);
    uint32_t *adjT = reinterpret_cast<uint32_t *>(dsmem) + NWB * 3 * W;
    if (a.adj_in_smem) {
        for (int x = threadIdx.x; x < W * Wp; x += blockDim.x) {
            const int w = x / Wp, u = x - w * Wp;
            adjT[x] = (u < n2) ? adj2[(int64_t)u * W + w] : 0u;
        }
    }
    // root
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) a.ped[0][0] = 0;
        for (int w = threadIdx.x; w < W; w += blockDim.x) a.used[0][w] = 0u;
    }
    block_sync();
    __syncwarp();
        grid.sync();

    int N = 1, lo = 0, cur = 0, ps = 0;
    int64_t children = 0, parents = 0, algb = 0;
    for (int i = 0; i < n1; ++i) {
        const int32_t *Pped = a.ped[cur];
        const uint32_t *Pused = a.used[cur];
        const MapT *Pmap = reinterpret_cast<const MapT *>(a.map[cur]);
        int32_t *Qped = a.ped[cur ^ 1];
        uint32_t *Qused = a.used[cur ^ 1];
        MapT *Qmap = reinterpret_cast<MapT *>(a.map[cur ^ 1]);
        const int pbeg = pptr[i], d = pptr[i + 1] - pbeg;
        const int32_t *pq = pqg + pbeg, *pl = plg + pbeg;
        const int vl1i = vl1[i];
        const int edd = c.edel * d, ee = c.edel + c.eins, pedDel = c.vdel + edd;
        const int chunk = (N + GW - 1) / GW;
        const int p0 = min(N, gw * chunk), p1 = min(N, p0 + chunk);
        int base = lo, below = 0;
        bool first = true, keepall = false;
        int tcode = 0, rq = 0;

        for (;;) { // ---------------- A + T ----------------
            for (int k = threadIdx.x; k < 256; k += blockDim.x) s_hist[k] = 0;
            if (threadIdx.x == 0) s_cnt = 0;
            if (blockIdx.x == 0)
                for (int k = threadIdx.x; k < 256; k += blockDim.x) a.hist[((ps + 1) % 3) * 256 + k] = 0;
            block_sync();
            int wcount = 0;
            for (int p = p0; p < p1; ++p) {
                const int pedp = Pped[p];
                const MapT *mrow = Pmap + (int64_t)p * a.n1s;
                for (int w = lane; w < W; w += 32) { sU[w] = Pused[(int64_t)p * W + w]; sB[w] = 0u; }
                __syncwarp();
                // B_p: images of the earlier g1 neighbours of v_i (PAPER.md:254 VFrom/VTo, reading C8)
                if (!LAB)
                    for (int k = lane; k < d; k += 32) {
                        const int t = mrow[pq[k]];
                        if (t != DELV) atomicOr(&sB[t >> 5], 1u << (t & 31));
                    }
                __syncwarp();
                // nonzero words of U (B is a subset of U)
                int nnz = 0;
                for (int w0 = 0; w0 < W; w0 += 32) {
                    const int w = w0 + lane;
                    const bool nz = (w < W) && sU[w] != 0u;
                    const unsigned m = __ballot_sync(FULL, nz);
                    if (nz) sNZ[nnz + __popc(m & lanemask_lt())] = w;
                    nnz += __popc(m);
                }
                __syncwarp();
                uint8_t *crow = a.codes + (int64_t)p * cs;
                int nvalid = 1;
                for (int u0 = 0; u0 < cs; u0 += 32) {
                    const int u = u0 + lane;
                    const bool sub = (u < n2) && !((sU[u >> 5] >> (u & 31)) & 1u);
                    const bool del = (u == n2);
                    int code = CODE_INVALID;
                    int ped = 0;
                    if (sub) {
                        int cnt = 0, cb = 0, mis = 0;
                        for (int z = 0; z < nnz; ++z) {
                            const int w = sNZ[z];
                            const uint32_t r = a.adj_in_smem ? adjT[(int64_t)w * Wp + u] : adj2[(int64_t)u * W + w];
                            cnt += __popc(r & sU[w]);
                            if (!LAB) cb += __popc(r & sB[w]);
                        }
                        if (LAB) {
                            for (int k = 0; k < d; ++k) {
                                const int t = mrow[pq[k]];
                                if (t == DELV) continue;
                                const int e = e2[(int64_t)t * pd.n2p + u];
                                cb += (e != 0);
                                mis += (e != 0) & (e != pl[k]);
                            }
                        }
                        ped = pedp + ((vl2[u] == vl1i) ? 0 : c.vsub) + edd + c.eins * cnt - ee * cb + c.esub * mis;
                    } else if (del) {
                        ped = pedp + pedDel;
                    }
                    if (sub || del) {
                        const int x = ped - base + 1;
                        code = x < 0 ? 0 : (x > win ? win + 1 : x);
                        if (code >= 1 && code <= win) atomicAdd(&s_hist[code], 1);
                    }
                    if (u < cs) crow[u] = (uint8_t)code;
                    nvalid += __popc(__ballot_sync(FULL, sub));
                }
                wcount += nvalid;
                __syncwarp();
            }
            if (first && lane == 0) atomicAdd((unsigned long long *)&s_cnt, (unsigned long long)wcount);
            block_sync();
            int *gh = a.hist + (ps % 3) * 256;
            for (int k = threadIdx.x; k < 256; k += blockDim.x)
                if (s_hist[k]) atomicAdd(&gh[k], s_hist[k]);
            if (first && threadIdx.x == 0) atomicAdd((unsigned long long *)&a.ci[i], (unsigned long long)s_cnt);
            block_sync();
        grid.sync();
            // T: every CTA derives the same threshold
            const int64_t ci = a.ci[i];
            keepall = (ci <= K);
            bool retry = false;
            if (!keepall) {
                // warp 0 of each block scans; broadcast via smem
                if (threadIdx.x == 0) {
                    int cum = below, t = 0;
                    for (int b = 1; b <= win; ++b) {
                        const int hv = gh[b];
                        if (cum + hv >= K) { t = b; break; }
                        cum += hv;
                    }
                    s_pre[0] = t;
                    s_pre[1] = t ? (K - cum) : (cum - below);
                }
                block_sync();
                tcode = s_pre[0];
                if (tcode) rq = s_pre[1];
                else { retry = true; below += s_pre[1]; }
                block_sync();
            }
            if (first) children += ci;
            ps++;
            first = false;
            if (!retry) break;
            base += win;
        }

        // ---------------- B: per-warp counts ----------------
        {
            int lt = 0, eq = 0;
            const uint32_t *cw = reinterpret_cast<const uint32_t *>(a.codes + (int64_t)p0 * cs);
            const int64_t nwords = (int64_t)(p1 - p0) * cs / 4;
            const uint32_t t4 = (uint32_t)tcode * 0x01010101u;
            for (int64_t x = lane; x < nwords; x += 32) {
                const uint32_t v = cw[x];
                if (keepall) lt += __popc(__vcmpne4(v, 0xffffffffu)) >> 3;
                else {
                    lt += __popc(__vcmpltu4(v, t4)) >> 3;
                    eq += __popc(__vcmpeq4(v, t4)) >> 3;
                }
            }
            lt = __reduce_add_sync(FULL, lt);
            eq = __reduce_add_sync(FULL, eq);
            if (lane == 0) { a.wlt[gw] = lt; a.weq[gw] = eq; }
        }
        block_sync();
        grid.sync();

        // ---------------- prefix for this CTA's warps (computed redundantly per CTA) ----------------
        {
            int slt = 0, seq = 0;
            const int first_w = blockIdx.x * NWB;
            for (int g = threadIdx.x; g < first_w; g += blockDim.x) { slt += a.wlt[g]; seq += a.weq[g]; }
            slt = __reduce_add_sync(FULL, slt);
            seq = __reduce_add_sync(FULL, seq);
            if (lane == 0) { s_red[0][wib] = slt; s_red[1][wib] = seq; }
            block_sync();
        }
        int ltpre = 0, eqpre = 0;
        for (int w = 0; w < NWB; ++w) { ltpre += s_red[0][w]; eqpre += s_red[1][w]; }
        for (int w = blockIdx.x * NWB; w < gw; ++w) { ltpre += a.wlt[w]; eqpre += a.weq[w]; }
        const int Nn = keepall ? (int)a.ci[i] : K;

        // ---------------- C1: compact survivors ----------------
        {
            int eq_seen = eqpre, out = ltpre + (keepall ? 0 : min(rq, eqpre));
            const unsigned lmask = lanemask_lt();
            for (int p = p0; p < p1; ++p) {
                const uint8_t *crow = a.codes + (int64_t)p * cs;
                for (int u0 = 0; u0 < cs; u0 += 32) {
                    const int u = u0 + lane;
                    const int code = (u < cs) ? crow[u] : CODE_INVALID;
                    const bool lt = keepall ? (code != CODE_INVALID) : (code < tcode);
                    const bool eq = !keepall && (code == tcode);
                    const unsigned eqm = __ballot_sync(FULL, eq);
                    const bool keep = lt || (eq && (eq_seen + __popc(eqm & lmask)) < rq);
                    const unsigned km = __ballot_sync(FULL, keep);
                    if (keep) {
                        const int pos = out + __popc(km & lmask);
                        a.sel_p[pos] = p;
                        a.sel_j[pos] = u;
                    }
                    out += __popc(km);
                    eq_seen += __popc(eqm);
                }
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0 && a.levels_out) {
            a.levels_out[3 * i] = N;
            a.levels_out[3 * i + 1] = a.ci[i];
            a.levels_out[3 * i + 2] = keepall ? -1 : (int64_t)(base + tcode - 1);
        }
        block_sync();
        grid.sync();

        // ---------------- C2: next frontier ----------------
        const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
        int mylo = 0x7fffffff;
        for (int k = gtid; k < Nn; k += gthreads) {
            const int p = a.sel_p[k], j = a.sel_j[k];
            const int code = a.codes[(int64_t)p * cs + j];
            int ped;
            if (code >= 1 && code <= win) ped = base + code - 1;
            else
                ped = large_child_scalar<MapT, LAB>(a, i, d, pq, pl, Pped[p], Pused + (int64_t)p * W,
                                                    Pmap + (int64_t)p * a.n1s, j, adj2, e2, vl1i, vl2);
            Qped[k] = ped;
            mylo = min(mylo, ped);
        }
        mylo = __reduce_min_sync(FULL, mylo);
        if (lane == 0 && mylo != 0x7fffffff) atomicMin(&a.lo[i + 1], mylo);
        for (int64_t x = gtid; x < (int64_t)Nn * W; x += gthreads) {
            const int k = (int)(x / W), w = (int)(x - (int64_t)k * W);
            const int p = a.sel_p[k], j = a.sel_j[k];
            uint32_t v = Pused[(int64_t)p * W + w];
            if (j < n2 && (j >> 5) == w) v |= 1u << (j & 31);
            Qused[x] = v;
        }
        {
            constexpr int EPW = 4 / sizeof(MapT); // map entries per 32-bit word
            const int wpr = (i + EPW) / EPW, hw = i / EPW, sh = (i % EPW) * 8 * (int)sizeof(MapT);
            const int rowwords = a.n1s * (int)sizeof(MapT) / 4;
            const uint32_t emask = (sizeof(MapT) == 1) ? 0xffu : 0xffffu;
            for (int64_t x = gtid; x < (int64_t)Nn * wpr; x += gthreads) {
                const int k = (int)(x / wpr), w = (int)(x - (int64_t)k * wpr);
                const int p = a.sel_p[k], j = a.sel_j[k];
                uint32_t word = reinterpret_cast<const uint32_t *>(Pmap)[(int64_t)p * rowwords + w];
                if (w == hw) {
                    const uint32_t e = (j == n2) ? (uint32_t)DELV : (uint32_t)j;
                    word = (word & ~(emask << sh)) | (e << sh);
                }
                reinterpret_cast<uint32_t *>(Qmap)[(int64_t)k * rowwords + w] = word;
            }
        }
        parents += N;
        algb += (int64_t)N * (4 + (int)sizeof(MapT) * d) + (int64_t)Nn * ((int)sizeof(MapT) * (2 * i + 1) + 8);
        block_sync();
        grid.sync();
        N = Nn;
        lo = a.lo[i + 1];
        cur ^= 1;
    }

    // ---------------- finalize: completion + argmin ----------------
    {
        const int32_t *Pped = a.ped[cur];
        const uint32_t *Pused = a.used[cur];
        for (int k = gw; k < N; k += GW) { // warp per survivor
            int usedc = 0, e2u2 = 0;
            for (int w = lane; w < W; w += 32) usedc += __popc(Pused[(int64_t)k * W + w]);
            for (int u = lane; u < n2; u += 32) {
                if (!((Pused[(int64_t)k * W + (u >> 5)] >> (u & 31)) & 1u)) continue;
                for (int w = 0; w < W; ++w) e2u2 += __popc(adj2[(int64_t)u * W + w] & Pused[(int64_t)k * W + w]);
            }
            usedc = __reduce_add_sync(FULL, usedc);
            e2u2 = __reduce_add_sync(FULL, e2u2);
            if (lane == 0) {
                const int64_t total = (int64_t)Pped[k] + (int64_t)c.vins * (n2 - usedc) +
                                      (int64_t)c.eins * (pd.m2 - e2u2 / 2);
                atomicMin(a.best, ((unsigned long long)total << 32) | (unsigned)k);
            }
        }
        block_sync();
        grid.sync();
        if (blockIdx.x == 0) {
            const unsigned long long best = *a.best;
            const int kb = (int)(best & 0xffffffffull);
            const MapT *row = reinterpret_cast<const MapT *>(a.map[cur]) + (int64_t)kb * a.n1s;
            for (int q = threadIdx.x; q < n1; q += blockDim.x) {
                const int t = row[q];
                a.map_out[q] = (t == DELV) ? -1 : t;
            }
            if (threadIdx.x == 0) {
                a.out[0] = (int64_t)(best >> 32);
                a.out[1] = children;
                a.out[2] = parents;
                a.out[3] = algb;
            }
        }
    }
}

} // namespace fg
