// shard_kernels.cuh -- one large (g1, g2) pair with its frontier sharded by parent over G ranks
// (§8(a) row a6).  The global frontier of level i is the concatenation, in rank
// order, of the ranks' local slices; every rank runs the same Branch / Rank / Update steps as the
// single-GPU kernels on its own parents, and the ranks exchange only what the exact selection
// needs (host-enqueued collectives between the phase kernels):
//   after Branch : all-reduce (sum) of the 256-bin rank-code histogram and of the candidate count
//   threshold    : computed identically on every rank from the reduced histogram (sh_thresh)
//   after Count  : all-gather of each rank's (codes < t, codes == t) totals -> the rank's global
//                  offset and its quota of ties at t (ties are admitted in global (parent, child)
//                  order = rank order, then local order, reading C12)
//   update       : survivors of a rank are children of its own parents, so they form a contiguous
//                  slice of the next global order (no state moves); optional contiguous rebalance
//   finalize     : all-reduce (min) of (total << 32 | global position), then the owner broadcasts
//                  the mapping.
// Frontier rows here are row-major (ped[K], used[K][W], lambda[K][n1s]) so a rebalance moves
// contiguous row ranges.
#pragma once
#include <cstdint>

#include "large_kernel.cuh"

namespace fg {

struct ShardArgs {
    const uint8_t *blob;
    PairDesc pd;
    Costs c;
    int32_t W, Wp, n1s, cs, win, adj_in_smem, K;
    const int32_t *ped;   // parents (local slice)
    const uint32_t *used;
    const void *map;
    int32_t *qped;        // children (next local slice)
    uint32_t *qused;
    void *qmap;
    uint8_t *codes;       // [Kloc][cs]
    int32_t *hist;        // [256] local histogram of the pass
    long long *ci;        // local candidate count
    int32_t *wlt, *weq;   // per-warp counts [grid * 8]
    int32_t *sel_p, *sel_j;
    int32_t *lomin;       // local min PED of the survivors
    unsigned long long *best;
};

// Status computed on the device from the reduced histogram (read by the host for control flow).
struct ShardStatus {
    int32_t keepall, tcode, r, retry, below_add, lo; // lo: the level's base PED (the previous level's minimum)
    long long ci;
};

template <typename MapT, bool LAB>
// base = *lo_dev (the previous level's survivor minimum, left on the device by the min all-reduce: the host
// does not wait for it) + base_off (the window slides of this level).
__global__ void __launch_bounds__(256) sh_branch(const ShardArgs a, int i, int N, const int32_t *lo_dev, int base_off, int first) {
    extern __shared__ __align__(16) uint8_t dsm[];
    const int base = *lo_dev + base_off;
    __shared__ int s_hist[256];
    __shared__ long long s_cnt;
    constexpr int NWB = 8;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * NWB + wib, GW = gridDim.x * NWB;
    const PairDesc pd = a.pd;
    const Costs c = a.c;
    const int n2 = pd.n2, W = a.W, Wp = a.Wp, cs = a.cs, win = a.win;
    constexpr int DELV = MapDel<MapT>::value;
    const int32_t *vl1 = reinterpret_cast<const int32_t *>(a.blob + pd.vl1);
    const int32_t *vl2 = reinterpret_cast<const int32_t *>(a.blob + pd.vl2);
    const int32_t *pptr = reinterpret_cast<const int32_t *>(a.blob + pd.pptr);
    const int32_t *pq = reinterpret_cast<const int32_t *>(a.blob + pd.pq) + pptr[i];
    const int32_t *pl = reinterpret_cast<const int32_t *>(a.blob + pd.pl) + pptr[i];
    const uint32_t *adj2 = reinterpret_cast<const uint32_t *>(a.blob + pd.adj2);
    const uint8_t *e2 = LAB ? (a.blob + pd.e2lab) : nullptr;
    const int d = pptr[i + 1] - pptr[i];
    const int vl1i = vl1[i];
    const int edd = c.edel * d, ee = c.edel + c.eins;
    uint32_t *sU = reinterpret_cast<uint32_t *>(dsm) + wib * 3 * W;
    uint32_t *sB = sU + W;
    int32_t *sNZ = reinterpret_cast<int32_t *>(sB + W);
    uint32_t *adjT = reinterpret_cast<uint32_t *>(dsm) + NWB * 3 * W;
    if (a.adj_in_smem)
        for (int x = threadIdx.x; x < W * Wp; x += blockDim.x) {
            const int w = x / Wp, u = x - w * Wp;
            adjT[x] = (u < n2) ? adj2[(int64_t)u * W + w] : 0u;
        }
    for (int k = threadIdx.x; k < 256; k += blockDim.x) s_hist[k] = 0;
    if (threadIdx.x == 0) s_cnt = 0;
    block_sync();
    const MapT *P = reinterpret_cast<const MapT *>(a.map);
    int wcount = 0;
    for (int p = gw; p < N; p += GW) { // warp per parent
        const int pedp = a.ped[p];
        const MapT *mrow = P + (int64_t)p * a.n1s;
        for (int w = lane; w < W; w += 32) { sU[w] = a.used[(int64_t)p * W + w]; sB[w] = 0u; }
        __syncwarp();
        if (!LAB)
            for (int k = lane; k < d; k += 32) {
                const int t = mrow[pq[k]];
                if (t != DELV) atomicOr(&sB[t >> 5], 1u << (t & 31));
            }
        __syncwarp();
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
            if (sub || del) {
                int ped;
                if (sub) {
                    int cnt = 0, cb = 0, mis = 0;
                    for (int z = 0; z < nnz; ++z) {
                        const int w = sNZ[z];
                        const uint32_t r = a.adj_in_smem ? adjT[(int64_t)w * Wp + u] : adj2[(int64_t)u * W + w];
                        cnt += __popc(r & sU[w]);
                        if (!LAB) cb += __popc(r & sB[w]);
                    }
                    if (LAB)
                        for (int k = 0; k < d; ++k) {
                            const int t = mrow[pq[k]];
                            if (t == DELV) continue;
                            const int e = e2[(int64_t)t * pd.n2p + u];
                            cb += (e != 0);
                            mis += (e != 0) & (e != pl[k]);
                        }
                    ped = pedp + ((vl2[u] == vl1i) ? 0 : c.vsub) + edd + c.eins * cnt - ee * cb + c.esub * mis;
                } else {
                    ped = pedp + c.vdel + edd;
                }
                code = rank_code(ped, base, win);
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
    for (int k = threadIdx.x; k < 256; k += blockDim.x)
        if (s_hist[k]) atomicAdd(&a.hist[k], s_hist[k]);
    if (first && threadIdx.x == 0 && s_cnt) atomicAdd((unsigned long long *)a.ci, (unsigned long long)s_cnt);
}

// Threshold from the globally reduced histogram (1 thread; identical on every rank).
__global__ void sh_thresh(const int32_t *hist, const long long *ci, int K, int win, int below, const int32_t *lo_dev,
                          ShardStatus *st) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    ShardStatus s{};
    s.ci = *ci;
    s.lo = *lo_dev;
    s.keepall = s.ci <= K;
    if (!s.keepall) {
        int cum = below, t = 0;
        for (int b = 1; b <= win; ++b) {
            if (cum + hist[b] >= K) { t = b; break; }
            cum += hist[b];
        }
        if (t) { s.tcode = t; s.r = K - cum; }
        else { s.retry = 1; s.below_add = cum - below; }
    }
    *st = s;
}

// Per-warp counts of codes < t / == t over contiguous parent chunks (warp w: parents [w*ch, (w+1)*ch)).
__global__ void __launch_bounds__(256) sh_count(const ShardArgs a, int N, int tcode, int keepall) {
    const int lane = threadIdx.x & 31, gw = blockIdx.x * 8 + (threadIdx.x >> 5), GW = gridDim.x * 8;
    const int ch = (N + GW - 1) / GW, p0 = min(N, gw * ch), p1 = min(N, p0 + ch);
    const uint32_t *cw = reinterpret_cast<const uint32_t *>(a.codes + (int64_t)p0 * a.cs);
    const int64_t nwords = (int64_t)(p1 - p0) * a.cs / 4;
    const uint32_t t4 = (uint32_t)tcode * 0x01010101u;
    int lt = 0, eq = 0;
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

// Local survivors in (parent, child) order.  rq_shard: ties at t this rank admits (global quota
// minus the ties of lower ranks, clamped); the rank's ties are admitted in local order.
__global__ void __launch_bounds__(256) sh_select(const ShardArgs a, int N, int tcode, int keepall, int rq_shard) {
    __shared__ int s_red[2][8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * 8 + wib, GW = gridDim.x * 8;
    const int ch = (N + GW - 1) / GW, p0 = min(N, gw * ch), p1 = min(N, p0 + ch);
    int slt = 0, seq = 0;
    for (int g = threadIdx.x; g < blockIdx.x * 8; g += blockDim.x) { slt += a.wlt[g]; seq += a.weq[g]; }
    slt = __reduce_add_sync(FULL, slt);
    seq = __reduce_add_sync(FULL, seq);
    if (lane == 0) { s_red[0][wib] = slt; s_red[1][wib] = seq; }
    block_sync();
    int ltpre = 0, eqpre = 0;
    for (int w = 0; w < 8; ++w) { ltpre += s_red[0][w]; eqpre += s_red[1][w]; }
    for (int w = blockIdx.x * 8; w < gw; ++w) { ltpre += a.wlt[w]; eqpre += a.weq[w]; }
    int eq_seen = eqpre, out = ltpre + (keepall ? 0 : min(rq_shard, eqpre));
    const unsigned lmask = lanemask_lt();
    for (int p = p0; p < p1; ++p) {
        const uint8_t *crow = a.codes + (int64_t)p * a.cs;
        for (int u0 = 0; u0 < a.cs; u0 += 32) {
            const int u = u0 + lane;
            const int code = (u < a.cs) ? crow[u] : CODE_INVALID;
            const bool lt = keepall ? (code != CODE_INVALID) : (code < tcode);
            const bool eq = !keepall && (code == tcode);
            const unsigned eqm = __ballot_sync(FULL, eq);
            const bool keep = lt || (eq && (eq_seen + __popc(eqm & lmask)) < rq_shard);
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

template <typename MapT, bool LAB>
__global__ void __launch_bounds__(256) sh_update(const ShardArgs a, int i, int Nn, int base) {
    const PairDesc pd = a.pd;
    const Costs c = a.c;
    const int n2 = pd.n2, W = a.W, win = a.win;
    constexpr int DELV = MapDel<MapT>::value;
    const int32_t *vl1 = reinterpret_cast<const int32_t *>(a.blob + pd.vl1);
    const int32_t *vl2 = reinterpret_cast<const int32_t *>(a.blob + pd.vl2);
    const int32_t *pptr = reinterpret_cast<const int32_t *>(a.blob + pd.pptr);
    const int32_t *pq = reinterpret_cast<const int32_t *>(a.blob + pd.pq) + pptr[i];
    const int32_t *pl = reinterpret_cast<const int32_t *>(a.blob + pd.pl) + pptr[i];
    const uint32_t *adj2 = reinterpret_cast<const uint32_t *>(a.blob + pd.adj2);
    const uint8_t *e2 = LAB ? (a.blob + pd.e2lab) : nullptr;
    const int d = pptr[i + 1] - pptr[i], vl1i = vl1[i];
    const MapT *P = reinterpret_cast<const MapT *>(a.map);
    MapT *Q = reinterpret_cast<MapT *>(a.qmap);
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
    int mylo = 0x7fffffff;
    for (int k = gtid; k < Nn; k += gthreads) {
        const int p = a.sel_p[k], j = a.sel_j[k];
        const int code = a.codes[(int64_t)p * a.cs + j];
        int ped;
        if (code >= 1 && code <= win) ped = base + code - 1;
        else {
            const int pedp = a.ped[p];
            if (j == n2) ped = pedp + c.vdel + c.edel * d;
            else {
                int cnt = 0, cb = 0, mis = 0;
                for (int w = 0; w < W; ++w) cnt += __popc(adj2[(int64_t)j * W + w] & a.used[(int64_t)p * W + w]);
                const MapT *mrow = P + (int64_t)p * a.n1s;
                for (int q = 0; q < d; ++q) {
                    const int t = mrow[pq[q]];
                    if (t == DELV) continue;
                    if (!LAB) cb += (adj2[(int64_t)j * W + (t >> 5)] >> (t & 31)) & 1u;
                    else {
                        const int e = e2[(int64_t)t * pd.n2p + j];
                        cb += (e != 0);
                        mis += (e != 0) & (e != pl[q]);
                    }
                }
                ped = pedp + ((vl2[j] == vl1i) ? 0 : c.vsub) + c.edel * d + c.eins * cnt - (c.edel + c.eins) * cb + c.esub * mis;
            }
        }
        a.qped[k] = ped;
        mylo = min(mylo, ped);
    }
    mylo = __reduce_min_sync(FULL, mylo);
    if ((threadIdx.x & 31) == 0 && mylo != 0x7fffffff) atomicMin(a.lomin, mylo);
    for (int64_t x = gtid; x < (int64_t)Nn * W; x += gthreads) {
        const int k = (int)(x / W), w = (int)(x - (int64_t)k * W);
        const int p = a.sel_p[k], j = a.sel_j[k];
        uint32_t v = a.used[(int64_t)p * W + w];
        if (j < n2 && (j >> 5) == w) v |= 1u << (j & 31);
        a.qused[x] = v;
    }
    constexpr int EPW = 4 / sizeof(MapT);
    const int rowwords = a.n1s * (int)sizeof(MapT) / 4;
    const int wpr = (i + EPW) / EPW, hw = i / EPW, sh = (i % EPW) * 8 * (int)sizeof(MapT);
    const uint32_t emask = (sizeof(MapT) == 1) ? 0xffu : 0xffffu;
    for (int64_t x = gtid; x < (int64_t)Nn * wpr; x += gthreads) {
        const int k = (int)(x / wpr), w = (int)(x - (int64_t)k * wpr);
        const int p = a.sel_p[k], j = a.sel_j[k];
        uint32_t word = reinterpret_cast<const uint32_t *>(P)[(int64_t)p * rowwords + w];
        if (w == hw) {
            const uint32_t e = (j == n2) ? (uint32_t)DELV : (uint32_t)j;
            word = (word & ~(emask << sh)) | (e << sh);
        }
        reinterpret_cast<uint32_t *>(Q)[(int64_t)k * rowwords + w] = word;
    }
}

// Completion + argmin over the local survivors; key = total << 32 | global position.
__global__ void __launch_bounds__(256) sh_final(const ShardArgs a, int N, int goff) {
    const PairDesc pd = a.pd;
    const int lane = threadIdx.x & 31, gw = blockIdx.x * 8 + (threadIdx.x >> 5), GW = gridDim.x * 8;
    const int n2 = pd.n2, W = a.W;
    const uint32_t *adj2 = reinterpret_cast<const uint32_t *>(a.blob + pd.adj2);
    for (int k = gw; k < N; k += GW) {
        int usedc = 0, e2u2 = 0;
        const uint32_t *U = a.used + (int64_t)k * W;
        for (int w = lane; w < W; w += 32) usedc += __popc(U[w]);
        for (int u = lane; u < n2; u += 32) {
            if (!((U[u >> 5] >> (u & 31)) & 1u)) continue;
            for (int w = 0; w < W; ++w) e2u2 += __popc(adj2[(int64_t)u * W + w] & U[w]);
        }
        usedc = __reduce_add_sync(FULL, usedc);
        e2u2 = __reduce_add_sync(FULL, e2u2);
        if (lane == 0) {
            const int64_t total = (int64_t)a.ped[k] + (int64_t)a.c.vins * (n2 - usedc) + (int64_t)a.c.eins * (pd.m2 - e2u2 / 2);
            atomicMin(a.best, ((unsigned long long)total << 32) | (unsigned)(goff + k));
        }
    }
}

template <typename MapT>
__global__ void sh_mapping(const void *map, int n1s, int k, int n1, int32_t *out) {
    constexpr int DELV = MapDel<MapT>::value;
    const MapT *row = reinterpret_cast<const MapT *>(map) + (int64_t)k * n1s;
    for (int q = threadIdx.x; q < n1; q += blockDim.x) out[q] = (row[q] == DELV) ? -1 : (int)row[q];
}

// tot[0] = sum of wlt[0..n), tot[1] = sum of weq[0..n)  (one block)
__global__ void reduce_totals(const int32_t *wlt, const int32_t *weq, int n, int64_t *tot) {
    __shared__ long long s[2][8];
    long long a = 0, b = 0;
    for (int x = threadIdx.x; x < n; x += blockDim.x) { a += wlt[x]; b += weq[x]; }
    for (int o = 16; o; o >>= 1) { a += __shfl_down_sync(FULL, a, o); b += __shfl_down_sync(FULL, b, o); }
    if ((threadIdx.x & 31) == 0) { s[0][threadIdx.x >> 5] = a; s[1][threadIdx.x >> 5] = b; }
    block_sync();
    if (threadIdx.x == 0) {
        long long ta = 0, tb = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { ta += s[0][w]; tb += s[1][w]; }
        tot[0] = ta;
        tot[1] = tb;
    }
}

// Loopback "collective" of the virtual-shard transport: element-wise sum or min over the G shards' buffers
// (all on this device), written back to every shard, with no host round trip.
template <typename T>
struct ShardPtrs {
    T *p[16];
};
template <typename T, int OP> // OP 0 = sum, 1 = min
__global__ void sh_combine(ShardPtrs<T> ps, int G, int n) {
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        T acc = ps.p[0][x];
        for (int g = 1; g < G; ++g) acc = OP == 0 ? acc + ps.p[g][x] : (ps.p[g][x] < acc ? ps.p[g][x] : acc);
        for (int g = 0; g < G; ++g) ps.p[g][x] = acc;
    }
}

} // namespace fg
