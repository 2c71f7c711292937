// Checks the large kernel's SWAR rank-code evaluation (two biased 16-bit lanes, packed min/max) against the
// plain per-slot formula on random inputs.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 swar_clamp.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__global__ void k(const uint32_t *in, int n, unsigned long long *bad, uint32_t *first) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t *r = in + 8 * t;
        const int pb = (int)r[0], vsub = r[1] & 7, eins = (r[1] >> 3) & 7, ee = (r[1] >> 6) & 15, win = (r[1] >> 10) & 1 ? 253 : 2;
        const uint32_t cvw = r[2], mnib = r[3] & 15;
        const int cb[4] = {(int)(r[4] & 31), (int)((r[4] >> 5) & 31), (int)((r[4] >> 10) & 31), (int)((r[4] >> 15) & 31)};
        const int d = 31;
        const int pbl = vsub + 255 * eins + 1, pbh = win + 2 + ee * d;
        uint32_t g = 0;
        for (int b = 0; b < 4; ++b) {
            const int x = pb + (int)((mnib >> b) & 1u) * vsub + eins * (int)((cvw >> (8 * b)) & 255u) - ee * cb[b];
            g |= (uint32_t)min(max(x, 0), win + 1) << (8 * b);
        }
        const uint32_t pbb = (uint32_t)(min(max(pb, -pbl), pbh) + 0x8000) * 0x00010001u;
        const uint32_t hiclamp = (uint32_t)(0x8000 + win + 1) * 0x00010001u;
        const uint32_t cnA = cvw & 0x00ff00ffu, cnB = (cvw >> 8) & 0x00ff00ffu;
        const uint32_t cbA = (uint32_t)cb[0] | ((uint32_t)cb[2] << 16), cbB = (uint32_t)cb[1] | ((uint32_t)cb[3] << 16);
        const uint32_t mA = (mnib & 1u) | ((mnib & 4u) << 14), mB = ((mnib >> 1) & 1u) | ((mnib & 8u) << 13);
        uint32_t XA = pbb + (uint32_t)vsub * mA + (uint32_t)eins * cnA - (uint32_t)ee * cbA;
        uint32_t XB = pbb + (uint32_t)vsub * mB + (uint32_t)eins * cnB - (uint32_t)ee * cbB;
        XA = __vminu2(__vmaxu2(XA, 0x80008000u), hiclamp) - 0x80008000u;
        XB = __vminu2(__vmaxu2(XB, 0x80008000u), hiclamp) - 0x80008000u;
        const uint32_t w = XA | (XB << 8);
        if (w != g && atomicAdd(bad, 1ull) == 0) {
            first[0] = t; first[1] = w; first[2] = g;
        }
    }
}
int main() {
    const int n = 1 << 22;
    uint32_t *h = (uint32_t *)malloc(32ull * n), *d;
    srand(1);
    for (int t = 0; t < n; ++t) {
        h[8 * t] = (uint32_t)(rand() % 1600 - 800);
        for (int j = 1; j < 8; ++j) h[8 * t + j] = ((uint32_t)rand() << 16) ^ (uint32_t)rand();
    }
    unsigned long long *bad; uint32_t *first;
    cudaMalloc(&d, 32ull * n); cudaMalloc(&bad, 8); cudaMalloc(&first, 12);
    cudaMemcpy(d, h, 32ull * n, cudaMemcpyHostToDevice); cudaMemset(bad, 0, 8);
    k<<<592, 256>>>(d, n, bad, first);
    unsigned long long nb; uint32_t f[3];
    cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost); cudaMemcpy(f, first, 12, cudaMemcpyDeviceToHost);
    printf("{\"cases\": %d, \"mismatches\": %llu", n, nb);
    if (nb) printf(", \"first\": {\"t\": %u, \"swar\": \"%08x\", \"plain\": \"%08x\", \"in\": [%d, %u, %08x, %u, %u]}", f[0], f[1], f[2], (int)h[8 * f[0]], h[8 * f[0] + 1], h[8 * f[0] + 2], h[8 * f[0] + 3], h[8 * f[0] + 4]);
    printf("}\n");
    return 0;
}
