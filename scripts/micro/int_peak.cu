// Integer issue-rate microbenchmark on the B200 ("__popc throughput before choosing
// the a1 formulation"; measure the integer peak used by the 'alu' roofline).
// Each thread runs 8 independent dependency chains of one instruction class; the grid fills every SM
// (148 x 8 CTAs x 256 threads).  Reports lane-operations per second per class, and for the MIX of the
// batched branch loop (per child, W = 2: 4 LOP3 AND, 4 POPC, 3 IADD3/IMAD, 2 IMNMX clamp, 1 shift).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu && ./int_peak > int_peak.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;
enum Op { LOP, IADD, IMAD, POPC, MNMX, MIX };

template <int OP>
__global__ void __launch_bounds__(256) bench(unsigned *out, int iters, unsigned seed) {
    unsigned x[CH], y = seed * 0x9E3779B9u + threadIdx.x, z = y ^ 0x5bd1e995u;
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = y + c * 0x1234567u;
    // inline PTX with volatile asm: every operation is issued as written (no folding of the chains)
#define LOP3(x, y, z) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(x) : "r"(y), "r"(z))
#define ADD3(x, y) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(y))
#define MAD(x, y, z) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z))
#define POP(x) asm volatile("popc.b32 %0, %0;" : "+r"(x))
#define MNX(x, y) asm volatile("min.u32 %0, %0, %1;" : "+r"(x) : "r"(y))
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == LOP) { LOP3(x[c], y, z); LOP3(x[c], z, y); LOP3(x[c], y, z); LOP3(x[c], z, y); }
            else if (OP == IADD) { ADD3(x[c], y); ADD3(x[c], z); ADD3(x[c], y); ADD3(x[c], z); }
            else if (OP == IMAD) { MAD(x[c], y, z); MAD(x[c], z, y); MAD(x[c], y, z); MAD(x[c], z, y); }
            else if (OP == POPC) { POP(x[c]); ADD3(x[c], y); POP(x[c]); ADD3(x[c], z); }
            else if (OP == MNMX) { MNX(x[c], y); ADD3(x[c], z); MNX(x[c], z); ADD3(x[c], y); }
            else { // MIX: one child of the W = 2 branch loop: 4 AND (lop3), 4 POPC, 3 MAD/ADD, 2 MIN/MAX, 1 ADD
                unsigned a0 = x[c], a1 = x[c], b0 = x[c], b1 = x[c];
                LOP3(a0, y, z); LOP3(a1, z, y); LOP3(b0, y, y); LOP3(b1, z, z);
                POP(a0); POP(a1); POP(b0); POP(b1);
                MAD(a0, y, a1); MAD(b0, z, b1); ADD3(a0, b0);
                MNX(a0, y); MNX(a0, z);
                ADD3(x[c], a0);
            }
        }
    }
    unsigned r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r ^= x[c];
    if (r == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int OP>
double run(int iters, double ops_per_step, int sms) {
    unsigned *out;
    cudaMalloc(&out, 148 * 8 * 256 * 16 * sizeof(unsigned));
    const int grid = sms * 8;
    bench<OP><<<grid, 256>>>(out, 16, 1u); // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        bench<OP><<<grid, 256>>>(out, iters, 7u + rep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    return (double)grid * 256 * iters * CH * ops_per_step / (best * 1e-3) / 1e9; // Gop/s
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    const int it = 4096;
    const double lop = run<LOP>(it, 4, sms), iadd = run<IADD>(it, 4, sms), imad = run<IMAD>(it, 4, sms);
    const double popc = run<POPC>(it, 4, sms), mnmx = run<MNMX>(it, 4, sms), mix = run<MIX>(it, 14, sms);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d, \"lop3_gops\": %.1f, \"iadd3_gops\": %.1f, "
           "\"imad_gops\": %.1f, \"popc_iadd_pairs_gops\": %.1f, \"min_iadd_pairs_gops\": %.1f, \"mix_gops\": %.1f, "
           "\"source\": \"scripts/micro/int_peak.cu on this GPU: lane-ops/s with 8 independent chains per thread, "
           "148x8 CTAs x 256 threads; popc/min rows count one POPC/MIN + one ADD as 2 ops; mix = one W=2 child of the batched branch loop (4 LOP3 + 4 POPC + 3 MAD/ADD + 2 MIN + 1 ADD = 14 lane-ops)\"}\n",
           p.name, sms, clk, lop, iadd, imad, popc, mnmx, mix);
    return 0;
}
