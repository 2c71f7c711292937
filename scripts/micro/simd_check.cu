#include <cstdio>
#include <cstdint>
__global__ void k(const uint32_t* v, uint32_t t4, uint32_t* out, int n) {
  int i = threadIdx.x; if (i >= n) return;
  out[4*i+0] = __vcmpltu4(v[i], t4);
  out[4*i+1] = __vcmpeq4(v[i], t4);
  out[4*i+2] = __vcmpne4(v[i], 0xffffffffu);
  out[4*i+3] = __vsub4(v[i], t4);
}
int main() {
  uint32_t h[8] = {0x03010000u, 0xff030101u, 0x00000000u, 0x01010101u, 0x80ff0102u, 0x7f000301u, 0x02020202u, 0x0100ff03u};
  uint32_t *dv, *dout; cudaMalloc(&dv, 32); cudaMalloc(&dout, 128);
  cudaMemcpy(dv, h, 32, cudaMemcpyHostToDevice);
  k<<<1,8>>>(dv, 0x01010101u, dout, 8);
  uint32_t o[32]; cudaMemcpy(o, dout, 128, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 8; ++i) printf("v=%08x lt1=%08x eq1=%08x ne255=%08x sub=%08x\n", h[i], o[4*i], o[4*i+1], o[4*i+2], o[4*i+3]);
}
