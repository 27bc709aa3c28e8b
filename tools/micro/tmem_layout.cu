// Probe of the tcgen05.ld/st .16x256b thread <-> (lane, column) mapping.
#include <cstdio>
#include <cstdint>
__global__ void k(int* out) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&taddr_s)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = taddr_s;
  // each warp w writes its quadrant: thread i -> lane 32*(w%4)+i, columns 0..7 value = lane*100 + col
  const uint32_t row = 32 * (warp % 4) + lane;
  uint32_t v[8];
  for (int c = 0; c < 8; ++c) v[c] = row * 100 + c;
  const uint32_t a = base + ((32u * (warp % 4)) << 16);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;\n");
  __syncthreads();
  if (warp < 4) {
    for (int h = 0; h < 2; ++h) {
      uint32_t r0, r1, r2, r3;
      const uint32_t la = base + ((32u * warp + 16u * h) << 16);
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(la));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
      int* o = out + ((warp * 2 + h) * 32 + lane) * 4;
      o[0] = r0; o[1] = r1; o[2] = r2; o[3] = r3;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(512));
}
int main() {
  int* d; cudaMalloc(&d, 8 * 32 * 4 * 4);
  k<<<1, 128>>>(d);
  int h[8 * 32 * 4];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(e));
  for (int q = 0; q < 3; ++q) {
    printf("warp %d h %d:\n", q / 2, q % 2);
    for (int t = 0; t < 32; ++t) printf(" t%02d: %5d %5d %5d %5d\n", t, h[(q * 32 + t) * 4], h[(q * 32 + t) * 4 + 1], h[(q * 32 + t) * 4 + 2], h[(q * 32 + t) * 4 + 3]);
  }
  return 0;
}
