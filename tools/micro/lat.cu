// Dependent-latency micro-benchmark for FP64 ops / shuffles / shared loads
// with 1..16 concurrently active warps in one CTA (development tool).
#include <cstdio>
template <int OP>
__global__ void lat(double* out, long long* cyc, int iters, int active_warps) {
  __shared__ double sm[1024];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 1) % 1024;
  __syncthreads();
  if (warp >= active_warps) return;
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) a = a + c;                                   // DADD chain
      if (OP == 1) a = fma(a, b, c);                            // DFMA chain
      if (OP == 2) a += __shfl_xor_sync(0xffffffffu, a, 1);     // 64-bit shuffle + DADD
      if (OP == 3) a = sm[(int)a & 1023];                       // LDS chase
      if (OP == 4) a = __shfl_xor_sync(0xffffffffu, a, 1);      // 64-bit shuffle only
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cyc[warp] = t1 - t0;
  out[threadIdx.x] = a;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 32 * 8);
  const char* nm[5] = {"DADD", "DFMA", "SHFL64+DADD", "LDS chase", "SHFL64"};
  const int iters = 256;
  for (int op = 0; op < 5; ++op) {
    for (int w : {1, 4, 8, 16}) {
      void (*k)(double*, long long*, int, int) = op == 0 ? lat<0> : op == 1 ? lat<1> : op == 2 ? lat<2> : op == 3 ? lat<3> : lat<4>;
      k<<<1, 512>>>(o, c, iters, w);
      cudaDeviceSynchronize();
      long long h[32]; cudaMemcpy(h, c, 32 * 8, cudaMemcpyDeviceToHost);
      printf("%-12s warps %2d: %.1f cycles/op\n", nm[op], w, h[0] / (16.0 * iters));
    }
  }
  return 0;
}
