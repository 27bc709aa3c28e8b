// Latency microbenchmarks (clock64) for the Householder panel step primitives on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ double sink;

__global__ void probe(long long* out, double seed) {
  __shared__ double sm[1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = seed + lane;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = seed * i;
  __syncthreads();
  long long t0, t1;
  // (a) 5-stage xor-shuffle reduction of a double, 100 times dependent
  t0 = clock64();
  for (int it = 0; it < 100; ++it) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / 100;
  // (b) dfma dependent chain
  t0 = clock64();
  for (int it = 0; it < 1000; ++it) v = fma(v, 0.999, 1e-3);
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / 1000;
  // (c) sqrt + div chain
  t0 = clock64();
  for (int it = 0; it < 100; ++it) { double b = -sqrt(fma(v, v, 1.0)); v = (b - v) / b + 1.0 / (v - b); }
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / 100;
  // (d) __syncthreads with the whole CTA
  t0 = clock64();
  for (int it = 0; it < 100; ++it) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / 100;
  // (e) LDS dependent chain (pointer chasing through smem)
  int idx = lane;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7 + 1) & 1023);
  __syncthreads();
  t0 = clock64();
  for (int it = 0; it < 100; ++it) idx = (int)sm[idx];
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / 100;
  // (f) dmma dependent chain
  double c0 = 0, c1 = 0;
  t0 = clock64();
  for (int it = 0; it < 100; ++it)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(v), "d"(v));
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / 100;
  // (g) shfl idx double
  t0 = clock64();
  for (int it = 0; it < 100; ++it) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31) * 1.0000001;
  t1 = clock64();
  if (threadIdx.x == 0) out[6] = (t1 - t0) / 100;
  sink = v + c0 + c1 + idx;
}

int main() {
  long long* d; cudaMalloc(&d, 64 * sizeof(long long));
  const char* names[] = {"xor5_reduce_f64", "dfma_lat", "sqrt_2div", "syncthreads_512", "lds_lat", "dmma_lat", "shfl_idx_f64"};
  for (int threads : {32, 512}) {
    probe<<<1, threads>>>(d, 1.5);
    long long h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads=%d:", threads);
    for (int i = 0; i < 7; ++i) printf(" %s=%lld", names[i], h[i]);
    printf("\n");
  }
  return 0;
}
