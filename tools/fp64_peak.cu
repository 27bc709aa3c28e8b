// FP64 throughput microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64 shapes).
// Purpose: MEASURED_PEAKS.json has no FP64 entry; the roofline denominator for the
// HBS compress path (all-fp64) is measured here.  Build: see tools/Makefile.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k4_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int iters = 4096;
  for (int bpsm : {1, 2, 4}) {
    for (int threads : {256, 512}) {
      int blocks = sms * bpsm;
      float ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
      double flops = 2.0 * 8 * iters * (double)blocks * threads;
      printf(", \"dfma_b%d_t%d_tflops\": %.2f", bpsm, threads, flops / ms / 1e9);
      ms = time_it([&] { dmma_m8n8k4_kernel<<<blocks, threads>>>(out, iters / 4); });
      flops = 2.0 * 256 * 8 * (iters / 4) * (double)blocks * (threads / 32);
      printf(", \"dmma_m8n8k4_b%d_t%d_tflops\": %.2f", bpsm, threads, flops / ms / 1e9);
      ms = time_it([&] { dmma_m16n8k4_kernel<<<blocks, threads>>>(out, iters / 4); });
      flops = 2.0 * 512 * 4 * (iters / 4) * (double)blocks * (threads / 32);
      printf(", \"dmma_m16n8k4_b%d_t%d_tflops\": %.2f", bpsm, threads, flops / ms / 1e9);
      ms = time_it([&] { dmma_m16n8k16_kernel<<<blocks, threads>>>(out, iters / 16); });
      flops = 2.0 * 2048 * 4 * (iters / 16) * (double)blocks * (threads / 32);
      printf(", \"dmma_m16n8k16_b%d_t%d_tflops\": %.2f", bpsm, threads, flops / ms / 1e9);
    }
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
