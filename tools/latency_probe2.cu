// Per-step latency pieces of the Householder panel on sm_100a (clock64).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ double sink2;
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}

__global__ void probe2(long long* out, double seed) {
  __shared__ uint64_t bars[64];
  __shared__ double col[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 64) mbar_init(&bars[threadIdx.x], 1);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) col[i] = seed + i;
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  // (a) ping-pong between warp 0 and warp 1 through mbarriers: 32 hand-offs
  long long t0 = clock64();
  for (int it = 0; it < 32; ++it) {
    if (warp == (it & 1)) {
      if (it > 0) mbar_wait(&bars[it - 1], 0);
      if (lane == 0) mbar_arrive(&bars[it]);
    }
  }
  if (warp == 1) mbar_wait(&bars[31], 0);
  long long t1 = clock64();
  if (threadIdx.x == 32) out[0] = (t1 - t0) / 32;
  __syncthreads();
  // (b) reflector: rsqrt + rcp chain
  double v = seed + lane;
  t0 = clock64();
  for (int it = 0; it < 100; ++it) {
    double s2 = fma(v, v, 1.0); double rho = rsqrt(s2); double nrm = s2 * rho;
    double tau = fma(fabs(v), rho, 1.0); double sc = copysign(__drcp_rn(fabs(v) + nrm), v);
    v = tau * 0.5 + sc;
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / 100;
  // (c) full step chain on one warp (MR=6 rows per lane), 32 steps
  double x[6], pv[6];
  for (int k = 0; k < 6; ++k) x[k] = seed + k + lane;
  t0 = clock64();
  if (warp == 0) {
    for (int j = 0; j < 32; ++j) {
      const double tau = col[j], scale = col[j + 1];
#pragma unroll
      for (int k = 0; k < 6; ++k) pv[k] = (lane + 32 * k > j) ? col[(lane + 32 * k) & 255] : 0.0;
      double d = 0, sxx = 0, spp = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) { d = fma(pv[k], x[k], d); sxx = fma(x[k], x[k], sxx); spp = fma(pv[k], pv[k], spp); }
      double rj = __shfl_sync(0xffffffffu, x[0], j);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
        spp += __shfl_xor_sync(0xffffffffu, spp, o);
      }
      const double f = tau * (rj + scale * d), gs = f * scale;
#pragma unroll
      for (int k = 0; k < 6; ++k) x[k] = fma(-gs, pv[k], x[k]);
      double nrm = fma(gs * gs, spp, fma(-2.0 * gs, d, sxx));
#pragma unroll
      for (int k = 0; k < 6; ++k) col[(lane + 32 * k) & 255] = x[k] * 1e-3;
      double alpha = __shfl_sync(0xffffffffu, x[0], (j + 1) & 31);
      __syncwarp();
      if (lane == 0) {
        double s2 = fma(alpha, alpha, fabs(nrm)); double rho = rsqrt(s2); double nn = s2 * rho;
        col[j + 1] = fma(fabs(alpha), rho, 1.0) * 1e-3; col[j + 2] = copysign(__drcp_rn(fabs(alpha) + nn), alpha) * 1e-3;
      }
      __syncwarp();
    }
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / 32;
  // (d) same chain but without the reflector
  t0 = clock64();
  if (warp == 0) {
    for (int j = 0; j < 32; ++j) {
      const double tau = col[j], scale = col[j + 1];
#pragma unroll
      for (int k = 0; k < 6; ++k) pv[k] = (lane + 32 * k > j) ? col[(lane + 32 * k) & 255] : 0.0;
      double d = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) d = fma(pv[k], x[k], d);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      const double f = tau * (1.0 + scale * d), gs = f * scale;
#pragma unroll
      for (int k = 0; k < 6; ++k) x[k] = fma(-gs, pv[k], x[k]);
#pragma unroll
      for (int k = 0; k < 6; ++k) col[(lane + 32 * k) & 255] = x[k] * 1e-3;
      __syncwarp();
    }
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / 32;
  sink2 = v + x[0] + x[5];
}

int main() {
  long long* d; cudaMalloc(&d, 64 * sizeof(long long));
  probe2<<<1, 512>>>(d, 1.5);
  long long h[4]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mbar_handoff=%lld reflector_rsqrt_rcp=%lld full_step=%lld step_no_reflector=%lld (err %s)\n", h[0], h[1], h[2], h[3],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
