// Micro-benchmark: cycles of one 192 x 32 panel factorisation (panel_factor_q)
// in isolation, one CTA of 256 threads (pure latency) -- development tool.
// Build: python gen_trace.py (writes pfq_trace.inc), then nvcc with the
// library objects of paper_2205_02990_b200/csrc/build (see git log).
#define HBS_TRACE
#ifndef PB_NBP
#define PB_NBP 32
#endif
#include "../../paper_2205_02990_b200/csrc/hqr.cu"
#include "pfq_trace.inc"
#include <cstdio>
#include <vector>
#include <random>

namespace hbs {
__global__ void __launch_bounds__(256, 1) pf_bench(const double* Ain, int m, int reps, long long* out) {
  extern __shared__ double sm[];
  const int lda = frag_ld(round_up(m, 32));
  double* s_tau = sm;
  double* s_scale = s_tau + 64;
  double* s_beta = s_scale + 64;
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_beta + 64);
  double* G = s_beta + 64 + 64;
  double* Tscr = G + kP * kLdT;
  double* A = Tscr + 384;
  if (threadIdx.x < 64) mbar_init(&bar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < lda * kP; e += blockDim.x) {
      const int i = e % lda, j = e / lda;
      A[e] = i < m ? Ain[i + j * m] : 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    panel_factor_r<6, 0>(A, lda, m, 0, PB_NBP, s_tau, s_scale, s_beta, bar, (unsigned)(r & 1), G);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot / reps;
}
__global__ void __launch_bounds__(256, 1) pf_trace(const double* Ain, int m, long long* trc) {
  extern __shared__ double sm[];
  const int lda = frag_ld(round_up(m, 32));
  double* s_tau = sm;
  double* s_scale = s_tau + 64;
  double* s_beta = s_scale + 64;
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_beta + 64);
  double* G = s_beta + 64 + 64;
  double* Tscr = G + kP * kLdT;
  double* A = Tscr + 384;
  if (threadIdx.x < 64) mbar_init(&bar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  for (int r = 0; r < 2; ++r) {
    for (int e = threadIdx.x; e < lda * kP; e += blockDim.x) {
      const int i = e % lda, j = e / lda;
      A[e] = i < m ? Ain[i + j * m] : 0.0;
    }
    __syncthreads();
    pfq_trace<24, 0>(A, lda, m, 0, kP, s_tau, s_scale, s_beta, bar, (unsigned)(r & 1), G, Tscr + 320, trc);
    __syncthreads();
  }
  if (threadIdx.x == 0) trc[399] = 7;
}
}  // namespace hbs

int main() {
  const int m = 192, reps = 20;
  std::vector<double> h(m * 32);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (auto& v : h) v = nd(rng);
  double* d; long long* o;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 148 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const int lda = hbs::frag_ld(hbs::round_up(m, 32));
  const size_t smem = (64 * 3 + 64 + 32 * 33 + 384 + (size_t)lda * 32) * 8;
  cudaFuncSetAttribute(hbs::pf_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int grid : {1, 148}) {
    hbs::pf_bench<<<grid, 256, smem>>>(d, m, reps, o);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
    printf("grid %d: %s  cycles/panel %lld  per step %.0f\n", grid, cudaGetErrorString(e), c, c / 32.0);
  }
  long long* trc; cudaMalloc(&trc, 400 * 8); cudaMemset(trc, 0, 400 * 8);
  cudaFuncSetAttribute(hbs::pf_trace, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  hbs::pf_trace<<<1, 256, smem>>>(d, m, trc);
  printf("trace: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  { long long z; cudaMemcpy(&z, trc + 399, 8, cudaMemcpyDeviceToHost); printf("marker %lld\n", z); }
  long long ht[400]; cudaMemcpy(ht, trc, 400 * 8, cudaMemcpyDeviceToHost);
  const char* nm[10] = {"wait", "pv+refl", "stau", "dots", "reduce", "update", "nrm", "need", "store", "arrive"};
  double acc[10] = {};
  for (int j = 0; j < 31; ++j) {
    printf("j=%2d start->next %6lld :", j, j < 30 ? ht[(j + 1) * 10] - ht[j * 10] : 0LL);
    for (int k = 1; k < 10; ++k) { printf(" %s %4lld", nm[k], ht[j * 10 + k] - ht[j * 10 + k - 1]); if (j > 0) acc[k] += ht[j * 10 + k] - ht[j * 10 + k - 1]; }
    if (j < 30) { printf(" | handoff %4lld", ht[(j + 1) * 10] - ht[j * 10 + 9]); acc[0] += ht[(j + 1) * 10] - ht[j * 10 + 9]; }
    printf("\n");
  }
  printf("avg:"); for (int k = 0; k < 10; ++k) printf(" %s %.0f", k ? nm[k] : "handoff", acc[k] / (k ? 30 : 29)); printf("\n");
  {
    long long pt[64];
    hbs::pf_bench<<<1, 256, smem>>>(d, m, 1, o);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(pt, hbs::g_pf_trace, sizeof(pt));
    long long t0 = pt[0];
    for (int w = 0; w < 8; ++w) t0 = pt[8 * w] < t0 ? pt[8 * w] : t0;
    for (int w = 0; w < 8; ++w) {
      printf("warp %d: loaded %6lld phase1 %6lld norm %6lld steps", w, pt[8 * w] - t0, pt[8 * w + 1] - t0, pt[8 * w + 2] - t0);
      for (int jl = 0; jl < 4; ++jl) printf(" %6lld", pt[8 * w + 3 + jl] - t0);
      printf("\n");
    }
    long long ps[64];
    cudaMemcpyFromSymbol(ps, hbs::g_pf_step, sizeof(ps));
    const char* nm[7] = {"start", "dots", "reduce", "refl", "update", "nrm", "publish"};
    for (int jl = 0; jl < 4; ++jl) {
      printf("warp 1 step %d:", jl);
      for (int i = 1; i < 7; ++i) printf(" %s %5lld", nm[i], ps[8 * jl + i] - ps[8 * jl + i - 1]);
      if (jl < 3) printf(" | next %5lld", ps[8 * (jl + 1)] - ps[8 * jl + 6]);
      printf("\n");
    }
  }
  return 0;
}
