// CTA-cooperative fp64 tensor-core (DMMA m8n8k4) GEMM on shared-memory tiles.
#pragma once
#include "common.cuh"

namespace hbs {

// Strided view of an smem matrix: element (i, j) at p[i * rs + j * cs].
struct SView {
  const double* p;
  int rs, cs;
  HBS_DEV double at(int i, int j) const { return p[i * rs + j * cs]; }
};
struct SViewW {
  double* p;
  int rs, cs;
  HBS_DEV double& at(int i, int j) const { return p[i * rs + j * cs]; }
};

// C(M x N) {=, +=} sgn * A(M x K) * B(K x N), all operands in shared memory.
// M, N multiples of 8; K multiple of 4 (callers zero-pad).  Work unit = a
// 16 x 16 warp tile (2 x 2 fragments); when there are fewer units than warps
// the K range is split across warps and the partial sums are reduced through
// `scratch` (needs ksplit * M * N doubles; may be null when ksplit == 1).
// Must be called by all threads of the CTA; ends with __syncthreads().
template <bool ACCUM>
HBS_DEV void cta_mma(int M, int N, int K, SView A, SView B, SViewW C, double sgn,
                     double* scratch = nullptr, int max_split = 1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int tm = (M + 15) >> 4, tn = (N + 15) >> 4;
  const int units = tm * tn;
  int ksplit = 1;
  if (scratch != nullptr) {
    while (ksplit * 2 <= max_split && units * ksplit * 2 <= nwarps && K / (ksplit * 2) >= 8) ksplit *= 2;
  }
  const int kchunk = ((K / ksplit) + 3) & ~3;
  for (int w = warp; w < units * ksplit; w += nwarps) {
    const int unit = w % units, ks = w / units;
    const int i0 = (unit / tn) * 16, j0 = (unit % tn) * 16;
    const int kb = ks * kchunk, ke = min(K, kb + kchunk);
    const bool m1 = i0 + 8 < M, n1 = j0 + 8 < N;
    double c[2][2][2] = {};
    for (int k = kb; k < ke; k += 4) {
      double a0 = A.at(i0 + g, k + t);
      double a1 = m1 ? A.at(i0 + 8 + g, k + t) : 0.0;
      double b0 = B.at(k + t, j0 + g);
      double b1 = n1 ? B.at(k + t, j0 + 8 + g) : 0.0;
      dmma8x8x4(c[0][0][0], c[0][0][1], a0, b0);
      dmma8x8x4(c[0][1][0], c[0][1][1], a0, b1);
      dmma8x8x4(c[1][0][0], c[1][0][1], a1, b0);
      dmma8x8x4(c[1][1][0], c[1][1][1], a1, b1);
    }
#pragma unroll
    for (int fi = 0; fi < 2; ++fi)
#pragma unroll
      for (int fj = 0; fj < 2; ++fj) {
        if ((fi && !m1) || (fj && !n1)) continue;
        const int i = i0 + fi * 8 + g, j = j0 + fj * 8 + 2 * t;
        if (ksplit == 1) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double v = sgn * c[fi][fj][e];
            if (ACCUM) v += C.at(i, j + e);
            C.at(i, j + e) = v;
          }
        } else {
          double* sp = scratch + (size_t)ks * M * N;
          sp[i * N + j] = c[fi][fj][0];
          sp[i * N + j + 1] = c[fi][fj][1];
        }
      }
  }
  __syncthreads();
  if (ksplit > 1) {
    for (int e = threadIdx.x; e < M * N; e += blockDim.x) {
      double v = 0.0;
      for (int ks = 0; ks < ksplit; ++ks) v += scratch[(size_t)ks * M * N + e];
      const int i = e / N, j = e % N;
      v *= sgn;
      if (ACCUM) v += C.at(i, j);
      C.at(i, j) = v;
    }
    __syncthreads();
  }
}

}  // namespace hbs
