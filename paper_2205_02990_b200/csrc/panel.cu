// Per-panel compact-WY factors and R diagonal-block inverses.
//
// For each (box, side, panel p) with reflectors j0 = p*NB ... j0+nbp-1:
//   T_p  : upper-triangular NB x NB with H_{j0} ... H_{j0+nbp-1} = I - V_p T_p V_p^T
//          (LAPACK dlarft, direct = 'F', storev = 'C' recurrence:
//           T(0:b, b) = -tau_b T(0:b, 0:b) (V_p(:, 0:b)^T v_b), T(b, b) = tau_b).
//          The Gram V_p^T V_p is formed on the FP64 tensor cores.
//   Rinv : inverse of R's diagonal block R(j0:j0+NB, j0:j0+NB) (one lane per column).
// These feed the tensor-core apply / triangular solve in applyq.cu.
#include "common.cuh"
#include "cta_mma.cuh"
#include "kernels.h"

namespace hbs {

__global__ void __launch_bounds__(128) panel_factors_kernel(PanelArgs args) {
  extern __shared__ double smem[];
  const int p = blockIdx.x;
  const int64_t b = blockIdx.y;
  const int side = blockIdx.z;
  const PanelSide& S = args.side[side];
  const int nb = box_rows(args.geo, b);
  const int n = args.n_is_rows ? nb : args.n_fixed;
  const int j0 = p * kNB;
  if (j0 >= n) return;
  const int nbp = min(kNB, n - j0);
  const int m = args.m;
  const int kpad = round_up(m - (j0 & ~3), 4);
  const int kb = j0 & ~3;
  const int ldv = frag_ld(kpad);
  const int ldg = kNB + 1;
  double* Vs = smem;                      // NB x ldv (columns kb .. m)
  double* G = Vs + kNB * ldv;             // NB x ldg
  double* T = G + kNB * ldg;              // NB x ldg
  double* Rs = T + kNB * ldg;             // NB x ldg

  const double* vt = S.vt + (size_t)b * S.vt_stride;
  for (int e = threadIdx.x; e < kNB * kpad; e += blockDim.x) {
    const int q = e / kpad, c = e % kpad;
    const int col = kb + c;
    Vs[q * ldv + c] = (q < nbp && col < m) ? vt[(size_t)(j0 + q) * S.ldvt + col] : 0.0;
  }
  const double* R = S.r + (size_t)b * S.r_stride;
  for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
    const int i = e / kNB, c = e % kNB;
    double v = (i == c) ? 1.0 : 0.0;
    if (i < nbp && c < nbp) v = R[(size_t)(j0 + i) * S.ldr + j0 + c];
    Rs[i * ldg + c] = v;
  }
  __syncthreads();
  // G = V_p^T V_p (NB x NB) on the tensor cores.
  cta_mma<false>(kNB, kNB, kpad, SView{Vs, ldv, 1}, SView{Vs, 1, ldv}, SViewW{G, ldg, 1}, 1.0);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* tau = S.tau + (size_t)b * S.tau_stride;
  if (warp == 0) {
    // dlarft recurrence; lane a owns row a of T.
    const int a = lane;
    for (int c = 0; c < kNB; ++c) {
      const double tc = (c < nbp) ? tau[j0 + c] : 0.0;
      double acc = 0.0;
      for (int q = a; q < c; ++q) acc = fma(T[a * ldg + q], G[q * ldg + c], acc);
      T[a * ldg + c] = (a < c) ? -tc * acc : (a == c ? tc : 0.0);
      __syncwarp();
    }
    double* tout = S.t + (size_t)b * S.t_stride + (size_t)p * kNB * kNB;
    for (int e = lane; e < kNB * kNB; e += 32) tout[e] = T[(e / kNB) * ldg + (e % kNB)];
  } else if (warp == 1) {
    // Rinv(:, c): back substitution R x = e_c, lane c.
    const int c = lane;
    double x[kNB];
#pragma unroll
    for (int i = kNB - 1; i >= 0; --i) {
      double acc = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = i + 1; k < kNB; ++k) acc = fma(-Rs[i * ldg + k], x[k], acc);
      x[i] = acc / Rs[i * ldg + i];
    }
    double* rout = S.rinv + (size_t)b * S.rinv_stride + (size_t)p * kNB * kNB;
#pragma unroll
    for (int i = 0; i < kNB; ++i) rout[i * kNB + c] = x[i];
  }
}

int launch_panel_factors(PanelArgs args, int nsides, cudaStream_t stream) {
  const int npanel = (args.n_max + kNB - 1) / kNB;
  const int kpad = round_up(args.m, 4);
  const size_t smem = ((size_t)kNB * frag_ld(kpad) + 3 * (size_t)kNB * (kNB + 1)) * sizeof(double);
  if (smem > kMaxSmemBytes) return kErrUnsupported;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(panel_factors_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(npanel, (unsigned)args.geo.nbox, nsides);
  panel_factors_kernel<<<grid, 128, smem, stream>>>(args);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

}  // namespace hbs
