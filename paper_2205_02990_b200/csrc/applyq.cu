// Apply the probe factorisation's Q to a tile of sample rows, then solve.
//
// For box tau with Omega_tau^T = Q R (complete Householder Q, geqrf.cu):
//   Y_tau Q = [Y Q1 | Y Q2]  (the transposed-side trailing update of the
//             partial QR of [Omega^T | Y^T]; blocked compact-WY on DMMA),
//   Y_tau Omega_tau^+ = (Y Q1) R^{-T}                 -- lstsq_right, linalg.py:65-90
//   Y_tau P           = (Y Q)(:, s-r:s)               -- nullspace + product, compress.py:169-171
// Rows of Y are independent, so each CTA owns a TW-row tile of one box.
#include "common.cuh"
#include "cta_mma.cuh"
#include "kernels.h"

namespace hbs {

template <int TW>
__global__ void __launch_bounds__(256) applyq_kernel(ApplyQArgs args) {
  extern __shared__ double smem[];
  const int tile = blockIdx.x;
  const int64_t b = blockIdx.y;
  const int side = blockIdx.z;
  const ApplyQSide& S = args.side[side];
  const int nb = box_rows(args.geo, b);
  const int n = args.n_is_rows ? nb : args.n_fixed;   // reflector count
  const int rows = nb;                                  // Y rows of this box
  const int row0 = tile * TW;
  if (row0 >= rows) return;
  const int trows = min(TW, rows - row0);
  const int s = args.s, r = args.r;
  const int spad = round_up(s, 8);
  const int lds = frag_ld(spad);
  constexpr int ldt = 36;  // frag_ld(32)
  double* Ys = smem;                    // TW x lds
  double* Vs = Ys + TW * lds;           // NB x lds  (also R rows in the solve phase)
  double* Ts = Vs + kNB * lds;          // NB x ldt
  double* Ws = Ts + kNB * ldt;          // TW x ldt
  double* W2 = Ws + TW * ldt;           // TW x ldt
  double* Ri = W2 + TW * ldt;           // NB x ldt
  double* scratch = Ri + kNB * ldt;     // 2 * TW * NB

  const int64_t rb = args.geo.row_begin[b];
  const double* y = S.y + S.y_c_rb * rb + S.y_c_b * b + (int64_t)row0 * S.ldy;
  for (int e = threadIdx.x; e < TW * spad; e += blockDim.x) {
    const int i = e / spad, c = e % spad;
    Ys[i * lds + c] = (i < trows && c < s) ? y[(int64_t)i * S.ldy + c] : 0.0;
  }

  const double* vt = S.vt + (size_t)b * S.vt_stride;
  const int npanel = (n + kNB - 1) / kNB;
  for (int p = 0; p < npanel; ++p) {
    const int j0 = p * kNB, nbp = min(kNB, n - j0);
    const int kb = j0 & ~7;
    __syncthreads();  // previous users of Vs / Ts are done
    for (int e = threadIdx.x; e < kNB * (spad - kb); e += blockDim.x) {
      const int q = e / (spad - kb), c = kb + e % (spad - kb);
      Vs[q * lds + c] = (q < nbp && c < s) ? vt[(size_t)(j0 + q) * S.ldvt + c] : 0.0;
    }
    const double* tp = S.t + (size_t)b * S.t_stride + (size_t)p * kNB * kNB;
    for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) Ts[(e / kNB) * ldt + e % kNB] = tp[e];
    __syncthreads();
    const int K = spad - kb;
    // W = Y(:, kb:) V_p(kb:, :)
    cta_mma<false>(TW, kNB, K, SView{Ys + kb, lds, 1}, SView{Vs + kb, 1, lds}, SViewW{Ws, ldt, 1}, 1.0,
                   scratch, 2);
    // W2 = W T_p
    cta_mma<false>(TW, kNB, kNB, SView{Ws, ldt, 1}, SView{Ts, ldt, 1}, SViewW{W2, ldt, 1}, 1.0, scratch, 2);
    // Y(:, kb:) -= W2 V_p(kb:, :)^T
    cta_mma<true>(TW, K, kNB, SView{W2, ldt, 1}, SView{Vs + kb, lds, 1}, SViewW{Ys + kb, lds, 1}, -1.0);
  }

  // Y P = (Y Q)(:, s-r:s)
  if (S.yp != nullptr) {
    double* yp = S.yp + (size_t)b * S.yp_stride + (size_t)row0 * S.ldyp;
    for (int e = threadIdx.x; e < trows * r; e += blockDim.x) {
      const int i = e / r, c = e % r;
      yp[(size_t)i * S.ldyp + c] = Ys[i * lds + s - r + c];
    }
  }
  __syncthreads();

  // X R^T = Y Q1, blocked back substitution over NB-column blocks (in place in Ys).
  const double* R = S.r + (size_t)b * S.r_stride;
  const int nblk = (n + kNB - 1) / kNB;
  for (int blk = nblk - 1; blk >= 0; --blk) {
    const int i0 = blk * kNB, nbi = min(kNB, n - i0);
    const int c0 = i0 + kNB;                  // first column of the already-solved part
    const int kr = n > c0 ? round_up(n - c0, 4) : 0;
    // acc = Y Q1(:, i0:i0+nbi) (masked), R rows i0.. cols c0..n, Rinv block
    for (int e = threadIdx.x; e < TW * kNB; e += blockDim.x) {
      const int i = e / kNB, c = e % kNB;
      Ws[i * ldt + c] = (c < nbi) ? Ys[i * lds + i0 + c] : 0.0;
    }
    for (int e = threadIdx.x; e < kNB * kr; e += blockDim.x) {
      const int q = e / kr, c = e % kr;
      Vs[q * lds + c] = (q < nbi && c0 + c < n) ? R[(size_t)(i0 + q) * S.ldr + c0 + c] : 0.0;
    }
    const double* ri = S.rinv + (size_t)b * S.rinv_stride + (size_t)blk * kNB * kNB;
    for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) Ri[(e / kNB) * ldt + e % kNB] = ri[e];
    __syncthreads();
    if (kr > 0) {
      // acc -= X(:, c0:n) R(i0:i0+NB, c0:n)^T
      cta_mma<true>(TW, kNB, kr, SView{Ys + c0, lds, 1}, SView{Vs, 1, lds}, SViewW{Ws, ldt, 1}, -1.0,
                    scratch, 2);
    }
    // X(:, blk) = acc Rinv^T  -> W2, then copy the valid columns back into Ys
    cta_mma<false>(TW, kNB, kNB, SView{Ws, ldt, 1}, SView{Ri, 1, ldt}, SViewW{W2, ldt, 1}, 1.0, scratch, 2);
    for (int e = threadIdx.x; e < TW * nbi; e += blockDim.x) {
      const int i = e / nbi, c = e % nbi;
      Ys[i * lds + i0 + c] = W2[i * ldt + c];
    }
    __syncthreads();
  }
  double* x = S.x + (size_t)b * S.x_stride + (size_t)row0 * S.ldx;
  for (int e = threadIdx.x; e < trows * n; e += blockDim.x) {
    const int i = e / n, c = e % n;
    x[(size_t)i * S.ldx + c] = Ys[i * lds + c];
  }
}

template <int TW>
static size_t applyq_smem(int s) {
  const int lds = frag_ld(round_up(s, 8));
  return ((size_t)TW * lds + (size_t)kNB * lds + (size_t)(kNB + 2 * TW + kNB) * 36 +
          2 * (size_t)TW * kNB) * sizeof(double);
}

template <int TW>
static int launch_applyq_tw(const ApplyQArgs& args, int nsides, cudaStream_t stream) {
  const size_t smem = applyq_smem<TW>(args.s);
  cudaFuncSetAttribute(applyq_kernel<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((args.n_max + TW - 1) / TW, (unsigned)args.geo.nbox, nsides);
  applyq_kernel<TW><<<grid, 256, smem, stream>>>(args);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

int launch_applyq(ApplyQArgs args, int nsides, cudaStream_t stream) {
  if (applyq_smem<32>(args.s) <= kMaxSmemBytes) return launch_applyq_tw<32>(args, nsides, stream);
  if (applyq_smem<16>(args.s) <= kMaxSmemBytes) return launch_applyq_tw<16>(args, nsides, stream);
  return kErrUnsupported;
}

}  // namespace hbs
