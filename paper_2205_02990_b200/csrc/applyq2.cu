// Apply the probe factorisation's Q to a tile of sample rows, then solve --
// warp-row-local tensor-core version.
//
// For box tau with Omega_tau^T = Q R (complete Householder Q from hqr.cu):
//   Y Q = Y - sum over panels of (Y V_p) T_p V_p^T   (compact WY, in panel order)
//   X   = (Y Q)(:, 0:n) R^{-T}   = Y Omega^+         (lstsq_right, linalg.py:65-90)
//   Y P = (Y Q)(:, s-r:s)                            (nullspace + product, compress.py:169-171)
// Each CTA owns 64 rows of one box; each warp owns 8 of them for the whole
// computation, so the three GEMMs per panel (Y V -> *T -> Y -= W V^T) and the
// blocked back substitution never leave the warp: intermediate W stays in
// DMMA accumulators and is re-laid out C-fragment -> A-fragment with quad
// shuffles.  V_p / T_p (and later R / Rinv blocks) stream through a
// double-buffered cp.async pipeline shared by the 8 warps.
#include "common.cuh"
#include "kernels.h"

namespace hbs {

namespace {
constexpr int kTW = 64;          // rows per CTA
constexpr int kLdT2 = 36;        // frag_ld(32)
}  // namespace

__global__ void __launch_bounds__(256) applyq2_kernel(ApplyQArgs args) {
  extern __shared__ __align__(16) double smem[];
  const int tile = blockIdx.x;
  const int64_t b = blockIdx.y;
  const int side = blockIdx.z;
  const ApplyQSide& S = args.side[side];
  const int nb = box_rows(args.geo, b);
  const int n = nb;
  const int row0 = tile * kTW;
  if (row0 >= nb) return;
  const int trows = min(kTW, nb - row0);
  const int s = args.s, r = args.r;
  const int spad = round_up(s, 8);
  const int lds = frag_ld(spad);
  double* Ys = smem;                              // kTW x lds
  double* Vst[2] = {Ys + kTW * lds, Ys + kTW * lds + kNB * lds};   // kNB x lds each
  double* Tst[2] = {Vst[1] + kNB * lds, Vst[1] + kNB * lds + kNB * kLdT2};

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rw = warp * 8;                        // my rows within the tile
  const int64_t rb = args.geo.row_begin[b];
  const double* y = S.y + S.y_c_rb * rb + S.y_c_b * b + (int64_t)row0 * S.ldy;
  const double* vt = S.vt + (size_t)b * S.vt_stride;
  const double* tglob = S.t + (size_t)b * S.t_stride;
  const double* R = S.r + (size_t)b * S.r_stride;
  const double* rinv = S.rinv + (size_t)b * S.rinv_stride;
  const int npanel = (n + kNB - 1) / kNB;
  const int nblk = npanel;

  // Y tile (zero rows >= trows, zero columns >= s)
  for (int e = threadIdx.x; e < kTW * spad; e += blockDim.x) {
    const int i = e / spad, c = e - i * spad;
    const bool ok = i < trows && c < s;
    cp_async8(&Ys[i * lds + c], ok ? y + (int64_t)i * S.ldy + c : y, ok);
  }
  // stage loader: panel p (p < npanel) or solve block (npanel + (nblk-1-blk))
  auto load_stage = [&](int stage, int buf) {
    if (stage < npanel) {
      const int j0 = stage * kNB, nbp = min(kNB, n - j0), kb = j0 & ~7;
      const int w = spad - kb;
      for (int e = threadIdx.x; e < kNB * w; e += blockDim.x) {
        const int q = e / w, c = kb + (e - q * w);
        const bool ok = q < nbp && c < s;
        cp_async8(&Vst[buf][q * lds + c], ok ? vt + (size_t)(j0 + q) * S.ldvt + c : vt, ok);
      }
      const double* tp = tglob + (size_t)stage * kNB * kNB;
      for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
        const int q = e >> 5, c = e & 31;
        cp_async8(&Tst[buf][q * kLdT2 + c], tp + e, true);
      }
    } else {
      const int blk = nblk - 1 - (stage - npanel);
      const int i0 = blk * kNB, nbi = min(kNB, n - i0), c0 = i0 + kNB;
      const int kr = n > c0 ? round_up(n - c0, 4) : 0;
      for (int e = threadIdx.x; e < kNB * kr; e += blockDim.x) {
        const int q = e / kr, c = e - q * kr;
        const bool ok = q < nbi && c0 + c < n;
        cp_async8(&Vst[buf][q * lds + c], ok ? R + (size_t)(i0 + q) * S.ldr + c0 + c : R, ok);
      }
      const double* rp = rinv + (size_t)blk * kNB * kNB;
      for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
        const int q = e >> 5, c = e & 31;
        cp_async8(&Tst[buf][q * kLdT2 + c], rp + e, true);
      }
    }
    cp_async_commit();
  };

  const int nstage = npanel + nblk;
  load_stage(0, 0);
  const double* yrow = Ys + (rw + g) * lds;
  for (int stage = 0; stage < nstage; ++stage) {
    const int buf = stage & 1;
    cp_async_wait<0>();
    __syncthreads();
    if (stage + 1 < nstage) load_stage(stage + 1, buf ^ 1);
    const double* V = Vst[buf];
    const double* T = Tst[buf];
    if (rw >= trows) continue;  // warp has no rows (still joins the barriers)
    if (stage < npanel) {
      const int j0 = stage * kNB, kb = j0 & ~7;
      // GEMM1: W = Y(:, kb:) V_p(kb:, :)   (8 x 32)
      double w[4][2] = {};
      for (int k = kb; k < spad; k += 4) {
        const double a = yrow[k + t];
#pragma unroll
        for (int f = 0; f < 4; ++f) dmma8x8x4(w[f][0], w[f][1], a, V[(8 * f + g) * lds + k + t]);
      }
      // GEMM2: W2 = W T_p
      double w2[4][2] = {};
#pragma unroll
      for (int kk = 0; kk < kNB; kk += 4) {
        const double a = cfrag_to_afrag<4>(w, kk, lane);
#pragma unroll
        for (int f = 0; f < 4; ++f) dmma8x8x4(w2[f][0], w2[f][1], a, T[(kk + t) * kLdT2 + 8 * f + g]);
      }
      double a3[kNB / 4];
#pragma unroll
      for (int kk = 0; kk < kNB; kk += 4) a3[kk / 4] = -cfrag_to_afrag<4>(w2, kk, lane);
      // GEMM3: Y(:, kb:) -= W2 V_p(kb:, :)^T
      double* yw = Ys + (rw + g) * lds;
      for (int n0 = kb; n0 < spad; n0 += 8) {
        double c0 = yw[n0 + 2 * t], c1 = yw[n0 + 2 * t + 1];
#pragma unroll
        for (int kk = 0; kk < kNB; kk += 4) dmma8x8x4(c0, c1, a3[kk / 4], V[(kk + t) * lds + n0 + g]);
        yw[n0 + 2 * t] = c0;
        yw[n0 + 2 * t + 1] = c1;
      }
      __syncwarp();
      if (stage == npanel - 1 && S.yp != nullptr) {
        // Y P = (Y Q)(:, s-r:s) for my rows (before the solve reuses Ys)
        double* yp = S.yp + (size_t)b * S.yp_stride + (size_t)(row0 + rw) * S.ldyp;
        const int myrows = min(8, trows - rw);
        for (int e = lane; e < myrows * r; e += 32) {
          const int i = e / r, c = e - i * r;
          yp[(size_t)i * S.ldyp + c] = Ys[(rw + i) * lds + s - r + c];
        }
      }
    } else {
      // blocked back substitution X R^T = Y Q1, block blk (from the last)
      const int blk = nblk - 1 - (stage - npanel);
      const int i0 = blk * kNB, c0 = i0 + kNB;
      const int kr = n > c0 ? round_up(n - c0, 4) : 0;
      double acc[4][2];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = i0 + 8 * f + 2 * t + e;
          acc[f][e] = c < n ? yrow[c] : 0.0;
        }
      for (int k = 0; k < kr; k += 4) {
        const double a = -yrow[c0 + k + t];
#pragma unroll
        for (int f = 0; f < 4; ++f) dmma8x8x4(acc[f][0], acc[f][1], a, V[(8 * f + g) * lds + k + t]);
      }
      double xb[4][2] = {};
#pragma unroll
      for (int kk = 0; kk < kNB; kk += 4) {
        const double a = cfrag_to_afrag<4>(acc, kk, lane);
#pragma unroll
        for (int f = 0; f < 4; ++f) dmma8x8x4(xb[f][0], xb[f][1], a, T[(8 * f + g) * kLdT2 + kk + t]);
      }
      __syncwarp();
      double* yw = Ys + (rw + g) * lds;
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = i0 + 8 * f + 2 * t + e;
          if (c < n) yw[c] = xb[f][e];
        }
      __syncwarp();
    }
  }
  // X rows of this warp
  if (rw < trows) {
    double* x = S.x + (size_t)b * S.x_stride + (size_t)(row0 + rw) * S.ldx;
    const int myrows = min(8, trows - rw);
    for (int e = lane; e < myrows * n; e += 32) {
      const int i = e / n, c = e - i * n;
      x[(size_t)i * S.ldx + c] = Ys[(rw + i) * lds + c];
    }
  }
}

size_t applyq2_smem_bytes(int s) {
  const int lds = frag_ld(round_up(s, 8));
  return ((size_t)kTW * lds + 2 * (size_t)kNB * lds + 2 * (size_t)kNB * kLdT2) * sizeof(double);
}

int launch_applyq2(ApplyQArgs args, int nsides, cudaStream_t stream) {
  const size_t smem = applyq2_smem_bytes(args.s);
  if (smem > kMaxSmemBytes) return kErrUnsupported;
  cudaFuncSetAttribute(applyq2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((args.n_max + kTW - 1) / kTW, (unsigned)args.geo.nbox, nsides);
  applyq2_kernel<<<grid, 256, smem, stream>>>(args);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

}  // namespace hbs
