// Probe factorisation by Gram / Cholesky + Householder reconstruction, for
// boxes whose probe block has nullity exactly r (s - n == r): every box of
// the BASELINE configurations except the config-3 leaves.
//
// Reference: nullspace() takes the last r columns of the complete Householder
// Q of Omega_tau^T (linalg.py:52-62) and lstsq_right() solves Y Omega_tau^+
// through an SVD (linalg.py:65-90), both called per node from
// compress_node_bases / compute_discrepancy (compress.py:155-197).  When the
// nullity equals r, span(P) = null(Omega_tau) and Y Omega^+ are unique, so any
// orthogonal Q with Omega^T = Q [R; 0] gives the same U, V and D.  This kernel
// builds one without a column-by-column Householder chain:
//
//   G = Omega Omega^T = R^T R                  (DMMA Gram, blocked Cholesky)
//   M = Omega_1^T - S R = V1 U'                (blocked LU, S = diag(+-1) chosen
//                                               per pivot as in dlarfg: -sign)
//   V2 = Omega_2^T U'^{-1}                      (block forward substitution)
//   T_p = -U'_pp R_pp^{-1} S_p V1,pp^{-T}       (diagonal 32 x 32 blocks)
//
// so that H = I - V T V^T (V = [V1; V2], unit lower trapezoidal) is orthogonal
// with H[:, :n] = Omega^T R^{-1} S: the Householder form of the QR of
// Omega^T with R_hh = S R (Ballard et al., "Reconstructing Householder
// vectors from tall-skinny QR").  The output is exactly what the Householder
// probe kernel leaves in shared memory -- V below the diagonal, R_hh on and
// above it, the compact-WY T of every 32-column panel -- and the fused kernel
// (hqr.cu, PRE mode) applies it to the box's Y rows and solves
// X = (Y H)(:, :n) R_hh^{-T}.
//
// One CTA (12 warps) per (box, side).  Shared memory: M (n x n, col-major),
// the streamed Omega column chunks, then G / R as 16 x 16 blocks of the upper
// block triangle (XOR-swizzled: conflict-free DMMA fragments either way).
//
// Fallback: a Cholesky breakdown, min R_ii < 1e-3 max R_ii (the Gram squares
// the condition number), a non-finite value, or a box shape outside
// (n % 16 == 0, n <= 128, s - n == r, s <= 256) flags the (box, side); the
// caller runs the LAPACK-convention Householder kernel on exactly those, which
// also applies the reference's sigma screen (linalg.py:73-78).
#include "common.cuh"
#include "kernels.h"

namespace hbs {
namespace {

constexpr int kGT = 384;     // threads per CTA (12 warps: 168 registers each)
constexpr int kGN = 128;     // max rows per box
constexpr int kLdX = 132;    // M leading dimension (frag_ld(128))
constexpr int kCh = 32;      // streamed Omega column chunk
constexpr int kLdC = 36;     // chunk row stride (frag_ld(32))
constexpr int kBlk = 256;    // one 16 x 16 block
constexpr double kFallbackRatio = 1e-3;

#ifdef HBS_TRACE
__device__ long long g_gram_trace[32];
#define GR_MARK(i) do { __syncthreads(); if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_gram_trace[i] = clock64(); } while (0)
#else
#define GR_MARK(i) do { } while (0)
#endif

HBS_DEV int bsw(int i, int j) { return i * 16 + (j ^ ((i & 3) << 2)); }
HBS_DEV int bidx(int nb, int bi, int bj) { return bi * nb - bi * (bi - 1) / 2 + (bj - bi); }

// upper block triangle of an n x n matrix in 16 x 16 blocks
struct GR {
  double* p;
  int nb;
  HBS_DEV double* blk(int bi, int bj) const { return p + bidx(nb, bi, bj) * kBlk; }
  HBS_DEV double& at(int i, int j) const { return blk(i >> 4, j >> 4)[bsw(i & 15, j & 15)]; }
};

// 1/sqrt(a) and 1/a from float seeds and two Newton steps in double, with
// exact power-of-two range reduction instead of the library slow paths (whose
// subroutine calls would push the callers' register arrays to local memory).
HBS_DEV double rsqrt_g(double a) {
  double sc = 1.0;
  // (one exact power-of-two step covers 1e-60 .. 1e60 -- far beyond any
  // Gram entry that passes the screens)
  if (a > 1e30) { a *= 0x1p-100; sc = 0x1p-50; }
  if (a < 1e-30 && a > 0.0) { a *= 0x1p100; sc = 0x1p50; }
  double y = static_cast<double>(rsqrtf(static_cast<float>(a)));
  const double ha = 0.5 * a;
  y = y * fma(-ha * y, y, 1.5);
  y = y * fma(-ha * y, y, 1.5);
  return y * sc;
}
HBS_DEV double rcp_g(double a) {
  double sc = 1.0;
  if (fabs(a) > 1e30) { a *= 0x1p-100; sc = 0x1p-100; }
  if (fabs(a) < 1e-30 && a != 0.0) { a *= 0x1p100; sc = 0x1p100; }
  float yf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(static_cast<float>(a)));   // (rcp.rn has a slow-path call)
  double y = static_cast<double>(yf);
  y = fma(y, fma(-a, y, 1.0), y);
  y = fma(y, fma(-a, y, 1.0), y);
  y = fma(y, fma(-a, y, 1.0), y);
  return y * sc;
}

// Cholesky of the diagonal block Bd (upper triangle = current Schur
// complement) in place.  Column-owned: lane k (and its mirror k + 16) holds
// column k; row j of R is broadcast through `row` (16 doubles of shared
// memory).  ri[j] = 1 / R_jj.  One warp; false on breakdown.
HBS_DEV bool chol16(double* Bd, double* ri, double* row, double floor_) {
  const int lane = threadIdx.x & 31, kc = lane & 15;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = Bd[bsw(i, kc)];   // rows > kc are don't-care (masked below)
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double d = __shfl_sync(0xffffffffu, c[j], j);
    ok = ok && (d > floor_) && (d < 1e300);
    const double rs = rsqrt_g(d);
    c[j] = (kc == j) ? d * rs : (kc > j ? c[j] * rs : 0.0);
    if (lane == j) ri[j] = rs;
    row[kc] = c[j];
    __syncwarp();
    const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      if (2 * h + 1 > j) {
        const double2 v = r2[h];
        if (2 * h > j) c[2 * h] = (2 * h <= kc) ? fma(-v.x, c[j], c[2 * h]) : c[2 * h];
        c[2 * h + 1] = (2 * h + 1 <= kc) ? fma(-v.y, c[j], c[2 * h + 1]) : c[2 * h + 1];
      }
    }
    __syncwarp();
  }
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i <= kc) Bd[bsw(i, kc)] = c[i];
  }
  return __all_sync(0xffffffffu, ok);
}

// Ri = R^{-1} (upper) of a finished diagonal block; lane i < 16: row i
// (x R = e_i, right-looking over columns); ri = 1 / R_jj.
HBS_DEV void rinv16(const double* Bd, const double* ri, double* Ri) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = (k == i) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    x[k] *= ri[k];
#pragma unroll
    for (int l = k + 1; l < 16; ++l) x[l] = fma(-x[k], Bd[bsw(k, l)], x[l]);
  }
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) Ri[bsw(i, k)] = x[k];
  }
}

// LU of the 16 x 16 diagonal block of M at (ko, ko) with the Householder sign
// rule, row-owned: pivot row j first loses s_j R(ko + j, ko + j:) with s_j =
// -sign of its current diagonal (|pivot| = |a| + R_jj), then is broadcast by
// shuffles.  Unit lower L below, U' on / above the diagonal (in X);
// sg[j] = s_j.
HBS_DEV void lu16(double* X, int ko, const double* Rd, double* sg) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double c[16], rr[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    c[k] = X[(ko + i) + (ko + k) * kLdX];
    rr[k] = (k >= i) ? Rd[bsw(i, k)] : 0.0;
  }
#pragma unroll 16
  for (int j = 0; j < 16; ++j) {
    // pivot row j (lane j) loses s_j R(j, j:) (branch-free: keeps c[] in registers)
    const double sj = c[j] >= 0.0 ? -1.0 : 1.0;
    const double sm = (i == j) ? -sj : 0.0;
#pragma unroll
    for (int k = j; k < 16; ++k) c[k] = fma(sm, rr[k], c[k]);
    if (lane == j) sg[j] = sj;
    const double dinv = __shfl_sync(0xffffffffu, rcp_g(c[j]), j);
    const double l = (i > j) ? c[j] * dinv : 0.0;
    if (i > j) c[j] = l;
#pragma unroll
    for (int k = j + 1; k < 16; ++k) {
      const double uk = __shfl_sync(0xffffffffu, c[k], j);
      c[k] = fma(-l, uk, c[k]);
    }
  }
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) X[(ko + i) + (ko + k) * kLdX] = c[k];
  }
}

// Li = L^{-1} (unit lower): lane i < 16 computes column i.
HBS_DEV void linv16(const double* X, int ko, double* Li) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double z[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) z[m] = (m == i) ? 1.0 : 0.0;
#pragma unroll
  for (int m = 0; m < 16; ++m)
#pragma unroll
    for (int q = m + 1; q < 16; ++q)
      if (m >= i) z[q] = fma(-X[(ko + q) + (ko + m) * kLdX], z[m], z[q]);
  if (lane < 16) {
#pragma unroll
    for (int m = 0; m < 16; ++m) Li[bsw(m, i)] = z[m];
  }
}

// Ui = U'^{-1} (upper): lane i < 16 computes column i (back substitution).
HBS_DEV void uinv16(const double* X, int ko, double* Ui) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double z[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) z[m] = (m == i) ? 1.0 : 0.0;
#pragma unroll
  for (int m = 15; m >= 0; --m) {
    if (m <= i) {
      z[m] *= rcp_g(X[(ko + m) + (ko + m) * kLdX]);
#pragma unroll
      for (int q = 0; q < m; ++q) z[q] = fma(-X[(ko + q) + (ko + m) * kLdX], z[m], z[q]);
    }
  }
  if (lane < 16) {
#pragma unroll
    for (int m = 0; m < 16; ++m) Ui[bsw(m, i)] = z[m];
  }
}

HBS_DEV void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace

__global__ void __launch_bounds__(kGT, 1) gram_factor_kernel(GramArgs args) {
  extern __shared__ __align__(16) double smem[];
  const int side = blockIdx.y;
  const int64_t b = blockIdx.x;
  const GramSide& S = args.side[side];
  const int n = box_rows(args.geo, b);
  const int s = args.s, r = args.r;
  int32_t* myflag = args.flag + (int64_t)side * args.geo.nbox + b;
  if ((n & 15) || n > kGN || n < 16 || s - n != r || s > 8 * kCh) {
    if (threadIdx.x == 0) *myflag = 1;
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nb = n >> 4;
  double* X = smem;                                  // M (n x n, col-major, ld kLdX)
  double* Yr = X + kGN * kLdX;                       // chunk buffers | G / R blocks
  double* Uinv = Yr + 2 * kGN * kLdC;                // inverses of U' diagonal blocks (V2)
  double* Rinv = Uinv + 8 * kBlk;                    // R_oo^{-1} of the current Cholesky block
  double* Linv = Rinv + kBlk;                        // L_oo^{-1} of the current LU block
  double* sg = Linv + kBlk;                          // Householder signs s_j
  double* rinvd = sg + kGN;                          // 1 / R_jj
  int* s_ok = reinterpret_cast<int*>(rinvd + kGN);
  const GR Gm{Yr, nb};

  const double* om = S.om + S.om_c_rb * args.geo.row_begin[b];
  GR_MARK(0);

  // ---------------------------------------------------------------- G = Omega Omega^T
  // Omega streams through two 32-column chunk buffers; the columns < n also
  // land in X as M = Omega_1^T (col-major).  Warp w accumulates 16 x 16
  // units (bi <= bj) w, w + 12, w + 24 of the upper block triangle.
  const int nch = (s + kCh - 1) / kCh;
  auto load_chunk = [&](int c) {
    double* buf = Yr + (c & 1) * kGN * kLdC;
    for (int e = threadIdx.x; e < n * kCh; e += kGT) {
      const int i = e >> 5, k = e & 31, colj = c * kCh + k;
      const bool ok = colj < s;
      const double* src = om + (int64_t)i * s + (ok ? colj : 0);
      cp_async8(&buf[i * kLdC + k], src, ok);
      if (ok && colj < n) cp_async8(&X[colj + i * kLdX], src, true);
    }
    cp_async_commit();
  };
  const int nunits = nb * (nb + 1) / 2;
  int ubi[3], ubj[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int bi = 0, rem = warp + 12 * q;
    if (rem >= nunits) rem = 0;
    while (rem >= nb - bi) { rem -= nb - bi; ++bi; }
    ubi[q] = bi; ubj[q] = bi + rem;
  }
  double acc[3][2][2][2];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) { acc[q][a][c][0] = 0.0; acc[q][a][c][1] = 0.0; }
  load_chunk(0);
  if (nch > 1) load_chunk(1);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const double* buf = Yr + (c & 1) * kGN * kLdC;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (warp + 12 * q < nunits) {
        const double* ra = buf + (16 * ubi[q] + g) * kLdC + t;
        const double* rb2 = buf + (16 * ubj[q] + g) * kLdC + t;
#pragma unroll
        for (int k = 0; k < kCh; k += 4) {
          const double a0 = ra[k], a1 = ra[8 * kLdC + k];
          const double b0 = rb2[k], b1 = rb2[8 * kLdC + k];
          dmma8x8x4(acc[q][0][0][0], acc[q][0][0][1], a0, b0);
          dmma8x8x4(acc[q][0][1][0], acc[q][0][1][1], a0, b1);
          dmma8x8x4(acc[q][1][0][0], acc[q][1][0][1], a1, b0);
          dmma8x8x4(acc[q][1][1][0], acc[q][1][1][1], a1, b1);
        }
      }
    }
    __syncthreads();
    if (c + 2 < nch) load_chunk(c + 2);
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    if (warp + 12 * q < nunits) {
      double* blk = Gm.blk(ubi[q], ubj[q]);
#pragma unroll
      for (int fi = 0; fi < 2; ++fi)
#pragma unroll
        for (int fj = 0; fj < 2; ++fj)
#pragma unroll
          for (int e = 0; e < 2; ++e) blk[bsw(8 * fi + g, 8 * fj + 2 * t + e)] = acc[q][fi][fj][e];
    }
  }
  __syncthreads();
  GR_MARK(1);

  // ---------------------------------------------------------------- Cholesky and LU, pipelined
  // Iteration it: Cholesky block o_c = it of G = R^T R, and LU block
  // o_l = it - 1 of M = Omega_1^T - S R (it needs R's block row o_l, final
  // since iteration it - 1).  (A) warp 0 factors / inverts R's diagonal
  // block, warp 1 the LU diagonal block (L^{-1}, U'^{-1}); (B) block row of
  // R, U12 = L^{-1} (M12 - S R12) and L21 = M21 U'^{-1} on the tensor cores;
  // (C) both trailing updates.
  double gmax = 0.0;
  for (int j = lane; j < n; j += 32) gmax = fmax(gmax, Gm.at(j, j));
  gmax = warp_max(gmax);
  const double floor_ = 1e-24 * gmax;
  for (int it = 0; it <= nb; ++it) {
    const int oc = it, ol = it - 1, kl = 16 * ol;
    // warps 0 / 3: Cholesky, then R_oo^{-1}; warps 1 / 2 / 4: LU, then L^{-1} and U'^{-1}
    if (oc < nb && (warp == 0 || warp == 3)) {
      if (warp == 0) {
        const bool ok = chol16(Gm.blk(oc, oc), rinvd + 16 * oc, Rinv, floor_);   // (Rinv: row buffer until warp 3 fills it)
        if (lane == 0) *s_ok = ok;
      }
      named_sync(1, 64);
      if (warp == 3) rinv16(Gm.blk(oc, oc), rinvd + 16 * oc, Rinv);
    } else if (ol >= 0 && (warp == 1 || warp == 2 || warp == 4)) {
      if (warp == 1) lu16(X, kl, Gm.blk(ol, ol), sg + kl);
      named_sync(2, 96);
      if (warp == 2) linv16(X, kl, Linv);
      if (warp == 4) uinv16(X, kl, Uinv + ol * kBlk);
    }
    __syncthreads();
    if (it == 2) GR_MARK(5);
    if (!*s_ok) {
      if (threadIdx.x == 0) *myflag = 1;
      return;
    }
    // (B) units of 16 x 8 (Cholesky / U12: one block column half) or 8 x 16 (L21)
    const int nbc = oc < nb ? nb - oc - 1 : 0;     // Cholesky block columns right of oc
    const int nbl = ol >= 0 ? nb - ol - 1 : 0;     // LU blocks right of / below ol
    const int ub = 2 * nbc + 4 * nbl;
    for (int u = warp; u < ub; u += kGT / 32) {
      if (u < 2 * nbc) {                           // R(oc, cb) = R_oo^{-T} G(oc, cb)
        const int cb = oc + 1 + (u >> 1), fj = u & 1;
        double* bc = Gm.blk(oc, cb);
        double acc2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          const double bv = bc[bsw(k + t, 8 * fj + g)];
#pragma unroll
          for (int fi = 0; fi < 2; ++fi) dmma8x8x4(acc2[fi][0], acc2[fi][1], Rinv[bsw(k + t, 8 * fi + g)], bv);
        }
        __syncwarp();
#pragma unroll
        for (int fi = 0; fi < 2; ++fi)
#pragma unroll
          for (int e = 0; e < 2; ++e) bc[bsw(8 * fi + g, 8 * fj + 2 * t + e)] = acc2[fi][e];
      } else if (u < 2 * nbc + 2 * nbl) {         // U12 = L^{-1} (M12 - S R12)
        const int v = u - 2 * nbc, cb = ol + 1 + (v >> 1), fj = v & 1;
        const double* rb2 = Gm.blk(ol, cb);
        const int col = 16 * cb + 8 * fj + g;
        double acc2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          const double bv = fma(-sg[kl + k + t], rb2[bsw(k + t, 8 * fj + g)], X[(kl + k + t) + col * kLdX]);
#pragma unroll
          for (int fi = 0; fi < 2; ++fi) dmma8x8x4(acc2[fi][0], acc2[fi][1], Linv[bsw(8 * fi + g, k + t)], bv);
        }
        __syncwarp();
#pragma unroll
        for (int fi = 0; fi < 2; ++fi)
#pragma unroll
          for (int e = 0; e < 2; ++e) X[(kl + 8 * fi + g) + (16 * cb + 8 * fj + 2 * t + e) * kLdX] = acc2[fi][e];
      } else {                                     // L21 = M21 U'^{-1}
        const int v = u - 2 * nbc - 2 * nbl, rbk = ol + 1 + (v >> 1), fi = v & 1;
        const int row = 16 * rbk + 8 * fi + g;
        const double* ui = Uinv + ol * kBlk;
        double acc2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          const double av = X[row + (kl + k + t) * kLdX];
#pragma unroll
          for (int fj = 0; fj < 2; ++fj) dmma8x8x4(acc2[fj][0], acc2[fj][1], av, ui[bsw(k + t, 8 * fj + g)]);
        }
        __syncwarp();
#pragma unroll
        for (int fj = 0; fj < 2; ++fj)
#pragma unroll
          for (int e = 0; e < 2; ++e) X[row + (kl + 8 * fj + 2 * t + e) * kLdX] = acc2[fj][e];
      }
    }
    __syncthreads();
    if (it == 2) GR_MARK(6);
    // (C) trailing updates in 16 x 16 units (four independent accumulator
    // chains): Cholesky (upper block triangle) then LU (square)
    const int mb = nbc;
    const int uc = mb * (mb + 1) / 2;
    const int ut = uc + nbl * nbl;
    for (int u = warp; u < ut; u += kGT / 32) {
      if (u < uc) {
        int q = u, bi = 0;
        while (q >= mb - bi) { q -= mb - bi; ++bi; }
        const int bj = bi + q + oc + 1;
        bi += oc + 1;
        const double* ra = Gm.blk(oc, bi);
        const double* rb2 = Gm.blk(oc, bj);
        double* cb = Gm.blk(bi, bj);
        double c[2][2][2];
#pragma unroll
        for (int fi = 0; fi < 2; ++fi)
#pragma unroll
          for (int fj = 0; fj < 2; ++fj)
#pragma unroll
            for (int e = 0; e < 2; ++e) c[fi][fj][e] = cb[bsw(8 * fi + g, 8 * fj + 2 * t + e)];
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          const double a0 = -ra[bsw(k + t, g)], a1 = -ra[bsw(k + t, 8 + g)];
          const double b0 = rb2[bsw(k + t, g)], b1 = rb2[bsw(k + t, 8 + g)];
          dmma8x8x4(c[0][0][0], c[0][0][1], a0, b0);
          dmma8x8x4(c[0][1][0], c[0][1][1], a0, b1);
          dmma8x8x4(c[1][0][0], c[1][0][1], a1, b0);
          dmma8x8x4(c[1][1][0], c[1][1][1], a1, b1);
        }
#pragma unroll
        for (int fi = 0; fi < 2; ++fi)
#pragma unroll
          for (int fj = 0; fj < 2; ++fj) {
            if (bi == bj && fi > fj) continue;
#pragma unroll
            for (int e = 0; e < 2; ++e) cb[bsw(8 * fi + g, 8 * fj + 2 * t + e)] = c[fi][fj][e];
          }
      } else {
        const int v = u - uc;
        const int c0r = kl + 16 + 16 * (v / nbl), d0 = kl + 16 + 16 * (v % nbl);
        double c[2][2][2];
#pragma unroll
        for (int fi = 0; fi < 2; ++fi)
#pragma unroll
          for (int fj = 0; fj < 2; ++fj)
#pragma unroll
            for (int e = 0; e < 2; ++e) c[fi][fj][e] = X[(c0r + 8 * fi + g) + (d0 + 8 * fj + 2 * t + e) * kLdX];
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          const double a0 = -X[(c0r + g) + (kl + k + t) * kLdX], a1 = -X[(c0r + 8 + g) + (kl + k + t) * kLdX];
          const double b0 = X[(kl + k + t) + (d0 + g) * kLdX], b1 = X[(kl + k + t) + (d0 + 8 + g) * kLdX];
          dmma8x8x4(c[0][0][0], c[0][0][1], a0, b0);
          dmma8x8x4(c[0][1][0], c[0][1][1], a0, b1);
          dmma8x8x4(c[1][0][0], c[1][0][1], a1, b0);
          dmma8x8x4(c[1][1][0], c[1][1][1], a1, b1);
        }
#pragma unroll
        for (int fi = 0; fi < 2; ++fi)
#pragma unroll
          for (int fj = 0; fj < 2; ++fj)
#pragma unroll
            for (int e = 0; e < 2; ++e) X[(c0r + 8 * fi + g) + (d0 + 8 * fj + 2 * t + e) * kLdX] = c[fi][fj][e];
      }
    }
    __syncthreads();
    if (it == 2) GR_MARK(7);
    if (it == 1) GR_MARK(8);
    if (it == nb - 1) GR_MARK(2);
  }
  // screen: the Gram squares cond(Omega); route doubtful boxes to Householder
  if (warp == 0) {
    double lo = INFINITY, hi = 0.0;
    for (int j = lane; j < n; j += 32) { const double d = Gm.at(j, j); lo = fmin(lo, d); hi = fmax(hi, d); }
    lo = warp_min(lo);
    hi = warp_max(hi);
    if (lane == 0) *s_ok = (hi > 0.0) && isfinite(hi) && lo >= kFallbackRatio * hi;
  }
  __syncthreads();
  GR_MARK(3);
  if (!*s_ok) {
    if (threadIdx.x == 0) *myflag = 1;
    return;
  }

  double* fac = S.fac + (size_t)b * S.fac_stride;   // n x s, row j = column j of [R_hh + V1; V2]
  if (warp < 8) {
    // ------------------------------------------------------------ V2 = Omega_2^T U'^{-1}
    // right-looking block forward substitution, 8 rows per warp: the
    // accumulators of every column block start as Omega_2^T (loads issued up
    // front) and lose V2(:, bb) U'(bb, cc) as soon as block bb is final.
    for (int rb = warp; 8 * rb < r; rb += 8) {
      const int q = 8 * rb + g;
      const bool qok = q < r;
      double acc[8][2][2];
#pragma unroll
      for (int bb = 0; bb < 8; ++bb)
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 16 * bb + 8 * f + 2 * t + e;
            acc[bb][f][e] = (bb < nb && qok) ? __ldg(om + (int64_t)col * s + n + q) : 0.0;
          }
#pragma unroll
      for (int bb = 0; bb < 8; ++bb) {
        if (bb < nb) {
          const double* ui = Uinv + bb * kBlk;
          double v[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
          for (int kk = 0; kk < 16; kk += 4) {
            const double a = cfrag_to_afrag<2>(acc[bb], kk, lane);
#pragma unroll
            for (int f = 0; f < 2; ++f) dmma8x8x4(v[f][0], v[f][1], a, ui[bsw(kk + t, 8 * f + g)]);
          }
          if (qok) {
#pragma unroll
            for (int f = 0; f < 2; ++f)
#pragma unroll
              for (int e = 0; e < 2; ++e) fac[(size_t)(16 * bb + 8 * f + 2 * t + e) * s + n + q] = v[f][e];
          }
          double va[4];
#pragma unroll
          for (int kk = 0; kk < 16; kk += 4) va[kk / 4] = -cfrag_to_afrag<2>(v, kk, lane);
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            if (cc > bb && cc < nb) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                for (int f = 0; f < 2; ++f)
                  dmma8x8x4(acc[cc][f][0], acc[cc][f][1], va[kk], X[(16 * bb + 4 * kk + t) + (16 * cc + 8 * f + g) * kLdX]);
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ T of panel p
    // lane i: row i of Z = U'_pp R_pp^{-1} (right-looking forward substitution),
    // then (Z S) V1,pp^{-T} in place; T_p = -result.
    const int p = warp - 8, j0 = 32 * p;
    if (j0 < n) {
      const int nbp = min(32, n - j0), i = lane;
      const int bo = j0 >> 4;
      const int bo1 = min(bo + 1, nb - 1);
      const double* Raa = Gm.blk(bo, bo);
      const double* Rab = Gm.blk(bo, bo1);
      const double* Rbb = Gm.blk(bo1, bo1);
      double z[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] = (j >= i && j < nbp && i < nbp) ? X[(j0 + i) + (j0 + j) * kLdX] : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < nbp) {
          z[k] *= rinvd[j0 + k];
#pragma unroll
          for (int l = 0; l < 32; ++l)
            if (l > k && l < nbp) {
              const double* rbl = (k >> 4) ? Rbb : ((l >> 4) ? Rab : Raa);
              z[l] = fma(-z[k], rbl[bsw(k & 15, l & 15)], z[l]);
            }
        }
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) z[k] = (k < nbp) ? z[k] * sg[j0 + k] : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < nbp) {
#pragma unroll
          for (int l = 0; l < 32; ++l)
            if (l > k && l < nbp) z[l] = fma(-z[k], X[(j0 + l) + (j0 + k) * kLdX], z[l]);
        }
      }
      // the fused kernel forms T from V and tau: tau_i = T_ii into row 0 of the panel's block
      double tii = 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) tii = (j == i) ? -z[j] : tii;
      S.t[(size_t)b * S.t_stride + (size_t)p * kNB * kNB + i] = tii;
    }
  }
  GR_MARK(9);
  // ------------------------------------------------------------ R_hh and V1 rows
  // fac row j (column j of the A layout), one warp per row: R_hh above and on
  // the diagonal, V1 below
  for (int j = warp; j < n; j += kGT / 32) {
    double* fr = fac + (size_t)j * s;
    const double* xr = X + j * kLdX;
    for (int i = lane; i < n; i += 32) fr[i] = (i <= j) ? sg[i] * Gm.at(i, j) : xr[i];
  }
  if (threadIdx.x == 0) {
    *myflag = 0;
    S.status[b] = kBoxOk;
  }
  GR_MARK(4);
}

size_t gram_smem_bytes() {
  return ((size_t)kGN * kLdX + 2 * kGN * kLdC + 10 * kBlk + 2 * kGN + 8) * sizeof(double);
}

bool gram_fits(int s, int n_max, int r) { return n_max <= kGN && s <= 8 * kCh && s - n_max == r && r >= 1; }

int launch_gram(const GramArgs& args, int nsides, cudaStream_t stream) {
  const size_t smem = gram_smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gram_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((unsigned)args.geo.nbox, nsides);
  gram_factor_kernel<<<grid, kGT, smem, stream>>>(args);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

extern "C" int hbs_debug_gram_trace(long long* out) {
#ifdef HBS_TRACE
  return cudaMemcpyFromSymbol(out, g_gram_trace, sizeof(long long) * 32) == cudaSuccess ? 0 : 4;
#else
  (void)out;
  return 6;
#endif
}

}  // namespace hbs
