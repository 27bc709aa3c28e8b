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

HBS_DEV double rsqrt_g(double a) {
  if (!(a > 1e-30 && a < 1e30)) return rsqrt(a);
  double y = static_cast<double>(rsqrtf(static_cast<float>(a)));
  const double ha = 0.5 * a;
  y = y * fma(-ha * y, y, 1.5);
  y = y * fma(-ha * y, y, 1.5);
  return y;
}
HBS_DEV double rcp_g(double a) {
  const double m = fabs(a);
  if (!(m > 1e-30 && m < 1e30)) return 1.0 / a;
  double y = static_cast<double>(__frcp_rn(static_cast<float>(a)));
  y = fma(y, fma(-a, y, 1.0), y);
  y = fma(y, fma(-a, y, 1.0), y);
  return y;
}

// Cholesky of the diagonal block Bd (upper triangle = current Schur
// complement) in place; rd[j] = R_jj, ri[j] = 1 / R_jj.  One warp; lane k
// (and its mirror k + 16) owns column k.  Returns false on breakdown.
HBS_DEV bool chol16(double* Bd, double* rd, double* ri, double* row, double floor_) {
  const int lane = threadIdx.x & 31, kc = lane & 15;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = Bd[bsw(i, kc)];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double d = __shfl_sync(0xffffffffu, c[j], j);
    ok = ok && (d > floor_) && (d < 1e300);
    const double rs = rsqrt_g(d);
    c[j] = (kc == j) ? d * rs : (kc > j ? c[j] * rs : 0.0);
    if (lane == j) { rd[j] = d * rs; ri[j] = rs; }
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

// LU of the 16 x 16 diagonal block of M at (ko, ko) with the Householder sign
// rule: pivot row j first loses s_j R(ko + j, ko + j:) with s_j = -sign of its
// current diagonal, so |pivot| = |a| + R_jj.  Unit lower L below, U' on and
// above the diagonal; sg[j] = s_j, pinv[j] = 1 / U'_jj.  One warp.
HBS_DEV void lu16(double* X, int ko, const double* Rd, double* sg, double* pinv, double* row) {
  const int lane = threadIdx.x & 31, kc = lane & 15;
  double c[16];
  double* col = X + ko + (ko + kc) * kLdX;
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = col[i];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double a = __shfl_sync(0xffffffffu, c[j], j);
    const double sj = a >= 0.0 ? -1.0 : 1.0;
    if (kc >= j) c[j] = fma(-sj, Rd[bsw(j, kc)], c[j]);
    const double d = __shfl_sync(0xffffffffu, c[j], j);
    const double dinv = rcp_g(d);
    if (lane == j) { sg[j] = sj; pinv[j] = dinv; }
    if (kc == j) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i > j) c[i] *= dinv;
    }
    if (lane == j) {
#pragma unroll
      for (int i = 0; i < 16; ++i) row[i] = c[i];
    }
    __syncwarp();
    if (kc > j) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i > j) c[i] = fma(-row[i], c[j], c[i]);
    }
    __syncwarp();
  }
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i) col[i] = c[i];
  }
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
  double* Uinv = Yr + 2 * kGN * kLdC;                // inverses of U' diagonal blocks
  double* rdiag = Uinv + 8 * kBlk;                   // R_jj
  double* rinvd = rdiag + kGN;                       // 1 / R_jj
  double* sg = rinvd + kGN;                          // Householder signs s_j
  double* pinv = sg + kGN;                           // 1 / U'_jj
  double* rowbuf = pinv + kGN;                       // 16 (+pad)
  int* s_ok = reinterpret_cast<int*>(rowbuf + 32);
  const GR Gm{Yr, nb};

  const double* om = S.om + S.om_c_rb * args.geo.row_begin[b];

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
  GR_MARK(0);

  // ---------------------------------------------------------------- Cholesky G = R^T R
  double gmax = 0.0;
  for (int j = lane; j < n; j += 32) gmax = fmax(gmax, Gm.at(j, j));
  gmax = warp_max(gmax);
  const double floor_ = 1e-24 * gmax;
  for (int o = 0; o < nb; ++o) {
    if (warp == 0) {
      const bool ok = chol16(Gm.blk(o, o), rdiag + 16 * o, rinvd + 16 * o, rowbuf, floor_);
      if (threadIdx.x == 0) *s_ok = ok;
    }
    __syncthreads();
    if (!*s_ok) {
      if (threadIdx.x == 0) *myflag = 1;
      return;
    }
    const int m = n - 16 * (o + 1);
    if (m > 0) {
      // block row o: R(o, c) = R_oo^{-T} G(o, c), one thread per column
      if (threadIdx.x < m) {
        const int cc = 16 * (o + 1) + threadIdx.x;
        double* bc = Gm.blk(o, cc >> 4);
        const double* bd = Gm.blk(o, o);
        const int cl = cc & 15;
        double x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = bc[bsw(i, cl)];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          x[i] *= rinvd[16 * o + i];
#pragma unroll
          for (int l = 0; l < 16; ++l)
            if (l > i) x[l] = fma(-bd[bsw(i, l)], x[i], x[l]);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) bc[bsw(i, cl)] = x[i];
      }
      __syncthreads();
      // trailing: G(bi, bj) -= R(o, bi)^T R(o, bj), o < bi <= bj (8 x 8 tiles)
      const int mb = nb - o - 1;
      const int units = mb * (mb + 1) / 2 * 4;
      for (int u = warp; u < units; u += kGT / 32) {
        int q = u >> 2, bi = 0;
        while (q >= mb - bi) { q -= mb - bi; ++bi; }
        const int bj = bi + q + o + 1;
        bi += o + 1;
        const int fi = (u >> 1) & 1, fj = u & 1;
        if (bi == bj && fi > fj) continue;
        const double* ra = Gm.blk(o, bi);
        const double* rb2 = Gm.blk(o, bj);
        double* cb = Gm.blk(bi, bj);
        double c0 = cb[bsw(8 * fi + g, 8 * fj + 2 * t)], c1 = cb[bsw(8 * fi + g, 8 * fj + 2 * t + 1)];
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          dmma8x8x4(c0, c1, -ra[bsw(k + t, 8 * fi + g)], rb2[bsw(k + t, 8 * fj + g)]);
        cb[bsw(8 * fi + g, 8 * fj + 2 * t)] = c0;
        cb[bsw(8 * fi + g, 8 * fj + 2 * t + 1)] = c1;
      }
      __syncthreads();
    }
  }
  // screen: the Gram squares cond(Omega); route doubtful boxes to Householder
  if (warp == 0) {
    double lo = INFINITY, hi = 0.0;
    for (int j = lane; j < n; j += 32) { lo = fmin(lo, rdiag[j]); hi = fmax(hi, rdiag[j]); }
    lo = warp_min(lo);
    hi = warp_max(hi);
    if (lane == 0) *s_ok = (hi > 0.0) && isfinite(hi) && lo >= kFallbackRatio * hi;
  }
  __syncthreads();
  GR_MARK(1);
  if (!*s_ok) {
    if (threadIdx.x == 0) *myflag = 1;
    return;
  }

  // ---------------------------------------------------------------- LU of M = Omega_1^T - S R
  for (int o = 0; o < nb; ++o) {
    const int ko = 16 * o;
    if (warp == 0) lu16(X, ko, Gm.blk(o, o), sg + ko, pinv + ko, rowbuf);
    __syncthreads();
    const int m = n - ko - 16;
    if (m > 0) {
      if (threadIdx.x < m) {
        // U12: column c of the block row, minus s_i R(ko + i, c), then L11^{-1}
        const int cc = ko + 16 + threadIdx.x;
        const double* rb2 = Gm.blk(o, cc >> 4);
        const int cl = cc & 15;
        double x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(-sg[ko + i], rb2[bsw(i, cl)], X[(ko + i) + cc * kLdX]);
#pragma unroll
        for (int i = 0; i < 16; ++i)
#pragma unroll
          for (int l = 0; l < 16; ++l)
            if (l > i) x[l] = fma(-X[(ko + l) + (ko + i) * kLdX], x[i], x[l]);
#pragma unroll
        for (int i = 0; i < 16; ++i) X[(ko + i) + cc * kLdX] = x[i];
      } else if (threadIdx.x >= 256 && threadIdx.x < 256 + m) {
        // L21: row c of the block column times U11^{-1}
        const int cr = ko + 16 + (threadIdx.x - 256);
        double y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) y[j] = X[cr + (ko + j) * kLdX];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          y[j] *= pinv[ko + j];
#pragma unroll
          for (int l = 0; l < 16; ++l)
            if (l > j) y[l] = fma(-X[(ko + j) + (ko + l) * kLdX], y[j], y[l]);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) X[cr + (ko + j) * kLdX] = y[j];
      }
      __syncthreads();
      // trailing M(c, d) -= L(c, ko:ko+16) U(ko:ko+16, d), 8 x 8 tiles
      const int mt = m >> 3;
      for (int u = warp; u < mt * mt; u += kGT / 32) {
        const int c0r = ko + 16 + 8 * (u / mt), d0 = ko + 16 + 8 * (u % mt);
        double* cp = X + (c0r + g) + (d0 + 2 * t) * kLdX;
        double c0 = cp[0], c1 = cp[kLdX];
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          dmma8x8x4(c0, c1, -X[(c0r + g) + (ko + k + t) * kLdX], X[(ko + k + t) + (d0 + g) * kLdX]);
        cp[0] = c0;
        cp[kLdX] = c1;
      }
      __syncthreads();
    }
  }
  GR_MARK(2);

  // inverses of U' diagonal blocks (for V2), one warp per block
  if (warp < nb) {
    const int kc = lane & 15, ko = 16 * warp;
    double z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = (i == kc) ? 1.0 : 0.0;
#pragma unroll
    for (int l = 15; l >= 0; --l) {
      z[l] *= pinv[ko + l];
#pragma unroll
      for (int i = 0; i < 15; ++i)
        if (i < l) z[i] = fma(-X[(ko + i) + (ko + l) * kLdX], z[l], z[i]);
    }
    if (lane < 16) {
#pragma unroll
      for (int i = 0; i < 16; ++i) Uinv[warp * kBlk + bsw(i, kc)] = z[i];
    }
  }
  __syncthreads();

  double* fac = S.fac + (size_t)b * S.fac_stride;   // n x s, row j = column j of [R_hh + V1; V2]
  if (warp < 8) {
    // ------------------------------------------------------------ V2 = Omega_2^T U'^{-1}
    for (int rb = warp; 8 * rb < r; rb += 8) {
      const int q = 8 * rb + g;
      const bool qok = q < r;
      double vf[8][4];
#pragma unroll
      for (int bb = 0; bb < 8; ++bb) {
        if (bb < nb) {
        double a[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) a[kk] = qok ? __ldg(om + (int64_t)(16 * bb + 4 * kk + t) * s + n + q) : 0.0;
        if (bb > 0) {
          double ac[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
          for (int pa = 0; pa < 8; ++pa) {
            if (pa < bb) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
#pragma unroll
              for (int f = 0; f < 2; ++f)
                dmma8x8x4(ac[f][0], ac[f][1], vf[pa][kk], X[(16 * pa + 4 * kk + t) + (16 * bb + 8 * f + g) * kLdX]);
            }
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) a[kk] -= cfrag_to_afrag<2>(ac, 4 * kk, lane);
        }
        double ac[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        const double* ui = Uinv + bb * kBlk;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int f = 0; f < 2; ++f) dmma8x8x4(ac[f][0], ac[f][1], a[kk], ui[bsw(4 * kk + t, 8 * f + g)]);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) vf[bb][kk] = cfrag_to_afrag<2>(ac, 4 * kk, lane);
        if (qok) {
#pragma unroll
          for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int e = 0; e < 2; ++e) fac[(size_t)(16 * bb + 8 * f + 2 * t + e) * s + n + q] = ac[f][e];
        }
        }
      }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ T of panel p
    const int p = warp - 8, j0 = 32 * p;
    if (j0 < n) {
      const int nbp = min(32, n - j0), i = lane;
      double z[32];   // row i of U'_pp R_pp^{-1}, then (in place) of -T_p
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        double a = (j >= i && j < nbp && i < nbp) ? X[(j0 + i) + (j0 + j) * kLdX] : 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (k < j) a = fma(-z[k], (j < nbp) ? Gm.at(j0 + k, j0 + j) : 0.0, a);
        z[j] = (j < nbp) ? a * rinvd[j0 + j] : 0.0;
      }
      // (Z S) V1^{-T}: forward substitution over j, in place (z[k < j] final)
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        double a = (j < nbp) ? z[j] * sg[j0 + j] : 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (k < j) a = fma(-z[k], (j < nbp) ? X[(j0 + j) + (j0 + k) * kLdX] : 0.0, a);
        z[j] = a;
      }
      double* tp = S.t + (size_t)b * S.t_stride + (size_t)p * kNB * kNB + (size_t)i * kNB;
#pragma unroll
      for (int j = 0; j < 32; ++j) tp[j] = -z[j];
    }
  }
  // ------------------------------------------------------------ R_hh and V1 rows
  for (int e = threadIdx.x; e < n * n; e += kGT) {
    const int j = e / n, i = e - j * n;
    const double v = (i <= j) ? sg[i] * Gm.at(i, j) : X[i + j * kLdX];
    fac[(size_t)j * s + i] = v;
  }
  if (threadIdx.x == 0) {
    *myflag = 0;
    S.status[b] = kBoxOk;
  }
  GR_MARK(3);
}

size_t gram_smem_bytes() {
  return ((size_t)kGN * kLdX + 2 * kGN * kLdC + 8 * kBlk + 4 * kGN + 40) * sizeof(double);
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
