// Batched orthonormal bases U = col(Y_tau P), V = col(Z_tau Q) by CholeskyQR2
// on the FP64 tensor cores.
//
// Reference: `col` (pkg/src/hbs/linalg.py:35-49) takes the Q factor of the
// reduced Householder QR of the n_tau x r block (numpy.linalg.qr), called from
// compress_node_bases (compress.py:155-175).  Only span(U) reaches the result:
// the discrepancy uses the projector U U^T (compress.py:192-197) and the lifted
// samples U^T(...) rotate with the basis, so the parent's samples and every
// later node see the same operator (the tests compare projectors and
// operators).  Any orthonormal basis of the same span
// is therefore a drop-in, and CholeskyQR2 reaches it with GEMM-shaped work:
//
//   pass 1:  G = A^T A (DMMA),  G = R^T R (blocked Cholesky),  A <- A R^{-1}
//   pass 2:  G = A^T A = I + E; if ||E||_F <= 1e-5, A <- A (I + E)^{-1/2} with
//            (I + E)^{-1/2} = I - E/2 + 3/8 E^2 + O(||E||^3) (the E^2 term
//            only when ||E||_F > 1e-8): tensor-core work, no sequential
//            step; else a second full Cholesky pass (classic CholeskyQR2).
//
// One CTA (8 warps, 2 CTAs per SM) per (box, side), the n x r block in shared
// memory.  A breakdown (a pivot below 1e-12 of its column's squared norm, i.e.
// condition number beyond about 1e6, a rank-deficient or zero block, or a
// non-finite value) flags the (box, side); the caller then re-runs the
// Householder kernel (hqr.cu, mode ortho) for the flagged blocks only.
#include <cstdlib>
#include "common.cuh"
#include "kernels.h"

namespace hbs {
namespace {

constexpr int kCT = 256;            // threads per CTA
constexpr int kLdG = 68;            // G / R / Z leading dimension (== 4 mod 16: conflict-free fragments)
constexpr int kRc = 64;             // max Cholesky dimension (r rounded up to 16)
constexpr int kNmax = 128;          // max rows per box

HBS_DEV void csync() { __syncthreads(); }

// 1/sqrt(a) from the float estimate and two Newton steps in double, for
// 1e-36 < a < 1e36 (callers check the range; the library routine's special-
// case branches dominate a Cholesky step).
HBS_DEV double rsqrt_nr(double a) {
  double y = static_cast<double>(rsqrtf(static_cast<float>(a)));
  const double ha = 0.5 * a;
  y = y * fma(-ha * y, y, 1.5);
  y = y * fma(-ha * y, y, 1.5);
  return y;
}

#ifdef HBS_TRACE
__device__ long long g_cq_trace[32];
#define CQ_MARK(i) do { __syncthreads(); if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_cq_trace[i] = clock64(); } while (0)
#else
#define CQ_MARK(i) do { } while (0)
#endif

// G(0:rp, 0:rp) = A^T A for A (npad x rp, row-major, ld lda) on the tensor
// cores; G column-major (G(i, j) at G[i + j*kLdG]); only blocks bi <= bj
// (diagonal blocks in full).
// With e2w != nullptr also forms ||G - I||_F^2 over the leading r x r part
// straight from the fragments: warp w stores its partial sum in e2w[w]
// (deterministic: the caller adds the eight partials in a fixed order).
HBS_DEV void gram(const double* A, int lda, int npad, int rp, double* G, double* e2w = nullptr, int r = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nbk = rp >> 3;
  const int nblk = nbk * (nbk + 1) / 2;
  double e2acc = 0.0;
  for (int q = warp; q < nblk; q += kCT / 32) {
    int bi = 0, rem = q;
    while (rem >= nbk - bi) { rem -= nbk - bi; ++bi; }
    const int bj = bi + rem;
    double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
    int k = 0;
    for (; k + 8 <= npad; k += 8) {
      dmma8x8x4(c0, c1, A[(k + t) * lda + 8 * bi + g], A[(k + t) * lda + 8 * bj + g]);
      dmma8x8x4(d0, d1, A[(k + 4 + t) * lda + 8 * bi + g], A[(k + 4 + t) * lda + 8 * bj + g]);
    }
    if (k < npad) dmma8x8x4(c0, c1, A[(k + t) * lda + 8 * bi + g], A[(k + t) * lda + 8 * bj + g]);
    const int i = 8 * bi + g, j = 8 * bj + 2 * t;
    G[i + j * kLdG] = c0 + d0;
    G[i + (j + 1) * kLdG] = c1 + d1;
    if (e2w) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jj = j + e;
        const double v = (e ? c1 + d1 : c0 + d0) - (i == jj ? 1.0 : 0.0);
        if (i <= jj && jj < r) e2acc = fma(i == jj ? v : 2.0 * v, v, e2acc);
      }
    }
  }
  if (e2w) {
    e2acc = warp_sum(e2acc);
    if (lane == 0) e2w[warp] = e2acc;
  }
}

// Cholesky of the 16 x 16 diagonal block at (o, o) of G (upper triangle holds
// the current Schur complement), in place: upper triangle <- R and
// rdinv[o + j] = 1 / R(j, j).  One warp: lane k (and its mirror k + 16) owns
// column o + k in registers; row j of R is broadcast through `row` (16
// doubles, 16-byte aligned).  Returns false (warp-uniform) on breakdown.
HBS_DEV bool chol16(double* G, int o, const double* gdiag, double* rdinv, double* row) {
  // branch-free body: every lane executes every shuffle and store (lanes
  // 16..31 duplicate lanes 0..15 and write the same values), so the compiler
  // needs no convergence barriers around the shuffles.
  const int lane = threadIdx.x & 31, kc = lane & 15;
  double c[16];
  double* col = G + o + (o + kc) * kLdG;
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = col[i];   // rows > kc are don't-care (masked below)
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double d = __shfl_sync(0xffffffffu, c[j], j);
    ok = ok && (d > 1e-12 * gdiag[o + j]) && (d > 1e-36) && (d < 1e36);
    const double rs = rsqrt_nr(d);
    c[j] = (kc == j) ? d * rs : (kc > j ? c[j] * rs : 0.0);
    rdinv[o + j] = rs;
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
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (i <= kc && lane < 16) col[i] = c[i];
  return __all_sync(0xffffffffu, ok);
}

// Block row o of R: R(o:o+16, c) = R_oo^{-T} S(o:o+16, c) for the trailing
// columns c in [o + 16, rc), one thread per column (threads 0 .. rc-o-17).
HBS_DEV void trsm_row(double* G, int o, int rc, const double* rdinv) {
  const int c = o + 16 + threadIdx.x;
  if (c >= rc) return;
  double* col = G + o + c * kLdG;
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = col[i];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    x[i] *= rdinv[o + i];
#pragma unroll
    for (int l = 1; l < 16; ++l)
      if (l > i) x[l] = fma(-G[(o + i) + (o + l) * kLdG], x[i], x[l]);   // R(o+i, o+l), broadcast
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) col[i] = x[i];
}

// Trailing Schur complement: S(c, d) -= R(o:o+16, c)^T R(o:o+16, d) for
// o + 16 <= c <= d < rc; all threads.
HBS_DEV void schur_update(double* G, int o, int rc) {
  const int m = rc - o - 16;
  for (int e = threadIdx.x; e < m * m; e += kCT) {
    const int ci = e % m, di = e / m;
    if (ci > di) continue;
    const int c = o + 16 + ci, d = o + 16 + di;
    const double* rc_ = G + o + c * kLdG;
    const double* rd_ = G + o + d * kLdG;
    double acc = G[c + d * kLdG];
#pragma unroll
    for (int l = 0; l < 16; ++l) acc = fma(-rc_[l], rd_[l], acc);
    G[c + d * kLdG] = acc;
  }
}

// Z = R_oo^{-1} of the 16 x 16 diagonal block at (o, o): stored transposed in
// the block's strictly lower triangle (Z(i, j), i < j, at
// G[(o + j) + (o + i) * kLdG]); its diagonal is rdinv.  One warp; lane k
// (k < 16) computes column k of Z by back substitution.
HBS_DEV void trinv16(double* G, int o, const double* rdinv) {
  const int lane = threadIdx.x & 31, kc = lane & 15;
  double z[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) z[i] = (i == kc) ? 1.0 : 0.0;
#pragma unroll
  for (int l = 15; l >= 0; --l) {
    z[l] *= rdinv[o + l];
#pragma unroll
    for (int i = 0; i < 15; ++i)
      if (i < l) z[i] = fma(-G[(o + i) + (o + l) * kLdG], z[l], z[i]);   // R(o+i, o+l)
  }
  __syncwarp();
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < kc) G[(o + kc) + (o + i) * kLdG] = z[i];
  }
}

// Z(i, j) (block-local indices) of the inverse diagonal block at origin o.
HBS_DEV double zval(const double* G, const double* rdinv, int o, int i, int j) {
  if (i > j) return 0.0;
  return i == j ? rdinv[o + i] : G[(o + j) + (o + i) * kLdG];
}

// A <- A R^{-1} by block forward substitution per 8-row block, in registers:
// Q_b = (A_b - sum_{a<b} Q_a R_ab) Z_bb over 16-column blocks b < rc/16.
HBS_DEV void apply_rinv(double* A, int lda, int npad, int rc, const double* G, const double* rdinv) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nb16 = rc >> 4;
  for (int rb = warp; rb < (npad >> 3); rb += kCT / 32) {
    double* arow = A + (8 * rb + g) * lda;
    double qf[4][4];   // A-fragments of the finished Q blocks
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (b >= nb16) break;
      const int o = 16 * b;
      double a[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) a[kk] = arow[o + 4 * kk + t];
      if (b > 0) {
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int pa = 0; pa < 4; ++pa) {
          if (pa >= b) break;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int f = 0; f < 2; ++f)
              dmma8x8x4(acc[f][0], acc[f][1], qf[pa][kk], G[(16 * pa + 4 * kk + t) + (o + 8 * f + g) * kLdG]);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) a[kk] -= cfrag_to_afrag<2>(acc, 4 * kk, lane);
      }
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int f = 0; f < 2; ++f) dmma8x8x4(acc[f][0], acc[f][1], a[kk], zval(G, rdinv, o, 4 * kk + t, 8 * f + g));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) qf[b][kk] = cfrag_to_afrag<2>(acc, 4 * kk, lane);
      __syncwarp();
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        arow[o + 8 * f + 2 * t] = acc[f][0];
        arow[o + 8 * f + 2 * t + 1] = acc[f][1];
      }
    }
  }
}

// E(i, j) = G(i, j) - delta_ij from the upper triangle of G; 0 in the padding.
HBS_DEV double eval_e(const double* G, int r, int i, int j) {
  if (i >= r || j >= r) return 0.0;
  return (i <= j ? G[i + j * kLdG] : G[j + i * kLdG]) - (i == j ? 1.0 : 0.0);
}

// B = (I + E)^{-1/2} ~ I - E/2 + 3/8 E^2 (error 5/16 ||E||^3), symmetric:
// strictly lower part into G's lower triangle, diagonal into bdiag.  E is read
// from the upper triangle only, so the writes do not race with the reads.
HBS_DEV void polar_b(double* G, int r, int rp, double* bdiag, bool second_order) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nbk = rp >> 3;
  const int nblk = nbk * (nbk + 1) / 2;
  for (int q = warp; q < nblk; q += kCT / 32) {
    int bj = 0, rem = q;
    while (rem >= nbk - bj) { rem -= nbk - bj; ++bj; }
    const int bi = bj + rem;   // bi >= bj
    double c0 = 0.0, c1 = 0.0;
    if (second_order)   // (3/8 ||E||^2 < 4e-17 otherwise)
      for (int l = 0; l < rp; l += 4)
        dmma8x8x4(c0, c1, eval_e(G, r, 8 * bi + g, l + t), eval_e(G, r, l + t, 8 * bj + g));
    const int i = 8 * bi + g;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 8 * bj + 2 * t + e;
      const double b = (i == j ? 1.0 : 0.0) - 0.5 * eval_e(G, r, i, j) + 0.375 * (e ? c1 : c0);
      if (i == j) bdiag[i] = b;
      else if (i > j) G[i + j * kLdG] = b;
    }
  }
}

// A <- A (I - F), F = upper triangle of E = G - I with the diagonal halved
// (the Cholesky factor of I + E is I + F + O(||E||^2)); only the MMAs of the
// upper block triangle are issued.
HBS_DEV void apply_first_order(double* A, int lda, int npad, int r, int rp, const double* G) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nbk = rp >> 3;
  for (int rb = warp; rb < (npad >> 3); rb += kCT / 32) {
    double* arow = A + (8 * rb) * lda;
    double a[kRc / 4];
#pragma unroll
    for (int kk = 0; kk < kRc / 4; ++kk) a[kk] = (4 * kk < rp) ? arow[g * lda + 4 * kk + t] : 0.0;
    double acc[kRc / 8][2];
#pragma unroll
    for (int f = 0; f < kRc / 8; ++f) { acc[f][0] = 0.0; acc[f][1] = 0.0; }
#pragma unroll
    for (int f = 0; f < kRc / 8; ++f) {
      if (f >= nbk) break;
#pragma unroll
      for (int kk = 0; kk < 2 * f + 2; ++kk) {   // k <= 8 f + 7: the blocks on / above the diagonal
        const int k = 4 * kk + t, c = 8 * f + g;
        const double gv = G[k + c * kLdG];
        const double fv = (k >= r || c >= r) ? 0.0 : (k < c ? gv : (k == c ? 0.5 * (gv - 1.0) : 0.0));
        dmma8x8x4(acc[f][0], acc[f][1], a[kk], fv);
      }
    }
    __syncwarp();
#pragma unroll
    for (int f = 0; f < kRc / 8; ++f) {
      if (f >= nbk) break;
      arow[g * lda + 8 * f + 2 * t] -= acc[f][0];
      arow[g * lda + 8 * f + 2 * t + 1] -= acc[f][1];
    }
  }
}

// A <- A B for the symmetric B of polar_b.
HBS_DEV void apply_b(double* A, int lda, int npad, int rp, const double* G, const double* bdiag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nbk = rp >> 3;
  for (int rb = warp; rb < (npad >> 3); rb += kCT / 32) {
    double* arow = A + (8 * rb) * lda;
    double a[kRc / 4];
#pragma unroll
    for (int kk = 0; kk < kRc / 4; ++kk) a[kk] = (4 * kk < rp) ? arow[g * lda + 4 * kk + t] : 0.0;
    double acc[kRc / 8][2];
#pragma unroll
    for (int f = 0; f < kRc / 8; ++f) { acc[f][0] = 0.0; acc[f][1] = 0.0; }
#pragma unroll
    for (int kk = 0; kk < kRc / 4; ++kk) {
      if (4 * kk >= rp) break;
#pragma unroll
      for (int f = 0; f < kRc / 8; ++f) {
        if (f >= nbk) break;
        const int k = 4 * kk + t, c = 8 * f + g;
        const double bv = k > c ? G[k + c * kLdG] : (k == c ? bdiag[k] : G[c + k * kLdG]);
        dmma8x8x4(acc[f][0], acc[f][1], a[kk], bv);
      }
    }
    __syncwarp();
#pragma unroll
    for (int f = 0; f < kRc / 8; ++f) {
      if (f >= nbk) break;
      arow[g * lda + 8 * f + 2 * t] = acc[f][0];
      arow[g * lda + 8 * f + 2 * t + 1] = acc[f][1];
    }
  }
}

// Full blocked Cholesky of G (rc x rc, 16-wide blocks) and A <- A R^{-1}.
// Returns false on breakdown.
HBS_DEV bool cholesky_pass(double* A, int lda, int npad, int rc, double* G, const double* gdiag, double* rdinv,
                           int* s_ok, double* rowbuf) {
  const int warp = uniform_warp(threadIdx.x >> 5);   // provably warp-uniform branches
  for (int o = 0; o < rc; o += 16) {
    if (warp == 0) {
      const bool ok = chol16(G, o, gdiag, rdinv, rowbuf);
      if (threadIdx.x == 0) *s_ok = ok;
    }
    csync();
    CQ_MARK(8 + o / 16);
    if (!*s_ok) return false;
    if (o + 16 < rc) {
      trsm_row(G, o, rc, rdinv);
      csync();
      schur_update(G, o, rc);
      csync();
    }
  }
  CQ_MARK(12);
  if (warp < (rc >> 4)) trinv16(G, 16 * warp, rdinv);
  csync();
  CQ_MARK(13);
  apply_rinv(A, lda, npad, rc, G, rdinv);
  csync();
  CQ_MARK(14);
  return true;
}

// NF / RF > 0: compile-time rows and rank (specialised launch for the boxes
// with exactly NF rows; the generic launch skips them via skip_rows).
template <int NF, int RF>
__global__ void __launch_bounds__(kCT, 2) cholqr_kernel(GeqrfArgs args, int32_t* flag) {
  extern __shared__ double smem[];
  const int side = blockIdx.y;
  const int64_t b = blockIdx.x;
  const GeqrfSide& S = args.side[side];
  const int nb_rt = box_rows(args.geo, b);
  if (NF ? nb_rt != NF : nb_rt == args.skip_rows) return;   // the other launch owns this box
  const int nb = NF ? NF : nb_rt;
  const int r = RF ? RF : args.n_fixed;
  const int rp = round_up(r, 8), rc = round_up(r, 16);
  const int npad = round_up(nb, 8);
  const int lda = frag_ld(rc);            // columns rp .. rc-1 stay zero
  double* G = smem;                       // kRc x kLdG
  double* gdiag = G + kRc * kLdG;         // kRc
  double* rdinv = gdiag + kRc;            // kRc
  double* rowbuf = rdinv + kRc;           // 32 (Cholesky row broadcast)
  int* s_ok = reinterpret_cast<int*>(rowbuf + 32);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(rowbuf + 34);
  double* s_e2 = rowbuf + 36;             // per-warp partials of ||G - I||_F^2
  double* A = rowbuf + 44;                // npad x lda (16-byte aligned rows)
  int32_t* myflag = flag + (int64_t)side * args.geo.nbox + b;

  CQ_MARK(0);
  const int64_t rb = args.geo.row_begin[b];
  const double* src = S.src + S.src_c_rb * rb + S.src_c_b * b;
  // rows are contiguous r-double runs: one TMA bulk copy per row when aligned
  const bool bulk = S.src_cs == 1 && (r & 1) == 0 && (S.src_rs & 1) == 0 &&
                    (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  if (bulk) {
    if (threadIdx.x == 0) {
      mbar_init(s_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    csync();
    if (threadIdx.x == 0) mbar_expect_tx(s_bar, (unsigned)(nb * r * sizeof(double)));
    csync();
    for (int i = threadIdx.x; i < nb; i += kCT) bulk_g2s(&A[i * lda], src + i * S.src_rs, (unsigned)(r * sizeof(double)), s_bar);
    for (int e = threadIdx.x; e < npad * rc; e += kCT) {
      const int i = e / rc, j = e - i * rc;
      if (i >= nb || j >= r) A[i * lda + j] = 0.0;
    }
  } else {
    for (int e = threadIdx.x; e < npad * rc; e += kCT) {
      const int i = e / rc, j = e - i * rc;
      A[i * lda + j] = (i < nb && j < r) ? __ldcg(src + i * S.src_rs + j * S.src_cs) : 0.0;
    }
  }
  for (int e = threadIdx.x; e < kRc * kLdG; e += kCT) G[e] = 0.0;
  if (bulk) mbar_wait(s_bar, 0);
  csync();
  CQ_MARK(1);

  bool fail = nb < r;
  for (int pass = 0; pass < 3 && !fail; ++pass) {
    gram(A, lda, npad, rp, G, pass ? s_e2 : nullptr, r);
    csync();
    CQ_MARK(2 + 3 * pass);
    if (pass == 0) {
      for (int j = threadIdx.x; j < rc; j += kCT) {
        if (j >= r) {   // identity padding of the Cholesky dimension
          for (int i = 0; i < rc; ++i) G[i + j * kLdG] = (i == j) ? 1.0 : 0.0;
        }
        gdiag[j] = G[j + j * kLdG];
      }
      csync();
    } else {
      // ||E||_F^2 (E = G - I, accumulated by gram): first-order Cholesky
      // finish when ||E||_F <= 1e-8, polar finish when <= 1e-5
      double e2 = 0.0;
#pragma unroll
      for (int w = 0; w < kCT / 32; ++w) e2 += s_e2[w];
      if (e2 <= 1e-16) {
        apply_first_order(A, lda, npad, r, rp, G);
        csync();
        CQ_MARK(16);
        break;
      }
      if (e2 <= 1e-10) {
        polar_b(G, r, rp, rdinv, true);
        csync();
        CQ_MARK(15);
        apply_b(A, lda, npad, rp, G, rdinv);
        csync();
        CQ_MARK(16);
        break;
      }
      if (pass == 2) { fail = true; break; }
      for (int j = threadIdx.x; j < rc; j += kCT) {
        if (j >= r)
          for (int i = 0; i < rc; ++i) G[i + j * kLdG] = (i == j) ? 1.0 : 0.0;
        gdiag[j] = 1.0;
      }
      csync();
    }
    if (!cholesky_pass(A, lda, npad, rc, G, gdiag, rdinv, s_ok, rowbuf)) fail = true;
  }
  if (threadIdx.x == 0) *myflag = fail ? 1 : 0;
  if (fail) return;
  double* q = S.q + S.q_c_rb * rb + S.q_c_b * b;
  for (int e = threadIdx.x; e < nb * r; e += kCT) {
    const int i = e / r, j = e - i * r;
    q[(int64_t)i * S.ldq + j] = A[i * lda + j];
  }
}

}  // namespace

bool cholqr_fits(int n_max, int r) { return n_max <= kNmax && r <= kRc && r >= 1; }

size_t cholqr_smem_bytes(int n_max, int r) {
  return ((size_t)kRc * kLdG + 2 * kRc + 44 + (size_t)round_up(n_max, 8) * frag_ld(round_up(r, 16))) * sizeof(double);
}

extern "C" int hbs_debug_cq_trace(long long* out) {
#ifdef HBS_TRACE
  return cudaMemcpyFromSymbol(out, g_cq_trace, sizeof(long long) * 32) == cudaSuccess ? 0 : 4;
#else
  (void)out;
  return 6;
#endif
}

template <int NF, int RF>
static int launch_cholqr_t(const GeqrfArgs& args, int nsides, int32_t* flag, size_t smem, cudaStream_t stream) {
  cudaFuncSetAttribute(cholqr_kernel<NF, RF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)args.geo.nbox, nsides);
  cholqr_kernel<NF, RF><<<grid, kCT, smem, stream>>>(args, flag);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

int launch_cholqr(GeqrfArgs args, int nsides, int32_t* flag, cudaStream_t stream) {
  const int nmax = args.m_max, r = args.n_fixed;
  if (!cholqr_fits(nmax, r)) return kErrUnsupported;
  size_t smem = cholqr_smem_bytes(nmax, r);
  // HBS_CQ_SOLO=1 (experiment): one CTA per SM instead of two
  static const bool solo = [] { const char* e = std::getenv("HBS_CQ_SOLO"); return e && e[0] == '1'; }();
  if (solo) smem = 120 * 1024;
  args.skip_rows = 0;
#ifndef HBS_NO_CHOLQR_SPECIAL
  if (nmax == 128 && r == 64) {   // config-4 shape: compile-time loop bounds
    const int rc = launch_cholqr_t<128, 64>(args, nsides, flag, smem, stream);
    if (rc != kOk) return rc;
    args.skip_rows = 128;
  }
#endif
  if (args.uniform && args.skip_rows == nmax) return kOk;   // every box went to the specialised launch
  return launch_cholqr_t<0, 0>(args, nsides, flag, smem, stream);
}

}  // namespace hbs
