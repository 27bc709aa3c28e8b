// Batched blocked Householder QR of small fp64 matrices (one CTA per matrix).
//
// Restates the reference's LAPACK path: numpy.linalg.qr -> dgeqrf (blocked,
// dlarfg reflectors, dlarft compact-WY T, dlarfb trailing update) and dorgqr,
// used by `nullspace` (linalg.py:52-62: complete Q of Omega_tau^T, last r
// columns) and `col` (linalg.py:35-49: reduced Q of Y_tau P).  The reflectors
// are the LAPACK ones, so the "last r columns" null-space subspace agrees with
// the reference when nullity > r.
//
// Structure per 32-column panel (512 threads, 16 warps):
//   * panel factorisation: each warp owns two panel columns in registers; one
//     __syncthreads per column; the compact-WY dots v_c . v_j are formed in the
//     same shuffle reductions as the column updates;
//   * T (dlarft recurrence) and R's diagonal-block inverse by two warps;
//   * trailing update A <- (I - V T^T V^T) A on the FP64 tensor cores
//     (DMMA m8n8k4), one 8-column strip per warp, W kept in registers and
//     re-laid out C-fragment -> B-fragment with shuffles.
// kOrtho then forms Q = H_0 ... H_{n-1} [I; 0] block-backward (dorgqr) with
// the same tensor-core block-reflector routine.
#include "common.cuh"
#include "kernels.h"

namespace hbs {

namespace {

constexpr int kP = 32;        // panel width (== kNB)
constexpr int kLdT = kP + 1;  // T / G smem leading dimension

struct Reflector {  // dlarfg for the current pivot
  double tau, beta, scale;
};

HBS_DEV Reflector make_reflector(double alpha, double xn2) {
  Reflector h{0.0, alpha, 0.0};
  if (xn2 != 0.0) {  // beta = -sign(alpha) * hypot(alpha, ||x||)
    h.beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
    h.tau = (h.beta - alpha) / h.beta;
    h.scale = 1.0 / (alpha - h.beta);
  }
  return h;
}

// V(i, q) of panel j0: unit lower trapezoidal, stored in A's panel columns
// (tails already scaled).  q >= nbp -> 0.
HBS_DEV double vval(const double* A, int lda, int j0, int nbp, int i, int q) {
  const int c = j0 + q;
  if (q >= nbp || i < c) return 0.0;
  return i == c ? 1.0 : A[i + c * lda];
}

// Fetch W(p, g) (p = kk + t) from C-fragments acc[f][e] (row g', col 2t'+e)
// into the B-fragment layout (row t, col g) of k-step kk.
template <int NF>
HBS_DEV double cfrag_to_bfrag(const double (&acc)[NF][2], int kk, int lane) {
  // kk is a compile-time constant in every (unrolled) caller, so acc[kk >> 3]
  // resolves to registers and only two shuffles are issued.
  const int g = lane >> 2, t = lane & 3;
  const int src = 4 * ((kk & 7) + t) + (g >> 1);
  const double v0 = __shfl_sync(0xffffffffu, acc[kk >> 3][0], src);
  const double v1 = __shfl_sync(0xffffffffu, acc[kk >> 3][1], src);
  return (g & 1) ? v1 : v0;
}

// A(j0:m, cb:ce) <- (I - V op(T) V^T) A(j0:m, cb:ce), V = panel j0 (nbp cols),
// op(T) = T^T when trans (dgeqrf trailing update, H^T from the left), else T
// (dorgqr).  T in smem (kP x kLdT).  mpad = rows rounded up to 8 (zero rows).
HBS_DEV void block_reflector_apply(double* A, int lda, int mpad, int j0, int nbp, const double* T, bool trans,
                                   int cb, int ce) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nstrip = (ce - cb + 7) >> 3;
  for (int sidx = warp; sidx < nstrip; sidx += nw) {
    const int c0 = cb + 8 * sidx;
    const bool colok = c0 + g < ce;
    // GEMM1: W = V^T A_strip  (32 x 8), K = rows j0 .. mpad
    double w[4][2] = {};
    for (int k = j0; k < mpad; k += 4) {
      const double bv = colok ? A[(k + t) + (c0 + g) * lda] : 0.0;
      if (k < j0 + kP) {
#pragma unroll
        for (int f = 0; f < 4; ++f) dmma8x8x4(w[f][0], w[f][1], vval(A, lda, j0, nbp, k + t, 8 * f + g), bv);
      } else {
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const double av = (8 * f + g < nbp) ? A[(k + t) + (j0 + 8 * f + g) * lda] : 0.0;
          dmma8x8x4(w[f][0], w[f][1], av, bv);
        }
      }
    }
    // GEMM2: W2 = op(T) W (32 x 8)
    double w2[4][2] = {};
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) {
      const double bv = cfrag_to_bfrag<4>(w, kk, lane);
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const int row = 8 * f + g, col = kk + t;
        const double av = trans ? T[col * kLdT + row] : T[row * kLdT + col];
        dmma8x8x4(w2[f][0], w2[f][1], av, bv);
      }
    }
    double bneg[kP / 4];
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) bneg[kk / 4] = -cfrag_to_bfrag<4>(w2, kk, lane);
    // GEMM3: A_strip -= V W2, 8-row blocks, four in flight
    const int col0 = c0 + 2 * t;
    const bool ok0 = col0 < ce, ok1 = col0 + 1 < ce;
    for (int ib = j0; ib < mpad; ib += 32) {
      double cv[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = ib + 8 * u + g;
        const bool rok = ib + 8 * u < mpad;
        cv[u][0] = (ok0 && rok) ? A[i + col0 * lda] : 0.0;
        cv[u][1] = (ok1 && rok) ? A[i + (col0 + 1) * lda] : 0.0;
      }
      if (ib < j0 + kP) {
#pragma unroll
        for (int kk = 0; kk < kP; kk += 4)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            dmma8x8x4(cv[u][0], cv[u][1], vval(A, lda, j0, nbp, ib + 8 * u + g, kk + t), bneg[kk / 4]);
      } else {
#pragma unroll
        for (int kk = 0; kk < kP; kk += 4) {
          const bool qok = kk + t < nbp;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double av = qok ? A[(ib + 8 * u + g) + (j0 + kk + t) * lda] : 0.0;
            dmma8x8x4(cv[u][0], cv[u][1], av, bneg[kk / 4]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = ib + 8 * u + g;
        if (ib + 8 * u < mpad) {
          if (ok0) A[i + col0 * lda] = cv[u][0];
          if (ok1) A[i + (col0 + 1) * lda] = cv[u][1];
        }
      }
    }
  }
}

// Factor panel j0 (nbp <= 32 columns) in place.  Leaves: pre-scale reflector
// values in A (finalised afterwards by the caller), tau/scale/beta in smem,
// G(c, j) = v_c . v_j (c < j) in G.
template <int MR, int CPW>
HBS_DEV void panel_factor(double* A, int lda, int m, int j0, int nbp, double* s_tau, double* s_scale,
                          double* s_beta, double* s_norm) {
  // Warp w owns panel columns j0 + w + nw*u (u < CPW), rows j0 + lane + 32k in x[u][k].
  constexpr int nw = 32 / CPW;        // warps per CTA (compile time)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kc = (m - j0 + 31) >> 5;  // row blocks of 32 from j0 (storage padded to 32)
  double x[CPW][MR];
  int clast = -1;
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    const int c = j0 + warp + nw * u;
    const bool own = (c - j0) < nbp;
    if (own) clast = c;
#pragma unroll
    for (int k = 0; k < MR; ++k) x[u][k] = (own && k < kc) ? A[(j0 + lane + 32 * k) + c * lda] : 0.0;
  }
  if (warp == 0) {  // reflector of the first pivot (column j0 is warp 0, slot u = 0)
    double p = 0.0;
#pragma unroll
    for (int k = 0; k < MR; ++k) {
      const int row = j0 + lane + 32 * k;
      if (k < kc && row > j0) p = fma(x[0][k], x[0][k], p);
    }
    p = warp_sum(p);
    const double alpha = __shfl_sync(0xffffffffu, x[0][0], 0);
    if (lane == 0) {
      const Reflector h = make_reflector(alpha, p);
      s_norm[0] = h.tau; s_norm[1] = h.scale; s_norm[2] = h.beta;
    }
  }
  __syncthreads();
  for (int j = 0; j < nbp; ++j) {
    const int jj = j0 + j;
    const double* sn = s_norm + 3 * (j & 1);
    const double tau = sn[0], scale = sn[1];
    if (threadIdx.x == 0) {
      s_tau[jj] = tau;
      s_scale[jj] = scale;
      s_beta[jj] = sn[2];
    }
    if (clast > jj) {
      double pv[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int row = j0 + lane + 32 * k;
        pv[k] = (k < kc && row > jj) ? A[row + jj * lda] : 0.0;
      }
      // which of my columns is the next pivot (its norm is folded into the same reduction)
      const int nxt = jj + 1;
      const int unx = (j + 1 < nbp && ((j + 1) & (nw - 1)) == warp) ? (j + 1) / nw : -1;
      double d[CPW], r_[CPW];
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        r_[u] = __shfl_sync(0xffffffffu, x[u][0], j);  // row jj sits in slot 0 of lane j
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < MR; ++k) a = fma(pv[k], x[u][k], a);
        d[u] = a;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int u = 0; u < CPW; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
      }
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        const int c = j0 + warp + nw * u;
        if (c > jj && (c - j0) < nbp) {
          const double f = tau * (r_[u] + scale * d[u]), gs = f * scale;
#pragma unroll
          for (int k = 0; k < MR; ++k) x[u][k] = fma(-gs, pv[k], x[u][k]);
          if (lane == j) x[u][0] -= f;
          if (u == unx) {
            double p = 0.0;
#pragma unroll
            for (int k = 0; k < MR; ++k) {
              const int row = j0 + lane + 32 * k;
              if (k < kc && row > nxt) p = fma(x[u][k], x[u][k], p);
            }
            const double nrm = warp_sum(p);
            // publish the next pivot: column, reflector
#pragma unroll
            for (int k = 0; k < MR; ++k)
              if (k < kc) A[(j0 + lane + 32 * k) + nxt * lda] = x[u][k];
            const double alpha = __shfl_sync(0xffffffffu, x[u][0], j + 1);
            if (lane == 0) {
              const Reflector h = make_reflector(alpha, nrm);
              double* so = s_norm + 3 * ((j + 1) & 1);
              so[0] = h.tau; so[1] = h.scale; so[2] = h.beta;
            }
          }
        }
      }
    }
    __syncthreads();
  }
  // write back the owned columns (final values, reflector tails unscaled)
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    const int c = j0 + warp + nw * u;
    if ((c - j0) < nbp) {
#pragma unroll
      for (int k = 0; k < MR; ++k)
        if (k < kc) A[(j0 + lane + 32 * k) + c * lda] = x[u][k];
    }
  }
  __syncthreads();
  // finalise: v tails = x * scale, diagonal = beta
  for (int q = 0; q < nbp; ++q) {
    const int c = j0 + q;
    const double sc = s_scale[c];
    for (int i = j0 + threadIdx.x; i < m; i += blockDim.x) {
      if (i > c) A[i + c * lda] *= sc;
      else if (i == c) A[i + c * lda] = s_beta[c];
    }
  }
  __syncthreads();
}

// G = V_p^T V_p (32 x 32) on the tensor cores; warp w < 16 computes one 8x8 block.
HBS_DEV void panel_gram(const double* A, int lda, int m, int j0, int nbp, double* G) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  for (int blk = warp; blk < 16; blk += nw) {
    const int fi = blk >> 2, fj = blk & 3;
    if (fi > fj) continue;  // only blocks on/above the diagonal are used
    double c0 = 0.0, c1 = 0.0;
    const int kend = round_up(m, 4);
    for (int k = j0; k < kend; k += 4) {
      const int i = k + t;
      double av, bv;
      if (k < j0 + kP) {
        av = vval(A, lda, j0, nbp, i, 8 * fi + g);
        bv = vval(A, lda, j0, nbp, i, 8 * fj + g);
      } else {
        av = (8 * fi + g < nbp) ? A[i + (j0 + 8 * fi + g) * lda] : 0.0;
        bv = (8 * fj + g < nbp) ? A[i + (j0 + 8 * fj + g) * lda] : 0.0;
      }
      dmma8x8x4(c0, c1, av, bv);
    }
    G[(8 * fi + g) * kLdT + 8 * fj + 2 * t] = c0;
    G[(8 * fi + g) * kLdT + 8 * fj + 2 * t + 1] = c1;
  }
}

// T (dlarft forward/columnwise) from G = V^T V and tau, whole CTA:
//   8x8 diagonal blocks by the column recurrence T(0:c, c) = -tau_c T(0:c,0:c) G(0:c, c)
//   (four warps in parallel), then the block formula
//   T = [[T1, -T1 G12 T2], [0, T2]]  for 8+8 -> 16 and 16+16 -> 32.
HBS_DEV void form_t(double* T, double* scratch, const double* G, const double* s_tau, int j0, int nbp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < kP * kLdT; e += blockDim.x) T[e] = 0.0;
  __syncthreads();
  if (warp < 4 && lane < 8) {
    const int base = 8 * warp, a = base + lane;
    double trow[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cc = base + c;
      const double tc = (cc < nbp) ? s_tau[j0 + cc] : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < c; ++q)
        if (q >= lane) acc = fma(trow[q], G[(base + q) * kLdT + cc], acc);
      trow[c] = (lane < c) ? -tc * acc : (lane == c ? tc : 0.0);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) T[a * kLdT + base + c] = trow[c];
  }
  __syncthreads();
  // combine: width 8 -> 16 (two pairs), then 16 -> 32
  for (int w = 8; w < kP; w *= 2) {
    const int npair = kP / (2 * w);
    // X = G12 T2 for every pair  (w x w each)
    for (int e = threadIdx.x; e < npair * w * w; e += blockDim.x) {
      const int pr = e / (w * w), rem = e % (w * w), i = rem / w, c = rem % w;
      const int o1 = 2 * w * pr, o2 = o1 + w;
      double acc = 0.0;
      for (int q = 0; q <= c; ++q) acc = fma(G[(o1 + i) * kLdT + o2 + q], T[(o2 + q) * kLdT + o2 + c], acc);
      scratch[e] = acc;
    }
    __syncthreads();
    // T12 = -T1 X
    for (int e = threadIdx.x; e < npair * w * w; e += blockDim.x) {
      const int pr = e / (w * w), rem = e % (w * w), i = rem / w, c = rem % w;
      const int o1 = 2 * w * pr, o2 = o1 + w;
      double acc = 0.0;
      for (int q = i; q < w; ++q) acc = fma(T[(o1 + i) * kLdT + o1 + q], scratch[pr * w * w + q * w + c], acc);
      T[(o1 + i) * kLdT + o2 + c] = -acc;
    }
    __syncthreads();
  }
}

}  // namespace

// Inverse of R's diagonal 32x32 blocks, one warp per (box, side, block):
// lane c computes column c of R_bb^{-1} (x = e_c; for i = 31..0: x_i /= R_ii,
// x_k -= R_ki x_i for k < i).  R is read from the QR kernel's output.
__global__ void __launch_bounds__(32) rinv_blocks_kernel(GeqrfArgs args) {
  const int p = blockIdx.x;
  const int64_t b = blockIdx.y;
  const GeqrfSide& S = args.side[blockIdx.z];
  const int nb = box_rows(args.geo, b);
  const int n = args.n_is_rows ? nb : args.n_fixed;
  const int j0 = p * kP;
  if (j0 >= n) return;
  const int nbp = min(kP, n - j0);
  __shared__ double Rs[kP][kP + 1];
  const double* R = S.r + (size_t)b * S.r_stride;
  const int c = threadIdx.x;
  for (int i = 0; i < kP; ++i) Rs[i][c] = (i < nbp && c < nbp) ? R[(size_t)(j0 + i) * S.ldr + j0 + c] : (i == c ? 1.0 : 0.0);
  __syncwarp();
  double x[kP];
#pragma unroll
  for (int i = 0; i < kP; ++i) x[i] = (i == c) ? 1.0 : 0.0;
#pragma unroll
  for (int i = kP - 1; i >= 0; --i) {
    x[i] = x[i] / Rs[i][i];
#pragma unroll
    for (int k = 0; k < i; ++k) x[k] = fma(-Rs[k][i], x[i], x[k]);
  }
  double* out = S.rinv + (size_t)b * S.rinv_stride + (size_t)p * kP * kP;
#pragma unroll
  for (int i = 0; i < kP; ++i) out[i * kP + c] = x[i];
}

namespace {
}  // namespace

template <int MR, bool SMEM, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) hqr_kernel(GeqrfArgs args) {
  constexpr int CPW = 1024 / NT;   // panel columns per warp
  extern __shared__ double smem[];
  const int side = blockIdx.y;
  const int64_t b = blockIdx.x;
  const GeqrfSide& S = args.side[side];
  const int nb = box_rows(args.geo, b);
  const int m = args.m_is_rows ? nb : args.m_fixed;
  const int n = args.n_is_rows ? nb : args.n_fixed;
  const int lda = args.lda_max;
  const int mpad = round_up(m, 32);
  const int npanel = (n + kP - 1) / kP;
  const int64_t rb = args.geo.row_begin[b];

  // smem: small vectors | T / G (per panel in ortho mode) | A (if SMEM)
  double* s_tau = smem;
  double* s_scale = s_tau + args.n_max;
  double* s_beta = s_scale + args.n_max;
  double* s_norm = s_beta + args.n_max;
  double* G = smem + round_up(3 * args.n_max + 6, 2);
  double* Tscr = G + kP * kLdT;     // 256-double scratch for form_t
  double* Tbase = Tscr + 256;
  const int tslots = (args.mode == kGeqrfOrtho) ? (args.n_max + kP - 1) / kP : 1;
  double* A = SMEM ? Tbase + (size_t)round_up(kP * kLdT * tslots, 2)
                   : args.gscratch + ((size_t)side * args.geo.nbox + b) * (size_t)lda * args.n_max;

  // load, zero-padding rows m .. mpad-1
  const double* src = S.src + S.src_c_rb * rb + S.src_c_b * b;
  if (S.src_rs == 1) {
    for (int j = 0; j < n; ++j)
      for (int i = threadIdx.x; i < mpad; i += blockDim.x) {
        const bool ok = i < m;
        if (SMEM) cp_async8(&A[i + j * lda], ok ? src + (int64_t)i + (int64_t)j * S.src_cs : src, ok);
        else A[i + j * lda] = ok ? src[(int64_t)i + (int64_t)j * S.src_cs] : 0.0;
      }
    if (SMEM) { cp_async_commit(); cp_async_wait<0>(); }
  } else {
    for (int e = threadIdx.x; e < mpad * n; e += blockDim.x) {
      const int i = e / n, j = e % n;
      A[i + j * lda] = (i < m) ? src[(int64_t)i * S.src_rs + (int64_t)j * S.src_cs] : 0.0;
    }
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5;
  for (int p = 0; p < npanel; ++p) {
    const int j0 = p * kP, nbp = min(kP, n - j0);
    double* T = Tbase + (args.mode == kGeqrfOrtho ? p * kP * kLdT : 0);
    panel_factor<MR, CPW>(A, lda, m, j0, nbp, s_tau, s_scale, s_beta, s_norm);
    panel_gram(A, lda, m, j0, nbp, G);
    __syncthreads();
    form_t(T, Tscr, G, s_tau, j0, nbp);
    if (args.mode == kGeqrfFactor) {
      double* tout = S.t + (size_t)b * S.t_stride + (size_t)p * kP * kP;
      for (int e = threadIdx.x; e < kP * kP; e += blockDim.x) tout[e] = T[(e / kP) * kLdT + e % kP];
    }
    if (j0 + kP < n) block_reflector_apply(A, lda, round_up(m, 8), j0, nbp, T, true, j0 + kP, n);
    __syncthreads();
  }

  if (args.mode == kGeqrfFactor) {
    if (threadIdx.x < 32) {  // sigma screen on diag(R)
      double lo = INFINITY, hi = 0.0;
      for (int j = threadIdx.x; j < n; j += 32) {
        const double d = fabs(A[j + j * lda]);
        lo = fmin(lo, d);
        hi = fmax(hi, d);
      }
      lo = warp_min(lo);
      hi = warp_max(hi);
      if (threadIdx.x == 0) {
        const bool bad = !(hi > 0.0) || lo < args.tol * hi || !isfinite(hi);
        S.status[b] = bad ? kBoxIllConditioned : kBoxOk;
      }
    }
    double* vt = S.vt + (size_t)b * S.vt_stride;
    for (int e = threadIdx.x; e < n * m; e += blockDim.x) {
      const int j = e / m, i = e % m;
      vt[(size_t)j * S.ldvt + i] = (i < j) ? 0.0 : (i == j ? 1.0 : A[i + j * lda]);
    }
    double* R = S.r + (size_t)b * S.r_stride;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, c = e % n;
      R[(size_t)i * S.ldr + c] = (i <= c) ? A[i + c * lda] : 0.0;
    }
    double* tau = S.tau + (size_t)b * S.tau_stride;
    for (int j = threadIdx.x; j < n; j += blockDim.x) tau[j] = s_tau[j];
    return;
  }

  // kOrtho: Q = H_0 ... H_{n-1} [I; 0], panels backwards (dorgqr).
  const int mp8 = round_up(m, 8);
  for (int p = npanel - 1; p >= 0; --p) {
    const int j0 = p * kP, nbp = min(kP, n - j0);
    const double* T = Tbase + p * kP * kLdT;
    // columns right of the panel already hold Q; apply the block reflector
    if (j0 + kP < n) block_reflector_apply(A, lda, mp8, j0, nbp, T, false, j0 + kP, n);
    // S = T V1^T (32 x 32) -> G, one 8x8 fragment per warp (V1 = V(j0:j0+32, :))
    {
      const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
      for (int blk = warp; blk < 16; blk += (int)(blockDim.x >> 5)) {
        const int fi = blk >> 2, fj = blk & 3;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < kP; kk += 4) {
          const double av = T[(8 * fi + g) * kLdT + kk + t];
          const double bv = vval(A, lda, j0, nbp, j0 + 8 * fj + g, kk + t);   // V1^T(q, c) = V(j0 + c, q)
          dmma8x8x4(c0, c1, av, bv);
        }
        G[(8 * fi + g) * kLdT + 8 * fj + 2 * t] = c0;
        G[(8 * fi + g) * kLdT + 8 * fj + 2 * t + 1] = c1;
      }
      __syncthreads();
      // Q panel rows j0.. in 8-row blocks: Q = E - V_p S (computed, then written after a barrier)
      const int nrb = (mp8 - j0) >> 3;
      const int nwarps = blockDim.x >> 5;
      for (int base = 0; base < nrb; base += 2 * nwarps) {
        double qv[2][4][2];   // up to 2 row blocks per warp per chunk
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int rbk = base + warp + u * nwarps;
#pragma unroll
          for (int f = 0; f < 4; ++f) { qv[u][f][0] = 0.0; qv[u][f][1] = 0.0; }
          if (rbk < nrb) {
            const int i = j0 + 8 * rbk + g;
#pragma unroll
            for (int kk = 0; kk < kP; kk += 4) {
              const double av = -vval(A, lda, j0, nbp, i, kk + t);
#pragma unroll
              for (int f = 0; f < 4; ++f) dmma8x8x4(qv[u][f][0], qv[u][f][1], av, G[(kk + t) * kLdT + 8 * f + g]);
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int rbk = base + warp + u * nwarps;
          if (rbk < nrb) {
            const int i = j0 + 8 * rbk + g;
#pragma unroll
            for (int f = 0; f < 4; ++f)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int c = 8 * f + 2 * t + e;
                if (c < nbp) A[i + (j0 + c) * lda] = qv[u][f][e] + (i == j0 + c ? 1.0 : 0.0);
              }
          }
        }
        __syncthreads();
      }
    }
    for (int e = threadIdx.x; e < j0 * nbp; e += blockDim.x) {
      const int c = e / j0, i = e % j0;
      A[i + (j0 + c) * lda] = 0.0;
    }
    __syncthreads();
  }
  double* q = S.q + S.q_c_rb * rb + S.q_c_b * b;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    q[(size_t)i * S.ldq + j] = A[i + j * lda];
  }
}

size_t hqr_smem_bytes(int m_max, int n_max, int mode, bool with_matrix) {
  const int lda = frag_ld(round_up(m_max, 32));
  const int np = (mode == kGeqrfOrtho) ? (n_max + kP - 1) / kP : 1;
  size_t d = round_up(3 * n_max + 6, 2) + kP * kLdT + 256 + round_up(kP * kLdT * np, 2);
  if (with_matrix) d += (size_t)lda * n_max;
  return d * sizeof(double);
}

size_t hqr_scratch_doubles(int m_max, int n_max, int64_t nbox) {
  return 2 * (size_t)nbox * (size_t)frag_ld(round_up(m_max, 32)) * n_max;
}

bool hqr_fits_smem(int m_max, int n_max, int mode) {
  return hqr_smem_bytes(m_max, n_max, mode, true) <= kMaxSmemBytes;
}

template <int MR, int NT>
static int launch_hqr_nt(GeqrfArgs& args, int nsides, cudaStream_t stream) {
  args.lda_max = frag_ld(round_up(args.m_max, 32));
  const bool fits = hqr_fits_smem(args.m_max, args.n_max, args.mode);
  if (!fits && args.gscratch == nullptr) return kErrWorkspace;
  const size_t smem = hqr_smem_bytes(args.m_max, args.n_max, args.mode, fits);
  dim3 grid((unsigned)args.geo.nbox, nsides);
  if (fits) {
    cudaFuncSetAttribute(hqr_kernel<MR, true, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    hqr_kernel<MR, true, NT><<<grid, NT, smem, stream>>>(args);
  } else {
    cudaFuncSetAttribute(hqr_kernel<MR, false, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    hqr_kernel<MR, false, NT><<<grid, NT, smem, stream>>>(args);
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

template <int MR>
static int launch_hqr_mr(GeqrfArgs& args, int nsides, cudaStream_t stream) {
  // The probe factorisation (one matrix per SM at config 4) uses 16 warps; the
  // smaller basis QR runs 8-warp CTAs so two boxes share an SM.
  if (args.mode != kGeqrfFactor) return launch_hqr_nt<MR, 256>(args, nsides, stream);
  const int rc = launch_hqr_nt<MR, 512>(args, nsides, stream);
  if (rc != kOk) return rc;
  dim3 grid((args.n_max + kP - 1) / kP, (unsigned)args.geo.nbox, nsides);
  rinv_blocks_kernel<<<grid, 32, 0, stream>>>(args);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

int launch_hqr(GeqrfArgs args, int nsides, cudaStream_t stream) {
  const int mr = (args.m_max + 31) / 32;
  switch (mr) {
    case 1: return launch_hqr_mr<1>(args, nsides, stream);
    case 2: return launch_hqr_mr<2>(args, nsides, stream);
    case 3: return launch_hqr_mr<3>(args, nsides, stream);
    case 4: return launch_hqr_mr<4>(args, nsides, stream);
    case 5: return launch_hqr_mr<5>(args, nsides, stream);
    case 6: return launch_hqr_mr<6>(args, nsides, stream);
    case 7: return launch_hqr_mr<7>(args, nsides, stream);
    case 8: return launch_hqr_mr<8>(args, nsides, stream);
    case 9: case 10: return launch_hqr_mr<10>(args, nsides, stream);
    case 11: case 12: return launch_hqr_mr<12>(args, nsides, stream);
    case 13: case 14: case 15: case 16: return launch_hqr_mr<16>(args, nsides, stream);
    default: return kErrUnsupported;
  }
}

}  // namespace hbs
