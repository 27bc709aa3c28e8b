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

#ifdef HBS_TRACE
__device__ long long g_hqr_trace[256];
__device__ int g_hqr_trace_mode = 0;   // record only kernels of this mode
#define HQR_MARK(i) do { __syncthreads(); if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && args.mode == g_hqr_trace_mode) g_hqr_trace[i] = clock64(); } while (0)
#define HQR_STEP(i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && j0 == 0) g_hqr_trace[64 + (i)] = clock64(); } while (0)
#define FUSED_MARK(i) do { if (blockIdx.x == 0 && blockIdx.y == 0) g_hqr_trace[128 + (i)] = clock64(); } while (0)
#define STEP_MARK(i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && j0 == 32 && lane == 0) g_hqr_trace[200 + (i)] = clock64(); } while (0)
__device__ long long g_pf_trace[64];
#ifndef PF_TRACE_J0
#define PF_TRACE_J0 0
#endif
#define PF_MARK(i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && j0 == PF_TRACE_J0 && lane == 0) g_pf_trace[8 * warp + (i)] = clock64(); } while (0)
__device__ long long g_pf_step[64];
#endif
#if defined(HBS_TRACE) && defined(HBS_TRACE_STEP)
// clock stamp once value v is available (warp 1 of the first panel only)
#define PF_DEP(i, v) do { if (blockIdx.x == 0 && blockIdx.y == 0 && j0 == 0 && lane == 0 && warp == 1) { \
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(G + kP * kLdT - 1)), "d"(v) : "memory"); \
    g_pf_step[8 * jl + (i)] = clock64(); } } while (0)
#else
#define PF_DEP(i, v) do { } while (0)
#endif
#ifndef HBS_TRACE
#define PF_MARK(i) do { } while (0)
#define FUSED_MARK(i) do { } while (0)
#define STEP_MARK(i) do { } while (0)
#define HQR_MARK(i) do { } while (0)
#define HQR_STEP(i) do { } while (0)
#endif

namespace {

constexpr int kP = 32;        // panel width (== kNB)
constexpr int kLdT = kP + 1;  // T / G smem leading dimension

struct Reflector {  // dlarfg for the current pivot
  double tau, beta, scale;
};

HBS_DEV Reflector make_reflector(double alpha, double xn2) {
  // dlarfg: beta = -sign(alpha) ||(alpha, x)||, tau = (beta - alpha) / beta,
  // x <- x / (alpha - beta).  Division-free form: with rho = 1 / ||(alpha, x)||,
  // tau = 1 + |alpha| rho and 1 / (alpha - beta) = sign(alpha) / (|alpha| + ||.||).
  Reflector h{0.0, alpha, 0.0};
  if (xn2 != 0.0) {
    const double s2 = fma(alpha, alpha, xn2);
    const double rho = rsqrt(s2);
    const double nrm = s2 * rho;
    h.beta = -copysign(nrm, alpha);
    h.tau = fma(fabs(alpha), rho, 1.0);
    h.scale = copysign(__drcp_rn(fabs(alpha) + nrm), alpha);
  }
  return h;
}

// make_reflector with the reciprocal square root and the reciprocal from
// float seeds refined by two Newton steps in double (about a tenth of the
// issue slots of the IEEE-exact library routines, which dominate a
// single-warp panel step); the library path covers operands outside the
// float seed's range.
HBS_DEV double rsqrt_nr(double a) {
#ifndef PF_EXP_NORANGE
  if (!(a > 1e-30 && a < 1e30)) return rsqrt(a);
#endif
  double y = static_cast<double>(rsqrtf(static_cast<float>(a)));
  const double ha = 0.5 * a;
  y = y * fma(-ha * y, y, 1.5);
  y = y * fma(-ha * y, y, 1.5);
  return y;
}
HBS_DEV double rcp_nr(double a) {
#ifndef PF_EXP_NORANGE
  if (!(a > 1e-30 && a < 1e30)) return __drcp_rn(a);
#endif
  double y = static_cast<double>(__frcp_rn(static_cast<float>(a)));
  y = fma(y, fma(-a, y, 1.0), y);
  y = fma(y, fma(-a, y, 1.0), y);
  return y;
}
HBS_DEV Reflector make_reflector_fast(double alpha, double xn2) {
  Reflector h{0.0, alpha, 0.0};
  if (xn2 != 0.0) {
    const double s2 = fma(alpha, alpha, xn2);
    const double rho = rsqrt_nr(s2);
    const double nrm = s2 * rho;
    h.beta = -copysign(nrm, alpha);
    h.tau = fma(fabs(alpha), rho, 1.0);
    h.scale = copysign(rcp_nr(fabs(alpha) + nrm), alpha);
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

// Warp-group synchronisation: NTG == 0 means the whole CTA (__syncthreads),
// otherwise named barrier 1 over the first NTG threads.
template <int NTG>
HBS_DEV void gsync() {
  if (NTG == 0) __syncthreads();
  else asm volatile("bar.sync 1, %0;\n" ::"n"(NTG) : "memory");
}
template <int NTG>
HBS_DEV int gthreads() { return NTG == 0 ? (int)blockDim.x : NTG; }
// Logical thread index of a warp group.  In the fused kernel (NTG == 256) the
// latency-critical panel group runs on physical warps 8..15, which the warp
// arbiter favours (highest warp id first), so logical = physical ^ 256.
template <int NTG>
HBS_DEV int ltid() { return NTG == 256 ? (int)(threadIdx.x ^ 256u) : (int)threadIdx.x; }

// A(j0:m, cb:ce) <- (I - V op(T) V^T) A(j0:m, cb:ce), V = panel j0 (nbp cols),
// op(T) = T^T when trans (dgeqrf trailing update, H^T from the left), else T
// (dorgqr).  T in smem (kP x kLdT).  mpad = rows rounded up to 8 (zero rows).
template <int NTG>
HBS_DEV void block_reflector_apply(double* A, int lda, int mpad, int j0, int nbp, const double* T, bool trans,
                                   int cb, int ce, int ldt = kLdT, int warp_base = 0) {
  const int warp = (ltid<NTG>() >> 5) - warp_base, lane = ltid<NTG>() & 31, nw = gthreads<NTG>() >> 5;
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
        const double av = trans ? T[col * ldt + row] : T[row * ldt + col];
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
// Panel factorisation in 8-column sub-panels.  In sub-panel q, warp w < 8 owns
// column cs + w (cs = j0 + 8q) in registers (rows j0 + lane + 32k).  Step j
// needs only pivot j: its owner publishes (column in A, tau/scale/beta in
// smem) and arrives on bar[j]; the others wait on bar[j] alone.  bar[] completes
// once per panel (parity = panel & 1).  The owners of earlier sub-panel columns
// form the compact-WY dots v_c . v_j on the fly (G8); after the 8 steps the
// sub-panel's block reflector is applied to the rest of the panel on the
// tensor cores, so only 8 warps ever contend for issue during a step.
template <int MR, int NTG>
HBS_DEV void panel_factor(double* A, int lda, int m, int j0, int nbp, double* s_tau, double* s_scale,
                          double* s_beta, uint64_t* bar, unsigned parity, double* G8, double* T8,
                          double* wpart, double* wfin) {
  constexpr int kSub = 8;
  const int warp = ltid<NTG>() >> 5, lane = ltid<NTG>() & 31, nw = gthreads<NTG>() >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int kc = (m - j0 + 31) >> 5;  // row blocks of 32 from j0 (storage padded to 32)
  for (int cs = j0; cs < j0 + nbp; cs += kSub) {
    const int nsub = min(kSub, j0 + nbp - cs);
    const int jq = cs - j0;           // step index of the sub-panel's first pivot
    if (warp < nsub) {
      const int c = cs + warp;
      double x[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) x[k] = (k < kc) ? A[(j0 + lane + 32 * k) + c * lda] : 0.0;
      if (warp == 0) {  // first pivot of the sub-panel: exact norm
        double p = 0.0;
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          const int row = j0 + lane + 32 * k;
          if (k < kc && row > cs) p = fma(x[k], x[k], p);
        }
        p = warp_sum(p);
        const double alpha = __shfl_sync(0xffffffffu, x[0], jq);   // row cs: slot 0, lane jq (< 32)
        if (lane == 0) {
          const Reflector h = make_reflector(alpha, p);
          s_tau[cs] = h.tau; s_scale[cs] = h.scale; s_beta[cs] = h.beta;
          mbar_arrive(&bar[jq]);
          HQR_STEP(jq);
        }
      }
      for (int i = 0; i < nsub; ++i) {
        const int jj = cs + i, j = jq + i;
        if (c == jj) continue;
        mbar_wait(&bar[j], parity);
        const double tau = s_tau[jj], scale = s_scale[jj];
        double pv[MR];
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          const int row = j0 + lane + 32 * k;
          pv[k] = (k < kc && row > jj) ? A[row + jj * lda] : 0.0;
        }
        const bool pub = (c == jj + 1);   // I publish the next pivot
        double d = 0.0, sxx = 0.0, spp = 0.0;
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          d = fma(pv[k], x[k], d);
          if (pub) {
            const int row = j0 + lane + 32 * k;
            if (row > jj + 1) { sxx = fma(x[k], x[k], sxx); spp = fma(pv[k], pv[k], spp); }
          }
        }
        const double rj = __shfl_sync(0xffffffffu, x[0], j);   // my value in row jj (slot 0, lane j < 32)
        double xn_old = 0.0, pn = 0.0;
        if (pub) {
          pn = __shfl_sync(0xffffffffu, pv[0], j + 1);
          xn_old = __shfl_sync(0xffffffffu, x[0], j + 1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          d += __shfl_xor_sync(0xffffffffu, d, o);
          if (pub) {
            sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
            spp += __shfl_xor_sync(0xffffffffu, spp, o);
          }
        }
        if (c < jj) {   // compact-WY dot v_c . v_jj (my column is a retired reflector)
          if (lane == 0) G8[(c - cs) * kSub + i] = s_scale[c] * (rj + scale * d);
          continue;
        }
        const double f = tau * (rj + scale * d), gs = f * scale;
#pragma unroll
        for (int k = 0; k < MR; ++k) x[k] = fma(-gs, pv[k], x[k]);
        if (lane == j) x[0] -= f;
        if (pub) {
          const double sxp = d - pn * xn_old;
          double nrm = fma(gs * gs, spp, fma(-2.0 * gs, sxp, sxx));
          if (!(nrm > 0.5 * sxx) || sxx == 0.0) {   // cancellation: recompute exactly
            double p = 0.0;
#pragma unroll
            for (int k = 0; k < MR; ++k) {
              const int row = j0 + lane + 32 * k;
              if (k < kc && row > jj + 1) p = fma(x[k], x[k], p);
            }
            nrm = warp_sum(p);
          }
#pragma unroll
          for (int k = 0; k < MR; ++k)
            if (k < kc) A[(j0 + lane + 32 * k) + c * lda] = x[k];
          const double alpha = __shfl_sync(0xffffffffu, x[0], j + 1);
          __syncwarp();
          if (lane == 0) {
            const Reflector h = make_reflector(alpha, nrm);
            s_tau[c] = h.tau; s_scale[c] = h.scale; s_beta[c] = h.beta;
            mbar_arrive(&bar[j + 1]);
            HQR_STEP(j + 1);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < MR; ++k)
        if (k < kc) A[(j0 + lane + 32 * k) + c * lda] = x[k];
    }
    gsync<NTG>();
    if (ltid<NTG>() == 0) HQR_STEP(40 + (jq >> 3) * 4);
    // finalise the sub-panel: v tails = x * scale, diagonal = beta
    for (int q = 0; q < nsub; ++q) {
      const int c = cs + q;
      const double sc = s_scale[c];
      for (int i = c + ltid<NTG>(); i < m; i += gthreads<NTG>()) {
        if (i > c) A[i + c * lda] *= sc;
        else A[i + c * lda] = s_beta[c];
      }
    }
    const int c1 = cs + kSub, c2 = j0 + nbp;   // remaining panel columns
    if (c1 < c2) {
      // T8 (dlarft recurrence, lanes 0..7 of warp 0); meanwhile warps 1..4
      // form partial W = V_sub^T X_rest over K chunks.
      if (warp == 0) {
        if (lane < kSub) {
          double trow[kSub];
#pragma unroll
          for (int cc = 0; cc < kSub; ++cc) {
            const double tc = (cc < nsub) ? s_tau[cs + cc] : 0.0;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < cc; ++q)
              if (q >= lane) acc = fma(trow[q], G8[q * kSub + cc], acc);
            trow[cc] = (lane < cc) ? -tc * acc : (lane == cc ? tc : 0.0);
          }
#pragma unroll
          for (int cc = 0; cc < kSub; ++cc) T8[lane * kSub + cc] = trow[cc];
        }
      }
      gsync<NTG>();   // finalised V visible
      if (ltid<NTG>() == 0) HQR_STEP(41 + (jq >> 3) * 4);
      const int kspan = round_up(m - cs, 4);
      const int nsplit = 4;
      const int kchunk = round_up((kspan + nsplit - 1) / nsplit, 4);
      if (warp >= 1 && warp <= nsplit) {
        const int ws = warp - 1;
        const int kb = cs + ws * kchunk, ke = min(cs + kspan, kb + kchunk);
        double w[3][2] = {};
        for (int k = kb; k < ke; k += 4) {
          const int i = k + t;
          // A = V_sub^T (row g = reflector, col = row index i)
          const double av = (g < nsub && i >= cs + g) ? (i == cs + g ? 1.0 : A[i + (cs + g) * lda]) : 0.0;
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            const int cc = c1 + 8 * f + g;
            const double bv = cc < c2 ? A[i + cc * lda] : 0.0;
            dmma8x8x4(w[f][0], w[f][1], av, bv);
          }
        }
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          wpart[ws * 192 + g * 24 + 8 * f + 2 * t] = w[f][0];
          wpart[ws * 192 + g * 24 + 8 * f + 2 * t + 1] = w[f][1];
        }
      }
      gsync<NTG>();
      if (ltid<NTG>() == 0) HQR_STEP(42 + (jq >> 3) * 4);
      // W' = T8^T (sum of partials)  (8 x 24)
      for (int e = ltid<NTG>(); e < 192; e += gthreads<NTG>()) {
        const int q = e / 24, cc = e % 24;
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < kSub; ++a) {
          const double wa = wpart[a * 24 + cc] + wpart[192 + a * 24 + cc] + wpart[384 + a * 24 + cc] +
                            wpart[576 + a * 24 + cc];
          acc = fma(T8[a * kSub + q], wa, acc);
        }
        wfin[e] = acc;
      }
      gsync<NTG>();
      // X_rest(rows cs.., c1..c2) -= V_sub W'
      const int nrb = (round_up(m, 8) - cs + 7) >> 3;
      for (int u = warp; u < nrb * 3; u += nw) {
        const int rbk = u / 3, f = u % 3;
        const int i = cs + 8 * rbk + g;
        const int col = c1 + 8 * f + 2 * t;
        if (c1 + 8 * f >= c2) continue;
        double c0v = (col < c2) ? A[i + col * lda] : 0.0;
        double c1v = (col + 1 < c2) ? A[i + (col + 1) * lda] : 0.0;
#pragma unroll
        for (int kk = 0; kk < kSub; kk += 4) {
          const int q = kk + t;
          const double av = (q < nsub && i >= cs + q) ? (i == cs + q ? 1.0 : A[i + (cs + q) * lda]) : 0.0;
          const double bv = -wfin[q * 24 + 8 * f + g];
          dmma8x8x4(c0v, c1v, av, bv);
        }
        if (col < c2) A[i + col * lda] = c0v;
        if (col + 1 < c2) A[i + (col + 1) * lda] = c1v;
      }
    }
    gsync<NTG>();
    if (ltid<NTG>() == 0) HQR_STEP(43 + (jq >> 3) * 4);
  }
}

// Whole-panel factorisation (no sub-panels).  NW warps; warp w owns panel
// columns j0 + w + NW*u (u < CPW = 32/NW) in registers (rows j0 + lane + 32k).
// Step j needs only pivot j: its owner publishes (column in A; tau / scale /
// beta in smem; next-pivot norm by the expansion
// ||x - g p||^2 = sxx - 2 g sxp + g^2 spp, recomputed exactly on
// cancellation) and arrives on bar[j]; every other warp waits on bar[j] only.
// Owners of retired columns form the compact-WY dots G(c, j) = v_c . v_j in
// the same reductions, so T needs no separate Gram.  bar[] completes once per
// panel (parity = panel & 1).
template <int MR, int NW, int NTG>
HBS_DEV void panel_factor_wide(double* A, int lda, int m, int j0, int nbp, double* s_tau, double* s_scale,
                               double* s_beta, uint64_t* bar, unsigned parity, double* G) {
  // G(q, j) is only written for q < j < nbp; zero it so form_t never reads
  // stale shared memory for partial panels.
  for (int e = ltid<NTG>(); e < kP * kLdT; e += gthreads<NTG>()) G[e] = 0.0;
  gsync<NTG>();
  constexpr int CPW = 32 / NW;
  const int warp = (ltid<NTG>() >> 5), lane = ltid<NTG>() & 31;
  const int kc = (m - j0 + 31) >> 5;
  double x[CPW][MR];
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    const int q = warp + NW * u;
#pragma unroll
    for (int k = 0; k < MR; ++k) x[u][k] = (q < nbp && k < kc) ? A[(j0 + lane + 32 * k) + (j0 + q) * lda] : 0.0;
  }
  if (warp == 0) {  // first pivot: column j0 (warp 0, u = 0), exact norm
    double p = 0.0;
#pragma unroll
    for (int k = 0; k < MR; ++k)
      if (k < kc && j0 + lane + 32 * k > j0) p = fma(x[0][k], x[0][k], p);
    p = warp_sum(p);
    const double alpha = __shfl_sync(0xffffffffu, x[0][0], 0);
    if (lane == 0) {
      const Reflector h = make_reflector(alpha, p);
      s_tau[j0] = h.tau; s_scale[j0] = h.scale; s_beta[j0] = h.beta;
      mbar_arrive(&bar[0]);
    }
  }
  for (int j = 0; j < nbp; ++j) {
    const int jj = j0 + j;
    const bool tr = (j == 6) && (((j + 1) % NW) == warp);
    if (tr) STEP_MARK(0);
    mbar_wait(&bar[j], parity);
    if (tr) STEP_MARK(1);
    const double tau = s_tau[jj], scale = s_scale[jj];
    double pv[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) {
      const int row = j0 + lane + 32 * k;
      pv[k] = (k < kc && row > jj) ? A[row + jj * lda] : 0.0;
    }
    const bool pubw = (j + 1 < nbp) && (((j + 1) % NW) == warp);   // I own the next pivot
    const int upub = (j + 1) / NW;
    double d[CPW], r_[CPW];
    double sxx = 0.0, spp = 0.0;
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      r_[u] = __shfl_sync(0xffffffffu, x[u][0], j);
      double a = 0.0;
#pragma unroll
      for (int k = 0; k < MR; ++k) a = fma(pv[k], x[u][k], a);
      d[u] = a;
      if (pubw && u == upub) {
#pragma unroll
        for (int k = 0; k < MR; ++k)
          if (j0 + lane + 32 * k > jj + 1) { sxx = fma(x[u][k], x[u][k], sxx); spp = fma(pv[k], pv[k], spp); }
      }
    }
    if (tr) STEP_MARK(2);
    double pn = 0.0, xn_old = 0.0;
    if (pubw) {
      pn = __shfl_sync(0xffffffffu, pv[0], j + 1);
#pragma unroll
      for (int u = 0; u < CPW; ++u)
        if (u == upub) xn_old = __shfl_sync(0xffffffffu, x[u][0], j + 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int u = 0; u < CPW; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
      if (pubw) {
        sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
        spp += __shfl_xor_sync(0xffffffffu, spp, o);
      }
    }
    if (tr) STEP_MARK(3);
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      const int q = warp + NW * u, c = j0 + q;
      if (q >= nbp || c == jj) continue;
      if (c < jj) {   // retired reflector: compact-WY dot v_c . v_jj
        if (lane == 0) G[q * kLdT + j] = s_scale[c] * (r_[u] + scale * d[u]);
        continue;
      }
      const double f = tau * (r_[u] + scale * d[u]), gs = f * scale;
#pragma unroll
      for (int k = 0; k < MR; ++k) x[u][k] = fma(-gs, pv[k], x[u][k]);
      if (lane == j) x[u][0] -= f;
      if (pubw && u == upub) {
        if (tr) STEP_MARK(4);
        const double sxp = d[u] - pn * xn_old;
        double nrm = fma(gs * gs, spp, fma(-2.0 * gs, sxp, sxx));
        if (!(nrm > 0.5 * sxx) || sxx == 0.0) {   // cancellation: recompute exactly
          double p = 0.0;
#pragma unroll
          for (int k = 0; k < MR; ++k)
            if (k < kc && j0 + lane + 32 * k > jj + 1) p = fma(x[u][k], x[u][k], p);
          nrm = warp_sum(p);
        }
#pragma unroll
        for (int k = 0; k < MR; ++k)
          if (k < kc) A[(j0 + lane + 32 * k) + c * lda] = x[u][k];
        if (tr) STEP_MARK(5);
        const double alpha = __shfl_sync(0xffffffffu, x[u][0], j + 1);
        __syncwarp();
        if (lane == 0) {
          const Reflector h = make_reflector(alpha, nrm);
          s_tau[c] = h.tau; s_scale[c] = h.scale; s_beta[c] = h.beta;
          if (tr) STEP_MARK(6);
          mbar_arrive(&bar[j + 1]);
          if (tr) STEP_MARK(7);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    const int q = warp + NW * u;
    if (q < nbp) {
#pragma unroll
      for (int k = 0; k < MR; ++k)
        if (k < kc) A[(j0 + lane + 32 * k) + (j0 + q) * lda] = x[u][k];
    }
  }
  gsync<NTG>();
  for (int q = 0; q < nbp; ++q) {   // finalise: v tails = x * scale, diagonal = beta
    const int c = j0 + q;
    const double sc = s_scale[c];
    for (int i = c + ltid<NTG>(); i < m; i += gthreads<NTG>()) {
      if (i > c) A[i + c * lda] *= sc;
      else A[i + c * lda] = s_beta[c];
    }
  }
  gsync<NTG>();
}

// Panel factorisation with 8-lane column groups (warps 0..7 of the CTA).
// Lane group lg = lane / 8 of warp w owns panel column q = 4w + lg; lane
// li = lane % 8 of the group holds rows j0 + li + 8k (k < MR8) in registers.
// Every column-dot reduction is a 3-stage xor shuffle inside the group, and
// the four groups of a warp reduce in the same shuffle instructions.  Step j
// needs only pivot j (mbarrier hand-off from the warp owning it); a step is
// bound by the FP64 and shuffle/shared pipes the active warps share, so warp
// w stops after step 4w+3 (its columns are all reflectors by then) and only
// the publishing warp runs the next pivot's norm.  The compact-WY dots
// V^T V for form_t come from one tensor-core Gram product afterwards.
template <int NTG>
HBS_DEV void panel_gram(const double* A, int lda, int m, int j0, int nbp, double* G);

// Transposed butterfly: four per-lane partial sums -> on return lanes
// 8s .. 8s+7 hold the warp-wide sum of slot s = lane >> 3 (6 shuffles, 5 stages).
HBS_DEV double reduce4_t(const double (&a)[4], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8;
  const double k0 = (b4 ? a[2] : a[0]) + __shfl_xor_sync(0xffffffffu, b4 ? a[0] : a[2], 16);
  const double k1 = (b4 ? a[3] : a[1]) + __shfl_xor_sync(0xffffffffu, b4 ? a[1] : a[3], 16);
  double k = (b3 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return k;
}

// Panel factorisation with warp-local column blocks (warps 0..7 of the group).
// Warp w holds panel columns 4w .. 4w+3 in registers, lane l rows j0 + l + 32k.
// It first applies the reflectors of the earlier warps' columns as they are
// published (mbarrier per reflector, one step behind the producer), then
// factors its own four columns with no cross-warp traffic: a step is the
// pivot's dots, one transposed 4-slot butterfly, the rank-1 update and the
// next pivot's norm by the update formula (exact recomputation on
// cancellation), so only every fourth pivot crosses warps.  Published
// columns hold the final R entries, beta and the dlarfg-scaled tails; the
// compact-WY dots V^T V for form_t come from one tensor-core Gram product.
template <int MR, int NTG>
HBS_DEV void panel_factor_r(double* A, int lda, int m, int j0, int nbp, double* s_tau, double* s_scale,
                            double* s_beta, uint64_t* bar, unsigned parity, double* G) {
  const int warp = ltid<NTG>() >> 5, lane = ltid<NTG>() & 31;
  if (warp < ((nbp + 3) >> 2)) {
    const int cb = 4 * warp;     // my first panel column
    const int mr = m - j0;       // panel rows; relative row of (lane, k) = lane + 32 k
    double x[4][MR];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int row = lane + 32 * k;
        x[c][k] = (cb + c < nbp && row < mr) ? A[(j0 + row) + (j0 + cb + c) * lda] : 0.0;
      }
    PF_MARK(0);
    // reflectors 0 .. cb-1 (earlier warps), applied as they are published
    for (int j = 0; j < cb; ++j) {
#ifdef PF_EXP_SLEEP
      mbar_wait_sleep(&bar[j], parity);
#else
      mbar_wait(&bar[j], parity);
#endif
      const double tau = s_tau[j0 + j];
      double v[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int row = lane + 32 * k;
        v[k] = (k > 0 || row > j) ? (row < mr ? A[(j0 + row) + (j0 + j) * lda] : 0.0) : (row == j ? 1.0 : 0.0);
      }
      double pc[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          if (k & 1) a1 = fma(v[k], x[c][k], a1);
          else a0 = fma(v[k], x[c][k], a0);
        }
        pc[c] = a0 + a1;
      }
      const double tot = tau * reduce4_t(pc, lane);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double w = __shfl_sync(0xffffffffu, tot, 8 * c);
#pragma unroll
        for (int k = 0; k < MR; ++k) x[c][k] = fma(-w, v[k], x[c][k]);
      }
    }
    PF_MARK(1);
    // my first pivot: exact norm below row cb, alpha = row cb (lane cb, slot 0)
    double nrm, alpha;
    {
      double pp = 0.0;
#pragma unroll
      for (int k = 0; k < MR; ++k)
        if (k > 0 || lane > cb) pp = fma(x[0][k], x[0][k], pp);
      nrm = warp_sum(pp);
      alpha = __shfl_sync(0xffffffffu, x[0][0], cb);
    }
    PF_MARK(2);
    // publish column j: R above, beta on the diagonal, scaled tail below
    auto publish = [&](int j, const Reflector& hh, const double (&xc)[MR]) {
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int row = lane + 32 * k;
        if (row < mr) A[(j0 + row) + (j0 + j) * lda] = row < j ? xc[k] : (row == j ? hh.beta : xc[k] * hh.scale);
      }
      if (lane == 0) { s_tau[j0 + j] = hh.tau; s_scale[j0 + j] = hh.scale; s_beta[j0 + j] = hh.beta; }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[j]);
    };
    Reflector hp{0.0, 0.0, 0.0};
    double xp[MR];
    int pubc = -1;
#pragma unroll
    for (int jl = 0; jl < 4; ++jl) {
      const int j = cb + jl;
      if (j >= nbp) break;
      PF_DEP(0, 0.0);
#ifdef PF_EXP_NOREFL
      const Reflector h{1.5 + 1e-300 * alpha, alpha, 0.5 + 1e-300 * nrm};
#elif defined(PF_EXP_FASTREFL)
      const Reflector h = make_reflector_fast(alpha, nrm);
#else
      const Reflector h = make_reflector(alpha, nrm);
#endif
#ifndef PF_EXP_NOPUB
      if (pubc >= 0) { publish(cb + pubc, hp, xp); pubc = -1; }
#endif
      double pv[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) pv[k] = (k > 0 || lane > j) ? x[jl][k] : 0.0;   // j < 32
      double pc[4] = {0.0, 0.0, 0.0, 0.0}, r[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int c = jl + 1; c < 4; ++c) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          if (k & 1) a1 = fma(pv[k], x[c][k], a1);
          else a0 = fma(pv[k], x[c][k], a0);
        }
        pc[c] = a0 + a1;
        r[c] = __shfl_sync(0xffffffffu, x[c][0], j);   // row j of column c
      }
      // next pivot (column jl+1): ||x||^2, ||pv||^2 over rows > j+1, row j+1 values
      double sxx = 0.0, spp = 0.0, xn_old = 0.0, pn = 0.0;
      if (jl < 3) {
#pragma unroll
        for (int k = 0; k < MR; ++k)
          if (k > 0 || lane > j + 1) { sxx = fma(x[jl + 1][k], x[jl + 1][k], sxx); spp = fma(pv[k], pv[k], spp); }
        xn_old = __shfl_sync(0xffffffffu, x[jl + 1][0], j + 1);
        pn = __shfl_sync(0xffffffffu, pv[0], j + 1);
      }
      PF_DEP(1, pc[3] + r[3] + sxx + spp);
      const double dsum = reduce4_t(pc, lane);
      PF_DEP(2, dsum);
      PF_DEP(3, h.tau * h.scale);
      if (jl < 3) { sxx = warp_sum(sxx); spp = warp_sum(spp); }
      double gsn = 0.0, dn = 0.0;
#pragma unroll
      for (int c = jl + 1; c < 4; ++c) {
        const double dc = __shfl_sync(0xffffffffu, dsum, 8 * c);
        const double f = h.tau * (r[c] + h.scale * dc), gs = f * h.scale;
#pragma unroll
        for (int k = 0; k < MR; ++k) x[c][k] = fma(-gs, pv[k], x[c][k]);
        if (lane == j) x[c][0] -= f;
        if (c == jl + 1) { gsn = gs; dn = dc; }
      }
      PF_DEP(4, x[3][0] + x[3][MR - 1]);
      if (jl < 3 && j + 1 < nbp) {
        // ||x'||^2 = sxx - 2 gs (x . pv) + gs^2 spp over rows > j+1
        double nn = fma(gsn * gsn, spp, fma(-2.0 * gsn, dn - pn * xn_old, sxx));
        alpha = fma(-gsn, pn, xn_old);
#ifndef PF_EXP_NONEED
        if (!(nn > 0.5 * sxx) || sxx == 0.0) {   // warp-uniform
          double pp = 0.0;
#pragma unroll
          for (int k = 0; k < MR; ++k)
            if (k > 0 || lane > j + 1) pp = fma(x[jl + 1][k], x[jl + 1][k], pp);
          nn = warp_sum(pp);
        }
#endif
        nrm = nn;
      }
      PF_DEP(5, nrm + alpha);
      // column j is published at the top of the next step (after that
      // step's reflector is issued) or after the loop
#ifdef PF_EXP_DEFER
      hp = h;
      pubc = jl;
#pragma unroll
      for (int k = 0; k < MR; ++k) xp[k] = x[jl][k];
#else
      publish(j, h, x[jl]);
#endif
      PF_MARK(3 + jl);
      PF_DEP(6, 0.0);
    }
    if (pubc >= 0) publish(cb + pubc, hp, xp);
  }
  gsync<NTG>();
  panel_gram<NTG>(A, lda, m, j0, nbp, G);   // compact-WY dots V^T V for form_t
  gsync<NTG>();
}

template <int MR8, int NTG>
HBS_DEV void panel_factor_q(double* A, int lda, int m, int j0, int nbp, double* s_tau, double* s_scale,
                            double* s_beta, uint64_t* bar, unsigned parity, double* G, double* s_an) {
  // s_an[j] = alpha (pre-reflection diagonal), s_an[32 + j] = ||x||^2 of pivot j:
  // the publisher stores only these; every warp forms the reflector itself,
  // overlapped with its own loads and reductions (off the critical chain).
  const int warp = (ltid<NTG>() >> 5), lane = ltid<NTG>() & 31;
  if (warp < 8) {
    const int lg = lane >> 3, li = lane & 7, gbase = lane & 24;
    // contiguous columns per warp: warp w retires after step 4w+3 and leaves
    // the pipes to the warps still updating
    const int q = 4 * warp + lg, c = j0 + q, jlast = 4 * warp + 3;
    const bool own = q < nbp;
    const int kc = (m - j0 + 7) >> 3;
    double x[MR8];
#pragma unroll
    for (int k = 0; k < MR8; ++k) x[k] = (own && k < kc) ? A[(j0 + li + 8 * k) + c * lda] : 0.0;
    if (warp == 0) {  // first pivot j0 = column q 0 (warp 0, group 0): exact norm
      double p = 0.0;
#pragma unroll
      for (int k = 0; k < MR8; ++k)
        if (k < kc && li + 8 * k > 0) p = fma(x[k], x[k], p);
      p += __shfl_xor_sync(0xffffffffu, p, 4);
      p += __shfl_xor_sync(0xffffffffu, p, 2);
      p += __shfl_xor_sync(0xffffffffu, p, 1);
      const double alpha = __shfl_sync(0xffffffffu, x[0], 0);
      if (lane == 0) {
        s_an[0] = alpha; s_an[32] = p;
        mbar_arrive(&bar[0]);
      }
    }
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {          // row slot of the pivot: kb = j / 8 (compile time)
      for (int jl = 0; jl < 8; ++jl) {
        const int j = 8 * kb + jl, jj = j0 + j;
        if (j >= nbp || j > jlast) break;
        const bool tr = (j == 6) && own && (q == 7) && li == 0;
        // warp-uniform: this warp owns pivot j+1 (group (j+1)%4 of warp (j+1)/4).
        // Only it runs the norm / publish work and its shuffles: the SM's
        // shuffle and shared-memory pipes, shared by the eight warps, bound a step.
        const bool pubw = warp == ((j + 1) >> 2) && j + 1 < nbp;
        mbar_wait(&bar[j], parity);
        if (tr) STEP_MARK(0);
        double pv[MR8];
#pragma unroll
        for (int k = 0; k < MR8; ++k) {
          const int row = j0 + li + 8 * k;
          pv[k] = (k < kc && row > jj) ? A[row + jj * lda] : 0.0;
        }
        const Reflector hj = make_reflector(s_an[j], s_an[32 + j]);
        const double tau = hj.tau, scale = hj.scale;
        if (tr) STEP_MARK(1);
        if (c == jj && li == 0) { s_tau[jj] = hj.tau; s_scale[jj] = hj.scale; s_beta[jj] = hj.beta; }
        if (tr) STEP_MARK(2);
        const bool pub = own && (q == j + 1);
        // my value in row jj (slot kb, lane jl of my group)
        const double r = __shfl_sync(0xffffffffu, x[kb], gbase | jl);
        double dd[8] = {};
#pragma unroll
        for (int k = 0; k < MR8; ++k) dd[k & 7] = fma(pv[k], x[k], dd[k & 7]);
        if (tr) STEP_MARK(3);
        double d = ((dd[0] + dd[1]) + (dd[2] + dd[3])) + ((dd[4] + dd[5]) + (dd[6] + dd[7]));
        // publisher warp: ||x||^2 and ||pv||^2 over rows > jj+1 (pre-update x),
        // and the row-(jj+1) values of x and pv
        double sxx = 0.0, spp = 0.0, xn_old = 0.0, pn = 0.0;
        if (pubw) {
          double sx[4] = {}, sp[4] = {};
#pragma unroll
          for (int k = 0; k < MR8; ++k)
            if (li + 8 * k > j + 1) { sx[k & 3] = fma(x[k], x[k], sx[k & 3]); sp[k & 3] = fma(pv[k], pv[k], sp[k & 3]); }
          sxx = (sx[0] + sx[1]) + (sx[2] + sx[3]);
          spp = (sp[0] + sp[1]) + (sp[2] + sp[3]);
          const int nl = (jl == 7) ? gbase : (gbase | (jl + 1));
          xn_old = __shfl_sync(0xffffffffu, (jl == 7) ? x[kb < 3 ? kb + 1 : kb] : x[kb], nl);
          pn = __shfl_sync(0xffffffffu, (jl == 7) ? pv[kb < 3 ? kb + 1 : kb] : pv[kb], nl);
        }
        d += __shfl_xor_sync(0xffffffffu, d, 4);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        if (tr) STEP_MARK(4);
        const double f = tau * (r + scale * d), gs = f * scale;
        if (own && c > jj) {
#pragma unroll
          for (int k = 0; k < MR8; ++k) x[k] = fma(-gs, pv[k], x[k]);
          if (li == jl) x[kb] -= f;
        }
        if (tr) STEP_MARK(5);
        if (pubw) {
          sxx += __shfl_xor_sync(0xffffffffu, sxx, 4);
          spp += __shfl_xor_sync(0xffffffffu, spp, 4);
          sxx += __shfl_xor_sync(0xffffffffu, sxx, 2);
          spp += __shfl_xor_sync(0xffffffffu, spp, 2);
          sxx += __shfl_xor_sync(0xffffffffu, sxx, 1);
          spp += __shfl_xor_sync(0xffffffffu, spp, 1);
          // next pivot: ||x'||^2 over rows > jj+1 = sxx - 2 gs sxp + gs^2 spp,
          // recomputed exactly on cancellation; alpha = updated row jj+1
          double nrm = fma(gs * gs, spp, fma(-2.0 * gs, d - pn * xn_old, sxx));
          const double alpha = fma(-gs, pn, xn_old);
          if (tr) STEP_MARK(6);
          const bool need = pub && (!(nrm > 0.5 * sxx) || sxx == 0.0);
          if (__any_sync(0xffffffffu, need)) {
            double pp = 0.0;
#pragma unroll
            for (int k = 0; k < MR8; ++k)
              if (k < kc && li + 8 * k > j + 1) pp = fma(x[k], x[k], pp);
            pp += __shfl_xor_sync(0xffffffffu, pp, 4);
            pp += __shfl_xor_sync(0xffffffffu, pp, 2);
            pp += __shfl_xor_sync(0xffffffffu, pp, 1);
            if (need) nrm = pp;
          }
          if (tr) STEP_MARK(7);
          if (pub) {
#pragma unroll
            for (int k = 0; k < MR8; ++k)
              if (k < kc) A[(j0 + li + 8 * k) + c * lda] = x[k];
          }
          __syncwarp();
          if (pub && li == 0) {
            s_an[j + 1] = alpha; s_an[32 + j + 1] = nrm;
            if (tr) STEP_MARK(8);
            mbar_arrive(&bar[j + 1]);
            if (tr) STEP_MARK(9);
          }
        }
      }
    }
    if (own) {
#pragma unroll
      for (int k = 0; k < MR8; ++k)
        if (k < kc) A[(j0 + li + 8 * k) + c * lda] = x[k];
    }
  }
  gsync<NTG>();
  for (int qq = 0; qq < nbp; ++qq) {   // finalise: v tails = x * scale, diagonal = beta
    const int cc = j0 + qq;
    const double sc = s_scale[cc];
    for (int i = cc + ltid<NTG>(); i < m; i += gthreads<NTG>()) {
      if (i > cc) A[i + cc * lda] *= sc;
      else A[i + cc * lda] = s_beta[cc];
    }
  }
  gsync<NTG>();
  panel_gram<NTG>(A, lda, m, j0, nbp, G);   // compact-WY dots V^T V for form_t
  gsync<NTG>();
}

// G = V_p^T V_p (32 x 32) on the tensor cores; warp w < 16 computes one 8x8 block.
template <int NTG>
HBS_DEV void panel_gram(const double* A, int lda, int m, int j0, int nbp, double* G) {
  const int warp = ltid<NTG>() >> 5, lane = ltid<NTG>() & 31, nw = gthreads<NTG>() >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int kend = round_up(m, 4);
  for (int blk = warp; blk < 16; blk += nw) {
    const int fi = blk >> 2, fj = blk & 3;
    if (fi > fj) continue;  // only blocks on/above the diagonal are used
    // four independent accumulator chains (k-steps interleaved); rows above
    // j0 + 8 fj are zero in column block fj
    double c[4][2] = {};
    int k = j0 + 8 * fj;
    for (; k < j0 + kP && k < kend; k += 4) {
      const int i = k + t;
      dmma8x8x4(c[(k >> 2) & 3][0], c[(k >> 2) & 3][1], vval(A, lda, j0, nbp, i, 8 * fi + g),
                vval(A, lda, j0, nbp, i, 8 * fj + g));
    }
    const bool oki = 8 * fi + g < nbp, okj = 8 * fj + g < nbp;
    const double* ci = A + (j0 + 8 * fi + g) * lda;
    const double* cj = A + (j0 + 8 * fj + g) * lda;
    for (; k < kend; k += 16) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = k + 4 * u + t;
        const bool in = k + 4 * u < kend;
        av[u] = (in && oki) ? ci[i] : 0.0;
        bv[u] = (in && okj) ? cj[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma8x8x4(c[u][0], c[u][1], av[u], bv[u]);
    }
    G[(8 * fi + g) * kLdT + 8 * fj + 2 * t] = (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
    G[(8 * fi + g) * kLdT + 8 * fj + 2 * t + 1] = (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
  }
}

// T (dlarft forward/columnwise) from G = V^T V and tau, whole CTA:
//   8x8 diagonal blocks by the column recurrence T(0:c, c) = -tau_c T(0:c,0:c) G(0:c, c)
//   (four warps in parallel), then the block formula
//   T = [[T1, -T1 G12 T2], [0, T2]]  for 8+8 -> 16 and 16+16 -> 32.
template <int NTG>
HBS_DEV void form_t(double* T, double* scratch, const double* G, const double* s_tau, int j0, int nbp) {
  const int warp = (ltid<NTG>() >> 5), lane = ltid<NTG>() & 31;
  for (int e = ltid<NTG>(); e < kP * kLdT; e += gthreads<NTG>()) T[e] = 0.0;
  gsync<NTG>();
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
  gsync<NTG>();
  // combine: width 8 -> 16 (two pairs), then 16 -> 32
  for (int w = 8; w < kP; w *= 2) {
    const int npair = kP / (2 * w);
    // X = G12 T2 for every pair  (w x w each)
    for (int e = ltid<NTG>(); e < npair * w * w; e += gthreads<NTG>()) {
      const int pr = e / (w * w), rem = e % (w * w), i = rem / w, c = rem % w;
      const int o1 = 2 * w * pr, o2 = o1 + w;
      double acc = 0.0;
      for (int q = 0; q <= c; ++q) acc = fma(G[(o1 + i) * kLdT + o2 + q], T[(o2 + q) * kLdT + o2 + c], acc);
      scratch[e] = acc;
    }
    gsync<NTG>();
    // T12 = -T1 X
    for (int e = ltid<NTG>(); e < npair * w * w; e += gthreads<NTG>()) {
      const int pr = e / (w * w), rem = e % (w * w), i = rem / w, c = rem % w;
      const int o1 = 2 * w * pr, o2 = o1 + w;
      double acc = 0.0;
      for (int q = i; q < w; ++q) acc = fma(T[(o1 + i) * kLdT + o1 + q], scratch[pr * w * w + q * w + c], acc);
      T[(o1 + i) * kLdT + o2 + c] = -acc;
    }
    gsync<NTG>();
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
  if (args.only && args.only[side * args.geo.nbox + b] == 0) return;
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
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_beta + args.n_max);   // 32 step barriers
  double* G = smem + round_up(3 * args.n_max + 32, 2);
  double* Tscr = G + kP * kLdT;     // 384-double scratch (form_t, sub-panel G8/T8/W')
  double* Tbase = Tscr + 384;
  const int tslots = (args.mode == kGeqrfOrtho) ? (args.n_max + kP - 1) / kP : 1;
  double* A = SMEM ? Tbase + (size_t)round_up(kP * kLdT * tslots, 2)
                   : args.gscratch + ((size_t)side * args.geo.nbox + b) * (size_t)lda * args.n_max;

  HQR_MARK(0);
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

  const int warp = (threadIdx.x >> 5);
  HQR_MARK(1);
  if (threadIdx.x < kP) mbar_init(&s_bar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  for (int p = 0; p < npanel; ++p) {
    const int j0 = p * kP, nbp = min(kP, n - j0);
    double* T = Tbase + (args.mode == kGeqrfOrtho ? p * kP * kLdT : 0);
    HQR_MARK(2 + 4 * p);
    if constexpr (MR <= 6) panel_factor_r<MR, 0>(A, lda, m, j0, nbp, s_tau, s_scale, s_beta, s_bar, (unsigned)(p & 1), G);
    else panel_factor_wide<MR, NT / 32, 0>(A, lda, m, j0, nbp, s_tau, s_scale, s_beta, s_bar, (unsigned)(p & 1), G);
    HQR_MARK(3 + 4 * p);
    form_t<0>(T, Tscr, G, s_tau, j0, nbp);
    if (args.mode == kGeqrfFactor) {
      double* tout = S.t + (size_t)b * S.t_stride + (size_t)p * kP * kP;
      for (int e = threadIdx.x; e < kP * kP; e += blockDim.x) tout[e] = T[(e / kP) * kLdT + e % kP];
    }
    HQR_MARK(4 + 4 * p);
    if (j0 + kP < n) block_reflector_apply<0>(A, lda, round_up(m, 8), j0, nbp, T, true, j0 + kP, n);
    HQR_MARK(5 + 4 * p);
    __syncthreads();
  }

  HQR_MARK(40);
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
    HQR_MARK(41);
    return;
  }

  // kOrtho: Q = H_0 ... H_{n-1} [I; 0], panels backwards (dorgqr).
  const int mp8 = round_up(m, 8);
  for (int p = npanel - 1; p >= 0; --p) {
    const int j0 = p * kP, nbp = min(kP, n - j0);
    const double* T = Tbase + p * kP * kLdT;
    // columns right of the panel already hold Q; apply the block reflector
    if (j0 + kP < n) block_reflector_apply<0>(A, lda, mp8, j0, nbp, T, false, j0 + kP, n);
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
  size_t d = round_up(3 * n_max + 32, 2) + kP * kLdT + 384 + round_up(kP * kLdT * np, 2);
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

extern "C" int hbs_debug_hqr_trace(long long* out) {
#ifdef HBS_TRACE
  if (cudaMemcpyFromSymbol(out + 256, g_pf_trace, sizeof(long long) * 64) != cudaSuccess) return 4;
  return cudaMemcpyFromSymbol(out, g_hqr_trace, sizeof(long long) * 256) == cudaSuccess ? 0 : 4;
#else
  (void)out;
  return 6;
#endif
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


// ============================================================================
// Fused probe QR + apply-Q + solve.
// ============================================================================
namespace {

// inverse of the 32x32 upper-triangular block R(j0:j0+32, j0:j0+32) (in A)
// into out (32 x kLdT) by the group: 8x8 diagonal blocks by lane-per-column
// back substitution, then inv([[A,B],[0,C]]) = [[A^-1, -A^-1 B C^-1],[0, C^-1]].
template <int NTG, int BAR>
HBS_DEV void ysync() { asm volatile("bar.sync %0, %1;\n" ::"n"(BAR), "n"(NTG) : "memory"); }

// Inverse of the 32x32 upper-triangular block R(j0:j0+32, j0:j0+32) (in A),
// by the warp group starting at warp `wb` (NTG threads, named barrier BAR):
// 8x8 diagonal blocks by lane-per-column back substitution, then
// inv([[A,B],[0,C]]) = [[A^-1, -A^-1 B C^-1],[0, C^-1]] for 8+8 and 16+16.
// out / scratch may live in global memory (row-major, ld 32 / 256 doubles).
template <int NTG, int BAR>
HBS_DEV void tri_inverse32(const double* A, int lda, int j0, int nbp, double* out, double* scratch, int wb) {
  const int tid = threadIdx.x - 32 * wb, warp = (tid >> 5), lane = tid & 31;
  auto R = [&](int i, int c) -> double {
    if (i >= nbp || c >= nbp) return i == c ? 1.0 : 0.0;
    return A[(j0 + i) + (j0 + c) * lda];
  };
  for (int e = tid; e < kP * kP; e += NTG) out[e] = 0.0;
  ysync<NTG, BAR>();
  if (warp < 4 && lane < 8) {
    const int base = 8 * warp, c = lane;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      x[i] = x[i] / R(base + i, base + i);
#pragma unroll
      for (int k = 0; k < i; ++k) x[k] = fma(-R(base + k, base + i), x[i], x[k]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) out[(base + i) * kP + base + c] = x[i];
  }
  __threadfence_block();
  ysync<NTG, BAR>();
  for (int w = 8; w < kP; w *= 2) {
    const int npair = kP / (2 * w);
    for (int e = tid; e < npair * w * w; e += NTG) {   // X = B C^-1
      const int pr = e / (w * w), rem = e % (w * w), i = rem / w, c = rem % w;
      const int o1 = 2 * w * pr, o2 = o1 + w;
      double acc = 0.0;
      for (int q = 0; q <= c; ++q) acc = fma(R(o1 + i, o2 + q), out[(o2 + q) * kP + o2 + c], acc);
      scratch[e] = acc;
    }
    __threadfence_block();
    ysync<NTG, BAR>();
    for (int e = tid; e < npair * w * w; e += NTG) {   // -A^-1 X
      const int pr = e / (w * w), rem = e % (w * w), i = rem / w, c = rem % w;
      const int o1 = 2 * w * pr, o2 = o1 + w;
      double acc = 0.0;
      for (int q = i; q < w; ++q) acc = fma(out[(o1 + i) * kP + o1 + q], scratch[pr * w * w + q * w + c], acc);
      out[(o1 + i) * kP + o2 + c] = -acc;
    }
    __threadfence_block();
    ysync<NTG, BAR>();
  }
}

}  // namespace

// Panel factorisation by CholeskyQR + Householder reconstruction (Ballard et
// al.), for the fused kernel's panel group (NTG threads, named barrier 1).
// The panel block P = A(j0:m, j0:j0+32) (rows below the finished R):
//   Gp = P^T P = R^T R (tensor cores; Cholesky, row-owned, one warp),
//   Q1 = P R^{-1} (tensor cores, in place),
//   Q1(0:32, :) - S = L U with s_j = -sign of the current pivot (one warp),
//   L2 = Q1(32:, :) U^{-1} (tensor cores, in place),
//   T = -U S L^{-T}, R_hh = S R.
// In exact arithmetic these are the reflectors (and T, R) the column-by-column
// Householder chain (dlarfg signs) produces -- Householder QR is unique for a
// given sign rule -- so the panel leaves A / T exactly as panel_factor_r +
// form_t would, without a 32-step reduction chain.  Returns false (group-
// uniform) for panels the chain must factor: partial panels, a Cholesky
// breakdown, or min R_ii < 1e-2 max R_ii (the Gram squares the panel's
// condition number; the chain also carries the reference's sigma screen).
template <int NTG>
__device__ __noinline__ bool panel_factor_gram(double* A, int lda, int m, int j0, int nbp, double* G, double* T,
                                               double* scr, int* s_flag) {
  if (nbp != kP) return false;
  const int warp = ltid<NTG>() >> 5, lane = ltid<NTG>() & 31, nw = gthreads<NTG>() >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mp = round_up(m, 8);
  double* sg = scr;   // signs s_j
  // 1. Gp = P^T P (32 x 32, row-major in G): 16 tiles of 8 x 8
  for (int tile = warp; tile < 16; tile += nw) {
    const int fi = tile >> 2, fj = tile & 3;
    const double* ci = A + (j0 + 8 * fi + g) * lda + t;
    const double* cj = A + (j0 + 8 * fj + g) * lda + t;
    double c[4][2] = {};
    for (int k = j0; k < mp; k += 16) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + 4 * u < mp) dmma8x8x4(c[u][0], c[u][1], ci[k + 4 * u], cj[k + 4 * u]);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
      G[(8 * fi + g) * kLdT + 8 * fj + 2 * t + e] = (c[0][e] + c[1][e]) + (c[2][e] + c[3][e]);
  }
  gsync<NTG>();
  // 2. Cholesky (row i in lane i), R into G's upper triangle; R^{-1} into T
  if (warp == 0) {
    double c[kP];
#pragma unroll
    for (int k = 0; k < kP; ++k) c[k] = (k >= lane) ? G[lane * kLdT + k] : 0.0;
    const double gmax = warp_max(G[lane * kLdT + lane]);
    bool ok = gmax > 0.0 && gmax < 1e300;
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      const double d = __shfl_sync(0xffffffffu, c[j], j);
      ok = ok && (d > 1e-4 * gmax);                  // R_jj >= 1e-2 max R_ii (approximately)
      const double rs = rsqrt_nr(d);
      if (lane == j) {
#pragma unroll
        for (int k = 0; k < kP; ++k)
          if (k >= j) c[k] *= rs;
      }
      double rji = 0.0;
#pragma unroll
      for (int k = j + 1; k < kP; ++k) {
        const double rk = __shfl_sync(0xffffffffu, c[k], j);
        if (k == lane) rji = rk;
        if (lane > j && k >= lane) c[k] = fma(-rji, rk, c[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < kP; ++k)
      if (k >= lane) G[lane * kLdT + k] = c[k];
    __syncwarp();
    // row lane of R^{-1}: x R = e_lane
#pragma unroll
    for (int k = 0; k < kP; ++k) c[k] = (k == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < kP; ++k) {
      c[k] *= rcp_nr(G[k * kLdT + k]);
#pragma unroll
      for (int l = k + 1; l < kP; ++l) c[l] = fma(-c[k], G[k * kLdT + l], c[l]);
    }
#pragma unroll
    for (int k = 0; k < kP; ++k) T[lane * kLdT + k] = c[k];
    if (lane == 0) *s_flag = __all_sync(0xffffffffu, ok) ? 1 : 0;
    else __all_sync(0xffffffffu, ok);
  }
  gsync<NTG>();
  if (!*s_flag) return false;
  // 3. Q1 = P R^{-1} in place, 8-row blocks per warp
  for (int r0 = j0 + 8 * warp; r0 < mp; r0 += 8 * nw) {
    double a[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) a[kk] = A[(r0 + g) + (j0 + 4 * kk + t) * lda];
    double acc[4][2] = {};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int f = 0; f < 4; ++f) dmma8x8x4(acc[f][0], acc[f][1], a[kk], T[(4 * kk + t) * kLdT + 8 * f + g]);
    __syncwarp();
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int e = 0; e < 2; ++e) A[(r0 + g) + (j0 + 8 * f + 2 * t + e) * lda] = acc[f][e];
  }
  gsync<NTG>();
  // 4. sign-chosen LU of the top 32 x 32 block (row lane in lane); U^{-1}
  //    into T (R^{-1} is dead); R_hh = S R into A's upper triangle (U is dead
  //    once U^{-1} and the T rows are formed); T = -U S L^{-T} rows into G
  if (warp == 0) {
    double c[kP];
#pragma unroll
    for (int k = 0; k < kP; ++k) c[k] = A[(j0 + lane) + (j0 + k) * lda];
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      double dinv = 0.0;
      if (lane == j) {
        const double sj = c[j] >= 0.0 ? -1.0 : 1.0;
        c[j] -= sj;
        sg[j] = sj;
        dinv = rcp_nr(c[j]);
      }
      dinv = __shfl_sync(0xffffffffu, dinv, j);
      const double l = c[j] * dinv;
      if (lane > j) c[j] = l;
#pragma unroll
      for (int k = j + 1; k < kP; ++k) {
        const double uk = __shfl_sync(0xffffffffu, c[k], j);
        if (lane > j) c[k] = fma(-l, uk, c[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < kP; ++k) A[(j0 + lane) + (j0 + k) * lda] = c[k];
    __syncwarp();
    // column lane of U^{-1}: U z = e_lane, back substitution (c reused)
#pragma unroll
    for (int k = 0; k < kP; ++k) c[k] = (k == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k = kP - 1; k >= 0; --k) {
      c[k] *= rcp_nr(A[(j0 + k) + (j0 + k) * lda]);
#pragma unroll
      for (int q = 0; q < k; ++q) c[q] = fma(-A[(j0 + q) + (j0 + k) * lda], c[k], c[q]);
    }
#pragma unroll
    for (int k = 0; k < kP; ++k) T[k * kLdT + lane] = c[k];
    // T row lane: -(U S) then forward substitution with L (unit lower)
#pragma unroll
    for (int k = 0; k < kP; ++k) c[k] = (k >= lane) ? -A[(j0 + lane) + (j0 + k) * lda] * sg[k] : 0.0;
#pragma unroll
    for (int k = 0; k < kP; ++k)
#pragma unroll
      for (int l = k + 1; l < kP; ++l) c[l] = fma(-c[k], A[(j0 + l) + (j0 + k) * lda], c[l]);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kP; ++k)
      if (k >= lane) A[(j0 + lane) + (j0 + k) * lda] = sg[lane] * G[lane * kLdT + k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kP; ++k) G[lane * kLdT + k] = c[k];
  }
  gsync<NTG>();
  // 5. L2 = Q1(32:, :) U^{-1} in place
  for (int r0 = j0 + kP + 8 * warp; r0 < mp; r0 += 8 * nw) {
    double a[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) a[kk] = A[(r0 + g) + (j0 + 4 * kk + t) * lda];
    double acc[4][2] = {};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int f = 0; f < 4; ++f) dmma8x8x4(acc[f][0], acc[f][1], a[kk], T[(4 * kk + t) * kLdT + 8 * f + g]);
    __syncwarp();
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int e = 0; e < 2; ++e) A[(r0 + g) + (j0 + 8 * f + 2 * t + e) * lda] = acc[f][e];
  }
  gsync<NTG>();
  // 6. T from G
  for (int e = ltid<NTG>(); e < kP * kP; e += gthreads<NTG>()) T[(e / kP) * kLdT + e % kP] = G[(e / kP) * kLdT + e % kP];
  gsync<NTG>();
  return true;
}

// TM: the box's Y rows live in tensor memory for the whole sweep (n_max <=
// 128 rows -> TMEM lanes, s <= 256 fp64 columns), so the Y group's three
// products per panel and the solve read and write Y there instead of
// round-tripping it through L2.
// NF / SF > 0: compile-time box rows and probe count (the launcher runs this
// specialisation for the boxes with exactly NF rows when s == SF, and the
// generic kernel (skip_rows = NF) for the others).
// PRE: the probe factorisation comes from the Gram kernel (gram.cu) in the
// same layout (fac: V below, R_hh on / above the diagonal; T in S.t): group P
// only loads it, and group Y applies it to the TMEM rows and solves.  With a
// Gram flag array, the PRE launch takes the (box, side)s whose flag is 0 and
// the Householder launch those whose flag is set.
template <int MR, bool TM, int NF = 0, int SF = 0, bool PRE = false>
__global__ void __launch_bounds__(512, 1) probe_fused_kernel(FusedArgs args) {
  extern __shared__ double smem[];
  const int side = blockIdx.y;
  const int64_t b = blockIdx.x;
  const FusedSide& S = args.side[side];
  const int nb_rt = box_rows(args.geo, b);
  if (NF ? nb_rt != NF : nb_rt == args.skip_rows) return;   // the other launch owns this box
  if (args.gflag != nullptr && ((args.gflag[(int64_t)side * args.geo.nbox + b] != 0) == PRE)) return;
  const int nb = NF ? NF : nb_rt;
  const int m = SF ? SF : args.s, n = nb, s = SF ? SF : args.s;
  const int lda = SF ? frag_ld_c(round_up_c(SF, 32)) : args.lda;
  const int nmax = NF ? NF : args.n_max;   // (the specialised launch has n_max == NF)
  const int mpad = round_up(m, 32);
  const int npanel = (n + kP - 1) / kP;
  const int64_t rb = args.geo.row_begin[b];
  const int warp = (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;

  double* s_tau = smem;
  double* s_scale = s_tau + nmax;
  double* s_beta = s_scale + nmax;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_beta + nmax);   // 32 step barriers
  uint64_t* s_ready = s_bar + kP;                                          // 16 panel-ready + 1 R-ready
  double* G = smem + round_up(3 * nmax + kP + 35, 2);
  double* Tscr = G + kP * kLdT;
  double* T = Tscr + 384;
  double* A = T + round_up(kP * kLdT, 2);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_ready + 34);
  int* s_pflag = reinterpret_cast<int*>(s_ready + 34) + 1;   // panel_factor_gram verdict

  // load Omega^T (s x n col-major == Omega rows), zero rows m .. mpad-1.
  // Each column is one contiguous Omega row: TMA bulk copies (one per column)
  // completing on an mbarrier when rows are 16-byte aligned, else cp.async.
  const double* src = PRE ? S.fac + (size_t)b * S.fac_stride : S.om + S.om_c_rb * rb;
  uint64_t* s_load = s_ready + 33;
  const bool bulk = ((s & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((lda & 1) == 0) &&
                    ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  if (threadIdx.x < kP + 34) mbar_init(&s_bar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  if (TM && warp == 0) tm_alloc512(s_tmem);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (bulk) {
    if (threadIdx.x == 0) mbar_expect_tx(s_load, (unsigned)(n * m * sizeof(double)));
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x)
      bulk_g2s(&A[j * lda], src + (int64_t)j * s, (unsigned)(m * sizeof(double)), s_load);
    const int zr = mpad - m;
    for (int e = threadIdx.x; e < zr * n; e += blockDim.x) A[m + e % zr + (e / zr) * lda] = 0.0;
    mbar_wait(s_load, 0);
  } else {
    for (int j = 0; j < n; ++j)
      for (int i = threadIdx.x; i < mpad; i += blockDim.x) {
        const bool ok = i < m;
        cp_async8(&A[i + j * lda], ok ? src + (int64_t)j * s + i : src, ok);
      }
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();

  double* tglob = S.t + (size_t)b * S.t_stride;
  double* rglob = S.rinv + (size_t)b * S.rinv_stride;
  if (threadIdx.x == 0) FUSED_MARK(0);
  double* yq = S.yq + (size_t)b * S.yq_stride;
  const int ngroups = (nb + 7) >> 3;
  // blocked back substitution X R^T = Y Q1 for one 8-row group, in place in
  // YQ (columns < n); R from shared memory, inverse diagonal blocks from rglob
  auto solve_rows = [&](int rg) {
    const int row = 8 * rg + g;
    const bool rok = row < nb;
    double* drow = yq + (size_t)row * s;
    for (int blk = npanel - 1; blk >= 0; --blk) {
      const int i0 = blk * kP, c0 = i0 + kP;
      const int kr = n > c0 ? round_up(n - c0, 4) : 0;
      double acc[4][2];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = i0 + 8 * f + 2 * t + e;
          acc[f][e] = (rok && c < n) ? __ldcg(drow + c) : 0.0;
        }
      for (int kc = 0; kc < kr; kc += 32) {
        double av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + kc + 4 * u + t;
          av[u] = (rok && c < n) ? -__ldcg(drow + c) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (kc + 4 * u >= kr) break;
          const int c = c0 + kc + 4 * u + t;
#pragma unroll
          for (int f = 0; f < 4; ++f) {
            const int i = i0 + 8 * f + g;
            const double bv = (i < n && c < n) ? A[i + c * lda] : 0.0;   // R(i, c), upper part
            dmma8x8x4(acc[f][0], acc[f][1], av[u], bv);
          }
        }
      }
      const double* ri = rglob + (size_t)blk * kP * kP;
      double xb[4][2] = {};
#pragma unroll
      for (int kk = 0; kk < kP; kk += 4) {
        const double a = cfrag_to_afrag<4>(acc, kk, lane);
#pragma unroll
        for (int f = 0; f < 4; ++f) dmma8x8x4(xb[f][0], xb[f][1], a, __ldcg(ri + (8 * f + g) * kP + kk + t));
      }
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = i0 + 8 * f + 2 * t + e;
          if (rok && c < n) drow[c] = xb[f][e];
        }
      __syncwarp();
    }
  };
#ifdef HBS_PRE_PAIRS   // experiment: measured slower (the T prologue is exposed), PRE at 8 Y warps is the default
  if constexpr (PRE && TM) {
    if (s <= 192) {
      // ---------------------------------------------------------- PRE, paired
      // The factorisation is final, so all 16 warps apply it: warp pair
      // (pi, pi + 8) owns TMEM rows R0 .. R0+15; warp half h computes the
      // products of its row group (rows R0 + 8h + g) and updates half of the
      // column chunks of Y for both row groups.  The two halves exchange
      // W2 = (Y V_p) T_p through the TMEM columns beyond Y (2s + 128 <= 512).
      const uint32_t tbase = *s_tmem;
      const int pi = warp & 7, half = warp >> 3;
      const int R0 = 32 * (pi & 3) + 16 * (pi >> 2);
      const uint32_t tl = tbase + ((uint32_t)R0 << 16);
      const int rowh[2] = {R0 + g, R0 + 8 + g};
      const bool okh[2] = {R0 + g < nb, R0 + 8 + g < nb};
      const int sig = (g >> 1) + ((g & 1) ? 4 : 0);
      const int spad = round_up(s, 8), scol = round_up(s, 16);
      const int xcol[2] = {192, 224};                 // fp64 exchange columns of the two halves
      const int pbar = 3 + pi;
      auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;\n" ::"r"(pbar) : "memory"); };
      if (half) {
        // panel T (dlarft from V^T V and the Gram kernel's tau) and R's
        // diagonal-block inverses, by the upper half (group barrier 1)
        const int lt = threadIdx.x ^ 256;
        for (int p = 0; p < npanel; ++p) {
          const int j0 = p * kP, nbp = min(kP, n - j0);
          for (int e = lt; e < nbp; e += 256) s_tau[j0 + e] = tglob[(size_t)p * kP * kP + e];
          gsync<256>();
          panel_gram<256>(A, lda, m, j0, nbp, G);
          gsync<256>();
          form_t<256>(T, Tscr, G, s_tau, j0, nbp);
          for (int e = lt; e < kP * kP; e += 256) tglob[(size_t)p * kP * kP + e] = T[(e / kP) * kLdT + e % kP];
          gsync<256>();
          tri_inverse32<256, 1>(A, lda, j0, nbp, rglob + (size_t)p * kP * kP, Tscr, 8);
          gsync<256>();
        }
      } else {
        // Y rows into TMEM (columns s .. zero: the solve's padded blocks)
        const int zcol = min(2 * 96, max(scol, round_up(n, 32) + 16));
        const double* y0 = S.y + S.y_c_rb * rb;
        for (int c0 = 0; c0 < zcol; c0 += 16) {
          double v[4][2];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = c0 + 4 * q + t;
              v[q][h] = (okh[h] && c < s) ? __ldcs(y0 + (size_t)rowh[h] * s + c) : 0.0;
            }
          tm_st16(tl + 2 * c0, v);
        }
        tm_wait_st();
      }
      __threadfence_block();
      tm_fence_before();
      __syncthreads();
      tm_fence_after();
      for (int p = 0; p < npanel; ++p) {
        const int j0 = p * kP, nbp = min(kP, n - j0), kb = j0 & ~7;
        const double* tp = tglob + (size_t)p * kP * kP;
        // GEMM1: W = Y(my rows, kb:) V_p   (8 x 32)
        double w[4][2] = {};
        for (int kc = kb & ~15; kc < spad; kc += 16) {
          double a[4][2];
          tm_ld16(tl + 2 * kc, a);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = kc + 4 * u;
            if (k < kb) continue;
            if (k >= spad) break;
            const double av = half ? a[u][1] : a[u][0];
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              const double bv = (k < j0 + kP) ? vval(A, lda, j0, nbp, k + t, 8 * f + g)
                                              : ((8 * f + g < nbp) ? A[(k + t) + (j0 + 8 * f + g) * lda] : 0.0);
              dmma8x8x4(w[f][0], w[f][1], av, bv);
            }
          }
        }
        // GEMM2: W2 = W T_p
        double w2[4][2] = {};
#pragma unroll
        for (int kk = 0; kk < kP; kk += 4) {
          const double a0 = cfrag_to_afrag<4>(w, kk, lane);
#pragma unroll
          for (int f = 0; f < 4; ++f) dmma8x8x4(w2[f][0], w2[f][1], a0, __ldcg(tp + (kk + t) * kP + 8 * f + g));
        }
        double a3[2][kP / 4];
#pragma unroll
        for (int kk = 0; kk < kP; kk += 4) a3[half][kk / 4] = -cfrag_to_afrag<4>(w2, kk, lane);
        // exchange -W2 (A fragments) with the partner through TMEM
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          double v[4][2];
#pragma unroll
          for (int rep = 0; rep < 4; ++rep) { v[rep][0] = a3[half][4 * q + rep]; v[rep][1] = a3[half][4 * q + rep]; }
          tm_st16(tl + 2 * (xcol[half] + 16 * q), v);
        }
        tm_wait_st();
        tm_fence_before();
        pair_sync();
        tm_fence_after();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          double v[4][2];
          tm_ld16(tl + 2 * (xcol[1 - half] + 16 * q), v);
#pragma unroll
          for (int rep = 0; rep < 4; ++rep) a3[1 - half][4 * q + rep] = half ? v[rep][0] : v[rep][1];
        }
        // GEMM3: Y(:, kb:) -= W2 V_p^T on my half of the 16-column chunks
        int ci = 0;
        for (int nc = kb & ~15; nc < spad; nc += 16, ++ci) {
          if ((ci & 1) != half) continue;
          double cv[4][2];
          tm_ld16(tl + 2 * nc, cv);
#pragma unroll
          for (int hb = 0; hb < 2; ++hb) {
            const int n0 = nc + 8 * hb;
            if (n0 < kb || n0 >= spad) continue;
            const int col = n0 + sig;
#pragma unroll
            for (int kk = 0; kk < kP; kk += 4) {
              const double bv = (n0 < j0 + kP) ? vval(A, lda, j0, nbp, col, kk + t)
                                               : ((kk + t < nbp) ? A[col + (j0 + kk + t) * lda] : 0.0);
              dmma8x8x4(cv[2 * hb][0], cv[2 * hb + 1][0], a3[0][kk / 4], bv);
              dmma8x8x4(cv[2 * hb][1], cv[2 * hb + 1][1], a3[1][kk / 4], bv);
            }
          }
          tm_st16(tl + 2 * nc, cv);
        }
        tm_wait_st();
        tm_fence_before();
        pair_sync();
        tm_fence_after();
      }
      // blocked back substitution X R^T = Y Q1 on the TMEM rows (lower half of each pair)
      if (!half) {
        for (int blk = npanel - 1; blk >= 0; --blk) {
          const int i0 = blk * kP, c0 = i0 + kP;
          const int kr = n > c0 ? round_up(n - c0, 4) : 0;
          double acc[2][4][2];
          {
            double v[4][2];
#pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
              tm_ld16(tl + 2 * (i0 + 16 * hq), v);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                acc[h][2 * hq][0] = v[0][h]; acc[h][2 * hq][1] = v[1][h];
                acc[h][2 * hq + 1][0] = v[2][h]; acc[h][2 * hq + 1][1] = v[3][h];
              }
            }
          }
          for (int kc = 0; kc < kr; kc += 16) {
            double av[4][2];
            tm_ld16(tl + 2 * (c0 + kc), av);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int k = kc + 4 * u;
              if (k >= kr) break;
              const int c = c0 + k + t;
#pragma unroll
              for (int f = 0; f < 4; ++f) {
                const int i = i0 + 8 * f + sig;
                const double bv = (i < n && c < n) ? A[i + c * lda] : 0.0;   // R(i, c)
                dmma8x8x4(acc[0][f][0], acc[0][f][1], -av[u][0], bv);
                dmma8x8x4(acc[1][f][0], acc[1][f][1], -av[u][1], bv);
              }
            }
          }
          const double* ri = rglob + (size_t)blk * kP * kP;
          double xb[2][4][2] = {};
#pragma unroll
          for (int kk = 0; kk < kP; kk += 4) {
            const double a0 = cfrag_to_afrag<4>(acc[0], kk, lane);
            const double a1 = cfrag_to_afrag<4>(acc[1], kk, lane);
            const int kq = (kk & 7) + t;
            const int kact = 8 * (kk >> 3) + (kq >> 1) + ((kq & 1) ? 4 : 0);
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              const double bv = __ldcg(ri + (8 * f + sig) * kP + kact);
              dmma8x8x4(xb[0][f][0], xb[0][f][1], a0, bv);
              dmma8x8x4(xb[1][f][0], xb[1][f][1], a1, bv);
            }
          }
          {
            double v[4][2];
#pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int ff = 0; ff < 2; ++ff) {
                  const int f = 2 * hq + ff;
                  const int cA = i0 + 8 * f + t, cB = cA + 4;
                  v[2 * ff][h] = cA < n ? xb[h][f][0] : acc[h][f][0];
                  v[2 * ff + 1][h] = cB < n ? xb[h][f][1] : acc[h][f][1];
                }
              tm_st16(tl + 2 * (i0 + 16 * hq), v);
            }
          }
          tm_wait_st();
        }
      }
      tm_fence_before();
      pair_sync();
      tm_fence_after();
      // Y Q (X in columns < n, Y P in columns s-r .. s-1) to the workspace, half the chunks each
      {
        int ci = 0;
        for (int c0 = 0; c0 < scol; c0 += 16, ++ci) {
          if ((ci & 1) != half) continue;
          double v[4][2];
          tm_ld16(tl + 2 * c0, v);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = c0 + 4 * q + t;
              if (okh[h] && c < s) yq[(size_t)rowh[h] * s + c] = v[q][h];
            }
        }
      }
      tm_fence_before();
      __syncthreads();
      tm_fence_after();
      if (warp == 0) tm_dealloc512(tbase);
      return;
    }
  }
#endif
  // s_ready[p] (p < 16): panel p factored (P -> Y);  s_ready[16 + p]: far
  // trailing update of panel p done (Y -> P);  s_ready[32]: all panels
  // applied to YQ (Y -> P);  s_ready[33]: operand load (TMA).
  if (warp >= 8) {
    // ------------------------------------------------------------ group P
    // (physical warps 8..15 = logical 0..7: the arbiter favours high warp ids)
    const int lt = threadIdx.x ^ 256;
    if constexpr (PRE) {
      // V and R are final; form each panel's compact-WY T (dlarft) from
      // V^T V and the tau the Gram kernel left in row 0 of the panel's T block
      for (int p = 0; p < npanel; ++p) {
        const int j0 = p * kP, nbp = min(kP, n - j0);
        for (int e = lt; e < nbp; e += 256) s_tau[j0 + e] = tglob[(size_t)p * kP * kP + e];
        gsync<256>();
        panel_gram<256>(A, lda, m, j0, nbp, G);
        gsync<256>();
        form_t<256>(T, Tscr, G, s_tau, j0, nbp);
        for (int e = lt; e < kP * kP; e += 256) tglob[(size_t)p * kP * kP + e] = T[(e / kP) * kLdT + e % kP];
        __threadfence_block();
        gsync<256>();
        if (lt == 0) mbar_arrive(&s_ready[p]);
      }
    }
    int nhh = 0;   // panels factored by the Householder chain so far (barrier parity)
    for (int p = 0; p < (PRE ? 0 : npanel); ++p) {
      const int j0 = p * kP, nbp = min(kP, n - j0);
      if (p >= 2) mbar_wait(&s_ready[16 + p - 2], 0);   // panels <= p-2 applied to my columns by group Y
      if (lt == 0) FUSED_MARK(21 + 2 * p);
      if (p >= 1) {                                      // look-ahead: apply panel p-1 to panel p's columns
        const int jp = j0 - kP;
        block_reflector_apply<256>(A, lda, round_up(m, 8), jp, kP, tglob + (size_t)(p - 1) * kP * kP, true, j0,
                                   j0 + nbp, kP);
        gsync<256>();
      }
      if (lt == 0) FUSED_MARK(22 + 2 * p);
#ifdef HBS_GRAM_PANEL   // experiment (measured slower: the single-warp 32-step factorisations)
      const bool gp = panel_factor_gram<256>(A, lda, m, j0, nbp, G, T, Tscr, s_pflag);
#else
      const bool gp = false;
      (void)s_pflag;
#endif
      if (!gp) {
        // Householder chain; the step barriers complete once per chain-factored panel
        if constexpr (MR <= 6) panel_factor_r<MR, 256>(A, lda, m, j0, nbp, s_tau, s_scale, s_beta, s_bar, (unsigned)(nhh & 1), G);
        else panel_factor_wide<MR, 8, 256>(A, lda, m, j0, nbp, s_tau, s_scale, s_beta, s_bar, (unsigned)(nhh & 1), G);
        ++nhh;
      }
      if (lt == 0) FUSED_MARK(42 + p);
      if (!gp) form_t<256>(T, Tscr, G, s_tau, j0, nbp);
      for (int e = lt; e < kP * kP; e += 256) tglob[(size_t)p * kP * kP + e] = T[(e / kP) * kLdT + e % kP];
      __threadfence_block();
      gsync<256>();
      if (lt == 0) { mbar_arrive(&s_ready[p]); FUSED_MARK(1 + 2 * p); }
    }
    if (!PRE && lt < 32) {  // sigma screen on diag(R) (PRE: the Gram kernel's status)
      double lo = INFINITY, hi = 0.0;
      for (int j = lt; j < n; j += 32) {
        const double d = fabs(A[j + j * lda]);
        lo = fmin(lo, d);
        hi = fmax(hi, d);
      }
      lo = warp_min(lo);
      hi = warp_max(hi);
      if (lt == 0) {
        const bool bad = !(hi > 0.0) || lo < args.tol * hi || !isfinite(hi);
        S.status[b] = bad ? kBoxIllConditioned : kBoxOk;
        FUSED_MARK(20);
      }
    }
    if constexpr (TM) {
      // the solve runs on the TMEM-resident rows (group Y); group P, idle
      // from here on, inverts R's last diagonal block for it while group Y
      // applies the last panel (scratch: Tscr, free after the last form_t)
      const int jl = (npanel - 1) * kP;
      tri_inverse32<256, 1>(A, lda, jl, min(kP, n - jl), rglob + (size_t)(npanel - 1) * kP * kP, Tscr, 8);
      __threadfence_block();
      gsync<256>();
      if (lt == 0) mbar_arrive(&s_ready[32]);
      return;
    }
    // group Y has applied every panel and inverted every diagonal block of R:
    // take row groups lt/32 (mod 16) of the solve
    mbar_wait(&s_ready[32], 0);
    for (int rg = lt >> 5; rg < ngroups; rg += 16) solve_rows(rg);
    return;
  }

  // -------------------------------------------------------------- group Y
  const int yw = warp;   // group Y: physical warps 0..7
  if constexpr (TM) {
    // warp yw owns rows R0 .. R0+15 (TMEM lanes of its quadrant); thread
    // (g, t) holds rows R0 + g and R0 + 8 + g.  C-fragments of an 8-column
    // block n0 are kept column-permuted: position 2t <-> column n0 + t,
    // 2t + 1 <-> n0 + 4 + t, i.e. sigma(j) = j/2 + 4 (j & 1).
    const uint32_t tbase = *s_tmem;
    const int R0 = 32 * (yw & 3) + 16 * (yw >> 2);
    const uint32_t tl = tbase + ((uint32_t)R0 << 16);
    const int rowh[2] = {R0 + g, R0 + 8 + g};
    const bool okh[2] = {R0 + g < nb, R0 + 8 + g < nb};
    const int sig = (g >> 1) + ((g & 1) ? 4 : 0);
    const int spad = round_up(s, 8), scol = round_up(s, 16);
    {
      // columns s .. are zero (the solve's padded blocks multiply them by 0)
      const int zcol = min(256, max(scol, round_up(n, 32) + 16));
      const double* y0 = S.y + S.y_c_rb * rb;
      for (int c0 = 0; c0 < zcol; c0 += 16) {
        double v[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = c0 + 4 * q + t;
            v[q][h] = (okh[h] && c < s) ? __ldcs(y0 + (size_t)rowh[h] * s + c) : 0.0;
          }
        tm_st16(tl + 2 * c0, v);
      }
      tm_wait_st();
    }
    for (int p = 0; p < npanel; ++p) {
      const int j0 = p * kP, nbp = min(kP, n - j0), kb = j0 & ~7;
      mbar_wait(&s_ready[p], 0);
      const double* tp = tglob + (size_t)p * kP * kP;
      if (!PRE && j0 + 2 * kP < n) {
        block_reflector_apply<256>(A, lda, round_up(m, 8), j0, nbp, tp, true, j0 + 2 * kP, n, kP, 8);
        ysync<256, 2>();
        if (yw == 0 && lane == 0) mbar_arrive(&s_ready[16 + p]);
      }
      if (p + 1 < npanel)   // (the last block is inverted by group P)
        tri_inverse32<256, 2>(A, lda, j0, nbp, rglob + (size_t)p * kP * kP, rglob + (size_t)npanel * kP * kP, 0);
      // GEMM1: W = Y(:, kb:) V_p   (16 x 32)
      double w[2][4][2] = {};
      for (int kc = kb & ~15; kc < spad; kc += 16) {
        double a[4][2];
        tm_ld16(tl + 2 * kc, a);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = kc + 4 * u;
          if (k < kb) continue;
          if (k >= spad) break;
#pragma unroll
          for (int f = 0; f < 4; ++f) {
            const double bv = (k < j0 + kP) ? vval(A, lda, j0, nbp, k + t, 8 * f + g)
                                            : ((8 * f + g < nbp) ? A[(k + t) + (j0 + 8 * f + g) * lda] : 0.0);
            dmma8x8x4(w[0][f][0], w[0][f][1], a[u][0], bv);
            dmma8x8x4(w[1][f][0], w[1][f][1], a[u][1], bv);
          }
        }
      }
      // GEMM2: W2 = W T_p
      double w2[2][4][2] = {};
#pragma unroll
      for (int kk = 0; kk < kP; kk += 4) {
        const double a0 = cfrag_to_afrag<4>(w[0], kk, lane);
        const double a1 = cfrag_to_afrag<4>(w[1], kk, lane);
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const double tb = __ldg(tp + (kk + t) * kP + 8 * f + g);
          dmma8x8x4(w2[0][f][0], w2[0][f][1], a0, tb);
          dmma8x8x4(w2[1][f][0], w2[1][f][1], a1, tb);
        }
      }
      double a3[2][kP / 4];
#pragma unroll
      for (int kk = 0; kk < kP; kk += 4) {
        a3[0][kk / 4] = -cfrag_to_afrag<4>(w2[0], kk, lane);
        a3[1][kk / 4] = -cfrag_to_afrag<4>(w2[1], kk, lane);
      }
      // GEMM3: Y(:, kb:) -= W2 V_p^T, two 8-column blocks per TMEM access
      for (int nc = kb & ~15; nc < spad; nc += 16) {
        double cv[4][2];
        tm_ld16(tl + 2 * nc, cv);
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          const int n0 = nc + 8 * hb;
          if (n0 < kb || n0 >= spad) continue;
          const int col = n0 + sig;
#pragma unroll
          for (int kk = 0; kk < kP; kk += 4) {
            const double bv = (n0 < j0 + kP) ? vval(A, lda, j0, nbp, col, kk + t)
                                             : ((kk + t < nbp) ? A[col + (j0 + kk + t) * lda] : 0.0);
            dmma8x8x4(cv[2 * hb][0], cv[2 * hb + 1][0], a3[0][kk / 4], bv);
            dmma8x8x4(cv[2 * hb][1], cv[2 * hb + 1][1], a3[1][kk / 4], bv);
          }
        }
        tm_st16(tl + 2 * nc, cv);
      }
      tm_wait_st();
      if (yw == 0 && lane == 0) FUSED_MARK(30 + p);
    }
    __threadfence_block();
    ysync<256, 2>();   // every diagonal-block inverse of R is in rglob ...
    mbar_wait(&s_ready[32], 0);   // ... including the last one (group P)
    if (yw == 0 && lane == 0) FUSED_MARK(40);
    // blocked back substitution X R^T = Y Q1 on the TMEM rows (columns < n)
    for (int blk = npanel - 1; blk >= 0; --blk) {
      const int i0 = blk * kP, c0 = i0 + kP;
      const int kr = n > c0 ? round_up(n - c0, 4) : 0;
      double acc[2][4][2];
      {
        double v[4][2];
#pragma unroll
        for (int hq = 0; hq < 2; ++hq) {
          tm_ld16(tl + 2 * (i0 + 16 * hq), v);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            acc[h][2 * hq][0] = v[0][h]; acc[h][2 * hq][1] = v[1][h];
            acc[h][2 * hq + 1][0] = v[2][h]; acc[h][2 * hq + 1][1] = v[3][h];
          }
        }
      }
      for (int kc = 0; kc < kr; kc += 16) {
        double av[4][2];
        tm_ld16(tl + 2 * (c0 + kc), av);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = kc + 4 * u;
          if (k >= kr) break;
          const int c = c0 + k + t;
#pragma unroll
          for (int f = 0; f < 4; ++f) {
            const int i = i0 + 8 * f + sig;
            const double bv = (i < n && c < n) ? A[i + c * lda] : 0.0;   // R(i, c)
            dmma8x8x4(acc[0][f][0], acc[0][f][1], -av[u][0], bv);
            dmma8x8x4(acc[1][f][0], acc[1][f][1], -av[u][1], bv);
          }
        }
      }
      const double* ri = rglob + (size_t)blk * kP * kP;
      double xb[2][4][2] = {};
#pragma unroll
      for (int kk = 0; kk < kP; kk += 4) {
        const double a0 = cfrag_to_afrag<4>(acc[0], kk, lane);
        const double a1 = cfrag_to_afrag<4>(acc[1], kk, lane);
        const int kq = (kk & 7) + t;
        const int kact = 8 * (kk >> 3) + (kq >> 1) + ((kq & 1) ? 4 : 0);
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const double bv = __ldcg(ri + (8 * f + sig) * kP + kact);   // R_blk^{-1}(j, k), permuted j and k
          dmma8x8x4(xb[0][f][0], xb[0][f][1], a0, bv);
          dmma8x8x4(xb[1][f][0], xb[1][f][1], a1, bv);
        }
      }
      {
        double v[4][2];
#pragma unroll
        for (int hq = 0; hq < 2; ++hq) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int ff = 0; ff < 2; ++ff) {
              const int f = 2 * hq + ff;
              const int cA = i0 + 8 * f + t, cB = cA + 4;   // columns of positions 2t, 2t+1
              v[2 * ff][h] = cA < n ? xb[h][f][0] : acc[h][f][0];
              v[2 * ff + 1][h] = cB < n ? xb[h][f][1] : acc[h][f][1];
            }
          tm_st16(tl + 2 * (i0 + 16 * hq), v);
        }
      }
      tm_wait_st();
    }
    // Y Q (X in columns < n, Y P in columns s-r .. s-1) back to the workspace
    for (int c0 = 0; c0 < scol; c0 += 16) {
      double v[4][2];
      tm_ld16(tl + 2 * c0, v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = c0 + 4 * q + t;
          if (okh[h] && c < s) yq[(size_t)rowh[h] * s + c] = v[q][h];
        }
    }
    tm_fence_before();
    ysync<256, 2>();
    tm_fence_after();
    if (yw == 0) tm_dealloc512(tbase);
    if (yw == 0 && lane == 0) FUSED_MARK(41);
    return;
  }
#ifdef HBS_TRACE_NOY
  // timing experiment only: keep the far-trailing / ready hand-shakes, skip the Y work
  for (int p = 0; p < npanel; ++p) {
    mbar_wait(&s_ready[p], 0);
    if (p * kP + 2 * kP < n) { ysync<256, 2>(); if (yw == 0 && lane == 0) mbar_arrive(&s_ready[16 + p]); }
  }
  ysync<256, 2>();
  if (yw == 0 && lane == 0) mbar_arrive(&s_ready[32]);
  return;
#endif
  const double* y0 = S.y + S.y_c_rb * rb;
  // 16-byte vector accesses only when every row start is 16-byte aligned
  const bool vec2 = ((s & 1) == 0) && ((reinterpret_cast<uintptr_t>(y0) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(yq) & 15) == 0);
  // (with odd s the pair (col, col+1) may end one past the row: the second
  // element is then neither read nor written)
  auto ld2 = [&](const double* p, bool second) -> double2 {
    if (vec2) return __ldcg(reinterpret_cast<const double2*>(p));
    return make_double2(__ldcg(p), second ? __ldcg(p + 1) : 0.0);
  };
  auto st2 = [&](double* p, double2 v, bool second) {
    if (vec2) *reinterpret_cast<double2*>(p) = v;
    else { p[0] = v.x; if (second) p[1] = v.y; }
  };
  const int spad = round_up(s, 8);
  for (int p = 0; p < npanel; ++p) {
    const int j0 = p * kP, nbp = min(kP, n - j0), kb = j0 & ~7;
    mbar_wait(&s_ready[p], 0);
    const double* tp = tglob + (size_t)p * kP * kP;
    // far trailing update: panel p applied to the columns beyond panel p+1
    if (j0 + 2 * kP < n) {
      block_reflector_apply<256>(A, lda, round_up(m, 8), j0, nbp, tp, true, j0 + 2 * kP, n, kP, 8);
      ysync<256, 2>();
      if (yw == 0 && lane == 0) mbar_arrive(&s_ready[16 + p]);
    }
    // R's diagonal block p is final: its inverse for the solve
    tri_inverse32<256, 2>(A, lda, j0, nbp, rglob + (size_t)p * kP * kP, rglob + (size_t)npanel * kP * kP, 0);
    for (int rg = yw; rg < ngroups; rg += 8) {
      const int row = 8 * rg + g;
      const bool rok = row < nb;
      const double* srow = (p == 0 ? y0 : yq) + (size_t)row * s;
      double* drow = yq + (size_t)row * s;
      // GEMM1: W = Y(:, kb:) V_p   (8 x 32); A-fragment loads issued 32 columns ahead
      double w[4][2] = {};
      for (int kc = kb; kc < spad; kc += 32) {
        double av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int col = kc + 4 * u + t;
          av[u] = (rok && col < s && kc + 4 * u < spad) ? __ldcg(srow + col) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = kc + 4 * u;
          if (k >= spad) break;
          if (k < j0 + kP) {
#pragma unroll
            for (int f = 0; f < 4; ++f) dmma8x8x4(w[f][0], w[f][1], av[u], vval(A, lda, j0, nbp, k + t, 8 * f + g));
          } else {
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              const double bv = (8 * f + g < nbp) ? A[(k + t) + (j0 + 8 * f + g) * lda] : 0.0;
              dmma8x8x4(w[f][0], w[f][1], av[u], bv);
            }
          }
        }
      }
      // GEMM2: W2 = W T_p
      double tb[kP / 4][4];
#pragma unroll
      for (int kk = 0; kk < kP; kk += 4)
#pragma unroll
        for (int f = 0; f < 4; ++f) tb[kk / 4][f] = __ldg(tp + (kk + t) * kP + 8 * f + g);
      double w2[4][2] = {};
#pragma unroll
      for (int kk = 0; kk < kP; kk += 4) {
        const double a = cfrag_to_afrag<4>(w, kk, lane);
#pragma unroll
        for (int f = 0; f < 4; ++f) dmma8x8x4(w2[f][0], w2[f][1], a, tb[kk / 4][f]);
      }
      double a3[kP / 4];
#pragma unroll
      for (int kk = 0; kk < kP; kk += 4) a3[kk / 4] = -cfrag_to_afrag<4>(w2, kk, lane);
      // GEMM3: Y(:, kb:) -= W2 V_p^T  (first panel also copies columns < kb);
      // C-fragment loads issued 4 column blocks ahead
      if (p == 0) {
        for (int c = 2 * t; c < kb; c += 8)
          if (rok) st2(drow + c, ld2(srow + c, c + 1 < kb), c + 1 < kb);
      }
      for (int nc = kb; nc < spad; nc += 32) {
        double2 cv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = nc + 8 * u + 2 * t;
          cv[u] = (rok && col < s) ? ld2(srow + col, col + 1 < s) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int n0 = nc + 8 * u;
          if (n0 >= spad) break;
          if (n0 < j0 + kP) {
#pragma unroll
            for (int kk = 0; kk < kP; kk += 4)
              dmma8x8x4(cv[u].x, cv[u].y, a3[kk / 4], vval(A, lda, j0, nbp, n0 + g, kk + t));
          } else {
#pragma unroll
            for (int kk = 0; kk < kP; kk += 4) {
              const double bv = (kk + t < nbp) ? A[(n0 + g) + (j0 + kk + t) * lda] : 0.0;
              dmma8x8x4(cv[u].x, cv[u].y, a3[kk / 4], bv);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = nc + 8 * u + 2 * t;
          if (rok && col < s && nc + 8 * u < spad) st2(drow + col, cv[u], col + 1 < s);
        }
      }
      __syncwarp();
    }
    if (yw == 0 && lane == 0) FUSED_MARK(30 + p);
  }
  // blocked back substitution, row groups shared with group P (which is idle
  // once its last panel is factored): Y takes rg = 8 + yw (mod 16)
  __threadfence_block();
  ysync<256, 2>();
  if (yw == 0 && lane == 0) { mbar_arrive(&s_ready[32]); FUSED_MARK(40); }
  for (int rg = 8 + yw; rg < ngroups; rg += 16) solve_rows(rg);
  if (yw == 0 && lane == 0) FUSED_MARK(41);
}

bool fused_fits(int s, int n_max) {
  const int lda = frag_ld(round_up(s, 32));
  const size_t d = round_up(3 * n_max + kP + 35, 2) + kP * kLdT + 384 + round_up(kP * kLdT, 2) + (size_t)lda * n_max;
  return n_max <= 16 * kP && d * sizeof(double) <= kMaxSmemBytes;
}

template <int MR, bool TM, int NF = 0, int SF = 0, bool PRE = false>
static int launch_fused_t(FusedArgs& args, int nsides, cudaStream_t stream) {
  args.lda = frag_ld(round_up(args.s, 32));
  const size_t d = round_up(3 * args.n_max + kP + 35, 2) + kP * kLdT + 384 + round_up(kP * kLdT, 2) +
                   (size_t)args.lda * args.n_max;
  const size_t smem = d * sizeof(double);
  cudaFuncSetAttribute(probe_fused_kernel<MR, TM, NF, SF, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)args.geo.nbox, nsides);
  probe_fused_kernel<MR, TM, NF, SF, PRE><<<grid, 512, smem, stream>>>(args);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

// Y rows in TMEM: at most 128 rows (lanes) and 256 fp64 columns per box
static bool fused_tmem_ok(const FusedArgs& args) {
#ifdef HBS_NO_TMEM
  return false;
#else
  return args.n_max <= 128 && round_up(args.s, 16) <= 256;
#endif
}

template <int MR>
static int launch_fused_mr(FusedArgs& args, int nsides, cudaStream_t stream) {
  args.skip_rows = -1;
  if (args.pre) {   // Gram-factored boxes: Y side only (TMEM rows)
    if (!fused_tmem_ok(args)) return kErrUnsupported;
#ifndef HBS_NO_FUSED_SPECIAL
    if constexpr (MR == 6) {
      if (args.s == 192 && args.n_max == 128) {
        const int rc = launch_fused_t<6, true, 128, 192, true>(args, nsides, stream);
        if (rc != kOk) return rc;
        args.skip_rows = 128;
      }
    }
#endif
    return launch_fused_t<MR, true, 0, 0, true>(args, nsides, stream);
  }
#ifndef HBS_NO_FUSED_SPECIAL
  if constexpr (MR == 6) {
    // config-4 shape: boxes of exactly 128 rows with s = 192 run a specialised
    // kernel (compile-time loop bounds); any other boxes of the level follow
    // in the generic kernel
    if (fused_tmem_ok(args) && args.s == 192 && args.n_max == 128) {
      const int rc = launch_fused_t<6, true, 128, 192>(args, nsides, stream);
      if (rc != kOk) return rc;
      args.skip_rows = 128;
    }
  }
#endif
  return fused_tmem_ok(args) ? launch_fused_t<MR, true>(args, nsides, stream)
                             : launch_fused_t<MR, false>(args, nsides, stream);
}

int launch_probe_fused(FusedArgs args, int nsides, cudaStream_t stream) {
  if (!fused_fits(args.s, args.n_max)) return kErrUnsupported;
  switch ((args.s + 31) / 32) {
    case 1: return launch_fused_mr<1>(args, nsides, stream);
    case 2: return launch_fused_mr<2>(args, nsides, stream);
    case 3: return launch_fused_mr<3>(args, nsides, stream);
    case 4: return launch_fused_mr<4>(args, nsides, stream);
    case 5: return launch_fused_mr<5>(args, nsides, stream);
    case 6: return launch_fused_mr<6>(args, nsides, stream);
    case 7: return launch_fused_mr<7>(args, nsides, stream);
    case 8: return launch_fused_mr<8>(args, nsides, stream);
    default: return kErrUnsupported;
  }
}

}  // namespace hbs
