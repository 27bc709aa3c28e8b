// Device-side building blocks of the blocked Householder kernels (hqr.cu) and
// the pipelined fused probe kernel (fused_pipe.cu): dlarfg reflectors, the
// warp-local panel factorisations, the tensor-core block-reflector update,
// compact-WY T, and the 32 x 32 triangular inverse.  Everything here has
// internal linkage (each translation unit gets its own copy).
#pragma once
#include "common.cuh"
#include "kernels.h"
namespace hbs {

#ifdef HBS_TRACE
static __device__ long long g_hqr_trace[256];
static __device__ int g_hqr_trace_mode = 0;   // record only kernels of this mode
#define HQR_MARK(i) do { __syncthreads(); if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && args.mode == g_hqr_trace_mode) g_hqr_trace[i] = clock64(); } while (0)
#define HQR_STEP(i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && j0 == 0) g_hqr_trace[64 + (i)] = clock64(); } while (0)
#define FUSED_MARK(i) do { if (blockIdx.x == 0 && blockIdx.y == 0) g_hqr_trace[128 + (i)] = clock64(); } while (0)
#define STEP_MARK(i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && j0 == 32 && lane == 0) g_hqr_trace[200 + (i)] = clock64(); } while (0)
static __device__ long long g_pf_trace[64];
#ifndef PF_TRACE_J0
#define PF_TRACE_J0 0
#endif
#define PF_MARK(i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && j0 == PF_TRACE_J0 && lane == 0) g_pf_trace[8 * warp + (i)] = clock64(); } while (0)
static __device__ long long g_pf_step[64];
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
#ifdef HBS_GROUPS_BY_SMSP
// (fused_pipe.cu) the two warp groups live on disjoint SM sub-partitions: a
// warp's sub-partition is warp % 4, group P = sub-partitions 0, 1 (logical
// threads 0..255), group Y = sub-partitions 2, 3 (logical threads 256..511).
template <int NTG>
HBS_DEV int ltid() {
  if (NTG != 256) return (int)threadIdx.x;
  const int w = threadIdx.x >> 5;
  return ((((w & 2) ? 8 : 0) + ((w >> 2) << 1) + (w & 1)) << 5) + (threadIdx.x & 31);
}
#else
template <int NTG>
HBS_DEV int ltid() { return NTG == 256 ? (int)(threadIdx.x ^ 256u) : (int)threadIdx.x; }
#endif

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
                            double* s_beta, uint64_t* bar, unsigned parity, double* G, uint64_t* pub = nullptr) {
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
  __threadfence_block();
  gsync<NTG>();
  // every reflector of the panel is in A: the pipelined kernel's group Y starts
  // the look-ahead product on it while T is formed
  if (pub != nullptr && ltid<NTG>() == 0) mbar_arrive(pub);
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
HBS_DEV void tri_inverse32(const double* A, int lda, int j0, int nbp, double* out, double* scratch, int wb,
                           int gtid = -1) {
  // gtid: the caller's index within its group (default: physical warps wb .. wb + NTG/32 - 1)
  const int tid = gtid >= 0 ? gtid : (int)threadIdx.x - 32 * wb, warp = (tid >> 5), lane = tid & 31;
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


}  // namespace hbs
