// Batched Householder QR of small fp64 matrices, one CTA per matrix.
//
// Restates the reference's LAPACK path (numpy.linalg.qr -> dgeqrf/dgeqr2 with
// the dlarfg reflector convention, then dorgqr/dorg2r), which the reference
// uses in `nullspace` (linalg.py:52-62, complete Q of Omega_tau^T) and `col`
// (linalg.py:35-49, reduced Q of Y_tau P).  Same reflectors => the same
// "last r columns" null-space subspace as the reference when nullity > r.
//
// Modes:
//   kFactor: A = Omega_tau^T (s x n_b).  Emits the reflectors as explicit rows
//            (Vt, n_b x s, unit diagonal, zeros above), R (n_b x n_b), tau and
//            the sigma-screen status used for IllConditionedProbeError.
//   kOrtho : A = Y_tau P (n_b x r).  Emits the explicit Q (n_b x r) = U_tau.
//
// The matrix lives in shared memory when it fits (every BASELINE config up to
// config 4), else in a global scratch slab (config 5 sizes) -- same code via
// generic addressing.
#include "common.cuh"
#include "kernels.h"

namespace hbs {

template <int MR>
HBS_DEV void householder_sweep(double* A, int lda, int m, int n, double* s_scale, double* s_tau,
                               double* s_beta, double* s_norm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (warp == 0) {
    double p = 0.0;
    for (int i = 1 + lane; i < m; i += 32) p += A[i] * A[i];
    p = warp_sum(p);
    if (lane == 0) s_norm[0] = p;
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double alpha = A[j + (size_t)j * lda];
    const double xn2 = s_norm[j & 1];
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (xn2 != 0.0) {  // dlarfg: beta = -sign(alpha) * hypot(alpha, ||x||)
      beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    double cj[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) {
      const int i = j + 1 + lane + 32 * k;
      cj[k] = (i < m) ? A[i + (size_t)j * lda] : 0.0;
    }
    // Two columns per pass for independent shuffle reductions.
    for (int c0 = j + 1 + warp; c0 < n; c0 += 2 * nw) {
      const int c1 = c0 + nw;
      const bool has1 = c1 < n;
      double* col0 = A + (size_t)c0 * lda;
      double* col1 = A + (size_t)(has1 ? c1 : c0) * lda;
      double a0[MR], a1[MR];
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int i = j + 1 + lane + 32 * k;
        a0[k] = (i < m) ? col0[i] : 0.0;
        a1[k] = (i < m && has1) ? col1[i] : 0.0;
        p0 = fma(cj[k], a0[k], p0);
        p1 = fma(cj[k], a1[k], p1);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, o);
        p1 += __shfl_xor_sync(0xffffffffu, p1, o);
      }
      const double f0 = tau * (col0[j] + scale * p0);
      const double f1 = tau * (col1[j] + scale * p1);
      const double g0 = f0 * scale, g1 = f1 * scale;
      double q0 = 0.0, q1 = 0.0;
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int i = j + 1 + lane + 32 * k;
        if (i < m) {
          a0[k] = fma(-g0, cj[k], a0[k]);
          col0[i] = a0[k];
          if (has1) {
            a1[k] = fma(-g1, cj[k], a1[k]);
            col1[i] = a1[k];
          }
          if (i >= j + 2) q0 = fma(a0[k], a0[k], q0);
        }
      }
      __syncwarp();
      if (lane == 0) {
        col0[j] -= f0;
        if (has1) col1[j] -= f1;
      }
      if (c0 == j + 1) {
        q0 = warp_sum(q0);
        if (lane == 0) s_norm[(j + 1) & 1] = q0;
      }
    }
    if (threadIdx.x == 0) {
      s_tau[j] = tau;
      s_scale[j] = scale;
      s_beta[j] = beta;
    }
    __syncthreads();
  }
  // Finalise: reflector tails v = x * scale (below the diagonal), R_jj = beta.
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int j = e / m, i = e % m;
    if (i > j) A[i + (size_t)j * lda] *= s_scale[j];
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) A[j + (size_t)j * lda] = s_beta[j];
  __syncthreads();
}

// dorg2r in place: A holds reflectors below the diagonal (finalised); V is a
// copy of those tails (so column j can be overwritten while other warps still
// read v_j).  On exit A(:, 0:n) = H_0 ... H_{n-1} [I; 0].
template <int MR>
HBS_DEV void householder_form_q(double* A, const double* V, int lda, int m, int n, const double* s_tau) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = n - 1; j >= 0; --j) {
    const double tau = s_tau[j];
    double vj[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) {
      const int i = j + lane + 32 * k;
      vj[k] = (i < m) ? (i == j ? 1.0 : V[i + (size_t)j * lda]) : 0.0;
    }
    // columns c > j: Q(j:m, c) -= tau v (v^T Q(j:m, c))
    for (int c = j + 1 + warp; c < n; c += nw) {
      double* col = A + (size_t)c * lda;
      double a[MR];
      double p = 0.0;
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int i = j + lane + 32 * k;
        a[k] = (i < m) ? col[i] : 0.0;
        p = fma(vj[k], a[k], p);
      }
      p = warp_sum(p) * tau;
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int i = j + lane + 32 * k;
        if (i < m) col[i] = fma(-p, vj[k], a[k]);
      }
    }
    // column j itself (owned by the last warp so it overlaps the others)
    if (warp == nw - 1) {
      double* col = A + (size_t)j * lda;
      for (int i = lane; i < m; i += 32) {
        double v;
        if (i < j) v = 0.0;
        else if (i == j) v = 1.0 - tau;
        else v = -tau * V[i + (size_t)j * lda];
        col[i] = v;
      }
    }
    __syncthreads();
  }
}

template <int MR>
__global__ void __launch_bounds__(512) geqrf_kernel(GeqrfArgs args) {
  extern __shared__ double smem[];
  const int side = blockIdx.y;
  const int64_t b = blockIdx.x;
  const GeqrfSide& S = args.side[side];
  const int nb = box_rows(args.geo, b);
  const int m = args.m_is_rows ? nb : args.m_fixed;
  const int n = args.n_is_rows ? nb : args.n_fixed;
  const int lda = m | 1;  // odd: row-wise traversals stay bank-conflict free
  const int64_t rb = args.geo.row_begin[b];

  double* small = smem;  // scale[nmax], tau[nmax], beta[nmax], norm[2]
  double* s_scale = small;
  double* s_tau = small + args.n_max;
  double* s_beta = small + 2 * args.n_max;
  double* s_norm = small + 3 * args.n_max;
  const int small_len = round_up(3 * args.n_max + 2, 2);
  double* A;
  double* V = nullptr;
  if (args.use_smem) {
    A = smem + small_len;
    V = A + (size_t)args.lda_max * args.n_max;
  } else {
    A = args.gscratch + ((size_t)side * args.geo.nbox + b) * (size_t)args.lda_max * args.n_max * 2;
    V = A + (size_t)args.lda_max * args.n_max;
  }

  // Load A(i, j) = src[off + i*rs + j*cs].
  const double* src = S.src + S.src_c_rb * rb + S.src_c_b * b;
  if (S.src_rs == 1) {
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
      const int j = e / m, i = e % m;
      A[i + (size_t)j * lda] = src[(int64_t)i + (int64_t)j * S.src_cs];
    }
  } else {
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
      const int i = e / n, j = e % n;
      A[i + (size_t)j * lda] = src[(int64_t)i * S.src_rs + (int64_t)j * S.src_cs];
    }
  }
  __syncthreads();

  householder_sweep<MR>(A, lda, m, n, s_scale, s_tau, s_beta, s_norm);

  if (args.mode == kGeqrfFactor) {
    // sigma screen on diag(R): sigma_min/sigma_max <= min|R_ii| / max|R_ii|
    if (threadIdx.x < 32) {
      double lo = INFINITY, hi = 0.0;
      for (int j = threadIdx.x; j < n; j += 32) {
        const double d = fabs(A[j + (size_t)j * lda]);
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
      double v = (i < j) ? 0.0 : (i == j ? 1.0 : A[i + (size_t)j * lda]);
      vt[(size_t)j * S.ldvt + i] = v;
    }
    double* R = S.r + (size_t)b * S.r_stride;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, c = e % n;
      R[(size_t)i * S.ldr + c] = (i <= c) ? A[i + (size_t)c * lda] : 0.0;
    }
    double* tau = S.tau + (size_t)b * S.tau_stride;
    for (int j = threadIdx.x; j < n; j += blockDim.x) tau[j] = s_tau[j];
  } else {
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
      const int j = e / m, i = e % m;
      V[i + (size_t)j * lda] = A[i + (size_t)j * lda];
    }
    __syncthreads();
    householder_form_q<MR>(A, V, lda, m, n, s_tau);
    double* q = S.q + S.q_c_rb * rb + S.q_c_b * b;
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
      const int i = e / n, j = e % n;
      q[(size_t)i * S.ldq + j] = A[i + (size_t)j * lda];
    }
  }
}

size_t geqrf_smem_bytes(int m_max, int n_max, int mode) {
  const int lda = m_max | 1;
  const size_t small_len = round_up(3 * n_max + 2, 2);
  const size_t mats = (mode == kGeqrfFactor ? 1 : 2) * (size_t)lda * n_max;
  return (small_len + mats) * sizeof(double);
}

size_t geqrf_scratch_doubles(int m_max, int n_max, int64_t nbox) {
  return 2 * (size_t)nbox * (size_t)(m_max | 1) * n_max * 2;
}

int launch_geqrf(GeqrfArgs args, int nsides, cudaStream_t stream) {
  args.lda_max = args.m_max | 1;
  const size_t full = geqrf_smem_bytes(args.m_max, args.n_max, args.mode);
  args.use_smem = full <= kMaxSmemBytes;
  if (!args.use_smem && args.gscratch == nullptr) return kErrWorkspace;
  const size_t smem = args.use_smem ? full : round_up(3 * args.n_max + 2, 2) * sizeof(double);
  const int mr = (args.m_max + 31) / 32;
  const int threads = args.n_max >= 96 ? 512 : (args.n_max >= 48 ? 256 : 128);
  dim3 grid((unsigned)args.geo.nbox, nsides);
#define HBS_GEQRF_CASE(R)                                                                        \
  case R:                                                                                        \
    if (smem > 48 * 1024)                                                                        \
      cudaFuncSetAttribute(geqrf_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    geqrf_kernel<R><<<grid, threads, smem, stream>>>(args);                                      \
    break;
  switch (mr) {
    HBS_GEQRF_CASE(1)
    HBS_GEQRF_CASE(2)
    HBS_GEQRF_CASE(3)
    HBS_GEQRF_CASE(4)
    HBS_GEQRF_CASE(5)
    HBS_GEQRF_CASE(6)
    HBS_GEQRF_CASE(7)
    HBS_GEQRF_CASE(8)
    HBS_GEQRF_CASE(10)
    HBS_GEQRF_CASE(12)
    HBS_GEQRF_CASE(16)
    default:
      if (mr == 9) { args.m_max = 320; return launch_geqrf(args, nsides, stream); }
      if (mr == 11) { args.m_max = 384; return launch_geqrf(args, nsides, stream); }
      if (mr > 12 && mr < 16) { args.m_max = 512; return launch_geqrf(args, nsides, stream); }
      return kErrUnsupported;
  }
#undef HBS_GEQRF_CASE
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

}  // namespace hbs
