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

#include <cstdlib>
#include "hqr_dev.cuh"

namespace hbs {


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
  if (NF ? nb_rt != NF : (nb_rt > args.skip_rows_lo && nb_rt <= args.skip_rows)) return;   // the other launch owns this box
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

  // load Omega^T (s x n col-major == Omega rows), zero rows m .. mpad-1.
  // Each column is one contiguous Omega row: TMA bulk copies (one per column)
  // completing on an mbarrier when rows are 16-byte aligned, else cp.async.
  const double* src = PRE ? S.fac + (size_t)b * S.fac_stride : S.om + S.om_c_rb * rb;
  uint64_t* s_load = s_ready + 33;
  const bool bulk = ((s & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((lda & 1) == 0) &&
                    ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  if (threadIdx.x < kP + 34) mbar_init(&s_bar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  // TMEM columns of this CTA: the Y rows (2 b32 columns per fp64 column) up to the
  // solve's padded width; small boxes leave room for the other CTAs of the SM
  const uint32_t tcols = TM ? tm_pow2_cols(2 * min(256, max(round_up(s, 16), round_up(n, 32) + 16))) : 0;
  if (TM && warp == 0) tm_alloc(s_tmem, tcols);
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
      // Householder chain; the step barriers complete once per panel
      if constexpr (MR <= 6) panel_factor_r<MR, 256>(A, lda, m, j0, nbp, s_tau, s_scale, s_beta, s_bar, (unsigned)(nhh & 1), G);
      else panel_factor_wide<MR, 8, 256>(A, lda, m, j0, nbp, s_tau, s_scale, s_beta, s_bar, (unsigned)(nhh & 1), G);
      ++nhh;
      if (lt == 0) FUSED_MARK(42 + p);
      form_t<256>(T, Tscr, G, s_tau, j0, nbp);
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
    if (yw == 0) tm_dealloc(tbase, tcols);
    if (yw == 0 && lane == 0) FUSED_MARK(41);
    return;
  }
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
  args.skip_rows_lo = -1;
  if (args.pre) {   // Gram-factored boxes: Y side only (TMEM rows)
    if (!fused_tmem_ok(args)) return kErrUnsupported;
#ifndef HBS_NO_FUSED_SPECIAL
    if constexpr (MR == 6) {
      if (args.s == 192 && args.n_max == 128) {
        const int rc = launch_fused_t<6, true, 128, 192, true>(args, nsides, stream);
        if (rc != kOk) return rc;
        args.skip_rows = 128;
        args.skip_rows_lo = 127;
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
    if (fused_tmem_ok(args) && args.s == 192 && args.n_max > 96 && args.n_max <= 128) {
      // the persistent pipelined kernels (fused_pipe.cu / fused_split.cu; HBS_PIPE=0 keeps the
      // one-shot kernel); they set the row range they covered in args.skip_rows(_lo)
      static const bool use_pipe = [] { const char* e = std::getenv("HBS_PIPE"); return !(e && e[0] == '0'); }();
      const int pr = use_pipe ? launch_probe_fused_pipe(args, nsides, stream) : 0;
      if (pr < 0) return kErrCuda;
      if (pr == 0 && args.n_max == 128) {
        const int rc = launch_fused_t<6, true, 128, 192>(args, nsides, stream);
        if (rc != kOk) return rc;
        args.skip_rows = 128;
        args.skip_rows_lo = 127;
      }
    }
  }
#endif
  // every box has n_max rows and a specialised launch took that shape: the generic launch would find no box
  if (args.uniform && args.n_max > args.skip_rows_lo && args.n_max <= args.skip_rows) return kOk;
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
