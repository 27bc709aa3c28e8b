// SMSP-split form of the persistent pipelined probe kernel (see fused_pipe.cu
// for the mathematics, the reference lines and the pipelining): the two warp
// groups live on disjoint SM sub-partitions.
//
// Why: the FP64 pipe is per sub-partition and shared by DFMA and DMMA; a DMMA
// stream from two warps of a sub-partition starves the DFMA chain of any other
// warp on it (tools/micro/fp64_contention.cu).  Group P (the dlarfg reflector
// chain, T, the look-ahead update and R's diagonal-block inverses) therefore
// runs on sub-partitions 0 / 1 (warps with (warp & 2) == 0) and group Y (far
// trailing update, apply-Q on the Y rows, solve) on sub-partitions 2 / 3.
// Tensor memory is reachable per sub-partition only (lanes 32 (warp % 4) ..),
// so group Y keeps box rows 64..127 in TMEM lanes 64..127 (four warps, 16 rows
// each) and streams rows 0..63 through L2 (four warps, two 8-row groups each).
//
// Boxes with 97..128 rows (uneven trees) run here too, zero-padded to 128:
// the missing columns of Omega^T are zero, so their reflectors are identities
// (dlarfg: tau = 0 for a zero column) and leave the real reflectors, R and Y Q
// untouched; the screen skips them, the R-block inverse treats their diagonal
// as 1, and the missing Y rows are zero in TMEM and never written back.
#define HBS_GROUPS_BY_SMSP
#include "hqr_dev.cuh"

namespace hbs {

#ifdef HBS_TRACE
static __device__ long long g_split_trace[96];
#define PIPE_MARK(i) do { if (blockIdx.x == 0 && it >= 1 && it <= 3) g_split_trace[32 * (it - 1) + (i)] = clock64(); } while (0)
#else
#define PIPE_MARK(i) do { } while (0)
#endif

namespace {

HBS_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

constexpr int kNBar = 64;   // 8-byte slots for mbarriers + the TMEM address
constexpr int kXch = 1024;  // look-ahead exchange (4 strips x 32 x 8)

template <int NF, int SF>
constexpr size_t split_smem_doubles() {
  return round_up_c(3 * NF + kNBar, 2) + kP * kLdT + 384 + round_up_c(kP * kLdT, 2) + kXch +
         (size_t)frag_ld_c(round_up_c(SF, 32)) * NF;
}


// Inverse of the 32 x 32 upper-triangular block R(j0:j0+32, j0:j0+32) (in A) by
// one warp, entirely in registers: lane c holds column c of the inverse and
// runs the back substitution x = e_c; for i = 31..0: x_i *= 1 / R_ii, x_k -= R_ki
// x_i (k < i) -- the rinv_blocks_kernel recurrence (hqr.cu); R entries are
// warp-uniform shared-memory reads.  out: 32 x 32 row-major.
__device__ __noinline__ void tri_inverse32_warp(const double* A, int lda, int j0, int nbp, double* out, int lane) {
  // lane i: 1 / R_ii (off the chain); columns >= nbp are zero padding: identity
  const double dinv = lane < nbp ? 1.0 / A[(j0 + lane) + (size_t)(j0 + lane) * lda] : 1.0;
  double x[kP];
#pragma unroll
  for (int i = 0; i < kP; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int i = kP - 1; i >= 0; --i) {
    const double* col = A + j0 + (size_t)(j0 + i) * lda;   // R(:, i) of the block
    x[i] *= __shfl_sync(0xffffffffu, dinv, i);
#pragma unroll
    for (int k = 0; k < i; ++k) x[k] = fma(-col[k], x[i], x[k]);
  }
#pragma unroll
  for (int i = 0; i < kP; ++i) out[i * kP + lane] = x[i];
}

}  // namespace

// PAD = false: boxes of exactly NF rows; PAD = true: boxes of NF-31 .. NF-1 rows (zero-padded).
template <int NF, int SF, bool PAD>
__global__ void __launch_bounds__(512, 1) probe_fused_split_kernel(FusedArgs args, int nsides) {
  static_assert(NF == 128 && SF % 32 == 0 && SF <= 192, "shape");
  extern __shared__ __align__(16) double smem[];
  constexpr int n = NF, m = SF, s = SF;
  constexpr int lda = frag_ld_c(round_up_c(SF, 32));
  constexpr int npanel = NF / kP;
  constexpr int MR = SF / 32;
  const int warp = (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t nbox = args.geo.nbox;
  const int64_t total = nbox * nsides;

  double* s_tau = smem;
  double* s_scale = s_tau + NF;
  double* s_beta = s_scale + NF;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_beta + NF);   // 32 step barriers
  uint64_t* s_ready = s_bar + kP;        // [p] panel p's T is in tglob                          (P -> Y)
  uint64_t* s_far = s_ready + 4;         // [p] panel p applied to the columns beyond panel p+1  (Y -> P)
  uint64_t* s_rinv = s_far + 4;          // R's diagonal-block inverses are in rglob             (P -> Y)
  uint64_t* s_load0 = s_rinv + 1;        // columns 0..31 of the item landed
  uint64_t* s_load1 = s_load0 + 1;       // columns 32..NF-1 landed
  uint64_t* s_ydone = s_load0 + 2;       // group Y no longer reads A of the item
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_load0 + 3);
  constexpr int kBarUsed = kP + 12;
  static_assert(kBarUsed + 1 <= kNBar, "barrier slots");
  double* G = smem + round_up_c(3 * NF + kNBar, 2);
  double* Tscr = G + kP * kLdT;
  double* T = Tscr + 384;
  double* xch = T + round_up_c(kP * kLdT, 2);
  double* A = xch + kXch;

  // items of this CTA: w = blockIdx.x + k gridDim.x whose box has NF rows
  auto next_item = [&](int64_t w) -> int64_t {
    for (w += gridDim.x; w < total; w += gridDim.x)
      if (const int rows = box_rows(args.geo, w % nbox); PAD ? (rows > NF - kP && rows < NF) : rows == NF) break;
    return w;
  };
  int64_t w = (int64_t)blockIdx.x - (int64_t)gridDim.x;
  w = next_item(w);

  if (threadIdx.x < kBarUsed) mbar_init(&s_bar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  if (warp == 2) tm_alloc512(s_tmem);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (w >= total) {
    if (warp == 2) tm_dealloc512(*s_tmem);
    return;
  }

  if ((warp & 2) == 0) {
    // ------------------------------------------------------------ group P (SM sub-partitions 0, 1)
    const int lt = ltid<256>();
    const int lw = lt >> 5;
    // TMA bulk copies, one per Omega row (= column of Omega^T)
    auto load_cols = [&](int64_t item, int c0, int c1, uint64_t* bar) {
      const FusedSide& S = args.side[item / nbox];
      const int64_t bi = item % nbox;
      const double* src = S.om + S.om_c_rb * args.geo.row_begin[bi];
      const int nb = PAD ? box_rows(args.geo, bi) : NF;
      const int ce = c1 < nb ? c1 : nb;              // real columns of the range
      const int z0 = c0 > nb ? c0 : nb;              // pad columns [z0, c1): zero
      for (int e = lt; e < (c1 - z0) * m; e += 256) A[(z0 + e / m) * lda + e % m] = 0.0;
      __threadfence_block();
      gsync<256>();
      if (lt == 0) mbar_expect_tx(bar, (unsigned)((ce - c0) * m * sizeof(double)));
      for (int j = c0 + lt; j < ce; j += 256)
        bulk_g2s(&A[j * lda], src + (int64_t)j * s, (unsigned)(m * sizeof(double)), bar);
    };
    unsigned nhh = 0;   // panels factored so far (step-barrier parity)
    load_cols(w, 0, kP, s_load0);
    load_cols(w, kP, n, s_load1);
    for (int it = 0; w < total; ++it) {
      const unsigned par = it & 1u;
      const int64_t b = w % nbox;
      const FusedSide& S = args.side[w / nbox];
      double* tglob = S.t + (size_t)b * S.t_stride;
      double* rglob = S.rinv + (size_t)b * S.rinv_stride;
      const int nb = PAD ? box_rows(args.geo, b) : NF;
#pragma unroll 1
      for (int p = 0; p < npanel; ++p) {
        const int j0 = p * kP;
        if (p == 0) {
          mbar_wait(s_load0, par);   // (it > 0: issued at the end of the previous item)
          if (lt == 0) PIPE_MARK(0);
        } else {
          if (p == 1) {
            if (it > 0) {
              mbar_wait(s_ydone, par ^ 1u);   // group Y has finished reading R of the previous item
              if (lt == 0) PIPE_MARK(13);
              fence_proxy_async();
              load_cols(w, kP, n, s_load1);
            }
            mbar_wait(s_load1, par);
          } else {
            mbar_wait(&s_far[p - 2], par);    // panels <= p-2 applied to my columns by group Y
          }
          if (lt == 0) PIPE_MARK(2 * p);
          // look-ahead: panel p-1 (T still in shared memory) applied to panel p's
          // columns, strip lw & 3 (8 columns), rows split between warps lw and lw ^ 4
          {
            const int jp = j0 - kP;
            const int strip = lw & 3, half = lw >> 2;
            const int c0 = j0 + 8 * strip;
            const int mid = jp + (((m - jp) / 2 + 15) & ~15);
            const int k0 = half ? mid : jp, k1 = half ? m : mid;
            double* xw = xch + strip * 256;
            double wl[4][2] = {};
            for (int k = k0; k < k1; k += 4) {
              const double bv = A[(k + t) + (c0 + g) * lda];
              if (k < jp + kP) {
#pragma unroll
                for (int f = 0; f < 4; ++f) dmma8x8x4(wl[f][0], wl[f][1], vval(A, lda, jp, kP, k + t, 8 * f + g), bv);
              } else {
#pragma unroll
                for (int f = 0; f < 4; ++f) dmma8x8x4(wl[f][0], wl[f][1], A[(k + t) + (jp + 8 * f + g) * lda], bv);
              }
            }
            if (half) {
#pragma unroll
              for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int e = 0; e < 2; ++e) xw[(2 * f + e) * 32 + lane] = wl[f][e];
            }
            gsync<256>();
            double w2l[4][2] = {};
            if (!half) {
#pragma unroll
              for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int e = 0; e < 2; ++e) wl[f][e] += xw[(2 * f + e) * 32 + lane];   // rows [jp, mid) + rows [mid, m)
#pragma unroll
              for (int kk = 0; kk < kP; kk += 4) {
                const double bv = cfrag_to_bfrag<4>(wl, kk, lane);
#pragma unroll
                for (int f = 0; f < 4; ++f) dmma8x8x4(w2l[f][0], w2l[f][1], T[(kk + t) * kLdT + 8 * f + g], bv);
              }
#pragma unroll
              for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int e = 0; e < 2; ++e) xw[(2 * f + e) * 32 + lane] = w2l[f][e];
            }
            gsync<256>();
            if (half) {
#pragma unroll
              for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int e = 0; e < 2; ++e) w2l[f][e] = xw[(2 * f + e) * 32 + lane];
            }
            double bneg[kP / 4];
#pragma unroll
            for (int kk = 0; kk < kP; kk += 4) bneg[kk / 4] = -cfrag_to_bfrag<4>(w2l, kk, lane);
            const int col0 = c0 + 2 * t;
            for (int ib = k0; ib < k1; ib += 32) {
              double cv[4][2];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = ib + 8 * u + g;
                const bool rok = ib + 8 * u < k1;
                cv[u][0] = rok ? A[i + col0 * lda] : 0.0;
                cv[u][1] = rok ? A[i + (col0 + 1) * lda] : 0.0;
              }
              if (ib < jp + kP) {
#pragma unroll
                for (int kk = 0; kk < kP; kk += 4)
#pragma unroll
                  for (int u = 0; u < 4; ++u)
                    dmma8x8x4(cv[u][0], cv[u][1], vval(A, lda, jp, kP, ib + 8 * u + g, kk + t), bneg[kk / 4]);
              } else {
#pragma unroll
                for (int kk = 0; kk < kP; kk += 4)
#pragma unroll
                  for (int u = 0; u < 4; ++u) {
                    const double av = (ib + 8 * u < k1) ? A[(ib + 8 * u + g) + (jp + kk + t) * lda] : 0.0;
                    dmma8x8x4(cv[u][0], cv[u][1], av, bneg[kk / 4]);
                  }
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = ib + 8 * u + g;
                if (ib + 8 * u < k1) {
                  A[i + col0 * lda] = cv[u][0];
                  A[i + (col0 + 1) * lda] = cv[u][1];
                }
              }
            }
            gsync<256>();
          }
        }
        if (lt == 0) PIPE_MARK(2 * p + 1);
        panel_factor_r<MR, 256>(A, lda, m, j0, kP, s_tau, s_scale, s_beta, s_bar, nhh & 1u, G);
        ++nhh;
        form_t<256>(T, Tscr, G, s_tau, j0, kP);
        for (int e = lt; e < kP * kP; e += 256) tglob[(size_t)p * kP * kP + e] = T[(e / kP) * kLdT + e % kP];
        __threadfence_block();
        gsync<256>();
        if (lt == 0) { mbar_arrive(&s_ready[p]); PIPE_MARK(8 + p); }
      }
      if (lt < 32) {   // sigma screen on diag(R)
        double lo = INFINITY, hi = 0.0;
        for (int j = lt; j < nb; j += 32) {
          const double d = fabs(A[j + j * lda]);
          lo = fmin(lo, d);
          hi = fmax(hi, d);
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        if (lt == 0) {
          const bool bad = !(hi > 0.0) || lo < args.tol * hi || !isfinite(hi);
          S.status[b] = bad ? kBoxIllConditioned : kBoxOk;
        }
      }
      // R's diagonal-block inverses for group Y's solve (it is still applying the last panel)
      if (lw < npanel) tri_inverse32_warp(A, lda, lw * kP, nb - lw * kP, rglob + (size_t)lw * kP * kP, lane);
      __threadfence_block();
      gsync<256>();
      if (lt == 0) { mbar_arrive(s_rinv); PIPE_MARK(12); }
      // next item's panel 0 into the dead columns 0..31: factored under group Y's tail
      w = next_item(w);
      if (w < total) {
        fence_proxy_async();
        load_cols(w, 0, kP, s_load0);
      }
    }
    return;
  }

  // -------------------------------------------------------------- group Y (SM sub-partitions 2, 3)
  const int ly = ltid<256>() - 256;
  const int yw = ly >> 5;                 // logical warp 0..7; sub-partition 2 + (yw & 1)
  const bool tmw = yw < 4;                // TMEM warps: 16 box rows each (64..127); the others stream rows 0..63 through L2
  const uint32_t tbase = *s_tmem;
  const int R0 = 32 * (2 + (yw & 1)) + 16 * ((yw >> 1) & 1);   // TMEM warps: first lane = first box row
  const uint32_t tl = tbase + ((uint32_t)R0 << 16);
  const int sig = (g >> 1) + ((g & 1) ? 4 : 0);
  const int rws[2] = {tmw ? R0 + g : 8 * (yw - 4) + g, tmw ? R0 + 8 + g : 32 + 8 * (yw - 4) + g};
  constexpr int scol = round_up_c(s, 16);
  for (int it = 0; w < total; ++it) {
    const unsigned par = it & 1u;
    const int64_t b = w % nbox;
    const FusedSide& S = args.side[w / nbox];
    const int64_t rb = args.geo.row_begin[b];
    double* tglob = S.t + (size_t)b * S.t_stride;
    double* rglob = S.rinv + (size_t)b * S.rinv_stride;
    double* yq = S.yq + (size_t)b * S.yq_stride;
    const double* y0 = S.y + S.y_c_rb * rb;
    const int nb = PAD ? box_rows(args.geo, b) : NF;
    const bool okh[2] = {!PAD || rws[0] < nb, !PAD || rws[1] < nb};   // (only TMEM rows can be missing: nb > 96)
    if (tmw) {
      for (int c0 = 0; c0 < scol; c0 += 16) {
        double v[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) v[q][h] = okh[h] ? __ldcs(y0 + (size_t)rws[h] * s + c0 + 4 * q + t) : 0.0;
        tm_st16(tl + 2 * c0, v);
      }
      tm_wait_st();
    }
    if (yw == 0 && lane == 0) PIPE_MARK(16);
    for (int p = 0; p < npanel; ++p) {
      const int j0 = p * kP;
      const double* tp = tglob + (size_t)p * kP * kP;
      mbar_wait(&s_ready[p], par);
      if (p == 0) mbar_wait(s_load1, par);
      if (j0 + 2 * kP < n) {   // far trailing update: panel p applied to the columns beyond panel p+1
        block_reflector_apply<256>(A, lda, m, j0, kP, tp, true, j0 + 2 * kP, n, kP, 8);
        __threadfence_block();
        ysync<256, 2>();
        if (yw == 0 && lane == 0) { mbar_arrive(&s_far[p]); PIPE_MARK(24 + p); }
      }
      if (tmw) {
        // GEMM1: W = Y(:, kb:) V_p   (16 x 32)
        double wv[2][4][2] = {};
        for (int kc = j0; kc < s; kc += 16) {
          double a[4][2];
          tm_ld16(tl + 2 * kc, a);
  #pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = kc + 4 * u;
                      #pragma unroll
            for (int f = 0; f < 4; ++f) {
              const double bv = (k < j0 + kP) ? vval(A, lda, j0, kP, k + t, 8 * f + g) : A[(k + t) + (j0 + 8 * f + g) * lda];
              dmma8x8x4(wv[0][f][0], wv[0][f][1], a[u][0], bv);
              dmma8x8x4(wv[1][f][0], wv[1][f][1], a[u][1], bv);
            }
          }
        }
        // GEMM2: W2 = W T_p
        double w2[2][4][2] = {};
  #pragma unroll
        for (int kk = 0; kk < kP; kk += 4) {
          const double a0 = cfrag_to_afrag<4>(wv[0], kk, lane);
          const double a1 = cfrag_to_afrag<4>(wv[1], kk, lane);
  #pragma unroll
          for (int f = 0; f < 4; ++f) {
            const double tb = __ldcg(tp + (kk + t) * kP + 8 * f + g);
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
        for (int nc = j0; nc < s; nc += 16) {
          double cv[4][2];
          tm_ld16(tl + 2 * nc, cv);
  #pragma unroll
          for (int hb = 0; hb < 2; ++hb) {
            const int n0 = nc + 8 * hb;
          
            const int col = n0 + sig;
  #pragma unroll
            for (int kk = 0; kk < kP; kk += 4) {
              const double bv = (n0 < j0 + kP) ? vval(A, lda, j0, kP, col, kk + t) : A[col + (j0 + kk + t) * lda];
              dmma8x8x4(cv[2 * hb][0], cv[2 * hb + 1][0], a3[0][kk / 4], bv);
              dmma8x8x4(cv[2 * hb][1], cv[2 * hb + 1][1], a3[1][kk / 4], bv);
            }
          }
          tm_st16(tl + 2 * nc, cv);
        }
        tm_wait_st();
      } else {
        // GEMM1: W = Y(:, j0:) V_p for my two row groups (2 x 8 x 32); A fragments from L2, 32 columns ahead
        const double* src = p == 0 ? y0 : yq;
        double wv[2][4][2] = {};
        for (int kc = j0; kc < s; kc += 32) {
          double av[2][8];
  #pragma unroll
          for (int h = 0; h < 2; ++h)
  #pragma unroll
            for (int u = 0; u < 8; ++u) av[h][u] = __ldcg(src + (size_t)rws[h] * s + kc + 4 * u + t);
  #pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = kc + 4 * u;
  #pragma unroll
            for (int f = 0; f < 4; ++f) {
              const double bv = (k < j0 + kP) ? vval(A, lda, j0, kP, k + t, 8 * f + g) : A[(k + t) + (j0 + 8 * f + g) * lda];
              dmma8x8x4(wv[0][f][0], wv[0][f][1], av[0][u], bv);
              dmma8x8x4(wv[1][f][0], wv[1][f][1], av[1][u], bv);
            }
          }
        }
        // GEMM2: W2 = W T_p
        double w2[2][4][2] = {};
  #pragma unroll
        for (int kk = 0; kk < kP; kk += 4) {
          const double a0 = cfrag_to_afrag<4>(wv[0], kk, lane);
          const double a1 = cfrag_to_afrag<4>(wv[1], kk, lane);
  #pragma unroll
          for (int f = 0; f < 4; ++f) {
            const double tb = __ldcg(tp + (kk + t) * kP + 8 * f + g);
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
        // GEMM3: Y(:, j0:) -= W2 V_p^T, four 8-column blocks in flight per row group
  #pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double* srow = src + (size_t)rws[h] * s;
          double* drow = yq + (size_t)rws[h] * s;
          for (int nc = j0; nc < s; nc += 32) {
            double2 cv[4];
  #pragma unroll
            for (int u = 0; u < 4; ++u) cv[u] = __ldcg(reinterpret_cast<const double2*>(srow + nc + 8 * u + 2 * t));
  #pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int n0 = nc + 8 * u;
  #pragma unroll
              for (int kk = 0; kk < kP; kk += 4) {
                const double bv = (n0 < j0 + kP) ? vval(A, lda, j0, kP, n0 + g, kk + t) : A[(n0 + g) + (j0 + kk + t) * lda];
                dmma8x8x4(cv[u].x, cv[u].y, a3[h][kk / 4], bv);
              }
            }
  #pragma unroll
            for (int u = 0; u < 4; ++u) *reinterpret_cast<double2*>(drow + nc + 8 * u + 2 * t) = cv[u];
          }
        }
        __syncwarp();
      }
      if (yw == 0 && lane == 0) PIPE_MARK(17 + p);
    }
    __threadfence_block();
    mbar_wait(s_rinv, par);   // every diagonal-block inverse of R is in rglob (group P)
    // blocked back substitution X R^T = Y Q1 (columns < n)
    if (tmw) {
      for (int blk = npanel - 1; blk >= 0; --blk) {
        const int i0 = blk * kP, c0 = i0 + kP;
        const int kr = n > c0 ? n - c0 : 0;
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
            const int c = c0 + kc + 4 * u + t;
  #pragma unroll
            for (int f = 0; f < 4; ++f) {
              const double bv = A[(i0 + 8 * f + sig) + c * lda];   // R(i, c)
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
                v[2 * ff][h] = xb[h][f][0];
                v[2 * ff + 1][h] = xb[h][f][1];
              }
            tm_st16(tl + 2 * (i0 + 16 * hq), v);
          }
        }
        tm_wait_st();
      }
    } else {
  #pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        double* drow = yq + (size_t)rws[h] * s;
        for (int blk = npanel - 1; blk >= 0; --blk) {
          const int i0 = blk * kP, c0 = i0 + kP;
          double acc[4][2];
  #pragma unroll
          for (int f = 0; f < 4; ++f) {
            const double2 d = __ldcg(reinterpret_cast<const double2*>(drow + i0 + 8 * f + 2 * t));
            acc[f][0] = d.x; acc[f][1] = d.y;
          }
          for (int kc = c0; kc < n; kc += 32) {
            double av[8];
  #pragma unroll
            for (int u = 0; u < 8; ++u) av[u] = -__ldcg(drow + kc + 4 * u + t);
  #pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int c = kc + 4 * u + t;
  #pragma unroll
              for (int f = 0; f < 4; ++f) dmma8x8x4(acc[f][0], acc[f][1], av[u], A[(i0 + 8 * f + g) + c * lda]);   // R(i, c)
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
          for (int f = 0; f < 4; ++f) *reinterpret_cast<double2*>(drow + i0 + 8 * f + 2 * t) = make_double2(xb[f][0], xb[f][1]);
          __syncwarp();
        }
      }
    }
    // shared memory of this item is dead for group Y: group P may overwrite it
    fence_proxy_async();
    ysync<256, 2>();
    if (yw == 0 && lane == 0) { mbar_arrive(s_ydone); PIPE_MARK(21); }
    if (tmw) {
      // Y Q (X in columns < n, Y P in columns s-r .. s-1) of the TMEM rows back to the workspace
      for (int c0 = 0; c0 < scol; c0 += 16) {
        double v[4][2];
        tm_ld16(tl + 2 * c0, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (okh[h]) yq[(size_t)rws[h] * s + c0 + 4 * q + t] = v[q][h];
      }
    }
    if (yw == 0 && lane == 0) PIPE_MARK(22);
    w = next_item(w);
  }
  tm_fence_before();
  ysync<256, 2>();
  tm_fence_after();
  if (warp == 2) tm_dealloc512(tbase);
}

// Launch on the 128-row boxes of a config-4 shaped level; same contract as
// launch_probe_fused_pipe (1 = ran, 0 = shape does not apply, < 0 = error).
int launch_probe_fused_split(FusedArgs& args, int nsides, cudaStream_t stream) {
  constexpr int NF = 128, SF = 192;
  if (args.s != SF || args.n_max > NF || args.n_max <= NF - kP || args.pre || args.gflag != nullptr) return 0;
  static const int n_sm = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  const int64_t total = args.geo.nbox * nsides;
  constexpr size_t smem = split_smem_doubles<NF, SF>() * sizeof(double);
  static_assert(smem <= kMaxSmemBytes, "shared memory");
  const unsigned grid = (unsigned)(total < n_sm ? total : n_sm);
  if (args.n_max == NF) {   // the full boxes (every box of a perfect tree)
    cudaFuncSetAttribute(probe_fused_split_kernel<NF, SF, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe_fused_split_kernel<NF, SF, false><<<grid, 512, smem, stream>>>(args, nsides);
    note_launch();
  }
  // boxes of NF-31 .. NF-1 rows (uneven trees; every CTA exits at once when there are none)
  if (!(args.uniform && args.n_max == NF)) {
  cudaFuncSetAttribute(probe_fused_split_kernel<NF, SF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_fused_split_kernel<NF, SF, true><<<grid, 512, smem, stream>>>(args, nsides);
  note_launch();
  }
  args.skip_rows = NF;
  args.skip_rows_lo = NF - kP;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

extern "C" int hbs_debug_split_trace(long long* out) {
#ifdef HBS_TRACE
  return cudaMemcpyFromSymbol(out, g_split_trace, sizeof(long long) * 96) == cudaSuccess ? 0 : 4;
#else
  (void)out;
  return 6;
#endif
}

}  // namespace hbs
