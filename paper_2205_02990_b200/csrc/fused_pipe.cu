// Persistent, software-pipelined form of the fused probe kernel (hqr.cu,
// probe_fused_kernel<6, true, NF, SF>) for levels with many boxes of one
// shape (config 4: 128-row boxes, s = 192).
//
// Same mathematics and per-(box, side) arithmetic as the one-shot kernel
// (reference: nullspace / lstsq_right, linalg.py:52-90, called per node from
// compress_node_bases / compute_discrepancy, compress.py:155-197): group P
// (warps 8..15) factors Omega_tau^T by the dlarfg Householder chain in shared
// memory, group Y (warps 0..7) applies every finished panel to the box's Y rows
// in tensor memory and solves X = (Y Q1) R^{-T}.
//
// What changes is the schedule, which is built around group P's reflector
// chain being the critical resource (measured: ~45k cycles per panel alone,
// ~65-75k next to group Y's tensor-core work, against ~220k of group Y work
// per item):
//  * one CTA per SM walks a strided list of (box, side) items; as soon as
//    group P has published the last panel of item i it loads panel 0 of item
//    i+1 into the shared-memory columns 0..31 (dead since panel 0 of item i
//    was applied) and factors it under group Y's last panel and solve.  The
//    other 96 columns follow by TMA once group Y has finished reading R
//    (s_ydone);
//  * group P runs nothing but the chain and T: the look-ahead update of the
//    next panel's columns is done by group Y (which has the slack), its K
//    range split over warp pairs, starting on the published reflectors
//    (s_pub) while group P still forms T; group Y also inverts every diagonal
//    block of R.
// (This kernel shares every SM sub-partition between the two groups; the
// default since round 2 is its SMSP-split successor, fused_split.cu, which
// launch_probe_fused_pipe dispatches to unless HBS_SPLIT=0.)
// All hand-offs are mbarriers whose phase parity is the item counter.  The
// look-ahead's split K sum (rows [j0, mid) + rows [mid, m), in that order)
// is the one difference in rounding from the one-shot kernel, so every
// 128-row box at s = 192 runs here, whatever the level size: a box's bits do
// not depend on how many boxes share its launch (multi-GPU partitions stay
// bitwise equal to the single-GPU sweep).
#include <cstdlib>
#include "hqr_dev.cuh"

namespace hbs {

#ifdef HBS_TRACE
static __device__ long long g_pipe_trace[96];
#define PIPE_MARK(i) do { if (blockIdx.x == 0 && it >= 1 && it <= 3) g_pipe_trace[32 * (it - 1) + (i)] = clock64(); } while (0)
#else
#define PIPE_MARK(i) do { } while (0)
#endif

namespace {

HBS_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

constexpr int kNBar = 64;   // 8-byte slots for mbarriers + the TMEM address
constexpr int kXch = 1024;  // look-ahead exchange (4 strips x 32 x 8)

template <int NF, int SF>
constexpr size_t pipe_smem_doubles() {
  return round_up_c(3 * NF + kNBar, 2) + kP * kLdT + 384 + round_up_c(kP * kLdT, 2) + kXch +
         (size_t)frag_ld_c(round_up_c(SF, 32)) * NF;
}

}  // namespace

template <int NF, int SF>
__global__ void __launch_bounds__(512, 1) probe_fused_pipe_kernel(FusedArgs args, int nsides) {
  static_assert(NF % kP == 0 && SF % 32 == 0 && SF <= 192 && NF <= 128, "shape");
  extern __shared__ double smem[];
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
  uint64_t* s_ready = s_bar + kP;        // [p] panel p's T is in tglob                  (P -> Y)
  uint64_t* s_pub = s_ready + 4;         // [p] panel p's reflectors are in A            (P -> Y)
  uint64_t* s_la = s_pub + 4;            // [p] panel p applied to panel p+1's columns   (Y -> P)
  uint64_t* s_load0 = s_la + 4;          // columns 0..31 of the item landed
  uint64_t* s_load1 = s_load0 + 1;       // columns 32..NF-1 landed
  uint64_t* s_ydone = s_load0 + 2;       // group Y no longer reads A of the item
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_load0 + 3);
  constexpr int kBarUsed = kP + 15;
  static_assert(kBarUsed + 1 <= kNBar, "barrier slots");
  double* G = smem + round_up_c(3 * NF + kNBar, 2);
  double* Tscr = G + kP * kLdT;
  double* T = Tscr + 384;
  double* xch = T + round_up_c(kP * kLdT, 2);
  double* A = xch + kXch;

  // items of this CTA: w = blockIdx.x + k gridDim.x whose box has NF rows
  auto next_item = [&](int64_t w) -> int64_t {
    for (w += gridDim.x; w < total; w += gridDim.x)
      if (box_rows(args.geo, w % nbox) == NF) break;
    return w;
  };
  int64_t w = (int64_t)blockIdx.x - (int64_t)gridDim.x;
  w = next_item(w);

  if (threadIdx.x < kBarUsed) mbar_init(&s_bar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  if (warp == 0) tm_alloc512(s_tmem);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (w >= total) {
    if (warp == 0) tm_dealloc512(*s_tmem);
    return;
  }

  if (warp >= 8) {
    // ------------------------------------------------------------ group P
    const int lt = threadIdx.x ^ 256;
    // TMA bulk copies, one per Omega row (= column of Omega^T)
    auto load_cols = [&](int64_t item, int c0, int c1, uint64_t* bar) {
      const FusedSide& S = args.side[item / nbox];
      const double* src = S.om + S.om_c_rb * args.geo.row_begin[item % nbox];
      if (lt == 0) mbar_expect_tx(bar, (unsigned)((c1 - c0) * m * sizeof(double)));
      gsync<256>();
      for (int j = c0 + lt; j < c1; j += 256)
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
#pragma unroll 1
      for (int p = 0; p < npanel; ++p) {
        const int j0 = p * kP;
        if (p == 0) {
          mbar_wait(s_load0, par);   // (it > 0: issued at the end of the previous item)
          if (lt == 0) PIPE_MARK(0);
        } else {
          if (p == 1 && it > 0) {
            mbar_wait(s_ydone, par ^ 1u);   // group Y has finished reading R of the previous item
            if (lt == 0) PIPE_MARK(13);
            fence_proxy_async();
            load_cols(w, kP, n, s_load1);
          }
          mbar_wait(&s_la[p - 1], par);   // panels < p applied to my columns by group Y
        }
        if (lt == 0) PIPE_MARK(2 * p + 1);
        panel_factor_r<MR, 256>(A, lda, m, j0, kP, s_tau, s_scale, s_beta, s_bar, nhh & 1u, G, &s_pub[p]);
        ++nhh;
        form_t<256>(T, Tscr, G, s_tau, j0, kP);
        for (int e = lt; e < kP * kP; e += 256) tglob[(size_t)p * kP * kP + e] = T[(e / kP) * kLdT + e % kP];
        __threadfence_block();
        gsync<256>();
        if (lt == 0) { mbar_arrive(&s_ready[p]); PIPE_MARK(8 + p); }
      }
      if (lt < 32) {   // sigma screen on diag(R)
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
        }
      }
      // next item's panel 0 into the dead columns 0..31: factored under group Y's tail
      w = next_item(w);
      if (w < total) {
        fence_proxy_async();
        load_cols(w, 0, kP, s_load0);
      }
    }
    return;
  }

  // -------------------------------------------------------------- group Y
  // warp yw owns rows R0 .. R0+15 (TMEM lanes of its quadrant); thread (g, t)
  // holds rows R0 + g and R0 + 8 + g.  C-fragments of an 8-column block n0 are
  // kept column-permuted: position 2t <-> column n0 + t, 2t + 1 <-> n0 + 4 + t,
  // i.e. sigma(j) = j/2 + 4 (j & 1)  (as in probe_fused_kernel, hqr.cu).
  const int yw = warp;
  const uint32_t tbase = *s_tmem;
  const int R0 = 32 * (yw & 3) + 16 * (yw >> 2);
  const uint32_t tl = tbase + ((uint32_t)R0 << 16);
  const int rowh[2] = {R0 + g, R0 + 8 + g};
  const int sig = (g >> 1) + ((g & 1) ? 4 : 0);
  constexpr int spad = round_up_c(s, 8), scol = round_up_c(s, 16);
  constexpr int zcol = scol > round_up_c(n, 32) + 16 ? scol : round_up_c(n, 32) + 16;
  for (int it = 0; w < total; ++it) {
    const unsigned par = it & 1u;
    const int64_t b = w % nbox;
    const FusedSide& S = args.side[w / nbox];
    const int64_t rb = args.geo.row_begin[b];
    double* tglob = S.t + (size_t)b * S.t_stride;
    double* rglob = S.rinv + (size_t)b * S.rinv_stride;
    double* yq = S.yq + (size_t)b * S.yq_stride;
    {
      const double* y0 = S.y + S.y_c_rb * rb;
      for (int c0 = 0; c0 < zcol; c0 += 16) {
        double v[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = c0 + 4 * q + t;
            v[q][h] = (c < s) ? __ldcs(y0 + (size_t)rowh[h] * s + c) : 0.0;
          }
        tm_st16(tl + 2 * c0, v);
      }
      tm_wait_st();
    }
    if (yw == 0 && lane == 0) PIPE_MARK(16);
    for (int p = 0; p < npanel; ++p) {
      const int j0 = p * kP, kb = j0;
      const double* tp = tglob + (size_t)p * kP * kP;
      if (p + 1 < npanel) {
        // look-ahead: panel p applied to the columns of panel p+1, strip yw & 3
        // (8 columns), rows split between the warps yw and yw ^ 4
        mbar_wait(&s_pub[p], par);
        if (p == 0) mbar_wait(s_load1, par);
        const int strip = yw & 3, half = yw >> 2;
        const int c0 = j0 + kP + 8 * strip;
        const int mid = j0 + (((m - j0) / 2 + 15) & ~15);
        const int k0 = half ? mid : j0, k1 = half ? m : mid;
        double* xw = xch + strip * 256;
        // GEMM1 (partial): W = V^T A_strip over my rows
        double wl[4][2] = {};
        for (int k = k0; k < k1; k += 4) {
          const double bv = A[(k + t) + (c0 + g) * lda];
          if (k < j0 + kP) {
#pragma unroll
            for (int f = 0; f < 4; ++f) dmma8x8x4(wl[f][0], wl[f][1], vval(A, lda, j0, kP, k + t, 8 * f + g), bv);
          } else {
#pragma unroll
            for (int f = 0; f < 4; ++f) dmma8x8x4(wl[f][0], wl[f][1], A[(k + t) + (j0 + 8 * f + g) * lda], bv);
          }
        }
        if (half) {
#pragma unroll
          for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int e = 0; e < 2; ++e) xw[(2 * f + e) * 32 + lane] = wl[f][e];
        }
        mbar_wait(&s_ready[p], par);   // T_p
        ysync<256, 2>();
        double w2l[4][2] = {};
        if (!half) {
#pragma unroll
          for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int e = 0; e < 2; ++e) wl[f][e] += xw[(2 * f + e) * 32 + lane];   // rows [j0, mid) + rows [mid, m)
          // GEMM2: W2 = T^T W (32 x 8)
#pragma unroll
          for (int kk = 0; kk < kP; kk += 4) {
            const double bv = cfrag_to_bfrag<4>(wl, kk, lane);
#pragma unroll
            for (int f = 0; f < 4; ++f) dmma8x8x4(w2l[f][0], w2l[f][1], __ldcg(tp + (kk + t) * kP + 8 * f + g), bv);
          }
#pragma unroll
          for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int e = 0; e < 2; ++e) xw[(2 * f + e) * 32 + lane] = w2l[f][e];
        }
        ysync<256, 2>();
        if (half) {
#pragma unroll
          for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int e = 0; e < 2; ++e) w2l[f][e] = xw[(2 * f + e) * 32 + lane];
        }
        double bneg[kP / 4];
#pragma unroll
        for (int kk = 0; kk < kP; kk += 4) bneg[kk / 4] = -cfrag_to_bfrag<4>(w2l, kk, lane);
        // GEMM3: A_strip -= V W2 on my rows, 8-row blocks, four in flight
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
          if (ib < j0 + kP) {
#pragma unroll
            for (int kk = 0; kk < kP; kk += 4)
#pragma unroll
              for (int u = 0; u < 4; ++u)
                dmma8x8x4(cv[u][0], cv[u][1], vval(A, lda, j0, kP, ib + 8 * u + g, kk + t), bneg[kk / 4]);
          } else {
#pragma unroll
            for (int kk = 0; kk < kP; kk += 4)
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const double av = (ib + 8 * u < k1) ? A[(ib + 8 * u + g) + (j0 + kk + t) * lda] : 0.0;
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
        __threadfence_block();
        ysync<256, 2>();
        if (yw == 0 && lane == 0) { mbar_arrive(&s_la[p]); PIPE_MARK(24 + p); }
      } else {
        mbar_wait(&s_ready[p], par);
      }
      if (j0 + 2 * kP < n) {   // far trailing update: panel p applied to the columns beyond panel p+1
        block_reflector_apply<256>(A, lda, m, j0, kP, tp, true, j0 + 2 * kP, n, kP, 8);
        ysync<256, 2>();
      }
      tri_inverse32<256, 2>(A, lda, j0, kP, rglob + (size_t)p * kP * kP, rglob + (size_t)npanel * kP * kP, 0);
      // GEMM1: W = Y(:, kb:) V_p   (16 x 32)
      double wv[2][4][2] = {};
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
            const double bv = (n0 < j0 + kP) ? vval(A, lda, j0, kP, col, kk + t) : A[col + (j0 + kk + t) * lda];
            dmma8x8x4(cv[2 * hb][0], cv[2 * hb + 1][0], a3[0][kk / 4], bv);
            dmma8x8x4(cv[2 * hb][1], cv[2 * hb + 1][1], a3[1][kk / 4], bv);
          }
        }
        tm_st16(tl + 2 * nc, cv);
      }
      tm_wait_st();
      if (yw == 0 && lane == 0) PIPE_MARK(17 + p);
    }
    __threadfence_block();
    ysync<256, 2>();   // every diagonal-block inverse of R is in rglob
    // blocked back substitution X R^T = Y Q1 on the TMEM rows (columns < n)
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
    // shared memory of this item is dead for group Y: group P may overwrite it
    fence_proxy_async();
    ysync<256, 2>();
    if (yw == 0 && lane == 0) { mbar_arrive(s_ydone); PIPE_MARK(21); }
    // Y Q (X in columns < n, Y P in columns s-r .. s-1) back to the workspace
    for (int c0 = 0; c0 < scol; c0 += 16) {
      double v[4][2];
      tm_ld16(tl + 2 * c0, v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = c0 + 4 * q + t;
          if (c < s) yq[(size_t)rowh[h] * s + c] = v[q][h];
        }
    }
    if (yw == 0 && lane == 0) PIPE_MARK(22);
    w = next_item(w);
  }
  tm_fence_before();
  ysync<256, 2>();
  tm_fence_after();
  if (yw == 0) tm_dealloc512(tbase);
}

// Launches the pipelined kernel on the boxes with exactly 128 rows of a
// config-4 shaped level (s = 192, n_max = 128), whatever the number of boxes.
// Returns 1 when it ran (the caller then skips those boxes), 0 when the shape
// does not apply, < 0 on a launch error.
int launch_probe_fused_pipe(FusedArgs& args, int nsides, cudaStream_t stream) {
  constexpr int NF = 128, SF = 192;
  if (args.s != SF || args.pre || args.gflag != nullptr) return 0;
  // default: the SMSP-split form (fused_split.cu); HBS_SPLIT=0 keeps this kernel
  static const bool use_split = [] { const char* e = std::getenv("HBS_SPLIT"); return !(e && e[0] == '0'); }();
  if (use_split) return launch_probe_fused_split(args, nsides, stream);
  if (args.n_max != NF) return 0;
  static const int n_sm = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  const int64_t total = args.geo.nbox * nsides;
  constexpr size_t smem = pipe_smem_doubles<NF, SF>() * sizeof(double);
  static_assert(smem <= kMaxSmemBytes, "shared memory");
  cudaFuncSetAttribute(probe_fused_pipe_kernel<NF, SF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_fused_pipe_kernel<NF, SF><<<(unsigned)(total < n_sm ? total : n_sm), 512, smem, stream>>>(args, nsides);
  note_launch();
  args.skip_rows = NF;
  args.skip_rows_lo = NF - 1;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

extern "C" int hbs_debug_pipe_trace(long long* out) {
#ifdef HBS_TRACE
  return cudaMemcpyFromSymbol(out, g_pipe_trace, sizeof(long long) * 96) == cudaSuccess ? 0 : 4;
#else
  (void)out;
  return 6;
#endif
}

}  // namespace hbs
