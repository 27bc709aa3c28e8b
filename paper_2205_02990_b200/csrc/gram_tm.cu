// The Gram / Householder-reconstruction probe factorisation (gram.cu) with
// the LU operand in tensor memory, sized so two CTAs share an SM and hide
// each other's Cholesky / LU chains.
//
// Same mathematics and outputs as gram_factor_kernel (see gram.cu for the
// derivation and the reference: linalg.py:52-90, compress.py:155-197):
//   G = Omega Omega^T = R^T R (Cholesky, 16 x 16 blocks in shared memory),
//   A = M^T = Omega_1 - R^T S (n x n, TMEM: lane i = box row i) factored as
//   A = U'^T V1^T by a Crout LU with the dlarfg sign rule (s_j = -sign of the
//   current pivot), V2 = Omega_2^T U'^{-1}, T_p = -U'_pp R_pp^{-1} S V1,pp^{-T}.
// Per (box, side): 8 warps, 256 TMEM columns, < 113 KB of shared memory.
// Warp w owns TMEM lanes (box rows) [32 (w % 4) + 16 (w / 4), +16): lane
// block b_w = 2 (w % 4) + w / 4.  TMEM tiles are 16 lanes x 16 fp64 columns
// (tcgen05.ld/st .16x256b.x4): thread (g, t) holds (row g + 8h, column
// c0 + 4 rep + t) -- the DMMA A-fragment layout of k-step rep.  A tile
// updated as a DMMA accumulator uses the column permutation
// sig(g) = g/2 + 4 (g & 1) on the B operand, so the C fragments land back in
// that layout (as in the fused kernel's TMEM path, hqr.cu).
#include "common.cuh"
#include "kernels.h"

namespace hbs {
namespace {

constexpr int kT = 256;       // threads (8 warps)
constexpr int kN = 128;       // max rows per box
constexpr int kCW = 8;        // streamed Omega column chunk
constexpr int kLdCh = 12;     // chunk row stride (== 4 mod 8; 8-byte, two k-steps)
constexpr int kLdP = 116;     // panel staging stride (>= 112, == 4 mod 16)
constexpr int kLdD = 17;      // diagonal-block scratch stride
constexpr int kBk = 256;      // one 16 x 16 block
constexpr double kFbRatio = 1e-3;

#ifdef HBS_TRACE
__device__ long long g_gtm_trace[32];
#define GT_MARK(i) do { __syncthreads(); if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_gtm_trace[i] = clock64(); } while (0)
#else
#define GT_MARK(i) do { } while (0)
#endif

HBS_DEV int bsw(int i, int j) { return i * 16 + (j ^ ((i & 3) << 2)); }
HBS_DEV int bidx(int nb, int bi, int bj) { return bi * nb - bi * (bi - 1) / 2 + (bj - bi); }
struct GR {
  double* p;
  int nb;
  HBS_DEV double* blk(int bi, int bj) const { return p + bidx(nb, bi, bj) * kBk; }
  HBS_DEV double& at(int i, int j) const { return blk(i >> 4, j >> 4)[bsw(i & 15, j & 15)]; }
};

HBS_DEV double rsqrt_t(double a) {
  double sc = 1.0;
  if (a > 1e30) { a *= 0x1p-100; sc = 0x1p-50; }
  if (a < 1e-30 && a > 0.0) { a *= 0x1p100; sc = 0x1p50; }
  double y = static_cast<double>(rsqrtf(static_cast<float>(a)));
  const double ha = 0.5 * a;
  y = y * fma(-ha * y, y, 1.5);
  y = y * fma(-ha * y, y, 1.5);
  return y * sc;
}
HBS_DEV double rcp_t(double a) {
  double sc = 1.0;
  if (fabs(a) > 1e30) { a *= 0x1p-100; sc = 0x1p-100; }
  if (fabs(a) < 1e-30 && a != 0.0) { a *= 0x1p100; sc = 0x1p100; }
  float yf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(static_cast<float>(a)));
  double y = static_cast<double>(yf);
  y = fma(y, fma(-a, y, 1.0), y);
  y = fma(y, fma(-a, y, 1.0), y);
  y = fma(y, fma(-a, y, 1.0), y);
  return y * sc;
}

HBS_DEV void tm_alloc256(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
      static_cast<unsigned>(__cvta_generic_to_shared(slot))));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
HBS_DEV void tm_dealloc256(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(taddr));
}
HBS_DEV uint32_t tmaddr(uint32_t base, int lane0, int col0) { return base + ((uint32_t)lane0 << 16) + 2u * col0; }

// Cholesky of a diagonal block (upper triangle = Schur complement) in place;
// column-owned, row j of R broadcast through `row`; ri[j] = 1 / R_jj.
HBS_DEV bool chol16(double* Bd, double* ri, double* row, double floor_) {
  const int lane = threadIdx.x & 31, kc = lane & 15;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = Bd[bsw(i, kc)];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double d = __shfl_sync(0xffffffffu, c[j], j);
    ok = ok && (d > floor_) && (d < 1e300);
    const double rs = rsqrt_t(d);
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

// Ri = R^{-1} (upper) of a finished diagonal block: lane i < 16 row i.
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

// Sign-chosen LU of the 16 x 16 block D (M orientation: D[i * kLdD + k] =
// M(i, k)), row-owned; Rd: R's diagonal block.  D <- L \ U'; sg[j] = s_j.
HBS_DEV void lu16(double* D, const double* Rd, double* sg) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double c[16], rr[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    c[k] = D[i * kLdD + k];
    rr[k] = (k >= i) ? Rd[bsw(i, k)] : 0.0;
  }
#pragma unroll 16
  for (int j = 0; j < 16; ++j) {
    const double sj = c[j] >= 0.0 ? -1.0 : 1.0;
    const double sm = (i == j) ? -sj : 0.0;
#pragma unroll
    for (int k = j; k < 16; ++k) c[k] = fma(sm, rr[k], c[k]);
    if (lane == j) sg[j] = sj;
    const double dinv = __shfl_sync(0xffffffffu, rcp_t(c[j]), j);
    const double l = (i > j) ? c[j] * dinv : 0.0;
    if (i > j) c[j] = l;
#pragma unroll
    for (int k = j + 1; k < 16; ++k) {
      const double uk = __shfl_sync(0xffffffffu, c[k], j);
      c[k] = fma(-l, uk, c[k]);
    }
  }
  __syncwarp();
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) D[i * kLdD + k] = c[k];
  }
  __syncwarp();
}

// Li = L^{-1} (unit lower) from D: lane i < 16 column i.
HBS_DEV void linv16(const double* D, double* Li) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double z[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) z[m] = (m == i) ? 1.0 : 0.0;
#pragma unroll
  for (int m = 0; m < 16; ++m)
#pragma unroll
    for (int q = m + 1; q < 16; ++q) z[q] = (m >= i) ? fma(-D[q * kLdD + m], z[m], z[q]) : z[q];
  if (lane < 16) {
#pragma unroll
    for (int m = 0; m < 16; ++m) Li[bsw(m, i)] = z[m];
  }
}

// Ui = U'^{-1} (upper) from D: lane i < 16 column i.
HBS_DEV void uinv16(const double* D, double* Ui) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double z[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) z[m] = (m == i) ? 1.0 : 0.0;
#pragma unroll
  for (int m = 15; m >= 0; --m) {
    const double zm = (m <= i) ? z[m] * rcp_t(D[m * kLdD + m]) : 0.0;
    z[m] = zm;
#pragma unroll
    for (int q = 0; q < m; ++q) z[q] = fma(-D[q * kLdD + m], zm, z[q]);
  }
  if (lane < 16) {
#pragma unroll
    for (int m = 0; m < 16; ++m) Ui[bsw(m, i)] = z[m];
  }
}

HBS_DEV void named_sync(int id, int nthreads) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory"); }

}  // namespace

__global__ void __launch_bounds__(kT, 2) gram_factor_tm_kernel(GramArgs args) {
  extern __shared__ __align__(16) double smem[];
  const int side = blockIdx.y;
  const int64_t b = blockIdx.x;
  const GramSide& S = args.side[side];
  const int n = box_rows(args.geo, b);
  const int s = args.s, r = args.r;
  int32_t* myflag = args.flag + (int64_t)side * args.geo.nbox + b;
  if ((n & 15) || n > kN || n < 16 || s - n != r || s > 256 || r > 64) {
    if (threadIdx.x == 0) *myflag = 1;
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nb = n >> 4;
  const int sig = (g >> 1) + ((g & 1) ? 4 : 0);
  const int myb = 2 * (warp & 3) + (warp >> 2);      // my TMEM lane block (rows 16 myb ..)
  double* Gb = smem;                                  // 36 G / R blocks        9216
  double* Ch = Gb + 36 * kBk;                         // chunk | panel staging  1856
  double* Uinv = Ch + 16 * kLdP;                      // U' diagonal-block inverses (8)
  double* Rinv = Uinv + 8 * kBk;                      // current R_oo^{-1}
  double* Linv = Rinv + kBk;                          // current L_oo^{-1}
  double* D16 = Linv + kBk;                           // 16 x 17 diagonal scratch (+ row buffer)
  double* sg = D16 + 16 * kLdD + 16;                  // signs s_j
  double* rinvd = sg + kN;                            // 1 / R_jj
  int* s_ok = reinterpret_cast<int*>(rinvd + kN);
  uint32_t* s_tm = reinterpret_cast<uint32_t*>(s_ok + 2);
  const GR Gm{Gb, nb};
  const double* om = S.om + S.om_c_rb * args.geo.row_begin[b];
  double* fac = S.fac + (size_t)b * S.fac_stride;

  if (warp == 0) tm_alloc256(s_tm);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tb = *s_tm;
  GT_MARK(0);

  // ------------------------------------------------------------- G = Omega Omega^T
  // 16 x 16 units (bi <= bj) accumulate in registers, five per warp at most,
  // over 8-column chunks of Omega staged in shared memory; the chunks with
  // columns < n also go to TMEM as A = Omega_1 (lane i = row i).
  {
    const int nunits = nb * (nb + 1) / 2;
    double acc[5][2][2][2];
#pragma unroll
    for (int q = 0; q < 5; ++q)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 2; ++c) { acc[q][a][c][0] = 0.0; acc[q][a][c][1] = 0.0; }
    int ubi[5], ubj[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      int bi = 0, rem = warp + 8 * q;
      if (rem >= nunits) rem = 0;
      while (rem >= nb - bi) { rem -= nb - bi; ++bi; }
      ubi[q] = bi; ubj[q] = bi + rem;
    }
    const int nch = (s + kCW - 1) / kCW;
    for (int c = 0; c < nch; ++c) {
      __syncthreads();   // previous chunk consumed
      for (int e = threadIdx.x; e < n * kCW; e += kT) {
        const int i = e >> 3, k = e & 7, col = c * kCW + k;
        const bool ok = col < s;
        cp_async8(&Ch[i * kLdCh + k], om + (int64_t)i * s + (ok ? col : 0), ok);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        if (warp + 8 * q < nunits) {
          const double* ra = Ch + (16 * ubi[q] + g) * kLdCh + t;
          const double* rb = Ch + (16 * ubj[q] + g) * kLdCh + t;
#pragma unroll
          for (int k = 0; k < kCW; k += 4) {
            const double a0 = ra[k], a1 = ra[8 * kLdCh + k], b0 = rb[k], b1 = rb[8 * kLdCh + k];
            dmma8x8x4(acc[q][0][0][0], acc[q][0][0][1], a0, b0);
            dmma8x8x4(acc[q][0][1][0], acc[q][0][1][1], a0, b1);
            dmma8x8x4(acc[q][1][0][0], acc[q][1][0][1], a1, b0);
            dmma8x8x4(acc[q][1][1][0], acc[q][1][1][1], a1, b1);
          }
        }
      }
      // columns < n: Omega_1 -> TMEM (my lane block, 8 columns = two 4-column reps)
      if (c * kCW < n && 16 * myb < n) {
        // tm_ld16 covers 16 columns; write the 8-column chunk as half a tile:
        // load the tile, replace reps 2 (c & 1) .. +1, store back.
        const int c0 = (c * kCW) & ~15, rep0 = ((c * kCW) & 15) >> 2;
        double v[4][2];
        tm_ld16(tmaddr(tb, 16 * myb, c0), v);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double x = Ch[(16 * myb + g + 8 * h) * kLdCh + 4 * rr + t];
            if (rep0 == 0) v[rr][h] = x;      // (compile-time indices keep v in registers)
            else v[2 + rr][h] = x;
          }
        tm_st16(tmaddr(tb, 16 * myb, c0), v);
        tm_wait_st();
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      if (warp + 8 * q < nunits) {
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
  }

  GT_MARK(1);
  // ------------------------------------------------------------- Cholesky + Crout LU, pipelined
  double gmax = 0.0;
  for (int j = lane; j < n; j += 32) gmax = fmax(gmax, Gm.at(j, j));
  gmax = warp_max(gmax);
  const double floor_ = 1e-24 * gmax;
  double ua[4][2];     // U'12^T of my lane block (A fragments of the trailing update), k-steps 0..3
  for (int it = 0; it <= nb; ++it) {
    const int oc = it, ol = it - 1, kl = 16 * ol;
    const int wd = (ol >= 0) ? ((ol & 1) ? 4 + (ol >> 1) : (ol >> 1)) : -1;   // owner warp of lane block ol
    const int wc = (wd == 7) ? 6 : 7;                                        // Cholesky warp
    const int wr = (wd == 5) ? 4 : 5;                                        // R^{-1} warp
    const int wu = (wd == 3) ? 2 : 3;                                        // U'^{-1} warp
    // (A) diagonal blocks
    if (oc < nb && (warp == wc || warp == wr)) {
      if (warp == wc) {
        const bool ok = chol16(Gm.blk(oc, oc), rinvd + 16 * oc, D16 + 16 * kLdD, floor_);
        if (lane == 0) *s_ok = ok;
      }
      named_sync(1, 64);
      if (warp == wr) rinv16(Gm.blk(oc, oc), rinvd + 16 * oc, Rinv);
    } else if (ol >= 0 && (warp == wd || warp == wu)) {
      if (warp == wd) {
        // TMEM diagonal tile (A orientation) -> D16 (M orientation), LU, back
        double v[4][2];
        tm_ld16(tmaddr(tb, kl, kl), v);
#pragma unroll
        for (int rep = 0; rep < 4; ++rep)
#pragma unroll
          for (int h = 0; h < 2; ++h) D16[(4 * rep + t) * kLdD + g + 8 * h] = v[rep][h];
        __syncwarp();
        lu16(D16, Gm.blk(ol, ol), sg + kl);
        // back to TMEM as A = M^T; V1 (strictly lower part of M) -> fac
#pragma unroll
        for (int rep = 0; rep < 4; ++rep)
#pragma unroll
          for (int h = 0; h < 2; ++h) v[rep][h] = D16[(4 * rep + t) * kLdD + g + 8 * h];
        tm_st16(tmaddr(tb, kl, kl), v);
        tm_wait_st();
        if (lane < 16) {
          for (int i = lane + 1; i < 16; ++i) fac[(size_t)(kl + lane) * s + kl + i] = D16[i * kLdD + lane];
          // tau_j = T_jj = -U'_jj s_j / R_jj, into row 0 of panel (kl + lane) / 32's T block
          // (the PRE kernel forms T itself from V and tau, dlarft)
          const int j = kl + lane;
          S.t[(size_t)b * S.t_stride + (size_t)(j >> 5) * kNB * kNB + (j & 31)] =
              -D16[lane * kLdD + lane] * sg[j] * rinvd[j];
        }
      }
      named_sync(2, 64);
      if (warp == wd) linv16(D16, Linv);
      if (warp == wu) uinv16(D16, Uinv + ol * kBk);
    }
    __syncthreads();
    if (it == 3) GT_MARK(3);
    if (!*s_ok) {
      if (warp == 0) tm_dealloc256(tb);
      if (threadIdx.x == 0) *myflag = 1;
      return;
    }
    // (B) Cholesky block row oc (units of 16 x 8, any warp); LU panel 1
    // (owner warps of lane blocks > ol: U'12^T = (A' - S R rows) V1^{-T}
    // in TMEM, fragments kept); LU panel 2 staging (owner of ol: rows ol of
    // A, columns > block, into Ch)
    const int nbc = oc < nb ? nb - oc - 1 : 0;
    for (int u = warp; u < 2 * nbc; u += kT / 32) {
      const int cb = oc + 1 + (u >> 1), fj = u & 1;
      double* bc = Gm.blk(oc, cb);
      double a2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int k = 0; k < 16; k += 4) {
        const double bv = bc[bsw(k + t, 8 * fj + g)];
#pragma unroll
        for (int fi = 0; fi < 2; ++fi) dmma8x8x4(a2[fi][0], a2[fi][1], Rinv[bsw(k + t, 8 * fi + g)], bv);
      }
      __syncwarp();
#pragma unroll
      for (int fi = 0; fi < 2; ++fi)
#pragma unroll
        for (int e = 0; e < 2; ++e) bc[bsw(8 * fi + g, 8 * fj + 2 * t + e)] = a2[fi][e];
    }
    if (ol >= 0) {
      if (myb > ol && myb < nb) {
        double v[4][2];
        tm_ld16(tmaddr(tb, 16 * myb, kl), v);
        // sign modification: A(j, kl + k) -= s_k R(kl + k, j)
#pragma unroll
        for (int rep = 0; rep < 4; ++rep)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            v[rep][h] = fma(-sg[kl + 4 * rep + t], Gm.at(kl + 4 * rep + t, 16 * myb + g + 8 * h), v[rep][h]);
        double c[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) { c[q][0] = 0.0; c[q][1] = 0.0; }
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          const int col = 8 * hb + sig;
#pragma unroll
          for (int rep = 0; rep < 4; ++rep) {
            const double bv = Linv[bsw(col, 4 * rep + t)];     // V1^{-T}(m, col) = L^{-1}(col, m)
            dmma8x8x4(c[2 * hb][0], c[2 * hb + 1][0], v[rep][0], bv);
            dmma8x8x4(c[2 * hb][1], c[2 * hb + 1][1], v[rep][1], bv);
          }
        }
        tm_st16(tmaddr(tb, 16 * myb, kl), c);
        tm_wait_st();
#pragma unroll
        for (int q = 0; q < 4; ++q) { ua[q][0] = c[q][0]; ua[q][1] = c[q][1]; }
      } else if (myb == ol) {
        // rows kl .. kl+15 of A, columns > block -> Ch (16 x m, row = k)
        for (int cb = ol + 1; cb < nb; ++cb) {
          double v[4][2];
          tm_ld16(tmaddr(tb, kl, 16 * cb), v);
#pragma unroll
          for (int rep = 0; rep < 4; ++rep)
#pragma unroll
            for (int h = 0; h < 2; ++h) Ch[(g + 8 * h) * kLdP + 16 * (cb - ol - 1) + 4 * rep + t] = v[rep][h];
        }
      }
    }
    __syncthreads();
    if (it == 3) GT_MARK(4);
    // (B2) LU panel 2: V1,21^T = U'11^{-T} (A rows block, cols > block), in place in
    // Ch (16 x 8 units, any warp); V1 -> fac
    const int nbl = ol >= 0 ? nb - ol - 1 : 0;
    for (int u = warp; u < 2 * nbl; u += kT / 32) {
      const int j0 = 8 * u;
      const double* ui = Uinv + ol * kBk;
      double a2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int k = 0; k < 16; k += 4) {
        const double bv = Ch[(k + t) * kLdP + j0 + g];
#pragma unroll
        for (int fi = 0; fi < 2; ++fi) dmma8x8x4(a2[fi][0], a2[fi][1], ui[bsw(k + t, 8 * fi + g)], bv);
      }
      __syncwarp();
#pragma unroll
      for (int fi = 0; fi < 2; ++fi)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          Ch[(8 * fi + g) * kLdP + j0 + 2 * t + e] = a2[fi][e];
          fac[(size_t)(kl + 8 * fi + g) * s + kl + 16 + j0 + 2 * t + e] = a2[fi][e];
        }
    }
    __syncthreads();
    if (it == 3) GT_MARK(5);
    // (C) Cholesky trailing (16 x 16 units, any warp) and LU trailing (owner
    // warps): A22 -= U'12^T V1,21^T
    const int uc = nbc * (nbc + 1) / 2;
    for (int u = warp; u < uc; u += kT / 32) {
      int q = u, bi = 0;
      while (q >= nbc - bi) { q -= nbc - bi; ++bi; }
      const int bj = bi + q + oc + 1;
      bi += oc + 1;
      const double* ra = Gm.blk(oc, bi);
      const double* rb = Gm.blk(oc, bj);
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
        const double b0 = rb[bsw(k + t, g)], b1 = rb[bsw(k + t, 8 + g)];
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
    }
    if (ol >= 0 && myb > ol && myb < nb) {
      for (int cb = ol + 1; cb < nb; ++cb) {
        double v[4][2];
        tm_ld16(tmaddr(tb, 16 * myb, 16 * cb), v);
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          const int col = 16 * (cb - ol - 1) + 8 * hb + sig;
#pragma unroll
          for (int rep = 0; rep < 4; ++rep) {
            const double bv = Ch[(4 * rep + t) * kLdP + col];
            dmma8x8x4(v[2 * hb][0], v[2 * hb + 1][0], -ua[rep][0], bv);
            dmma8x8x4(v[2 * hb][1], v[2 * hb + 1][1], -ua[rep][1], bv);
          }
        }
        tm_st16(tmaddr(tb, 16 * myb, 16 * cb), v);
      }
      tm_wait_st();
    }
    __syncthreads();
    if (it == 3) GT_MARK(6);
    if (it == 2) GT_MARK(2);
  }
  GT_MARK(7);
  // screen (the Gram squares cond(Omega); route doubtful boxes to Householder)
  if (warp == 0) {
    double lo = INFINITY, hi = 0.0;
    for (int j = lane; j < n; j += 32) { const double d = Gm.at(j, j); lo = fmin(lo, d); hi = fmax(hi, d); }
    lo = warp_min(lo);
    hi = warp_max(hi);
    if (lane == 0) *s_ok = (hi > 0.0) && isfinite(hi) && lo >= kFbRatio * hi;
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (!*s_ok) {
    if (warp == 0) tm_dealloc256(tb);
    if (threadIdx.x == 0) *myflag = 1;
    return;
  }

  // ------------------------------------------------------------- R_hh
  for (int j = warp; j < n; j += kT / 32) {
    double* fr = fac + (size_t)j * s;
    for (int i = lane; i <= j; i += 32) fr[i] = sg[i] * Gm.at(i, j);
  }
  __syncthreads();

  GT_MARK(8);
  // ------------------------------------------------------------- V2 = Omega_2^T U'^{-1}
  // V2^T = U'^{-T} Omega_2 (U'^T: lower part of A in TMEM), right-looking over
  // lane blocks with Omega_2 in shared memory (the G region; R is done):
  //   X_bb = U'_bb^{-T} C_bb (all warps, 8-column units), then the owner
  //   warp of every later block cc: C_cc -= U'^T_{cc,bb} X_bb.
  constexpr int kLdX = 68;
  double* Cm = Gb;                                    // n x kLdX
  for (int e = threadIdx.x; e < n * r; e += kT) {
    const int j = e / r, q = e - j * r;
    Cm[j * kLdX + q] = __ldg(om + (int64_t)j * s + n + q);
  }
  __syncthreads();
  for (int bb = 0; bb < nb; ++bb) {
    const double* ui = Uinv + bb * kBk;
    for (int u = warp; 8 * u < r; u += kT / 32) {
      double x2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int k = 0; k < 16; k += 4) {
        const double bv = Cm[(16 * bb + k + t) * kLdX + 8 * u + g];
#pragma unroll
        for (int fi = 0; fi < 2; ++fi) dmma8x8x4(x2[fi][0], x2[fi][1], ui[bsw(k + t, 8 * fi + g)], bv);
      }
      __syncwarp();
#pragma unroll
      for (int fi = 0; fi < 2; ++fi)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int q = 8 * u + 2 * t + e, row = 16 * bb + 8 * fi + g;
          Cm[row * kLdX + q] = x2[fi][e];
          if (q < r) fac[(size_t)row * s + n + q] = x2[fi][e];
        }
    }
    __syncthreads();
    if (myb > bb && myb < nb) {
      double v[4][2];
      tm_ld16(tmaddr(tb, 16 * myb, 16 * bb), v);
      for (int u = 0; 8 * u < r; ++u) {
        double c[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e) c[h][e] = Cm[(16 * myb + g + 8 * h) * kLdX + 8 * u + 2 * t + e];
#pragma unroll
        for (int rep = 0; rep < 4; ++rep) {
          const double bv = Cm[(16 * bb + 4 * rep + t) * kLdX + 8 * u + g];
          dmma8x8x4(c[0][0], c[0][1], -v[rep][0], bv);
          dmma8x8x4(c[1][0], c[1][1], -v[rep][1], bv);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e) Cm[(16 * myb + g + 8 * h) * kLdX + 8 * u + 2 * t + e] = c[h][e];
      }
    }
    __syncthreads();
  }
  GT_MARK(9);
  if (threadIdx.x == 0) {
    *myflag = 0;
    S.status[b] = kBoxOk;
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (warp == 0) tm_dealloc256(tb);
}

size_t gram_tm_smem_bytes() {
  return ((size_t)36 * kBk + 16 * kLdP + 10 * kBk + 16 * kLdD + 16 + 2 * kN + 8) * sizeof(double);
}

int launch_gram_tm(const GramArgs& args, int nsides, cudaStream_t stream) {
  const size_t smem = gram_tm_smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gram_factor_tm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((unsigned)args.geo.nbox, nsides);
  gram_factor_tm_kernel<<<grid, kT, smem, stream>>>(args);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

extern "C" int hbs_debug_gram_tm_trace(long long* out) {
#ifdef HBS_TRACE
  return cudaMemcpyFromSymbol(out, g_gtm_trace, sizeof(long long) * 32) == cudaSuccess ? 0 : 4;
#else
  (void)out;
  return 6;
#endif
}

}  // namespace hbs
