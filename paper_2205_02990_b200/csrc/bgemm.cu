// Batched, variable-size fp64 GEMM on the FP64 tensor cores (DMMA m8n8k4),
// one launch per level-wide product (box b = tile group of blockIdx.x):
//     C_b = alpha * op(A_b) op(B_b) + beta * C0_b
// Operand bases are derived from the level geometry (row starts, packed
// square-block offsets), so the same kernel serves the discrepancy algebra
// (compress.py:192-197), the parent-sample lift (compress.py:209-227) and the
// telescoping apply used by the HBS sampler (factorization.py:89-143).
//
// 64 x 64 CTA tile, 4 warps of 32 x 32 (16 MMAs per 8 fragment loads per
// k-step), BK = 16, double-buffered cp.async with 16-byte copies when every
// operand row start of the box is 16-byte aligned; 96 registers and 41 KB of
// shared memory give 5 CTAs per SM (measured best for the K = 64..192
// per-box products: more resident warps beat deeper pipelines).  Each operand is staged in the
// orientation it has in global memory (contiguous runs stay contiguous), and
// both staging layouts give bank-conflict-free m8n8k4 fragment loads.
#include "common.cuh"
#include "kernels.h"

namespace hbs {

namespace {
#ifndef BGEMM_BK
#define BGEMM_BK 16
#endif
#ifndef BGEMM_NSTAGE
#define BGEMM_NSTAGE 2
#endif
#ifndef BGEMM_MINB
#define BGEMM_MINB 5   // 5 CTAs (20 warps) per SM: these short-K products are latency-bound
#endif
constexpr int BM = 64, BN = 64, BK = BGEMM_BK, NSTAGE = BGEMM_NSTAGE, NT = 128;
constexpr int LDK = BK + 4;   // k-contiguous staging: [row][k]  (== 4 mod 16)
constexpr int LDR = BM + 4;   // row-contiguous staging: [k][row]
constexpr int STAGE = BM * LDK > BK * LDR ? BM * LDK : BK * LDR;   // doubles per operand stage

HBS_DEV int64_t op_off(const BOperand& o, const LevelGeo& g, int64_t b) {
  int64_t off = o.c_b * b;
  if (o.c_rb) off += o.c_rb * g.row_begin[b];
  if (o.c_sq) off += o.c_sq * g.sq_off[b];
  return off;
}

HBS_DEV void cp_async16(double* dst, const double* src, int bytes) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(src), "r"(bytes));
}

// Stage a 64 x 16 (rows x k) operand tile whose global element (i, k) sits at
// p[i * ld + k] (KC = true: k contiguous) or p[k * ld + i] (KC = false).
// KC: smem [i][k] (ld LDK); else smem [k][i] (ld LDR).
template <bool KC>
HBS_DEV void stage_tile(double* s, const double* p, int ld, int i0, int k0, int I, int K, int tid, bool vec) {
  if (vec) {
#pragma unroll
    for (int e = 0; e < (BM * BK / 2) / NT; ++e) {
      const int idx = tid + e * NT;
      int i, k;
      if (KC) { i = idx / (BK / 2); k = 2 * (idx % (BK / 2)); }
      else { k = idx >> 5; i = 2 * (idx & 31); }
      const int gi = i0 + i, gk = k0 + k;
      int bytes;
      const double* src;
      if (KC) {
        bytes = (gi < I && gk < K) ? (gk + 1 < K ? 16 : 8) : 0;
        src = p + (int64_t)gi * ld + gk;
      } else {
        bytes = (gi < I && gk < K) ? (gi + 1 < I ? 16 : 8) : 0;
        src = p + (int64_t)gk * ld + gi;
      }
      cp_async16(KC ? &s[i * LDK + k] : &s[k * LDR + i], bytes ? src : p, bytes);
    }
  } else {
#pragma unroll
    for (int e = 0; e < (BM * BK) / NT; ++e) {
      const int idx = tid + e * NT;
      int i, k;
      if (KC) { i = idx / BK; k = idx % BK; }
      else { k = idx >> 6; i = idx & 63; }
      const int gi = i0 + i, gk = k0 + k;
      const bool ok = gi < I && gk < K;
      const double* src = KC ? p + (int64_t)gi * ld + gk : p + (int64_t)gk * ld + gi;
      cp_async8(KC ? &s[i * LDK + k] : &s[k * LDR + i], ok ? src : p, ok);
    }
  }
}

// Interior tile of an aligned operand: 16-byte copies with no bounds checks.
template <bool KC>
HBS_DEV void stage_tile_full(double* s, const double* p, int ld, int i0, int k0, int tid) {
#pragma unroll
  for (int e = 0; e < (BM * BK / 2) / NT; ++e) {
    const int idx = tid + e * NT;
    int i, k;
    if (KC) { i = idx / (BK / 2); k = 2 * (idx % (BK / 2)); }
    else { k = idx >> 5; i = 2 * (idx & 31); }
    const double* src = KC ? p + (int64_t)(i0 + i) * ld + (k0 + k) : p + (int64_t)(k0 + k) * ld + (i0 + i);
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(KC ? &s[i * LDK + k] : &s[k * LDR + i]));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(src));
  }
}

// fragment element (row, k) of a staged tile
template <bool KC>
HBS_DEV double frag(const double* s, int row, int k) {
  return KC ? s[row * LDK + k] : s[k * LDR + row];
}

}  // namespace

// A(i, k): trans = 0 -> A[i*lda + k] (k contiguous); B(k, j): trans = 1 -> B[j*ldb + k] (k contiguous).
HBS_DEV bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <bool AKC, bool BKC>
__global__ void __launch_bounds__(NT, BGEMM_MINB) bgemm_kernel(BgemmArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                       // NSTAGE x STAGE
  double* Bs = smem + NSTAGE * STAGE;      // NSTAGE x STAGE
  // blockIdx.x = box * (tiles_m * tiles_n) + tile: a box's tiles run back to back (L2 reuse)
  const int tn_max = (args.N_max + BN - 1) / BN, tm_max = (args.M_max + BM - 1) / BM;
  const int64_t b = blockIdx.x / (tm_max * tn_max);
  const int tile = blockIdx.x % (tm_max * tn_max);
  const int rows = args.geo.row_begin ? box_rows(args.geo, b) : 0;
  const int M = args.M.fixed + args.M.rows_mult * rows;
  const int N = args.N.fixed + args.N.rows_mult * rows;
  const int K = args.K.fixed + args.K.rows_mult * rows;
  const int m0 = (tile / tn_max) * BM, n0 = (tile % tn_max) * BN;
  if (m0 >= M || n0 >= N) return;
  const int lda = args.A.ld_rows ? rows : args.A.ld_fixed;
  const int ldb = args.B.ld_rows ? rows : args.B.ld_fixed;
  const double* A = args.A.p + op_off(args.A, args.geo, b);
  const double* B = args.B.p + op_off(args.B, args.geo, b);
  const int tid = threadIdx.x;
  // 16-byte staging when every row start of this box's operands is aligned
  const bool vec = al16(A) && al16(B) && (lda % 2 == 0) && (ldb % 2 == 0);

  // interior tiles of aligned operands stage without bounds checks
  const bool full = vec && m0 + BM <= M && n0 + BN <= N && (K % BK) == 0;
  auto load = [&](int stage, int k0) {
    if (full) {
      stage_tile_full<AKC>(As + stage * STAGE, A, lda, m0, k0, tid);
      stage_tile_full<BKC>(Bs + stage * STAGE, B, ldb, n0, k0, tid);
    } else {
      stage_tile<AKC>(As + stage * STAGE, A, lda, m0, k0, M, K, tid, vec);
      stage_tile<BKC>(Bs + stage * STAGE, B, ldb, n0, k0, N, K, tid, vec);
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;   // 2 x 2 warps, warp tile 32 x 32
  double acc[4][4][2] = {};
  const int nk = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nk) load(s, s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    {   // refill the stage consumed last iteration
      const int kn = kt + NSTAGE - 1;
      if (kn < nk) load(kn % NSTAGE, kn * BK);
      cp_async_commit();
    }
    const double* as = As + (kt % NSTAGE) * STAGE;
    const double* bs = Bs + (kt % NSTAGE) * STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int fi = 0; fi < 4; ++fi) af[fi] = frag<AKC>(as, wm * 32 + fi * 8 + g, kk + t);
#pragma unroll
      for (int fj = 0; fj < 4; ++fj) bf[fj] = frag<BKC>(bs, wn * 32 + fj * 8 + g, kk + t);
#pragma unroll
      for (int fi = 0; fi < 4; ++fi)
#pragma unroll
        for (int fj = 0; fj < 4; ++fj) dmma8x8x4(acc[fi][fj][0], acc[fi][fj][1], af[fi], bf[fj]);
    }
  }
  cp_async_wait<0>();

  const int ldc = args.ldc_rows ? rows : args.ldc_fixed;
  double* C = args.C + args.cc_b * b + (args.cc_rb ? args.cc_rb * args.geo.row_begin[b] : 0) +
              (args.cc_sq ? args.cc_sq * args.geo.sq_off[b] : 0);
  const bool has_c0 = args.beta != 0.0;
  const int ldc0 = args.C0.ld_rows ? rows : args.C0.ld_fixed;
  const double* C0 = has_c0 ? args.C0.p + op_off(args.C0, args.geo, b) : nullptr;
  const bool cvec = al16(C) && (ldc % 2 == 0);
  if (full && cvec && !has_c0) {   // interior tile, no C0: unpredicated 16-byte stores
#pragma unroll
    for (int fi = 0; fi < 4; ++fi)
#pragma unroll
      for (int fj = 0; fj < 4; ++fj) {
        const int i = m0 + wm * 32 + fi * 8 + g;
        const int j = n0 + wn * 32 + fj * 8 + 2 * t;
        *reinterpret_cast<double2*>(C + (int64_t)i * ldc + j) =
            make_double2(args.alpha * acc[fi][fj][0], args.alpha * acc[fi][fj][1]);
      }
    return;
  }
#pragma unroll
  for (int fi = 0; fi < 4; ++fi)
#pragma unroll
    for (int fj = 0; fj < 4; ++fj) {
      const int i = m0 + wm * 32 + fi * 8 + g;
      const int j = n0 + wn * 32 + fj * 8 + 2 * t;
      if (i >= M) continue;
      double v0 = args.alpha * acc[fi][fj][0], v1 = args.alpha * acc[fi][fj][1];
      if (has_c0) {
        if (args.C0.trans) {
          if (j < N) v0 = fma(args.beta, C0[(int64_t)j * ldc0 + i], v0);
          if (j + 1 < N) v1 = fma(args.beta, C0[(int64_t)(j + 1) * ldc0 + i], v1);
        } else {
          if (j < N) v0 = fma(args.beta, C0[(int64_t)i * ldc0 + j], v0);
          if (j + 1 < N) v1 = fma(args.beta, C0[(int64_t)i * ldc0 + j + 1], v1);
        }
      }
      double* cp = C + (int64_t)i * ldc + j;
      if (cvec && j + 1 < N) {
        *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
      } else {
        if (j < N) cp[0] = v0;
        if (j + 1 < N) cp[1] = v1;
      }
    }
}

namespace {

template <bool AKC, bool BKC>
int launch_t(const BgemmArgs& args, dim3 grid, cudaStream_t stream) {
  const size_t smem = 2 * NSTAGE * STAGE * sizeof(double);
  cudaFuncSetAttribute(bgemm_kernel<AKC, BKC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bgemm_kernel<AKC, BKC><<<grid, NT, smem, stream>>>(args);
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

}  // namespace

int launch_bgemm(const BgemmArgs& args, cudaStream_t stream) {
  if (args.geo.nbox <= 0 || args.M_max <= 0 || args.N_max <= 0) return kOk;
  const int64_t tiles = (int64_t)((args.N_max + BN - 1) / BN) * ((args.M_max + BM - 1) / BM);
  if (tiles * args.geo.nbox >= (1ll << 31)) return kErrUnsupported;
  dim3 grid((unsigned)(tiles * args.geo.nbox));
  note_launch();
  const bool akc = !args.A.trans, bkc = args.B.trans != 0;
  if (akc && bkc) return launch_t<true, true>(args, grid, stream);
  if (akc) return launch_t<true, false>(args, grid, stream);
  if (bkc) return launch_t<false, true>(args, grid, stream);
  return launch_t<false, false>(args, grid, stream);
}

}  // namespace hbs
