// Batched, variable-size fp64 GEMM on the FP64 tensor cores (DMMA m8n8k4),
// one launch per level-wide product (box b = blockIdx.z):
//     C_b = alpha * op(A_b) op(B_b) + beta * C0_b
// Operand bases are derived from the level geometry (row starts, packed
// square-block offsets), so the same kernel serves the discrepancy algebra
// (compress.py:192-197), the parent-sample lift (compress.py:209-227) and the
// telescoping apply used by the HBS sampler (factorization.py:89-143).
// 64 x 64 CTA tile, BK = 16, cp.async double buffering, 8 warps of 32 x 16.
#include "common.cuh"
#include "kernels.h"

namespace hbs {

namespace {
constexpr int BM = 64, BN = 64, BK = 16;
constexpr int LDA_S = 20;  // BK + 4  (== 4 mod 16)
constexpr int LDB_S = 68;  // BN + 4

HBS_DEV int64_t op_off(const BOperand& o, const LevelGeo& g, int64_t b) {
  int64_t off = o.c_b * b;
  if (o.c_rb) off += o.c_rb * g.row_begin[b];
  if (o.c_sq) off += o.c_sq * g.sq_off[b];
  return off;
}

}  // namespace

__global__ void __launch_bounds__(256) bgemm_kernel(BgemmArgs args) {
  __shared__ __align__(16) double As[2][BM * LDA_S];
  __shared__ __align__(16) double Bs[2][BK * LDB_S];
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

  auto load_tile = [&](int buf, int k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      int i, k;
      if (!args.A.trans) { i = idx >> 4; k = idx & 15; }
      else { i = idx & 63; k = idx >> 6; }
      const bool ok = (m0 + i < M) && (k0 + k < K);
      const double* src = args.A.trans ? A + (int64_t)(k0 + k) * lda + (m0 + i)
                                       : A + (int64_t)(m0 + i) * lda + (k0 + k);
      cp_async8(&As[buf][i * LDA_S + k], ok ? src : A, ok);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      int k, j;
      if (!args.B.trans) { k = idx >> 6; j = idx & 63; }
      else { j = idx >> 4; k = idx & 15; }
      const bool ok = (k0 + k < K) && (n0 + j < N);
      const double* src = args.B.trans ? B + (int64_t)(n0 + j) * ldb + (k0 + k)
                                       : B + (int64_t)(k0 + k) * ldb + (n0 + j);
      cp_async8(&Bs[buf][k * LDB_S + j], ok ? src : B, ok);
    }
    cp_async_commit();
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;   // 2 x 4 warps, warp tile 32 x 16
  double acc[4][2][2] = {};
  const int nk = (K + BK - 1) / BK;
  if (nk > 0) load_tile(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      load_tile(buf ^ 1, (kt + 1) * BK);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As[buf];
    const double* bs = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int fi = 0; fi < 4; ++fi) af[fi] = as[(wm * 32 + fi * 8 + g) * LDA_S + kk + t];
#pragma unroll
      for (int fj = 0; fj < 2; ++fj) bf[fj] = bs[(kk + t) * LDB_S + wn * 16 + fj * 8 + g];
#pragma unroll
      for (int fi = 0; fi < 4; ++fi)
#pragma unroll
        for (int fj = 0; fj < 2; ++fj) dmma8x8x4(acc[fi][fj][0], acc[fi][fj][1], af[fi], bf[fj]);
    }
    __syncthreads();
  }

  const int ldc = args.ldc_rows ? rows : args.ldc_fixed;
  double* C = args.C + args.cc_b * b + (args.cc_rb ? args.cc_rb * args.geo.row_begin[b] : 0) +
              (args.cc_sq ? args.cc_sq * args.geo.sq_off[b] : 0);
  const bool has_c0 = args.beta != 0.0;
  const int ldc0 = args.C0.ld_rows ? rows : args.C0.ld_fixed;
  const double* C0 = has_c0 ? args.C0.p + op_off(args.C0, args.geo, b) : nullptr;
#pragma unroll
  for (int fi = 0; fi < 4; ++fi)
#pragma unroll
    for (int fj = 0; fj < 2; ++fj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = m0 + wm * 32 + fi * 8 + g;
        const int j = n0 + wn * 16 + fj * 8 + 2 * t + e;
        if (i < M && j < N) {
          double v = args.alpha * acc[fi][fj][e];
          if (has_c0) {
            const double c0 = args.C0.trans ? C0[(int64_t)j * ldc0 + i] : C0[(int64_t)i * ldc0 + j];
            v = fma(args.beta, c0, v);
          }
          C[(int64_t)i * ldc + j] = v;
        }
      }
}

int launch_bgemm(const BgemmArgs& args, cudaStream_t stream) {
  if (args.geo.nbox <= 0 || args.M_max <= 0 || args.N_max <= 0) return kOk;
  const int64_t tiles = (int64_t)((args.N_max + BN - 1) / BN) * ((args.M_max + BM - 1) / BM);
  if (tiles * args.geo.nbox >= (1ll << 31)) return kErrUnsupported;
  dim3 grid((unsigned)(tiles * args.geo.nbox));
  bgemm_kernel<<<grid, 256, 0, stream>>>(args);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

}  // namespace hbs
