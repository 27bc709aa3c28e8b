// Internal (C++) launch interface of the HBS kernels.  The public C-ABI lives
// in include/hbs_b200.h and is implemented in capi.cu on top of these.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace hbs {

enum Status : int {
  kOk = 0,
  kErrDimension = 1,      // -> DimensionError
  kErrConfiguration = 2,  // -> ConfigurationError
  kErrIllConditioned = 3, // -> IllConditionedProbeError (see status arrays)
  kErrCuda = 4,
  kErrWorkspace = 5,
  kErrUnsupported = 6,
};

constexpr size_t kMaxSmemBytes = 227 * 1024;

// Count of kernels this library has launched (process-wide, for the bench's
// gpu_launches claim); incremented by every launch_* helper.
void note_launch();

// ---------------------------------------------------------------- geqrf
enum GeqrfMode : int { kGeqrfFactor = 0, kGeqrfOrtho = 1 };

struct GeqrfSide {
  // source: element (i, j) of box b at src + src_c_rb*row_begin[b] + src_c_b*b + i*src_rs + j*src_cs
  const double* src;
  int64_t src_c_rb, src_c_b;
  int64_t src_rs, src_cs;
  // kFactor outputs (uniform per-box strides)
  double* vt; int64_t vt_stride; int ldvt;
  double* r; int64_t r_stride; int ldr;
  double* tau; int64_t tau_stride;
  double* t; int64_t t_stride;        // hqr: npanel x 32 x 32 compact-WY T blocks
  double* rinv; int64_t rinv_stride;  // hqr: npanel x 32 x 32 inverses of R's diagonal blocks
  int32_t* status;
  // kOrtho output: q + q_c_rb*row_begin[b] + q_c_b*b, row-major, ld = ldq
  double* q; int64_t q_c_rb, q_c_b; int ldq;
};

struct GeqrfArgs {
  LevelGeo geo;
  GeqrfSide side[2];
  int mode;
  int m_fixed, n_fixed, m_is_rows, n_is_rows;
  int m_max, n_max, lda_max;
  double tol;
  double* gscratch;  // needed when the matrix does not fit in shared memory
  int use_smem;
  const int32_t* only;  // if set: process (box b, side) only when only[side*nbox + b] != 0
  int skip_rows;        // cholqr generic kernel: boxes with this many rows went to a specialised launch (0: none)
  int uniform;          // every box of the level has m_max rows (host hint)
};

// Blocked Householder (hqr.cu): kFactor also emits the per-panel T and R
// diagonal-block inverses (PanelSide layout) through GeqrfSide::t / rinv.
size_t hqr_smem_bytes(int m_max, int n_max, int mode, bool with_matrix);
size_t hqr_scratch_doubles(int m_max, int n_max, int64_t nbox);
bool hqr_fits_smem(int m_max, int n_max, int mode);
int launch_hqr(GeqrfArgs args, int nsides, cudaStream_t stream);

// ---------------------------------------------------------------- CholeskyQR2 bases
// Orthonormal basis of each box's (rows x r) block (GeqrfArgs in kOrtho form:
// side[].src/q addressing, n_fixed = r, m_max = max rows).  flag[side*nbox + b]
// = 1 marks a breakdown; those blocks go to launch_hqr with only = flag.
bool cholqr_fits(int n_max, int r);
int launch_cholqr(GeqrfArgs args, int nsides, int32_t* flag, cudaStream_t stream);

// ---------------------------------------------------------------- fused probe QR + apply Q + solve
// Per (box, side): Householder QR of Omega_tau^T in shared memory (warps 0-7)
// while warps 8-15 apply each finished panel to the box's Y rows (streamed
// from L2) and finally solve X = (Y Q1) R^{-T}.  Output YQ (rows x s per box):
// columns 0..n-1 hold X = Y Omega^+, columns s-r..s-1 hold Y P.
struct FusedSide {
  const double* om; int64_t om_c_rb;       // Omega rows of box b at om + om_c_rb*row_begin[b], ld = s
  const double* y; int64_t y_c_rb;         // Y rows, ld = s
  double* yq; int64_t yq_stride;           // per box rows x s (ld = s), uniform stride
  double* t; int64_t t_stride;             // npanel x 32 x 32 compact-WY T blocks
  double* rinv; int64_t rinv_stride;       // npanel x 32 x 32 R diagonal-block inverses
  int32_t* status;
  const double* fac; int64_t fac_stride;   // PRE: Gram-kernel factorisation (n x s per box)
};
struct FusedArgs {
  LevelGeo geo;
  FusedSide side[2];
  int s, n_max, lda;
  double tol;
  int skip_rows;   // generic kernel: boxes with skip_rows_lo < rows <= skip_rows were done by a specialised launch (-1: none)
  int skip_rows_lo;
  int uniform;     // every box of the level has n_max rows (host hint): generic launches with no box are skipped
  int pre;                  // 1: apply the Gram factorisation (fac) instead of factoring Omega
  const int32_t* gflag;     // Gram flags (side*nbox + b): PRE takes flag 0, Householder flag != 0
};
bool fused_fits(int s, int n_max);
int launch_probe_fused(FusedArgs args, int nsides, cudaStream_t stream);
// Persistent pipelined form for config-4 shaped levels (fused_pipe.cu): 1 = ran on the
// 128-row boxes, 0 = shape or size does not apply, < 0 = launch error.
int launch_probe_fused_pipe(FusedArgs& args, int nsides, cudaStream_t stream);
// Same with the two warp groups on disjoint SM sub-partitions (fused_split.cu; HBS_SPLIT=1).
int launch_probe_fused_split(FusedArgs& args, int nsides, cudaStream_t stream);

// ---------------------------------------------------------------- Gram probe factorisation
// Per (box, side) with nullity s - n == r: Cholesky of Omega Omega^T and
// Householder reconstruction by a sign-chosen LU (gram.cu).  fac (n x s per
// box, uniform stride): row j = column j of [R_hh + V1 (strictly lower); V2],
// the layout the Householder kernel leaves in shared memory; t: compact-WY T
// of each 32-column panel.  flag[side*nbox + b] = 1 routes the (box, side) to
// the Householder path (shape, breakdown or doubtful conditioning).
struct GramSide {
  const double* om; int64_t om_c_rb;       // Omega rows of box b at om + om_c_rb*row_begin[b], ld = s
  double* fac; int64_t fac_stride;
  double* t; int64_t t_stride;
  int32_t* status;
};
struct GramArgs {
  LevelGeo geo;
  GramSide side[2];
  int s, r;
  int32_t* flag;
};
bool gram_fits(int s, int n_max, int r);
int launch_gram(const GramArgs& args, int nsides, cudaStream_t stream);
// Same factorisation with the LU operand in TMEM, two CTAs per SM (gram_tm.cu).
int launch_gram_tm(const GramArgs& args, int nsides, cudaStream_t stream);

// ---------------------------------------------------------------- apply Q + solve
// Per (row tile, box, side): Yt <- Y_tile * Q (blocked WY), then
// X_tile = (Y Q)(:, 0:n) R^{-T} and P-projection = (Y Q)(:, s-r:s).
struct ApplyQSide {
  const double* y; int64_t y_c_rb, y_c_b; int ldy;  // rows of Y for box b (row-major, ld)
  const double* vt; int64_t vt_stride; int ldvt;
  const double* r; int64_t r_stride; int ldr;
  const double* t; int64_t t_stride;
  const double* rinv; int64_t rinv_stride;
  double* x; int64_t x_stride; int ldx;      // n_b x n_b per box (uniform stride)
  double* yp; int64_t yp_stride; int ldyp;   // n_b x r per box (may be null)
};
struct ApplyQArgs {
  LevelGeo geo;
  ApplyQSide side[2];
  int s, r;
  int n_fixed, n_is_rows, n_max;
};
int launch_applyq(ApplyQArgs args, int nsides, cudaStream_t stream);
size_t applyq2_smem_bytes(int s);
int launch_applyq2(ApplyQArgs args, int nsides, cudaStream_t stream);

// ---------------------------------------------------------------- batched GEMM
// Operand addressing for box b: base + c_rb*row_begin[b] + c_b*b + c_sq*sq_off[b];
// element (i, j) at [i*ld + j] (trans = 0) or [j*ld + i] (trans = 1);
// ld = ld_fixed, or the box's row count when ld_rows != 0.
struct BOperand {
  const double* p;
  int64_t c_rb, c_b, c_sq;
  int ld_fixed, ld_rows, trans;
};
struct BDim {
  int fixed, rows_mult;  // value = fixed + rows_mult * rows_b
};
struct BgemmArgs {
  LevelGeo geo;
  BDim M, N, K;
  int M_max, N_max;
  BOperand A, B, C0;
  double* C; int64_t cc_rb, cc_b, cc_sq; int ldc_fixed, ldc_rows;
  double alpha, beta;  // C = alpha * op(A) op(B) + beta * C0
};
int launch_bgemm(const BgemmArgs& args, cudaStream_t stream);

}  // namespace hbs
