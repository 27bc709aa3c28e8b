/*
 * hbs_b200.h -- C-ABI of the B200-native HBS compress-from-samples path.
 *
 * Drop-in boundary for the hot path of the reference `hbs` package
 * (arXiv 2205.02990, /root/reference/pkg/src/hbs):
 *
 *   reference (Python)                                   this ABI
 *   ---------------------------------------------------  ------------------------------------
 *   compress_from_samples, per-level body                 hbs_compress_level
 *     (compress.py:250-269: compress_node_bases            (all boxes of one level, both sides)
 *      155-175, compute_discrepancy 178-197,
 *      lift_to_parent 200-227)
 *   compress_from_samples, root (compress.py:271-279,     hbs_compress_root
 *     compute_root 230-233)
 *   nullspace / col / lstsq_right (linalg.py:35-90)       (inside the two calls above)
 *   apply_matrix (factorization.py:89-143) = the HBS      hbs_apply
 *     sampler behind hbs_oracle (operators.py:221-228)
 *   dense_oracle a @ x / a.T @ x (operators.py:213-218)   hbs_dense_apply
 *   IllConditionedProbeError(node_id, level)              per-box int32 status arrays
 *     (errors.py:12-19, compress.py:260-265)                (+ HBS_ERR_ILL_CONDITIONED)
 *
 * Conventions.  All matrices are fp64, row-major (numpy C order).  Every
 * pointer is a DEVICE pointer unless stated; the library allocates nothing:
 * the caller passes a workspace sized by the *_workspace_bytes queries.
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 * stream-ordered and never synchronise the host.
 *
 * Level geometry.  A level has `nbox` boxes; box b owns rows
 * [row_begin[b], row_begin[b+1]) of the level's sample quadruple
 * (leaf level: the global samples; coarser levels: the lifted 2r-row blocks).
 * sq_off[b] = sum_{c<b} rows_c^2 (packed square blocks).
 *
 * Outputs of a level: U, V packed as (total_rows x r) with box b at row
 * row_begin[b]; D packed as consecutive rows_b x rows_b blocks at sq_off[b];
 * the lifted parent quadruple (nbox*r x s, child b at rows [b*r, (b+1)*r)).
 */
#ifndef HBS_B200_H_
#define HBS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define HBS_OK 0
#define HBS_ERR_DIMENSION 1        /* -> DimensionError */
#define HBS_ERR_CONFIGURATION 2    /* -> ConfigurationError (nullity s - rows < r) */
#define HBS_ERR_ILL_CONDITIONED 3  /* -> IllConditionedProbeError (see status) */
#define HBS_ERR_CUDA 4
#define HBS_ERR_WORKSPACE 5
#define HBS_ERR_UNSUPPORTED 6

/* Library version / build identification (sm_100a). */
const char* hbs_b200_version(void);

/* Workspace needed by hbs_compress_level for a level of `nbox` boxes of at
 * most `max_rows` rows with s probes and rank r.  Replaces the reference's
 * per-node temporaries (compress.py:155-227). */
int hbs_level_workspace_bytes(int64_t nbox, int max_rows, int s, int r, size_t* bytes);

/* One level of the sweep (compress.py:250-269 for every node of the level,
 * plus lift_to_parent for the next level, compress.py:254-256/200-227).
 *   omega, psi, y, z : level quadruple, rows x s, ld = s
 *   u, v, d          : outputs (see header comment)
 *   lift_*           : parent quadruple outputs (nbox*r x s) or all NULL
 *   status           : int32[2*nbox]; status[side*nbox + b] != 0 marks box b's
 *                      side (0: omega, 1: psi) as failing the sigma test of
 *                      lstsq_right (linalg.py:73-78) with tolerance `tol`.
 * Returns HBS_ERR_CONFIGURATION when s - max_rows < r (compress.py:164-168). */
int hbs_compress_level(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows,
                       int s, int r, double tol,
                       const double* omega, const double* psi, const double* y, const double* z,
                       double* u, double* v, double* d,
                       double* lift_omega, double* lift_psi, double* lift_y, double* lift_z,
                       void* workspace, size_t workspace_bytes, int32_t* status, void* stream);

/* Same as hbs_compress_level, but records CUDA events between its phases and
 * writes their durations (ms) to the HOST array phase_ms[6]: probe QR,
 * panel factors, apply-Q + solve, basis QR (col), discrepancy GEMMs, lift
 * GEMMs.  Synchronises the stream; for measurement only. */
int hbs_compress_level_profiled(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows,
                                int s, int r, double tol,
                                const double* omega, const double* psi, const double* y, const double* z,
                                double* u, double* v, double* d,
                                double* lift_omega, double* lift_psi, double* lift_y, double* lift_z,
                                void* workspace, size_t workspace_bytes, int32_t* status, void* stream,
                                float* phase_ms);

/* Building block: batched Householder QR of Omega_tau^T for every box of a
 * level -- the factorisation numpy.linalg.qr(mode="complete") performs inside
 * the reference's nullspace() (linalg.py:52-62), with LAPACK's dlarfg
 * reflector convention.  Per box b (uniform strides by max_rows = nr):
 *   vt   : nr x s, reflector j as row j (unit diagonal, zeros before it)
 *   r    : nr x nr upper triangular R  (Omega_tau^T = Q R)
 *   tau  : nr reflector scalars
 *   t    : ceil(nr/32) compact-WY T blocks (32 x 32, row-major)
 *   rinv : ceil(nr/32) inverses of R's 32 x 32 diagonal blocks
 *   status[b] = 1 when min|R_ii| < tol max|R_ii| (rank-deficient probe block)
 * scratch: hbs_probe_qr_scratch_bytes (0 unless a matrix exceeds shared memory). */
int hbs_probe_qr_scratch_bytes(int64_t nbox, int max_rows, int s, size_t* bytes);
int hbs_probe_qr(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows, int s,
                 double tol, const double* omega, double* vt, double* r, double* tau, double* t, double* rinv,
                 double* scratch, int32_t* status, void* stream);

/* Building block: the same factorisation of Omega_tau^T by Gram / Cholesky and
 * a sign-chosen LU that reconstructs the Householder form (gram.cu), for
 * boxes with nullity s - rows == r.  Per box b (uniform stride rows x s):
 *   fac  : row j = column j of [R (upper, on/above the diagonal) + V1 (below); V2],
 *          i.e. hbs_probe_qr's r and vt in one array
 *   t    : ceil(rows/32) compact-WY T blocks (32 x 32, row-major)
 *   flag[b] = 1 when the box needs the Householder kernel instead (shape,
 *          Cholesky breakdown or min R_ii < 1e-3 max R_ii); status[b] = 0
 *          otherwise.  Needs max_rows <= 128, s <= 256. */
int hbs_gram_probe_factor(int64_t nbox, const int64_t* row_begin, int max_rows, int s, int r,
                          const double* omega, double* fac, double* t, int32_t* flag, int32_t* status,
                          void* stream);

/* Building block: batched reduced Householder QR with explicit Q -- the
 * reference's col() (linalg.py:35-49: np.linalg.qr(b)[0][:, :r]) for every
 * box of a level.  b and q are packed (rows x r) row-major with box b at row
 * row_begin[b]; q may alias nothing in b.  scratch: hbs_basis_qr_scratch_bytes. */
int hbs_basis_qr_scratch_bytes(int64_t nbox, int max_rows, int r, size_t* bytes);
int hbs_basis_qr(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows, int r,
                 const double* b, double* q, double* scratch, void* stream);

/* Building block: the orthonormal bases hbs_compress_level uses for col()
 * (linalg.py:35-49): CholeskyQR2 on the FP64 tensor cores, any orthonormal
 * basis of span(b) (the reference's result only depends on the span, see
 * cholqr.cu), with the Householder kernel re-run for blocks whose Cholesky
 * breaks down (rank-deficient, zero, or condition number beyond ~1e6).
 * flags: nbox int32 scratch; on return flags[b] = 1 where the fallback ran.
 * Needs max_rows <= 128 and r <= 64, else HBS_ERR_UNSUPPORTED. */
int hbs_basis_orth(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows, int r,
                   const double* b, double* q, int32_t* flags, double* scratch, void* stream);

/* Number of CUDA kernels launched by this library so far (process-wide). */
unsigned long long hbs_launch_counter(void);

/* Optional hint for the NEXT hbs_compress_level / hbs_compress_level_profiled
 * call of the calling thread: the smallest box of the level has `min_rows`
 * rows (the host knows the tree, tree.py:63-102; the library only sees device
 * pointers).  When min_rows == max_rows every box has the shape the
 * specialised kernels cover, and the generic launches that would find no box
 * are skipped.  Results do not depend on the hint; 0 (the default after every
 * level call) means unknown. */
void hbs_level_hint(int min_rows);

/* Root core D_root = Y_root Omega_root^+ (compress.py:230-233), rows = 2r.
 * `row_begin`/`sq_off` describe the single root box ({0, 2r} / {0, 4r^2}). */
int hbs_root_workspace_bytes(int rows, int s, size_t* bytes);
int hbs_compress_root(const int64_t* row_begin, const int64_t* sq_off, int rows, int s, double tol,
                      const double* omega, const double* y, double* root,
                      void* workspace, size_t workspace_bytes, int32_t* status, void* stream);

/* Telescoping apply out = A q (transpose = 0) or A^T q (transpose = 1) of a
 * packed factorization (factorization.py:89-143).  Host arrays of length
 * depth+1 hold per-level DEVICE pointers (index 0 unused): row_begin[l],
 * sq_off[l] (2^l + 1 entries each), u[l], v[l], d[l].  q, out: n x c. */
int hbs_apply_workspace_bytes(int depth, int r, int64_t c, size_t* bytes);
int hbs_apply(int depth, int r, int64_t n, int64_t c,
              const int64_t* const* row_begin, const int64_t* const* sq_off,
              const double* const* u, const double* const* v, const double* const* d,
              const double* root, const double* q, double* out, int transpose,
              void* workspace, size_t workspace_bytes, void* stream);

/* The three sweeps of hbs_apply, exposed for the subtree-partitioned sampler
 * (one process per GPU: local upward pass, all-gather of qhat at the
 * partition level, replicated top, local downward pass).  Per-level host
 * arrays are indexed by level number: nbox[l], row_begin[l], sq_off[l]
 * (device), basis[l] / d[l] (device), qhat[l] / uhat[l] (device, box b's
 * r x c block at b*r*c).
 *   up:   qhat[l] = basis_l^T (l == level_hi ? q : qhat[l+1]),  l = level_hi .. level_lo
 *   root: uhat1 = root^(T) qhat1                                  (2r x c)
 *   down: (l == level_hi ? out : uhat[l+1]) = basis_l uhat[l] + d_l^(T) (l == level_hi ? q : qhat[l+1]),
 *         l = level_lo .. level_hi; max_rows_hi = largest box at level_hi. */
int hbs_apply_up(int level_hi, int level_lo, int r, int64_t c, const int64_t* nbox,
                 const int64_t* const* row_begin, const int64_t* const* sq_off, const double* const* basis,
                 const double* q, double* const* qhat, void* stream);
int hbs_apply_root(int r, int64_t c, const double* root, int transpose, const double* qhat1, double* uhat1,
                   void* stream);
int hbs_apply_down(int level_lo, int level_hi, int r, int64_t c, const int64_t* nbox,
                   const int64_t* const* row_begin, const int64_t* const* sq_off, int max_rows_hi,
                   const double* const* basis, const double* const* d, int transpose_d, double* const* uhat,
                   const double* const* qhat, const double* q, double* out, void* stream);

/* Dense sampler out = A q or A^T q for an explicit n x n row-major A
 * (operators.py:213-218). */
int hbs_dense_apply(int64_t n, int64_t c, const double* a, const double* q, double* out,
                    int transpose, void* stream);

/* Config-3 operator generator: A_ij = log|x_i - x_j| (i != j), A_ii = 1 with
 * x_i = (cos t_i, 0.5 sin t_i), t_i = 2 pi i / n.  Fills rows [row0, row0+rows). */
int hbs_fill_log_kernel(int64_t n, int64_t row0, int64_t rows, double* a, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HBS_B200_H_ */
