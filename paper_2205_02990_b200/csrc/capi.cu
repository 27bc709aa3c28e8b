// C-ABI implementation (include/hbs_b200.h): level orchestration of the
// batched kernels, workspace carving, and the samplers.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include "../../include/hbs_b200.h"
#include "kernels.h"

#include <atomic>

namespace hbs {
static std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {

// Optional per-phase timing of hbs_compress_level (hbs_compress_level_profiled).
struct PhaseTimer {
  cudaEvent_t ev[8];
  int n = 0;
  bool on = false;
  cudaStream_t st = nullptr;
  void start(cudaStream_t s) {
    on = true; st = s; n = 0;
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventRecord(ev[n++], st);
  }
  void mark() { if (on && n < 8) cudaEventRecord(ev[n++], st); }
  void finish(float* out, int nphase) {
    if (!on) return;
    cudaEventSynchronize(ev[n - 1]);
    for (int i = 0; i < nphase; ++i) {
      out[i] = 0.f;
      if (i + 1 < n) cudaEventElapsedTime(&out[i], ev[i], ev[i + 1]);
    }
    for (auto& e : ev) cudaEventDestroy(e);
    on = false;
  }
};
PhaseTimer g_timer;  // only used by the profiled entry point (not thread-safe by design)

// Side stream for the four lift products that need only the bases (V^T Omega,
// U^T Psi, U^T Y, V^T Z): they run next to the discrepancy chain, which matters
// on the upper levels where a single short GEMM cannot fill the GPU.  Forked
// and joined with events, so a CUDA-graph capture of the caller's stream keeps
// the concurrency.  HBS_LIFT_OVERLAP=0 keeps everything on one stream.
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, e1 = nullptr, join = nullptr;
  bool ok = false;
  SideStream() {
    const char* e = std::getenv("HBS_LIFT_OVERLAP");
    if (e && e[0] == '0') return;
    ok = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess;
  }
};
SideStream& side_stream() {
  thread_local SideStream s;
  return s;
}

constexpr size_t kAlign = 256;

// HBS_GRAM_V3=1: the one-CTA-per-SM Gram kernel (gram.cu) instead of the TMEM one (gram_tm.cu)
bool gram_v3() {
  static const bool v = [] { const char* e = std::getenv("HBS_GRAM_V3"); return e && e[0] == '1'; }();
  return v;
}

struct Carver {
  char* base;
  size_t used = 0;
  template <typename T>
  T* take(size_t count) {
    used = (used + kAlign - 1) / kAlign * kAlign;
    T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
    used += count * sizeof(T);
    return p;
  }
};

// Per-level scratch (uniform per-box strides, max_rows = nr).
struct LevelWs {
  double* vt[2]; double* R[2]; double* tau[2]; double* T[2]; double* Rinv[2];
  double* X[2];   // Y Omega^+ and Z Psi^+
  double* P[2];   // Y P and Z Q
  double* G1; double* M3; double* M4; double* E1; double* E2;
  double* gscratch;
  int32_t* qr_flag;   // 2 x nbox CholeskyQR2 breakdown flags
  bool fused;
  bool gram;          // Gram / Householder-reconstruction probe factorisation (gram.cu)
  double* fac[2];     // its output (rows x s per box)
  int32_t* gflag;     // 2 x nbox: 1 = Householder fallback
  // where the solve results live after factor_and_solve
  const double* Xp[2]; int ldX; int64_t strideX;   // Y Omega^+ / Z Psi^+
  const double* Pp[2]; int ldP; int64_t strideP;   // Y P / Z Q
};

size_t carve_level(Carver& c, LevelWs& w, int64_t nbox, int nr, int s, int r, bool root_only) {
  const size_t nb = (size_t)nbox;
  const int npanel = (nr + kNB - 1) / kNB;
  const int sides = root_only ? 1 : 2;
  // HBS_PROBE_SPLIT=1 (experiments only): separate QR + apply-Q kernels
  static const bool force_split = std::getenv("HBS_PROBE_SPLIT") != nullptr;
  w.fused = fused_fits(s, nr) && !force_split;
  // HBS_GRAM=1: Gram / Householder-reconstruction probe factorisation for the
  // eligible boxes (experimental; HBS_GRAM=0 or unset: Householder only).
  // The root needs only Y Omega^+ (unique for any nullity); other levels need
  // nullity == r for the null-space pick to be basis independent.
  static const bool use_gram = [] { const char* e = std::getenv("HBS_GRAM"); return e && e[0] == '1'; }();
  w.gram = w.fused && use_gram && gram_fits(s, nr, root_only ? s - nr : r);
  for (int sd = 0; sd < 2; ++sd) {
    const bool on = sd < sides;
    w.fac[sd] = (on && w.gram) ? c.take<double>(nb * nr * s) : nullptr;
    // vt doubles as the fused kernel's Y Q buffer (rows x s per box)
    w.vt[sd] = on ? c.take<double>(nb * nr * s) : nullptr;
    w.R[sd] = (on && !w.fused) ? c.take<double>(nb * nr * nr) : nullptr;
    w.tau[sd] = (on && !w.fused) ? c.take<double>(nb * nr) : nullptr;
    w.T[sd] = on ? c.take<double>(nb * npanel * kNB * kNB) : nullptr;
    w.Rinv[sd] = on ? c.take<double>(nb * (npanel + 1) * kNB * kNB) : nullptr;   // + scratch block
    w.X[sd] = (on && !w.fused) ? c.take<double>(nb * nr * nr) : nullptr;
    w.P[sd] = (on && !root_only && !w.fused) ? c.take<double>(nb * nr * r) : nullptr;
  }
  if (!root_only) {
    w.G1 = c.take<double>(nb * r * nr);
    w.M3 = c.take<double>(nb * r * r);
    w.M4 = c.take<double>(nb * r * nr);
    w.E1 = c.take<double>(nb * r * nr);
    w.E2 = c.take<double>(nb * r * nr);
    w.qr_flag = c.take<int32_t>(2 * nb);
  } else {
    w.G1 = w.M3 = w.M4 = w.E1 = w.E2 = nullptr;
    w.qr_flag = nullptr;
  }
  w.gflag = w.gram ? c.take<int32_t>(2 * nb) : nullptr;
  const bool big_factor = !hqr_fits_smem(s, nr, kGeqrfFactor);
  const bool big_ortho = !root_only && !hqr_fits_smem(nr, r, kGeqrfOrtho);
  w.gscratch = (big_factor || big_ortho)
                   ? c.take<double>(hqr_scratch_doubles(s > nr ? s : nr, nr > r ? nr : r, nbox))
                   : nullptr;
  return c.used + kAlign;
}

BOperand op(const double* p, int64_t c_rb, int64_t c_b, int64_t c_sq, int ld, bool ld_rows, bool trans) {
  BOperand o;
  o.p = p; o.c_rb = c_rb; o.c_b = c_b; o.c_sq = c_sq;
  o.ld_fixed = ld; o.ld_rows = ld_rows ? 1 : 0; o.trans = trans ? 1 : 0;
  return o;
}
BDim dfix(int v) { return BDim{v, 0}; }
BDim drows() { return BDim{0, 1}; }

int gemm(const LevelGeo& geo, BDim M, BDim N, BDim K, int mmax, int nmax, BOperand A, BOperand B,
         double* C, int64_t cc_rb, int64_t cc_b, int64_t cc_sq, int ldc, bool ldc_rows, double alpha,
         double beta, BOperand C0, cudaStream_t st) {
  BgemmArgs a;
  a.geo = geo; a.M = M; a.N = N; a.K = K; a.M_max = mmax; a.N_max = nmax;
  a.A = A; a.B = B; a.C0 = C0;
  a.C = C; a.cc_rb = cc_rb; a.cc_b = cc_b; a.cc_sq = cc_sq; a.ldc_fixed = ldc; a.ldc_rows = ldc_rows ? 1 : 0;
  a.alpha = alpha; a.beta = beta;
  return launch_bgemm(a, st);
}

#define HBS_TRY(x) do { int _e = (x); if (_e != kOk) return _e; } while (0)

// hbs_level_hint: smallest box of the next level call (0 = unknown), consumed by that call
thread_local int g_min_rows_hint = 0;
thread_local int g_level_uniform = 0;   // the running level call: min rows == max rows

// Probe factorisation + apply/solve for both sides of a level (or side 0 only).
int factor_and_solve(const LevelGeo& geo, int nr, int s, int r, double tol, int nsides,
                     const double* om0, const double* om1, const double* y0, const double* y1,
                     LevelWs& w, int32_t* status, double* root_out, cudaStream_t st) {
  const int npanel_f = (nr + kNB - 1) / kNB;
  if (w.fused) {
    FusedArgs f;
    std::memset(&f, 0, sizeof(f));
    f.geo = geo; f.s = s; f.n_max = nr; f.tol = tol;
    f.uniform = g_level_uniform;
    const double* oms[2] = {om0, om1};
    const double* ys[2] = {y0, y1};
    for (int sd = 0; sd < nsides; ++sd) {
      FusedSide& S = f.side[sd];
      S.om = oms[sd]; S.om_c_rb = s;
      S.y = ys[sd]; S.y_c_rb = s;
      S.yq = w.vt[sd]; S.yq_stride = (int64_t)nr * s;
      S.t = w.T[sd]; S.t_stride = (int64_t)npanel_f * kNB * kNB;
      S.rinv = w.Rinv[sd]; S.rinv_stride = (int64_t)(npanel_f + 1) * kNB * kNB;
      S.status = status + sd * geo.nbox;
      w.Xp[sd] = w.vt[sd];
      w.Pp[sd] = w.vt[sd] + (s - r);
    }
    w.ldX = s; w.strideX = (int64_t)nr * s;
    w.ldP = s; w.strideP = (int64_t)nr * s;
    if (w.gram) {
      // Gram factorisation of every (box, side); the fused kernel applies it
      // to Y (PRE) and factors the flagged ones by Householder.
      GramArgs ga;
      std::memset(&ga, 0, sizeof(ga));
      ga.geo = geo; ga.s = s; ga.r = s - nr; ga.flag = w.gflag;
      for (int sd = 0; sd < nsides; ++sd) {
        GramSide& G = ga.side[sd];
        G.om = oms[sd]; G.om_c_rb = s;
        G.fac = w.fac[sd]; G.fac_stride = (int64_t)nr * s;
        G.t = w.T[sd]; G.t_stride = (int64_t)npanel_f * kNB * kNB;
        G.status = status + sd * geo.nbox;
        f.side[sd].fac = w.fac[sd]; f.side[sd].fac_stride = (int64_t)nr * s;
      }
      HBS_TRY(gram_v3() ? launch_gram(ga, nsides, st) : launch_gram_tm(ga, nsides, st));
      f.gflag = w.gflag;
      f.pre = 1;
      HBS_TRY(launch_probe_fused(f, nsides, st));
      f.pre = 0;
    }
    HBS_TRY(launch_probe_fused(f, nsides, st));
    g_timer.mark(); g_timer.mark(); g_timer.mark();   // (QR, panel factors and apply are one kernel)
    if (root_out) {
      if (cudaMemcpy2DAsync(root_out, nr * sizeof(double), w.vt[0], s * sizeof(double), nr * sizeof(double), nr,
                            cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return kErrCuda;
    }
    return kOk;
  }
  for (int sd = 0; sd < nsides; ++sd) { w.Xp[sd] = w.X[sd]; w.Pp[sd] = w.P[sd]; }
  w.ldX = nr; w.strideX = (int64_t)nr * nr;
  w.ldP = r; w.strideP = (int64_t)nr * r;
  GeqrfArgs g;
  std::memset(&g, 0, sizeof(g));
  g.geo = geo; g.mode = kGeqrfFactor;
  g.m_fixed = s; g.m_is_rows = 0; g.n_fixed = 0; g.n_is_rows = 1;
  g.m_max = s; g.n_max = nr; g.tol = tol; g.gscratch = w.gscratch;
  const double* oms[2] = {om0, om1};
  const int npanel = (nr + kNB - 1) / kNB;
  for (int sd = 0; sd < nsides; ++sd) {
    GeqrfSide& S = g.side[sd];
    S.src = oms[sd]; S.src_c_rb = s; S.src_c_b = 0; S.src_rs = 1; S.src_cs = s;
    S.vt = w.vt[sd]; S.vt_stride = (int64_t)nr * s; S.ldvt = s;
    S.r = w.R[sd]; S.r_stride = (int64_t)nr * nr; S.ldr = nr;
    S.tau = w.tau[sd]; S.tau_stride = nr;
    S.t = w.T[sd]; S.t_stride = (int64_t)npanel * kNB * kNB;
    S.rinv = w.Rinv[sd]; S.rinv_stride = (int64_t)npanel * kNB * kNB;
    S.status = status + sd * geo.nbox;
  }
  HBS_TRY(launch_hqr(g, nsides, st));
  g_timer.mark();
  g_timer.mark();  // (panel factors are produced inside the QR kernel)

  ApplyQArgs a;
  std::memset(&a, 0, sizeof(a));
  a.geo = geo; a.s = s; a.r = r; a.n_fixed = 0; a.n_is_rows = 1; a.n_max = nr;
  const double* ys[2] = {y0, y1};
  for (int sd = 0; sd < nsides; ++sd) {
    ApplyQSide& S = a.side[sd];
    S.y = ys[sd]; S.y_c_rb = s; S.y_c_b = 0; S.ldy = s;
    S.vt = w.vt[sd]; S.vt_stride = (int64_t)nr * s; S.ldvt = s;
    S.r = w.R[sd]; S.r_stride = (int64_t)nr * nr; S.ldr = nr;
    S.t = w.T[sd]; S.t_stride = (int64_t)npanel * kNB * kNB;
    S.rinv = w.Rinv[sd]; S.rinv_stride = (int64_t)npanel * kNB * kNB;
    if (root_out) {
      S.x = root_out; S.x_stride = 0; S.ldx = nr;
      S.yp = nullptr;
    } else {
      S.x = w.X[sd]; S.x_stride = (int64_t)nr * nr; S.ldx = nr;
      S.yp = w.P[sd]; S.yp_stride = (int64_t)nr * r; S.ldyp = r;
    }
  }
  if (applyq2_smem_bytes(s) <= kMaxSmemBytes) HBS_TRY(launch_applyq2(a, nsides, st));
  else HBS_TRY(launch_applyq(a, nsides, st));
  g_timer.mark();
  return kOk;
}

}  // namespace
}  // namespace hbs

using namespace hbs;

extern "C" {

const char* hbs_b200_version(void) { return "hbs_b200 0.1 (sm_100a, fp64 DMMA)"; }

int hbs_level_workspace_bytes(int64_t nbox, int max_rows, int s, int r, size_t* bytes) {
  if (nbox < 1 || max_rows < 1 || s < 1 || r < 1 || !bytes) return HBS_ERR_DIMENSION;
  Carver c{nullptr};
  LevelWs w;
  *bytes = carve_level(c, w, nbox, max_rows, s, r, false);
  return HBS_OK;
}

int hbs_compress_level(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows, int s,
                       int r, double tol, const double* omega, const double* psi, const double* y,
                       const double* z, double* u, double* v, double* d, double* lift_omega,
                       double* lift_psi, double* lift_y, double* lift_z, void* workspace,
                       size_t workspace_bytes, int32_t* status, void* stream) {
  g_level_uniform = (g_min_rows_hint == max_rows) ? 1 : 0;   // hbs_level_hint, consumed here
  g_min_rows_hint = 0;
  if (nbox < 1 || max_rows < 1 || s < 1 || r < 1 || max_rows < r) return HBS_ERR_DIMENSION;
  if (s - max_rows < r) return HBS_ERR_CONFIGURATION;
  if (s > 512) return HBS_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carver c{static_cast<char*>(workspace)};
  LevelWs w;
  if (carve_level(c, w, nbox, max_rows, s, r, false) > workspace_bytes) return HBS_ERR_WORKSPACE;
  const LevelGeo geo{row_begin, sq_off, nbox};
  const int nr = max_rows;

  HBS_TRY(factor_and_solve(geo, nr, s, r, tol, 2, omega, psi, y, z, w, status, nullptr, st));

  // U = col(Y P), V = col(Z Q): Householder QR + explicit Q (linalg.py:35-49).
  GeqrfArgs g;
  std::memset(&g, 0, sizeof(g));
  g.geo = geo; g.mode = kGeqrfOrtho;
  g.m_fixed = 0; g.m_is_rows = 1; g.n_fixed = r; g.n_is_rows = 0;
  g.m_max = nr; g.n_max = r; g.tol = tol; g.gscratch = w.gscratch;
  double* outs[2] = {u, v};
  for (int sd = 0; sd < 2; ++sd) {
    GeqrfSide& S = g.side[sd];
    S.src = w.Pp[sd]; S.src_c_rb = 0; S.src_c_b = w.strideP; S.src_rs = w.ldP; S.src_cs = 1;
    S.q = outs[sd]; S.q_c_rb = r; S.q_c_b = 0; S.ldq = r;
  }
  // CholeskyQR2 bases on the tensor cores (Householder only for flagged
  // blocks) when they are interchangeable with the reference's: the basis of
  // a node reaches the parent only through its span and a rotation of the
  // parent's probe rows, and the parent's null-space pick (the last r columns
  // of its complete Householder Q, linalg.py:52-62) is rotation-invariant
  // exactly when its nullity s - 2r equals r.  Every BASELINE config has
  // s = 3r; otherwise keep LAPACK's reflector-defined bases.
  g.uniform = g_level_uniform;
  if (cholqr_fits(nr, r) && s <= 3 * r) {
    HBS_TRY(launch_cholqr(g, 2, w.qr_flag, st));
    g.only = w.qr_flag;
  }
  HBS_TRY(launch_hqr(g, 2, st));
  g_timer.mark();

  // Discrepancy D = X - U [U^T X - U^T W^T + (U^T W^T V) V^T]  (compress.py:192-197)
  const BOperand none = op(nullptr, 0, 0, 0, 0, false, false);
  const BOperand Ut = op(u, r, 0, 0, r, false, true);   // U^T  (r x rows)
  const BOperand Un = op(u, r, 0, 0, r, false, false);  // U    (rows x r)
  const BOperand Vt = op(v, r, 0, 0, r, false, true);
  const BOperand Vn = op(v, r, 0, 0, r, false, false);
  const int64_t sqs = (int64_t)nr * nr, rs = (int64_t)r * nr;
  const BOperand Om = op(omega, s, 0, 0, s, false, false);
  const BOperand Ps = op(psi, s, 0, 0, s, false, false);
  const BOperand Yn = op(y, s, 0, 0, s, false, false);
  const BOperand Zn = op(z, s, 0, 0, s, false, false);
  const int64_t prs = (int64_t)r * s;
  // the lift products that need only the bases go to the side stream (not under the
  // phase timer, whose events live on the caller's stream)
  SideStream& side = side_stream();
  const bool overlap = lift_omega != nullptr && side.ok && !g_timer.on;
  cudaStream_t ls = overlap ? side.st : st;
  auto lift_base = [&]() -> int {
    HBS_TRY(gemm(geo, dfix(r), dfix(s), drows(), r, s, Vt, Om, lift_omega, 0, prs, 0, s, false, 1.0, 0.0, none, ls));
    HBS_TRY(gemm(geo, dfix(r), dfix(s), drows(), r, s, Ut, Ps, lift_psi, 0, prs, 0, s, false, 1.0, 0.0, none, ls));
    HBS_TRY(gemm(geo, dfix(r), dfix(s), drows(), r, s, Ut, Yn, lift_y, 0, prs, 0, s, false, 1.0, 0.0, none, ls));
    HBS_TRY(gemm(geo, dfix(r), dfix(s), drows(), r, s, Vt, Zn, lift_z, 0, prs, 0, s, false, 1.0, 0.0, none, ls));
    return HBS_OK;
  };
  if (overlap) {
    if (cudaEventRecord(side.fork, st) != cudaSuccess || cudaStreamWaitEvent(side.st, side.fork, 0) != cudaSuccess)
      return HBS_ERR_CUDA;
    HBS_TRY(lift_base());
  }
  const BOperand Xn = op(w.Xp[0], 0, w.strideX, 0, w.ldX, false, false);
  const BOperand Wt = op(w.Xp[1], 0, w.strideX, 0, w.ldX, false, true);
  const BOperand G1 = op(w.G1, 0, rs, 0, nr, false, false);
  const BOperand M3 = op(w.M3, 0, (int64_t)r * r, 0, r, false, false);
  const BOperand M4 = op(w.M4, 0, rs, 0, nr, false, false);
  HBS_TRY(gemm(geo, dfix(r), drows(), drows(), r, nr, Ut, Wt, w.G1, 0, rs, 0, nr, false, 1.0, 0.0, none, st));
  HBS_TRY(gemm(geo, dfix(r), dfix(r), drows(), r, r, G1, Vn, w.M3, 0, (int64_t)r * r, 0, r, false, 1.0, 0.0,
               none, st));
  // E1 = G1 - M3 V^T (= U^T D, reused by the lift), M4 = U^T X - E1
  const BOperand E1 = op(w.E1, 0, rs, 0, nr, false, false);
  HBS_TRY(gemm(geo, dfix(r), drows(), dfix(r), r, nr, M3, Vt, w.E1, 0, rs, 0, nr, false, -1.0, 1.0, G1, st));
  if (overlap) {   // U^T (Y - D Omega) = U^T Y - E1 Omega needs nothing beyond E1: finish it on the side stream
    if (cudaEventRecord(side.e1, st) != cudaSuccess || cudaStreamWaitEvent(side.st, side.e1, 0) != cudaSuccess)
      return HBS_ERR_CUDA;
    HBS_TRY(gemm(geo, dfix(r), dfix(s), drows(), r, s, E1, Om, lift_y, 0, prs, 0, s, false, -1.0, 1.0,
                 op(lift_y, 0, prs, 0, s, false, false), side.st));
    if (cudaEventRecord(side.join, side.st) != cudaSuccess) return HBS_ERR_CUDA;
  }
  HBS_TRY(gemm(geo, dfix(r), drows(), drows(), r, nr, Ut, Xn, w.M4, 0, rs, 0, nr, false, 1.0, -1.0, E1, st));
  HBS_TRY(gemm(geo, drows(), drows(), dfix(r), nr, nr, Un, M4, d, 0, 0, 1, 0, true, -1.0, 1.0, Xn, st));
  g_timer.mark();

  if (lift_omega) {
    // Parent quadruple rows of child b: [b*r, (b+1)*r)  (compress.py:209-227)
    const BOperand Dt = op(d, 0, 0, 1, 0, true, true);
    // U^T D = E1 from the discrepancy algebra (U^T U = I); V^T D^T directly
    const BOperand E2 = op(w.E2, 0, rs, 0, nr, false, false);
    HBS_TRY(gemm(geo, dfix(r), drows(), drows(), r, nr, Vt, Dt, w.E2, 0, rs, 0, nr, false, 1.0, 0.0, none, st));
    if (overlap) {
      if (cudaStreamWaitEvent(st, side.join, 0) != cudaSuccess) return HBS_ERR_CUDA;
    } else {
      HBS_TRY(lift_base());
      HBS_TRY(gemm(geo, dfix(r), dfix(s), drows(), r, s, E1, Om, lift_y, 0, prs, 0, s, false, -1.0, 1.0,
                   op(lift_y, 0, prs, 0, s, false, false), st));
    }
    HBS_TRY(gemm(geo, dfix(r), dfix(s), drows(), r, s, E2, Ps, lift_z, 0, prs, 0, s, false, -1.0, 1.0,
                 op(lift_z, 0, prs, 0, s, false, false), st));
  }
  g_timer.mark();
  return HBS_OK;
}

unsigned long long hbs_launch_counter(void) { return g_launches.load(); }

void hbs_level_hint(int min_rows) { g_min_rows_hint = min_rows; }

int hbs_compress_level_profiled(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows,
                                int s, int r, double tol, const double* omega, const double* psi,
                                const double* y, const double* z, double* u, double* v, double* d,
                                double* lift_omega, double* lift_psi, double* lift_y, double* lift_z,
                                void* workspace, size_t workspace_bytes, int32_t* status, void* stream,
                                float* phase_ms) {
  g_timer.start(static_cast<cudaStream_t>(stream));
  const int rc = hbs_compress_level(nbox, row_begin, sq_off, max_rows, s, r, tol, omega, psi, y, z, u, v, d,
                                    lift_omega, lift_psi, lift_y, lift_z, workspace, workspace_bytes, status,
                                    stream);
  g_timer.finish(phase_ms, 6);
  return rc;
}

int hbs_probe_qr(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows, int s,
                 double tol, const double* omega, double* vt, double* r, double* tau, double* t, double* rinv,
                 double* scratch, int32_t* status, void* stream) {
  if (nbox < 1 || max_rows < 1 || s < max_rows) return HBS_ERR_DIMENSION;
  if (s > 512) return HBS_ERR_UNSUPPORTED;
  const LevelGeo geo{row_begin, sq_off, nbox};
  const int nr = max_rows, npanel = (nr + kNB - 1) / kNB;
  GeqrfArgs g;
  std::memset(&g, 0, sizeof(g));
  g.geo = geo; g.mode = kGeqrfFactor;
  g.m_fixed = s; g.m_is_rows = 0; g.n_fixed = 0; g.n_is_rows = 1;
  g.m_max = s; g.n_max = nr; g.tol = tol; g.gscratch = scratch;
  GeqrfSide& S = g.side[0];
  S.src = omega; S.src_c_rb = s; S.src_c_b = 0; S.src_rs = 1; S.src_cs = s;
  S.vt = vt; S.vt_stride = (int64_t)nr * s; S.ldvt = s;
  S.r = r; S.r_stride = (int64_t)nr * nr; S.ldr = nr;
  S.tau = tau; S.tau_stride = nr;
  S.t = t; S.t_stride = (int64_t)npanel * kNB * kNB;
  S.rinv = rinv; S.rinv_stride = (int64_t)npanel * kNB * kNB;
  S.status = status;
  return launch_hqr(g, 1, static_cast<cudaStream_t>(stream));
}

int hbs_gram_probe_factor(int64_t nbox, const int64_t* row_begin, int max_rows, int s, int r,
                          const double* omega, double* fac, double* t, int32_t* flag, int32_t* status,
                          void* stream) {
  if (nbox < 1 || max_rows < 1 || s < max_rows || !flag) return HBS_ERR_DIMENSION;
  if (!gram_fits(s, max_rows, r)) return HBS_ERR_UNSUPPORTED;
  GramArgs ga;
  std::memset(&ga, 0, sizeof(ga));
  ga.geo = LevelGeo{row_begin, nullptr, nbox};
  ga.s = s; ga.r = r; ga.flag = flag;
  GramSide& G = ga.side[0];
  G.om = omega; G.om_c_rb = s;
  G.fac = fac; G.fac_stride = (int64_t)max_rows * s;
  G.t = t; G.t_stride = (int64_t)((max_rows + kNB - 1) / kNB) * kNB * kNB;
  G.status = status;
  return gram_v3() ? launch_gram(ga, 1, static_cast<cudaStream_t>(stream))
                   : launch_gram_tm(ga, 1, static_cast<cudaStream_t>(stream));
}

int hbs_basis_qr(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows, int r,
                 const double* b, double* q, double* scratch, void* stream) {
  if (nbox < 1 || max_rows < r || r < 1) return HBS_ERR_DIMENSION;
  if (max_rows > 512) return HBS_ERR_UNSUPPORTED;
  GeqrfArgs g;
  std::memset(&g, 0, sizeof(g));
  g.geo = LevelGeo{row_begin, sq_off, nbox}; g.mode = kGeqrfOrtho;
  g.m_fixed = 0; g.m_is_rows = 1; g.n_fixed = r; g.n_is_rows = 0;
  g.m_max = max_rows; g.n_max = r; g.gscratch = scratch;
  for (int sd = 0; sd < 1; ++sd) {
    GeqrfSide& S = g.side[sd];
    S.src = b; S.src_c_rb = r; S.src_c_b = 0; S.src_rs = r; S.src_cs = 1;
    S.q = q; S.q_c_rb = r; S.q_c_b = 0; S.ldq = r;
  }
  return launch_hqr(g, 1, static_cast<cudaStream_t>(stream));
}

int hbs_basis_orth(int64_t nbox, const int64_t* row_begin, const int64_t* sq_off, int max_rows, int r,
                   const double* b, double* q, int32_t* flags, double* scratch, void* stream) {
  if (nbox < 1 || max_rows < r || r < 1 || !flags) return HBS_ERR_DIMENSION;
  if (!cholqr_fits(max_rows, r)) return HBS_ERR_UNSUPPORTED;
  GeqrfArgs g;
  std::memset(&g, 0, sizeof(g));
  g.geo = LevelGeo{row_begin, sq_off, nbox}; g.mode = kGeqrfOrtho;
  g.m_fixed = 0; g.m_is_rows = 1; g.n_fixed = r; g.n_is_rows = 0;
  g.m_max = max_rows; g.n_max = r; g.gscratch = scratch;
  GeqrfSide& S = g.side[0];
  S.src = b; S.src_c_rb = r; S.src_c_b = 0; S.src_rs = r; S.src_cs = 1;
  S.q = q; S.q_c_rb = r; S.q_c_b = 0; S.ldq = r;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HBS_TRY(launch_cholqr(g, 1, flags, st));
  g.only = flags;
  return launch_hqr(g, 1, st);
}

int hbs_basis_qr_scratch_bytes(int64_t nbox, int max_rows, int r, size_t* bytes) {
  if (!bytes) return HBS_ERR_DIMENSION;
  *bytes = hqr_fits_smem(max_rows, r, kGeqrfOrtho) ? 0 : hqr_scratch_doubles(max_rows, r, nbox) * sizeof(double);
  return HBS_OK;
}

int hbs_probe_qr_scratch_bytes(int64_t nbox, int max_rows, int s, size_t* bytes) {
  if (!bytes) return HBS_ERR_DIMENSION;
  *bytes = hqr_fits_smem(s, max_rows, kGeqrfFactor) ? 0 : hqr_scratch_doubles(s, max_rows, nbox) * sizeof(double);
  return HBS_OK;
}

int hbs_root_workspace_bytes(int rows, int s, size_t* bytes) {
  if (rows < 1 || s < 1 || !bytes) return HBS_ERR_DIMENSION;
  Carver c{nullptr};
  LevelWs w;
  *bytes = carve_level(c, w, 1, rows, s, 1, true);
  return HBS_OK;
}

int hbs_compress_root(const int64_t* row_begin, const int64_t* sq_off, int rows, int s, double tol,
                      const double* omega, const double* y, double* root, void* workspace,
                      size_t workspace_bytes, int32_t* status, void* stream) {
  g_level_uniform = 0;   // (a level hint never applies to the root call)
  g_min_rows_hint = 0;
  if (rows < 1 || s < rows) return HBS_ERR_DIMENSION;
  if (s > 512) return HBS_ERR_UNSUPPORTED;
  Carver c{static_cast<char*>(workspace)};
  LevelWs w;
  if (carve_level(c, w, 1, rows, s, 1, true) > workspace_bytes) return HBS_ERR_WORKSPACE;
  const LevelGeo geo{row_begin, sq_off, 1};
  return factor_and_solve(geo, rows, s, 1, tol, 1, omega, nullptr, y, nullptr, w, status, root,
                          static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------------ samplers
int hbs_apply_up(int level_hi, int level_lo, int r, int64_t c, const int64_t* nbox,
                 const int64_t* const* row_begin, const int64_t* const* sq_off, const double* const* basis,
                 const double* q, double* const* qhat, void* stream) {
  if (level_lo < 0 || level_hi < level_lo || r < 1 || c < 1 || c > (1 << 30)) return HBS_ERR_DIMENSION;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cc = (int)c;
  const BOperand none = op(nullptr, 0, 0, 0, 0, false, false);
  for (int l = level_hi; l >= level_lo; --l) {
    const LevelGeo geo{row_begin[l], sq_off[l], nbox[l]};
    const double* src = (l == level_hi) ? q : qhat[l + 1];
    HBS_TRY(gemm(geo, dfix(r), dfix(cc), drows(), r, cc, op(basis[l], r, 0, 0, r, false, true),
                 op(src, cc, 0, 0, cc, false, false), qhat[l], 0, (int64_t)r * cc, 0, cc, false, 1.0, 0.0, none, st));
  }
  return HBS_OK;
}

int hbs_apply_root(int r, int64_t c, const double* root, int transpose, const double* qhat1, double* uhat1,
                   void* stream) {
  if (r < 1 || c < 1 || c > (1 << 30)) return HBS_ERR_DIMENSION;
  const LevelGeo geo{nullptr, nullptr, 1};
  const int cc = (int)c;
  return gemm(geo, dfix(2 * r), dfix(cc), dfix(2 * r), 2 * r, cc, op(root, 0, 0, 0, 2 * r, false, transpose != 0),
              op(qhat1, 0, 0, 0, cc, false, false), uhat1, 0, 0, 0, cc, false, 1.0, 0.0,
              op(nullptr, 0, 0, 0, 0, false, false), static_cast<cudaStream_t>(stream));
}

int hbs_apply_down(int level_lo, int level_hi, int r, int64_t c, const int64_t* nbox,
                   const int64_t* const* row_begin, const int64_t* const* sq_off, int max_rows_hi,
                   const double* const* basis, const double* const* d, int transpose_d, double* const* uhat,
                   const double* const* qhat, const double* q, double* out, void* stream) {
  if (level_lo < 0 || level_hi < level_lo || r < 1 || c < 1 || c > (1 << 30) || max_rows_hi < 1)
    return HBS_ERR_DIMENSION;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cc = (int)c;
  const BOperand none = op(nullptr, 0, 0, 0, 0, false, false);
  for (int l = level_lo; l <= level_hi; ++l) {
    const LevelGeo geo{row_begin[l], sq_off[l], nbox[l]};
    const bool last = (l == level_hi);
    double* dst = last ? out : uhat[l + 1];
    const double* rhs = last ? q : qhat[l + 1];
    const int mmax = last ? max_rows_hi : 2 * r;
    HBS_TRY(gemm(geo, drows(), dfix(cc), dfix(r), mmax, cc, op(basis[l], r, 0, 0, r, false, false),
                 op(uhat[l], 0, (int64_t)r * cc, 0, cc, false, false), dst, cc, 0, 0, cc, false, 1.0, 0.0, none, st));
    HBS_TRY(gemm(geo, drows(), dfix(cc), drows(), mmax, cc, op(d[l], 0, 0, 1, 0, true, transpose_d != 0),
                 op(rhs, cc, 0, 0, cc, false, false), dst, cc, 0, 0, cc, false, 1.0, 1.0,
                 op(dst, cc, 0, 0, cc, false, false), st));
  }
  return HBS_OK;
}

int hbs_apply_workspace_bytes(int depth, int r, int64_t c, size_t* bytes) {
  if (depth < 1 || r < 1 || c < 1 || !bytes) return HBS_ERR_DIMENSION;
  // qhat and uhat for every level: sum_l 2^l r c, twice.
  const size_t per = ((size_t(1) << (depth + 1)) - 2) * (size_t)r * (size_t)c;
  *bytes = 2 * per * sizeof(double) + 2 * kAlign;
  return HBS_OK;
}

int hbs_apply(int depth, int r, int64_t n, int64_t c, const int64_t* const* row_begin,
              const int64_t* const* sq_off, const double* const* u, const double* const* v,
              const double* const* d, const double* root, const double* q, double* out, int transpose,
              void* workspace, size_t workspace_bytes, void* stream) {
  if (depth < 1 || depth > 60 || r < 1 || n < 2 || c < 1) return HBS_ERR_DIMENSION;
  if (c > (1 << 30)) return HBS_ERR_UNSUPPORTED;
  size_t need;
  hbs_apply_workspace_bytes(depth, r, c, &need);
  if (need > workspace_bytes) return HBS_ERR_WORKSPACE;
  double* base = static_cast<double*>(workspace);
  double* qhat[64];
  double* uhat[64];
  int64_t nbox[64];
  size_t off = 0;
  for (int l = 1; l <= depth; ++l) { qhat[l] = base + off; off += ((size_t)1 << l) * r * c; }
  for (int l = 1; l <= depth; ++l) { uhat[l] = base + off; off += ((size_t)1 << l) * r * c; }
  for (int l = 0; l <= depth; ++l) nbox[l] = (int64_t)1 << l;
  const int leaf_max = (int)((n + ((int64_t)1 << depth) - 1) >> depth);
  const double* const* up = transpose ? u : v;
  const double* const* down = transpose ? v : u;
  HBS_TRY(hbs_apply_up(depth, 1, r, c, nbox, row_begin, sq_off, up, q, qhat, stream));
  HBS_TRY(hbs_apply_root(r, c, root, transpose, qhat[1], uhat[1], stream));
  return hbs_apply_down(1, depth, r, c, nbox, row_begin, sq_off, leaf_max, down, d, transpose, uhat, qhat, q, out,
                        stream);
}

int hbs_dense_apply(int64_t n, int64_t c, const double* a, const double* q, double* out, int transpose,
                    void* stream) {
  if (n < 1 || c < 1) return HBS_ERR_DIMENSION;
  if (n > (1 << 30) || c > (1 << 30)) return HBS_ERR_UNSUPPORTED;
  // single "box" spanning all rows: geometry {0, n}
  static_assert(sizeof(int64_t) == 8, "");
  const int nn = (int)n, cc = (int)c;
  BgemmArgs g;
  std::memset(&g, 0, sizeof(g));
  g.geo = LevelGeo{nullptr, nullptr, 1};
  g.M = dfix(nn); g.N = dfix(cc); g.K = dfix(nn); g.M_max = nn; g.N_max = cc;
  g.A = op(a, 0, 0, 0, nn, false, transpose != 0);
  g.B = op(q, 0, 0, 0, cc, false, false);
  g.C0 = op(nullptr, 0, 0, 0, 0, false, false);
  g.C = out; g.ldc_fixed = cc; g.alpha = 1.0; g.beta = 0.0;
  return launch_bgemm(g, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
