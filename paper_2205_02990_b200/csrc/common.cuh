// Shared device helpers for the HBS compress-from-samples kernels (sm_100a, fp64).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define HBS_DEV __device__ __forceinline__

namespace hbs {

// Per-box status written by the kernels (0 = ok).  The host maps a nonzero
// status onto IllConditionedProbeError(node_id, level) -- errors.py:12-19.
enum BoxStatus : int32_t { kBoxOk = 0, kBoxIllConditioned = 1 };

// Panel width of the blocked Householder representation (compact WY T blocks,
// diagonal-block inverses of R).
constexpr int kNB = 32;

// Row geometry of one tree level: box b owns rows [row_begin[b], row_begin[b+1]).
struct LevelGeo {
  const int64_t* row_begin;  // nbox + 1
  const int64_t* sq_off;     // nbox + 1, prefix sums of rows^2 (packed D blocks)
  int64_t nbox;
};

HBS_DEV int box_rows(const LevelGeo& g, int64_t b) {
  return static_cast<int>(g.row_begin[b + 1] - g.row_begin[b]);
}

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).
// Fragment ownership (lane = 4*g + t): A(g, t); B(t, g); C(g, 2t), C(g, 2t+1).
HBS_DEV void dmma8x8x4(double& c0, double& c1, double a, double b) {
  // not volatile: pure register semantics, so the compiler may hoist the
  // operand loads of later k-steps above earlier MMAs.
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Warp index broadcast from lane 0: provably warp-uniform to the compiler, so
// branches on it do not force WARPSYNC.COLLECTIVE around later shuffles.
HBS_DEV int uniform_warp(int w) { return __shfl_sync(0xffffffffu, w, 0); }

HBS_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

HBS_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

HBS_DEV double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Leading dimension (in doubles) for an smem tile whose rows hold `cols`
// doubles: rounded up so ld % 16 == 4, which makes every m8n8k4 fragment load
// (row- or column-ordered) bank-conflict free.

inline __host__ __device__ int frag_ld(int cols) {
  int ld = (cols + 3) & ~3;
  while ((ld & 15) != 4) ld += 4;
  return ld;
}

inline __host__ __device__ int round_up(int x, int m) { return (x + m - 1) / m * m; }
// compile-time forms of round_up / frag_ld (template-specialised kernels)
constexpr int round_up_c(int x, int m) { return (x + m - 1) / m * m; }
constexpr int frag_ld_c(int cols) {
  int ld = (cols + 3) & ~3;
  while ((ld & 15) != 4) ld += 4;
  return ld;
}

// mbarrier helpers (shared::cta).
HBS_DEV void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
HBS_DEV void mbar_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(a) : "memory");
}
HBS_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}
// Same, with a suspend-time hint: the waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-issuing try_wait, leaving the
// issue slots of its SM sub-partition to the warps doing the work.
HBS_DEV void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity), "r"(1000000u) : "memory");
}

// Warp-uniform wait: one lane spins (acquire), then __syncwarp re-converges the
// warp and orders the other lanes' later reads after the acquire.  Waiting in
// every lane leaves the compiler unable to prove convergence afterwards, and
// it then emits WARPSYNC.COLLECTIVE sequences around every later shuffle.
HBS_DEV void mbar_wait_warp(uint64_t* bar, unsigned parity) {
  if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
  __syncwarp();
}

// TMA bulk copy global -> shared with mbarrier completion (cp.async.bulk).
HBS_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
HBS_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}

// cp.async (LDGSTS) helpers: 8-byte element copies with zero fill.
HBS_DEV void cp_async8(double* dst, const double* src, bool pred) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(src), "r"(pred ? 8 : 0));
}
HBS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
HBS_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// C-fragment (row g, cols 2t, 2t+1 of 8x8 block f) -> A-fragment (row g, col
// kk + t) of the same row block, for k-step kk of a K = 8*NF operand held as
// NF C-fragments.  Pure quad shuffles (lanes sharing g).
template <int NF>
HBS_DEV double cfrag_to_afrag(const double (&acc)[NF][2], int kk, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const int col = (kk & 7) + t;
  const int src = 4 * g + (col >> 1);
  const double v0 = __shfl_sync(0xffffffffu, acc[kk >> 3][0], src);
  const double v1 = __shfl_sync(0xffffffffu, acc[kk >> 3][1], src);
  return (col & 1) ? v1 : v0;
}

// ---------------------------------------------------------------- TMEM (tcgen05) as an fp64 scratchpad
// fp64 element (lane i, column c) occupies 32-bit TMEM columns 2c (low word)
// and 2c + 1 (high word).  A .16x256b access by a warp covers 16 lanes
// (rows) x 4 fp64 columns per repetition; thread (g = lane/4, t = lane%4)
// holds (row g, col c0 + t) and (row g + 8, col c0 + t) -- the m8n8k4
// A-fragment layout of two 8-row groups.  Warp w may only touch lanes
// 32 (w % 4) .. 32 (w % 4) + 31.
HBS_DEV void tm_alloc512(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
      static_cast<unsigned>(__cvta_generic_to_shared(slot))));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
// Runtime column count (a power of two in 32 .. 512): a CTA that needs fewer
// than 512 columns leaves the rest to the other CTAs resident on its SM.
HBS_DEV void tm_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
      static_cast<unsigned>(__cvta_generic_to_shared(slot))), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
HBS_DEV void tm_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols));
}
HBS_DEV uint32_t tm_pow2_cols(int need) {
  uint32_t c = 32;
  while ((int)c < need) c <<= 1;
  return c;
}
HBS_DEV void tm_dealloc512(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr));
}
HBS_DEV void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
HBS_DEV void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
HBS_DEV void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// 16 columns (4 repetitions): v[rep][h] = (row g + 8h, col c0 + 4 rep + t)
HBS_DEV void tm_ld16(uint32_t taddr, double (&v)[4][2]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[q][0] = __hiloint2double((int)r[4 * q + 1], (int)r[4 * q + 0]);
    v[q][1] = __hiloint2double((int)r[4 * q + 3], (int)r[4 * q + 2]);
  }
}
HBS_DEV void tm_st16(uint32_t taddr, const double (&v)[4][2]) {
  uint32_t r[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    r[4 * q + 0] = (uint32_t)__double2loint(v[q][0]);
    r[4 * q + 1] = (uint32_t)__double2hiint(v[q][0]);
    r[4 * q + 2] = (uint32_t)__double2loint(v[q][1]);
    r[4 * q + 3] = (uint32_t)__double2hiint(v[q][1]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

}  // namespace hbs
