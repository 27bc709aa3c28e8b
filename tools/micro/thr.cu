// Single-warp issue-rate micro-benchmark: 8 independent chains per op
// (development tool).
#include <cstdio>
template <int OP>
__global__ void thr(double* out, long long* cyc, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) a[i] = fma(a[i], b, c);
        if (OP == 1) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 3));
        if (OP == 2) a[i] = __int_as_float(__shfl_xor_sync(0xffffffffu, __float_as_int((float)a[i]), 1 + (i & 3)));
        if (OP == 3) a[i] = rsqrt(a[i] + 2.0);
        if (OP == 4) a[i] = a[i] * 0.5 + __shfl_sync(0xffffffffu, a[i], i);
      }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[threadIdx.x] = s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  const char* nm[5] = {"DFMA", "SHFL64 (2 instr)", "SHFL32", "rsqrt f64", "SHFL64.IDX+DFMA"};
  for (int op = 0; op < 5; ++op) {
    void (*k)(double*, long long*, int) = op == 0 ? thr<0> : op == 1 ? thr<1> : op == 2 ? thr<2> : op == 3 ? thr<3> : thr<4>;
    for (int nw : {32, 128}) {
      k<<<1, nw>>>(o, c, 64);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%-18s threads %3d: %.2f cycles per warp-op\n", nm[op], nw, h / (64.0 * 32));
    }
  }
  return 0;
}
