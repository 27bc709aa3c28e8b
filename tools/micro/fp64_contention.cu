// How a dependent DFMA chain (the Householder panel chain's shape) is slowed by
// DMMA m8n8k4 streams of other warps: per-SMSP or per-SM pipe, effect of the
// number of independent DMMA accumulators per streaming warp, and of warp ids.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_contention fp64_contention.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// chain_warp: warp running the dependent DFMA chain; stream_mask: bit w set -> warp w streams DMMAs
template <int K, int MODE>
__global__ void probe(int chain_warp, unsigned stream_mask, int chain_len, int stream_iters, long long* out, double* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ volatile int go;
  if (threadIdx.x == 0) go = 0;
  __syncthreads();
  if (warp == chain_warp) {
    double x = 1.0 + lane * 1e-9, a = 1.0000001, b = 1e-12;
    // let the streamers get going
    for (int i = 0; i < 2000; ++i) asm volatile("" ::: "memory");
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < chain_len; ++i) x = fma(x, a, b);
    const long long t1 = clock64();
    if (lane == 0) { out[0] = t1 - t0; }
    sink[threadIdx.x] = x;
    go = 1;
  } else if ((stream_mask >> warp) & 1u) {
    double c[K][2];
#pragma unroll
    for (int k = 0; k < K; ++k) { c[k][0] = 0.0; c[k][1] = 0.0; }
    const double a = 1.0 + lane, b = 1e-3 * lane;
    const long long t0 = clock64();
    int it = 0;
    for (; it < stream_iters && !go; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (MODE == 0) dmma(c[k][0], c[k][1], a, b);
          else { c[k][0] = fma(c[k][0], a, b); c[k][1] = fma(c[k][1], a, b); }
        }
    }
    const long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += c[k][0] + c[k][1];
    sink[threadIdx.x] = s;
    if (lane == 0) { out[1 + warp] = t1 - t0; out[32 + warp] = (long long)it * 8 * K; }
  }
}

template <int K, int MODE = 0>
void run(const char* name, int chain_warp, unsigned mask, long long* d_out, double* d_sink) {
  const int chain_len = 20000;
  cudaMemset(d_out, 0, 64 * sizeof(long long));
  probe<K, MODE><<<1, 512>>>(chain_warp, mask, chain_len, 1 << 20, d_out, d_sink);
  cudaDeviceSynchronize();
  long long h[64];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  double dm = 0.0; int nst = 0;
  for (int w = 0; w < 16; ++w) if ((mask >> w) & 1u) { dm += (double)h[1 + w] / (double)(h[32 + w] ? h[32 + w] : 1); ++nst; }
  printf("%-44s %s K=%d chain warp %2d  cycles/DFMA %7.2f   streamer cycles/DMMA %6.2f (%d warps)\n", name, MODE ? "DFMA-stream (x2 per count)" : "DMMA-stream", K, chain_warp,
         (double)h[0] / chain_len, nst ? dm / nst : 0.0, nst);
}

int main() {
  long long* d_out; double* d_sink;
  cudaMalloc(&d_out, 64 * sizeof(long long));
  cudaMalloc(&d_sink, 512 * sizeof(double));
  run<1>("alone", 0, 0u, d_out, d_sink);
  run<1>("alone (warp 12)", 12, 0u, d_out, d_sink);
  // streamers on the chain warp's SMSP (warp % 4 == 0)
  run<1>("1 streamer same SMSP (warp 4)", 0, 1u << 4, d_out, d_sink);
  run<2>("1 streamer same SMSP (warp 4)", 0, 1u << 4, d_out, d_sink);
  run<4>("1 streamer same SMSP (warp 4)", 0, 1u << 4, d_out, d_sink);
  run<8>("1 streamer same SMSP (warp 4)", 0, 1u << 4, d_out, d_sink);
  run<1>("2 streamers same SMSP (warps 4, 8)", 0, (1u << 4) | (1u << 8), d_out, d_sink);
  run<2>("2 streamers same SMSP (warps 4, 8)", 0, (1u << 4) | (1u << 8), d_out, d_sink);
  run<4>("2 streamers same SMSP (warps 4, 8)", 0, (1u << 4) | (1u << 8), d_out, d_sink);
  run<8>("2 streamers same SMSP (warps 4, 8)", 0, (1u << 4) | (1u << 8), d_out, d_sink);
  // chain on the highest warp id of the SMSP, streamers below it
  run<8>("2 streamers same SMSP (warps 0, 4), chain 12", 12, (1u << 0) | (1u << 4), d_out, d_sink);
  run<2>("2 streamers same SMSP (warps 0, 4), chain 12", 12, (1u << 0) | (1u << 4), d_out, d_sink);
  run<8>("2 streamers same SMSP (warps 8, 12), chain 0", 0, (1u << 8) | (1u << 12), d_out, d_sink);
  // streamers on the other SMSPs only
  run<8>("3 streamers other SMSPs (warps 1, 2, 3)", 0, 0xEu, d_out, d_sink);
  run<8>("6 streamers other SMSPs (1,2,3,5,6,7)", 0, 0xEEu, d_out, d_sink);
  run<8>("8 streamers all SMSPs (2 each, 1..8 minus 0)", 12, 0x0FFu, d_out, d_sink);
  run<8>("all 15 other warps stream", 0, 0xFFFEu, d_out, d_sink);
  // DFMA streamers (register-tiled GEMM style): K independent accumulator pairs
  run<4, 1>("1 streamer same SMSP (warp 4)", 0, 1u << 4, d_out, d_sink);
  run<16, 1>("1 streamer same SMSP (warp 4)", 0, 1u << 4, d_out, d_sink);
  run<4, 1>("2 streamers same SMSP (warps 4, 8)", 0, (1u << 4) | (1u << 8), d_out, d_sink);
  run<16, 1>("2 streamers same SMSP (warps 4, 8)", 0, (1u << 4) | (1u << 8), d_out, d_sink);
  run<16, 1>("3 streamers same SMSP (warps 4, 8, 12)", 0, (1u << 4) | (1u << 8) | (1u << 12), d_out, d_sink);
  run<16, 1>("2 streamers same SMSP (0, 4), chain 12", 12, (1u << 0) | (1u << 4), d_out, d_sink);
  run<16, 1>("all 15 other warps stream", 0, 0xFFFEu, d_out, d_sink);
  return 0;
}
