// Synthetic operator generator for config 3:
// points on the ellipse (cos t, 0.5 sin t), t_i = 2 pi i / n,
// A_ij = log|x_i - x_j| (i != j), A_ii = 1.  Row-major, rows [row0, row0+rows).
#include <cmath>
#include "../../include/hbs_b200.h"
#include "kernels.h"

namespace hbs {
__global__ void fill_log_kernel(int64_t n, int64_t row0, int64_t rows, double* a) {
  const int64_t total = rows * n;
  const double h = 2.0 * 3.14159265358979323846 / (double)n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row0 + e / n, j = e % n;
    double v = 1.0;
    if (i != j) {
      double si, ci, sj, cj;
      sincos(h * (double)i, &si, &ci);
      sincos(h * (double)j, &sj, &cj);
      const double dx = ci - cj, dy = 0.5 * (si - sj);
      v = log(sqrt(dx * dx + dy * dy));
    }
    a[e] = v;
  }
}
}  // namespace hbs

extern "C" int hbs_fill_log_kernel(int64_t n, int64_t row0, int64_t rows, double* a, void* stream) {
  if (n < 1 || rows < 0 || row0 < 0 || row0 + rows > n) return HBS_ERR_DIMENSION;
  if (rows == 0) return HBS_OK;
  hbs::fill_log_kernel<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(n, row0, rows, a);
  hbs::note_launch();
  return cudaGetLastError() == cudaSuccess ? HBS_OK : HBS_ERR_CUDA;
}
