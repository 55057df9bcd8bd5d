// layout.cuh — rhs-major <-> index-major vectors of the public apply calls
// (include/pmmf_b200.h stores rhs r at [r*n, (r+1)*n); the kernels keep
// v[i * nrhs + r] so a rotation touches contiguous rhs lanes).
#pragma once

#include "common.cuh"

namespace pmmf_b200 {
namespace {

// out (cols x rows, row-major) = in (rows x cols, row-major)^T through a
// 32 x 33 shared tile: both sides coalesced.
__global__ void k_transpose_tiled(const double* __restrict__ in, double* __restrict__ out, i64 rows, i64 cols) {
  __shared__ double t[32][33];
  const i64 c0 = static_cast<i64>(blockIdx.x) * 32, r0 = static_cast<i64>(blockIdx.y) * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const i64 r = r0 + y, c = c0 + threadIdx.x;
    if (r < rows && c < cols) t[y][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const i64 c = c0 + y, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = t[threadIdx.x][y];
  }
}

inline void transpose_tiled(const double* in, double* out, i64 rows, i64 cols, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  dim3 g(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32)), b(32, 8);
  k_transpose_tiled<<<g, b, 0, s>>>(in, out, rows, cols);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  PMMF_CUDA(cudaGetLastError());
}
// rhs-major (nrhs x n) -> index-major (n x nrhs) and back
inline void to_index_major(const double* in, double* out, i64 n, int nrhs, cudaStream_t s) {
  transpose_tiled(in, out, nrhs, n, s);
}
inline void to_rhs_major(const double* in, double* out, i64 n, int nrhs, cudaStream_t s) {
  transpose_tiled(in, out, n, nrhs, s);
}

}  // namespace
}  // namespace pmmf_b200
