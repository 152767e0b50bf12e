// slab_kernels.cu -- row copies for the slab decomposition's halo exchanges (SURVEY.md §8e
// PAR-2): pack own rows into contiguous send buffers, unpack received rows into the extended
// stage field.  One launch moves the same row range of every plane of a batch.
#include "common.cuh"

namespace ld {

// plane pl (pl in [0, nplanes)) of the source is  src + (pl * s_step + s_off) * s_rows * N,
// its row y of interest is s_row0 + y;  the destination likewise.  Rows y in [0, count).
__global__ void __launch_bounds__(256)
copy_rows_kernel(float* __restrict__ dst, int d_step, int d_off, int d_rows, int d_row0, const float* __restrict__ src,
                 int s_step, int s_off, int s_rows, int s_row0, int nplanes, int count, int N) {
  const size_t per_plane = (size_t)count * N / 4;   // float4 units (N % 4 == 0)
  const size_t total = per_plane * nplanes;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const int pl = (int)(t / per_plane);
    const size_t k = (t - (size_t)pl * per_plane) * 4;
    const int y = (int)(k / N), x = (int)(k - (size_t)y * N);
    const float4 v = *reinterpret_cast<const float4*>(src + ((size_t)(pl * s_step + s_off) * s_rows + s_row0 + y) * N + x);
    *reinterpret_cast<float4*>(dst + ((size_t)(pl * d_step + d_off) * d_rows + d_row0 + y) * N + x) = v;
  }
}

cudaError_t launch_copy_rows(float* dst, int d_step, int d_off, int d_rows, int d_row0, const float* src, int s_step,
                             int s_off, int s_rows, int s_row0, int nplanes, int count, int N, cudaStream_t st) {
  if (count <= 0 || nplanes <= 0) return cudaSuccess;
  const size_t total = (size_t)nplanes * count * N / 4;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  copy_rows_kernel<<<blocks, 256, 0, st>>>(dst, d_step, d_off, d_rows, d_row0, src, s_step, s_off, s_rows, s_row0,
                                           nplanes, count, N);
  return cudaGetLastError();
}

}  // namespace ld
