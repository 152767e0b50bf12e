// misc.cu -- finiteness check (SURVEY.md §5 failure detection; SPEC-style "simulation
// divergence" error naming the step).
#include "common.cuh"

namespace ld {

__global__ void nonfinite_check_kernel(const float* __restrict__ u, size_t n, int step, int* flag) {
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    bad |= !isfinite(u[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(flag, step);
}

cudaError_t launch_nonfinite_check(const float* u, size_t n, int step, int* flag, cudaStream_t st) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  nonfinite_check_kernel<<<blocks, 256, 0, st>>>(u, n, step, flag);
  return cudaGetLastError();
}

}  // namespace ld
