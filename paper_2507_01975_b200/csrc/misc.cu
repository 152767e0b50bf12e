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

// NEXT-3 ring of the last k_c step inputs, [B][k_c][2][N][N]: slot s <- slot s+1, the newest slot
// <- u.  Each thread owns one float4 index of an element's field across all slots, so the shift
// reads every slot before overwriting it.
__global__ void hist_push_kernel(float4* __restrict__ hist, const float4* __restrict__ u, int B, int kc, size_t f4) {
  const size_t total = (size_t)B * f4;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const size_t b = t / f4, i = t - b * f4;
    float4* h = hist + b * kc * f4 + i;
    for (int s = 0; s + 1 < kc; ++s) h[s * f4] = h[(s + 1) * f4];
    h[(size_t)(kc - 1) * f4] = u[t];
  }
}

cudaError_t launch_hist_push(float* hist, const float* u, int B, int kc, size_t field_per_elem, cudaStream_t st) {
  const size_t f4 = field_per_elem / 4, total = (size_t)B * f4;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  hist_push_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<float4*>(hist), reinterpret_cast<const float4*>(u), B, kc,
                                          f4);
  return cudaGetLastError();
}

cudaError_t launch_nonfinite_check(const float* u, size_t n, int step, int* flag, cudaStream_t st) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  nonfinite_check_kernel<<<blocks, 256, 0, st>>>(u, n, step, flag);
  return cudaGetLastError();
}

// Block-mean downsampling fine -> coarse (the paper's training data are
// fine-grid DNS fields "downsampled ... to the desired coarse grid resolutions", P:141, P:344,
// Table S1; finite-volume reading: a coarse cell holds the mean of the f x f fine cells it
// covers).  coarse[p][J][I] = mean_{dj,di < f} fine[p][J f + dj][I f + di] for every plane p.
__global__ void downsample_kernel(const float* __restrict__ fine, int nf, int f, size_t nplanes,
                                  float* __restrict__ coarse) {
  const int nc = nf / f;
  const size_t total = nplanes * nc * nc;
  const float inv = 1.0f / ((float)f * (float)f);
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const int I = (int)(t % nc);
    const size_t r = t / nc;
    const int J = (int)(r % nc);
    const size_t pl = r / nc;
    const float* src = fine + (pl * nf + (size_t)J * f) * nf + (size_t)I * f;
    float acc = 0.f;
    for (int dj = 0; dj < f; ++dj)
      for (int di = 0; di < f; ++di) acc += src[(size_t)dj * nf + di];
    coarse[t] = acc * inv;
  }
}

cudaError_t launch_downsample(const float* fine, int nf, int f, size_t nplanes, float* coarse, cudaStream_t st) {
  const size_t total = nplanes * (size_t)(nf / f) * (nf / f);
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  downsample_kernel<<<blocks, 256, 0, st>>>(fine, nf, f, nplanes, coarse);
  return cudaGetLastError();
}

}  // namespace ld
