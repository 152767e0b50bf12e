// store_microbench.cu -- global store throughput per SM (STG.128, each warp instruction writing
// 512 contiguous bytes), L2-resident target, 148 CTAs x W warps.  Measurement aid only.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void st128(float4* buf, size_t per_cta_f4, int reps, long long* out) {
  float4* b = buf + (size_t)blockIdx.x * per_cta_f4;
  const float4 v = make_float4(threadIdx.x, 1.f, 2.f, 3.f);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < per_cta_f4; i += blockDim.x) b[i] = v;
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  const size_t per_cta = 128 * 1024;   // bytes per CTA per rep (one conv tile's output)
  float4* buf;
  cudaMalloc(&buf, per_cta * 148);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int threads : {128, 256, 512, 1024}) {
    const int reps = 50;
    st128<<<148, threads>>>(buf, per_cta / 16, reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("threads %4d: %.1f B/clk/SM (%s)\n", threads, per_cta * (double)reps / avg, cudaGetErrorString(e));
  }
  return 0;
}
