// copy_microbench.cu -- global(L2-resident) -> shared copy throughput per SM on B200, for the
// operand producer of the tcgen05 conv.  Measurement aid only.
//   mode 0: cp.async 16 B, a warp covers 512 contiguous bytes
//   mode 1: cp.async.bulk, 160-B runs (one lane per run)
//   mode 2: cp.async.bulk, 2-KB runs
//   mode 3: TMA tensor 3D box {4 floats, 10 rows, 6 cols} per op (1920 B)   [strip box]
//   mode 4: TMA tensor 5D box with an overlapping "strip" dimension (8 strips x 6 cols x 2 q) (15 KB)
// All 148 SMs, 1 CTA each, each CTA streams `iters` stages of ~30 KB into a 4-deep ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o copy_mb copy_microbench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su32(b)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(n), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma5(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4,
                                     uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(bar))
      : "memory");
}

constexpr int STAGE = 32768, NST = 4;

__global__ void __launch_bounds__(128, 1) kern(int mode, int iters, const uint8_t* src, size_t src_bytes,
                                               const __grid_constant__ CUtensorMap m3,
                                               const __grid_constant__ CUtensorMap m5, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NST];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(full + s, mode == 0 ? 128 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // each CTA reads its own ~1 MB region (L2 resident across the 148 CTAs: ~150 MB? no: wrap in 32 MB)
  const size_t region = (size_t)blockIdx.x * 196608 % (src_bytes - 2 * 1048576);
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    const int slot = k % NST;
    if (k >= NST) mbar_wait(full + slot, ((k / NST) - 1) & 1);   // previous use of the slot landed
    __syncthreads();
    uint8_t* st = sm + slot * STAGE;
    const uint8_t* g = src + region + (size_t)(k % 16) * 65536;
    if (mode == 0) {
      for (int i = tid; i < STAGE / 16; i += 128)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(st + i * 16)), "l"(g + i * 16) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(full + slot)) : "memory");
    } else if (warp == 0) {
      if (lane == 0) mbar_expect(full + slot, mode == 4 ? 15360 * 2 : (mode == 3 ? 32 * 960 : (mode == 1 ? 204 * 160 : STAGE)));
      __syncwarp();
      if (mode == 1) {
        for (int i = lane; i < 204; i += 32) bulk(st + i * 160, g + (size_t)i * 4096, 160, full + slot);
      } else if (mode == 2) {
        for (int i = lane; i < STAGE / 2048; i += 32) bulk(st + i * 2048, g + (size_t)i * 4096, 2048, full + slot);
      } else if (mode == 3) {
        tma3(st + lane * 1024, &m3, 0, (lane * 8) % 504, (k * 4 + lane) % 58, full + slot);
      } else {
        if (lane < 2) tma5(st + lane * 15360, &m5, 0, 0, (k * 7 + lane * 6) % 58, 0, 0, full + slot);
      }
    }
  }
  for (int k = iters - NST; k < iters; ++k) mbar_wait(full + k % NST, (k / NST) & 1);
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  const size_t bytes = 64ull << 20;
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  // tensor maps over a float buffer viewed as [cols 64][rows 514][4 floats]  (3D strip box)
  CUtensorMap m3, m5;
  {
    cuuint64_t dims[3] = {4, 514, 64};
    cuuint64_t strides[2] = {16, 514 * 16};
    cuuint32_t box[3] = {4, 10, 6};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, src, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode 3d: %d\n", (int)r);
  }
  {
    // 5D with overlapping strip dim: e(4) r(10, 16 B) x(66 cols, 1056 B... stride 66*16) q(2) yb(8, stride 128 B)
    cuuint64_t dims[5] = {4, 10, 66, 2, 8};
    cuuint64_t strides[4] = {16, 66 * 16, 66 * 66 * 16, 128};
    cuuint32_t box[5] = {4, 10, 6, 2, 8};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m5, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, src, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode 5d overlapping: %d\n", (int)r);
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE);
  const char* names[5] = {"cp.async 16B coalesced", "bulk 160B runs", "bulk 2KB runs", "TMA 3D strip box 960B x32",
                          "TMA 5D 8-strip box 15KB"};
  for (int mode = 0; mode < 5; ++mode) {
    const int iters = 400;
    kern<<<148, 128, NST * STAGE>>>(mode, iters, src, bytes, m3, m5, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double per_stage = mode == 4 ? 30720.0 : (mode == 3 ? 30720.0 : (mode == 1 ? 204 * 160.0 : (double)STAGE));
    printf("%-28s %7.1f cycles/stage  %6.1f B/clk/SM  (%s)\n", names[mode], avg / iters, per_stage * iters / avg,
           cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
