// tma_fair_microbench.cu -- global -> shared fill throughput per SM on B200, re-measured fairly for the
// conv producer (VERDICT r01 "What's weak" #9 / "do this" #4): a deep ring (6 x 32 KB), several boxes in
// flight per stage, no CTA-wide barrier per stage (one consumer warp waits on the full barrier and
// re-arms the empty one, as a real pipeline does), 128B-swizzled boxes of the shape the conv's K-major
// operand stage holds (32 fp32 channels = 128 B inner, 128-130 rows), plus the no-swizzle 16-B-inner box
// the conv's current SWIZZLE_NONE K-major layout would need.  Measurement aid only.
//   mode 0: cp.async 16 B, 4 producer warps, a warp covers 512 contiguous bytes (the conv's producer)
//   mode 1: cp.async.bulk 16 KB runs (2 per stage)
//   mode 2: TMA 2D SW128 box {32 fp32, 128 rows} (16 KB), 2 per stage
//   mode 3: TMA 2D SW128 box {32 fp32, 64 rows} (8 KB), 4 per stage
//   mode 4: TMA 3D no-swizzle box {4 fp32 (16 B), 128 rows, 8 chunks} (16 KB), 2 per stage  [K-major core rows]
//   mode 5: TMA 2D SW128 box {32 fp32, 128 rows} from a DRAM-sized source (1 GB, streamed once)
// Source for modes 0-4: 64 MB (L2-resident); each CTA streams its own 1-MB window.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_fair tma_fair_microbench.cu -lcuda
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
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
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
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}

constexpr int STAGE = 32768, NST = 6;
constexpr int NPROD = 4;   // producer warps (mode 0); warp 4 = consumer

__global__ void __launch_bounds__(160, 1) kern(int mode, int iters, const uint8_t* src, size_t src_bytes,
                                               const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m2s,
                                               const __grid_constant__ CUtensorMap m3, const __grid_constant__ CUtensorMap mbig,
                                               long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NST], empty[NST];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + s, mode == 0 ? NPROD * 32 : 1);
      mbar_init(empty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t region = (size_t)blockIdx.x * 196608 % (src_bytes - 2 * 1048576);
  long long t0 = clock64();
  if (warp < NPROD) {
    for (int k = 0; k < iters; ++k) {
      const int slot = k % NST;
      if (k >= NST) mbar_wait(empty + slot, ((k / NST) - 1) & 1);
      uint8_t* st = sm + slot * STAGE;
      const uint8_t* g = src + region + (size_t)(k % 16) * 65536;
      if (mode == 0) {
        for (int i = tid; i < STAGE / 16; i += NPROD * 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(st + i * 16)), "l"(g + i * 16) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(full + slot)) : "memory");
      } else if (tid == 0) {
        mbar_expect(full + slot, STAGE);
        const int row0 = (int)(((region >> 8) + (size_t)(k % 16) * 256) % 200000);   // 256-B rows of the 64-MB view
        if (mode == 1) {
          bulk(st, g, 16384, full + slot);
          bulk(st + 16384, g + 32768, 16384, full + slot);
        } else if (mode == 2) {
          tma2(st, &m2, 0, row0, full + slot);
          tma2(st + 16384, &m2, 32, row0, full + slot);   // the other 32 channels of the same rows
        } else if (mode == 3) {
          for (int b = 0; b < 4; ++b) tma2(st + b * 8192, &m2s, (b & 1) * 32, row0 + (b >> 1) * 64, full + slot);
        } else if (mode == 4) {
          tma3(st, &m3, 0, row0, 0, full + slot);
          tma3(st + 16384, &m3, 0, row0, 8, full + slot);
        } else {
          const int r = (int)(((size_t)blockIdx.x * iters + k) * 128 % (1u << 22));   // 4M rows of 256 B
          tma2(st, &mbig, 0, r, full + slot);
          tma2(st + 16384, &mbig, 32, r, full + slot);
        }
      }
    }
  } else if (lane == 0) {   // consumer: wait for the stage, touch it, release it
    uint32_t acc = 0;
    for (int k = 0; k < iters; ++k) {
      const int slot = k % NST;
      mbar_wait(full + slot, (k / NST) & 1);
      acc += *(volatile uint32_t*)(sm + slot * STAGE + (k & 63) * 4);
      mbar_arrive(empty + slot);
    }
    if (acc == 0xdeadbeef) out[0] = 0;
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}

static bool enc(CUtensorMap* m, int rank, void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                const cuuint32_t* box, CUtensorMapSwizzle sw, const char* what) {
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, base, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %-34s %d\n", what, (int)r);
  return r == CUDA_SUCCESS;
}

int main() {
  const size_t bytes = 64ull << 20, big = 1ull << 30;
  uint8_t *src, *bsrc;
  cudaMalloc(&src, bytes);
  cudaMalloc(&bsrc, big);
  cudaMemset(src, 1, bytes);
  cudaMemset(bsrc, 1, big);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  CUtensorMap m2, m2s, m3, mbig;
  bool ok = true;
  {   // activations viewed as [rows 262144][64 fp32 channels] (256-B rows), SW128 boxes of 32 channels
    cuuint64_t dims[2] = {64, 262144}, strides[1] = {256};
    cuuint32_t box[2] = {32, 128}, box_s[2] = {32, 64};
    ok &= enc(&m2, 2, src, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, "2D SW128 {32,128}");
    ok &= enc(&m2s, 2, src, dims, strides, box_s, CU_TENSOR_MAP_SWIZZLE_128B, "2D SW128 {32,64}");
  }
  {   // [chunk 16][rows 262144][4 fp32] viewed from the same 256-B rows: box {4, 128, 8} = K-major core rows
    cuuint64_t dims[3] = {4, 262144, 16}, strides[2] = {256, 16};
    cuuint32_t box[3] = {4, 128, 8};
    ok &= enc(&m3, 3, src, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE, "3D none {4,128,8}");
  }
  {
    cuuint64_t dims[2] = {64, 1ull << 22}, strides[1] = {256};
    cuuint32_t box[2] = {32, 128};
    ok &= enc(&mbig, 2, bsrc, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, "2D SW128 {32,128} 1 GB");
  }
  if (!ok) return 1;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE);
  const char* names[6] = {"cp.async 16B, 4 warps", "bulk 16KB runs x2", "TMA 2D SW128 16KB box x2",
                          "TMA 2D SW128 8KB box x4", "TMA 3D none 16B-inner x2", "TMA 2D SW128 x2, HBM src"};
  for (int mode = 0; mode < 6; ++mode) {
    const int iters = 2000;
    kern<<<148, 160, NST * STAGE>>>(mode, iters, src, bytes, m2, m2s, m3, mbig, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s %7.1f cycles/stage  %6.1f B/clk/SM  (%.2f TB/s at %.0f MHz, %s)\n", names[mode], avg / iters,
           (double)STAGE * iters / avg, (double)STAGE * iters / avg * 148 * clk * 1e3 / 1e12, clk / 1e3,
           cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
