// umma_microbench.cu -- measure tcgen05.mma (kind::tf32, SS operands) issue-to-completion
// cycles for the operand layouts the conv kernel uses.  Debug/measurement aid only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_mb umma_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int kind_f16, int M, int N) {
  // kind::tf32: a/b format 2; kind::f16 with bf16: a/b format 1
  return (1u << 4) | ((kind_f16 ? 0u : 2u) << 7) | ((kind_f16 ? 0u : 2u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

template <int KIND_F16>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (KIND_F16)
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
  else
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

// mode 0: conv-like shifted A (SBO = 160, tap offsets); 1: aligned contiguous A (SBO = 128)
template <int N, int KIND_F16>
__global__ void bench(int mode, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* A = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);   // 64 KB
  uint8_t* B = A + 65536;                                                 // 128 KB
  for (int i = threadIdx.x; i < (65536 + 131072) / 16; i += blockDim.x)
    reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(KIND_F16, 128, N);
    const uint32_t a0 = su32(A), b0 = su32(B);
    const uint32_t LBO_A = mode == 0 ? 181 * 16 : 128 * 16 * 2, SBO_A = mode == 0 ? 160 : 128;
    const uint32_t LBO_B = N * 16, SBO_B = 128;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int tap = 0; tap < 9; ++tap) {
        const uint32_t aoff = mode == 0 ? (uint32_t)(((tap / 3) * 10 + tap % 3) * 16) : 0u;
        for (int j = 0; j < 8; ++j) {
          uint64_t ad, bd;
          if (mode == 2) {   // SWIZZLE_128B K-major: 8-row x 128-B atoms, SBO = 1024, K-step = +32 B
            ad = sdesc(a0 + (j >> 2) * 16384 + (j & 3) * 32, 16, 1024, 2);
            const uint32_t nblk = 131072 / (N * 128);
            bd = sdesc(b0 + ((tap * 2 + (j >> 2)) % nblk) * (N * 128) + (j & 3) * 32, 16, 1024, 2);
          } else {
            ad = sdesc(a0 + 2 * (j & 3) * LBO_A + aoff, LBO_A, SBO_A, 0);
            const uint32_t nkq = 131072 / LBO_B - 1;
            bd = sdesc(b0 + ((tap * 16 + 2 * j) % nkq) * LBO_B, LBO_B, SBO_B, 0);
          }
          mma<KIND_F16>(tm, ad, bd, id, (r | tap | j) != 0);
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @P1 bra D; bra W; D:}" ::"r"(
        su32(&bar)));
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

// Fast issue: whole warp 0 runs the loop; descriptors = base + constant (unrolled); elect.sync issues.
__device__ float g_sink;
template <int N, int KIND_F16>
__global__ void bench_fast(int reps, long long* out, int fill, int alu_mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* A = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* B = A + 65536;
  for (int i = threadIdx.x; i < (65536 + 131072) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + 12345u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    float f = fill ? ((float)(h & 0xffff) / 32768.f - 1.f) : 0.f;
    uint32_t bits;
    if (KIND_F16) { __half2 hh = __floats2half2_rn(f, -0.5f * f); bits = *reinterpret_cast<uint32_t*>(&hh); }
    else bits = __float_as_uint(f);
    reinterpret_cast<uint32_t*>(sm)[i] = bits;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const int issuer_warp = (alu_mode & 4) ? 12 : 0;
  if ((int)(threadIdx.x >> 5) == issuer_warp) {
    constexpr uint32_t id = idesc(KIND_F16, 128, N);
    constexpr uint32_t LBO_A = 181 * 16, SBO_A = 160, LBO_B = N * 16, SBO_B = 128;
    const uint64_t a0 = sdesc(su32(A), LBO_A, SBO_A, 0), b0 = sdesc(su32(B), LBO_B, SBO_B, 0);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint64_t ad = a0 + (uint64_t)(((2 * (j & 3)) * LBO_A + ((tap / 3) * 10 + tap % 3) * 16) >> 4);
          const uint64_t bd = b0 + (uint64_t)((((tap * 16 + 2 * j) % 60) * LBO_B) >> 4);
          uint32_t is_leader;
          asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p;}" : "=r"(is_leader));
          if (is_leader) mma<KIND_F16>(tm, ad, bd, id, (r | tap | j) != 0);
          __syncwarp();
        }
      }
    }
    if ((threadIdx.x & 31) == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @P1 bra D; bra W; D:}" ::"r"(
          su32(&bar)));
      out[blockIdx.x] = clock64() - t0;
      asm volatile("st.volatile.shared.u32 [%0], 1;" ::"r"(su32(&slot) + 4096));
    }
  } else if (alu_mode & 3) {
    // concurrent ALU load (GELU via erff, alu_mode 1; plain FFMA chains, alu_mode 2)
    float x = threadIdx.x * 1e-3f, acc = 0.f;
    for (int it = 0; it < reps * 300; ++it) {
      if ((alu_mode & 3) == 1) {
        if (alu_mode & 8) {          // MUFU only
#pragma unroll
          for (int q = 0; q < 8; ++q) acc += __expf(x + q * 0.1f);
        } else if (alu_mode & 16) {  // ALU select/compare only
#pragma unroll
          for (int q = 0; q < 8; ++q) { const float y = x + q; acc += (y > 1.5f ? y : -y) + (y < 2.f ? 0.25f : 0.75f); }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) { const float y = x + q * 0.1f; acc += 0.5f * y * (1.f + erff(y * 0.7071f)); }
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = fmaf(acc, 0.999f, x + q);
      }
      x += 1e-4f;
    }
    if (acc == 12345.f) g_sink = acc;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

template <int N, int F16>
void run_fast(const char* name, int fill = 0, int alu = 0) {
  const int grid = 148, reps = 50;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  const int smem = 65536 + 131072 + 1024;
  cudaFuncSetAttribute(bench_fast<N, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench_fast<N, F16><<<grid, alu ? 416 : 128, smem>>>(reps, d, fill, alu);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  const double nmma = reps * 72.0;
  const double flops = nmma * 2.0 * 128 * N * (F16 ? 16 : 8);
  printf("%-34s N=%3d fill=%d alu=%d fast : %.1f cycles/MMA, %.0f flop/clk/SM (%s)\n", name, N, fill, alu, avg / nmma, flops / avg,
         cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int F16>
void run(int mode, const char* name) {
  const int grid = 148, reps = 50;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  const int smem = 65536 + 131072 + 1024;
  cudaFuncSetAttribute(bench<N, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<N, F16><<<grid, 128, smem>>>(mode, reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  const double nmma = reps * 72.0;
  const double flops = nmma * 2.0 * 128 * N * (F16 ? 16 : 8);
  printf("%-34s N=%3d mode=%d: %.1f cycles/MMA, %.0f flop/clk/SM (%s)\n", name, N, mode, avg / nmma, flops / avg,
         cudaGetErrorString(e));
  cudaFree(d);
}


// Accumulator-rotation probe: is the ~75-cycle floor of an M=128, N<=128 MMA a dependency
// latency on its accumulator (then NACC independent accumulators hide it) or a per-instruction
// cost (then they do not)?  One thread issues reps*72 MMAs; MMA i accumulates into D[i % NACC].
template <int N, int F16, int NACC>
__global__ void bench_acc(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* A = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* B = A + 65536;
  for (int i = threadIdx.x; i < (65536 + 131072) / 16; i += blockDim.x)
    reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc(F16, 128, N);
    constexpr uint32_t LBO_A = 181 * 16, SBO_A = 160, LBO_B = N * 16, SBO_B = 128;
    const uint64_t a0 = sdesc(su32(A), LBO_A, SBO_A, 0), b0 = sdesc(su32(B), LBO_B, SBO_B, 0);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = tap * 8 + j;
          const uint64_t ad = a0 + (uint64_t)(((2 * (j & 3)) * LBO_A + ((tap / 3) * 10 + tap % 3) * 16) >> 4);
          const uint64_t bd = b0 + (uint64_t)((((tap * 16 + 2 * j) % 60) * LBO_B) >> 4);
          mma<F16>(tm + (uint32_t)((i % NACC) * N), ad, bd, id, (r | (i >= NACC)) != 0);
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @P1 bra D; bra W; D:}" ::"r"(
        su32(&bar)));
    out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int N, int F16, int NACC>
void run_acc(const char* name) {
  const int grid = 148, reps = 50;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  const int smem = 65536 + 131072 + 1024;
  cudaFuncSetAttribute(bench_acc<N, F16, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench_acc<N, F16, NACC><<<grid, 128, smem>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  const double nmma = reps * 72.0;
  const double flops = nmma * 2.0 * 128 * N * (F16 ? 16 : 8);
  printf("%-20s N=%3d NACC=%d: %.1f cycles/MMA, %.0f flop/clk/SM (%s)\n", name, N, NACC, avg / nmma, flops / avg,
         cudaGetErrorString(e));
  cudaFree(d);
}


// The conv_xn K-step: 3 dy x 6 input columns, N = 64,128,192,192,128,64 (x CO=64), D offsets
// p_lo*64, A = conv layout (LBO 2560, SBO 160, +16 B per dy, +5120 B per column), B = [dy][q][192][16B].
// shape 0: as the conv; 1: every MMA N=192 at D offset 0; 2: every MMA N=128; 3: N=64 at offset 0;
// 4: as the conv but all D offsets 0 (same columns)
__global__ void bench_conv(int shape, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2[4];
  __shared__ uint32_t slot;
  uint8_t* A = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);   // 30720 B
  uint8_t* Bm = A + 30720;                                                // 18432 B
  for (int i = threadIdx.x; i < (30720 + 18432) / 16; i += blockDim.x)
    reinterpret_cast<float4*>(A)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint64_t a0 = sdesc(su32(A), 2560, 160, 0), b0 = sdesc(su32(Bm), 3072, 128, 0);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy) {
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          int plo = c - 2 > 0 ? c - 2 : 0, phi = c < 3 ? c : 3, nb = phi - plo + 1, jlo = plo - (c - 2);
          if (shape == 1) { nb = 3; plo = 0; jlo = 0; }
          if (shape == 2) { nb = 2; plo = 0; jlo = 0; }
          if (shape == 3) { nb = 1; plo = 0; jlo = 0; }
          if (shape == 4) { plo = 0; }
          const uint64_t ad = a0 + (uint64_t)((c * 5120 + dy * 16) >> 4);
          const uint64_t bd = b0 + (uint64_t)((dy * 6144 + jlo * 1024) >> 4);
          mma<0>(tm + plo * 64, ad, bd, idesc(0, 128, nb * 64), (r | dy | c) != 0);
        }
      }
      if (shape >= 5) {   // per K-step handshake like the conv: commit to a stage barrier
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[r & 3])));
      }
      if (shape >= 6) {   // ... and wait for the K-step 3 back to retire (4-deep ring)
        if (r >= 3) {
          const uint32_t par = ((r - 3) >> 2) & 1;
          asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @P1 bra D; bra W; D:}" ::"r"(
              su32(&bar2[(r - 3) & 3])), "r"(par));
        }
      }
      if (shape >= 7) asm volatile("fence.proxy.async.shared::cta;");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @P1 bra D; bra W; D:}" ::"r"(
        su32(&bar)));
    out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

void run_conv(int shape, const char* name) {
  const int grid = 148, reps = 100;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  const int smem = 30720 + 18432 + 1024;
  cudaFuncSetAttribute(bench_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench_conv<<<grid, 128, smem>>>(shape, reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  printf("conv K-step shape %d %-28s: %.1f cycles per K-step (18 MMAs) (%s)\n", shape, name, avg / reps, cudaGetErrorString(e));
  cudaFree(d);
}


// The conv_xn MMA loop as in the kernel: 4-stage ring of 48 KB stages (A 30720 B + W 18432 B),
// 8 K-steps per tile, two 256-column accumulators alternating per tile, one commit per K-step
// (to a stage barrier) and one per tile.  mode 0: one thread issues; mode 1: convergent warp +
// elect.sync region per K-step (as conv_xn now does).
__global__ void bench_ring(int mode, int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t slot;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 4 * 49152 / 16; i += blockDim.x) {
    if (mode >= 7) {   // random-looking operands (mode 7) instead of mostly zeros
      uint32_t h = (uint32_t)i * 2654435761u + 12345u;
      float f[4];
      for (int q = 0; q < 4; ++q) {
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        f[q] = (float)(h & 0xffff) / 32768.f - 1.f;
      }
      reinterpret_cast<float4*>(base)[i] = make_float4(f[0], f[1], f[2], f[3]);
    } else {
      reinterpret_cast<float4*>(base)[i] = make_float4(0.01f * (i & 7), 0.f, 0.02f, 0.f);
    }
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < 8; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  volatile __shared__ int done_flag;
  if (threadIdx.x == 0) done_flag = 0;
  __syncthreads();
  if (threadIdx.x >= 32) {
    // interference warps (mode 2: cp.async streaming into a scratch region; 3: tcgen05.ld of
    // the accumulators; 4: FFMA chains; 5: STG stores of 512-B runs)
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    uint8_t* scratch = base + 4 * 49152;
    const uint8_t* gsrc = reinterpret_cast<const uint8_t*>(out) + 0;   // dummy, replaced below
    (void)gsrc;
    float acc = threadIdx.x * 1e-3f;
    int it = 0;
    while (!done_flag) {
      if (mode == 2) {
        extern __device__ float4 g_buf[];
        for (int i = threadIdx.x - 32; i < 32768 / 16; i += blockDim.x - 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(scratch + i * 16)),
                       "l"(g_buf + ((size_t)blockIdx.x * 8192 + (it & 3) * 2048 + i)) : "memory");
        asm volatile("cp.async.wait_all;" ::: "memory");
      } else if (mode == 3) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(tm + ((uint32_t)((w & 3) * 32) << 16) + (uint32_t)((it & 15) * 32)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += __uint_as_float(r[ln & 31]);
      } else if (mode == 4) {
#pragma unroll
        for (int q = 0; q < 64; ++q) acc = fmaf(acc, 0.999f, 1e-3f * q);
      } else if (mode == 6) {   // bulk copies (TMA engine) of 16 KB into the scratch, back to back
        if (ln == 0 && w == 1) {
          extern __device__ float4 g_buf[];
          uint64_t* bb = reinterpret_cast<uint64_t*>(scratch + 16384 + 8192);
          if (it == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bb)));
            asm volatile("fence.mbarrier_init.release.cluster;");
          }
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bb)), "r"(16384) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           su32(scratch)),
                       "l"(g_buf + (size_t)blockIdx.x * 8192 + (it & 3) * 1024), "r"(16384), "r"(su32(bb))
                       : "memory");
          asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @P1 bra D; bra W; D:}" ::"r"(
              su32(bb)), "r"(it & 1));
        }
      } else if (mode == 5) {
        extern __device__ float4 g_buf[];
        for (int q = 0; q < 16; ++q)
          g_buf[(size_t)blockIdx.x * 8192 + ((it * 16 + q) & 15) * 512 + (threadIdx.x - 32)] = make_float4(acc, acc, acc, acc);
      }
      ++it;
    }
    if (acc == 12345.f) out[0] = 1;
  }
  if (threadIdx.x < 32) {
    const uint32_t s0 = su32(base);
    long long t0 = clock64();
    int k = 0;
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dacc = tm + (t & 1) * 256;
      for (int ks = 0; ks < 8; ++ks, ++k) {
        const int st = k & 3;
        if (k >= 4) {   // wait for the K-step that last used this stage to retire
          const uint32_t par = ((k - 4) >> 2) & 1;
          asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @P1 bra D; bra W; D:}" ::"r"(
              su32(&bars[st])), "r"(par));
        }
        const uint64_t ad = sdesc(s0 + st * 49152, 2560, 160, 0), bd = sdesc(s0 + st * 49152 + 30720, 3072, 128, 0);
        bool go = mode == 1 || threadIdx.x == 0;
        if (mode == 1) {
          uint32_t p;
          asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
          go = p;
        }
        if (go) {
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) {
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              const int plo = c - 2 > 0 ? c - 2 : 0, phi = c < 3 ? c : 3, nb = phi - plo + 1, jlo = plo - (c - 2);
              mma<0>(dacc + plo * 64, ad + (uint64_t)((c * 5120 + dy * 16) >> 4),
                     bd + (uint64_t)((dy * 6144 + jlo * 1024) >> 4), idesc(0, 128, nb * 64), (ks | dy | c) != 0);
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bars[st])));
          if (ks == 7)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bars[4 + (t & 1)])));
        }
        __syncwarp();
      }
    }
    // drain: wait the last commit of the last K-step's stage
    {
      const int kl = k - 1, st = kl & 3;
      const uint32_t par = (kl >> 2) & 1;
      asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @P1 bra D; bra W; D:}" ::"r"(
          su32(&bars[st])), "r"(par));
    }
    if (threadIdx.x == 0) { out[blockIdx.x] = clock64() - t0; done_flag = 1; }
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}
__device__ float4 g_buf[148 * 8192];

void run_ring(int mode, int nextra = 1) {
  const int grid = 148, tiles = 20;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  const int smem = 4 * 49152 + 32768 + 1024;
  cudaFuncSetAttribute(bench_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench_ring<<<grid, mode >= 2 ? 32 + 32 * nextra : 128, smem>>>(mode, tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  printf("ring mode %d (+%d warps): %.0f cycles per tile (8 K-steps), %.1f per K-step (%s)\n", mode, nextra, avg / tiles, avg / tiles / 8,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run_conv(0, "as the conv");
  run_ring(0);
  run_ring(1);
  run_ring(2, 4);
  run_ring(3, 16);
  run_ring(4, 16);
  run_ring(5, 16);
  run_ring(6, 1);
  run_ring(7, 1);
  return 0;
}
