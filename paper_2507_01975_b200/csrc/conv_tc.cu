// conv_tc.cu -- 3x3 periodic conv layer as an implicit GEMM on the 5th-gen tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), SURVEY.md §8a rows a1-a2 (LD_CONV_TF32).
//
//   D[m][co] = sum_{tap, ci} A[m][tap, ci] * Wt[tap][ci][co]      (+ bias, activation)
//   m = cell of an 8 (x) x 16 (y) tile  ->  GEMM M = 128, N = CO (64 or 32), K = 9 * CI.
//
// The im2col operand is never materialised.  The CTA stages one periodic halo tile of
// 10 x 18 cells x CI channels in shared memory in the canonical K-major, no-swizzle
// UMMA layout  [ci/4][position][4 x fp32]  (core matrix = 8 consecutive x-cells x 16 B).
// Because 8 consecutive x-cells are 16 B apart and consecutive tile rows are PW*16 B
// apart (the descriptor's stride-byte-offset), the operand of tap (dy, dx) is the same
// buffer with its start address moved by ((1+dy)*PW + (1+dx)) * 16 bytes: 9 descriptors,
// one halo load.  All 9*CI x CO weights stay resident in shared memory for the CTA's
// lifetime (persistent CTAs, one per SM, static round-robin over tiles).
//
// Warp roles (288 threads):
//   warps 0-3 : producer  -- cp.async the next halo tile (periodic wrap on the fly),
//                            fence.proxy.async, arrive a_full
//   warp  8   : MMA issuer -- one thread issues 9 * CI/8 tcgen05.mma per tile into one of
//                            two TMEM accumulators, tcgen05.commit -> a_empty, tm_full[buf]
//   warps 4-7 : epilogue  -- tcgen05.ld its 32 TMEM lanes, release the accumulator, add
//                            bias, apply ReLU/GELU(erf), store (NHWC hidden / planar w, e)
#include <cuda.h>

#include "common.cuh"

namespace ld {

namespace tc {

constexpr int TX = 8, TY = 16;
constexpr int PW = TX + 2;                 // halo pitch (positions per tile row)
constexpr int NPOS = (TY + 2) * PW + 1;    // 181 positions (odd: conflict-free 16-B cp.async stores)
constexpr int kThreads = 288;

LD_DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

LD_DEVINL void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
LD_DEVINL void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
LD_DEVINL void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
LD_DEVINL void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
LD_DEVINL void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
LD_DEVINL void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
LD_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
LD_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
LD_DEVINL void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}

// UMMA shared-memory descriptor, K-major SWIZZLE_NONE: start, leading-byte-offset (K
// direction between 16-B core-matrix columns), stride-byte-offset (M/N direction between
// 8-row core matrices), version 1 (sm_100), base offset 0, layout 0.
LD_DEVINL uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Instruction descriptor kind::tf32: D fp32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

LD_DEVINL void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
LD_DEVINL void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
LD_DEVINL void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int CI, int CO>
struct Cfg {
  static constexpr int NQ = CI / 4;                    // 16-B K chunks per tap
  static constexpr int W_BYTES = 9 * NQ * CO * 16;     // [tap*NQ + q][co][16 B]
  static constexpr int A_BYTES = NQ * NPOS * 16;       // [q][pos][16 B]
  static constexpr uint32_t LBO_A = NPOS * 16, SBO_A = PW * 16;
  static constexpr uint32_t LBO_B = CO * 16, SBO_B = 128;
  static constexpr int TMEM_COLS = (2 * CO) < 32 ? 32 : 2 * CO;   // two accumulators
  static constexpr int SMEM = W_BYTES + A_BYTES + 512;
};

enum { OUT_NHWC = 0, OUT_STENCIL = 1 };

template <int CI, int CO, int OUT_MODE>
__global__ void __launch_bounds__(kThreads, 1)
conv_tc_kernel(const float* __restrict__ in, int N, int B, const float* __restrict__ Wtc,
               const float* __restrict__ bias, int act, int co_real, float* __restrict__ out0,
               float* __restrict__ out1) {
  using C = Cfg<CI, CO>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sW = smem;
  uint8_t* sA = smem + C::W_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + C::A_BYTES);   // 8-B aligned (A_BYTES % 16 == 0)
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 1;
  uint64_t* tm_full = bars + 2;    // [2]
  uint64_t* tm_empty = bars + 4;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
  float* sBias = reinterpret_cast<float*>(bars + 8);                // CO floats (<= 64)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---- one-time setup: weights + bias to smem, barriers, TMEM allocation
  {
    const float4* src = reinterpret_cast<const float4*>(Wtc);
    float4* dst = reinterpret_cast<float4*>(sW);
    for (int i = threadIdx.x; i < C::W_BYTES / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    for (int i = threadIdx.x; i < CO; i += blockDim.x) sBias[i] = bias[i];
  }
  if (threadIdx.x == 0) {
    mbar_init(a_full, 128);
    mbar_init(a_empty, 1);
    mbar_init(tm_full + 0, 1);
    mbar_init(tm_full + 1, 1);
    mbar_init(tm_empty + 0, 128);
    mbar_init(tm_empty + 1, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async();   // weights written by the generic proxy, read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles_x = N / TX, tiles_y = N / TY;
  const int ntiles = B * tiles_x * tiles_y;

  if (warp < 4) {
    // ================= producer: periodic halo tile -> sA =================
    const int tid = threadIdx.x;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int b = tile / (tiles_x * tiles_y), rem = tile - b * tiles_x * tiles_y;
      const int y0 = (rem / tiles_x) * TY, x0 = (rem % tiles_x) * TX;
      mbar_wait(a_empty, (it & 1) ^ 1);
      const float* inb = in + (size_t)b * N * N * CI;
      for (int idx = tid; idx < C::NQ * (NPOS - 1); idx += 128) {
        const int p = idx / C::NQ, q = idx - p * C::NQ;
        const int hy = p / PW, hx = p - hy * PW;
        const int gy = wrap(y0 - 1 + hy, N), gx = wrap(x0 - 1 + hx, N);
        cp_async16(sA + ((size_t)q * NPOS + p) * 16, inb + ((size_t)gy * N + gx) * CI + q * 4);
      }
      cp_async_wait_all();
      fence_proxy_async();
      mbar_arrive(a_full);
    }
  } else if (warp == 8) {
    // ================= MMA issuer (single thread) =================
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(128, CO);
      const uint32_t a0 = smem_u32(sA), w0 = smem_u32(sW);
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int ab = it & 1;
        mbar_wait(a_full, it & 1);
        mbar_wait(tm_empty + ab, ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + ab * CO;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int dy = tap / 3, dx = tap % 3;   // (1+dy, 1+dx) of the halo origin
          const uint32_t aoff = (uint32_t)((dy * PW + dx) * 16);
#pragma unroll
          for (int j = 0; j < C::NQ / 2; ++j) {
            const uint64_t ad = sdesc(a0 + 2 * j * C::LBO_A + aoff, C::LBO_A, C::SBO_A);
            const uint64_t bd = sdesc(w0 + (tap * C::NQ + 2 * j) * C::LBO_B, C::LBO_B, C::SBO_B);
            mma_tf32(d, ad, bd, idesc, (tap | j) != 0);
          }
        }
        tc_commit(a_empty);
        tc_commit(tm_full + ab);
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue: TMEM -> registers -> global =================
    const int qd = warp - 4;                  // TMEM lane quarter
    const int m = qd * 32 + lane;             // GEMM row = cell (x = m % 8, y = m / 8)
    const int cx = m & 7, cy = m >> 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int b = tile / (tiles_x * tiles_y), rem = tile - b * tiles_x * tiles_y;
      const int y0 = (rem / tiles_x) * TY, x0 = (rem % tiles_x) * TX;
      const int ab = it & 1;
      mbar_wait(tm_full + ab, (it >> 1) & 1);
      tc_fence_after();
      uint32_t r[CO];
      const uint32_t taddr = tmem_base + ((uint32_t)(qd * 32) << 16) + ab * CO;
      tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      if (CO == 64) tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[CO == 64 ? 32 : 0]));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(tm_empty + ab);
      const int gx = x0 + cx, gy = y0 + cy;
      float v[CO];
#pragma unroll
      for (int o = 0; o < CO; ++o) {
        float t = __uint_as_float(r[o]) + sBias[o];
        if (act == 0) t = fmaxf(t, 0.f);
        else if (act == 1) t = gelu_erf(t);
        v[o] = t;
      }
      if (OUT_MODE == OUT_NHWC) {
        float4* dst = reinterpret_cast<float4*>(out0 + (((size_t)b * N + gy) * N + gx) * CO);
#pragma unroll
        for (int o = 0; o < CO / 4; ++o) dst[o] = make_float4(v[4 * o], v[4 * o + 1], v[4 * o + 2], v[4 * o + 3]);
      } else {
        const size_t plane = (size_t)N * N, pix = (size_t)gy * N + gx;
        float* wb = out0 + (size_t)b * 24 * plane + pix;
#pragma unroll
        for (int o = 0; o < 24; ++o) wb[o * plane] = v[o];
        if (out1 != nullptr && co_real > 24) {
          out1[((size_t)b * 2 + 0) * plane + pix] = v[24];
          out1[((size_t)b * 2 + 1) * plane + pix] = v[25];
        }
      }
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                 : "memory");
  }
}

template <int CI, int CO, int OM>
cudaError_t set_attr() {
  return cudaFuncSetAttribute(conv_tc_kernel<CI, CO, OM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              Cfg<CI, CO>::SMEM);
}

template <int CI, int CO, int OM>
cudaError_t launch(const float* in, int N, int B, const float* W, const float* bias, int act, int co_real, float* o0,
                   float* o1, cudaStream_t st) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int ntiles = B * (N / TX) * (N / TY);
  const int grid = ntiles < sms ? ntiles : sms;
  conv_tc_kernel<CI, CO, OM><<<grid, kThreads, Cfg<CI, CO>::SMEM, st>>>(in, N, B, W, bias, act, co_real, o0, o1);
  return cudaGetLastError();
}

}  // namespace tc

bool tc_conv_available() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0;
}

cudaError_t tc_conv_prepare() {
  cudaError_t e;
  if ((e = tc::set_attr<64, 64, tc::OUT_NHWC>()) != cudaSuccess) return e;
  if ((e = tc::set_attr<64, 32, tc::OUT_STENCIL>()) != cudaSuccess) return e;
  if ((e = tc::set_attr<32, 32, tc::OUT_NHWC>()) != cudaSuccess) return e;
  return tc::set_attr<32, 32, tc::OUT_STENCIL>();
}

size_t tc_weight_floats(int ci, int co_pad) { return (size_t)9 * ci * co_pad; }

// [tap][ci][co_pad] -> [tap*ci/4 + q][co][4]  (K-major 16-B chunks per output channel)
void tc_pack_weights(const float* Wt, int ci, int co_pad, float* dst) {
  const int nq = ci / 4;
  for (int tap = 0; tap < 9; ++tap)
    for (int q = 0; q < nq; ++q)
      for (int co = 0; co < co_pad; ++co)
        for (int e = 0; e < 4; ++e)
          dst[(((size_t)tap * nq + q) * co_pad + co) * 4 + e] = Wt[((size_t)tap * ci + 4 * q + e) * co_pad + co];
}

cudaError_t launch_conv_tc_ci(const float* in, int Ci, int N, int B, const float* Wtc, const float* bias, int co_pad,
                              int act, int out_mode, int co_real, float* out0, float* out1, cudaStream_t st) {
  if (N % tc::TY != 0 || N % tc::TX != 0) return cudaErrorInvalidValue;
  if (Ci == 64 && co_pad == 64 && out_mode == 0)
    return tc::launch<64, 64, tc::OUT_NHWC>(in, N, B, Wtc, bias, act, co_real, out0, out1, st);
  if (Ci == 64 && co_pad == 32 && out_mode == 1)
    return tc::launch<64, 32, tc::OUT_STENCIL>(in, N, B, Wtc, bias, act, co_real, out0, out1, st);
  if (Ci == 32 && co_pad == 32 && out_mode == 0)
    return tc::launch<32, 32, tc::OUT_NHWC>(in, N, B, Wtc, bias, act, co_real, out0, out1, st);
  if (Ci == 32 && co_pad == 32 && out_mode == 1)
    return tc::launch<32, 32, tc::OUT_STENCIL>(in, N, B, Wtc, bias, act, co_real, out0, out1, st);
  return cudaErrorInvalidValue;
}

}  // namespace ld
