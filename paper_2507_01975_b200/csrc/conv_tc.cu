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
//   warps 0-3 : producer  -- cp.async the next half-K stage of a halo tile (periodic wrap
//                            on the fly) into a 3-deep stage ring, fence.proxy.async, arrive
//   warp  8   : MMA issuer -- one elected thread issues 9 * K/32B tcgen05.mma per tile into
//                            one of two TMEM accumulators; tcgen05.commit frees each stage
//   warps 4-7 : epilogue  -- tcgen05.ld its 32 TMEM lanes, release the accumulator, add
//                            bias, apply ReLU/GELU(erf), store (NHWC hidden / planar w, e)
//
// Operand element type T: float (kind::tf32, LD_CONV_TF32) or __half (kind::f16 with fp32
// accumulation, LD_CONV_F16: same 11-bit significand as TF32, half the operand bytes).
// Measured on B200 (tests/tools/umma_microbench.cu): an M=128 SS-mode MMA costs ~74 cycles
// for N <= 128 -- the A operand (4 KB) is read from shared memory at ~64 B/clk -- so with
// N = 64 output channels the A read, not the MMA datapath, bounds this kernel.  Halving the
// operand bytes (f16) doubles the MACs per A byte.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdlib>
#include <cstdio>

#include "common.cuh"

namespace ld {

namespace tc {

constexpr int TX = 8, TY = 16;
constexpr int PW = TX + 2;                 // halo pitch (positions per tile row)
constexpr int NPOS = (TY + 2) * PW + 1;    // 181 positions (odd: conflict-free 16-B cp.async stores)
constexpr int kThreads = 416;     // 4 producer + 8 epilogue + 1 MMA warps

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

// Instruction descriptor: D fp32 (c_format 1); A/B format 2 = TF32 (kind::tf32) or 0 = F16
// (kind::f16); both K-major; N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_mma(bool f16, int M, int N) {
  return (1u << 4) | ((f16 ? 0u : 2u) << 7) | ((f16 ? 0u : 2u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

template <bool F16>
LD_DEVINL void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (F16)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

LD_DEVINL uint32_t elect_one() {
  uint32_t p;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p;
}
LD_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
LD_DEVINL void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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
LD_DEVINL void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
LD_DEVINL void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }


template <typename T, int CI, int CO>
struct Cfg {
  static constexpr bool F16 = sizeof(T) == 2;
  static constexpr int NQ = CI * (int)sizeof(T) / 16;  // 16-B K chunks per tap
  static constexpr int NSPLIT = 2;                     // K halves per tile (pipeline stages)
  static constexpr int QS = NQ / NSPLIT;               // chunks per stage
  static constexpr int W_BYTES = 9 * NQ * CO * 16;     // [tap*NQ + q][co][16 B]
  static constexpr int STAGE_BYTES = QS * NPOS * 16;   // [q][pos][16 B]
  static constexpr int NSTAGE_FIT = (227 * 1024 - W_BYTES - 1024) / STAGE_BYTES;
  static constexpr int NSTAGE = NSTAGE_FIT > 4 ? 4 : NSTAGE_FIT;   // operand ring depth
  static_assert(NSTAGE >= 3, "operand ring needs >= 3 stages");
  static constexpr uint32_t LBO_A = NPOS * 16, SBO_A = PW * 16;
  static constexpr uint32_t LBO_B = CO * 16, SBO_B = 128;
  static constexpr int TMEM_COLS = (2 * CO) < 32 ? 32 : 2 * CO;   // two accumulators
  static constexpr int SMEM = W_BYTES + NSTAGE * STAGE_BYTES + 512;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

enum { OUT_NHWC = 0, OUT_STENCIL = 1, OUT_PLANAR_ALL = 2 };

// Hidden-layer GELU deferred to a post-MMA phase of the same kernel (see below).
// Measured slower on B200 (the extra read-modify-write pass costs more than the MMA/ALU
// interference it removes), so off by default.
#ifndef LD_TC_DEFER_GELU
#define LD_TC_DEFER_GELU 0
#endif

template <typename T>
LD_DEVINL void store_nhwc(T* dst, const float* v, int n);
template <>
LD_DEVINL void store_nhwc<float>(float* dst, const float* v, int n) {
  float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int o = 0; o < 16; ++o)
    if (4 * o < n) d[o] = make_float4(v[4 * o], v[4 * o + 1], v[4 * o + 2], v[4 * o + 3]);
}
template <>
LD_DEVINL void store_nhwc<__half>(__half* dst, const float* v, int n) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    if (8 * o >= n) break;
    __half2 h0 = __floats2half2_rn(v[8 * o], v[8 * o + 1]), h1 = __floats2half2_rn(v[8 * o + 2], v[8 * o + 3]);
    __half2 h2 = __floats2half2_rn(v[8 * o + 4], v[8 * o + 5]), h3 = __floats2half2_rn(v[8 * o + 6], v[8 * o + 7]);
    d[o] = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                      *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
  }
}

template <typename T, int CI, int CO, int OUT_MODE>
__global__ void __launch_bounds__(kThreads, 1)
conv_tc_kernel(const T* __restrict__ in, int N, int B, const uint8_t* __restrict__ Wtc,
               const float* __restrict__ bias, int act, int co_real, void* __restrict__ out0_,
               float* __restrict__ out1, int dbg, unsigned long long* __restrict__ ts) {
  // dbg (measurement knob, 0 in production, env LD_TC_DEBUG): bit0 producer skips the copies,
  // bit1 epilogue skips math and stores, bit2 MMA warp skips the MMAs (commits only)
  using C = Cfg<T, CI, CO>;
  constexpr bool kDeferGelu = LD_TC_DEFER_GELU && OUT_MODE == OUT_NHWC;
#ifndef LD_TC_KNOBS
  dbg = 0;   // measurement knobs compiled out: every dbg test below folds away
#endif
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sW = smem;
  uint8_t* sA = smem + C::W_BYTES;                                   // NSTAGE x STAGE_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + C::NSTAGE * C::STAGE_BYTES);
  uint64_t* a_full = bars;                     // [NSTAGE]
  uint64_t* a_empty = bars + C::NSTAGE;        // [NSTAGE]
  uint64_t* tm_full = bars + 2 * C::NSTAGE;    // [2]
  uint64_t* tm_empty = tm_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + 2);
  float* sBias = reinterpret_cast<float*>(tm_empty + 4);             // CO floats (<= 64)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto trace = [&](int slot) {   // debug trace of CTA 0 only (ts[2048 + slot]); -DLD_TC_TRACE
#ifdef LD_TC_TRACE
    if (ts != nullptr && blockIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[2048 + slot] = t;
    }
#else
    (void)slot;
#endif
  };
  auto stamp = [&](int slot) {
    if (ts != nullptr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[blockIdx.x * 8 + slot] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  // ---- prologue (independent of the previous kernel: overlaps it under PDL)
  {
    const uint4* src = reinterpret_cast<const uint4*>(Wtc);
    uint4* dst = reinterpret_cast<uint4*>(sW);
    for (int i = threadIdx.x; i < C::W_BYTES / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    for (int i = threadIdx.x; i < CO; i += blockDim.x) sBias[i] = bias[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NSTAGE; ++s) {
      mbar_init(a_full + s, 128);
      mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tm_full + s, 1);
      mbar_init(tm_empty + s, 256);
    }
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
  if (threadIdx.x == 0) stamp(1);
  pdl_launch();          // let the next kernel start its own prologue as SMs free up
  pdl_wait();            // inputs written by the previous kernel are visible after this
  if (threadIdx.x == 0) stamp(2);

  const int tiles_x = N / TX, tiles_y = N / TY;
  const int ntiles = B * tiles_x * tiles_y;

  if (warp < 4) {
    // ================= producer: periodic halo tile, one K half per stage =================
    // cp.async commit groups keep NSTAGE-1 stages in flight: stage k is published (fence +
    // arrive) only after stage k+NSTAGE-2 has been issued, so L2 latency overlaps.
    constexpr int INFLIGHT = C::NSTAGE - 1;
    const int tid = threadIdx.x;
    int k = 0;   // global stage counter
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int b = tile / (tiles_x * tiles_y), rem = tile - b * tiles_x * tiles_y;
      const int y0 = (rem / tiles_x) * TY, x0 = (rem % tiles_x) * TX;
      const uint8_t* inb = reinterpret_cast<const uint8_t*>(in + (size_t)b * N * N * CI);
      for (int h = 0; h < C::NSPLIT; ++h, ++k) {
        const int slot = k % C::NSTAGE;
        mbar_wait(a_empty + slot, ((k / C::NSTAGE) & 1) ^ 1);
        uint8_t* st = sA + slot * C::STAGE_BYTES;
        for (int idx = tid; idx < ((dbg & 1) ? 0 : C::QS * (NPOS - 1)); idx += 128) {
          const int p = idx / C::QS, q = idx - p * C::QS;
          const int hy = p / PW, hx = p - hy * PW;
          const int gy = wrap(y0 - 1 + hy, N), gx = wrap(x0 - 1 + hx, N);
          cp_async16(st + ((size_t)q * NPOS + p) * 16,
                     inb + ((size_t)gy * N + gx) * CI * sizeof(T) + (size_t)(h * C::QS + q) * 16);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (k >= INFLIGHT - 1) {
          asm volatile("cp.async.wait_group %0;" ::"n"(INFLIGHT - 1) : "memory");
          fence_proxy_async();
          mbar_arrive(a_full + (k - (INFLIGHT - 1)) % C::NSTAGE);
          if (tid == 0 && k - (INFLIGHT - 1) < 16) trace(200 + k - (INFLIGHT - 1));   // producer: stage published
        }
      }
    }
    // drain: publish the last INFLIGHT-1 stages
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    fence_proxy_async();
    for (int j = k - (INFLIGHT - 1); j < k; ++j)
      if (j >= 0) mbar_arrive(a_full + j % C::NSTAGE);
    if (threadIdx.x == 0) stamp(3);
  } else if (warp == 12) {
    // ================= MMA issuer (whole warp loops, one elected lane issues) =================
    constexpr uint32_t idesc = idesc_mma(C::F16, 128, CO);
    const uint32_t a0 = smem_u32(sA), w0 = smem_u32(sW);
    const uint64_t adesc0 = sdesc(a0, C::LBO_A, C::SBO_A), bdesc0 = sdesc(w0, C::LBO_B, C::SBO_B);
    int k = 0, it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int ab = it & 1;
      mbar_wait(tm_empty + ab, ((it >> 1) & 1) ^ 1);
      if (lane == 0 && it < 16) trace(it * 8 + 0);        // MMA: accumulator free
      for (int h = 0; h < C::NSPLIT; ++h, ++k) {
        const int slot = k % C::NSTAGE;
        mbar_wait(a_full + slot, (k / C::NSTAGE) & 1);
        if (lane == 0 && it < 16) trace(it * 8 + 1 + h);    // MMA: stage h data ready
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ast = adesc0 + (uint64_t)((slot * C::STAGE_BYTES) >> 4);
          const uint32_t d = tmem_base + ab * CO;
#pragma unroll 1
          for (int tap = 0; tap < 9; ++tap) {
            const uint32_t aoff = (uint32_t)(((tap / 3) * PW + tap % 3) * 16);
#pragma unroll
            for (int j = 0; j < C::QS / 2; ++j) {
              const uint64_t ad = ast + (uint64_t)((2 * j * C::LBO_A + aoff) >> 4);
              const uint64_t bd = bdesc0 + (uint64_t)(((tap * C::NQ + h * C::QS + 2 * j) * C::LBO_B) >> 4);
              if (!(dbg & 4)) mma_ss<C::F16>(d, ad, bd, idesc, (h | tap | j) != 0);
            }
          }
          tc_commit(a_empty + slot);                        // stage free once these MMAs retire
          if (h == C::NSPLIT - 1) tc_commit(tm_full + ab);  // accumulator complete
          if (it < 16) trace(it * 8 + 3 + h);               // MMA: stage h issued
        }
        __syncwarp();
      }
    }
  } else {
    // ================= epilogue: TMEM -> registers -> global =================
    // (MMA loop end is stamped as slot 4 below)
    // warps 4..11: TMEM lane quarter = warp % 4 (hardware rule), column half = (warp - 4) / 4
    constexpr int HC = CO / 2;                // columns per thread
    const int qd = warp & 3, ch = (warp - 4) >> 2;
    const int m = qd * 32 + lane;             // GEMM row = cell (x = m % 8, y = m / 8)
    const int cx = m & 7, cy = m >> 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int b = tile / (tiles_x * tiles_y), rem = tile - b * tiles_x * tiles_y;
      const int y0 = (rem / tiles_x) * TY, x0 = (rem % tiles_x) * TX;
      const int ab = it & 1;
      mbar_wait(tm_full + ab, (it >> 1) & 1);
      if (threadIdx.x == 128 && it < 16) trace(it * 8 + 5);   // epilogue: accumulator ready
      tc_fence_after();
      uint32_t r[32];
      const uint32_t taddr = tmem_base + ((uint32_t)(qd * 32) << 16) + ab * CO + ch * HC;
      if (HC == 32) tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      else tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(tm_empty + ab);
      if (threadIdx.x == 128 && it < 16) trace(it * 8 + 6);   // epilogue: TMEM drained
      if (dbg & 2) continue;
      const int gx = x0 + cx, gy = y0 + cy;
      float v[HC];
#pragma unroll
      for (int o = 0; o < HC; ++o) {
        float t = __uint_as_float(r[o]) + sBias[ch * HC + o];
        if (act == 0 || (dbg & 32)) t = fmaxf(t, 0.f);
        else if (act == 1 && !(kDeferGelu && !(dbg & 64))) t = gelu_erf(t);
        v[o] = t;
      }
      const size_t plane = (size_t)N * N, pix = (size_t)gy * N + gx;
      if (dbg & 16) {
        if (v[0] == 12345.f) out1[0] = v[1];   // keep the math live
        continue;
      }
      if (OUT_MODE == OUT_NHWC) {
        T* dst = reinterpret_cast<T*>(out0_) + (((size_t)b * N + gy) * N + gx) * CO + ch * HC;
        store_nhwc<T>(dst, v, HC);
      } else if (OUT_MODE == OUT_STENCIL) {
        float* wb = reinterpret_cast<float*>(out0_) + (size_t)b * 24 * plane + pix;
#pragma unroll
        for (int o = 0; o < HC; ++o) {
          const int co = ch * HC + o;
          if (co < 24) wb[co * plane] = v[o];
          else if (out1 != nullptr && co < co_real) out1[((size_t)b * 2 + (co - 24)) * plane + pix] = v[o];
        }
      } else {
        float* ob = reinterpret_cast<float*>(out0_) + (size_t)b * co_real * plane + pix;
#pragma unroll
        for (int o = 0; o < HC; ++o)
          if (ch * HC + o < co_real) ob[(ch * HC + o) * plane] = v[o];
      }
    }
  }
  // ---- deferred GELU (hidden layers): applied in place to this CTA's own tiles after its
  // last MMA, so the erf arithmetic does not run concurrently with the tensor core (measured:
  // concurrent ALU issue slows these A-read-bound MMAs ~2x; tests/tools/umma_microbench.cu).
  if (kDeferGelu && act == 1 && !(dbg & 2) && !(dbg & 64)) {
    __syncthreads();   // this CTA's pre-activation stores are visible to all its threads
    constexpr int EPV = 16 / (int)sizeof(T);           // elements per 16-B vector
    constexpr int VPC = CO / EPV;                       // vectors per cell
    constexpr int PER_TILE = TX * TY * VPC;
    constexpr int U = 4;                                // loads in flight per thread
    const int my_tiles = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int total = my_tiles * PER_TILE;
    for (int i0 = threadIdx.x; i0 < total; i0 += U * blockDim.x) {
      uint4* ptr[U];
      uint4 q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * blockDim.x;
        ptr[u] = nullptr;
        if (i < total) {
          const int lt = i / PER_TILE, w = i - lt * PER_TILE;
          const int tile = blockIdx.x + lt * gridDim.x;
          const int b = tile / (tiles_x * tiles_y), rem = tile - b * tiles_x * tiles_y;
          const int y0 = (rem / tiles_x) * TY, x0 = (rem % tiles_x) * TX;
          const int cell = w / VPC, vq = w - cell * VPC;
          ptr[u] = reinterpret_cast<uint4*>(reinterpret_cast<T*>(out0_) + (size_t)b * N * N * CO +
                                            ((size_t)(y0 + cell / TX) * N + x0 + (cell % TX)) * CO) + vq;
          q[u] = *ptr[u];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ptr[u] == nullptr) continue;
        if (sizeof(T) == 2) {
          __half2* hq = reinterpret_cast<__half2*>(&q[u]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __half22float2(hq[e]);
            hq[e] = __floats2half2_rn(gelu_erf(f.x), gelu_erf(f.y));
          }
        } else {
          float* fq = reinterpret_cast<float*>(&q[u]);
#pragma unroll
          for (int e = 0; e < 4; ++e) fq[e] = gelu_erf(fq[e]);
        }
        *ptr[u] = q[u];
      }
    }
  }
  if (threadIdx.x == 12 * 32) stamp(4);
  if (threadIdx.x == 4 * 32) stamp(5);
  __syncthreads();
  if (threadIdx.x == 0) stamp(6);
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                 : "memory");
  }
}

template <typename T, int CI, int CO, int OM>
cudaError_t set_attr() {
  return cudaFuncSetAttribute(conv_tc_kernel<T, CI, CO, OM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              Cfg<T, CI, CO>::SMEM);
}

template <typename T, int CI, int CO, int OM>
cudaError_t launch(const void* in, int N, int B, const void* W, const float* bias, int act, int co_real, void* o0,
                   float* o1, cudaStream_t st) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int ntiles = B * (N / TX) * (N / TY);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ntiles < sms ? ntiles : sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg<T, CI, CO>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int dbg = -1;
  if (dbg < 0) {
    const char* e = getenv("LD_TC_DEBUG");
    dbg = e ? atoi(e) : 0;
  }
  static unsigned long long* ts = nullptr;
  static int dumped = 0;
  const bool want_ts = (dbg & 8) && CI == 64 && CO == 64 && dumped < 3;
  if (want_ts && ts == nullptr) {
    cudaMalloc(&ts, 4096 * sizeof(unsigned long long));
    cudaMemset(ts, 0, 4096 * sizeof(unsigned long long));
  }
  cudaError_t err = cudaLaunchKernelEx(&cfg, conv_tc_kernel<T, CI, CO, OM>, reinterpret_cast<const T*>(in), N, B,
                                       reinterpret_cast<const uint8_t*>(W), bias, act, co_real, o0, o1, dbg & ~8,
                                       want_ts ? ts : nullptr);
  if (want_ts) {   // debug: per-CTA phase timestamps (ns), printed for the first few launches
    ++dumped;
    unsigned long long h[148 * 8];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, ts, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    const int g = (int)cfg.gridDim.x;
    for (int i = 0; i < g; ++i) t0 = h[i * 8] < t0 ? h[i * 8] : t0;
    double avg[8] = {0};
    unsigned long long mx[8] = {0};
    for (int i = 0; i < g; ++i)
      for (int k = 0; k < 7; ++k) {
        const unsigned long long d = h[i * 8 + k] - t0;
        avg[k] += (double)d / g;
        mx[k] = d > mx[k] ? d : mx[k];
      }
    fprintf(stderr, "[conv_tc ts] grid=%d  (avg/max ns from first CTA start) entry %.0f/%llu  prologue %.0f/%llu  "
            "pdl_wait %.0f/%llu  producer_end %.0f/%llu  mma_end %.0f/%llu  epi_end %.0f/%llu  exit %.0f/%llu\n",
            g, avg[0], mx[0], avg[1], mx[1], avg[2], mx[2], avg[3], mx[3], avg[4], mx[4], avg[5], mx[5], avg[6], mx[6]);
    unsigned long long tr[2048];
    cudaMemcpy(tr, ts + 2048, sizeof(tr), cudaMemcpyDeviceToHost);
    const unsigned long long c0 = h[0];
    for (int it = 0; it < 8; ++it)
      fprintf(stderr, "  tile %d: acc_free %lld  A0_ready %lld  A1_ready %lld  A0_issued %lld  A1_issued %lld  epi_ready %lld  epi_drained %lld | prod_pub %lld %lld\n",
              it, (long long)(tr[it * 8 + 0] - c0), (long long)(tr[it * 8 + 1] - c0), (long long)(tr[it * 8 + 2] - c0),
              (long long)(tr[it * 8 + 3] - c0), (long long)(tr[it * 8 + 4] - c0), (long long)(tr[it * 8 + 5] - c0),
              (long long)(tr[it * 8 + 6] - c0), (long long)(tr[200 + 2 * it] - c0), (long long)(tr[201 + 2 * it] - c0));
  }
  return err;
}

}  // namespace tc

bool tc_conv_available() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0;
}

#define LD_TC_VARIANTS(X)                                                                          \
  X(float, 64, 64, tc::OUT_NHWC) X(float, 64, 32, tc::OUT_STENCIL) X(float, 64, 32, tc::OUT_PLANAR_ALL) \
  X(float, 32, 32, tc::OUT_NHWC) X(float, 32, 32, tc::OUT_STENCIL) X(float, 32, 32, tc::OUT_PLANAR_ALL) \
  X(__half, 64, 64, tc::OUT_NHWC) X(__half, 64, 32, tc::OUT_STENCIL) X(__half, 64, 32, tc::OUT_PLANAR_ALL) \
  X(__half, 32, 32, tc::OUT_NHWC) X(__half, 32, 32, tc::OUT_STENCIL) X(__half, 32, 32, tc::OUT_PLANAR_ALL)

cudaError_t tc_conv_prepare() {
  cudaError_t e = cudaSuccess;
#define LD_SET(T, CI, CO, OM) \
  if (e == cudaSuccess) e = tc::set_attr<T, CI, CO, OM>();
  LD_TC_VARIANTS(LD_SET)
#undef LD_SET
  return e;
}

// bytes of the packed tcgen05 weight operand of one layer
size_t tc_weight_bytes(int ci, int co_pad, int f16) { return (size_t)9 * ci * co_pad * (f16 ? 2 : 4); }

// Wt [tap][ci][co_pad] (fp32) -> [tap*NQ + q][co][16 B]  (K-major 16-B chunks per output channel;
// 4 fp32 or 8 fp16 consecutive input channels per chunk)
void tc_pack_weights(const float* Wt, int ci, int co_pad, int f16, uint8_t* dst) {
  const int epc = f16 ? 8 : 4, nq = ci / epc;
  for (int tap = 0; tap < 9; ++tap)
    for (int q = 0; q < nq; ++q)
      for (int co = 0; co < co_pad; ++co)
        for (int e = 0; e < epc; ++e) {
          const float w = Wt[((size_t)tap * ci + epc * q + e) * co_pad + co];
          const size_t idx = (((size_t)tap * nq + q) * co_pad + co) * epc + e;
          if (f16) reinterpret_cast<__half*>(dst)[idx] = __float2half_rn(w);
          else reinterpret_cast<float*>(dst)[idx] = w;
        }
}

cudaError_t launch_conv_tc_ci(const void* in, int Ci, int N, int B, const void* Wtc, const float* bias, int co_pad,
                              int f16, int act, int out_mode, int co_real, void* out0, float* out1, cudaStream_t st) {
  if (N % tc::TY != 0 || N % tc::TX != 0) return cudaErrorInvalidValue;
#define LD_LAUNCH(T, CI, CO, OM)                                                                      \
  if ((sizeof(T) == 2) == (f16 != 0) && Ci == CI && co_pad == CO && out_mode == OM)                   \
    return tc::launch<T, CI, CO, OM>(in, N, B, Wtc, bias, act, co_real, out0, out1, st);
  LD_TC_VARIANTS(LD_LAUNCH)
#undef LD_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace ld
