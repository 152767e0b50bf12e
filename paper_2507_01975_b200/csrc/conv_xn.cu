// conv_xn.cu -- 3x3 periodic conv layer as an implicit GEMM on the 5th-gen tensor cores
// (tcgen05.mma, accumulators in TMEM), PAPER.md P:246-250 as
// generalised by BASELINE.json (readings R1, R6).
//
//   out[b, y, x, co] = phi( bias[co] + sum_{dy,dx,ci} W[(dy+1)*3+(dx+1)][ci][co] * in[b, y+dy, x+dx, ci] )
//
// Why this shape (measured, profiles/r01_umma_*.log): one M=128 tcgen05.mma costs ~60-78 cycles
// for ANY N <= 128 but reaches the hardware floor M*N/256 cycles at N >= 128.  With the output
// channels alone as N (64) the conv is capped near 25-50% of the tensor pipe.  So the x
// direction goes into N as well:
//
//   GEMM rows (M = 128 TMEM lanes) = 16 "strips" x 8 consecutive y-cells, all at one x offset;
//   GEMM cols (N)                  = (output x position p, co);  XP = 4 positions per strip.
//
// For input column x_in = xbase + c - 1 (c = 0..5) and row shift dy, ONE MMA with
//   B = [W(dy, dx=+1) | W(dy, 0) | W(dy, -1)]   (N = 3 * CO = 192)
// adds the contributions of that input column to the three outputs x_in - dx, i.e. to the
// TMEM accumulator columns of positions p = c-2, c-1, c: the x-shift of the stencil is a
// column offset of D, the y-shift (dy) a 16-byte start offset of the A descriptor (each strip
// is stored as 10 rows = 8 + a periodic 1-cell halo on each side, SBO = 160 B, so every 8-lane
// core-matrix group carries its own halo and strips may sit anywhere in the domain).
// At the tile edge (c = 0, 1, 4, 5) the MMA shrinks to N = 64 / 128.  Per K-step of 32 bytes:
// 3 dy x 6 columns = 18 MMAs, ~88% of the floor of the pure-N=192 shape.
//
// Activations in HBM: [b][K-step][q][x][y][16 B] (q = which 16-B half of the 32-B K-step), so the
// producer's loads and the epilogue's stores are contiguous runs along y.
// Shared memory per pipeline stage (one K-step = 32 B of channels per cell):
//   A [c 0..5][q 0..1][strip 0..15][row 0..9][16 B]      30720 B (K-major, no swizzle)
//   W [dy 0..2][q 0..1][n 0..3*CO-1][16 B]              18432 B (CO = 64), one bulk copy
// 4 stages (192 KB).  TMEM: two accumulators of XP*CO columns (512 for CO = 64).
//
// Warp roles (672 threads): warps 0-3 producer (coalesced 16-B cp.async of the activation runs
// with periodic wrap + one bulk copy of the pre-packed W block per stage), warps 4-19 epilogue
// (one output position each: tcgen05.ld -> bias -> activation -> store), warp 20 MMA issuer (one
// thread, fully unrolled).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>

#include <cuda_bf16.h>
#include <type_traits>

#include "common.cuh"

namespace ld {
namespace xn {

constexpr int XP = 4;          // output x positions per strip (N-blocks of CO columns)
constexpr int NG = 16;         // strips per tile (8 TMEM lanes each)
constexpr int RY = 8;          // y-cells per strip
constexpr int RH = RY + 2;     // stored rows per strip (periodic halo)
constexpr int NCOL = XP + 2;   // input x columns per tile

LD_DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
LD_DEVINL void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
LD_DEVINL void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
LD_DEVINL void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
LD_DEVINL void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nXN_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra XN_DONE;\nbra XN_WAIT;\nXN_DONE:\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// Waiters that are not on the MMA issue path back off between polls, so their spin loops do not
// take issue slots from the single MMA-issuing thread (which shares an SMSP with 5 other warps).
LD_DEVINL bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
LD_DEVINL void mbar_wait_backoff(uint64_t* b, uint32_t parity) {
  while (!mbar_try(b, parity)) __nanosleep(64);
}

LD_DEVINL void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// the same copy with an L2 eviction-priority hint (createpolicy): operands read once per layer marked
// evict_first, so the lines the next kernel reads (this layer's output) are the ones L2 keeps
LD_DEVINL void cp_async16_hint(void* dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "l"(pol)
               : "memory");
}
LD_DEVINL uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
LD_DEVINL void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
LD_DEVINL void prefetch_l2(const void* src, uint32_t bytes) {   // bulk L2 prefetch (16-B multiple)
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
LD_DEVINL void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
LD_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
LD_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
LD_DEVINL void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
LD_DEVINL uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;   // sm_100 descriptor version
  return d;
}
// D fp32; A/B TF32 (format 2, kind::tf32), F16 (format 0) or BF16 (format 1, both kind::f16);
// both K-major.
__host__ __device__ constexpr uint32_t idesc(int fmt, int M, int N) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
template <bool F16>
LD_DEVINL void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (F16)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
LD_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
LD_DEVINL uint32_t elect_one() {
  uint32_t p;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p;
}
LD_DEVINL void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// 32 lanes x 32 consecutive fp32 columns; completes at the next tmem_ld_wait()
LD_DEVINL void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
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
// the registers of an async tcgen05.ld are defined at its wait: keep every use below it
template <int n>
LD_DEVINL void tmem_regs_ready(uint32_t (&r)[n]) {
#pragma unroll
  for (int i = 0; i < n; ++i) asm volatile("" : "+r"(r[i]));
}
// 32 lanes x 16 consecutive fp32 columns; completes at the next tmem_ld_wait()
LD_DEVINL void tmem_ld16_async(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
template <int n>
LD_DEVINL void tmem_ld_async(uint32_t taddr, uint32_t (&r)[n]) {
  if constexpr (n == 16) tmem_ld16_async(taddr, r);
  else tmem_ld32_async(taddr, r);
}
#define XN_TSC 296   // measurement stamps: CTA slots (2 per SM)
#ifndef XN_GELU2
#define XN_GELU2 1   // epilogue GELU on packed fp32 pairs
#endif
#ifndef XN_EPI_CH
#define XN_EPI_CH 32   // epilogue chunk (TMEM columns per tcgen05.ld) for the blocked output
#endif


// CT ("contiguous tile"): the 16 strips of every tile are one 128-row column segment (N_y % 128
// == 0), so the operand stage stores each input column as 130 consecutive rows (SBO = 128 B) instead
// of 16 separate 10-row strips (SBO = 160 B): 19% fewer operand bytes, and a stage small enough for
// the TF32 weights to stay resident beside 3 stages.
// DU ("dual"): two CTAs per SM, each with half the resources (3 producer + 8 epilogue warps, one
// TMEM accumulator, 2 streamed stages), so one CTA's prologue / epilogue overlaps the other's
// MMAs -- for grids of at most ~2 tiles per SM, where a CTA otherwise runs its last epilogue
// and its first operand fill alone.
// XPT: output x positions per tile (4; 8 for the contiguous-tile output layer with the flux epilogue,
// whose 32-column accumulators leave TMEM room for 2 x 8 positions)
template <typename T, int CI, int CO, bool CT = false, bool DU = false, int XPT = XP>
struct Cfg {
  static constexpr int XP_ = XPT, NCOL_ = XPT + 2;       // positions, input columns per tile
  static constexpr int ARH = CT ? NG * RY + 2 : NG * RH;   // stored rows per (column, core column)
  static constexpr int A_QBYTES = ARH * 16;
  static constexpr int A_STAGE = NCOL_ * 2 * A_QBYTES;     // 24960 (CT) / 30720 at XPT = 4
  static constexpr uint32_t LBO_A = A_QBYTES, SBO_A = CT ? RY * 16 : RH * 16;
  static constexpr bool F16 = sizeof(T) == 2;            // kind::f16 (F16 or BF16 operands)
  static constexpr int FMT = sizeof(T) == 4 ? 2 : (std::is_same<T, __nv_bfloat16>::value ? 1 : 0);
  static constexpr int EPC = 16 / (int)sizeof(T);        // channels per 16-B core column
  static constexpr bool PLANAR_IN = CI == 2;              // first layer: planar velocity (u, v)
  static constexpr int NKS = PLANAR_IN ? 1 : CI / (2 * EPC);   // K-steps (32 B of channels each)
  static constexpr int KBE = 2 * EPC;                     // channels per K-step block (8 fp32 / 16 fp16)
  static constexpr int NKS_OUT = CO / KBE;                // K-step blocks of the output activation
  static constexpr int NB = 3 * CO;                       // B rows: (dx block, co)
  static constexpr int W_DY = 2 * NB * 16;                // bytes of one dy block
  static constexpr int W_STAGE = 3 * W_DY;
  static constexpr uint32_t LBO_B = NB * 16, SBO_B = 128;
  // Weights resident in shared memory for the CTA's lifetime when they fit beside >= 3 operand
  // stages (loaded once, not re-streamed per tile: saves 9*CI*CO*4 B of L2 traffic per tile);
  // otherwise one weight block travels with every stage.
  static constexpr int W_TOTAL = NKS * W_STAGE;
  static constexpr int SMEM_CAP = DU ? 113 * 1024 : 227 * 1024;   // per CTA
#ifndef XN_CT_STREAM_W
#define XN_CT_STREAM_W 0   // measurement build: contiguous tiles stream W per stage (deeper ring)
#endif
  static constexpr bool W_RES = W_TOTAL + 3 * A_STAGE + 2048 <= SMEM_CAP && !(CT && XN_CT_STREAM_W);   // measured: 2 stages are too shallow
  static constexpr int W_OFF = W_RES ? W_TOTAL : 0;
  static constexpr int STAGE = W_RES ? A_STAGE : A_STAGE + W_STAGE;
  static constexpr int NST_FIT = (SMEM_CAP - W_OFF - 2048) / STAGE;
#ifndef XN_MAXSTAGE
#define XN_MAXSTAGE 4
#endif
  static constexpr int NSTAGE = NST_FIT >= XN_MAXSTAGE ? XN_MAXSTAGE : NST_FIT;
  static constexpr int NPW = DU ? 3 : 4;                  // producer warps
  static constexpr int NPT = 32 * NPW;                    // producer threads
  static constexpr int NEW = DU ? 8 : 16;                 // epilogue warps (XP * 4 / NEW positions each)
  static constexpr int MMA_WARP = NPW + NEW;
  static constexpr int THREADS = 32 * (NPW + NEW + 1);
  static constexpr int MINB = DU ? 2 : 1;                 // CTAs per SM
  static constexpr int NACC = DU ? 1 : 2;                 // TMEM accumulators
  static constexpr int ACC_COLS = XP_ * CO;               // one accumulator
  static constexpr int TMEM_COLS = NACC * ACC_COLS;       // 128, 256 or 512 (power of two)
  static constexpr int SMEM = W_OFF + NSTAGE * STAGE + 1024;   // + barriers, bias, strip origins
  static_assert(NSTAGE >= 2, "pipeline depth");
  static_assert(TMEM_COLS <= 512, "TMEM columns");
  static_assert(NKS >= 1, "K steps");
};

enum { OUT_BLOCKED = 0, OUT_STENCIL = 1, OUT_PLANAR_ALL = 2, OUT_FLUX = 3 };

// OUT_FLUX (output layer, Ny % 128 == 0): instead of the 24 stencils the epilogue writes the face
// fluxes of each cell's own faces, F[b][x][y][4] = (F^x_u, F^x_v at i-1/2, F^y_u, F^y_v at j-1/2), applying
// the cell's stencils to the stage field in registers (the same fp32 operations in the same order as K2).
// The field's tile neighbourhood -- the 128 y x 4 x cells of the tile plus a radius-3 halo, both
// components -- is staged by the epilogue warps in shared memory behind the CTA's operand ring while the
// tile's MMAs run.
constexpr int FE_ROWS = NG * RY + 6;   // 134 rows x (XP + 6 used + 1 pad) floats per component
template <int XPn>
constexpr int fe_pitch() { return XPn + 7; }
template <int XPn>
constexpr int fe_smem() { return 2 * FE_ROWS * fe_pitch<XPn>() * 4; }
// positions per tile of a kernel variant
template <int OM, bool CT, bool DU>
constexpr int xp_of() { return (OM == OUT_FLUX && CT && !DU) ? 8 : XP; }

// operand type code of the launch interface: 0 fp32 (TF32 MMA), 1 fp16, 2 bf16
template <typename T>
constexpr int type_code() {
  return sizeof(T) == 4 ? 0 : (std::is_same<T, __nv_bfloat16>::value ? 2 : 1);
}

template <typename T>
LD_DEVINL void store_vec(T* dst, const float* v, int n);
template <>
LD_DEVINL void store_vec<float>(float* dst, const float* v, int n) {
  float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int o = 0; o < 8; ++o)
    if (4 * o < n) d[o] = make_float4(v[4 * o], v[4 * o + 1], v[4 * o + 2], v[4 * o + 3]);
}
template <>
LD_DEVINL void store_vec<__half>(__half* dst, const float* v, int n) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    if (8 * o >= n) break;
    __half2 h[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2half2_rn(v[8 * o + 2 * e], v[8 * o + 2 * e + 1]);
    d[o] = *reinterpret_cast<uint4*>(h);
  }
}
template <>
LD_DEVINL void store_vec<__nv_bfloat16>(__nv_bfloat16* dst, const float* v, int n) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    if (8 * o >= n) break;
    __nv_bfloat162 h[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * o + 2 * e], v[8 * o + 2 * e + 1]);
    d[o] = *reinterpret_cast<uint4*>(h);
  }
}

// strip s -> (b, x0, y0): s = (b * (Nx/XP) + xb) * (Ny/RY) + yb  (y-blocks fastest, so the 16
// strips of a tile are a contiguous column segment when Ny >= 128)
LD_DEVINL void strip_origin(int s, int Nx, int Ny, int xp, int& b, int& x0, int& y0) {
  const int nyb = Ny / RY, nxb = Nx / xp;
  const int yb = s % nyb, t = s / nyb;
  const int xb = t % nxb;
  b = t / nxb;
  x0 = xb * xp;
  y0 = yb * RY;
}


// The MMAs of one K-step (3 dy x (XPn + 2) input columns), fully unrolled: every descriptor is the
// stage base plus a compile-time offset.  Input column c (x0 - 1 + c) feeds positions p = c - 2 .. c.
// FIRST: the tile's first K-step, whose dy = -1 pass clears the accumulator.  Per group of 4 positions
// g (XPn = 4: one group; 8: two) the clearing order is the XP = 4 one -- column 4g + 2 (positions
// 4g .. 4g + 2) and 4g + 5 (position 4g + 3) with accumulate = 0, then 4g, 4g + 1, 4g + 3, 4g + 4 --
// with every MMA restricted to the group's positions, so each output receives its contributions in the
// same order for any XPn (bitwise the same accumulators).  All other passes: columns ascending.
template <bool F16, int FMT, int CO, int A_QBYTES, int XPn>
LD_DEVINL void mma_cols(uint32_t dacc, uint64_t ad, uint64_t bd, int dyi, int c, int plo, int phi, uint32_t accf) {
  constexpr uint32_t W_DY = 2 * 3 * CO * 16;
  const int p_lo = c - 2 > plo ? c - 2 : plo;
  const int p_hi = c < phi ? c : phi;
  if (p_hi < p_lo) return;
  const int nblk = p_hi - p_lo + 1;
  const int j_lo = p_lo - (c - 2);
  const uint64_t a = ad + (uint64_t)((c * 2 * A_QBYTES + dyi * 16) >> 4);
  const uint64_t b = bd + (uint64_t)((dyi * W_DY + j_lo * CO * 16) >> 4);
  const uint32_t id = idesc(FMT, 128, nblk * CO);
  mma<F16>(dacc + (uint32_t)(p_lo * CO), a, b, id, accf);
}
template <bool F16, int FMT, int CO, bool FIRST, int A_QBYTES, int XPn = XP>
LD_DEVINL void issue_kstep(uint32_t dacc, uint64_t ad, uint64_t bd) {
  constexpr int NC = XPn + 2;
#pragma unroll
  for (int dyi = 0; dyi < 3; ++dyi) {
    if (FIRST && dyi == 0) {
#pragma unroll
      for (int g = 0; g < XPn / 4; ++g) {
#pragma unroll
        for (int ci = 0; ci < 6; ++ci) {
          const int cr = ci == 0 ? 2 : ci == 1 ? 5 : ci - 2 + (ci >= 4 ? 1 : 0);   // 2,5,0,1,3,4
          mma_cols<F16, FMT, CO, A_QBYTES, XPn>(dacc, ad, bd, 0, 4 * g + cr, 4 * g, 4 * g + 3, ci >= 2 ? 1u : 0u);
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) mma_cols<F16, FMT, CO, A_QBYTES, XPn>(dacc, ad, bd, dyi, c, 0, XPn - 1, 1u);
    }
  }
}

// FUSE1: the net's first layer (2 -> CI channels: the planar stage field u, its SIMT-layout weights
// W1 [9][2][CI] and bias b1) is recomputed on the fly by the producer warps in fp32 (paired FFMA2) for
// every K-step's channels and written straight into the operand stage, instead of being read from the
// first layer's 256-B/cell output -- the first conv launch and its output round trip through HBM
// disappear (contiguous-tile hidden layers only).
template <typename T, int CI, int CO, bool CT, bool DU>
__host__ __device__ constexpr bool C_PLANAR_IN_() { return Cfg<T, CI, CO, CT, DU>::PLANAR_IN; }

struct Fuse1 {
  const float* u;
  const float* W1;
  const float* b1;
  int act;
};

template <typename T, int CI, int CO, int OUT_MODE, int ACT, bool CT, bool DU, bool FUSE1 = false>
__global__ void __launch_bounds__(Cfg<T, CI, CO, CT, DU>::THREADS, Cfg<T, CI, CO, CT, DU>::MINB)
conv_xn_kernel(const T* __restrict__ in, int N, int Ny, int B, const uint8_t* __restrict__ Wp,
               const float* __restrict__ bias, int co_real, void* __restrict__ out0_,
               float* __restrict__ out1, int planar_async, int pf, int dbg, unsigned long long* __restrict__ ts,
               Fuse1 f1, int bulkA_, FluxEpi fe) {
  // bulkA: the contiguous-tile operand stages are filled by cp.async.bulk copies (one per (column, q) run
  // of 130 rows, split at the periodic wrap) issued by producer warp 0, completing on the stage's
  // mbarrier -- the copies run on the async (TMA) engine instead of 1560 16-B LSU requests per stage
  const bool bulkA = CT && !C_PLANAR_IN_<T, CI, CO, CT, DU>() && !FUSE1 && (bulkA_ & 1) != 0;
  // bulkA_ bit1: the producer's activation copies carry an L2 evict_first hint (read once per layer)
  const bool l2ef = (bulkA_ & 2) != 0;
  // dbg: measurement knobs, compiled in only with -DLD_XN_KNOBS (env LD_XN_DEBUG): bit0 the
  // producer skips the A copies, bit1 the epilogue skips math and stores, bit2 the MMA thread
  // skips the MMAs (commits only), bit3 the producer skips the W bulk copies, bit4 ReLU instead
  // of GELU, bit5 the epilogue skips the stores
#ifndef LD_XN_KNOBS
  dbg = 0;
#endif
  constexpr int XPK = xp_of<OUT_MODE, CT, DU>();
  using C = Cfg<T, CI, CO, CT, DU, XPK>;
  constexpr int NCOL = C::NCOL_, XP = C::XP_;   // this variant's columns / positions per tile
  constexpr int FE_PITCH = fe_pitch<XP>();
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* const stages = smem + C::W_OFF;   // [W (resident)] [NSTAGE stages] [barriers ...]
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + C::NSTAGE * C::STAGE);
  uint64_t* full = bars;                     // [NSTAGE]
  uint64_t* empty = bars + C::NSTAGE;        // [NSTAGE]
  uint64_t* tm_full = bars + 2 * C::NSTAGE;  // [2]
  uint64_t* tm_empty = tm_full + 2;          // [2]
  uint64_t* wbar = tm_empty + 2;             // resident weights landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + 3);
  float* sBias = reinterpret_cast<float*>(tm_empty + 4);   // CO floats (then 32 words of strip origins)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto stamp = [&](int slot) {   // measurement only (-DLD_XN_KNOBS, LD_XN_DEBUG bit 6)
#if defined(LD_XN_KNOBS)
    if (ts != nullptr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[blockIdx.x * 8 + slot] = t;
    }
#else
    (void)slot;
#endif
  };
  auto tacc = [&](int slot, long long cyc) {   // per-role wait-cycle totals (measurement only)
#if defined(LD_XN_KNOBS) && !defined(LD_XN_NOTIMING)
    if (ts != nullptr) atomicAdd(ts + XN_TSC * 8 + blockIdx.x * 8 + slot, (unsigned long long)cyc);
#else
    (void)slot; (void)cyc;
#endif
  };
  auto tstamp = [&](int tile_it, int ev) {   // per-tile event times, tiles 0 and 1 of the CTA (measurement)
#if defined(LD_XN_KNOBS)
    if (ts != nullptr && tile_it < 2) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[2 * XN_TSC * 8 + blockIdx.x * 16 + ev * 2 + tile_it] = t;
    }
#else
    (void)tile_it; (void)ev;
#endif
  };
  if (threadIdx.x == 0) stamp(0);
  // Domain: N (x, periodic, power of two) by Ny (y, periodic, any multiple of RY: the slab
  // decomposition runs the net on extended slabs whose wrapped edge rows are discarded)
  const int nstrips = B * (N / XP) * (Ny / RY);
  const int ntiles = (nstrips + NG - 1) / NG;
  // streamed weights: the first NSTAGE stages' W blocks are issued before the PDL wait (they do
  // not depend on the previous kernel), the producer loop skips them
  const int my_tiles = (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1;
  const int w_pre = (C::W_RES || (dbg & 8)) ? 0 : (my_tiles * C::NKS < C::NSTAGE ? my_tiles * C::NKS : C::NSTAGE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NSTAGE; ++s) {
      // producer arrivals (+ the per-stage W expect_tx); bulk-copy A fills: one expect_tx arrival
      mbar_init(full + s, bulkA ? (C::W_RES ? 1 : 2) : (C::W_RES ? C::NPT : C::NPT + 1));
      mbar_init(empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tm_full + s, 1);
      mbar_init(tm_empty + s, 32 * C::NEW);   // every epilogue thread
    }
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (C::W_RES) {   // resident weights: one bulk copy, independent of the previous kernel (PDL)
      mbar_arrive_tx(wbar, C::W_TOTAL);
      for (int off = 0; off < C::W_TOTAL; off += 65536) {
        const int nb = C::W_TOTAL - off < 65536 ? C::W_TOTAL - off : 65536;
        bulk_g2s(smem + off, Wp + off, (uint32_t)nb, wbar);
      }
    }
    for (int k = 0; k < w_pre; ++k) {
      mbar_arrive_tx(full + k, C::W_STAGE);
      bulk_g2s(stages + k * C::STAGE + C::A_STAGE, Wp + (size_t)(k % C::NKS) * C::W_STAGE, C::W_STAGE, full + k);
    }
  }
  if (C::PLANAR_IN && !C::F16 && planar_async) {   // TF32 first layer: zero words stay zero (see producer)
    for (int i = threadIdx.x; i < C::NSTAGE * C::STAGE / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(stages)[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) stamp(1);
  pdl_launch();   // the next kernel may start its prologue as SMs free up
  // The previous kernel's output (our input) is visible after griddepcontrol.wait.  Only the
  // producer reads it; it waits after setting up its first tile.  Everything else this CTA
  // does (MMAs, epilogue stores into the buffer the previous kernel read) is ordered after
  // the producer's copies through the stage / accumulator barriers.
  if (warp >= C::NPW) pdl_wait();
  if (threadIdx.x == 0) stamp(2);

  auto wy = [Ny](int y) { return y < 0 ? y + Ny : (y >= Ny ? y - Ny : y); };

  if (warp < C::NPW) {
    // ===================== producer (4 warps, coalesced cp.async) =====================
    // Activation layout [b][ks][q][x][y][16 B]; the stage's 1920 16-B chunks are numbered
    // idx = ((c * 2 + q) * 16 + g) * 10 + r (= their shared-memory slot), and thread t copies
    // idx = t + NPT i: consecutive lanes take consecutive rows of a strip and strips are
    // consecutive in y, so a warp instruction reads ~512 contiguous bytes (measured
    // tests/tools/copy_microbench.cu: ~64 B/clk/SM; profiles/r01_copy_engines.log).  Completion
    // is signalled with cp.async.mbarrier.arrive.noinc, so the producer never waits for its
    // own copies; the MMA thread issues the proxy fence after acquiring the stage.
    constexpr int NCH = NCOL * 2 * C::ARH;          // 1920 (1560 with CT) chunks per stage
    constexpr int CPT = (NCH + C::NPT - 1) / C::NPT;   // 15 (13) per thread with 128 producer threads
    const int tid = threadIdx.x;
    uint32_t* sOrg = reinterpret_cast<uint32_t*>(sBias + 64);   // per-strip chunk offset base [16]
    const size_t ks_stride = (size_t)2 * N * Ny;                // 16-B chunks per K-step block
    int k = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      // strip origins of this tile -> per-chunk offsets (in 16-B units, K-step 0)
      uint32_t off[CPT];
      {
        asm volatile("bar.sync 1, %0;" ::"n"(C::NPT) : "memory");   // previous tile's sOrg reads are done
        if (tid < NG) {
          int s = tile * NG + tid;
          if (s >= nstrips) s = 0;   // ragged last tile: load anything valid, never stored
          int b, x0, y0;
          strip_origin(s, N, Ny, XP, b, x0, y0);
          sOrg[tid] = (uint32_t)b;
          sOrg[16 + tid] = (uint32_t)(x0 | (y0 << 16));
        }
        asm volatile("bar.sync 1, %0;" ::"n"(C::NPT) : "memory");
        // first layer, 4-byte async gather (planar_async): work item j = tid + NPT i takes (row (g, r), column
        // c) with c fastest, so a warp instruction reads ~5 rows x 6 consecutive x of the planar field (a few
        // sectors) instead of 32 rows (32 sectors, 4 B used in each); the q = 1 chunks (zero) are skipped
        const bool gather_x = C::PLANAR_IN && !C::F16 && !CT && planar_async && !(bulkA_ & 4);
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
          if (gather_x) {
            const int j = tid + C::NPT * i;
            if (j >= NCOL * NG * RH) { off[i] = 0x80000000u; continue; }
            const int c = j % NCOL, rest = j / NCOL, g = rest / RH, r = rest - g * RH;
            const uint32_t b = sOrg[g], xy = sOrg[16 + g];
            const int x0 = (int)(xy & 0xffff), y0 = (int)(xy >> 16);
            off[i] = (uint32_t)(((size_t)b * 2 * Ny + wy(y0 - 1 + r)) * N + wrap(x0 - 1 + c, N));
            continue;
          }
          const int idx = tid + C::NPT * i < NCH ? tid + C::NPT * i : NCH - 1;
          int r, g, cq;
          if constexpr (CT) {   // rows r of the tile's column (all strips: origin of strip 0)
            r = idx % C::ARH; g = 0; cq = idx / C::ARH;
          } else {
            r = idx % RH; g = (idx / RH) % NG; cq = idx / (RH * NG);
          }
          const int q = cq & 1, c = cq >> 1;
          const uint32_t b = sOrg[g], xy = sOrg[16 + g];
          const int x0 = (int)(xy & 0xffff), y0 = (int)(xy >> 16);
          if constexpr (C::PLANAR_IN)   // element offset of (b, y, x) in the planar field
            off[i] = (uint32_t)(((size_t)b * 2 * Ny + wy(y0 - 1 + r)) * N + wrap(x0 - 1 + c, N)) |
                     (q == 1 ? 0x80000000u : 0u);
          else
            off[i] = (uint32_t)((((size_t)b * C::NKS * 2 + q) * N + wrap(x0 - 1 + c, N)) * Ny + wy(y0 - 1 + r));
        }
      }
      if (tile == (int)blockIdx.x) pdl_wait();   // first tile set up: now the input is needed
      if constexpr (!C::PLANAR_IN) {
        // L2 prefetch of the operand runs of this CTA's tile `pf` tiles ahead: the DRAM latency of
        // the activations is paid while the current tiles run, so the cp.async stages (all the
        // shared memory the ring has) only wait for L2
        const int nt = tile + pf * (int)gridDim.x;
        if (pf > 0 && nt < ntiles) {
          constexpr int ITEMS = C::NKS * 2 * NCOL * (CT ? 1 : NG);
          for (int it2 = tid; it2 < ITEMS; it2 += C::NPT) {
            const int g = CT ? 0 : it2 % NG;
            int r = CT ? it2 : it2 / NG;
            const int c = r % NCOL;
            r /= NCOL;
            const int q = r & 1, ks = r >> 1;
            const int sn = nt * NG + g;
            if (sn >= nstrips) continue;
            int b, x0, y0;
            strip_origin(sn, N, Ny, XP, b, x0, y0);
            const uint4* src = reinterpret_cast<const uint4*>(in) +
                               ((((size_t)b * C::NKS + ks) * 2 + q) * N + wrap(x0 - 1 + c, N)) * Ny + y0;
            // CT: the tile's 128 rows of this column (one 2-KB run); else the strip's 8 rows (128 B)
            prefetch_l2(src, CT ? (uint32_t)(NG * RY * 16) : (uint32_t)(RY * 16));
          }
        }
      }
      for (int ks = 0; ks < C::NKS; ++ks, ++k) {
        const int slot = k % C::NSTAGE;
        mbar_wait_backoff(empty + slot, ((k / C::NSTAGE) & 1) ^ 1);
        uint8_t* stA = stages + slot * C::STAGE;
        if (tid == 0 && !C::W_RES && k >= w_pre) {
          if (dbg & 8) {
            mbar_arrive(full + slot);
          } else {
            mbar_arrive_tx(full + slot, C::W_STAGE);
            bulk_g2s(stA + C::A_STAGE, Wp + (size_t)ks * C::W_STAGE, C::W_STAGE, full + slot);
          }
        }
        if (C::PLANAR_IN && !C::F16 && planar_async) {
          // first layer, TF32, grids of several tiles per CTA (planar_async): u and v land in
          // words 0 and 1 of each q = 0 chunk by 4-byte cp.async (the stages were zeroed at
          // start-up and the other words never change), so the producer does not wait for its
          // loads (c3 first layer 145 -> 123 us; at c2, two tiles per CTA, the zeroing costs more)
          const float* up = reinterpret_cast<const float*>(in);
          const uint32_t st0 = smem_u32(stA);
          const bool gx = !CT && !(bulkA_ & 4);   // item order of the gather above (c fastest)
#pragma unroll
          for (int i = 0; i < CPT; ++i) {
            if (tid + C::NPT * i >= NCH) break;
            if (!(off[i] & 0x80000000u)) {
              int slot_idx = tid + C::NPT * i;
              if (gx) {   // chunk ((c * 2 + 0) * NG + g) * RH + r of item j
                const int j = slot_idx, c = j % NCOL, rest = j / NCOL, g = rest / RH, r = rest - g * RH;
                slot_idx = (c * 2 * NG + g) * RH + r;
              }
              const uint32_t d = st0 + (uint32_t)slot_idx * 16u;
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(up + off[i]) : "memory");
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d + 4u), "l"(up + off[i] + (size_t)N * Ny)
                           : "memory");
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + slot)) : "memory");
        } else if constexpr (FUSE1) {
          // layer 1 of this K-step's KBE channels for the tile's NCOL x ARH cells, fp32, into the stage
          static_assert(CT, "FUSE1 needs the contiguous-tile layout");
          const int ch0 = ks * C::KBE;
          const uint32_t b = sOrg[0], xy = sOrg[16];
          const int x0 = (int)(xy & 0xffff), y0 = (int)(xy >> 16);
          const float* ub = f1.u + (size_t)b * 2 * N * Ny;
          for (int cell = tid; cell < NCOL * C::ARH; cell += C::NPT) {
            const int c = cell / C::ARH, r = cell - c * C::ARH;
            unsigned long long z[C::KBE / 2];
#pragma unroll
            for (int k = 0; k < C::KBE / 2; ++k) z[k] = 0ull;
#pragma unroll 1
            for (int dy = -1; dy <= 1; ++dy) {
              const int yy = wy(y0 - 1 + r + dy);
#pragma unroll
              for (int dx = -1; dx <= 1; ++dx) {
                const int xx = wrap(x0 - 1 + c + dx, N);
                const int tap = (dy + 1) * 3 + (dx + 1);
#pragma unroll
                for (int ci = 0; ci < 2; ++ci) {
                  const unsigned long long vv = f2_splat(__ldg(ub + ((size_t)ci * Ny + yy) * N + xx));
                  const float4* wq = reinterpret_cast<const float4*>(f1.W1 + (tap * 2 + ci) * CI + ch0);
#pragma unroll
                  for (int k4 = 0; k4 < C::KBE / 4; ++k4) {
                    const float4 wv = __ldg(wq + k4);
                    z[2 * k4] = f2_fma(f2_pack(wv.x, wv.y), vv, z[2 * k4]);
                    z[2 * k4 + 1] = f2_fma(f2_pack(wv.z, wv.w), vv, z[2 * k4 + 1]);
                  }
                }
              }
            }
            float v[C::KBE];
#pragma unroll
            for (int k = 0; k < C::KBE / 2; ++k) {
              float a0, a1;
              f2_unpack(z[k], a0, a1);
              const float bb0 = __ldg(f1.b1 + ch0 + 2 * k), bb1 = __ldg(f1.b1 + ch0 + 2 * k + 1);
              if (f1.act == 1) {
                gelu_fast2(a0, a1, bb0, bb1, v[2 * k], v[2 * k + 1]);
              } else {
                v[2 * k] = fmaxf(a0 + bb0, 0.f);
                v[2 * k + 1] = fmaxf(a1 + bb1, 0.f);
              }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q)
              store_vec<T>(reinterpret_cast<T*>(stA + ((c * 2 + q) * C::ARH + r) * 16), v + q * C::EPC, C::EPC);
          }
          fence_proxy_async();
          mbar_arrive(full + slot);
        } else if (C::PLANAR_IN) {
          // first layer: channels (u, v, 0, ..., 0) assembled from the planar fp32 field
          // [b][2][N][N] -- 2 real channels of the 16 (F16 / BF16) of one K-step
          const float* up = reinterpret_cast<const float*>(in);
#pragma unroll
          for (int i = 0; i < CPT; ++i) {
            if (tid + C::NPT * i >= NCH) break;
            uint4 val = make_uint4(0u, 0u, 0u, 0u);
            if (!(off[i] & 0x80000000u)) {
              const float a = __ldg(up + off[i]), bb = __ldg(up + off[i] + (size_t)N * Ny);
              if (C::FMT == 1) {
                const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, bb);
                val.x = *reinterpret_cast<const uint32_t*>(&h2);
              } else if (C::F16) {
                const __half2 h2 = __floats2half2_rn(a, bb);
                val.x = *reinterpret_cast<const uint32_t*>(&h2);
              } else {
                val.x = __float_as_uint(a);
                val.y = __float_as_uint(bb);
              }
            }
            *reinterpret_cast<uint4*>(stA + (tid + C::NPT * i) * 16) = val;
          }
          fence_proxy_async();
          mbar_arrive(full + slot);
        } else {
          if (dbg & 512) {   // measurement knob: the same byte count from one linear region
            const uint4* src = reinterpret_cast<const uint4*>(in) + ((size_t)tile * C::NKS + ks) * NCH;
#pragma unroll
            for (int i = 0; i < CPT; ++i)
              if (tid + C::NPT * i < NCH) cp_async16(stA + (tid + C::NPT * i) * 16, src + tid + C::NPT * i);
          } else if (bulkA) {
            if (tid < 32) {
              if (tid == 0) mbar_arrive_tx(full + slot, (uint32_t)(NCOL * 2 * C::ARH * 16));
              __syncwarp();
              if (tid < NCOL * 2) {
                const int c = tid >> 1, q = tid & 1;
                const uint32_t b = sOrg[0], xy = sOrg[16];
                const int x0 = (int)(xy & 0xffff), y0 = (int)(xy >> 16);
                const uint4* col = reinterpret_cast<const uint4*>(in) +
                                   ((((size_t)b * C::NKS + ks) * 2 + q) * N + wrap(x0 - 1 + c, N)) * Ny;
                uint8_t* dst = stA + (size_t)(c * 2 + q) * C::ARH * 16;
                for (int r0 = 0; r0 < C::ARH;) {   // rows y0-1 .. y0+128, split where they wrap
                  const int gy = wy(y0 - 1 + r0);
                  const int len = C::ARH - r0 < Ny - gy ? C::ARH - r0 : Ny - gy;
                  bulk_g2s(dst + r0 * 16, col + gy, (uint32_t)(len * 16), full + slot);
                  r0 += len;
                }
              }
            }
            continue;   // no per-thread arrival: the expect_tx arrival completes with the copies' bytes
          } else if (!(dbg & 1)) {
            const uint4* src = reinterpret_cast<const uint4*>(in) + (size_t)ks * ks_stride;
            if (l2ef) {
              const uint64_t pol = l2_policy_evict_first();
#pragma unroll
              for (int i = 0; i < CPT; ++i)
                if (tid + C::NPT * i < NCH) cp_async16_hint(stA + (tid + C::NPT * i) * 16, src + off[i], pol);
            } else {
#pragma unroll
              for (int i = 0; i < CPT; ++i)
                if (tid + C::NPT * i < NCH) cp_async16(stA + (tid + C::NPT * i) * 16, src + off[i]);
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + slot))
                       : "memory");
        }
      }
    }
    if (threadIdx.x == 0) stamp(3);
  } else if (warp == C::MMA_WARP) {
    // ===================== MMA issuer =====================
    // The whole warp runs the loop convergently (waits by all lanes); each K-step's 18 MMAs and
    // its commits are issued from ONE elect.sync region.  Issuing from a divergent `lane == 0`
    // branch made the compiler wrap every tcgen05.mma in its own elect / waterfall loop (5 extra
    // dependent instructions per MMA), and the measured single-thread issue latency then paced
    // the N = 64 / 128 MMAs (ncu warp sampling: MMA warp in "wait" / "not selected").
    const uint32_t s0 = smem_u32(stages);
    const uint64_t adesc0 = sdesc(s0, C::LBO_A, C::SBO_A);
    const uint64_t bdesc0 = C::W_RES ? sdesc(smem_u32(smem), C::LBO_B, C::SBO_B)
                                     : sdesc(s0 + C::A_STAGE, C::LBO_B, C::SBO_B);
    if (C::W_RES) mbar_wait(wbar, 0);
    int k = 0, it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int ab = it % C::NACC;
      const long long c0 = clock64();
      mbar_wait(tm_empty + ab, ((it / C::NACC) & 1) ^ 1);
      if (lane == 0) tacc(2, clock64() - c0);
      tc_fence_after();
      const uint32_t dacc = tmem_base + (uint32_t)(ab * C::ACC_COLS);
      for (int ks = 0; ks < C::NKS; ++ks, ++k) {
        const int slot = k % C::NSTAGE;
        const long long c1 = clock64();
        mbar_wait(full + slot, (k / C::NSTAGE) & 1);
        if (lane == 0) tacc(3, clock64() - c1);
        if (!(dbg & 256)) fence_proxy_async();   // cp.async (generic proxy) writes -> tcgen05.mma (async proxy) reads
        tc_fence_after();
        const uint64_t ad = adesc0 + (uint64_t)((slot * C::STAGE) >> 4);
        const uint64_t bd = bdesc0 + (uint64_t)(((C::W_RES ? ks * C::W_STAGE : slot * C::STAGE)) >> 4);
        const long long ci0 = clock64();
        if (lane == 0 && ks == 0) tstamp(it, 0);
        if (elect_one()) {
          if (dbg & 4) {
          } else if (ks == 0) {
            issue_kstep<C::F16, C::FMT, CO, true, C::A_QBYTES, XP>(dacc, ad, bd);
          } else {
            issue_kstep<C::F16, C::FMT, CO, false, C::A_QBYTES, XP>(dacc, ad, bd);
          }
          tc_commit(empty + slot);
          if (ks == C::NKS - 1) tc_commit(tm_full + ab);
        }
        __syncwarp();
        if (lane == 0) tacc(6, clock64() - ci0);
        if (lane == 0 && ks == C::NKS - 1) tstamp(it, 1);
      }
    }
    if (lane == 0) stamp(4);
  } else if (warp >= C::NPW) {
    // ===================== epilogue =====================
    // warp w: TMEM lane quarter w % 4 (hardware rule); epilogue warp e = w - NPW covers output
    // positions p = e / 4 + j * NEW / 4 (one position with 16 warps, two with 8)
    const int qd = warp & 3, e_w = warp - C::NPW;
    const int m = qd * 32 + lane;                      // TMEM lane = GEMM row
    const int g = m >> 3, i = m & 7;
    const size_t plane = (size_t)N * Ny;
    const int ep0 = 32 * C::NPW;                       // first epilogue thread (measurement stamps)
    // the bias is staged by the epilogue warps themselves (named barrier 2), off the CTA's
    // start-up path: they have nothing else to do before the first accumulator is ready
    for (int i = threadIdx.x - ep0; i < CO; i += 32 * C::NEW) sBias[i] = __ldg(bias + i);
    asm volatile("bar.sync 2, %0;" ::"n"(32 * C::NEW) : "memory");
    int it = 0;
    float* const Us = reinterpret_cast<float*>(smem + C::SMEM);   // OUT_FLUX: [2][FE_ROWS][FE_PITCH]
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int ab = it % C::NACC;
      if constexpr (OUT_MODE == OUT_FLUX) {
        // the tile's field neighbourhood (rows y0-3 .. y0+130, columns x0-3 .. x0+6, periodic wrap); the
        // previous tile's readers are done (named barrier 3 at the end of every tile)
        int fb, fx0, fy0;
        strip_origin(tile * NG, N, Ny, XP, fb, fx0, fy0);
        const float* Ub = fe.U + (size_t)fb * 2 * N * Ny;
        constexpr int FEC = XP + 6;   // staged columns x0 - 3 .. x0 + XP + 2
        for (int j = threadIdx.x - ep0; j < 2 * FE_ROWS * FEC; j += 32 * C::NEW) {
          const int c = j / (FE_ROWS * FEC), r = j - c * (FE_ROWS * FEC), ry = r / FEC, rx = r - ry * FEC;
          int gyy = fy0 - 3 + ry;
          gyy = gyy < 0 ? gyy + Ny : (gyy >= Ny ? gyy - Ny : gyy);
          Us[(c * FE_ROWS + ry) * FE_PITCH + rx] = __ldg(Ub + ((size_t)c * Ny + gyy) * N + ((fx0 - 3 + rx) & (N - 1)));
        }
        asm volatile("bar.sync 3, %0;" ::"n"(32 * C::NEW) : "memory");
      }
      const long long c0 = clock64();
      mbar_wait_backoff(tm_full + ab, (it / C::NACC) & 1);
      const long long c1 = clock64();
      if (threadIdx.x == ep0) tacc(4, c1 - c0);
      if (threadIdx.x == ep0) tstamp(it, 2);
      tc_fence_after();
      const int s = tile * NG + g;
      const bool valid = s < nstrips;   // ragged last tile: lanes of missing strips store nothing
      int b, x0, y0;
      strip_origin(valid ? s : 0, N, Ny, XP, b, x0, y0);
      const int gy = y0 + i;
#pragma unroll 1
      for (int pj = 0; pj < XP * 4 / C::NEW; ++pj) {
      const int p = (e_w >> 2) + pj * (C::NEW / 4);
      const int gx = x0 + p;
      const bool last_p = pj == XP * 4 / C::NEW - 1;
      // CH-column chunks (CH live values); the accumulator is released after the last chunk is
      // in registers.  (Measured: issuing chunk h+1's tcgen05.ld before activating chunk h is
      // 5% slower at c2.)
      constexpr int CH = OUT_MODE == OUT_BLOCKED ? XN_EPI_CH : 32;
#pragma unroll
      for (int h = 0; h < CO / CH; ++h) {
        uint32_t r1[CH];
        if (!(dbg & 128))
          tmem_ld_async<CH>(tmem_base + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ab * C::ACC_COLS + p * CO + h * CH), r1);
        tmem_ld_wait();
        tmem_regs_ready<CH>(r1);
        if (h == CO / CH - 1 && last_p) {
          tc_fence_before();
          mbar_arrive(tm_empty + ab);
        }
        float v[CH];
        if (dbg & 2) {   // measurement knob: no epilogue math (loop-invariant branch)
#pragma unroll
          for (int o = 0; o < CH; ++o) v[o] = __uint_as_float(r1[o]);
        } else if (ACT == 0 || (dbg & 16)) {
#pragma unroll
          for (int o = 0; o < CH; ++o) v[o] = fmaxf(__uint_as_float(r1[o]) + sBias[h * CH + o], 0.f);
        } else {
#if XN_GELU2
          if constexpr (ACT == 1) {   // packed fp32 pairs (FFMA2 / FMUL2 / FADD2)
#pragma unroll
            for (int o = 0; o < CH; o += 2)
              gelu_fast2(__uint_as_float(r1[o]), __uint_as_float(r1[o + 1]), sBias[h * CH + o],
                         sBias[h * CH + o + 1], v[o], v[o + 1]);
          } else
#endif
#pragma unroll
          for (int o = 0; o < CH; ++o) {
            const float t = __uint_as_float(r1[o]) + sBias[h * CH + o];
            v[o] = ACT == 1 ? gelu_fast(t) : t;
          }
        }
        if (!valid || (dbg & 2) || ((dbg & 32) && v[0] != 1234.5f)) {
        } else if (OUT_MODE == OUT_BLOCKED) {
          // act[b][ks][q][x][y][16 B]: the 32 lanes of a warp are 32 consecutive y, so every
          // 16-B store instruction writes one contiguous 512-B run
#pragma unroll
          for (int kk = 0; kk < CH / C::EPC; ++kk) {
            const int c0 = h * CH + kk * C::EPC;   // first channel of this 16-B run
            const int ks = c0 / C::KBE, qq = (c0 / C::EPC) & 1;
            T* dst = reinterpret_cast<T*>(out0_) +
                     (((((size_t)b * C::NKS_OUT + ks) * 2 + qq) * N + gx) * Ny + gy) * C::EPC;
            if (dbg & 2048)   // measurement knob: every CTA stores into its own 16-KB-per-warp scratch
              dst = reinterpret_cast<T*>(out0_) + ((size_t)blockIdx.x * 16 + (warp - 4)) * 32 * 32 * 4 +
                    (size_t)kk * 32 * 4 + lane * C::EPC;
            store_vec<T>(dst, v + kk * C::EPC, C::EPC);
          }
        } else if constexpr (OUT_MODE == OUT_FLUX) {
          // own faces of cell (gx, gy): tile-local row m (the 16 strips are one 128-row segment), column p
          const float* ux = Us + (0 * FE_ROWS + m + 3) * FE_PITCH + p;   // x-face taps x-3 .. x+2
          const float* vx = Us + (1 * FE_ROWS + m + 3) * FE_PITCH + p;
          float uI, uD, vI, vD;
          face_taps2<1>(v, ux, vx, uI, uD, vI, vD);
          float gu = uD * fe.inv_h, gv = vD * fe.inv_h;
          float adv = fe.gamma * uI;
          const float fxu = adv * uI - fe.nu * gu, fxv = adv * vI - fe.nu * gv;
          const float* uy = Us + (0 * FE_ROWS + m) * FE_PITCH + p + 3;       // y-face taps y-3 .. y+2
          const float* vy = Us + (1 * FE_ROWS + m) * FE_PITCH + p + 3;
          face_taps2<FE_PITCH>(v + 12, uy, vy, uI, uD, vI, vD);
          gu = uD * fe.inv_h; gv = vD * fe.inv_h;
          adv = fe.gamma * vI;
          const float fyu = adv * uI - fe.nu * gu, fyv = adv * vI - fe.nu * gv;
          const size_t cell = ((size_t)b * N + gx) * Ny + gy;
          reinterpret_cast<float4*>(out0_)[cell] = make_float4(fxu, fxv, fyu, fyv);
          if (out1 != nullptr && co_real > 24)
            *reinterpret_cast<float2*>(out1 + cell * 2) = make_float2(v[24], v[25]);
        } else if (OUT_MODE == OUT_STENCIL) {
          // x-major stencils w[b][x][y][24] and TC term e[b][x][y][2] (CO = 32): a warp writes
          // 32 consecutive cells = one contiguous 3-KB run
          const size_t cell = ((size_t)b * N + gx) * Ny + gy;
          float4* w4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(out0_) + cell * 24);
#pragma unroll
          for (int o = 0; o < 6; ++o) w4[o] = make_float4(v[4 * o], v[4 * o + 1], v[4 * o + 2], v[4 * o + 3]);
          if (out1 != nullptr && co_real > 24)
            *reinterpret_cast<float2*>(out1 + cell * 2) = make_float2(v[24], v[25]);
        } else {
          float* ob = reinterpret_cast<float*>(out0_) + (size_t)b * co_real * plane + (size_t)gy * N + gx;
#pragma unroll
          for (int o = 0; o < CH; ++o)
            if (h * CH + o < co_real) ob[(size_t)(h * CH + o) * plane] = v[o];
        }
      }
      }   // positions
      if (threadIdx.x == ep0) tacc(5, clock64() - c1);
      if (threadIdx.x == ep0) tstamp(it, 3);
      if constexpr (OUT_MODE == OUT_FLUX) asm volatile("bar.sync 3, %0;" ::"n"(32 * C::NEW) : "memory");
    }
    if (threadIdx.x == 32 * C::NPW) stamp(5);
  }
  __syncthreads();
  if (threadIdx.x == 0) stamp(6);
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                 : "memory");
  }
}

template <typename T, int CI, int CO, int OM, int ACT, bool CT, bool DU = false, bool FUSE1 = false>
cudaError_t set_attr() {
  constexpr int XPK = xp_of<OM, CT, DU>();
  return cudaFuncSetAttribute(conv_xn_kernel<T, CI, CO, OM, ACT, CT, DU, FUSE1>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              Cfg<T, CI, CO, CT, DU, XPK>::SMEM + (OM == OUT_FLUX ? fe_smem<XPK>() : 0));
}

template <typename T, int CI, int CO, int OM, int ACT, bool CT, bool DU = false, bool FUSE1 = false>
cudaError_t launch(const void* in, int N, int Ny, int B, const void* Wp, const float* bias, int co_real, void* o0,
                   float* o1, cudaStream_t st, Fuse1 f1 = Fuse1{nullptr, nullptr, nullptr, 0},
                   FluxEpi fe = FluxEpi{nullptr, 0.f, 0.f, 0.f}) {
  constexpr int XPK = xp_of<OM, CT, DU>();
  using C = Cfg<T, CI, CO, CT, DU, XPK>;
  static_assert(OM != OUT_FLUX || C::SMEM + fe_smem<XPK>() <= (DU ? 113 : 227) * 1024, "flux epilogue smem");
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int nstrips = B * (N / XPK) * (Ny / RY);
  const int ntiles = (nstrips + NG - 1) / NG;
  cudaLaunchConfig_t cfg = {};
  const int slots = C::MINB * sms;
  cfg.gridDim = dim3(ntiles < slots ? ntiles : slots);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM + (OM == OUT_FLUX ? fe_smem<XPK>() : 0);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // contiguous-tile stages by cp.async.bulk (LD_XN_BULKA=0/1 overrides; default below)
  static const int bulk_env = getenv("LD_XN_BULKA") ? atoi(getenv("LD_XN_BULKA")) : -1;
  const int bulkA = bulk_env >= 0 ? bulk_env : 0;
  // L2 evict_first on the activation reads, per layer kind (bit0 output layer with the flux epilogue,
  // bit1 hidden layers); LD_XN_L2EF overrides (measurement)
  static const int l2ef_env = getenv("LD_XN_L2EF") ? atoi(getenv("LD_XN_L2EF")) : -1;
  const int l2ef_mask = l2ef_env >= 0 ? l2ef_env : 0;
  const bool l2ef = (OM == OUT_FLUX && (l2ef_mask & 1)) || (OM == OUT_BLOCKED && CI != 2 && (l2ef_mask & 2));
  // first layer's 4-byte gather in the old row-per-lane order (LD_XN_GATHER_Y=1, measurement)
  static const bool gather_y = getenv("LD_XN_GATHER_Y") != nullptr;
  // L2 prefetch lead of the producer in tiles (0 = off); LD_XN_PF overrides (measurement)
  static const int pf_env = getenv("LD_XN_PF") ? atoi(getenv("LD_XN_PF")) : -1;
  const int pf = pf_env >= 0 ? pf_env : 0;   // measured: no gain on the hidden layers, 2x slower last layer
  static int dbg = -1;
  if (dbg < 0) {
    const char* e = getenv("LD_XN_DEBUG");
    dbg = e ? atoi(e) : 0;
  }
  unsigned long long* ts = nullptr;
#ifdef LD_XN_KNOBS
  static unsigned long long* ts_buf = nullptr;
  static int dumped = 0;
  static const int ts_ci = getenv("LD_XN_TS_CI") ? atoi(getenv("LD_XN_TS_CI")) : 64;   // layer to stamp
  static const int ts_co = getenv("LD_XN_TS_CO") ? atoi(getenv("LD_XN_TS_CO")) : 64;
  const bool want_ts = (dbg & 64) && CI == ts_ci && CO == ts_co && dumped < 4;
  if (want_ts) {
    if (ts_buf == nullptr) cudaMalloc(&ts_buf, (2 * XN_TSC * 8 + XN_TSC * 16) * sizeof(unsigned long long));
    cudaMemsetAsync(ts_buf, 0, (2 * XN_TSC * 8 + XN_TSC * 16) * sizeof(unsigned long long), st);
    ts = ts_buf;
  }
#endif
  cudaError_t err = cudaLaunchKernelEx(&cfg, conv_xn_kernel<T, CI, CO, OM, ACT, CT, DU, FUSE1>,
                                       reinterpret_cast<const T*>(in), N, Ny, B, reinterpret_cast<const uint8_t*>(Wp),
                                       bias, co_real, o0, o1, (int)(CI == 2 && ntiles > 2 * (int)cfg.gridDim.x), pf,
                                       dbg, ts, f1, bulkA | (l2ef ? 2 : 0) | (gather_y ? 4 : 0), fe);
#ifdef LD_XN_KNOBS
  if (want_ts) {   // per-CTA phase timestamps (ns from the first CTA's start): avg / max over CTAs
    ++dumped;
    unsigned long long h[2 * XN_TSC * 8 + XN_TSC * 16];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, ts_buf, sizeof(h), cudaMemcpyDeviceToHost);
    const int g = (int)cfg.gridDim.x;
    unsigned long long t0 = ~0ull;
    for (int i = 0; i < g; ++i) t0 = h[i * 8] < t0 ? h[i * 8] : t0;
    fprintf(stderr, "[conv_xn ts] grid=%d", g);
    const char* nm[7] = {"entry", "alloc", "pdl", "prod_end", "mma_end", "epi_end", "exit"};
    for (int k = 0; k < 7; ++k) {
      double avg = 0; unsigned long long mx = 0;   // (per-CTA, 8 words each)
      for (int i = 0; i < g; ++i) { const unsigned long long d = h[i * 8 + k] - t0; avg += (double)d / g; mx = d > mx ? d : mx; }
      fprintf(stderr, "  %s %.0f/%llu", nm[k], avg, mx);
    }
    const char* wn[7] = {"prod_wait_empty", "prod_wait_copies", "mma_wait_tmem", "mma_wait_full", "epi_wait_full",
                         "epi_work", "mma_issue"};
    {   // per-tile events of the CTAs that ran 2 tiles: avg ns from the CTA's entry
      const char* en[4] = {"mma_first", "mma_last_commit", "epi_start", "epi_end"};
      double avg[4][2] = {{0}};
      int cnt = 0;
      for (int i = 0; i < g; ++i) {
        const unsigned long long* q = h + 2 * XN_TSC * 8 + i * 16;
        if (q[3 * 2 + 1] == 0) continue;   // one tile only
        ++cnt;
        for (int e2 = 0; e2 < 4; ++e2)
          for (int t = 0; t < 2; ++t) avg[e2][t] += (double)(q[e2 * 2 + t] - h[i * 8]) / 1.0;
      }
      {   // tile 0 of every CTA, ns from the first CTA's entry: avg / max
        double a0[4] = {0}; unsigned long long m0[4] = {0};
        for (int i = 0; i < g; ++i)
          for (int e2 = 0; e2 < 4; ++e2) {
            const unsigned long long d = h[2 * XN_TSC * 8 + i * 16 + e2 * 2] - t0;
            a0[e2] += (double)d / g; m0[e2] = d > m0[e2] ? d : m0[e2];
          }
        fprintf(stderr, "\n   tile 0, all CTAs (ns from first entry, avg/max):");
        for (int e2 = 0; e2 < 4; ++e2) fprintf(stderr, "  %s %.0f/%llu", en[e2], a0[e2], m0[e2]);
      }
      fprintf(stderr, "\n   2-tile CTAs (%d), ns from entry:", cnt);
      for (int t = 0; t < 2; ++t)
        for (int e2 = 0; e2 < 4; ++e2) fprintf(stderr, "  t%d.%s %.0f", t, en[e2], cnt ? avg[e2][t] / cnt : 0.0);
    }
    fprintf(stderr, "\n   cycles (avg over CTAs):");
    for (int k = 0; k < 7; ++k) {
      double avg = 0;
      for (int i = 0; i < g; ++i) avg += (double)h[XN_TSC * 8 + i * 8 + k] / g;
      fprintf(stderr, "  %s %.0f", wn[k], avg);
    }
    fprintf(stderr, "\n");
  }
#endif
  return err;
}

}  // namespace xn

bool tc_conv_available() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0;
}

// (T, CI, CO, out mode, activation): hidden layers (CI = CO = width, ReLU or GELU) and the
// linear output layer (CO = 32 padded, step layout or planar eval layout)
#define LD_XN_VARIANTS_T(X, T)                                                                           \
  X(T, 2, 64, xn::OUT_BLOCKED, 0, false) X(T, 2, 64, xn::OUT_BLOCKED, 1, false)                          \
  X(T, 2, 32, xn::OUT_BLOCKED, 0, false) X(T, 2, 32, xn::OUT_BLOCKED, 1, false)                          \
  X(T, 64, 64, xn::OUT_BLOCKED, 0, false) X(T, 64, 64, xn::OUT_BLOCKED, 1, false)                        \
  X(T, 64, 32, xn::OUT_STENCIL, -1, false) X(T, 64, 32, xn::OUT_PLANAR_ALL, -1, false)                   \
  X(T, 32, 32, xn::OUT_BLOCKED, 0, false) X(T, 32, 32, xn::OUT_BLOCKED, 1, false)                        \
  X(T, 32, 32, xn::OUT_STENCIL, -1, false) X(T, 32, 32, xn::OUT_PLANAR_ALL, -1, false)                   \
  X(T, 64, 64, xn::OUT_BLOCKED, 0, true) X(T, 64, 64, xn::OUT_BLOCKED, 1, true)                          \
  X(T, 32, 32, xn::OUT_BLOCKED, 0, true) X(T, 32, 32, xn::OUT_BLOCKED, 1, true)                          \
  X(T, 64, 32, xn::OUT_FLUX, -1, false) X(T, 32, 32, xn::OUT_FLUX, -1, false)                         \
  X(T, 64, 32, xn::OUT_FLUX, -1, true)
#define LD_XN_VARIANTS(X) LD_XN_VARIANTS_T(X, float) LD_XN_VARIANTS_T(X, __half) LD_XN_VARIANTS_T(X, __nv_bfloat16)
// two-CTAs-per-SM hidden layers (grids of <= ~2 tiles per SM)
#define LD_XN_DUAL_VARIANTS(X)                                                                           \
  X(float, 64, 64, xn::OUT_BLOCKED, 1, false) X(__half, 64, 64, xn::OUT_BLOCKED, 1, false)                 \
  X(float, 2, 64, xn::OUT_BLOCKED, 1, false) X(float, 64, 32, xn::OUT_STENCIL, -1, false)                 \
  X(float, 64, 32, xn::OUT_FLUX, -1, false)

cudaError_t tc_conv_prepare() {
  cudaError_t e = cudaSuccess;
#define LD_SET(T, CI, CO, OM, ACT, CT) \
  if (e == cudaSuccess) e = xn::set_attr<T, CI, CO, OM, ACT, CT>();
  LD_XN_VARIANTS(LD_SET)
#undef LD_SET
#define LD_SET_DU(T, CI, CO, OM, ACT, CT) \
  if (e == cudaSuccess) e = xn::set_attr<T, CI, CO, OM, ACT, CT, true>();
  LD_XN_DUAL_VARIANTS(LD_SET_DU)
#undef LD_SET_DU
#define LD_SET_F1(T, ACT) \
  if (e == cudaSuccess) e = xn::set_attr<T, 64, 64, xn::OUT_BLOCKED, ACT, true, false, true>();
  LD_SET_F1(float, 0) LD_SET_F1(float, 1) LD_SET_F1(__half, 0) LD_SET_F1(__half, 1)
  LD_SET_F1(__nv_bfloat16, 0) LD_SET_F1(__nv_bfloat16, 1)
#undef LD_SET_F1
  return e;
}

// The second layer with the first recomputed in its producer (FUSE1): 64 -> 64 hidden layer in the
// contiguous-tile form (Ny % 128 == 0); u planar [B][2][Ny][N] fp32, W1 / b1 the first layer's SIMT-
// layout weights [9][2][64] / bias [64].  Returns cudaErrorNotSupported when the shape does not qualify.
cudaError_t launch_conv_tc_fused1(const float* u, const float* W1, const float* b1, int act1, int N, int Ny, int B,
                                  const void* Wtc, const float* bias, int f16, int act, void* out0, cudaStream_t st) {
  if (Ny % (xn::NG * xn::RY) != 0 || N % xn::XP != 0) return cudaErrorNotSupported;
  const xn::Fuse1 f1{u, W1, b1, act1};
#define LD_L1(T, ACT)                                                                                        \
  if (xn::type_code<T>() == f16 && act == ACT)                                                               \
    return xn::launch<T, 64, 64, xn::OUT_BLOCKED, ACT, true, false, true>(nullptr, N, Ny, B, Wtc, bias, 64, out0, \
                                                                          nullptr, st, f1);
  LD_L1(float, 0) LD_L1(float, 1) LD_L1(__half, 0) LD_L1(__half, 1) LD_L1(__nv_bfloat16, 0) LD_L1(__nv_bfloat16, 1)
#undef LD_L1
  return cudaErrorNotSupported;
}

// bytes of the packed tcgen05 weight operand of one layer
size_t tc_weight_bytes(int ci, int co_pad, int f16) {
  const int kpad = ci < (f16 ? 16 : 8) ? (f16 ? 16 : 8) : ci;   // first layer: K padded to one K-step
  return (size_t)9 * kpad * co_pad * (f16 ? 2 : 4);
}

// Wt [tap][ci][co_pad] (fp32, tap = (dy+1)*3 + (dx+1)) -> per K-step blocks
//   [ks][dy 0..2][q 0..1][n = dxblk*co_pad + co][epc]   with dxblk 0,1,2 <-> dx = +1, 0, -1
// (K-major 16-B core columns: epc = 4 fp32 or 8 fp16 consecutive input channels).
void tc_pack_weights(const float* Wt, int ci, int co_pad, int f16, uint8_t* dst) {
  const int epc = f16 ? 8 : 4, nks = ci < 2 * epc ? 1 : ci / (2 * epc), nb = 3 * co_pad;
  for (int ks = 0; ks < nks; ++ks)
    for (int dy = 0; dy < 3; ++dy)
      for (int q = 0; q < 2; ++q)
        for (int n = 0; n < nb; ++n)
          for (int e = 0; e < epc; ++e) {
            const int dxblk = n / co_pad, co = n % co_pad, dx = 1 - dxblk;
            const int tap = dy * 3 + (dx + 1);
            const int c = ks * 2 * epc + q * epc + e;
            const float w = c < ci ? Wt[((size_t)tap * ci + c) * co_pad + co] : 0.f;   // zero-padded K
            const size_t idx = ((((size_t)ks * 3 + dy) * 2 + q) * nb + n) * epc + e;
            if (f16 == 2) reinterpret_cast<__nv_bfloat16*>(dst)[idx] = __float2bfloat16_rn(w);
            else if (f16) reinterpret_cast<__half*>(dst)[idx] = __float2half_rn(w);
            else reinterpret_cast<float*>(dst)[idx] = w;
          }
}

cudaError_t launch_conv_tc_ci(const void* in, int Ci, int N, int Ny, int B, const void* Wtc, const float* bias,
                              int co_pad,
                              int f16, int act, int out_mode, int co_real, void* out0, float* out1, cudaStream_t st,
                              const FluxEpi* fe) {
  if (Ny % xn::RY != 0 || N % xn::XP != 0) return cudaErrorInvalidValue;
  if (out_mode == xn::OUT_FLUX && (fe == nullptr || Ny % (xn::NG * xn::RY) != 0)) return cudaErrorInvalidValue;
  const FluxEpi fev = fe ? *fe : FluxEpi{nullptr, 0.f, 0.f, 0.f};
  // contiguous-tile operand layout whenever the 16 strips of a tile share one column
  static const bool ct_enabled = getenv("LD_XN_NO_CT") == nullptr;   // measurement knob
  // (hidden layers only: measured slower for the 32-column output layer, whose weights are resident
  // either way)
  // the output layer with the flux epilogue in the contiguous-tile form too (its tile is one 128-row column
  // segment anyway): c4 418 -> 410 us, c3 201 -> 197 us per launch; LD_XN_NO_CT_OUT=1 restores the strip form
  static const bool ct_out = getenv("LD_XN_NO_CT_OUT") == nullptr;
  const bool ct = ct_enabled && Ci != 2 && Ny % (xn::NG * xn::RY) == 0 &&
                  (out_mode == xn::OUT_BLOCKED ||
                   (ct_out && out_mode == xn::OUT_FLUX && Ci == 64 && co_pad == 32 && N % 8 == 0));
  // Two CTAs per SM (Cfg::DU) when the grid is at most two tiles per SM: measured at c2 (256
  // tiles) the step is 5% faster with the hidden and output layers in this form -- a finishing
  // CTA's slot takes the next layer's CTA (PDL) while its partner still runs -- and slower with
  // the first layer or F16 operands.  LD_XN_DUAL overrides (bit0 hidden, bit1 first, bit2 output).
  static const int dual_env = getenv("LD_XN_DUAL") ? atoi(getenv("LD_XN_DUAL")) : -1;
  const int layer_bit = Ci == 2 ? 2 : (out_mode == xn::OUT_BLOCKED ? 1 : 4);   // (OUT_FLUX: the output layer)
  const int ntiles = (B * (N / xn::XP) * (Ny / xn::RY) + xn::NG - 1) / xn::NG;
  const int dual_mode = dual_env >= 0 ? dual_env : (!f16 && ntiles <= 2 * 148 ? 1 | 4 : 0);
  const bool dual = (dual_mode & layer_bit) && !ct;
  if (dual) {
#define LD_LAUNCH_DU(T, CI, CO, OM, ACT, CT)                                                         \
    if (xn::type_code<T>() == f16 && Ci == CI && co_pad == CO && out_mode == OM && act == ACT) \
      return xn::launch<T, CI, CO, OM, ACT, CT, true>(in, N, Ny, B, Wtc, bias, co_real, out0, out1, st,      \
                                                      xn::Fuse1{nullptr, nullptr, nullptr, 0}, fev);
    LD_XN_DUAL_VARIANTS(LD_LAUNCH_DU)
#undef LD_LAUNCH_DU
  }
#define LD_LAUNCH(T, CI, CO, OM, ACT, CT)                                                            \
  if (xn::type_code<T>() == f16 && Ci == CI && co_pad == CO && out_mode == OM && act == ACT &&  \
      ct == CT)                                                                                      \
    return xn::launch<T, CI, CO, OM, ACT, CT>(in, N, Ny, B, Wtc, bias, co_real, out0, out1, st,              \
                                              xn::Fuse1{nullptr, nullptr, nullptr, 0}, fev);
  LD_XN_VARIANTS(LD_LAUNCH)
#undef LD_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace ld
