// common.cuh -- shared device helpers for the LDSolver sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define LD_DEVINL __device__ __forceinline__

namespace ld {

// Per-stage RK combination coefficients (Shu-Osher form):
//   out = a * u^n + b * X + c * dt * T + q * dt * acc  (+ e when add_e)
//   acc_out = (acc_init ? 0 : acc_in) + r * T        (RK4 only, when r != 0)
struct StageCoef {
  float a, b, c, q, r;
  int acc_init;   // 1: acc_in treated as zero (first RK4 stage)
  int add_e;      // 1: add the temporal-correction field e
};

// Fixed (base) stencils, channels as in w: wIx[6] wDx[6] wIy[6] wDy[6].
struct BaseStencil { float w[24]; };

// Physics parameters the fused flux kernel needs.
struct FluxParams {
  int n;            // N
  int batch;
  float h, inv_h;
  float nu;
  float gamma;      // 1/2 Burgers, 1 NS (R9)
  float dt;
  float drag;       // alpha
  int forced;       // 1 if force_amp != 0 or drag != 0
  const float* force_row;  // [N]: force_amp * sin(force_k * y_j), fp64-evaluated at init
  // Domain of the stage field X, the stencils w and the TC term e: N (x) by ny (y) rows, periodic
  // in both (single domain: ny = N).  The kernel computes the rows [y_off, y_off + rows) of it;
  // row y_off is global row gy0 (forcing).  out, u^n and acc are [B][2][*_rows][N] planes whose
  // row *_row0 is the first computed row (single domain: all N and 0).
  int ny, y_off, rows, gy0, o_rows, o_row0, un_rows, un_row0, a_rows, a_row0;
  // NEXT-2 branch on the faces [B][8][ny][N] (nullptr: off): added to the stencil face values
  // (x-face: interp u, v, d/dx u, v; y-face: interp u, v, d/dy u, v)
  const float* fno = nullptr;
};

// Flux epilogue of the net's output layer (conv_xn.cu OUT_FLUX): the stage field the net reads and the
// physics of the face fluxes (as in FluxParams).
struct FluxEpi {
  const float* U;   // planar [B][2][N][N] stage field
  float gamma, nu, inv_h;
};

// Arguments of the pencil projection passes (pencil.cu), shared with the host orchestration.
struct PencilArgs {
  int N, B, P, rank;       // grid, batch, ranks, this rank
  float half_inv_h, scale; // 1/(2h); 1/N^2
  // stage field U* (own rows): element (b, c, y, x) at U[((b * 2 + c) * rows + row0 + y) * N + x]
  const float* U;
  int rows, row0;
  // v rows just below / above the own rows (y0 - 1, y0 + n): element (b, x) at vb[b * vstride + x]
  const float* vbelow;
  const float* vabove;
  long long vstride;
};

// erf by Abramowitz & Stegun 7.1.26: erf(z) = 1 - t (a1 + t (a2 + ... a5 t)) exp(-z^2),
// t = 1 / (1 + p z), |error| <= 1.5e-7 (<= 6e-7 with fp32 evaluation, i.e. fp32 rounding
// level).  Branch- and select-free: 2 MUFU (rcp, ex2) + 8 FMA-pipe ops, about half the
// instructions of erff(); the epilogue GELU is issued concurrently with tcgen05 MMAs, and
// measured ALU issue pressure slows those MMAs (tests/tools/umma_microbench.cu).
LD_DEVINL float erf_as(float z) {
  const float az = fabsf(z);
  const float t = __fdividef(1.0f, fmaf(0.3275911f, az, 1.0f));
  const float poly =
      t * fmaf(fmaf(fmaf(fmaf(1.061405429f, t, -1.453152027f), t, 1.421413741f), t, -0.284496736f), t, 0.254829592f);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-az * az * 1.4426950408889634f));
  return copysignf(fmaf(-poly, e, 1.0f), z);
}

// GELU with the exact-erf definition 1/2 x (1 + erf(x / sqrt 2)) (R6); erff is the CUDA
// single-precision erf (<= 2 ulp).  erf_as above is kept as a measured alternative: it
// issues fewer instructions but two MUFU ops, and measured no faster inside the conv.
LD_DEVINL float gelu_erf(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// GELU for the tensor-core paths, whose next layer rounds activations to an 11-bit significand
// (TF32 / FP16 operands, relative step 2^-11):  GELU(x) = x Phi(x) = (x + |x| E)/2 with
// E = erf(|x|/sqrt 2) = 1 - q^-16, q = 1 + a1 z + ... + a6 z^6 (Abramowitz & Stegun 7.1.28,
// |error of E| <= 3e-7), so GELU = relu(x) - |x| q^-16 / 2: 6 FMA + 4 MUL + 1 MUFU.RCP and no
// branch, i.e. no per-element control flow and full ILP across an epilogue's values.
// Absolute error <= 1.5e-7 |x| -- far below the 2^-11 operand rounding that follows.
LD_DEVINL float gelu_fast(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  float q = fmaf(fmaf(fmaf(fmaf(fmaf(fmaf(0.0000430638f, z, 0.0002765672f), z, 0.0001520143f), z, 0.0092705272f), z,
                          0.0422820123f), z, 0.0705230784f), z, 1.0f);
  q = q * q;
  q = q * q;
  q = q * q;
  q = q * q;
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));   // q >= 1: no denormal / special path
  return fmaf(-0.5f * fabsf(x), r, fmaxf(x, 0.f));
}

// The same GELU on a pair of values with the packed fp32 pipe ops of sm_100 (FFMA2 / FMUL2 /
// FADD2: one instruction for two lanes' worth of fp32 arithmetic), bias added in the same
// pass: (y0, y1) = GELU(x0 + b0), GELU(x1 + b1).  Same operations, same order, same rounding
// per element as gelu_fast(x + b).
LD_DEVINL unsigned long long f2_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
LD_DEVINL void f2_unpack(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
LD_DEVINL unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
LD_DEVINL unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
LD_DEVINL unsigned long long f2_add(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
LD_DEVINL unsigned long long f2_splat(float c) { return f2_pack(c, c); }
LD_DEVINL void gelu_fast2(float x0, float x1, float b0, float b1, float& y0, float& y1) {
  const unsigned long long t = f2_add(f2_pack(x0, x1), f2_pack(b0, b1));
  float t0, t1;
  f2_unpack(t, t0, t1);
  const unsigned long long a = f2_pack(fabsf(t0), fabsf(t1));
  const unsigned long long z = f2_mul(a, f2_splat(0.70710678118654752f));
  unsigned long long q = f2_fma(f2_splat(0.0000430638f), z, f2_splat(0.0002765672f));
  q = f2_fma(q, z, f2_splat(0.0001520143f));
  q = f2_fma(q, z, f2_splat(0.0092705272f));
  q = f2_fma(q, z, f2_splat(0.0422820123f));
  q = f2_fma(q, z, f2_splat(0.0705230784f));
  q = f2_fma(q, z, f2_splat(1.0f));
  q = f2_mul(q, q);
  q = f2_mul(q, q);
  q = f2_mul(q, q);
  q = f2_mul(q, q);
  float q0, q1, r0, r1;
  f2_unpack(q, q0, q1);
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(q0));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(q1));
  const unsigned long long h = f2_mul(a, f2_splat(-0.5f));
  f2_unpack(f2_fma(h, f2_pack(r0, r1), f2_pack(fmaxf(t0, 0.f), fmaxf(t1, 0.f))), y0, y1);
}

LD_DEVINL int wrap(int i, int n) { return i & (n - 1); }  // n is a power of two

LD_DEVINL float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
LD_DEVINL float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
LD_DEVINL float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
LD_DEVINL float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// The 6-tap interpolation / derivative sums of u and v at one face on packed fp32 pairs (FFMA2: (uI, vI)
// and (uD, vD) in one instruction each); per element the same fma.rn sequence as four scalar chains, so
// the results are bitwise those of the scalar form.  Shared by K2 (flux.cu), the output layer's flux
// epilogue (conv_xn.cu) and, in its scalar form, the fused stage kernel (fft.cu).
template <int STRIDE>
LD_DEVINL void face_taps2(const float* wv, const float* u0, const float* v0, float& uI, float& uD, float& vI,
                          float& vD) {
  unsigned long long I = 0ull, D = 0ull;   // (uI, vI), (uD, vD)
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const unsigned long long uv = f2_pack(u0[t * STRIDE], v0[t * STRIDE]);
    I = f2_fma(f2_splat(wv[t]), uv, I);
    D = f2_fma(f2_splat(wv[6 + t]), uv, D);
  }
  f2_unpack(I, uI, vI);
  f2_unpack(D, uD, vD);
}

}  // namespace ld
