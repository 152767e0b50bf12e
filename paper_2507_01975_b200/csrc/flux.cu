// flux.cu -- K2: fused stencil application -> face fluxes -> divergence -> forcing/drag
// -> RK stage combination.
//
// Per cell (i, j) (Eq.4; readings R2, R3, R9, R12):
//   x-face i-1/2 (owned by cell i):  c^x = sum_t wIx[t] c(i-3+t, j),  dc^x = (1/h) sum_t wDx[t] c(i-3+t, j)
//   y-face j-1/2 (owned by cell j):  same with shifts in j and the y stencils
//   F^x_c = gamma u^x c^x - nu dc^x,  F^y_c = gamma v^y c^y - nu dc^y
//   T_c   = -[F^x_c(i+1) - F^x_c(i) + F^y_c(j+1) - F^y_c(j)] / h  (+ f_j - alpha u, - alpha v)
//   out   = a u^n + b X + c dt T + q dt acc (+ e)           (Shu-Osher stage, R13)
//
// Layout: X, u^n, out, acc: planar [B][2][N][N] (y rows, x fastest); stencils w: x-major
// cell-major [B][N(x)][N(y)][24] (channels wIx[6] wDx[6] wIy[6] wDy[6], as the tcgen05 conv
// epilogue writes them: one 96-B run per cell, read as 6 x 16 B); TC term e: [B][N(x)][N(y)][2].
// CTA tile TX x TY cells, one thread per cell.  The stage field with a radius-3 halo (periodic
// wrap) and the stencils of the extra +x / +y face owners are staged once in shared memory;
// every face flux is computed exactly once (conservative) into shared memory.  All global
// loads a thread needs (its stencils, u^n, acc, e) are issued before the first barrier so
// their latencies overlap.
#include "common.cuh"

namespace ld {

struct BaseStencil { float w[24]; };

template <bool FIXED>
__global__ void __launch_bounds__(256, 4)
flux_rk_kernel(FluxParams P, StageCoef S, BaseStencil base,
               const float* __restrict__ X, const float* un,
               const float* __restrict__ w, const float* __restrict__ e,
               float* acc, float* out, int write_T)
{
  extern __shared__ float sm[];
  const int TX = blockDim.x, TY = blockDim.y;
  const int N = P.n;
  const int HX = TX + 6, HY = TY + 6;
  float* us = sm;                       // [2][HY][HX]
  float* Fx = us + 2 * HY * HX;         // [2][TY][TX+1]
  float* Fy = Fx + 2 * TY * (TX + 1);   // [2][TY+1][TX]
  float* wxe = Fy + 2 * (TY + 1) * TX;  // [TY][12]  x-face stencils of the cells at x0 + TX
  float* wye = wxe + TY * 12;           // [TX][12]  y-face stencils of the cells at y0 + TY

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TX + tx, nthr = TX * TY;
  const size_t plane = (size_t)N * N;
  const float* Xb = X + (size_t)b * 2 * plane;
  const int gy = y0 + ty, gx = x0 + tx;
  const size_t pix = (size_t)gy * N + gx;
  const size_t cell = ((size_t)b * N + gx) * N + gy;   // x-major index of w and e

  // ---- issue every global load of this thread first
  float wx[12], wy[12];
  if (FIXED) {
#pragma unroll
    for (int t = 0; t < 12; ++t) { wx[t] = base.w[t]; wy[t] = base.w[12 + t]; }
  } else {
    const float4* w4 = reinterpret_cast<const float4*>(w + cell * 24);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const float4 a = __ldg(w4 + q), c = __ldg(w4 + 3 + q);
      wx[4 * q] = a.x; wx[4 * q + 1] = a.y; wx[4 * q + 2] = a.z; wx[4 * q + 3] = a.w;
      wy[4 * q] = c.x; wy[4 * q + 1] = c.y; wy[4 * q + 2] = c.z; wy[4 * q + 3] = c.w;
    }
  }
  const size_t i0 = (size_t)b * 2 * plane + pix, i1 = i0 + plane;
  float un0 = 0.f, un1 = 0.f, ac0 = 0.f, ac1 = 0.f;
  float2 ee = make_float2(0.f, 0.f);
  const bool need_acc = S.q != 0.f || (S.r != 0.f && !S.acc_init);
  if (!write_T) {
    if (S.a != 0.f) { un0 = un[i0]; un1 = un[i1]; }
    if (need_acc) { ac0 = acc[i0]; ac1 = acc[i1]; }
    if (S.add_e) ee = *reinterpret_cast<const float2*>(e + cell * 2);
  }

  // ---- stage the halo tile and the stencils of the extra face owners
  for (int idx = tid; idx < 2 * HY * HX; idx += nthr) {
    const int c = idx / (HY * HX), rem = idx - c * (HY * HX);
    const int ry = rem / HX, rx = rem - ry * HX;
    us[idx] = Xb[c * plane + (size_t)wrap(y0 - 3 + ry, N) * N + wrap(x0 - 3 + rx, N)];
  }
  if (!FIXED) {
    const float* wb = w + (size_t)b * plane * 24;
    for (int idx = tid; idx < (TY + TX) * 12; idx += nthr) {
      if (idx < TY * 12) {
        const int r = idx / 12, t = idx - r * 12;
        wxe[idx] = __ldg(wb + ((size_t)wrap(x0 + TX, N) * N + y0 + r) * 24 + t);
      } else {
        const int k = idx - TY * 12, xx = k / 12, t = k - xx * 12;
        wye[k] = __ldg(wb + ((size_t)(x0 + xx) * N + wrap(y0 + TY, N)) * 24 + 12 + t);
      }
    }
  }
  __syncthreads();

  auto U = [&](int c, int ry, int rx) { return us[(c * HY + ry) * HX + rx]; };

  // x-face flux of local cell (ly in [0,TY), lx in [0,TX]) with its 6 interp + 6 deriv taps
  auto xface = [&](int ly, int lx, const float* ww) {
    float uI = 0.f, uD = 0.f, vI = 0.f, vD = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const float uu = U(0, ly + 3, lx + t), vv = U(1, ly + 3, lx + t);
      uI = fmaf(ww[t], uu, uI); uD = fmaf(ww[6 + t], uu, uD);
      vI = fmaf(ww[t], vv, vI); vD = fmaf(ww[6 + t], vv, vD);
    }
    const float adv = P.gamma * uI;
    Fx[(0 * TY + ly) * (TX + 1) + lx] = adv * uI - P.nu * (uD * P.inv_h);
    Fx[(1 * TY + ly) * (TX + 1) + lx] = adv * vI - P.nu * (vD * P.inv_h);
  };
  // y-face flux of local cell (ly in [0,TY], lx in [0,TX))
  auto yface = [&](int ly, int lx, const float* ww) {
    float uI = 0.f, uD = 0.f, vI = 0.f, vD = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const float uu = U(0, ly + t, lx + 3), vv = U(1, ly + t, lx + 3);
      uI = fmaf(ww[t], uu, uI); uD = fmaf(ww[6 + t], uu, uD);
      vI = fmaf(ww[t], vv, vI); vD = fmaf(ww[6 + t], vv, vD);
    }
    const float adv = P.gamma * vI;
    Fy[(0 * (TY + 1) + ly) * TX + lx] = adv * uI - P.nu * (uD * P.inv_h);
    Fy[(1 * (TY + 1) + ly) * TX + lx] = adv * vI - P.nu * (vD * P.inv_h);
  };

  xface(ty, tx, wx);
  yface(ty, tx, wy);
  if (tx == TX - 1) xface(ty, TX, FIXED ? base.w : wxe + ty * 12);
  if (ty == TY - 1) yface(TY, tx, FIXED ? base.w + 12 : wye + tx * 12);
  __syncthreads();

  float T[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float t = -((Fx[(c * TY + ty) * (TX + 1) + tx + 1] - Fx[(c * TY + ty) * (TX + 1) + tx]) +
                (Fy[(c * (TY + 1) + ty + 1) * TX + tx] - Fy[(c * (TY + 1) + ty) * TX + tx])) * P.inv_h;
    if (P.forced) {
      if (c == 0) t += P.force_row[gy];
      t -= P.drag * U(c, ty + 3, tx + 3);
    }
    T[c] = t;
  }
  if (write_T) {
    out[i0] = T[0];
    out[i1] = T[1];
    return;
  }
  const float unv[2] = {un0, un1}, acv[2] = {ac0, ac1}, ev[2] = {ee.x, ee.y};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float v = S.a * unv[c] + S.b * U(c, ty + 3, tx + 3) + S.c * P.dt * T[c];
    if (S.q != 0.f) v += S.q * P.dt * acv[c];
    if (S.add_e) v += ev[c];
    const size_t idx = c ? i1 : i0;
    if (S.r != 0.f) acc[idx] = acv[c] + S.r * T[c];
    out[idx] = v;
  }
}

cudaError_t launch_flux_rk(const FluxParams& P, const StageCoef& S, const float* base24,
                           const float* X, const float* un, const float* w, const float* e,
                           float* acc, float* out, int write_T, cudaStream_t st) {
  const int TX = P.n >= 32 ? 32 : P.n, TY = P.n >= 8 ? 8 : P.n;
  dim3 block(TX, TY), grid(P.n / TX, P.n / TY, P.batch);
  const size_t smem = sizeof(float) * (2 * (TY + 6) * (TX + 6) + 2 * TY * (TX + 1) + 2 * (TY + 1) * TX +
                                       (TY + TX) * 12);
  BaseStencil bs;
  for (int i = 0; i < 24; ++i) bs.w[i] = base24 ? base24[i] : 0.f;
  if (w == nullptr)
    flux_rk_kernel<true><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
  else
    flux_rk_kernel<false><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
  return cudaGetLastError();
}

}  // namespace ld
