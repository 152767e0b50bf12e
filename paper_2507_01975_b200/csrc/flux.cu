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
// Layout: X, u^n, out, e, acc: [B][2][N][N]; w: planar [B][24][N][N] (coalesced per tap).
// CTA tile TX x 8 cells; the stage field with a radius-3 halo (periodic wrap) is staged
// once in shared memory; face fluxes are computed once per face (conservative) into
// shared memory, including the extra column/row of faces owned by the +x / +y neighbours.
#include "common.cuh"

namespace ld {

struct BaseStencil { float w[24]; };

constexpr int kFluxTY = 8;

template <bool FIXED>
__global__ void __launch_bounds__(256)
flux_rk_kernel(FluxParams P, StageCoef S, BaseStencil base,
               const float* __restrict__ X, const float* un,
               const float* __restrict__ w, const float* __restrict__ e,
               float* acc, float* out, int write_T)
{
  extern __shared__ float sm[];
  const int TX = blockDim.x, TY = kFluxTY;
  const int N = P.n;
  const int HX = TX + 6, HY = TY + 6;
  float* us = sm;                       // [2][HY][HX]
  float* Fx = us + 2 * HY * HX;         // [2][TY][TX+1]
  float* Fy = Fx + 2 * TY * (TX + 1);   // [2][TY+1][TX]

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TX + tx, nthr = TX * TY;
  const size_t plane = (size_t)N * N;
  const float* Xb = X + (size_t)b * 2 * plane;

  // prefetch this thread's stencil weights (and those of the extra +x / +y face owners) so
  // their L2/HBM latency overlaps the halo staging below
  const float* wb = w + (size_t)b * 24 * plane;
  float wx[12], wy[12], wx2[12], wy2[12];
  const bool xtra = tx == TX - 1, ytra = ty == TY - 1;
  {
    const size_t pix = (size_t)(y0 + ty) * N + (x0 + tx);
    const size_t pix_x = (size_t)(y0 + ty) * N + wrap(x0 + TX, N);
    const size_t pix_y = (size_t)wrap(y0 + TY, N) * N + (x0 + tx);
#pragma unroll
    for (int t = 0; t < 12; ++t) {
      wx[t] = FIXED ? base.w[t] : __ldg(wb + (size_t)t * plane + pix);
      wy[t] = FIXED ? base.w[12 + t] : __ldg(wb + (size_t)(12 + t) * plane + pix);
      wx2[t] = (FIXED || !xtra) ? wx[t] : __ldg(wb + (size_t)t * plane + pix_x);
      wy2[t] = (FIXED || !ytra) ? wy[t] : __ldg(wb + (size_t)(12 + t) * plane + pix_y);
    }
    if (FIXED) {
#pragma unroll
      for (int t = 0; t < 12; ++t) { wx2[t] = base.w[t]; wy2[t] = base.w[12 + t]; }
    }
  }

  for (int idx = tid; idx < 2 * HY * HX; idx += nthr) {
    const int c = idx / (HY * HX), rem = idx % (HY * HX);
    const int ry = rem / HX, rx = rem % HX;
    us[idx] = Xb[c * plane + (size_t)wrap(y0 - 3 + ry, N) * N + wrap(x0 - 3 + rx, N)];
  }
  __syncthreads();

  auto U = [&](int c, int ry, int rx) { return us[(c * HY + ry) * HX + rx]; };

  // x-face flux of local cell (ly in [0,TY), lx in [0,TX]) with its 6 interp + 6 deriv taps
  auto xface = [&](int ly, int lx, const float (&ww)[12]) {
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
  auto yface = [&](int ly, int lx, const float (&ww)[12]) {
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
  if (xtra) xface(ty, TX, wx2);
  if (ytra) yface(TY, tx, wy2);
  __syncthreads();

  const int gy = y0 + ty, gx = x0 + tx;
  const size_t pix = (size_t)gy * N + gx;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float T = -((Fx[(c * TY + ty) * (TX + 1) + tx + 1] - Fx[(c * TY + ty) * (TX + 1) + tx]) +
                (Fy[(c * (TY + 1) + ty + 1) * TX + tx] - Fy[(c * (TY + 1) + ty) * TX + tx])) * P.inv_h;
    const float xc = U(c, ty + 3, tx + 3);
    if (P.forced) {
      if (c == 0) T += P.force_row[gy];
      T -= P.drag * xc;
    }
    const size_t idx = ((size_t)b * 2 + c) * plane + pix;
    if (write_T) { out[idx] = T; continue; }
    float v = S.a * un[idx] + S.b * xc + S.c * P.dt * T;
    float a_in = 0.f;
    if (S.q != 0.f || (S.r != 0.f && !S.acc_init)) a_in = acc[idx];
    if (S.q != 0.f) v += S.q * P.dt * a_in;
    if (S.add_e) v += e[idx];
    if (S.r != 0.f) acc[idx] = a_in + S.r * T;
    out[idx] = v;
  }
}

cudaError_t launch_flux_rk(const FluxParams& P, const StageCoef& S, const float* base24,
                           const float* X, const float* un, const float* w, const float* e,
                           float* acc, float* out, int write_T, cudaStream_t st) {
  const int TX = P.n >= 32 ? 32 : P.n;
  dim3 block(TX, kFluxTY), grid(P.n / TX, P.n / kFluxTY, P.batch);
  const size_t smem = sizeof(float) * (2 * (kFluxTY + 6) * (TX + 6) + 2 * kFluxTY * (TX + 1) +
                                       2 * (kFluxTY + 1) * TX);
  BaseStencil bs;
  for (int i = 0; i < 24; ++i) bs.w[i] = base24 ? base24[i] : 0.f;
  if (w == nullptr)
    flux_rk_kernel<true><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
  else
    flux_rk_kernel<false><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
  return cudaGetLastError();
}

}  // namespace ld
