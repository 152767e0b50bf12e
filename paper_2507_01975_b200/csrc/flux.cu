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

template <int TX, int TY, bool FIXED>
__global__ void __launch_bounds__(TX * TY, 2048 / (TX * TY) < 4 ? 2048 / (TX * TY) : 4)
flux_rk_kernel(FluxParams P, StageCoef S, BaseStencil base,
               const float* __restrict__ X, const float* un,
               const float* __restrict__ w, const float* __restrict__ e,
               float* acc, float* out, int write_T)
{
  // TX x TY tile, one thread per cell; compile-time tile sizes turn every staging index
  // computation into shifts and constant multiplies
  extern __shared__ __align__(16) float sm[];
  const int N = P.n;
  constexpr int HX = TX + 6, HY = TY + 6;
  float* ws = sm;                       // [TX+1][TY+1][24] stencils of the tile (+ the +x / +y face owners)
  float* us = ws + (TX + 1) * (TY + 1) * 24;   // [2][HY][HX]
  float* Fx = us + 2 * HY * HX;         // [2][TY][TX+1]
  float* Fy = Fx + 2 * TY * (TX + 1);   // [2][TY+1][TX]

  const int b = blockIdx.z;
  const int NY = P.ny;
  auto wy = [NY](int y) { return y < 0 ? y + NY : (y >= NY ? y - NY : y); };
  const int x0 = blockIdx.x * TX, y0 = P.y_off + blockIdx.y * TY;   // tile origin in the X / w domain
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TX + tx;
  constexpr int nthr = TX * TY;
  const size_t plane = (size_t)N * NY;
  const float* Xb = X + (size_t)b * 2 * plane;
  const int gy = y0 + ty, gx = x0 + tx;          // cell in the X / w domain
  const int oy = P.o_row0 + blockIdx.y * TY + ty;   // its row in the u^n / out / acc planes
  const size_t opl = (size_t)P.o_rows * N;

  // ---- stencils: for each of the TX+1 columns x, the TY+1 cells y0 .. y0+TY are one contiguous
  // (TY+1) x 96-B run of the x-major layout w[b][x][y][24] (two runs where y0+TY wraps to 0):
  // coalesced 16-B cp.async into shared memory
  if (!FIXED) {
    constexpr int CPC = (TY + 1) * 6;   // 16-B chunks per column
#pragma unroll
    for (int idx = tid; idx < (TX + 1) * CPC; idx += nthr) {
      const int cx = idx / CPC, k = idx - cx * CPC;
      const int cy = k / 6, q = k - cy * 6;
      const size_t cell = ((size_t)b * N + wrap(x0 + cx, N)) * NY + wy(y0 + cy);
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ws + ((cx * (TY + 1) + cy) * 24 + q * 4));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(w + cell * 24 + q * 4) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // ---- per-thread loads of the RK combination, issued early
  const size_t i0 = (size_t)b * 2 * opl + (size_t)oy * N + gx, i1 = i0 + opl;   // out
  const int ly = blockIdx.y * TY + ty;
  const size_t unpl = (size_t)P.un_rows * N, apl = (size_t)P.a_rows * N;
  const size_t n0 = (size_t)b * 2 * unpl + (size_t)(P.un_row0 + ly) * N + gx, n1 = n0 + unpl;   // u^n
  const size_t a0 = (size_t)b * 2 * apl + (size_t)(P.a_row0 + ly) * N + gx, a1 = a0 + apl;       // acc
  float un0 = 0.f, un1 = 0.f, ac0 = 0.f, ac1 = 0.f;
  float2 ee = make_float2(0.f, 0.f);
  const bool need_acc = S.q != 0.f || (S.r != 0.f && !S.acc_init);
  if (!write_T) {
    if (S.a != 0.f) { un0 = un[n0]; un1 = un[n1]; }
    if (need_acc) { ac0 = acc[a0]; ac1 = acc[a1]; }
    if (S.add_e) ee = *reinterpret_cast<const float2*>(e + (((size_t)b * N + gx) * NY + gy) * 2);
  }
  // ---- halo tile of the stage field (periodic wrap), coalesced along x
#pragma unroll
  for (int idx = tid; idx < 2 * HY * HX; idx += nthr) {
    const int c = idx / (HY * HX), rem = idx - c * (HY * HX);
    const int ry = rem / HX, rx = rem - ry * HX;
    us[idx] = Xb[c * plane + (size_t)wy(y0 - 3 + ry) * N + wrap(x0 - 3 + rx, N)];
  }
  if (!FIXED) asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  auto U = [&](int c, int ry, int rx) { return us[(c * HY + ry) * HX + rx]; };
  auto W = [&](int lx, int ly, int t) { return FIXED ? base.w[t] : ws[(lx * (TY + 1) + ly) * 24 + t]; };

  // x-face flux of local cell (ly in [0,TY), lx in [0,TX]) with its 6 interp + 6 deriv taps
  auto xface = [&](int ly, int lx) {
    float uI = 0.f, uD = 0.f, vI = 0.f, vD = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const float uu = U(0, ly + 3, lx + t), vv = U(1, ly + 3, lx + t);
      const float wi = W(lx, ly, t), wd = W(lx, ly, 6 + t);
      uI = fmaf(wi, uu, uI); uD = fmaf(wd, uu, uD);
      vI = fmaf(wi, vv, vI); vD = fmaf(wd, vv, vD);
    }
    const float adv = P.gamma * uI;
    Fx[(0 * TY + ly) * (TX + 1) + lx] = adv * uI - P.nu * (uD * P.inv_h);
    Fx[(1 * TY + ly) * (TX + 1) + lx] = adv * vI - P.nu * (vD * P.inv_h);
  };
  // y-face flux of local cell (ly in [0,TY], lx in [0,TX))
  auto yface = [&](int ly, int lx) {
    float uI = 0.f, uD = 0.f, vI = 0.f, vD = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const float uu = U(0, ly + t, lx + 3), vv = U(1, ly + t, lx + 3);
      const float wi = W(lx, ly, 12 + t), wd = W(lx, ly, 18 + t);
      uI = fmaf(wi, uu, uI); uD = fmaf(wd, uu, uD);
      vI = fmaf(wi, vv, vI); vD = fmaf(wd, vv, vD);
    }
    const float adv = P.gamma * vI;
    Fy[(0 * (TY + 1) + ly) * TX + lx] = adv * uI - P.nu * (uD * P.inv_h);
    Fy[(1 * (TY + 1) + ly) * TX + lx] = adv * vI - P.nu * (vD * P.inv_h);
  };

  xface(ty, tx);
  yface(ty, tx);
  if (tx == TX - 1) xface(ty, TX);
  if (ty == TY - 1) yface(TY, tx);
  __syncthreads();

  float T[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float t = -((Fx[(c * TY + ty) * (TX + 1) + tx + 1] - Fx[(c * TY + ty) * (TX + 1) + tx]) +
                (Fy[(c * (TY + 1) + ty + 1) * TX + tx] - Fy[(c * (TY + 1) + ty) * TX + tx])) * P.inv_h;
    if (P.forced) {
      if (c == 0) t += P.force_row[P.gy0 + blockIdx.y * TY + ty];
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
    if (S.r != 0.f) acc[c ? a1 : a0] = acv[c] + S.r * T[c];
    out[c ? i1 : i0] = v;
  }
}

template <int TX, int TY>
static void launch_flux_t(const FluxParams& P, const StageCoef& S, const BaseStencil& bs, const float* X,
                          const float* un, const float* w, const float* e, float* acc, float* out, int write_T,
                          cudaStream_t st) {
  dim3 block(TX, TY), grid(P.n / TX, P.rows / TY, P.batch);
  const size_t smem = sizeof(float) * ((size_t)(TX + 1) * (TY + 1) * 24 + 2 * (TY + 6) * (TX + 6) +
                                       2 * TY * (TX + 1) + 2 * (TY + 1) * TX);
  if (w == nullptr)
    flux_rk_kernel<TX, TY, true><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
  else
    flux_rk_kernel<TX, TY, false><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
}

cudaError_t launch_flux_rk(const FluxParams& P, const StageCoef& S, const float* base24,
                           const float* X, const float* un, const float* w, const float* e,
                           float* acc, float* out, int write_T, cudaStream_t st) {
  BaseStencil bs;
  for (int i = 0; i < 24; ++i) bs.w[i] = base24 ? base24[i] : 0.f;
  if (P.n >= 32) launch_flux_t<32, 8>(P, S, bs, X, un, w, e, acc, out, write_T, st);
  else if (P.n == 16) launch_flux_t<16, 8>(P, S, bs, X, un, w, e, acc, out, write_T, st);
  else launch_flux_t<8, 8>(P, S, bs, X, un, w, e, acc, out, write_T, st);
  return cudaGetLastError();
}

}  // namespace ld
