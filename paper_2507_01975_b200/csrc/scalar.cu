// scalar.cu -- passive-scalar transport of the shear-flow case ("a coupled
// advection-diffusion equation alongside the NSE"; SURVEY.md §8f lower row; readings S1-S4 in
// DESIGN.md §8h).  Per RK stage, after the stage's net has written the stencils w:
//   x-face of cell i (owner i): u^x = sum_t wIx[t] u(i-3+t), s^x = sum_t wIx[t] s(i-3+t),
//                               ds^x = (1/h) sum_t wDx[t] s(i-3+t);  F^x_s = u^x s^x - D ds^x
//   (y-face likewise), T_s = -[F^x_s(i+1) - F^x_s(i) + F^y_s(j+1) - F^y_s(j)] / h,
//   s_out = a s^n + b s_X + c dt T_s (+ q dt acc), acc <- acc + r T_s (RK4), the momentum's Shu-Osher
//   coefficients; no projection, no forcing, no TC term on s.
// Layout: velocity X [B][2][N][N], scalar [B][N][N], stencils w x-major [B][N(x)][N(y)][24] (the conv
// epilogue's layout; nullptr = the base stencils).  One thread per cell; each thread evaluates its own
// two faces and the +x / +y neighbours' (the scalar is a small share of the step).
#include "common.cuh"

namespace ld {

__global__ void scalar_rk_kernel(FluxParams P, StageCoef S, BaseStencil base, float D, const float* __restrict__ X,
                                 const float* __restrict__ w, const float* __restrict__ sX, const float* sn,
                                 float* acc, float* out) {
  const int N = P.n;
  const size_t NN = (size_t)N * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)P.batch * NN) return;
  const int b = (int)(idx / NN), cell = (int)(idx % NN), j = cell / N, i = cell % N;
  const float* u = X + (size_t)b * 2 * NN;
  const float* v = u + NN;
  const float* s = sX + (size_t)b * NN;
  auto stencil = [&](int ci, int cj, int k) {   // channel k of the stencils of cell (ci, cj)
    return w ? w[(((size_t)b * N + ci) * N + cj) * 24 + k] : base.w[k];
  };
  auto xflux = [&](int ci) {   // flux through the x-face owned by cell (ci, j)
    float uf = 0.f, sf = 0.f, df = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const size_t o = (size_t)j * N + wrap(ci - 3 + t, N);
      const float wi = stencil(ci, j, t), wd = stencil(ci, j, 6 + t);
      uf = fmaf(wi, u[o], uf);
      sf = fmaf(wi, s[o], sf);
      df = fmaf(wd, s[o], df);
    }
    return uf * sf - D * (df * P.inv_h);
  };
  auto yflux = [&](int cj) {   // flux through the y-face owned by cell (i, cj)
    float vf = 0.f, sf = 0.f, df = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const size_t o = (size_t)wrap(cj - 3 + t, N) * N + i;
      const float wi = stencil(i, cj, 12 + t), wd = stencil(i, cj, 18 + t);
      vf = fmaf(wi, v[o], vf);
      sf = fmaf(wi, s[o], sf);
      df = fmaf(wd, s[o], df);
    }
    return vf * sf - D * (df * P.inv_h);
  };
  const float T = -((xflux(wrap(i + 1, N)) - xflux(i)) + (yflux(wrap(j + 1, N)) - yflux(j))) * P.inv_h;
  const bool need_acc = S.q != 0.f || (S.r != 0.f && !S.acc_init);
  const float av = need_acc ? acc[idx] : 0.f;
  float o = S.a * sn[idx] + S.b * s[cell] + S.c * P.dt * T;
  if (S.q != 0.f) o += S.q * P.dt * av;
  if (S.r != 0.f) acc[idx] = av + S.r * T;
  out[idx] = o;
}

cudaError_t launch_scalar_rk(const FluxParams& P, const StageCoef& S, const float* base24, float D, const float* X,
                             const float* w, const float* sX, const float* sn, float* acc, float* out, cudaStream_t st) {
  BaseStencil bs;
  for (int k = 0; k < 24; ++k) bs.w[k] = base24 ? base24[k] : 0.f;
  const size_t n = (size_t)P.batch * P.n * P.n;
  scalar_rk_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(P, S, bs, D, X, w, sX, sn, acc, out);
  return cudaGetLastError();
}

}  // namespace ld

// ---------------------------------------------------------------------------
// The paper's constant 5x4 face kernels (stencil_mode LD_STENCIL_5X4; O_P + O_L =
// (W_P + W_L) * u, W in R^{5x4}; readings F1-F3 in DESIGN.md §8i).  W (constrained at ld_init) is
// [axis][op][b 5 tangential][a 4 normal]; x-face of cell (i, j): taps (i - 2 + a, j - 2 + b); y-face:
// taps (i - 2 + b, j - 2 + a).  Fluxes, divergence, source and the Shu-Osher combination as K2
// (flux.cu).  One thread per cell; each thread evaluates its two faces and the +x / +y neighbours'.
// ---------------------------------------------------------------------------
namespace ld {

struct W5x4 {
  float w[80];
};

__global__ void flux5x4_rk_kernel(FluxParams P, StageCoef S, W5x4 W, const float* __restrict__ X, const float* un,
                                  float* acc, float* out, int write_T) {
  const int N = P.n;
  const size_t NN = (size_t)N * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)P.batch * NN) return;
  const int b = (int)(idx / NN), cell = (int)(idx % NN), j = cell / N, i = cell % N;
  const float* u = X + (size_t)b * 2 * NN;
  const float* v = u + NN;
  // face values of the x-face (ax 0) owned by cell (ci, cj) or the y-face (ax 1): interp / deriv of u, v
  auto faces = [&](int ax, int ci, int cj, float& uI, float& vI, float& uD, float& vD) {
    uI = vI = uD = vD = 0.f;
    const float* wi = W.w + ax * 40;
    const float* wd = wi + 20;
#pragma unroll
    for (int bb = 0; bb < 5; ++bb)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int x = ax == 0 ? ci - 2 + a : ci - 2 + bb, y = ax == 0 ? cj - 2 + bb : cj - 2 + a;
        const size_t o = (size_t)wrap(y, N) * N + wrap(x, N);
        const float uu = u[o], vv = v[o];
        uI = fmaf(wi[bb * 4 + a], uu, uI); vI = fmaf(wi[bb * 4 + a], vv, vI);
        uD = fmaf(wd[bb * 4 + a], uu, uD); vD = fmaf(wd[bb * 4 + a], vv, vD);
      }
  };
  float F[4][2];   // x-face (i), x-face (i+1), y-face (j), y-face (j+1); components u, v
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int ax = f >> 1;
    const int ci = (f == 1) ? wrap(i + 1, N) : i, cj = (f == 3) ? wrap(j + 1, N) : j;
    float uI, vI, uD, vD;
    faces(ax, ci, cj, uI, vI, uD, vD);
    const float adv = P.gamma * (ax == 0 ? uI : vI);   // face-normal advecting velocity (R3)
    F[f][0] = adv * uI - P.nu * (uD * P.inv_h);
    F[f][1] = adv * vI - P.nu * (vD * P.inv_h);
  }
  const bool need_acc = S.q != 0.f || (S.r != 0.f && !S.acc_init);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float t = -((F[1][c] - F[0][c]) + (F[3][c] - F[2][c])) * P.inv_h;
    const size_t o = (size_t)b * 2 * NN + c * NN + cell;
    if (P.forced) {
      if (c == 0) t += P.force_row[j];
      t -= P.drag * X[o];
    }
    if (write_T) {
      out[o] = t;
      continue;
    }
    const float av = need_acc ? acc[o] : 0.f;
    float val = S.a * un[o] + S.b * X[o] + S.c * P.dt * t;
    if (S.q != 0.f) val += S.q * P.dt * av;
    if (S.r != 0.f) acc[o] = av + S.r * t;
    out[o] = val;
  }
}

cudaError_t launch_flux5x4_rk(const FluxParams& P, const StageCoef& S, const float* w80, const float* X, const float* un,
                              float* acc, float* out, int write_T, cudaStream_t st) {
  W5x4 W;
  for (int k = 0; k < 80; ++k) W.w[k] = w80[k];
  const size_t n = (size_t)P.batch * P.n * P.n;
  flux5x4_rk_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(P, S, W, X, un, acc, out, write_T);
  return cudaGetLastError();
}

}  // namespace ld
