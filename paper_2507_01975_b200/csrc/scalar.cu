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
