// adjoint.cu -- NEXT-4: the vector-Jacobian product of one LDSolver step, i.e. the
// reverse pass that training needs ("fully differentiable"; autoregressive rollout
// trained on the MSE loss of P:348-352).  For a cotangent g of u^{n+1} it returns
//   u_bar = (d u^{n+1} / d u^n)^T g   and   theta_bar += (d u^{n+1} / d theta)^T g.
//
// Reverse order of the forward step (readings as the forward, DESIGN.md §2 / §8g):
//   RK stages (Shu-Osher / classical RK4) in reverse, the projection P being self-adjoint
//   (G_c = -D_c^T, P orthogonal: the forward kernels apply it to the cotangents);
//   per stage: divergence -> face fluxes -> face values (adjoint face stencils: a gather over the
//   face owners) and the stencil cotangent w_bar; R_bar = Pi w_bar (Pi symmetric, R4) plus e_bar on
//   the TC channels at the stage-1 net (R8); the conv net in reverse: weight / bias gradients
//   (wgrad kernel), input gradients (the SIMT conv with flipped, transposed weights), GELU' / ReLU'.
// Arithmetic: fp32 SIMT throughout (the fp32-exact net of LD_CONV_FP32 for the forward recompute),
// whatever conv_precision the handle's forward uses.  The forward stage fields are recomputed and
// kept; each stage's net activations are recomputed when that stage is differentiated.
//
// Layouts (all [b][j][i] = [y][x] row-major, i fastest): fields planar [B][2][N][N]; net tensors
// NHWC [B][N][N][C]; constrained stencils w cell-major [B][N][N][24] (x-interp, x-deriv, y-interp,
// y-deriv, 6 taps each); face fluxes [B][4][N][N] (F^x_u, F^x_v, F^y_u, F^y_v of the cell's faces);
// face cotangents [B][8][N][N] (x-face: uI, vI, uD, vD; y-face: uJ, vJ, uE, vE).
#include "common.cuh"

namespace ld {

namespace adj {

constexpr int RS = 32;   // channel stride of the raw net output R / its cotangent (n_out <= 26, padded)

// Pi per (axis, op): Pi_I r = r - mean(r); Pi_D r = r - mean(r) - s (s.r)/|s|^2, s = t - 5/2 (R4)
LD_DEVINL void apply_pi(const float* r, float* out /*24*/) {
#pragma unroll
  for (int blk = 0; blk < 4; ++blk) {
    float sum = 0.f, sr = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      sum += r[blk * 6 + t];
      sr += ((float)t - 2.5f) * r[blk * 6 + t];
    }
    const float mean = sum * (1.f / 6.f), proj = (blk & 1) ? sr * (1.f / 17.5f) : 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) out[blk * 6 + t] = r[blk * 6 + t] - mean - ((float)t - 2.5f) * proj;
  }
}

struct Base24 {
  float w[24];
};

// forward: constrained stencils w (from R or the base) and the face fluxes of every cell
__global__ void fwd_faces_kernel(const float* __restrict__ U, const float* __restrict__ R, Base24 base, int N, int B,
                                 float inv_h, float nu, float gamma, float* __restrict__ w_out,
                                 float* __restrict__ F4) {
  const size_t NN = (size_t)N * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)B * NN) return;
  const int b = (int)(idx / NN), cell = (int)(idx % NN), j = cell / N, i = cell % N;
  float w[24];
  if (R) {
    float pr[24];
    apply_pi(R + idx * RS, pr);
#pragma unroll
    for (int k = 0; k < 24; ++k) w[k] = base.w[k] + pr[k];
  } else {
#pragma unroll
    for (int k = 0; k < 24; ++k) w[k] = base.w[k];
  }
#pragma unroll
  for (int k = 0; k < 24; ++k) w_out[idx * 24 + k] = w[k];
  const float* u = U + (size_t)b * 2 * NN;
  const float* v = u + NN;
  float uI = 0.f, vI = 0.f, uD = 0.f, vD = 0.f, uJ = 0.f, vJ = 0.f, uE = 0.f, vE = 0.f;
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const size_t ox = (size_t)j * N + wrap(i - 3 + t, N), oy = (size_t)wrap(j - 3 + t, N) * N + i;
    uI = fmaf(w[t], u[ox], uI); vI = fmaf(w[t], v[ox], vI);
    uD = fmaf(w[6 + t], u[ox], uD); vD = fmaf(w[6 + t], v[ox], vD);
    uJ = fmaf(w[12 + t], u[oy], uJ); vJ = fmaf(w[12 + t], v[oy], vJ);
    uE = fmaf(w[18 + t], u[oy], uE); vE = fmaf(w[18 + t], v[oy], vE);
  }
  float* f = F4 + (size_t)b * 4 * NN + cell;
  f[0] = gamma * uI * uI - nu * (uD * inv_h);
  f[NN] = gamma * uI * vI - nu * (vD * inv_h);
  f[2 * NN] = gamma * vJ * uJ - nu * (uE * inv_h);
  f[3 * NN] = gamma * vJ * vJ - nu * (vE * inv_h);
}

// forward: T = -div F + f - alpha u (Tout, optional) and Y = a un + b U + cdt T + ec E (Y, optional;
// E planar, the stage-1 net's TC term)
__global__ void fwd_combine_kernel(const float* __restrict__ F4, const float* __restrict__ U,
                                   const float* __restrict__ un, const float* __restrict__ E, int N, int B,
                                   float inv_h, int forced, const float* __restrict__ force_row, float drag,
                                   float a, float bb, float cdt, float ec, float* __restrict__ Tout,
                                   float* __restrict__ Y) {
  const size_t NN = (size_t)N * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)B * NN) return;
  const int b = (int)(idx / NN), cell = (int)(idx % NN), j = cell / N, i = cell % N;
  const float* f = F4 + (size_t)b * 4 * NN;
  const size_t xp = (size_t)j * N + wrap(i + 1, N), yp = (size_t)wrap(j + 1, N) * N + i;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const float* fx = f + c * NN;
    const float* fy = f + (2 + c) * NN;
    float t = -((fx[xp] - fx[cell]) + (fy[yp] - fy[cell])) * inv_h;
    const size_t o = (size_t)b * 2 * NN + c * NN + cell;
    if (forced) {
      if (c == 0) t += force_row[j];
      t -= drag * U[o];
    }
    if (Tout) Tout[o] = t;
    if (Y) {
      float y = a * un[o] + bb * U[o] + cdt * t;
      if (ec != 0.f) y += ec * E[o];
      Y[o] = y;
    }
  }
}

// backward: face cotangents (8 per cell) and R_bar = Pi w_bar (+ e_bar on channels 24, 25)
__global__ void bwd_faces_kernel(const float* __restrict__ U, const float* __restrict__ w, const float* __restrict__ Tb,
                                 const float* __restrict__ eb, int N, int B, float inv_h, float nu, float gamma,
                                 float* __restrict__ Fadj, float* __restrict__ Rb) {
  const size_t NN = (size_t)N * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)B * NN) return;
  const int b = (int)(idx / NN), cell = (int)(idx % NN), j = cell / N, i = cell % N;
  const float* u = U + (size_t)b * 2 * NN;
  const float* v = u + NN;
  const float* tb = Tb + (size_t)b * 2 * NN;
  const float* wc = w + idx * 24;
  const size_t xm = (size_t)j * N + wrap(i - 1, N), ym = (size_t)wrap(j - 1, N) * N + i;
  // T(i) = -(F^x(i+1) - F^x(i) + ...)/h  =>  F^x_bar(i) = (T_bar(i) - T_bar(i-1)) / h
  const float Fxu = (tb[cell] - tb[xm]) * inv_h, Fxv = (tb[NN + cell] - tb[NN + xm]) * inv_h;
  const float Fyu = (tb[cell] - tb[ym]) * inv_h, Fyv = (tb[NN + cell] - tb[NN + ym]) * inv_h;
  float ux[6], vx[6], uy[6], vy[6];
  float uI = 0.f, vI = 0.f, uJ = 0.f, vJ = 0.f;
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const size_t ox = (size_t)j * N + wrap(i - 3 + t, N), oy = (size_t)wrap(j - 3 + t, N) * N + i;
    ux[t] = u[ox]; vx[t] = v[ox]; uy[t] = u[oy]; vy[t] = v[oy];
    uI = fmaf(wc[t], ux[t], uI); vI = fmaf(wc[t], vx[t], vI);
    uJ = fmaf(wc[12 + t], uy[t], uJ); vJ = fmaf(wc[12 + t], vy[t], vJ);
  }
  // F^x_u = g uI uI - nu uD/h, F^x_v = g uI vI - nu vD/h; F^y_u = g vJ uJ - nu uE/h, F^y_v = g vJ vJ - nu vE/h
  const float uIb = gamma * (2.f * uI * Fxu + vI * Fxv), vIb = gamma * uI * Fxv;
  const float uDb = -nu * inv_h * Fxu, vDb = -nu * inv_h * Fxv;
  const float uJb = gamma * vJ * Fyu, vJb = gamma * (uJ * Fyu + 2.f * vJ * Fyv);
  const float uEb = -nu * inv_h * Fyu, vEb = -nu * inv_h * Fyv;
  float* fa = Fadj + (size_t)b * 8 * NN + cell;
  fa[0] = uIb; fa[NN] = vIb; fa[2 * NN] = uDb; fa[3 * NN] = vDb;
  fa[4 * NN] = uJb; fa[5 * NN] = vJb; fa[6 * NN] = uEb; fa[7 * NN] = vEb;
  if (Rb) {
    float wb[24];
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      wb[t] = uIb * ux[t] + vIb * vx[t];
      wb[6 + t] = uDb * ux[t] + vDb * vx[t];
      wb[12 + t] = uJb * uy[t] + vJb * vy[t];
      wb[18 + t] = uEb * uy[t] + vEb * vy[t];
    }
    float rb[24];
    apply_pi(wb, rb);
    float* r = Rb + idx * RS;
#pragma unroll
    for (int k = 0; k < 24; ++k) r[k] = rb[k];
    r[24] = eb ? eb[(size_t)b * 2 * NN + cell] : 0.f;
    r[25] = eb ? eb[(size_t)b * 2 * NN + NN + cell] : 0.f;
#pragma unroll
    for (int k = 26; k < RS; ++k) r[k] = 0.f;
  }
}

// backward: U_bar += adjoint face stencils (gather over the face owners) - alpha T_bar
__global__ void bwd_gather_kernel(const float* __restrict__ Fadj, const float* __restrict__ w,
                                  const float* __restrict__ Tb, int N, int B, int forced, float drag,
                                  float* __restrict__ Ub) {
  const size_t NN = (size_t)N * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)B * NN) return;
  const int b = (int)(idx / NN), cell = (int)(idx % NN), j = cell / N, i = cell % N;
  const float* fa = Fadj + (size_t)b * 8 * NN;
  const float* wb = w + (size_t)b * NN * 24;
  float su = 0.f, sv = 0.f;
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    // the x-face of cell (i+3-t, j) reads this cell with tap t; the y-face of (i, j+3-t) likewise
    const size_t ox = (size_t)j * N + wrap(i + 3 - t, N), oy = (size_t)wrap(j + 3 - t, N) * N + i;
    const float* wx = wb + ox * 24;
    const float* wy = wb + oy * 24;
    su += wx[t] * fa[ox] + wx[6 + t] * fa[2 * NN + ox] + wy[12 + t] * fa[4 * NN + oy] + wy[18 + t] * fa[6 * NN + oy];
    sv += wx[t] * fa[NN + ox] + wx[6 + t] * fa[3 * NN + ox] + wy[12 + t] * fa[5 * NN + oy] + wy[18 + t] * fa[7 * NN + oy];
  }
  const size_t o = (size_t)b * 2 * NN + cell;
  if (forced) {
    su -= drag * Tb[o];
    sv -= drag * Tb[o + NN];
  }
  Ub[o] += su;
  Ub[o + NN] += sv;
}

// e = R[..., 24:26] (NHWC, stride RS) -> planar [B][2][N][N]
__global__ void extract_e_kernel(const float* __restrict__ R, int N, int B, float* __restrict__ E) {
  const size_t NN = (size_t)N * N;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)B * NN) return;
  const size_t b = idx / NN, cell = idx % NN;
  E[b * 2 * NN + cell] = R[idx * RS + 24];
  E[b * 2 * NN + NN + cell] = R[idx * RS + 25];
}

LD_DEVINL float gelu_grad_f(float x) {
  return 0.5f * (1.f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * __expf(-0.5f * x * x);
}

// mode 0: y = phi(z) (forward); mode 1: y = y * phi'(z) (backward, in place on the cotangent)
__global__ void act_kernel(const float* __restrict__ z, float* __restrict__ y, size_t n, int act, int mode) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const float x = z[k];
  if (mode == 0) y[k] = act == 1 ? gelu_erf(x) : fmaxf(x, 0.f);
  else y[k] *= act == 1 ? gelu_grad_f(x) : (x > 0.f ? 1.f : 0.f);
}

// out = a x + b y + c z (null inputs skipped); out may alias x
__global__ void lin3_kernel(float* out, float a, const float* x, float b, const float* y, float c, const float* z,
                            size_t n) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  float s = 0.f;
  if (x) s += a * x[k];
  if (y) s += b * y[k];
  if (z) s += c * z[k];
  out[k] = s;
}

// Weight / bias gradients of one 3x3 layer: Wb[tap][ci][co] += sum_cells G[cell][co] H[cell + shift(tap)][ci],
// bb[co] += sum_cells G[cell][co].  H: NHWC [B][N][N][CI] or planar [B][CI][N][N]; G: NHWC [B][N][N][CO].
// CTA (blockIdx.y) = one (CIB input channels) x (COB output channels) block; thread = one (ci, co) pair
// with its 9 tap accumulators in registers; 8x8 cell tiles (grid-stride over blockIdx.x) staged in
// shared memory with the periodic halo; one atomic add per accumulator at the end.
template <int CI, int CO, int CIB, int COB, bool PLANAR>
__global__ void __launch_bounds__(CIB * COB) wgrad_kernel(const float* __restrict__ H, const float* __restrict__ G, int N,
                                                          int B, float* __restrict__ Wb, float* __restrict__ bb) {
  constexpr int NT = CIB * COB, NCOB = CO / COB;
  __shared__ float hs[CIB][10][10];
  __shared__ float gs[64][COB];
  const int cib = blockIdx.y / NCOB, cob = blockIdx.y % NCOB;
  const int ci_l = threadIdx.x / COB, co_l = threadIdx.x % COB;
  const int tiles_x = N / 8, ntiles = B * tiles_x * tiles_x;
  const size_t NN = (size_t)N * N;
  float acc[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) acc[t] = 0.f;
  float bacc = 0.f;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int b = tile / (tiles_x * tiles_x), tt = tile % (tiles_x * tiles_x);
    const int y0 = (tt / tiles_x) * 8, x0 = (tt % tiles_x) * 8;
    __syncthreads();
    for (int k = threadIdx.x; k < 64 * COB; k += NT) {
      const int c = k / COB, o = k % COB;
      gs[c][o] = G[(((size_t)b * N + y0 + c / 8) * N + x0 + c % 8) * CO + cob * COB + o];
    }
    for (int k = threadIdx.x; k < CIB * 100; k += NT) {
      const int c = k / 100, hy = (k % 100) / 10, hx = k % 10;
      const int gy = wrap(y0 - 1 + hy, N), gx = wrap(x0 - 1 + hx, N), ci = cib * CIB + c;
      hs[c][hy][hx] = PLANAR ? H[((size_t)b * CI + ci) * NN + (size_t)gy * N + gx]
                             : H[(((size_t)b * N + gy) * N + gx) * CI + ci];
    }
    __syncthreads();
    for (int c = 0; c < 64; ++c) {
      const float g = gs[c][co_l];
      const int cy = c / 8, cx = c % 8;
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) acc[ky * 3 + kx] = fmaf(g, hs[ci_l][cy + ky][cx + kx], acc[ky * 3 + kx]);
      bacc += g;
    }
  }
  const int ci = cib * CIB + ci_l, co = cob * COB + co_l;
#pragma unroll
  for (int t = 0; t < 9; ++t) atomicAdd(Wb + ((size_t)t * CI + ci) * CO + co, acc[t]);
  if (cib == 0 && ci_l == 0) atomicAdd(bb + co, bacc);
}

// transposed, tap-flipped weights of the backward data conv: Wt[tap'][o][c] = W[8 - tap'][c][o]
// (W: [9][ci][co_pad] of the forward SIMT conv; Wt: [9][co_pad][cout_pad], zero for c >= ci)
__global__ void transpose_w_kernel(const float* __restrict__ W, int ci, int co_pad, int cout_pad, float* __restrict__ Wt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= 9 * co_pad * cout_pad) return;
  const int tap = k / (co_pad * cout_pad), o = (k / cout_pad) % co_pad, c = k % cout_pad;
  Wt[k] = c < ci ? W[((size_t)(8 - tap) * ci + c) * co_pad + o] : 0.f;
}

// gradient accumulators ([9][ci][co_pad] + [co_pad]) -> += the blob layout W[co][ky][kx][ci], b[co]
__global__ void pack_grads_kernel(const float* __restrict__ Wb, const float* __restrict__ bb, int ci, int co, int co_pad,
                                  float* __restrict__ blob) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int nw = co * 9 * ci;
  if (k < nw) {
    const int o = k / (9 * ci), tap = (k / ci) % 9, c = k % ci;
    blob[k] += Wb[((size_t)tap * ci + c) * co_pad + o];
  } else if (k < nw + co) {
    blob[k] += bb[k - nw];
  }
}

}  // namespace adj

static inline unsigned nblk(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

cudaError_t adj_fwd_faces(const float* U, const float* R, const float* base24, int N, int B, float inv_h, float nu,
                          float gamma, float* w_out, float* F4, cudaStream_t st) {
  adj::Base24 bs;
  for (int k = 0; k < 24; ++k) bs.w[k] = base24[k];
  adj::fwd_faces_kernel<<<nblk((size_t)B * N * N), 256, 0, st>>>(U, R, bs, N, B, inv_h, nu, gamma, w_out, F4);
  return cudaGetLastError();
}
cudaError_t adj_extract_e(const float* R, int N, int B, float* E, cudaStream_t st) {
  adj::extract_e_kernel<<<nblk((size_t)B * N * N), 256, 0, st>>>(R, N, B, E);
  return cudaGetLastError();
}
cudaError_t adj_fwd_combine(const float* F4, const float* U, const float* un, const float* E, int N, int B, float inv_h,
                            int forced, const float* force_row, float drag, float a, float b, float cdt, float ec,
                            float* Tout, float* Y, cudaStream_t st) {
  adj::fwd_combine_kernel<<<nblk((size_t)B * N * N), 256, 0, st>>>(F4, U, un, E, N, B, inv_h, forced, force_row, drag,
                                                                   a, b, cdt, ec, Tout, Y);
  return cudaGetLastError();
}
cudaError_t adj_bwd_faces(const float* U, const float* w, const float* Tb, const float* eb, int N, int B, float inv_h,
                          float nu, float gamma, float* Fadj, float* Rb, cudaStream_t st) {
  adj::bwd_faces_kernel<<<nblk((size_t)B * N * N), 256, 0, st>>>(U, w, Tb, eb, N, B, inv_h, nu, gamma, Fadj, Rb);
  return cudaGetLastError();
}
cudaError_t adj_bwd_gather(const float* Fadj, const float* w, const float* Tb, int N, int B, int forced, float drag,
                           float* Ub, cudaStream_t st) {
  adj::bwd_gather_kernel<<<nblk((size_t)B * N * N), 256, 0, st>>>(Fadj, w, Tb, N, B, forced, drag, Ub);
  return cudaGetLastError();
}
cudaError_t adj_act(const float* z, float* y, size_t n, int act, int mode, cudaStream_t st) {
  adj::act_kernel<<<nblk(n), 256, 0, st>>>(z, y, n, act, mode);
  return cudaGetLastError();
}
cudaError_t adj_lin3(float* out, float a, const float* x, float b, const float* y, float c, const float* z, size_t n,
                     cudaStream_t st) {
  adj::lin3_kernel<<<nblk(n), 256, 0, st>>>(out, a, x, b, y, c, z, n);
  return cudaGetLastError();
}
cudaError_t adj_wgrad(const float* H, bool planar, int ci, const float* G, int co_pad, int N, int B, float* Wb, float* bb,
                      cudaStream_t st) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int ntiles = B * (N / 8) * (N / 8);
  const int gx = ntiles < 2 * sms ? ntiles : 2 * sms;
#define LD_WG(CI_, CO_, CIB_, COB_, PL_)                                                                        \
  if (ci == CI_ && co_pad == CO_ && planar == PL_) {                                                          \
    adj::wgrad_kernel<CI_, CO_, CIB_, COB_, PL_><<<dim3(gx, (CI_ / CIB_) * (CO_ / COB_)), CIB_ * COB_, 0, st>>>( \
        H, G, N, B, Wb, bb);                                                                                    \
    return cudaGetLastError();                                                                                 \
  }
  LD_WG(2, 64, 2, 64, true) LD_WG(2, 32, 2, 32, true) LD_WG(64, 64, 16, 16, false) LD_WG(64, 32, 16, 16, false)
  LD_WG(32, 32, 16, 16, false)
#undef LD_WG
  return cudaErrorInvalidValue;
}
cudaError_t adj_transpose_w(const float* W, int ci, int co_pad, int cout_pad, float* Wt, cudaStream_t st) {
  adj::transpose_w_kernel<<<nblk((size_t)9 * co_pad * cout_pad), 256, 0, st>>>(W, ci, co_pad, cout_pad, Wt);
  return cudaGetLastError();
}
cudaError_t adj_pack_grads(const float* Wb, const float* bb, int ci, int co, int co_pad, float* blob, cudaStream_t st) {
  adj::pack_grads_kernel<<<nblk((size_t)co * 9 * ci + co), 256, 0, st>>>(Wb, bb, ci, co, co_pad, blob);
  return cudaGetLastError();
}

}  // namespace ld
