// fft.cu -- the FFT pressure projection for N <= 128:
//
//   d = D_c U*,  d_hat = DFT2(d),  p_hat = -d_hat / (kx_hat^2 + ky_hat^2)  (0 on the four null
//   modes mx, my in {0, N/2}),  p = IDFT2(p_hat),  U = U* - G_c p
//   with k_hat_m = sin(2 pi m / N) / h (exactly 0 at m = 0, N/2)
// (Eq.13-15, "spectral solver" P:315; readings R10, R23).
// Twiddles exp(-2 pi i k / N) and the symbol k_hat^2 are evaluated in fp64 on the host at
// ld_init and rounded once to fp32.  N >= 256 (and the slab decomposition) use pencil.cu.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "warpfft.cuh"
#ifndef LD_PROJ_RELAXED
#define LD_PROJ_RELAXED 1
#endif

namespace ld {

// ---------------------------------------------------------------------------
// Register-blocked Stockham autosort FFT (natural order in and out) for the fused small-N
// projection: radix-8 passes (radix 4/2 for the remainder), each pass = every thread loads
// its butterflies' R inputs into registers, one barrier, every thread stores -- so an
// N = 64 transform costs 2 barrier pairs instead of 6 radix-2 stages.
//   pass (R, Ns): for butterfly j in [0, N/R): k = j % Ns,
//     v_r = x[j + r N/R] * w^{r k / (Ns R)},  v = DFT_R(v),  y[(j/Ns) Ns R + k + r Ns] = v_r
// ---------------------------------------------------------------------------
LD_DEVINL float2 twid(const float2* __restrict__ tw, int m, int n) {   // e^{-2 pi i m / n}, m in [0, n)
  const float2 w = __ldg(tw + (m & (n / 2 - 1)));
  return (m & (n / 2)) ? make_float2(-w.x, -w.y) : w;
}

template <int R>
LD_DEVINL void dft_small(float2 (&v)[8], bool inv) {
  const float sg = inv ? 1.f : -1.f;   // exponent sign
  if (R == 2) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b); v[1] = csub(a, b);
  } else if (R == 4) {
    const float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    const float2 b0 = cadd(v[1], v[3]), b1 = csub(v[1], v[3]);
    const float2 jb1 = make_float2(-sg * b1.y, sg * b1.x);   // (sg i) * b1
    v[0] = cadd(a0, b0); v[2] = csub(a0, b0);
    v[1] = cadd(a1, jb1); v[3] = csub(a1, jb1);
  } else {   // R == 8: two radix-4 on even/odd, then combine with w8^k
    float2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    auto r4 = [&](float2 (&x)[4]) {
      const float2 a0 = cadd(x[0], x[2]), a1 = csub(x[0], x[2]);
      const float2 b0 = cadd(x[1], x[3]), b1 = csub(x[1], x[3]);
      const float2 jb1 = make_float2(-sg * b1.y, sg * b1.x);
      x[0] = cadd(a0, b0); x[2] = csub(a0, b0);
      x[1] = cadd(a1, jb1); x[3] = csub(a1, jb1);
    };
    r4(e); r4(o);
    const float c = 0.70710678118654752f;
    const float2 w1 = make_float2(c, sg * c), w2 = make_float2(0.f, sg), w3 = make_float2(-c, sg * c);
    const float2 o1 = cmul(w1, o[1]), o2 = cmul(w2, o[2]), o3 = cmul(w3, o[3]);
    v[0] = cadd(e[0], o[0]); v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);   v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);   v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);   v[7] = csub(e[3], o3);
  }
}

// out-of-place pass src -> dst (separate buffers, so no register blocking is needed and the
// code stays compact: one loop per radix)
template <int R>
LD_DEVINL void stockham_pass(const float2* src, float2* dst, int pitch, int nseq, int n, int Ns,
                             const float2* __restrict__ tw, bool inv) {
  const int nb = n / R, total = nseq * nb;
#pragma unroll 1
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int q = t / nb, j = t - q * nb, k = j % Ns;
    const float2* x = src + q * pitch;
    float2 v[8];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float2 a = x[j + r * nb];
      if (r > 0 && Ns > 1) {
        float2 w = twid(tw, (r * k * (n / (Ns * R))) & (n - 1), n);
        if (inv) w.y = -w.y;
        a = cmul(a, w);
      }
      v[r] = a;
    }
    dft_small<R>(v, inv);
    float2* y = dst + q * pitch + (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) y[r * Ns] = v[r];
  }
  __syncthreads();
}

// whole transform of nseq sequences of length n (power of two >= 8), natural order, ping-pong
// between *a and *b; returns the buffer holding the result
__device__ __noinline__ float2* fft_stockham(float2* a, float2* b, int pitch, int nseq, int n,
                                             const float2* __restrict__ tw, bool inv) {
  int Ns = 1;
  while (Ns < n) {
    const int rem = n / Ns;
    if (rem >= 8) { stockham_pass<8>(a, b, pitch, nseq, n, Ns, tw, inv); Ns *= 8; }
    else if (rem == 4) { stockham_pass<4>(a, b, pitch, nseq, n, Ns, tw, inv); Ns *= 4; }
    else { stockham_pass<2>(a, b, pitch, nseq, n, Ns, tw, inv); Ns *= 2; }
    float2* t = a; a = b; b = t;
  }
  return a;
}

// Fused single-CTA projection for N < 32 (one element per CTA), natural-order Stockham FFTs.
//   Z [N/2][N] row pairs, S [N/2+1][N] column-major half spectrum, W scratch (size of S)
__global__ void __launch_bounds__(512)
proj_fused_stockham(const float* Ustar, float* Uout, int N, float half_inv_h, const float2* __restrict__ tw,
                    const float* __restrict__ ksym2, float inv_n2) {
  extern __shared__ float2 s2[];
  const int H = N / 2 + 1;
  float2* Z = s2;
  float2* S = s2 + (N / 2) * N;
  float2* W = S + H * N;
  const int b = blockIdx.x;
  const size_t plane = (size_t)N * N;
  const float* u = Ustar + (size_t)b * 2 * plane;
  const float* v = u + plane;
  for (int idx = threadIdx.x; idx < (N / 2) * N; idx += blockDim.x) {
    const int rp = idx / N, i = idx - rp * N;
    float d[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = 2 * rp + r;
      const float du = u[(size_t)j * N + wrap(i + 1, N)] - u[(size_t)j * N + wrap(i - 1, N)];
      const float dv = v[(size_t)wrap(j + 1, N) * N + i] - v[(size_t)wrap(j - 1, N) * N + i];
      d[r] = (du + dv) * half_inv_h;
    }
    Z[idx] = make_float2(d[0], d[1]);
  }
  __syncthreads();
  const float2* Zf = fft_stockham(Z, W, N, N / 2, N, tw, false);     // row FFTs
  for (int idx = threadIdx.x; idx < (N / 2) * H; idx += blockDim.x) {
    const int rp = idx / H, k = idx - rp * H;
    const float2 zk = Zf[rp * N + k], zn = conjf2(Zf[rp * N + ((N - k) & (N - 1))]);
    const float2 sum = cadd(zk, zn), dif = csub(zk, zn);
    S[k * N + 2 * rp] = make_float2(0.5f * sum.x, 0.5f * sum.y);
    S[k * N + 2 * rp + 1] = make_float2(0.5f * dif.y, -0.5f * dif.x);
  }
  __syncthreads();
  float2* Sf = fft_stockham(S, W, N, H, N, tw, false);               // column FFTs
  for (int idx = threadIdx.x; idx < H * N; idx += blockDim.x) {
    const int kx = idx / N, my = idx - kx * N;
    const bool null_mode = (kx == 0 || kx == N / 2) && (my == 0 || my == N / 2);
    const float scale = null_mode ? 0.f : -inv_n2 / (__ldg(ksym2 + kx) + __ldg(ksym2 + my));
    const float2 z = Sf[idx];
    Sf[idx] = make_float2(z.x * scale, z.y * scale);
  }
  __syncthreads();
  float2* other = (Sf == S) ? W : S;
  const float2* Si = fft_stockham(Sf, other, N, H, N, tw, true);     // inverse columns
  for (int idx = threadIdx.x; idx < (N / 2) * N; idx += blockDim.x) {
    const int rp = idx / N, k = idx - rp * N;
    float2 X, Y;
    if (k <= N / 2) {
      X = Si[k * N + 2 * rp]; Y = Si[k * N + 2 * rp + 1];
      if (k == 0 || k == N / 2) { X.y = 0.f; Y.y = 0.f; }
    } else {
      X = conjf2(Si[(N - k) * N + 2 * rp]); Y = conjf2(Si[(N - k) * N + 2 * rp + 1]);
    }
    Z[idx] = make_float2(X.x - Y.y, X.y + Y.x);
  }
  __syncthreads();
  float2* scratch = (Si == W) ? S : W;
  const float2* Pz = fft_stockham(Z, scratch, N, N / 2, N, tw, true);  // inverse rows
  auto P = [&](int j, int i) { const float2 z = Pz[(j >> 1) * N + i]; return (j & 1) ? z.y : z.x; };
  float* uo = Uout + (size_t)b * 2 * plane;
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    const int j = idx / N, i = idx - j * N;
    const float gx = (P(j, wrap(i + 1, N)) - P(j, wrap(i - 1, N))) * half_inv_h;
    const float gy = (P(wrap(j + 1, N), i) - P(wrap(j - 1, N), i)) * half_inv_h;
    const float a = u[idx], c = v[idx];
    uo[idx] = a - gx;
    uo[plane + idx] = c - gy;
  }
}


// Fused projection of ONE batch element, N = 32 E <= 128, on a thread-block cluster of CL CTAs.
// The divergence is transformed as a complex field z = d + 0 i (each element on its own: packing
// two elements into one complex FFT would halve the arithmetic but couple their rounding, and
// batch permutation must permute the outputs bitwise -- SURVEY.md §8c Pin-14).
// CTA r of the cluster owns rows [r R, (r+1) R), R = N / CL, as Z [R][N+1] float2 in its shared
// memory; the column pass reads and writes the other CTAs' rows through distributed shared
// memory (the whole pair stays on chip: U* is read once, U written once).
//   1. rows:    z = D_c U*  -> FFT along x            (own rows)
//   2. columns: FFT along y, * -1/(N^2 (kx^2+ky^2)), inverse FFT along y   (own column range)
//   3. rows:    inverse FFT along x -> (p_b0, p_b1)   (own rows)
//   4. U = U* - G_c p                                  (own rows; y +- 1 rows of the neighbours)
template <int E>
__global__ void __launch_bounds__(512)
proj_cluster(const float* Ustar, float* Uout, int B, float half_inv_h, const float2* __restrict__ tw_g,
                  const float* __restrict__ ksym2_g, float scale) {
  namespace cg = cooperative_groups;
  constexpr int N = 32 * E, NP = N + 1;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  const int R = N / CL;
  extern __shared__ float2 s2[];
  float2* Z = s2;                              // [R][NP] own rows
  float2* tw = Z + R * NP;                     // [N]
  float* ks = reinterpret_cast<float*>(tw + N);   // [N]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int b0 = blockIdx.x / CL;
  constexpr bool two = false;
  const size_t plane = (size_t)N * N;
  const int y0 = rank * R;
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    const float2 w = tw_g[m & (N / 2 - 1)];
    tw[m] = (m & (N / 2)) ? make_float2(-w.x, -w.y) : w;
    ks[m] = ksym2_g[m];
  }
  const float* u0 = Ustar + (size_t)b0 * 2 * plane;
  const float* u1 = u0;
  __syncthreads();
  // 1. own rows: z = D_c U* -> FFT along x
  for (int yl = warp; yl < R; yl += nw) {
    const int y = y0 + yl;
    float2 v[E];
    const int ym = wrap(y - 1, N), yp = wrap(y + 1, N);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int x = lane + 32 * e, xm = wrap(x - 1, N), xp = wrap(x + 1, N);
      const float d0 = (__ldg(u0 + (size_t)y * N + xp) - __ldg(u0 + (size_t)y * N + xm) +
                        __ldg(u0 + plane + (size_t)yp * N + x) - __ldg(u0 + plane + (size_t)ym * N + x)) * half_inv_h;
      const float d1 = two ? (__ldg(u1 + (size_t)y * N + xp) - __ldg(u1 + (size_t)y * N + xm) +
                              __ldg(u1 + plane + (size_t)yp * N + x) - __ldg(u1 + plane + (size_t)ym * N + x)) *
                                 half_inv_h
                           : 0.f;
      v[e] = make_float2(d0, d1);
    }
    warp_fft_fwd<E>(v, tw);
    const int kb = E * bitrev5(lane);
#pragma unroll
    for (int k = 0; k < E; ++k) Z[yl * NP + kb + k] = v[k];
  }
  cluster.sync();
  // 2. own column range [rank N/CL, (rank+1) N/CL): rows of every CTA through DSMEM
  {
    const int C0 = rank * (N / CL), C1 = C0 + N / CL;
    float2* rowbase[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int y = lane + 32 * e;
      rowbase[e] = cluster.map_shared_rank(Z, y / R) + (y % R) * NP;
    }
    for (int kx = C0 + warp; kx < C1; kx += nw) {
      float2 v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = rowbase[e][kx];
      warp_fft_fwd<E>(v, tw);
      const int kb = E * bitrev5(lane);
      const bool xnull = kx == 0 || kx == N / 2;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int ky = kb + k;
        const bool nul = xnull && (ky == 0 || ky == N / 2);
        const float f = nul ? 0.f : -scale / (ks[kx] + ks[ky]);
        v[k] = make_float2(v[k].x * f, v[k].y * f);
      }
      warp_fft_inv<E>(v, tw);
#pragma unroll
      for (int e = 0; e < E; ++e) rowbase[e][kx] = v[e];
    }
  }
  cluster.sync();
  // 3. own rows: inverse along x -> (p_b0, p_b1)(x, y), in place
  for (int yl = warp; yl < R; yl += nw) {
    float2 v[E];
    const int kb = E * bitrev5(lane);
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = Z[yl * NP + kb + k];
    __syncwarp();
    warp_fft_inv<E>(v, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) Z[yl * NP + lane + 32 * e] = v[e];
  }
  cluster.sync();
  // 4. U = U* - G_c p on own rows (rows y0 - 1 and y0 + R from the neighbouring CTAs)
  {
    const float2* below = cluster.map_shared_rank(Z, (rank + CL - 1) % CL) + (R - 1) * NP;   // row y0 - 1
    const float2* above = cluster.map_shared_rank(Z, (rank + 1) % CL);                       // row y0 + R
    float* o0 = Uout + (size_t)b0 * 2 * plane;
    float* o1 = o0 + 2 * plane;
    for (int idx = threadIdx.x; idx < R * N; idx += blockDim.x) {
      const int yl = idx / N, x = idx - yl * N;
      const size_t gi = (size_t)(y0 + yl) * N + x;
      const float2 gx = csub(Z[yl * NP + wrap(x + 1, N)], Z[yl * NP + wrap(x - 1, N)]);
      const float2 pu = yl + 1 < R ? Z[(yl + 1) * NP + x] : above[x];
      const float2 pd = yl > 0 ? Z[(yl - 1) * NP + x] : below[x];
      const float2 gy = csub(pu, pd);
      o0[gi] = u0[gi] - gx.x * half_inv_h;
      o0[plane + gi] = u0[plane + gi] - gy.x * half_inv_h;
      if (two) {
        o1[gi] = u1[gi] - gx.y * half_inv_h;
        o1[plane + gi] = u1[plane + gi] - gy.y * half_inv_h;
      }
    }
  }
  // no CTA leaves while a neighbour may still read its rows: the neighbours' DSMEM reads have
  // returned (their values were stored) before they arrive, so no release / acquire is needed
  // (a release here would wait for this CTA's global stores to drain)
  if (LD_PROJ_RELAXED) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  } else {
    cluster.sync();
  }
}

// ---------------------------------------------------------------------------
// Fused K2 + projection for one RK stage of the single-domain step, N = 32 E <= 64 (c2): the
// flux / divergence / RK kernel (flux.cu, rows a3-a5) and proj_cluster (row a6) in one
// cluster-per-element kernel, so U* never leaves shared memory and the two launches, their
// gap and the U* write + re-read disappear.  CTA r of the cluster owns rows [r R, (r+1) R):
//   F0. U rows y0-3 .. y0+R+2 (periodic) -> smem
//   F1. face fluxes of the own cells + the y-faces of row y0+R (same formulas as flux.cu)
//   F2. T, forcing / drag, Shu-Osher combination -> U* own rows (smem; acc to global)
//   P1-P4. as proj_cluster, with U* and its rows y0-1 / y0+R read from (distributed) smem
// The arithmetic of every value is the same sequence of fp32 operations as the two-kernel
// path, so the fused step is bitwise identical to it.
template <int E, bool FIXED, bool FNO>
__global__ void __launch_bounds__(512)
flux_proj_cluster(FluxParams P, StageCoef S, BaseStencil base, const float* __restrict__ X, const float* un,
                  const float* __restrict__ w, const float* __restrict__ e, float* acc, float* Uout,
                  float half_inv_h, const float2* __restrict__ tw_g, const float* __restrict__ ksym2_g,
                  float scale) {
  namespace cg = cooperative_groups;
  constexpr int N = 32 * E, NP = N + 1;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  const int R = N / CL, HR = R + 6;
  const int b = blockIdx.x / CL;
  const int y0 = rank * R;
  const size_t plane = (size_t)N * N;
  extern __shared__ __align__(16) float smf[];
  // every global input of the stage is staged with cp.async at entry (one latency period):
  float* Us = smf;                                   // [2][R][N] U* own rows (to the end)
  float* us = Us + 2 * R * N;                        // [2][HR][N] U rows y0-3 .. y0+R+2
  float* uns = us + 2 * HR * N;                      // [2][R][N] u^n own rows
  float* accs = uns + 2 * R * N;                     // [2][R][N] RK4 accumulator own rows
  float* es = accs + 2 * R * N;                      // [N][R][2] TC term e (x-major like e)
  float* Fx = es + 2 * R * N;                        // [2][R][N]
  float* Fy = Fx + 2 * R * N;                        // [2][R+1][N]
  float* ws = Fy + 2 * (R + 1) * N;                  // [N][R+1][24] stencils of rows y0 .. y0+R
  float2* Z = reinterpret_cast<float2*>(ws);         // P: [R][NP] (aliases ws, dead after F1)
  const int wsz = FIXED ? 2 * R * NP : std::max(N * (R + 1) * 24, 2 * R * NP);
  float2* tw = reinterpret_cast<float2*>(ws + wsz);  // [N]
  float* ks = reinterpret_cast<float*>(tw + N);       // [N]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool need_acc = S.q != 0.f || (S.r != 0.f && !S.acc_init);
  auto cp16 = [](float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
  };
  // F0: stage U halo rows, w of rows y0 .. y0+R (x-major runs of R+1 cells, split at the wrap),
  // u^n / acc own rows, e.  Warp-per-row loops: a lane's 16-B chunk index is its lane (+32 k),
  // so the per-chunk cost is an add and the copy.
  {
    constexpr int C4 = N / 4;                      // 16-B chunks per field row
    const float* Xb = X + (size_t)b * 2 * plane;
    for (int ry = warp; ry < HR; ry += nw) {       // U halo rows, both components
      const float* src = Xb + (size_t)wrap(y0 - 3 + ry, N) * N;
      for (int j = lane; j < 2 * C4; j += 32) {
        const int c = j / C4, x4 = j - c * C4;
        cp16(us + (c * HR + ry) * N + 4 * x4, src + c * plane + 4 * x4);
      }
    }
    if (S.a != 0.f || need_acc) {
      for (int ly = warp; ly < R; ly += nw) {
        for (int j = lane; j < 2 * C4; j += 32) {
          const int c = j / C4, x4 = j - c * C4;
          const size_t gi = ((size_t)b * 2 + c) * plane + (size_t)(y0 + ly) * N + 4 * x4;
          if (S.a != 0.f) cp16(uns + (c * R + ly) * N + 4 * x4, un + gi);
          if (need_acc) cp16(accs + (c * R + ly) * N + 4 * x4, acc + gi);
        }
      }
    }
    if (S.add_e) {   // e[b][x][y][2]: per x a run of R cells x 8 B (R even: whole 16-B chunks)
      const float* eb = e + (size_t)b * plane * 2;
      for (int x = warp; x < N; x += nw)
        for (int j = lane; j < R / 2; j += 32) cp16(es + (x * R + 2 * j) * 2, eb + ((size_t)x * N + y0 + 2 * j) * 2);
    }
    if (!FIXED) {   // cell (x, ly) at ws[(x (R+1) + ly) 24]: per x one run of (R+1) 6 chunks
      const float* wb = w + (size_t)b * plane * 24;
      const int rwrap = (N - y0) * 6;              // chunks at / past this index wrap to y = 0
      for (int x = warp; x < N; x += nw) {
        const float* src = wb + ((size_t)x * N + y0) * 24;
        float* dst = ws + x * (R + 1) * 24;
        for (int r = lane; r < (R + 1) * 6; r += 32)
          cp16(dst + 4 * r, src + 4 * r - (r >= rwrap ? N * 24 : 0));
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    const float2 t = tw_g[m & (N / 2 - 1)];
    tw[m] = (m & (N / 2)) ? make_float2(-t.x, -t.y) : t;
    ks[m] = ksym2_g[m];
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // F1: x-face of cell (x, ly) and y-face of cell (x, ly) (ly = R: the +y neighbour row)
  auto wload = [&](int x, int ly, int off, float (&wv)[12]) {
    if (FIXED) {
#pragma unroll
      for (int t = 0; t < 12; ++t) wv[t] = base.w[off + t];
    } else {
      const float4* w4 = reinterpret_cast<const float4*>(ws + (x * (R + 1) + ly) * 24 + off);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const float4 v = w4[q];
        wv[4 * q] = v.x; wv[4 * q + 1] = v.y; wv[4 * q + 2] = v.z; wv[4 * q + 3] = v.w;
      }
    }
  };
  for (int idx = threadIdx.x; idx < (R + 1) * N; idx += blockDim.x) {
    const int ly = idx / N, x = idx - ly * N;
    if (ly < R) {   // x-face i-1/2 of cell (x, y0+ly): taps x-3 .. x+2 of row ly+3
      float wv[12];
      wload(x, ly, 0, wv);
      const float* u0 = us + (0 * HR + ly + 3) * N;
      const float* v0 = us + (1 * HR + ly + 3) * N;
      float uI = 0.f, uD = 0.f, vI = 0.f, vD = 0.f;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const int xt = wrap(x - 3 + t, N);
        const float uu = u0[xt], vv = v0[xt];
        uI = fmaf(wv[t], uu, uI); uD = fmaf(wv[6 + t], uu, uD);
        vI = fmaf(wv[t], vv, vI); vD = fmaf(wv[6 + t], vv, vD);
      }
      float gu = uD * P.inv_h, gv = vD * P.inv_h;
      if (FNO) {   // NEXT-2 branch at this x-face (channels 0-3)
        const size_t fi = ((size_t)b * 8 * N + y0 + ly) * N + x;
        uI += P.fno[fi]; vI += P.fno[fi + plane]; gu += P.fno[fi + 2 * plane]; gv += P.fno[fi + 3 * plane];
      }
      const float adv = P.gamma * uI;
      Fx[(0 * R + ly) * N + x] = adv * uI - P.nu * gu;
      Fx[(1 * R + ly) * N + x] = adv * vI - P.nu * gv;
    }
    {   // y-face j-1/2 of cell (x, y0+ly): taps rows ly .. ly+5 (y-3 .. y+2)
      float wv[12];
      wload(x, ly, 12, wv);
      const float* u0 = us + (0 * HR + ly) * N + x;
      const float* v0 = us + (1 * HR + ly) * N + x;
      float uI = 0.f, uD = 0.f, vI = 0.f, vD = 0.f;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const float uu = u0[t * N], vv = v0[t * N];
        uI = fmaf(wv[t], uu, uI); uD = fmaf(wv[6 + t], uu, uD);
        vI = fmaf(wv[t], vv, vI); vD = fmaf(wv[6 + t], vv, vD);
      }
      float gu = uD * P.inv_h, gv = vD * P.inv_h;
      if (FNO) {   // NEXT-2 branch at this y-face (channels 4-7)
        const size_t fi = ((size_t)b * 8 * N + wrap(y0 + ly, N)) * N + x + 4 * plane;
        uI += P.fno[fi]; vI += P.fno[fi + plane]; gu += P.fno[fi + 2 * plane]; gv += P.fno[fi + 3 * plane];
      }
      const float adv = P.gamma * vI;
      Fy[(0 * (R + 1) + ly) * N + x] = adv * uI - P.nu * gu;
      Fy[(1 * (R + 1) + ly) * N + x] = adv * vI - P.nu * gv;
    }
  }
  __syncthreads();
  // F2: divergence, forcing / drag, Shu-Osher stage -> U* (own rows, smem)
  for (int idx = threadIdx.x; idx < R * N; idx += blockDim.x) {
    const int ly = idx / N, x = idx - ly * N, y = y0 + ly;
    float T[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float t = -((Fx[(c * R + ly) * N + wrap(x + 1, N)] - Fx[(c * R + ly) * N + x]) +
                  (Fy[(c * (R + 1) + ly + 1) * N + x] - Fy[(c * (R + 1) + ly) * N + x])) * P.inv_h;
      if (P.forced) {
        if (c == 0) t += P.force_row[y];
        t -= P.drag * us[(c * HR + ly + 3) * N + x];
      }
      T[c] = t;
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float unv = S.a != 0.f ? uns[(c * R + ly) * N + x] : 0.f;
      const float acv = need_acc ? accs[(c * R + ly) * N + x] : 0.f;
      float v = S.a * unv + S.b * us[(c * HR + ly + 3) * N + x] + S.c * P.dt * T[c];
      if (S.q != 0.f) v += S.q * P.dt * acv;
      if (S.add_e) v += es[(x * R + ly) * 2 + c];
      if (S.r != 0.f) acc[((size_t)b * 2 + c) * plane + (size_t)y * N + x] = acv + S.r * T[c];
      Us[(c * R + ly) * N + x] = v;
    }
  }
  cluster.sync();   // U* rows visible to the neighbours; the F buffers are free for Z
  // P1: own rows: z = D_c U* -> FFT along x
  {
    const float* vbelow = cluster.map_shared_rank(Us, (rank + CL - 1) % CL) + (2 * R - 1) * N;   // v row y0-1
    const float* vabove = cluster.map_shared_rank(Us, (rank + 1) % CL) + R * N;                  // v row y0+R
    for (int yl = warp; yl < R; yl += nw) {
      const float* ur = Us + yl * N;
      const float* vp = yl + 1 < R ? Us + (R + yl + 1) * N : vabove;
      const float* vm = yl > 0 ? Us + (R + yl - 1) * N : vbelow;
      float2 v[E];
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int x = lane + 32 * q;
        const float d0 = (ur[wrap(x + 1, N)] - ur[wrap(x - 1, N)] + vp[x] - vm[x]) * half_inv_h;
        v[q] = make_float2(d0, 0.f);
      }
      warp_fft_fwd<E>(v, tw);
      const int kb = E * bitrev5(lane);
#pragma unroll
      for (int k = 0; k < E; ++k) Z[yl * NP + kb + k] = v[k];
    }
  }
  cluster.sync();
  // P2: own column range through DSMEM (as proj_cluster)
  {
    const int C0 = rank * (N / CL), C1 = C0 + N / CL;
    float2* rowbase[E];
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int y = lane + 32 * q;
      rowbase[q] = cluster.map_shared_rank(Z, y / R) + (y % R) * NP;
    }
    for (int kx = C0 + warp; kx < C1; kx += nw) {
      float2 v[E];
#pragma unroll
      for (int q = 0; q < E; ++q) v[q] = rowbase[q][kx];
      warp_fft_fwd<E>(v, tw);
      const int kb = E * bitrev5(lane);
      const bool xnull = kx == 0 || kx == N / 2;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int ky = kb + k;
        const bool nul = xnull && (ky == 0 || ky == N / 2);
        const float f = nul ? 0.f : -scale / (ks[kx] + ks[ky]);
        v[k] = make_float2(v[k].x * f, v[k].y * f);
      }
      warp_fft_inv<E>(v, tw);
#pragma unroll
      for (int q = 0; q < E; ++q) rowbase[q][kx] = v[q];
    }
  }
  cluster.sync();
  // P3: own rows: inverse along x -> p (real part)
  for (int yl = warp; yl < R; yl += nw) {
    float2 v[E];
    const int kb = E * bitrev5(lane);
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = Z[yl * NP + kb + k];
    __syncwarp();
    warp_fft_inv<E>(v, tw);
#pragma unroll
    for (int q = 0; q < E; ++q) Z[yl * NP + lane + 32 * q] = v[q];
  }
  cluster.sync();
  // P4: U = U* - G_c p on own rows
  {
    const float2* below = cluster.map_shared_rank(Z, (rank + CL - 1) % CL) + (R - 1) * NP;
    const float2* above = cluster.map_shared_rank(Z, (rank + 1) % CL);
    float* o0 = Uout + (size_t)b * 2 * plane;
    for (int idx = threadIdx.x; idx < R * N; idx += blockDim.x) {
      const int yl = idx / N, x = idx - yl * N;
      const size_t gi = (size_t)(y0 + yl) * N + x;
      const float2 gx = csub(Z[yl * NP + wrap(x + 1, N)], Z[yl * NP + wrap(x - 1, N)]);
      const float2 pu = yl + 1 < R ? Z[(yl + 1) * NP + x] : above[x];
      const float2 pd = yl > 0 ? Z[(yl - 1) * NP + x] : below[x];
      const float2 gy = csub(pu, pd);
      o0[gi] = Us[yl * N + x] - gx.x * half_inv_h;
      o0[plane + gi] = Us[(R + yl) * N + x] - gy.x * half_inv_h;
    }
  }
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");   // neighbours done reading
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

static size_t flux_proj_smem_bytes(int N, int CL, bool fixed) {
  const int R = N / CL, HR = R + 6, NP = N + 1;
  const int wsz = fixed ? 2 * R * NP : std::max(N * (R + 1) * 24, 2 * R * NP);
  return sizeof(float) * ((size_t)2 * R * N * 5 + 2 * HR * N + 2 * (R + 1) * N + wsz + 3 * (size_t)N);
}

bool fused_stage_available(int n) { return (n == 32 || n == 64) && getenv("LD_NO_FUSED_STAGE") == nullptr; }

// Fused stage (flux + projection) for the single-domain NS step; returns cudaErrorNotSupported
// when the shape has no fused form (the caller then runs the two kernels).
cudaError_t launch_flux_projection(const FluxParams& P, const StageCoef& S, const float* base24, const float* X,
                                   const float* un, const float* w, const float* e, float* acc, float* Uout,
                                   const float2* tw, const float* ksym2, cudaStream_t st) {
  const int N = P.n, B = P.batch;
  if ((N != 32 && N != 64) || P.ny != N || P.rows != N || P.y_off != 0) return cudaErrorNotSupported;
  if (getenv("LD_NO_FUSED_STAGE") != nullptr) return cudaErrorNotSupported;   // knob: the two-kernel path
  const int min_rows = B >= 16 ? 16 : 4;
  int CL = 1;
  while (CL < 8 && B * CL < 148 && N / (2 * CL) >= min_rows) CL *= 2;
  while (N / CL > 16 && N == 64) CL *= 2;   // shared memory: at most 16 own rows at N = 64 (162 KB)
  BaseStencil bs;
  for (int i = 0; i < 24; ++i) bs.w[i] = base24 ? base24[i] : 0.f;
  const float half_inv_h = 0.5f / P.h;   // as launch_projection
  const float scale = 1.0f / ((float)N * (float)N);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B * CL);
  cfg.blockDim = dim3(512);
  const bool fixed = w == nullptr;
  cfg.dynamicSmemBytes = flux_proj_smem_bytes(N, CL, fixed);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define LD_FP(E, F, O) \
  return cudaLaunchKernelEx(&cfg, flux_proj_cluster<E, F, O>, P, S, bs, X, un, w, e, acc, Uout, half_inv_h, tw, ksym2, scale)
  const bool fno = P.fno != nullptr;   // (the branch needs learned stencils: never with fixed)
  if (N == 32) { if (fixed) LD_FP(1, true, false); else if (fno) LD_FP(1, false, true); else LD_FP(1, false, false); }
  if (fixed) LD_FP(2, true, false); else if (fno) LD_FP(2, false, true); else LD_FP(2, false, false);
#undef LD_FP
}

static size_t cluster_smem_bytes(int N, int CL) {
  return sizeof(float2) * ((size_t)(N / CL) * (N + 1) + N) + sizeof(float) * N;
}

template <int E>
static cudaError_t launch_proj_cluster(int CL, const float* Ustar, float* Uout, int B, float half_inv_h, const float2* tw,
                               const float* ksym2, float scale, cudaStream_t st) {
  constexpr int N = 32 * E;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B * CL);
  cfg.blockDim = dim3(N / CL >= 16 ? 512 : 256);
  cfg.dynamicSmemBytes = cluster_smem_bytes(N, CL);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, proj_cluster<E>, Ustar, Uout, B, half_inv_h, tw, ksym2, scale);
}



static size_t fused_smem_bytes(int N) { return sizeof(float2) * ((size_t)(N / 2) * N + 2 * (size_t)(N / 2 + 1) * N); }

cudaError_t launch_projection_pencil(const float* Ustar, float* Uout, float2* spec, float* p, int N, int B, float h,
                                     const float2* tw, const float* ksym2, cudaStream_t st);
cudaError_t pencil_set_smem_limits();

// N = 128 goes through the real-data pencil passes, measured faster than the cluster kernel at c3
// (59.8 vs 73.1 us per projection).  The choice depends on N only, never on the batch, so a batch and
// any shard or chunk of it run the same arithmetic (Pin-14, the pipelined host path);
// LD_PROJ_CLUSTER128=1 keeps the cluster kernel (measurement knob).
bool projection_uses_pencil(int N, int B) {
  (void)B;
  static const bool cluster128 = getenv("LD_PROJ_CLUSTER128") != nullptr;
  return N >= 256 || (N == 128 && !cluster128);
}

// Dispatch (every N a power of two in [8, 8192]):
//   N < 32        : proj_fused_stockham, one CTA per element (test sizes)
//   32 <= N <= 128: proj_cluster, one element per thread-block cluster (c1-c3)
//   N >= 256      : the pencil passes of pencil.cu (c4, c5; also the slab decomposition)
cudaError_t launch_projection(const float* Ustar, float* Uout, float2* spec, float* p, int N, int B, float h,
                              const float2* tw, const float* ksym2, cudaStream_t st) {
  const float half_inv_h = 0.5f / h;
  // N = 256 through one cluster-per-element kernel (proj_cluster<8>, 8 CTAs of 32 rows) instead of the
  // four pencil passes: measured slower at c4 (254-280 vs 162 us: latency-bound, 25% warps active), so
  // only with the measurement knob LD_PROJ_CLUSTER256=1
  static const bool cluster256 = getenv("LD_PROJ_CLUSTER256") != nullptr;
  if (N == 256 && cluster256)
    return launch_proj_cluster<8>(8, Ustar, Uout, B, half_inv_h, tw, ksym2, 1.0f / ((float)N * (float)N), st);
  if (projection_uses_pencil(N, B)) return launch_projection_pencil(Ustar, Uout, spec, p, N, B, h, tw, ksym2, st);
  if (N >= 32) {
    // cluster size: enough CTAs to cover the SMs, at most 8 (portable), at least 16 rows per CTA
    // (4 when the batch is small)
    const float scale = 1.0f / ((float)N * (float)N);
    // (measured at c2, N = 64, B = 32: CL = 4 -- 16 rows per CTA -- 12.7 us, CL = 8 14.1 us)
    const int min_rows = B >= 16 ? 16 : 4;
    int CL = 1;
    while (CL < 8 && B * CL < 148 && N / (2 * CL) >= min_rows) CL *= 2;
    static const int cl_env = getenv("LD_PROJ_CL") ? atoi(getenv("LD_PROJ_CL")) : 0;   // measurement knob
    if (cl_env > 0 && N / cl_env >= 2) CL = cl_env;
    if (N == 32) return launch_proj_cluster<1>(CL, Ustar, Uout, B, half_inv_h, tw, ksym2, scale, st);
    if (N == 64) return launch_proj_cluster<2>(CL, Ustar, Uout, B, half_inv_h, tw, ksym2, scale, st);
    return launch_proj_cluster<4>(CL, Ustar, Uout, B, half_inv_h, tw, ksym2, scale, st);
  }
  proj_fused_stockham<<<B, 512, fused_smem_bytes(N), st>>>(Ustar, Uout, N, half_inv_h, tw, ksym2,
                                                           1.0f / ((float)N * (float)N));
  return cudaGetLastError();
}

// Dynamic shared-memory limits of the projection kernels on the CURRENT device (function attributes
// are per device): called by ld_init, errors reported there.
cudaError_t projection_set_smem_limits() {
  cudaError_t e = pencil_set_smem_limits();
  if (e != cudaSuccess) return e;
  {
    const int mx = (int)flux_proj_smem_bytes(64, 4, false);   // >= every launched shape
#define LD_FPA(E, F, O)                                                                                   \
    if (e == cudaSuccess)                                                                                \
      e = cudaFuncSetAttribute(flux_proj_cluster<E, F, O>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    LD_FPA(1, false, false) LD_FPA(1, true, false) LD_FPA(2, false, false) LD_FPA(2, true, false)
    LD_FPA(1, false, true) LD_FPA(2, false, true)
#undef LD_FPA
    if (e != cudaSuccess) return e;
  }
  e = cudaFuncSetAttribute(proj_cluster<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cluster_smem_bytes(128, 1));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(proj_cluster<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cluster_smem_bytes(256, 8));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(proj_fused_stockham, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)fused_smem_bytes(16));
}

}  // namespace ld
