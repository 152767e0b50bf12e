// spectral.cu -- the frequency-domain operator O_F (Eq. 8; SURVEY.md §8f
// NEXT-2; readings N2-1..N2-4 in DESIGN.md §8c):
//
//   O_F(u) = Q( F^{-1}( R_L ... R_1 . F(u) ) ),  modes |kx|, |ky| <= K retained,
//   R_l(-k) = conj(R_l(k)) (real output), Q pointwise C -> 8.
//
// The L per-mode layers and Q are linear, so ld_spectral_create composes them on the host (in
// fp64, rounded once) into one 8 x 2 complex matrix per half-plane mode, M(k) = Q R_L(k)..R_1(k);
// the kernel then evaluates a truncated DFT directly -- with K << N only (K+1)(2K+1) of the N^2
// modes are non-zero, so partial DFT sums (x then y, and back) beat a full FFT:
//   1. A_c(y, kx)   = sum_x u_c(y, x) e^{-2 pi i kx x / N}              kx in [0, K]
//   2. U_c(kx, ky)  = sum_y A_c(y, kx) e^{-2 pi i ky y / N}             ky in [-K, K]
//   3. O_j(kx, ky)  = sum_c M_jc(kx, ky) U_c(kx, ky)                    half plane
//   4. B_j(y, kx)   = sum_ky O_j(kx, ky) e^{+2 pi i ky y / N}  (kx = 0: O_j(0,0) + 2 Re sum_{ky>0})
//   5. o_j(y, x)    = (B_j(y, 0) + 2 Re sum_{kx>0} B_j(y, kx) e^{+2 pi i kx x / N}) / N^2
// One CTA per (element, group of JG output channels): the forward part (1-2) is recomputed per
// group (it is ~15% of the work) so the grid has 8/JG CTAs per element.
#include <algorithm>
#include <cooperative_groups.h>

#include "common.cuh"

namespace ld {


// C[M][Nc] = A[M][Kd] (row stride lda) x B[Kd][Nc] (row stride ldb, 16-B aligned rows) with 4 x 4
// register tiles per thread; st(m0, n0, acc) stores a tile.  M, Nc multiples of 4.  Threads of a
// warp take consecutive column tiles, so B rows are read as float4 by few distinct addresses and
// the A column values are broadcast within a tile row (lda = 1 mod 8 keeps tile rows on distinct
// banks).
template <class Store>
LD_DEVINL void sp_gemm44(const float* A, int lda, const float* Bm, int ldb, int M, int Nc, int Kd, Store st) {
  const int tn = Nc / 4, tiles = (M / 4) * tn;
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    const int m0 = (t / tn) * 4, n0 = (t - (t / tn) * tn) * 4;
    float acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = 0.f;
    const float* a0 = A + m0 * lda;
    for (int k = 0; k < Kd; ++k) {
      const float4 b = *reinterpret_cast<const float4*>(Bm + k * ldb + n0);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float a = a0[r * lda + k];
        acc[r][0] = fmaf(a, b.x, acc[r][0]);
        acc[r][1] = fmaf(a, b.y, acc[r][1]);
        acc[r][2] = fmaf(a, b.z, acc[r][2]);
        acc[r][3] = fmaf(a, b.w, acc[r][3]);
      }
    }
    st(m0, n0, acc);
  }
}

struct SpDims {
  int N, K, KX, KY, W2, LA, L4, L5, SP_JG;   // SP_JG: output channels per CTA
  int CIN, G, ROWS, CHUNK;                   // input channels, CTAs per element (cluster), rows
  __host__ __device__ SpDims(int n, int k, int jg, int cin, int g)
      : N(n), K(k), KX(k + 1), KY(2 * k + 1), SP_JG(jg), CIN(cin), G(g), ROWS(cin * n), CHUNK(cin * n / g) {
    W2 = 2 * (KX + (KX & 1));            // complex columns (re, im interleaved), multiple of 4
    LA = N + 1;                          // us rows (= 1 mod 8 for N % 8 == 0)
    L4 = ((2 * KY + 7) / 8) * 8 + 1;     // E4 rows
    L5 = ((W2 + 7) / 8) * 8 + 1;         // C4 rows
  }
  // float offsets of the shared-memory regions: region X first (us for step 1, then E4 + C4)
  __host__ __device__ int x_size() const {
    const int a = CHUNK * LA, e = N * L4 + SP_JG * N * L5;
    return a > e ? a : e;
  }
  __host__ __device__ int o_E1() const { return x_size(); }
  __host__ __device__ int o_Ar() const { return o_E1() + N * W2; }
  __host__ __device__ int o_Uh() const { return o_Ar() + ROWS * W2; }
  __host__ __device__ int o_B4() const { return o_Uh() + CIN * KX * KY * 2; }
  __host__ __device__ int o_E5() const { return o_B4() + SP_JG * 2 * KY * W2; }
  __host__ __device__ int o_tw() const { return o_E5() + W2 * N; }
  __host__ __device__ int total() const { return o_tw() + 2 * N; }
};

// O_F as three small dense products (forward x, inverse y, inverse x) and one per-mode pass:
//   1. Ar[(c,y)][2kx+{re,im}] = us[(c,y)][x] . E1[x][2kx+..]          E1 = (cos, -sin)(2 pi kx x / N)
//   2. Uh[c][kx][ky]          = sum_y A[c][y][kx] e^{-2 pi i ky y / N}     (loop, ~5% of the work)
//   3. O_j(kx, ky) = M_j(k) Uh(k) on the half plane, its mirror conj on kx = 0, ky < 0, expanded
//      into the real 2 x 2 blocks of B4[2ky'+{0,1}][2kx+{re,im}]
//   4. C4[y][2kx+..] = E4[y][2ky'+..] . B4                               E4 = (cos, sin)(2 pi ky y / N)
//   5. out[y][x]     = C4[y][..] . E5[..][x]     E5 rows (w cos, w (-sin))(2 pi kx x / N), w = 2/N^2
//                                                (1/N^2 and 0 for kx = 0: the Hermitian sum)
// cin input channels ([B][cin][N][N]) -> cout outputs; out_mode 0: planar [B][cout][N][N],
// 1: cell-major [B][N(x)][N(y)][cout] (the TC-term layout the flux kernels read).
template <int SP_JG>
__global__ void __launch_bounds__(256)
spectral_kernel(const float* __restrict__ u, float* __restrict__ out, int N, int K, int cin, int cout, int out_mode,
                const float2* __restrict__ M, const float2* __restrict__ tw_g) {
  extern __shared__ __align__(16) float sp[];
  const SpDims d(N, K, SP_JG, cin, cout / SP_JG);
  const int KX = d.KX, KY = d.KY, W2 = d.W2;
  float* us = sp;
  float* E1 = sp + d.o_E1();
  float* Ar = sp + d.o_Ar();
  float2* Uh = reinterpret_cast<float2*>(sp + d.o_Uh());
  float* B4 = sp + d.o_B4();
  float* E5 = sp + d.o_E5();
  float2* tw = reinterpret_cast<float2*>(sp + d.o_tw());
  float* E4 = sp;                  // after step 1 (aliases us)
  float* C4 = sp + N * d.L4;       // [JG][N][L5]
  // the 8 / JG CTAs of an element form a cluster (grid y): each runs the forward x-DFT on its
  // share of the 2N rows, the y-DFT on its share of the modes, and the spectrum is exchanged
  // through distributed shared memory instead of being recomputed per output-channel group
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int G = d.G, rk = (int)cl.block_rank();
  const int chunk = d.CHUNK, r0 = rk * chunk;   // rows (c, y) of this CTA
  const int b = blockIdx.x, j0 = blockIdx.y * SP_JG;
  const size_t plane = (size_t)N * N;
  const int msk = N - 1;           // N is a power of two
  const float* ub = u + (size_t)b * cin * plane + (size_t)r0 * N;
  for (int i = threadIdx.x; i < chunk * N; i += blockDim.x) {
    const int r = i / N, x = i - r * N;
    us[r * d.LA + x] = __ldg(ub + i);
  }
  for (int m = threadIdx.x; m < N; m += blockDim.x) tw[m] = __ldg(tw_g + m);
  __syncthreads();
  const float inv_n2 = 1.0f / ((float)N * (float)N);
  for (int i = threadIdx.x; i < N * W2; i += blockDim.x) {   // E1 [x][2kx+..] and E5 [2kx+..][x]
    const int x = i / W2, j = i - x * W2, kx = j >> 1;
    const float2 w = kx < KX ? tw[(kx * x) & msk] : make_float2(0.f, 0.f);
    E1[i] = (j & 1) ? w.y : w.x;
    const float wt = kx == 0 ? inv_n2 : 2.f * inv_n2;
    E5[j * N + x] = (j & 1) ? (kx == 0 ? 0.f : wt * w.y) : wt * w.x;
  }
  __syncthreads();
  // 1. forward x-DFT of this CTA's rows (Ar keeps the global row index)
  sp_gemm44(us, d.LA, E1, W2, chunk, W2, N, [&](int m0, int n0, float (&acc)[4][4]) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
      *reinterpret_cast<float4*>(Ar + (r0 + m0 + r) * W2 + n0) =
          make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
  });
  cl.sync();   // every CTA's rows of Ar visible cluster-wide
  // 2. forward y-DFT, ky in [-K, K]; E4 [y][2ky'+..] = (cos, sin)(2 pi ky y / N) into the freed us region
  const int nout2 = cin * KX * KY, o_lo = rk * nout2 / G, o_hi = (rk + 1) * nout2 / G;
  for (int o = o_lo + threadIdx.x; o < o_hi; o += blockDim.x) {
    const int kyi = o % KY, kx = (o / KY) % KX, c = o / (KY * KX);
    const int ky = kyi - K;
    float re = 0.f, im = 0.f;
    for (int y = 0; y < N; ++y) {
      const int row = c * N + y;
      const float* arow = cl.map_shared_rank(Ar, row / chunk) + row * W2;
      const float2 a = *reinterpret_cast<const float2*>(arow + 2 * kx);
      const float2 w = tw[(ky * y) & msk];
      re = fmaf(a.x, w.x, fmaf(-a.y, w.y, re));
      im = fmaf(a.x, w.y, fmaf(a.y, w.x, im));
    }
    for (int g = 0; g < G; ++g) cl.map_shared_rank(Uh, g)[(c * KX + kx) * KY + kyi] = make_float2(re, im);
  }
  for (int i = threadIdx.x; i < N * d.L4; i += blockDim.x) {
    const int y = i / d.L4, j = i - y * d.L4, kyi = j >> 1;
    float v = 0.f;
    if (j < 2 * KY) {
      const float2 w = tw[((kyi - K) * y) & msk];
      v = (j & 1) ? -w.y : w.x;
    }
    E4[i] = v;
  }
  cl.sync();   // the whole spectrum Uh in every CTA; no remote access after this point
  // 3. per-mode 8 x 2 matrices (this CTA's rows), expanded into B4 (zero padding columns)
  for (int o = threadIdx.x; o < SP_JG * KY * (W2 / 2); o += blockDim.x) {
    const int kx = o % (W2 / 2), kyi = (o / (W2 / 2)) % KY, jj = o / ((W2 / 2) * KY);
    float2 r = make_float2(0.f, 0.f);
    if (kx < KX) {
      const bool mirror = kx == 0 && kyi < K;          // (0, ky < 0) = conj of (0, -ky)
      const int kys = mirror ? 2 * K - kyi : kyi;
      const int mode = kx == 0 ? kys - K : (K + 1) + (kx - 1) * KY + kys;   // ldgen/spectral.py order
      const float2* m = M + ((size_t)mode * cout + (j0 + jj)) * cin;
      for (int c = 0; c < cin; ++c) {
        const float2 mc = __ldg(m + c), uc = Uh[(c * KX + kx) * KY + kys];
        r.x = fmaf(mc.x, uc.x, fmaf(-mc.y, uc.y, r.x));
        r.y = fmaf(mc.x, uc.y, fmaf(mc.y, uc.x, r.y));
      }
      if (mirror) r.y = -r.y;
    }
    float* bb = B4 + jj * 2 * KY * W2;
    bb[(2 * kyi) * W2 + 2 * kx] = r.x;
    bb[(2 * kyi) * W2 + 2 * kx + 1] = r.y;
    bb[(2 * kyi + 1) * W2 + 2 * kx] = -r.y;
    bb[(2 * kyi + 1) * W2 + 2 * kx + 1] = r.x;
  }
  __syncthreads();
  // 4. inverse y-DFT per output channel
  for (int jj = 0; jj < SP_JG; ++jj) {
    float* c4 = C4 + jj * N * d.L5;
    sp_gemm44(E4, d.L4, B4 + jj * 2 * KY * W2, W2, N, W2, 2 * KY, [&](int m0, int n0, float (&acc)[4][4]) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) c4[(m0 + r) * d.L5 + n0 + q] = acc[r][q];
    });
  }
  __syncthreads();
  // 5. inverse x-DFT (real part, Hermitian weights folded into E5) straight to global
  for (int jj = 0; jj < SP_JG; ++jj) {
    float* ob = out + ((size_t)b * cout + j0 + jj) * plane;
    sp_gemm44(C4 + jj * N * d.L5, d.L5, E5, N, N, N, W2, [&](int m0, int n0, float (&acc)[4][4]) {
      if (out_mode == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
          *reinterpret_cast<float4*>(ob + (size_t)(m0 + r) * N + n0) =
              make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      } else {   // [b][x][y][cout]: rows m0.. are y, columns n0.. are x
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            out[(((size_t)b * N + n0 + q) * N + m0 + r) * cout + j0 + jj] = acc[r][q];
      }
    });
  }
}

// ---------------------------------------------------------------------------
// Large-N form (the operator's tables and rows exceed shared memory: N > 128 for O_F, N > 64 for the
// history TC): the same truncated transforms as three global-memory passes with small scratch.
//   s1: A[b][c][y][kx]  = sum_x u_c(y, x) e^{-2 pi i kx x / N}                     (kx in [0, K])
//   s2: per (b, kx): Uh_c(ky) = sum_y A e^{-2 pi i ky y / N}, O_j = M_j(k) Uh (mirror at kx = 0, ky < 0),
//       Bj[b][j][y][kx] = sum_ky O_j(ky) e^{+2 pi i ky y / N}
//   s3: o_j(y, x) = sum_kx w_kx Re(Bj(y, kx) e^{+2 pi i kx x / N}), w_0 = 1/N^2, w_kx>0 = 2/N^2
// Scratch (caller's workspace): A B cin N (K+1) and Bj B cout N (K+1) complex values.
// ---------------------------------------------------------------------------
__global__ void spec_big_x(const float* __restrict__ u, float2* __restrict__ A, int N, int B, int K, int cin,
                           const float2* __restrict__ tw) {
  const int KX = K + 1, msk = N - 1;
  const size_t total = (size_t)B * cin * N * KX;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const int kx = (int)(t % KX);
    const size_t row = t / KX;   // (b, c, y)
    const float* ur = u + row * N;
    float re = 0.f, im = 0.f;
    for (int x = 0; x < N; ++x) {
      const float v = __ldg(ur + x);
      const float2 w = __ldg(tw + ((kx * x) & msk));
      re = fmaf(v, w.x, re);
      im = fmaf(v, w.y, im);
    }
    A[t] = make_float2(re, im);
  }
}

__global__ void spec_big_modes(const float2* __restrict__ A, float2* __restrict__ Bj, int N, int K, int cin, int cout,
                               const float2* __restrict__ M, const float2* __restrict__ tw) {
  extern __shared__ float2 sb[];
  const int KX = K + 1, KY = 2 * K + 1, msk = N - 1;
  const int b = blockIdx.x / KX, kx = blockIdx.x % KX;
  float2* Ac = sb;                   // [cin][N]
  float2* Uh = Ac + cin * N;         // [cin][KY]
  float2* O = Uh + cin * KY;         // [cout][KY]
  for (int i = threadIdx.x; i < cin * N; i += blockDim.x) Ac[i] = A[((size_t)b * cin * N + i) * KX + kx];
  __syncthreads();
  for (int o = threadIdx.x; o < cin * KY; o += blockDim.x) {
    const int c = o / KY, ky = o % KY - K;
    float re = 0.f, im = 0.f;
    for (int y = 0; y < N; ++y) {
      const float2 a = Ac[c * N + y], w = __ldg(tw + ((ky * y) & msk));
      re = fmaf(a.x, w.x, fmaf(-a.y, w.y, re));
      im = fmaf(a.x, w.y, fmaf(a.y, w.x, im));
    }
    Uh[o] = make_float2(re, im);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < cout * KY; o += blockDim.x) {
    const int j = o / KY, kyi = o % KY;
    const bool mirror = kx == 0 && kyi < K;          // (0, ky < 0) = conj of (0, -ky)
    const int kys = mirror ? 2 * K - kyi : kyi;
    const int mode = kx == 0 ? kys - K : (K + 1) + (kx - 1) * KY + kys;
    const float2* m = M + ((size_t)mode * cout + j) * cin;
    float2 r = make_float2(0.f, 0.f);
    for (int c = 0; c < cin; ++c) {
      const float2 mc = __ldg(m + c), uc = Uh[c * KY + kys];
      r.x = fmaf(mc.x, uc.x, fmaf(-mc.y, uc.y, r.x));
      r.y = fmaf(mc.x, uc.y, fmaf(mc.y, uc.x, r.y));
    }
    if (mirror) r.y = -r.y;
    O[o] = r;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < cout * N; o += blockDim.x) {
    const int j = o / N, y = o % N;
    float re = 0.f, im = 0.f;
    for (int kyi = 0; kyi < KY; ++kyi) {
      const float2 v = O[j * KY + kyi], w = __ldg(tw + (((kyi - K) * y) & msk));   // conj(w): e^{+i}
      re = fmaf(v.x, w.x, fmaf(v.y, w.y, re));
      im = fmaf(v.y, w.x, fmaf(-v.x, w.y, im));
    }
    Bj[(((size_t)b * cout + j) * N + y) * KX + kx] = make_float2(re, im);
  }
}

__global__ void spec_big_ix(const float2* __restrict__ Bj, float* __restrict__ out, int N, int B, int K, int cout,
                            int out_mode, const float2* __restrict__ tw) {
  const int KX = K + 1, msk = N - 1;
  const float inv_n2 = 1.0f / ((float)N * (float)N);
  if (out_mode == 0) {      // planar [b][j][y][x]: x fastest
    const size_t total = (size_t)B * cout * N * N;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
      const int x = (int)(t % N);
      const float2* br = Bj + (t / N) * KX;     // row (b, j, y)
      float s = 0.f;
      for (int kx = 0; kx < KX; ++kx) {
        const float2 v = br[kx], w = __ldg(tw + ((kx * x) & msk));   // Re(v conj(w))
        s += (kx == 0 ? 1.f : 2.f) * (v.x * w.x + v.y * w.y);
      }
      out[t] = s * inv_n2;
    }
    return;
  }
  // cell-major [b][x][y][j]: one thread per cell writes its cout outputs contiguously (coalesced)
  const size_t cells = (size_t)B * N * N;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < cells; t += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)(t % N), x = (int)((t / N) % N);
    const size_t b = t / ((size_t)N * N);
    for (int j = 0; j < cout; ++j) {
      const float2* br = Bj + ((b * cout + j) * N + y) * KX;
      float s = 0.f;
      for (int kx = 0; kx < KX; ++kx) {
        const float2 v = br[kx], w = __ldg(tw + ((kx * x) & msk));
        s += (kx == 0 ? 1.f : 2.f) * (v.x * w.x + v.y * w.y);
      }
      out[t * cout + j] = s * inv_n2;
    }
  }
}

// Warp-per-row forms of s1 / s3 (KX <= 16, the twiddle table [KX][N] in shared memory): s1 keeps the
// 2 KX partial sums of a row in registers and folds them with a 31-shuffle transpose reduction (lane l
// ends with value l); s3 broadcasts a row's weighted coefficients to registers and streams x.  The
// generic kernels above read every twiddle from global (L1) per term and stay as the fallback.
LD_DEVINL void big_twiddle_table(float2* E, int N, int KX, const float2* __restrict__ tw) {
  const int msk = N - 1;
  for (int i = threadIdx.x; i < KX * N; i += blockDim.x) {
    const int kx = i / N, x = i - kx * N;
    E[i] = __ldg(tw + ((kx * x) & msk));
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) spec_big_x_w(const float* __restrict__ u, float* __restrict__ A, int N,
                                                    int rows, int KX, const float2* __restrict__ tw) {
  extern __shared__ float2 E[];   // [KX][N]
  big_twiddle_table(E, N, KX, tw);
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    const float* ur = u + (size_t)row * N;
    for (int x = lane; x < N; x += 32) {
      const float a = __ldg(ur + x);
#pragma unroll
      for (int kx = 0; kx < 16; ++kx)
        if (kx < KX) {
          const float2 w = E[kx * N + x];
          v[2 * kx] = fmaf(a, w.x, v[2 * kx]);
          v[2 * kx + 1] = fmaf(a, w.y, v[2 * kx + 1]);
        }
    }
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
      const bool up = (lane & sft) != 0;
#pragma unroll
      for (int i = 0; i < sft; ++i) {
        const float send = up ? v[i] : v[i + sft], keep = up ? v[i + sft] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
      }
    }
    if (lane < 2 * KX) A[(size_t)row * 2 * KX + lane] = v[0];
  }
}

// s3, planar output [b][j][y][x]: a warp per (b, j, y) row
__global__ void __launch_bounds__(256) spec_big_ix_w(const float2* __restrict__ Bj, float* __restrict__ out, int N,
                                                     int rows, int KX, const float2* __restrict__ tw) {
  extern __shared__ float2 E[];
  big_twiddle_table(E, N, KX, tw);
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  const float inv_n2 = 1.0f / ((float)N * (float)N);
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    float2 c = lane < KX ? Bj[(size_t)row * KX + lane] : make_float2(0.f, 0.f);
    const float wk = (lane == 0 ? 1.f : 2.f) * inv_n2;
    c.x *= wk;
    c.y *= wk;
    float cr[16], ci[16];
#pragma unroll
    for (int kx = 0; kx < 16; ++kx) {
      cr[kx] = __shfl_sync(0xffffffffu, c.x, kx);
      ci[kx] = __shfl_sync(0xffffffffu, c.y, kx);
    }
    float* orow = out + (size_t)row * N;
    for (int x = lane; x < N; x += 32) {
      float s = 0.f;
#pragma unroll
      for (int kx = 0; kx < 16; ++kx)
        if (kx < KX) {
          const float2 w = E[kx * N + x];
          s = fmaf(cr[kx], w.x, fmaf(ci[kx], w.y, s));
        }
      orow[x] = s;
    }
  }
}

// s3, cell-major output [b][x][y][2] (the history TC's e): a warp per (b, 32 rows y, 32 columns x); lane
// = y keeps its two rows' coefficients in registers, the twiddle of the common x is a broadcast, and each
// x writes 32 consecutive (e_u, e_v) pairs
__global__ void __launch_bounds__(256) spec_big_ix_t2(const float2* __restrict__ Bj, float* __restrict__ out,
                                                      int N, int B, int KX, const float2* __restrict__ tw) {
  extern __shared__ float2 E[];
  big_twiddle_table(E, N, KX, tw);
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5, nb = N / 32;
  const float inv_n2 = 1.0f / ((float)N * (float)N);
  const int units = B * nb * nb;
  for (int un = blockIdx.x * wpb + (threadIdx.x >> 5); un < units; un += gridDim.x * wpb) {
    const int xb = un % nb, yb = (un / nb) % nb, b = un / (nb * nb);
    const int y = yb * 32 + lane;
    float r0[16], i0[16], r1[16], i1[16];
#pragma unroll
    for (int kx = 0; kx < 16; ++kx) {
      float2 c0 = make_float2(0.f, 0.f), c1 = c0;
      if (kx < KX) {
        const float wk = (kx == 0 ? 1.f : 2.f) * inv_n2;
        c0 = Bj[(((size_t)b * 2 + 0) * N + y) * KX + kx];
        c1 = Bj[(((size_t)b * 2 + 1) * N + y) * KX + kx];
        c0.x *= wk; c0.y *= wk; c1.x *= wk; c1.y *= wk;
      }
      r0[kx] = c0.x; i0[kx] = c0.y; r1[kx] = c1.x; i1[kx] = c1.y;
    }
    for (int x = xb * 32; x < xb * 32 + 32; ++x) {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int kx = 0; kx < 16; ++kx)
        if (kx < KX) {
          const float2 w = E[kx * N + x];
          s0 = fmaf(r0[kx], w.x, fmaf(i0[kx], w.y, s0));
          s1 = fmaf(r1[kx], w.x, fmaf(i1[kx], w.y, s1));
        }
      *reinterpret_cast<float2*>(out + (((size_t)b * N + x) * N + y) * 2) = make_float2(s0, s1);
    }
  }
}

static bool big_fast(int N, int KX) { return KX <= 16 && N % 32 == 0 && (size_t)KX * N * sizeof(float2) <= 160 * 1024; }

size_t spectral_big_scratch_bytes(int N, int B, int K, int cin, int cout) {
  return sizeof(float2) * (size_t)B * N * (K + 1) * (cin + cout) + 256;
}

cudaError_t launch_spectral_big(const float* u, float* out, int N, int B, int K, int cin, int cout, int out_mode,
                                const float2* M, const float2* tw, void* scratch, cudaStream_t st) {
  if (!scratch) return cudaErrorInvalidValue;
  float2* A = reinterpret_cast<float2*>(scratch);
  float2* Bj = A + (size_t)B * cin * N * (K + 1);
  const int KX = K + 1;
  static const bool generic = getenv("LD_SPEC_BIG_GENERIC") != nullptr;   // measurement knob: generic s1 / s3
  const bool fast = big_fast(N, KX) && !generic;
  const size_t tsm = sizeof(float2) * (size_t)KX * N;
  if (fast) {
    static int attr_dev = -1;       // the table may exceed the 48 KB default (N >= 512)
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
      for (const void* f : {(const void*)spec_big_x_w, (const void*)spec_big_ix_w, (const void*)spec_big_ix_t2}) {
        const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        if (e != cudaSuccess) return e;
      }
      attr_dev = dev;
    }
  }
  const size_t n1 = (size_t)B * cin * N * KX;
  if (fast) {
    const int rows = B * cin * N;
    spec_big_x_w<<<(unsigned)std::min(( rows + 7) / 8, 148 * 4), 256, tsm, st>>>(u, reinterpret_cast<float*>(A), N,
                                                                                  rows, KX, tw);
  } else {
    spec_big_x<<<(unsigned)std::min<size_t>((n1 + 255) / 256, 148 * 16), 256, 0, st>>>(u, A, N, B, K, cin, tw);
  }
  const size_t smem = sizeof(float2) * ((size_t)cin * N + (size_t)(cin + cout) * (2 * K + 1));
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(spec_big_modes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  spec_big_modes<<<B * KX, 256, smem, st>>>(A, Bj, N, K, cin, cout, M, tw);
  if (fast && out_mode == 0) {
    const int rows = B * cout * N;
    spec_big_ix_w<<<(unsigned)std::min((rows + 7) / 8, 148 * 4), 256, tsm, st>>>(Bj, out, N, rows, KX, tw);
  } else if (fast && cout == 2) {
    const int units = B * (N / 32) * (N / 32);
    spec_big_ix_t2<<<(unsigned)std::min((units + 7) / 8, 148 * 4), 256, tsm, st>>>(Bj, out, N, B, KX, tw);
  } else {
    const size_t n3 = out_mode == 0 ? (size_t)B * cout * N * N : (size_t)B * N * N;
    spec_big_ix<<<(unsigned)std::min<size_t>((n3 + 255) / 256, 148 * 16), 256, 0, st>>>(Bj, out, N, B, K, cout,
                                                                                         out_mode, tw);
  }
  return cudaGetLastError();
}

// output channels per CTA (cout = 8): the CTA count B * 8 / JG near one or two per SM
// (measured at N = 64, B = 32: JG = 2 26.7 us, JG = 1 31.4, JG = 4 33.5; N = 128, B = 128: JG = 4
// 195 us, JG = 2 283); cout = 2 (history TC): one channel per CTA, two CTAs per element
static int spectral_jg(int B, int cout) {
  if (cout == 2) return 1;
  return B <= 48 ? 2 : (B <= 256 ? 4 : 8);
}
static size_t spectral_smem_jg(int N, int K, int jg, int cin, int cout) {
  return sizeof(float) * (size_t)SpDims(N, K, jg, cin, cout / jg).total();
}
size_t spectral_smem_bytes(int N, int K) { return spectral_smem_jg(N, K, 2, 2, 8); }   // O_F: the smallest form
size_t spectral_smem_bytes_io(int N, int K, int cin, int cout) {
  return spectral_smem_jg(N, K, spectral_jg(1, cout) == 1 && cout == 2 ? 1 : 2, cin, cout);
}

template <int JG>
static cudaError_t launch_spectral_jg(const float* u, float* out, int N, int B, int K, int cin, int cout, int out_mode,
                                      const float2* M, const float2* tw, cudaStream_t st) {
  const size_t smem = spectral_smem_jg(N, K, JG, cin, cout);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B, cout / JG);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;   // the channel groups of an element
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = cout / JG;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, spectral_kernel<JG>, u, out, N, K, cin, cout, out_mode, M, tw);
}

// Dynamic shared-memory limit (the 227 KB opt-in maximum) of every spectral_kernel instance on the
// CURRENT device (function attributes are per device): called by ld_init / ld_spectral_create.
cudaError_t spectral_set_smem_limits() {
  const int mx = 227 * 1024;
  cudaError_t e = cudaFuncSetAttribute(spectral_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(spectral_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(spectral_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(spectral_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  return e;
}

cudaError_t launch_spectral_io(const float* u, float* out, int N, int B, int K, int cin, int cout, int out_mode,
                               const float2* M, const float2* tw, cudaStream_t st) {
  int jg = spectral_jg(B, cout);
  while (jg > 2 && spectral_smem_jg(N, K, jg, cin, cout) > 227 * 1024) jg /= 2;
  if (jg == 1) return launch_spectral_jg<1>(u, out, N, B, K, cin, cout, out_mode, M, tw, st);
  if (jg == 2) return launch_spectral_jg<2>(u, out, N, B, K, cin, cout, out_mode, M, tw, st);
  if (jg == 4) return launch_spectral_jg<4>(u, out, N, B, K, cin, cout, out_mode, M, tw, st);
  return launch_spectral_jg<8>(u, out, N, B, K, cin, cout, out_mode, M, tw, st);
}

cudaError_t launch_spectral(const float* u, float* out, int N, int B, int K, const float2* M, const float2* tw,
                            cudaStream_t st) {
  return launch_spectral_io(u, out, N, B, K, 2, 8, 0, M, tw, st);
}

}  // namespace ld
