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
#include "common.cuh"

namespace ld {

constexpr int SP_JG = 2;   // output channels per CTA

__global__ void __launch_bounds__(256)
spectral_kernel(const float* __restrict__ u, float* __restrict__ out, int N, int K,
                const float2* __restrict__ M, const float2* __restrict__ tw_g) {
  extern __shared__ __align__(16) float sp[];
  const int KX = K + 1, KY = 2 * K + 1;
  float* us = sp;                                          // [2][N][N]
  float2* tw = reinterpret_cast<float2*>(us + 2 * N * N);  // [N]  e^{-2 pi i m / N}
  float2* A = tw + N;                                      // [2][N][KX]
  float2* Uh = A + 2 * N * KX;                             // [2][KX][KY]
  float2* Oh = Uh + 2 * KX * KY;                           // [JG][KX][KY]
  float2* Bj = Oh + SP_JG * KX * KY;                       // [JG][N][KX]
  const int b = blockIdx.x, j0 = blockIdx.y * SP_JG;
  const size_t plane = (size_t)N * N;
  const float* ub = u + (size_t)b * 2 * plane;
  for (int i = threadIdx.x; i < 2 * N * N / 4; i += blockDim.x)
    reinterpret_cast<float4*>(us)[i] = __ldg(reinterpret_cast<const float4*>(ub) + i);
  for (int m = threadIdx.x; m < N; m += blockDim.x) tw[m] = __ldg(tw_g + m);
  __syncthreads();
  const int msk = N - 1;   // N is a power of two
  // 1. x-DFT of both components, kx in [0, K]
  for (int o = threadIdx.x; o < 2 * N * KX; o += blockDim.x) {
    const int kx = o % KX, y = (o / KX) % N, c = o / (KX * N);
    const float* row = us + (c * N + y) * N;
    float re = 0.f, im = 0.f;
    for (int x = 0; x < N; ++x) {
      const float2 w = tw[(kx * x) & msk];
      re = fmaf(row[x], w.x, re);
      im = fmaf(row[x], w.y, im);
    }
    A[(c * N + y) * KX + kx] = make_float2(re, im);
  }
  __syncthreads();
  // 2. y-DFT, ky in [-K, K]
  for (int o = threadIdx.x; o < 2 * KX * KY; o += blockDim.x) {
    const int kyi = o % KY, kx = (o / KY) % KX, c = o / (KY * KX);
    const int ky = kyi - K;
    float re = 0.f, im = 0.f;
    for (int y = 0; y < N; ++y) {
      const float2 a = A[(c * N + y) * KX + kx], w = tw[(ky * y) & msk];
      re = fmaf(a.x, w.x, fmaf(-a.y, w.y, re));
      im = fmaf(a.x, w.y, fmaf(a.y, w.x, im));
    }
    Uh[(c * KX + kx) * KY + kyi] = make_float2(re, im);
  }
  __syncthreads();
  // 3. per-mode 8 x 2 complex matrix (this CTA's JG rows), half plane: kx = 0 keeps ky >= 0
  for (int o = threadIdx.x; o < SP_JG * KX * KY; o += blockDim.x) {
    const int kyi = o % KY, kx = (o / KY) % KX, jj = o / (KY * KX);
    float2 r = make_float2(0.f, 0.f);
    if (kx > 0 || kyi >= K) {
      const int mode = kx == 0 ? kyi - K : (K + 1) + (kx - 1) * KY + kyi;   // storage order (ldgen/spectral.py)
      const float2* m = M + ((size_t)mode * 8 + (j0 + jj)) * 2;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float2 mc = __ldg(m + c), uc = Uh[(c * KX + kx) * KY + kyi];
        r.x = fmaf(mc.x, uc.x, fmaf(-mc.y, uc.y, r.x));
        r.y = fmaf(mc.x, uc.y, fmaf(mc.y, uc.x, r.y));
      }
    }
    Oh[(jj * KX + kx) * KY + kyi] = r;
  }
  __syncthreads();
  // 4. inverse y-DFT (e^{+i}): B_j(y, kx)
  for (int o = threadIdx.x; o < SP_JG * N * KX; o += blockDim.x) {
    const int kx = o % KX, y = (o / KX) % N, jj = o / (KX * N);
    const float2* oh = Oh + (jj * KX + kx) * KY;
    float re = 0.f, im = 0.f;
    if (kx > 0) {
      for (int kyi = 0; kyi < KY; ++kyi) {
        const float2 a = oh[kyi], w = tw[((kyi - K) * y) & msk];   // e^{+i t} = (w.x, -w.y)
        re = fmaf(a.x, w.x, fmaf(a.y, w.y, re));
        im = fmaf(a.y, w.x, fmaf(-a.x, w.y, im));
      }
    } else {
      for (int kyi = K + 1; kyi < KY; ++kyi) {   // 2 Re sum_{ky > 0}
        const float2 a = oh[kyi], w = tw[((kyi - K) * y) & msk];
        re = fmaf(a.x, w.x, fmaf(a.y, w.y, re));
      }
      re = fmaf(2.f, re, oh[K].x);
    }
    Bj[(jj * N + y) * KX + kx] = make_float2(re, im);
  }
  __syncthreads();
  // 5. inverse x-DFT, real part: o_j(y, x)
  const float inv_n2 = 1.0f / ((float)N * (float)N);
  for (int o = threadIdx.x; o < SP_JG * N * N; o += blockDim.x) {
    const int x = o % N, y = (o / N) % N, jj = o / (N * N);
    const float2* bj = Bj + (jj * N + y) * KX;
    float s = 0.f;
    for (int kx = 1; kx < KX; ++kx) {
      const float2 a = bj[kx], w = tw[(kx * x) & msk];
      s = fmaf(a.x, w.x, fmaf(a.y, w.y, s));
    }
    out[((size_t)b * 8 + j0 + jj) * plane + (size_t)y * N + x] = fmaf(2.f, s, bj[0].x) * inv_n2;
  }
}

size_t spectral_smem_bytes(int N, int K) {
  const size_t KX = K + 1, KY = 2 * K + 1;
  return sizeof(float) * 2 * (size_t)N * N +
         sizeof(float2) * ((size_t)N + 2 * N * KX + 2 * KX * KY + SP_JG * KX * KY + SP_JG * N * KX);
}

cudaError_t launch_spectral(const float* u, float* out, int N, int B, int K, const float2* M, const float2* tw,
                            cudaStream_t st) {
  const size_t smem = spectral_smem_bytes(N, K);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(spectral_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  spectral_kernel<<<dim3(B, 8 / SP_JG), 256, smem, st>>>(u, out, N, K, M, tw);
  return cudaGetLastError();
}

}  // namespace ld
