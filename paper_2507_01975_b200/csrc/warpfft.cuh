// warpfft.cuh -- register-resident warp FFT shared by the projection kernels (fft.cu, pencil.cu).
#pragma once
#include "common.cuh"

namespace ld {

// ---------------------------------------------------------------------------
// Register-resident warp FFT (four-step, N = 32 E points, E = N/32 complex values per lane).
// Lane l holds x[l + 32 e], e = 0..E-1 (natural order).  Forward:
//   1. E-point DFT over the lane's registers, 2. twiddle W_N^{l k1},
//   3. 32-point DFT across lanes by 5 radix-2 DIF shuffle stages (xor partners 16 .. 1);
// afterwards lane l, register k1 holds X[k1 + E * bitrev5(l)] (scrambled).  The inverse runs the
// transposed steps in reverse order (DIT shuffle stages 1 .. 16 with conjugate twiddles, conj
// twiddle, inverse E-point DFT), so it takes the scrambled spectrum and returns natural order:
// no data movement between a forward and an inverse.  Unnormalised (the caller scales by
// 1/N per transform pair).  tw[m] = W_N^m = e^{-2 pi i m / N}, m in [0, N), in shared memory.
// ---------------------------------------------------------------------------
template <int E, bool INV>
LD_DEVINL void reg_dft(float2 (&v)[E], const float2* tw, int N) {
  // radix-2 DIT over the E registers (natural in, natural out), twiddles W_E^j = W_N^{32 j}
  if constexpr (E == 1) {
    return;
  } else {
    float2 a[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {   // bit-reverse permutation (compile time)
      int r = 0;
#pragma unroll
      for (int b = 1, t = i; b < E; b <<= 1, t >>= 1) r = (r << 1) | (t & 1);
      a[r] = v[i];
    }
#pragma unroll
    for (int m = 1; m < E; m <<= 1) {
#pragma unroll
      for (int g = 0; g < E; g += 2 * m) {
#pragma unroll
        for (int j = 0; j < m; ++j) {
          float2 w = tw[(32 * j * (E / (2 * m))) & (N - 1)];
          if (INV) w.y = -w.y;
          const float2 t = cmul(w, a[g + j + m]);
          a[g + j + m] = csub(a[g + j], t);
          a[g + j] = cadd(a[g + j], t);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = a[i];
  }
}

template <int E>
LD_DEVINL void warp_fft_fwd(float2 (&v)[E], const float2* tw) {
  constexpr int N = 32 * E;
  const int lane = threadIdx.x & 31;
  reg_dft<E, false>(v, tw, N);
#pragma unroll
  for (int k = 1; k < E; ++k) v[k] = cmul(v[k], tw[(lane * k) & (N - 1)]);
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = lane & s;
    const float2 w = tw[(lane & (s - 1)) * (N / (2 * s))];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, v[k].x, s), __shfl_xor_sync(0xffffffffu, v[k].y, s));
      v[k] = up ? cmul(csub(o, v[k]), w) : cadd(v[k], o);
    }
  }
}

template <int E>
LD_DEVINL void warp_fft_inv(float2 (&v)[E], const float2* tw) {
  constexpr int N = 32 * E;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 1; s <= 16; s <<= 1) {
    const bool up = lane & s;
    const float2 w = conjf2(tw[(lane & (s - 1)) * (N / (2 * s))]);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, v[k].x, s), __shfl_xor_sync(0xffffffffu, v[k].y, s));
      v[k] = up ? csub(o, cmul(v[k], w)) : cadd(v[k], cmul(o, w));
    }
  }
#pragma unroll
  for (int k = 1; k < E; ++k) v[k] = cmul(v[k], conjf2(tw[(lane * k) & (N - 1)]));
  reg_dft<E, true>(v, tw, N);
}

LD_DEVINL int bitrev5(int l) { return (int)(__brev((unsigned)l) >> 27); }

}  // namespace ld
