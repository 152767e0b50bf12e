// fft256.cuh -- 256-point complex FFT on a half-warp (16 lanes x 16 registers), natural order in and out,
// for the N = 256 projection passes (pencil.cu *_n256; PAPER.md P:315 spectral solve, c4).
//
// Four-step with N = 16 x 16:  n = n2 + 16 n1, k = k1 + 16 k2,
//   X[k1 + 16 k2] = sum_n2 W16^{n2 k2} W256^{n2 k1} sum_n1 x[n2 + 16 n1] W16^{n1 k1}.
// Lane h of the half-warp holds x[h + 16 j] in register j.  Forward: (1) an in-register 16-point DFT over
// n1 (lane h = n2), (2) the twiddle W256^{h k1}, (3) a transpose through shared memory S[k1][n2]
// (XOR-swizzled: conflict-free both ways), (4) an in-register 16-point DFT over n2 (lane h = k1); lane h then
// holds X[h + 16 k2] in register k2 -- natural order again.  The inverse runs the same steps with
// conjugate twiddles on that layout and returns x[h + 16 j].  Unnormalised (the caller scales).
// Compared with the 32-lane shuffle FFT (warpfft.cuh: 5 shuffle stages of 8 values per lane) the data
// crosses lanes once through shared memory: about a third of the instructions per point.
#pragma once
#include "common.cuh"

namespace ld {

// 4-point DFT in place (natural order); INV: W4 = +i instead of -i
template <bool INV>
LD_DEVINL void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  const float2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = csub(a1, a3);
  // -i d13 = (d13.y, -d13.x);  +i d13 = (-d13.y, d13.x)
  const float2 r = INV ? make_float2(-d13.y, d13.x) : make_float2(d13.y, -d13.x);
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, r);
  a3 = csub(d02, r);
}

// W16^m for m in [0, 16) (compile-time constants; INV: conjugate)
template <bool INV>
LD_DEVINL float2 w16(int m) {
  constexpr float C1 = 0.92387953251128674f, S1 = 0.38268343236508977f, C2 = 0.70710678118654752f;
  float c, s;   // W16^m = cos(2 pi m / 16) - i sin(2 pi m / 16)
  switch (m & 15) {
    case 0: c = 1.f; s = 0.f; break;
    case 1: c = C1; s = S1; break;
    case 2: c = C2; s = C2; break;
    case 3: c = S1; s = C1; break;
    case 4: c = 0.f; s = 1.f; break;
    case 5: c = -S1; s = C1; break;
    case 6: c = -C2; s = C2; break;
    case 7: c = -C1; s = S1; break;
    case 8: c = -1.f; s = 0.f; break;
    case 9: c = -C1; s = -S1; break;
    case 10: c = -C2; s = -C2; break;
    case 11: c = -S1; s = -C1; break;
    case 12: c = 0.f; s = -1.f; break;
    case 13: c = S1; s = -C1; break;
    case 14: c = C2; s = -C2; break;
    default: c = C1; s = -S1; break;
  }
  return make_float2(c, INV ? s : -s);
}

// 16-point DFT over the registers, natural order in and out: n = 4a + b, k = c + 4d,
// X[c + 4d] = sum_b W4^{bd} (W16^{bc} sum_a x[4a + b] W4^{ac})
template <bool INV>
LD_DEVINL void dft16(float2 (&x)[16]) {
#pragma unroll
  for (int b = 0; b < 4; ++b) dft4<INV>(x[b], x[4 + b], x[8 + b], x[12 + b]);   // x[4c + b] = U_b[c]
#pragma unroll
  for (int b = 1; b < 4; ++b)
#pragma unroll
    for (int c = 1; c < 4; ++c) x[4 * c + b] = cmul(x[4 * c + b], w16<INV>(b * c));
  float2 y[16];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float2 a0 = x[4 * c], a1 = x[4 * c + 1], a2 = x[4 * c + 2], a3 = x[4 * c + 3];
    dft4<INV>(a0, a1, a2, a3);   // over b -> d
    y[c] = a0; y[c + 4] = a1; y[c + 8] = a2; y[c + 12] = a3;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = y[i];
}

// tw16[k1 * 16 + h] = W256^{h k1} (forward); a 16 x 16 table built from tw_g (W256^m, m < 128)
LD_DEVINL void load_tw16x16(float2* tw16, const float2* __restrict__ tw_g, int tid, int nt) {
  for (int i = tid; i < 256; i += nt) {
    const int m = (i >> 4) * (i & 15);   // k1 * h < 225
    const float2 w = tw_g[m & 127];
    tw16[i] = (m & 128) ? make_float2(-w.x, -w.y) : w;
  }
}

// The half-warp FFT.  S: this half-warp's 256-float2 scratch, element (row r, column c) at r * 16 + (c ^ r)
// (XOR swizzle: conflict-free for the row-wise writes and the column-wise reads).  h = lane & 15.
template <bool INV>
LD_DEVINL void fft256_hw(float2 (&v)[16], float2* S, const float2* tw16, int h) {
  dft16<INV>(v);   // forward: over n1 (lane = n2); inverse: over k2 (lane = k1)
#pragma unroll
  for (int k = 1; k < 16; ++k) {
    const float2 w = tw16[k * 16 + h];   // W256^{h k}
    v[k] = cmul(v[k], INV ? conjf2(w) : w);
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) S[k * 16 + (h ^ k)] = v[k];   // (row k, column h)
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = S[h * 16 + (k ^ h)];   // (row h, column k)
  __syncwarp();
  dft16<INV>(v);   // forward: over n2 (lane = k1) -> X[h + 16 k2]; inverse: over k1 -> x[h + 16 n1]
}

}  // namespace ld
