// pencil.cu -- FFT pressure projection for large grids (N >= 256) and for the slab
// decomposition: rows -> (all-to-all) -> columns -> (all-to-all)
// -> rows, each pass a register-resident warp FFT (fft.cu: warp_fft_fwd / warp_fft_inv).
//
//   d = D_c U*;  d_hat = DFT2(d);  p_hat = -d_hat / (kx_hat^2 + ky_hat^2) (0 on the four null
//   modes);  p = IDFT2(p_hat);  U = U* - G_c p       (Eq.13-15; R10, R23)
//
// Spectrum layout.  A row transform leaves lane l, register k1 holding X[k1 + E bitrev5(l)];
// it is stored as it stands at position pos = l E + k1 (one contiguous E-run per lane, i.e.
// coalesced), so "positions" are a fixed permutation of kx:  kx(pos) = pos % E + E bitrev5(pos / E).
// The inverse row transform reads the same permuted order, so nothing is ever un-permuted; the
// column pass only needs kx(pos) for the multiplier.
//
// Work distribution over P slab ranks (P = 1: single domain).  Rank r owns rows
// [r n, (r+1) n), n = N / P.  After the row pass its spectrum rows are stored as P blocks
//   send[s][b][y_local][c],  c in [0, m), m = N / P   (block s = positions [s m, (s+1) m))
// which is exactly an all-to-all send buffer: after the exchange rank s holds
//   recv[r][b][y_local][c] = all N rows (y = r n + y_local) of its m positions,
// the column pass transforms those in place, the reverse all-to-all returns them, and the
// inverse row pass reads rank r's rows back from the P blocks.  With P = 1 both buffers are
// the same [1][B][N][N] array and no exchange happens.
#include <cstdlib>

#include "common.cuh"
#include "warpfft.cuh"
#include "fft256.cuh"

namespace ld {


LD_DEVINL int pos_to_k(int pos, int E) { return pos % E + E * (int)(__brev((unsigned)(pos / E)) >> 27); }

// ---- pass 1: d = D_c U* on the own rows, forward FFT along x, stored as P position blocks
template <int E>
__global__ void __launch_bounds__(256)
pen_rows_fwd(PencilArgs A, float2* __restrict__ send, const float2* __restrict__ tw_g) {
  constexpr int N = 32 * E;
  __shared__ float2 tw[N];
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    const float2 w = tw_g[m & (N / 2 - 1)];
    tw[m] = (m & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();
  const int n = N / A.P, m = N / A.P;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // (b, y) of the own rows
  if (row >= A.B * n) return;
  const int b = row / n, y = row - b * n;
  const float* u = A.U + ((size_t)(b * 2 + 0) * A.rows + A.row0) * N;
  const float* v = A.U + ((size_t)(b * 2 + 1) * A.rows + A.row0) * N;
  const float* vdn = y > 0 ? v + (size_t)(y - 1) * N : A.vbelow + (size_t)b * A.vstride;
  const float* vup = y + 1 < n ? v + (size_t)(y + 1) * N : A.vabove + (size_t)b * A.vstride;
  float2 z[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int x = lane + 32 * e;
    const float d = (__ldg(u + (size_t)y * N + ((x + 1) & (N - 1))) - __ldg(u + (size_t)y * N + ((x - 1) & (N - 1))) +
                     __ldg(vup + x) - __ldg(vdn + x)) * A.half_inv_h;
    z[e] = make_float2(d, 0.f);
  }
  warp_fft_fwd<E>(z, tw);
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int pos = lane * E + k, s = pos / m, c = pos - s * m;
    send[(((size_t)s * A.B + b) * n + y) * m + c] = z[k];
  }
}

// ---- pass 2: for CC consecutive own positions of element b: FFT along y (all N rows, read
// from the P row blocks), * -scale / (kx^2 + ky^2), inverse FFT along y, in place
template <int E, int CC>
__global__ void __launch_bounds__(256)
pen_cols(PencilArgs A, float2* __restrict__ buf, const float2* __restrict__ tw_g, const float* __restrict__ ks_g) {
  constexpr int N = 32 * E, NP = N + 1;
  extern __shared__ float2 sm2[];
  float2* T = sm2;                   // [CC][NP] columns
  float2* tw = T + CC * NP;          // [N]
  float* ks = reinterpret_cast<float*>(tw + N);
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float2 w = tw_g[i & (N / 2 - 1)];
    tw[i] = (i & (N / 2)) ? make_float2(-w.x, -w.y) : w;
    ks[i] = ks_g[i];
  }
  const int n = N / A.P, m = N / A.P;
  const int nblk = m / CC;
  const int b = blockIdx.x / nblk, c0 = (blockIdx.x - b * nblk) * CC;
  // coalesced load: for every y, CC consecutive complex of block (y / n)
  for (int i = threadIdx.x; i < N * CC; i += blockDim.x) {
    const int y = i / CC, c = i - y * CC;
    const int r = y / n, yl = y - r * n;
    T[c * NP + y] = buf[(((size_t)r * A.B + b) * n + yl) * m + c0 + c];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < CC; c += nw) {
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = T[c * NP + lane + 32 * e];
    warp_fft_fwd<E>(v, tw);
    const int kx = pos_to_k(A.rank * m + c0 + c, E);
    const bool xnull = kx == 0 || kx == N / 2;
    const int kb = E * (int)(__brev((unsigned)lane) >> 27);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int ky = kb + k;
      const bool nul = xnull && (ky == 0 || ky == N / 2);
      const float f = nul ? 0.f : -A.scale / (ks[kx] + ks[ky]);
      v[k] = make_float2(v[k].x * f, v[k].y * f);
    }
    warp_fft_inv<E>(v, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) T[c * NP + lane + 32 * e] = v[e];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < N * CC; i += blockDim.x) {
    const int y = i / CC, c = i - y * CC;
    const int r = y / n, yl = y - r * n;
    buf[(((size_t)r * A.B + b) * n + yl) * m + c0 + c] = T[c * NP + y];
  }
}

// ---- pass 3: inverse FFT along x of the own rows (positions gathered from the P blocks) -> p
template <int E>
__global__ void __launch_bounds__(256)
pen_rows_inv(PencilArgs A, const float2* __restrict__ recv, float* __restrict__ p, const float2* __restrict__ tw_g) {
  constexpr int N = 32 * E;
  __shared__ float2 tw[N];
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float2 w = tw_g[i & (N / 2 - 1)];
    tw[i] = (i & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();
  const int n = N / A.P, m = N / A.P;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= A.B * n) return;
  const int b = row / n, y = row - b * n;
  float2 z[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int pos = lane * E + k, s = pos / m, c = pos - s * m;
    z[k] = recv[(((size_t)s * A.B + b) * n + y) * m + c];
  }
  warp_fft_inv<E>(z, tw);
#pragma unroll
  for (int e = 0; e < E; ++e) p[((size_t)b * n + y) * N + lane + 32 * e] = z[e].x;
}

// ---------------------------------------------------------------------------
// Real-data form of the single-domain projection (P = 1, N = 256 .. 1024; PAPER.md P:315 spectral
// solve, BASELINE north_star "batched real FFT"): two real rows per complex transform.
//   r2 rows:  z_m(x) = d_{2m}(x) + i d_{2m+1}(x)  ->  Z_m(kx)  (N/2 transforms per element, not N)
//   r2 cols:  for each pair {kx, -kx} (N/2 + 1 pairs): D_{2m}(kx) = (Z_m(kx) + conj Z_m(-kx)) / 2,
//             D_{2m+1}(kx) = (Z_m(kx) - conj Z_m(-kx)) / 2i; one column FFT along y, the Poisson
//             divide, the inverse; P_y(-kx) = conj P_y(kx) (p real) repacks
//             Z'_m(+-kx) = P_{2m}(+-kx) + i P_{2m+1}(+-kx)            (N/2 + 1 column FFTs, not N)
//   r2 inv:   inverse row FFT of Z'_m -> p_{2m} + i p_{2m+1}
// Spectrum rows [B][N/2][N positions] (half the bytes of the complex form).
// ---------------------------------------------------------------------------
LD_DEVINL int k_to_pos(int k, int E) { return E * (int)(__brev((unsigned)(k / E)) >> 27) + k % E; }

template <int E>
__global__ void __launch_bounds__(128, E <= 8 ? 16 : (E == 16 ? 8 : 2))
pen_rows_fwd_r2(PencilArgs A, float2* __restrict__ spec, const float2* __restrict__ tw_g) {
  constexpr int N = 32 * E;
  __shared__ float2 tw[N];
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    const float2 w = tw_g[m & (N / 2 - 1)];
    tw[m] = (m & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // (b, row pair mm)
  if (row >= A.B * (N / 2)) return;
  const int b = row / (N / 2), mm = row - b * (N / 2);
  const float* u = A.U + (size_t)(b * 2 + 0) * N * N;
  const float* v = A.U + (size_t)(b * 2 + 1) * N * N;
  float2 z[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int x = lane + 32 * e, xp = (x + 1) & (N - 1), xm = (x - 1) & (N - 1);
    float d[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int y = 2 * mm + h, yp = (y + 1) & (N - 1), ym = (y - 1) & (N - 1);
      d[h] = (__ldg(u + (size_t)y * N + xp) - __ldg(u + (size_t)y * N + xm) + __ldg(v + (size_t)yp * N + x) -
              __ldg(v + (size_t)ym * N + x)) * A.half_inv_h;
    }
    z[e] = make_float2(d[0], d[1]);
  }
  warp_fft_fwd<E>(z, tw);
  float4* dst = reinterpret_cast<float4*>(spec + ((size_t)b * (N / 2) + mm) * N + lane * E);   // 16-B stores
#pragma unroll
  for (int k = 0; k < E; k += 2) dst[k / 2] = make_float4(z[k].x, z[k].y, z[k + 1].x, z[k + 1].y);
}

template <int E, int CC>
__global__ void __launch_bounds__(128)
pen_cols_r2(PencilArgs A, float2* __restrict__ spec, const float2* __restrict__ tw_g, const float* __restrict__ ks_g) {
  constexpr int N = 32 * E, H = N / 2, NPAIR = N / 2 + 1;
  extern __shared__ float2 sm2[];
  float2* T1 = sm2;                  // [CC][H] Z_m(kx)
  float2* T2 = T1 + CC * H;          // [CC][H] Z_m(-kx)
  float2* tw = T2 + CC * H;          // [N]
  float* ks = reinterpret_cast<float*>(tw + N);
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float2 w = tw_g[i & (N / 2 - 1)];
    tw[i] = (i & (N / 2)) ? make_float2(-w.x, -w.y) : w;
    ks[i] = ks_g[i];
  }
  const int nblk = (NPAIR + CC - 1) / CC;
  const int b = blockIdx.x / nblk, q0 = (blockIdx.x - b * nblk) * CC;
  const float2* sb = spec + (size_t)b * H * N;
  for (int i = threadIdx.x; i < CC * H; i += blockDim.x) {
    const int c = i / H, m = i - c * H, kx = q0 + c;
    if (kx < NPAIR) {
      T1[c * H + m] = sb[(size_t)m * N + k_to_pos(kx, E)];
      T2[c * H + m] = sb[(size_t)m * N + k_to_pos((N - kx) & (N - 1), E)];
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < CC; c += nw) {
    const int kx = q0 + c;
    if (kx >= NPAIR) break;
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {   // D_y(kx), y = lane + 32 e
      const int y = lane + 32 * e, m = y >> 1;
      const float2 a = T1[c * H + m], bb = conjf2(T2[c * H + m]);
      v[e] = (y & 1) ? make_float2(0.5f * (a.y - bb.y), -0.5f * (a.x - bb.x)) : make_float2(0.5f * (a.x + bb.x), 0.5f * (a.y + bb.y));
    }
    warp_fft_fwd<E>(v, tw);
    const bool xnull = kx == 0 || kx == N / 2;
    const int kb = E * bitrev5(lane);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int ky = kb + k;
      const bool nul = xnull && (ky == 0 || ky == N / 2);
      const float f = nul ? 0.f : -A.scale / (ks[kx] + ks[ky]);
      v[k] = make_float2(v[k].x * f, v[k].y * f);
    }
    warp_fft_inv<E>(v, tw);
    // repack: even lanes hold P_{2m}, lane + 1 holds P_{2m+1} (y = lane + 32 e, m = y / 2)
    const int p1 = k_to_pos(kx, E), p2 = k_to_pos((N - kx) & (N - 1), E);
    float2* db = spec + (size_t)b * H * N;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float2 o = make_float2(__shfl_down_sync(0xffffffffu, v[e].x, 1), __shfl_down_sync(0xffffffffu, v[e].y, 1));
      if (!(lane & 1)) {
        const int m = (lane + 32 * e) >> 1;
        if (xnull) {   // self-paired column: P real up to rounding
          db[(size_t)m * N + p1] = make_float2(v[e].x, o.x);
        } else {
          db[(size_t)m * N + p1] = make_float2(v[e].x - o.y, v[e].y + o.x);
          db[(size_t)m * N + p2] = make_float2(v[e].x + o.y, o.x - v[e].y);
        }
      }
    }
  }
}

// pen_cols_r2 with coalesced memory passes: the CTA's CC columns are loaded row-major (for every row
// pair m the CC consecutive positions of kx and of -kx: 64-B runs) and the repacked results are
// staged back in shared memory and written the same way, instead of one 8-B store per row and lane
// pair.  NW warps, one column at a time per warp.  The same fp32 arithmetic as pen_cols_r2.
template <int E, int CC>
constexpr size_t cols_r2s_smem() { return sizeof(float2) * ((size_t)2 * (CC + 1) * 16 * E + 32 * E) + sizeof(float) * 32 * E; }
template <int E, int CC, int NW>
__global__ void __launch_bounds__(32 * NW, E <= 8 ? 8 : 4)
pen_cols_r2s(PencilArgs A, float2* __restrict__ spec, const float2* __restrict__ tw_g, const float* __restrict__ ks_g) {
  constexpr int N = 32 * E, H = N / 2, NPAIR = N / 2 + 1, NT = 32 * NW, PC = CC + 1;   // PC: padded pitch
  extern __shared__ float2 sm2[];
  float2* T1 = sm2;                  // [H][PC] Z_m(kx), then P-packed values at position(kx)
  float2* T2 = T1 + PC * H;          // [H][PC] Z_m(-kx), then at position(-kx)
  float2* tw = T2 + PC * H;          // [N]
  float* ks = reinterpret_cast<float*>(tw + N);
  for (int i = threadIdx.x; i < N; i += NT) {
    const float2 w = tw_g[i & (N / 2 - 1)];
    tw[i] = (i & (N / 2)) ? make_float2(-w.x, -w.y) : w;
    ks[i] = ks_g[i];
  }
  const int nblk = (NPAIR + CC - 1) / CC;
  const int b = blockIdx.x / nblk, q0 = (blockIdx.x - b * nblk) * CC;
  float2* sb = spec + (size_t)b * H * N;
  for (int i = threadIdx.x; i < CC * H; i += NT) {
    const int m = i / CC, c = i - m * CC, kx = q0 + c;
    if (kx < NPAIR) {
      T1[m * PC + c] = sb[(size_t)m * N + k_to_pos(kx, E)];
      T2[m * PC + c] = sb[(size_t)m * N + k_to_pos((N - kx) & (N - 1), E)];
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < CC; c += NW) {
    const int kx = q0 + c;
    if (kx >= NPAIR) break;
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {   // D_y(kx), y = lane + 32 e
      const int y = lane + 32 * e, m = y >> 1;
      const float2 a = T1[m * PC + c], bb = conjf2(T2[m * PC + c]);
      v[e] = (y & 1) ? make_float2(0.5f * (a.y - bb.y), -0.5f * (a.x - bb.x)) : make_float2(0.5f * (a.x + bb.x), 0.5f * (a.y + bb.y));
    }
    __syncwarp();   // every lane has read column c before it is overwritten below
    warp_fft_fwd<E>(v, tw);
    const bool xnull = kx == 0 || kx == N / 2;
    const int kb = E * bitrev5(lane);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int ky = kb + k;
      const bool nul = xnull && (ky == 0 || ky == N / 2);
      const float f = nul ? 0.f : -A.scale / (ks[kx] + ks[ky]);
      v[k] = make_float2(v[k].x * f, v[k].y * f);
    }
    warp_fft_inv<E>(v, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float2 o = make_float2(__shfl_down_sync(0xffffffffu, v[e].x, 1), __shfl_down_sync(0xffffffffu, v[e].y, 1));
      if (!(lane & 1)) {
        const int m = (lane + 32 * e) >> 1;
        if (xnull) {   // self-paired column: P real up to rounding
          T1[m * PC + c] = make_float2(v[e].x, o.x);
        } else {
          T1[m * PC + c] = make_float2(v[e].x - o.y, v[e].y + o.x);
          T2[m * PC + c] = make_float2(v[e].x + o.y, o.x - v[e].y);
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < CC * H; i += NT) {
    const int m = i / CC, c = i - m * CC, kx = q0 + c;
    if (kx < NPAIR) {
      sb[(size_t)m * N + k_to_pos(kx, E)] = T1[m * PC + c];
      if (kx != 0 && kx != N / 2) sb[(size_t)m * N + k_to_pos(N - kx, E)] = T2[m * PC + c];
    }
  }
}

template <int E>
__global__ void __launch_bounds__(256)
pen_rows_inv_r2(PencilArgs A, const float2* __restrict__ spec, float* __restrict__ p, const float2* __restrict__ tw_g) {
  constexpr int N = 32 * E;
  __shared__ float2 tw[N];
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float2 w = tw_g[i & (N / 2 - 1)];
    tw[i] = (i & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= A.B * (N / 2)) return;
  const int b = row / (N / 2), mm = row - b * (N / 2);
  float2 z[E];
#pragma unroll
  for (int k = 0; k < E; ++k) z[k] = spec[((size_t)b * (N / 2) + mm) * N + lane * E + k];
  warp_fft_inv<E>(z, tw);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    p[((size_t)b * N + 2 * mm) * N + lane + 32 * e] = z[e].x;
    p[((size_t)b * N + 2 * mm + 1) * N + lane + 32 * e] = z[e].y;
  }
}

// ---- r2 pass 3 fused with the correction (P = 1): the CTA owns rows y0 .. y0 + 2R - 1 (R row pairs);
// R + 1 warps inverse-transform the pairs mm0 - 1 .. mm0 + R (one halo pair on each side: the
// centred y-difference needs p rows y0 - 1 and y0 + 2R) into shared memory, then every thread applies
// U = U* - G_c p to float4 runs of the own rows.  p never reaches global memory: per cell the pass
// reads the half spectrum 4 B (x (R + 2) / R) and U* 8 B and writes U 8 B, instead of the inverse
// pass's 4 + 4 and the correction's 4 + 8 + 8.  The same fp32 operations as pen_rows_inv_r2 +
// pen_correct (explicitly rounded, no contraction), so the result is bitwise the two-pass one.
constexpr int R2_CORR_R = 8;
template <int E, int R>
constexpr size_t inv_corr_smem() {   // twiddles, p rows, the first correction iteration's U* (2 float4 per thread)
  return sizeof(float2) * 32 * E + sizeof(float) * 2 * (R + 2) * 32 * E + sizeof(float4) * 2 * 32 * (R + 1);
}

template <int E, int R>
__global__ void __launch_bounds__(32 * (R + 1), E <= 8 ? 7 : 2)
pen_inv_correct_r2(PencilArgs A, const float2* __restrict__ spec, const float2* __restrict__ tw_g, float* Uout) {
  constexpr int N = 32 * E, H = N / 2, NT = 32 * (R + 1);
  extern __shared__ float2 smr[];
  float2* tw = smr;                                     // [N]
  float* ps = reinterpret_cast<float*>(smr + N);        // [2 (R + 2)][N]: rows y0 - 2 .. y0 + 2R + 1
  float4* pre = reinterpret_cast<float4*>(ps + 2 * (R + 2) * N);   // [2][NT]: U* of iteration 0
  constexpr int nblk = H / R, Q = N / 4;   // Q: float4 runs per row
  const int b = blockIdx.x / nblk, mm0 = (blockIdx.x - b * nblk) * R;
  const size_t plane = (size_t)N * N;
  {   // the first correction iteration's U* loads are in flight during the inverse transforms
    const int r = threadIdx.x / Q, x = (threadIdx.x - r * Q) * 4;
    const float* src = A.U + ((size_t)(b * 2) * N + 2 * mm0 + r) * N + x;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(pre + threadIdx.x)),
                 "l"(src) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(pre + NT + threadIdx.x)),
                 "l"(src + plane) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int i = threadIdx.x; i < N; i += NT) {
    const float2 w = tw_g[i & (N / 2 - 1)];
    tw[i] = (i & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warps 0 .. R-1: pairs mm0 .. mm0+R-1 (smem pair slot w + 1); warp R: the halo pairs mm0 - 1 (slot 0)
  // and mm0 + R (slot R + 1), one after the other (R + 1 warps: 7 CTAs per SM at N = 256, one wave at c4)
  for (int t = 0; t < (warp == R ? 2 : 1); ++t) {
    const int slot = warp < R ? warp + 1 : (t == 0 ? 0 : R + 1);
    const int mm = (mm0 - 1 + slot) & (H - 1);   // periodic in y (N even: pairs wrap with the rows)
    float2 z[E];
    const float4* srcz = reinterpret_cast<const float4*>(spec + ((size_t)b * H + mm) * N + lane * E);   // 16-B loads
#pragma unroll
    for (int k = 0; k < E; k += 2) {
      const float4 q = srcz[k / 2];
      z[k] = make_float2(q.x, q.y);
      z[k + 1] = make_float2(q.z, q.w);
    }
    warp_fft_inv<E>(z, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      ps[(2 * slot) * N + lane + 32 * e] = z[e].x;
      ps[(2 * slot + 1) * N + lane + 32 * e] = z[e].y;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  static_assert(NT <= 2 * R * Q, "every thread has an iteration 0");
  for (int i = threadIdx.x; i < 2 * R * Q; i += NT) {
    const int r = i / Q, x = (i - r * Q) * 4;
    const int y = 2 * mm0 + r;
    const float* pr = ps + (r + 2) * N;   // smem row of y
    const float4 pc = *reinterpret_cast<const float4*>(pr + x);
    const float pl = pr[(x - 1) & (N - 1)], prr = pr[(x + 4) & (N - 1)];
    const float4 pu = *reinterpret_cast<const float4*>(pr + N + x), pd = *reinterpret_cast<const float4*>(pr - N + x);
    const size_t iu = ((size_t)(b * 2) * N + y) * N + x;
    const bool first = i == (int)threadIdx.x;
    const float4 uu = first ? pre[threadIdx.x] : *reinterpret_cast<const float4*>(A.U + iu);
    const float4 vv = first ? pre[NT + threadIdx.x] : *reinterpret_cast<const float4*>(A.U + iu + plane);
    float4 ou, ov;
    ou.x = __fsub_rn(uu.x, __fmul_rn(__fsub_rn(pc.y, pl), A.half_inv_h));
    ou.y = __fsub_rn(uu.y, __fmul_rn(__fsub_rn(pc.z, pc.x), A.half_inv_h));
    ou.z = __fsub_rn(uu.z, __fmul_rn(__fsub_rn(pc.w, pc.y), A.half_inv_h));
    ou.w = __fsub_rn(uu.w, __fmul_rn(__fsub_rn(prr, pc.z), A.half_inv_h));
    ov.x = __fsub_rn(vv.x, __fmul_rn(__fsub_rn(pu.x, pd.x), A.half_inv_h));
    ov.y = __fsub_rn(vv.y, __fmul_rn(__fsub_rn(pu.y, pd.y), A.half_inv_h));
    ov.z = __fsub_rn(vv.z, __fmul_rn(__fsub_rn(pu.z, pd.z), A.half_inv_h));
    ov.w = __fsub_rn(vv.w, __fmul_rn(__fsub_rn(pu.w, pd.w), A.half_inv_h));
    *reinterpret_cast<float4*>(Uout + iu) = ou;
    *reinterpret_cast<float4*>(Uout + iu + plane) = ov;
  }
}

// ---------------------------------------------------------------------------
// N = 256 real-data passes on half-warp FFTs (fft256.cuh): the same three passes as the *_r2 kernels --
// rows (two real rows per complex transform, divergence fused), columns (pairs {kx, -kx}, Poisson divide),
// inverse rows fused with the correction -- but each 256-point transform runs on 16 lanes x 16 registers
// with one shared-memory transpose instead of the 32-lane shuffle FFT, and the spectrum rows are stored in
// natural kx order ([B][N/2][N], 4 B per cell).
// ---------------------------------------------------------------------------
constexpr int HW_S = 256;   // float2 per half-warp transpose scratch

__global__ void __launch_bounds__(128, 8)
pen_rows_fwd_n256(PencilArgs A, float2* __restrict__ spec, const float2* __restrict__ tw_g) {
  constexpr int N = 256, H = 128;
  __shared__ float2 tw16[256];
  __shared__ float2 Ssh[8 * HW_S];
  load_tw16x16(tw16, tw_g, threadIdx.x, 128);
  __syncthreads();
  const int hw = threadIdx.x >> 4, h = threadIdx.x & 15;
  const int row = blockIdx.x * 8 + hw;   // (b, row pair mm)
  if (row >= A.B * H) return;             // (whole half-warps: the FFT's __syncwarp stays uniform)
  const int b = row / H, mm = row - b * H;
  const float* u = A.U + (size_t)(b * 2 + 0) * N * N;
  const float* v = A.U + (size_t)(b * 2 + 1) * N * N;
  const int y0 = 2 * mm, y1 = 2 * mm + 1, ym = (y0 - 1) & (N - 1), yp = (y1 + 1) & (N - 1);
  float2 z[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int x = h + 16 * j, xp = (x + 1) & (N - 1), xm = (x - 1) & (N - 1);
    const float d0 = (__ldg(u + y0 * N + xp) - __ldg(u + y0 * N + xm) + __ldg(v + y1 * N + x) - __ldg(v + ym * N + x)) * A.half_inv_h;
    const float d1 = (__ldg(u + y1 * N + xp) - __ldg(u + y1 * N + xm) + __ldg(v + yp * N + x) - __ldg(v + y0 * N + x)) * A.half_inv_h;
    z[j] = make_float2(d0, d1);
  }
  fft256_hw<false>(z, Ssh + hw * HW_S, tw16, h);
  float2* dst = spec + ((size_t)b * H + mm) * N;
#pragma unroll
  for (int j = 0; j < 16; ++j) dst[h + 16 * j] = z[j];   // natural kx: 16 lanes, 128 contiguous B
}

// columns: the CTA's 8 column pairs (kx = q0 .. q0 + 7 and -kx), one per half-warp; loads and stores
// row-major through shared memory as in pen_cols_r2s
__global__ void __launch_bounds__(128, 8)
pen_cols_n256(PencilArgs A, float2* __restrict__ spec, const float2* __restrict__ tw_g, const float* __restrict__ ks_g) {
  constexpr int N = 256, H = 128, NPAIR = 129, CC = 8, PC = CC + 1;
  // [m][c] Z_m(kx) | Z_m(-kx); between the unpack and the repack the same memory is the 8 half-warps'
  // FFT scratch (8 x 256 float2 <= 2 x 128 x 9)
  __shared__ float2 TT[2 * H * PC];
  float2* T1 = TT;
  float2* T2 = TT + H * PC;
  __shared__ float2 tw16[256];
  __shared__ float ks[N];
  load_tw16x16(tw16, tw_g, threadIdx.x, 128);
  for (int i = threadIdx.x; i < N; i += 128) ks[i] = ks_g[i];
  constexpr int nblk = (NPAIR + CC - 1) / CC;
  const int b = blockIdx.x / nblk, q0 = (blockIdx.x - b * nblk) * CC;
  float2* sb = spec + (size_t)b * H * N;
  for (int i = threadIdx.x; i < CC * H; i += 128) {
    const int m = i / CC, c = i - m * CC, kx = q0 + c;
    if (kx < NPAIR) {
      T1[m * PC + c] = sb[(size_t)m * N + kx];
      T2[m * PC + c] = sb[(size_t)m * N + ((N - kx) & (N - 1))];
    }
  }
  __syncthreads();
  const int hw = threadIdx.x >> 4, h = threadIdx.x & 15, c = hw, kx = q0 + c;
  const bool live = kx < NPAIR;   // (dead half-warps of the last block transform zeros, write nothing)
  float2 v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {   // D_y(kx), y = h + 16 j
    const int y = h + 16 * j, m = y >> 1;
    const float2 a = live ? T1[m * PC + c] : make_float2(0.f, 0.f);
    const float2 bb = live ? conjf2(T2[m * PC + c]) : make_float2(0.f, 0.f);
    v[j] = (y & 1) ? make_float2(0.5f * (a.y - bb.y), -0.5f * (a.x - bb.x)) : make_float2(0.5f * (a.x + bb.x), 0.5f * (a.y + bb.y));
  }
  __syncthreads();   // every column read: T1 / T2 become the transpose scratch
  float2* S = TT + hw * HW_S;
  fft256_hw<false>(v, S, tw16, h);   // lane h, register j: ky = h + 16 j
  const bool xnull = kx == 0 || kx == N / 2;
  const int kxs = live ? kx : 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int ky = h + 16 * j;
    const bool nul = xnull && (ky == 0 || ky == N / 2);
    const float f = nul ? 0.f : -A.scale / (ks[kxs] + ks[ky]);
    v[j] = make_float2(v[j].x * f, v[j].y * f);
  }
  fft256_hw<true>(v, S, tw16, h);    // lane h, register j: y = h + 16 j
  __syncthreads();   // every half-warp's scratch use is over: T1 / T2 take the repacked values
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    // even lanes hold P_{2m}, lane h + 1 holds P_{2m+1} (y = h + 16 j, m = y / 2)
    const float2 o = make_float2(__shfl_down_sync(0xffffffffu, v[j].x, 1, 16), __shfl_down_sync(0xffffffffu, v[j].y, 1, 16));
    if (live && !(h & 1)) {
      const int m = (h + 16 * j) >> 1;
      if (xnull) {   // self-paired column: P real up to rounding
        T1[m * PC + c] = make_float2(v[j].x, o.x);
      } else {
        T1[m * PC + c] = make_float2(v[j].x - o.y, v[j].y + o.x);
        T2[m * PC + c] = make_float2(v[j].x + o.y, o.x - v[j].y);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < CC * H; i += 128) {
    const int m = i / CC, c2 = i - m * CC, k2 = q0 + c2;
    if (k2 < NPAIR) {
      sb[(size_t)m * N + k2] = T1[m * PC + c2];
      if (k2 != 0 && k2 != N / 2) sb[(size_t)m * N + (N - k2)] = T2[m * PC + c2];
    }
  }
}

// inverse rows fused with the correction (as pen_inv_correct_r2): R = 8 own row pairs + 2 halo pairs, one
// per half-warp (5 warps), p rows in shared memory, U = U* - G_c p on float4 runs of the 16 own rows
__global__ void __launch_bounds__(160, 8)
pen_inv_correct_n256(PencilArgs A, const float2* __restrict__ spec, const float2* __restrict__ tw_g, float* Uout) {
  constexpr int N = 256, H = 128, R = 8, NT = 160, Q = N / 4;
  __shared__ float2 tw16[256];
  // rows y0 - 2 .. y0 + 2R + 1; half-warp hw's two rows (2 KB) are first its FFT scratch
  __shared__ __align__(16) float ps[2 * (R + 2) * N];
  __shared__ float4 pre[2 * NT];                         // U* of the first correction iteration
  constexpr int nblk = H / R;
  const int b = blockIdx.x / nblk, mm0 = (blockIdx.x - b * nblk) * R;
  const size_t plane = (size_t)N * N;
  {
    const int r = threadIdx.x / Q, x = (threadIdx.x - r * Q) * 4;
    const float* src = A.U + ((size_t)(b * 2) * N + 2 * mm0 + r) * N + x;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(pre + threadIdx.x)),
                 "l"(src) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(pre + NT + threadIdx.x)),
                 "l"(src + plane) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  load_tw16x16(tw16, tw_g, threadIdx.x, NT);
  __syncthreads();
  {
    const int hw = threadIdx.x >> 4, h = threadIdx.x & 15;   // half-warp hw: pair slot hw (0: mm0 - 1)
    const int mm = (mm0 - 1 + hw) & (H - 1);
    const float2* src = spec + ((size_t)b * H + mm) * N;
    float2 z[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) z[j] = src[h + 16 * j];
    fft256_hw<true>(z, reinterpret_cast<float2*>(ps + 2 * hw * N), tw16, h);   // (ends with __syncwarp)
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      ps[(2 * hw) * N + h + 16 * j] = z[j].x;
      ps[(2 * hw + 1) * N + h + 16 * j] = z[j].y;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * R * Q; i += NT) {
    const int r = i / Q, x = (i - r * Q) * 4;
    const int y = 2 * mm0 + r;
    const float* pr = ps + (r + 2) * N;
    const float4 pc = *reinterpret_cast<const float4*>(pr + x);
    const float pl = pr[(x - 1) & (N - 1)], prr = pr[(x + 4) & (N - 1)];
    const float4 pu = *reinterpret_cast<const float4*>(pr + N + x), pd = *reinterpret_cast<const float4*>(pr - N + x);
    const size_t iu = ((size_t)(b * 2) * N + y) * N + x;
    const bool first = i == (int)threadIdx.x;
    const float4 uu = first ? pre[threadIdx.x] : *reinterpret_cast<const float4*>(A.U + iu);
    const float4 vv = first ? pre[NT + threadIdx.x] : *reinterpret_cast<const float4*>(A.U + iu + plane);
    float4 ou, ov;
    ou.x = __fsub_rn(uu.x, __fmul_rn(__fsub_rn(pc.y, pl), A.half_inv_h));
    ou.y = __fsub_rn(uu.y, __fmul_rn(__fsub_rn(pc.z, pc.x), A.half_inv_h));
    ou.z = __fsub_rn(uu.z, __fmul_rn(__fsub_rn(pc.w, pc.y), A.half_inv_h));
    ou.w = __fsub_rn(uu.w, __fmul_rn(__fsub_rn(prr, pc.z), A.half_inv_h));
    ov.x = __fsub_rn(vv.x, __fmul_rn(__fsub_rn(pu.x, pd.x), A.half_inv_h));
    ov.y = __fsub_rn(vv.y, __fmul_rn(__fsub_rn(pu.y, pd.y), A.half_inv_h));
    ov.z = __fsub_rn(vv.z, __fmul_rn(__fsub_rn(pu.z, pd.z), A.half_inv_h));
    ov.w = __fsub_rn(vv.w, __fmul_rn(__fsub_rn(pu.w, pd.w), A.half_inv_h));
    *reinterpret_cast<float4*>(Uout + iu) = ou;
    *reinterpret_cast<float4*>(Uout + iu + plane) = ov;
  }
}

static cudaError_t projection_n256(const PencilArgs& A, float2* spec, const float2* tw, const float* ks, float* Uout,
                                   cudaStream_t st) {
  const int pairs = A.B * 128;
  pen_rows_fwd_n256<<<(pairs + 7) / 8, 128, 0, st>>>(A, spec, tw);
  pen_cols_n256<<<A.B * 17, 128, 0, st>>>(A, spec, tw, ks);
  pen_inv_correct_n256<<<A.B * 16, 160, 0, st>>>(A, spec, tw, Uout);
  return cudaGetLastError();
}

// r2 forward + column passes; with fuse_corr the inverse row pass and the correction run as one kernel
// (pen_inv_correct_r2, Uout written) -- otherwise the inverse pass writes p and the caller corrects
template <int E>
static cudaError_t projection_r2(const PencilArgs& A, float2* spec, float* p, const float2* tw, const float* ks,
                                 cudaStream_t st, float* Uout = nullptr) {
  constexpr int N = 32 * E;
  const int rows = A.B * (N / 2);
  pen_rows_fwd_r2<E><<<(rows + 3) / 4, 128, 0, st>>>(A, spec, tw);
  constexpr int CC = E >= 32 ? 4 : 8;
  const int nblk = (N / 2 + 1 + CC - 1) / CC;
  const size_t smem = sizeof(float2) * ((size_t)2 * CC * (N / 2) + N) + sizeof(float) * N;
  static const bool cols_old = getenv("LD_PEN_COLS_OLD") != nullptr;   // measurement knob
  if (cols_old) pen_cols_r2<E, CC><<<A.B * nblk, 128, smem, st>>>(A, spec, tw, ks);
  else pen_cols_r2s<E, CC, 4><<<A.B * nblk, 128, cols_r2s_smem<E, CC>(), st>>>(A, spec, tw, ks);
  if (Uout != nullptr) {
    constexpr int R = R2_CORR_R;
    pen_inv_correct_r2<E, R><<<A.B * (N / 2 / R), 32 * (R + 1), inv_corr_smem<E, R>(), st>>>(A, spec, tw, Uout);
  } else {
    pen_rows_inv_r2<E><<<(rows + 3) / 4, 128, 0, st>>>(A, spec, p, tw);
  }
  return cudaGetLastError();
}

// ---- pass 4: U = U* - G_c p on the own rows; p rows y0 - 1 / y0 + n from pbelow / pabove
// ([B][N] each; for P = 1 they are rows N-1 / 0 of p itself).  In place allowed (Uout == U*).
// One thread per float4 run of a row (N a power of two >= 4): 32-bit index arithmetic by shifts
// (the earlier grid-stride form spent its time in 64-bit divisions), explicitly rounded operations.
__global__ void __launch_bounds__(256)
pen_correct(PencilArgs A, const float* __restrict__ p, const float* pbelow, const float* pabove, long long pstride,
            float* Uout, int out_rows, int out_row0) {
  const int N = A.N, n = N / A.P;
  const int lq = __ffs(N) - 3;   // log2(N / 4)
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int by = t >> lq, x = (t & ((N >> 2) - 1)) << 2;
  if (by >= A.B * n) return;
  const int b = by / n, y = by - b * n;
  const float* pr = p + ((size_t)b * n + y) * N;
  const float* pdn = y > 0 ? pr - N : pbelow + (size_t)b * pstride;
  const float* pup = y + 1 < n ? pr + N : pabove + (size_t)b * pstride;
  const float4 pc = *reinterpret_cast<const float4*>(pr + x);
  const float pl = pr[(x - 1) & (N - 1)], prr = pr[(x + 4) & (N - 1)];
  const float4 pu = *reinterpret_cast<const float4*>(pup + x), pd = *reinterpret_cast<const float4*>(pdn + x);
  const size_t iu = ((size_t)(b * 2) * A.rows + A.row0 + y) * N + x;
  const size_t iv = iu + (size_t)A.rows * N;
  const size_t ou = ((size_t)(b * 2) * out_rows + out_row0 + y) * N + x;
  const size_t ov = ou + (size_t)out_rows * N;
  const float4 uu = *reinterpret_cast<const float4*>(A.U + iu);
  const float4 vv = *reinterpret_cast<const float4*>(A.U + iv);
  float4 ru, rv;
  ru.x = __fsub_rn(uu.x, __fmul_rn(__fsub_rn(pc.y, pl), A.half_inv_h));
  ru.y = __fsub_rn(uu.y, __fmul_rn(__fsub_rn(pc.z, pc.x), A.half_inv_h));
  ru.z = __fsub_rn(uu.z, __fmul_rn(__fsub_rn(pc.w, pc.y), A.half_inv_h));
  ru.w = __fsub_rn(uu.w, __fmul_rn(__fsub_rn(prr, pc.z), A.half_inv_h));
  rv.x = __fsub_rn(vv.x, __fmul_rn(__fsub_rn(pu.x, pd.x), A.half_inv_h));
  rv.y = __fsub_rn(vv.y, __fmul_rn(__fsub_rn(pu.y, pd.y), A.half_inv_h));
  rv.z = __fsub_rn(vv.z, __fmul_rn(__fsub_rn(pu.z, pd.z), A.half_inv_h));
  rv.w = __fsub_rn(vv.w, __fmul_rn(__fsub_rn(pu.w, pd.w), A.half_inv_h));
  *reinterpret_cast<float4*>(Uout + ou) = ru;
  *reinterpret_cast<float4*>(Uout + ov) = rv;
}

// ---------------------------------------------------------------------------
// N = N1 N2 >= 2048 (four-step over warp FFTs, N1 = 64, N2 = N / 64 in {32, 64}).  One CTA per
// transform, data in shared memory.  With n = N2 n1 + n2 and k = k1 + N1 k2:
//   X[k1 + N1 k2] = sum_n2 W_N2^{n2 k2} W_N^{n2 k1} sum_n1 x[N2 n1 + n2] W_N1^{n1 k1}
// forward: (1) N2 warp FFTs of length N1 over n1 (stride N2) -> S[k1][n2] * W_N^{n2 k1};
// (3) N1 warp FFTs of length N2 over n2 -> lane l, register j of sequence k1 holds
// X[k1 + N1 (j + E2 bitrev5(l))], stored at position pos = k1 N2 + l E2 + j.  The inverse runs
// the transposed steps: (3') inverse warp FFTs of the N1 position runs (scrambled in, natural
// n2 out), conj twiddle, (1') inverse warp FFTs over k1 (scrambled in, natural n1 out).
// ---------------------------------------------------------------------------
template <int N2>
LD_DEVINL int pos_to_k4(int pos) {
  constexpr int N1 = 64, E2 = N2 / 32;
  const int k1 = pos / N2, t = pos - k1 * N2;
  return k1 + N1 * (t % E2 + E2 * (int)(__brev((unsigned)(t / E2)) >> 27));
}
LD_DEVINL int padx(int n) { return n + (n >> 6); }   // one complex of padding per 64: conflict-free stride-N2 reads

// forward: X natural (padded) -> X in positions order (unpadded).  twN = W_N, tw1 = W_64, tw2 = W_N2.
template <int N2>
LD_DEVINL void block_fft_fwd(float2* X, float2* S, const float2* twN, const float2* tw1, const float2* tw2) {
  constexpr int N1 = 64, N = N1 * N2, E1 = 2, E2 = N2 / 32;
  constexpr int SP = N2 + 1;   // S row pitch
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int br = (int)(__brev((unsigned)lane) >> 27);
  for (int n2 = warp; n2 < N2; n2 += nw) {
    float2 v[E1];
#pragma unroll
    for (int e = 0; e < E1; ++e) v[e] = X[padx(N2 * (lane + 32 * e) + n2)];
    warp_fft_fwd<E1>(v, tw1);
#pragma unroll
    for (int j = 0; j < E1; ++j) {
      const int k1 = j + E1 * br;
      S[k1 * SP + n2] = cmul(v[j], twN[(n2 * k1) & (N - 1)]);
    }
  }
  __syncthreads();
  for (int k1 = warp; k1 < N1; k1 += nw) {
    float2 v[E2];
#pragma unroll
    for (int e = 0; e < E2; ++e) v[e] = S[k1 * SP + lane + 32 * e];
    warp_fft_fwd<E2>(v, tw2);
#pragma unroll
    for (int j = 0; j < E2; ++j) X[k1 * N2 + lane * E2 + j] = v[j];   // positions, unpadded
  }
  __syncthreads();
}

// inverse: X in positions order (unpadded) -> X natural (padded)
template <int N2>
LD_DEVINL void block_fft_inv(float2* X, float2* S, const float2* twN, const float2* tw1, const float2* tw2) {
  constexpr int N1 = 64, N = N1 * N2, E1 = 2, E2 = N2 / 32;
  constexpr int SP = N2 + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int br = (int)(__brev((unsigned)lane) >> 27);
  for (int k1 = warp; k1 < N1; k1 += nw) {
    float2 v[E2];
#pragma unroll
    for (int j = 0; j < E2; ++j) v[j] = X[k1 * N2 + lane * E2 + j];
    warp_fft_inv<E2>(v, tw2);
#pragma unroll
    for (int e = 0; e < E2; ++e) {
      const int n2 = lane + 32 * e;
      S[k1 * SP + n2] = cmul(v[e], conjf2(twN[(n2 * k1) & (N - 1)]));
    }
  }
  __syncthreads();
  for (int n2 = warp; n2 < N2; n2 += nw) {
    float2 v[E1];
#pragma unroll
    for (int j = 0; j < E1; ++j) v[j] = S[(j + E1 * br) * SP + n2];
    warp_fft_inv<E1>(v, tw1);
#pragma unroll
    for (int e = 0; e < E1; ++e) X[padx(N2 * (lane + 32 * e) + n2)] = v[e];
  }
  __syncthreads();
}

// shared tables for the four-step kernels: twN [N], tw1 [64], tw2 [N2]
template <int N2>
LD_DEVINL void load_tables4(float2* twN, float2* tw1, float2* tw2, const float2* __restrict__ tw_g) {
  constexpr int N1 = 64, N = N1 * N2;
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    const float2 w = tw_g[m & (N / 2 - 1)];
    twN[m] = (m & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();
  for (int m = threadIdx.x; m < N1; m += blockDim.x) tw1[m] = twN[m * N2];
  for (int m = threadIdx.x; m < N2; m += blockDim.x) tw2[m] = twN[m * N1];
  __syncthreads();
}

template <int N2>
constexpr size_t smem4_bytes(int cols) {
  // twN + tw1 + tw2 + cols x padded transforms + S scratch + ks (floats)
  return sizeof(float2) * ((size_t)64 * N2 + 64 + N2 + (size_t)cols * (64 * N2 + N2 + 1) + 64 * (N2 + 1)) +
         sizeof(float) * 64 * N2;
}

template <int N2>
__global__ void __launch_bounds__(512)
pen_rows_fwd_4s(PencilArgs A, float2* __restrict__ send, const float2* __restrict__ tw_g) {
  constexpr int N1 = 64, N = N1 * N2;
  extern __shared__ float2 sm4[];
  float2* twN = sm4;
  float2* tw1 = twN + N;
  float2* tw2 = tw1 + N1;
  float2* X = tw2 + N2;                       // [padx(N)]
  float2* S = X + (N + N2 + 1);               // [N1][N2+1]
  load_tables4<N2>(twN, tw1, tw2, tw_g);
  const int n = N / A.P, m = N / A.P;
  // persistent: the CTA walks rows blockIdx.x, + gridDim.x, ... (the 48 KB of tables loaded once)
  for (int row = blockIdx.x; row < A.B * n; row += gridDim.x) {
  if (row != (int)blockIdx.x) __syncthreads();   // the previous row's X reads are done
  const int b = row / n, y = row - b * n;
  const float* u = A.U + ((size_t)(b * 2 + 0) * A.rows + A.row0) * N;
  const float* v = A.U + ((size_t)(b * 2 + 1) * A.rows + A.row0) * N;
  const float* vdn = y > 0 ? v + (size_t)(y - 1) * N : A.vbelow + (size_t)b * A.vstride;
  const float* vup = y + 1 < n ? v + (size_t)(y + 1) * N : A.vabove + (size_t)b * A.vstride;
  for (int x = threadIdx.x; x < N; x += blockDim.x) {
    const float d = (__ldg(u + (size_t)y * N + ((x + 1) & (N - 1))) - __ldg(u + (size_t)y * N + ((x - 1) & (N - 1))) +
                     __ldg(vup + x) - __ldg(vdn + x)) * A.half_inv_h;
    X[padx(x)] = make_float2(d, 0.f);
  }
  __syncthreads();
  block_fft_fwd<N2>(X, S, twN, tw1, tw2);
  for (int pos = threadIdx.x; pos < N; pos += blockDim.x) {
    const int s = pos / m, c = pos - s * m;
    send[(((size_t)s * A.B + b) * n + y) * m + c] = X[pos];
  }
  }
}

template <int N2>
__global__ void __launch_bounds__(512)
pen_rows_inv_4s(PencilArgs A, const float2* __restrict__ recv, float* __restrict__ p, const float2* __restrict__ tw_g) {
  constexpr int N1 = 64, N = N1 * N2;
  extern __shared__ float2 sm4[];
  float2* twN = sm4;
  float2* tw1 = twN + N;
  float2* tw2 = tw1 + N1;
  float2* X = tw2 + N2;
  float2* S = X + (N + N2 + 1);
  load_tables4<N2>(twN, tw1, tw2, tw_g);
  const int n = N / A.P, m = N / A.P;
  for (int row = blockIdx.x; row < A.B * n; row += gridDim.x) {   // persistent (see pen_rows_fwd_4s)
    if (row != (int)blockIdx.x) __syncthreads();
    const int b = row / n, y = row - b * n;
    for (int pos = threadIdx.x; pos < N; pos += blockDim.x) {
      const int s = pos / m, c = pos - s * m;
      X[pos] = recv[(((size_t)s * A.B + b) * n + y) * m + c];
    }
    __syncthreads();
    block_fft_inv<N2>(X, S, twN, tw1, tw2);
    for (int x = threadIdx.x; x < N; x += blockDim.x) p[((size_t)b * n + y) * N + x] = X[padx(x)].x;
  }
}

// columns for N >= 2048: CC columns of element b per CTA, one four-step transform at a time
template <int N2, int CC>
__global__ void __launch_bounds__(512)
pen_cols_4s(PencilArgs A, float2* __restrict__ buf, const float2* __restrict__ tw_g, const float* __restrict__ ks_g) {
  constexpr int N1 = 64, N = N1 * N2, XP = N + N2 + 1;
  extern __shared__ float2 sm4[];
  float2* twN = sm4;
  float2* tw1 = twN + N;
  float2* tw2 = tw1 + N1;
  float2* T = tw2 + N2;                       // [CC][XP] columns (padded natural y)
  float2* S = T + CC * XP;                    // [N1][N2+1]
  float* ks = reinterpret_cast<float*>(S + N1 * (N2 + 1));
  load_tables4<N2>(twN, tw1, tw2, tw_g);
  for (int i = threadIdx.x; i < N; i += blockDim.x) ks[i] = ks_g[i];
  const int n = N / A.P, m = N / A.P;
  const int nblk = m / CC;
  for (int blk = blockIdx.x; blk < A.B * nblk; blk += gridDim.x) {   // persistent (tables loaded once)
  if (blk != (int)blockIdx.x) __syncthreads();
  const int b = blk / nblk, c0 = (blk - b * nblk) * CC;
  for (int i = threadIdx.x; i < N * CC; i += blockDim.x) {
    const int y = i / CC, c = i - y * CC;
    const int r = y / n, yl = y - r * n;
    T[c * XP + padx(y)] = buf[(((size_t)r * A.B + b) * n + yl) * m + c0 + c];
  }
  __syncthreads();
  for (int c = 0; c < CC; ++c) {
    float2* X = T + c * XP;
    block_fft_fwd<N2>(X, S, twN, tw1, tw2);   // X now in positions order along y
    const int kx = pos_to_k4<N2>(A.rank * m + c0 + c);
    const bool xnull = kx == 0 || kx == N / 2;
    for (int pos = threadIdx.x; pos < N; pos += blockDim.x) {
      const int ky = pos_to_k4<N2>(pos);
      const bool nul = xnull && (ky == 0 || ky == N / 2);
      const float f = nul ? 0.f : -A.scale / (ks[kx] + ks[ky]);
      X[pos] = make_float2(X[pos].x * f, X[pos].y * f);
    }
    __syncthreads();
    block_fft_inv<N2>(X, S, twN, tw1, tw2);   // back to natural y (padded)
  }
  for (int i = threadIdx.x; i < N * CC; i += blockDim.x) {
    const int y = i / CC, c = i - y * CC;
    const int r = y / n, yl = y - r * n;
    buf[(((size_t)r * A.B + b) * n + yl) * m + c0 + c] = T[c * XP + padx(y)];
  }
  }
}

// ---------------------------------------------------------------------------
// N = 4096 column pass on half-warp FFTs (fft256.cuh): 4096 = 16 x 256, n = n2 + 16 n1, k = k1 + 256 k2,
//   X[k1 + 256 k2] = sum_n2 W16^{n2 k2} W4096^{n2 k1} sum_n1 x[n2 + 16 n1] W256^{n1 k1}.
// A column is transformed by a group of 256 threads (16 half-warps): half-warp n2 runs the 256-point FFT
// over n1 (lane h, register j: n1 / k1 = h + 16 j), the twiddle W4096^{n2 k1}, a transpose through the
// column's shared buffer (k1-major, pitch 17), then thread t = k1 runs the 16-point DFT over n2 and holds
// X[t + 256 k2] -- natural ky, so the Poisson divide happens in registers and the inverse runs the same
// steps backwards.  Two columns per CTA (512 threads, one per group), the same load / store layout as
// pen_cols_4s (P position blocks, slab-ready).  Replaces the 64 x 64 shuffle-FFT block transform of
// pen_cols_4s<64, CC> (c5a; LD_PEN4_OLD=1 keeps it).
// ---------------------------------------------------------------------------
constexpr int C4K_COL = 4096 + 256;   // float2 per column buffer: natural y at n + (n >> 4), or k1 * 17 + n2
constexpr size_t cols4k_smem() { return sizeof(float2) * ((size_t)2 * C4K_COL + 4096 + 256); }

template <int MB>
__global__ void __launch_bounds__(512, MB)
pen_cols_4k_hw(PencilArgs A, float2* __restrict__ buf, const float2* __restrict__ tw_g, const float* __restrict__ ks_g) {
  constexpr int N = 4096, N2 = 64;
  extern __shared__ float2 smk[];
  float2* T = smk;                        // [2][C4K_COL]
  float2* twN = T + 2 * C4K_COL;          // [4096] W4096^m
  float2* tw16 = twN + N;                 // [256] W256^{h k1}
  for (int m2 = threadIdx.x; m2 < N; m2 += blockDim.x) {
    const float2 w = tw_g[m2 & (N / 2 - 1)];
    twN[m2] = (m2 & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();   // tw16 is read from twN entries other warps wrote
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tw16[i] = twN[((i >> 4) * (i & 15)) * 16];   // W256^m = W4096^{16 m}
  __syncthreads();
  const int n = N / A.P, m = N / A.P;
  constexpr int CC = 2;
  const int nblk = m / CC;
  const int g = threadIdx.x >> 8, t = threadIdx.x & 255;   // column group, thread in group
  const int hw = t >> 4, h = t & 15;                          // half-warp (n2), lane
  float2* Tg = T + g * C4K_COL;
  auto gbar = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory"); };   // the group's 256 threads
  for (int blk = blockIdx.x; blk < A.B * nblk; blk += gridDim.x) {
    const int b = blk / nblk, c0 = (blk - b * nblk) * CC;
    __syncthreads();   // the previous block's stores have read T
    for (int i = threadIdx.x; i < N * CC; i += blockDim.x) {   // coalesced: CC consecutive complex per row y
      const int y = i / CC, c = i - y * CC;
      const int r = y / n, yl = y - r * n;
      T[c * C4K_COL + y + (y >> 4)] = buf[(((size_t)r * A.B + b) * n + yl) * m + c0 + c];
    }
    __syncthreads();
    // ---- forward: half-warp n2 = hw, 256-point FFT over n1 of x[n2 + 16 n1]
    float2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int y = hw + 16 * (h + 16 * j);
      v[j] = Tg[y + (y >> 4)];
    }
    gbar();   // every input read: the buffer is the FFT scratch (half-warp hw: 256 float2 at hw * 256)
    fft256_hw<false>(v, Tg + hw * 256, tw16, h);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = cmul(v[j], twN[hw * (h + 16 * j)]);   // W4096^{n2 k1}
    gbar();
#pragma unroll
    for (int j = 0; j < 16; ++j) Tg[(h + 16 * j) * 17 + hw] = v[j];   // (k1, n2)
    gbar();
    float2 w[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) w[q] = Tg[t * 17 + q];   // k1 = t, n2 = q
    dft16<false>(w);                                        // w[k2] = X[t + 256 k2]
    // ---- Poisson divide (natural ky = t + 256 k2)
    const int kx = pos_to_k4<N2>(A.rank * m + c0 + g);
    const bool xnull = kx == 0 || kx == N / 2;
    const float kxs = __ldg(ks_g + kx);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int ky = t + 256 * q;
      const bool nul = xnull && (ky == 0 || ky == N / 2);
      const float f = nul ? 0.f : -A.scale / (kxs + __ldg(ks_g + ky));
      w[q] = make_float2(w[q].x * f, w[q].y * f);
    }
    // ---- inverse: thread t = k1: 16-point inverse DFT over k2, conj twiddle, transpose, half-warp FFTs over k1
    dft16<true>(w);   // w[n2]
#pragma unroll
    for (int q = 0; q < 16; ++q) w[q] = cmul(w[q], conjf2(twN[q * t]));
    gbar();   // the (k1, n2) reads above are done
#pragma unroll
    for (int q = 0; q < 16; ++q) Tg[t * 17 + q] = w[q];
    gbar();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = Tg[(h + 16 * j) * 17 + hw];   // k1 = h + 16 j, n2 = hw
    gbar();
    fft256_hw<true>(v, Tg + hw * 256, tw16, h);   // x[n2 + 16 n1], n1 = h + 16 j
    gbar();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int y = hw + 16 * (h + 16 * j);
      Tg[y + (y >> 4)] = v[j];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N * CC; i += blockDim.x) {
      const int y = i / CC, c = i - y * CC;
      const int r = y / n, yl = y - r * n;
      buf[(((size_t)r * A.B + b) * n + yl) * m + c0 + c] = T[c * C4K_COL + y + (y >> 4)];
    }
  }
}

// ---------------------------------------------------------------------------
// N = 4096 row passes on half-warp FFTs: the same 16 x 256 four-step as pen_cols_4k_hw, one row per group of
// 256 threads, two rows per CTA.  The spectrum row is stored in the "positions" order of the shuffle-FFT
// passes (pos_to_k4<64>: kx = k1 + 64 hi at pos = 64 k1 + (hi & 1) + 2 bitrev5(hi >> 1)) through a padded
// shared row (padx: the stride-64 scatter is conflict-free), so the column pass, the slab all-to-all blocks
// and pen_correct are unchanged.  LD_PEN4_OLD=1 keeps pen_rows_fwd_4s / pen_rows_inv_4s.
// ---------------------------------------------------------------------------
LD_DEVINL int k_to_pos4k(int kx) {
  const int hi = kx >> 6;
  return ((kx & 63) << 6) + (hi & 1) + 2 * (int)(__brev((unsigned)(hi >> 1)) >> 27);
}

template <int MB>
__global__ void __launch_bounds__(512, MB)
pen_rows_fwd_4k_hw(PencilArgs A, float2* __restrict__ send, const float2* __restrict__ tw_g) {
  constexpr int N = 4096;
  extern __shared__ float2 smk[];
  float2* T = smk;                        // [2][C4K_COL]
  float2* twN = T + 2 * C4K_COL;          // [4096] W4096^m
  float2* tw16 = twN + N;                 // [256] W256^{h k1}
  for (int m2 = threadIdx.x; m2 < N; m2 += blockDim.x) {
    const float2 w = tw_g[m2 & (N / 2 - 1)];
    twN[m2] = (m2 & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();   // tw16 is read from twN entries other warps wrote
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tw16[i] = twN[((i >> 4) * (i & 15)) * 16];
  __syncthreads();
  const int n = N / A.P, m = N / A.P;
  const int g = threadIdx.x >> 8, t = threadIdx.x & 255;   // row group, thread in group
  const int hw = t >> 4, h = t & 15;                          // half-warp (n2), lane
  float2* Tg = T + g * C4K_COL;
  float* Tf = reinterpret_cast<float*>(Tg);
  auto gbar = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory"); };
  const int npair = (A.B * n) >> 1;       // n is even: the two rows of a pair belong to one element
  for (int blk = blockIdx.x; blk < npair; blk += gridDim.x) {
    const int row = 2 * blk + g;
    const int b = row / n, y = row - b * n;
    const float* u = A.U + ((size_t)(b * 2 + 0) * A.rows + A.row0) * N;
    const float* v_ = A.U + ((size_t)(b * 2 + 1) * A.rows + A.row0) * N;
    const float* vdn = y > 0 ? v_ + (size_t)(y - 1) * N : A.vbelow + (size_t)b * A.vstride;
    const float* vup = y + 1 < n ? v_ + (size_t)(y + 1) * N : A.vabove + (size_t)b * A.vstride;
    gbar();   // the previous row's stores have read Tg
    for (int x = t; x < N; x += 256) {
      const float d = (__ldg(u + (size_t)y * N + ((x + 1) & (N - 1))) - __ldg(u + (size_t)y * N + ((x - 1) & (N - 1))) +
                       __ldg(vup + x) - __ldg(vdn + x)) * A.half_inv_h;
      Tf[x + (x >> 4)] = d;
    }
    gbar();
    float2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int x = hw + 16 * (h + 16 * j);
      v[j] = make_float2(Tf[x + (x >> 4)], 0.f);
    }
    gbar();   // every input read: the buffer is the FFT scratch
    fft256_hw<false>(v, Tg + hw * 256, tw16, h);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = cmul(v[j], twN[hw * (h + 16 * j)]);   // W4096^{n2 k1}
    gbar();
#pragma unroll
    for (int j = 0; j < 16; ++j) Tg[(h + 16 * j) * 17 + hw] = v[j];   // (k1, n2)
    gbar();
    float2 w[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) w[q] = Tg[t * 17 + q];
    dft16<false>(w);                                        // w[k2] = X[t + 256 k2]
    gbar();   // the (k1, n2) reads are done
#pragma unroll
    for (int q = 0; q < 16; ++q) Tg[padx(k_to_pos4k(t + 256 * q))] = w[q];
    gbar();
    for (int pos = t; pos < N; pos += 256) {
      const int s = pos / m, c = pos - s * m;
      send[(((size_t)s * A.B + b) * n + y) * m + c] = Tg[padx(pos)];
    }
  }
}

template <int MB>
__global__ void __launch_bounds__(512, MB)
pen_rows_inv_4k_hw(PencilArgs A, const float2* __restrict__ recv, float* __restrict__ p, const float2* __restrict__ tw_g) {
  constexpr int N = 4096;
  extern __shared__ float2 smk[];
  float2* T = smk;
  float2* twN = T + 2 * C4K_COL;
  float2* tw16 = twN + N;
  for (int m2 = threadIdx.x; m2 < N; m2 += blockDim.x) {
    const float2 w = tw_g[m2 & (N / 2 - 1)];
    twN[m2] = (m2 & (N / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tw16[i] = twN[((i >> 4) * (i & 15)) * 16];
  __syncthreads();
  const int n = N / A.P, m = N / A.P;
  const int g = threadIdx.x >> 8, t = threadIdx.x & 255;
  const int hw = t >> 4, h = t & 15;
  float2* Tg = T + g * C4K_COL;
  float* Tf = reinterpret_cast<float*>(Tg);
  auto gbar = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory"); };
  const int npair = (A.B * n) >> 1;
  for (int blk = blockIdx.x; blk < npair; blk += gridDim.x) {
    const int row = 2 * blk + g;
    const int b = row / n, y = row - b * n;
    gbar();   // the previous row's stores have read Tf
    for (int pos = t; pos < N; pos += 256) {
      const int s = pos / m, c = pos - s * m;
      Tg[padx(pos)] = recv[(((size_t)s * A.B + b) * n + y) * m + c];
    }
    gbar();
    float2 w[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) w[q] = Tg[padx(k_to_pos4k(t + 256 * q))];   // X[t + 256 k2]
    dft16<true>(w);   // over k2 -> n2
#pragma unroll
    for (int q = 0; q < 16; ++q) w[q] = cmul(w[q], conjf2(twN[q * t]));
    gbar();   // the positions reads are done
#pragma unroll
    for (int q = 0; q < 16; ++q) Tg[t * 17 + q] = w[q];
    gbar();
    float2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = Tg[(h + 16 * j) * 17 + hw];   // k1 = h + 16 j, n2 = hw
    gbar();
    fft256_hw<true>(v, Tg + hw * 256, tw16, h);   // x[n2 + 16 n1], n1 = h + 16 j
    gbar();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int x = hw + 16 * (h + 16 * j);
      Tf[x + (x >> 4)] = v[j].x;
    }
    gbar();
    for (int x = t; x < N; x += 256) p[((size_t)b * n + y) * N + x] = Tf[x + (x >> 4)];
  }
}

// ------------------------------------------------------------------ host side
template <int E>
static cudaError_t pencil_passes_fwd(const PencilArgs& A, float2* send, const float2* tw, cudaStream_t st) {
  const int n = A.N / A.P;
  const int rows = A.B * n;
  static const int rb = getenv("LD_PEN_RB") ? atoi(getenv("LD_PEN_RB")) : 4;   // rows (warps) per CTA (knob)
  pen_rows_fwd<E><<<(rows + rb - 1) / rb, 32 * rb, 0, st>>>(A, send, tw);
  return cudaGetLastError();
}

template <int E>
static cudaError_t pencil_passes_cols(const PencilArgs& A, float2* buf, const float2* tw, const float* ks,
                                      cudaStream_t st) {
  constexpr int N = 32 * E;
  constexpr int CC = N >= 1024 ? 8 : (N >= 512 ? 16 : 32);
  const int m = N / A.P;
  const int cc = m < CC ? m : CC;
  if (cc != CC) return cudaErrorInvalidValue;   // m must be a multiple of CC (P <= N / CC)
  // N = 256: 8 columns per CTA and 4 warps (2048 CTAs at c4, 16 resident per SM: no 1.15-wave tail as
  // with 32 columns per CTA; measured 156 vs 163 us per projection at c4); LD_PEN_CC32=1 restores 32
  static const bool cc8 = getenv("LD_PEN_CC32") == nullptr;
  if (E == 8 && cc8 && m % 8 == 0) {
    const size_t smem8 = sizeof(float2) * ((size_t)8 * (N + 1) + N) + sizeof(float) * N;
    pen_cols<E, 8><<<A.B * (m / 8), 128, smem8, st>>>(A, buf, tw, ks);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(float2) * ((size_t)CC * (N + 1) + N) + sizeof(float) * N;
  pen_cols<E, CC><<<A.B * (m / CC), 256, smem, st>>>(A, buf, tw, ks);
  return cudaGetLastError();
}

template <int E>
static cudaError_t pencil_passes_inv(const PencilArgs& A, const float2* recv, float* p, const float2* tw,
                                     cudaStream_t st) {
  const int n = A.N / A.P;
  const int rows = A.B * n;
  static const int rb = getenv("LD_PEN_RB") ? atoi(getenv("LD_PEN_RB")) : 4;
  pen_rows_inv<E><<<(rows + rb - 1) / rb, 32 * rb, 0, st>>>(A, recv, p, tw);
  return cudaGetLastError();
}

// persistent four-step grids: as many CTAs as fit at once (by shared memory; 512 threads each), at most
// the number of work items
static int grid4(int items, size_t smem) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = (int)((228u * 1024u) / (smem + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);   // 512 threads: at most 4 per SM
  const int g = sms * per_sm;
  return items < g ? items : g;
}

template <int N2>
static cudaError_t pencil4_fwd(const PencilArgs& A, float2* send, const float2* tw, cudaStream_t st) {
  const int n = A.N / A.P;
  static const bool old4 = getenv("LD_PEN4_OLD") != nullptr;
  if (N2 == 64 && !old4 && n % 2 == 0) {   // N = 4096: half-warp FFT rows, two per CTA
    // two CTAs per SM (64 registers, 52 B of spills) by default; LD_PEN4_ROWS_LB1=1: one (128 registers)
    static const bool lb1 = getenv("LD_PEN4_ROWS_LB1") != nullptr;
    if (lb1) pen_rows_fwd_4k_hw<1><<<grid4(A.B * n / 2, cols4k_smem()), 512, cols4k_smem(), st>>>(A, send, tw);
    else pen_rows_fwd_4k_hw<2><<<grid4(A.B * n / 2, cols4k_smem()), 512, cols4k_smem(), st>>>(A, send, tw);
    return cudaGetLastError();
  }
  pen_rows_fwd_4s<N2><<<grid4(A.B * n, smem4_bytes<N2>(1) - sizeof(float) * 64 * N2), 512,
                        smem4_bytes<N2>(1) - sizeof(float) * 64 * N2, st>>>(A, send, tw);
  return cudaGetLastError();
}
template <int N2>
static cudaError_t pencil4_inv(const PencilArgs& A, const float2* recv, float* p, const float2* tw, cudaStream_t st) {
  const int n = A.N / A.P;
  static const bool old4 = getenv("LD_PEN4_OLD") != nullptr;
  if (N2 == 64 && !old4 && n % 2 == 0) {
    static const bool lb1 = getenv("LD_PEN4_ROWS_LB1") != nullptr;
    if (lb1) pen_rows_inv_4k_hw<1><<<grid4(A.B * n / 2, cols4k_smem()), 512, cols4k_smem(), st>>>(A, recv, p, tw);
    else pen_rows_inv_4k_hw<2><<<grid4(A.B * n / 2, cols4k_smem()), 512, cols4k_smem(), st>>>(A, recv, p, tw);
    return cudaGetLastError();
  }
  pen_rows_inv_4s<N2><<<grid4(A.B * n, smem4_bytes<N2>(1) - sizeof(float) * 64 * N2), 512,
                        smem4_bytes<N2>(1) - sizeof(float) * 64 * N2, st>>>(A, recv, p, tw);
  return cudaGetLastError();
}
template <int N2>
static cudaError_t pencil4_cols(const PencilArgs& A, float2* buf, const float2* tw, const float* ks, cudaStream_t st) {
  // 4 columns per CTA (32-B runs per row: whole sectors; 216 KB of shared memory at N = 4096);
  // LD_PEN4_CC2=1 keeps 2 (measurement)
  static const bool cc2 = getenv("LD_PEN4_CC2") != nullptr;
  const int m = A.N / A.P;
  // N = 4096: the half-warp FFT column pass (LD_PEN4_OLD=1 keeps the 64 x 64 shuffle-FFT form)
  static const bool old4 = getenv("LD_PEN4_OLD") != nullptr;
  if (N2 == 64 && !old4 && !cc2 && m % 2 == 0) {
    // one CTA per SM (128 registers); LD_PEN4_COLS_LB2=1: two (64 registers) -- measured slower at c5a
    // (projection 4.65 -> 5.2 ms: the column loads / stores of 4 columns per SM thrash more than the extra
    // warps hide), unlike the row passes
    static const bool lb1 = getenv("LD_PEN4_COLS_LB2") == nullptr;
    if (lb1) pen_cols_4k_hw<1><<<grid4(A.B * (m / 2), cols4k_smem()), 512, cols4k_smem(), st>>>(A, buf, tw, ks);
    else pen_cols_4k_hw<2><<<grid4(A.B * (m / 2), cols4k_smem()), 512, cols4k_smem(), st>>>(A, buf, tw, ks);
    return cudaGetLastError();
  }
  if (!cc2 && m % 4 == 0) {
    pen_cols_4s<N2, 4><<<grid4(A.B * (m / 4), smem4_bytes<N2>(4)), 512, smem4_bytes<N2>(4), st>>>(A, buf, tw, ks);
    return cudaGetLastError();
  }
  constexpr int CC = 2;
  if (m % CC != 0) return cudaErrorInvalidValue;
  pen_cols_4s<N2, CC><<<grid4(A.B * (m / CC), smem4_bytes<N2>(CC)), 512, smem4_bytes<N2>(CC), st>>>(A, buf, tw, ks);
  return cudaGetLastError();
}

#define LD_PENCIL_DISPATCH(fn, fn4, ...)         \
  switch (A.N) {                                 \
    case 256: return fn<8>(__VA_ARGS__);         \
    case 512: return fn<16>(__VA_ARGS__);        \
    case 1024: return fn<32>(__VA_ARGS__);       \
    case 2048: return fn4<32>(__VA_ARGS__);      \
    case 4096: return fn4<64>(__VA_ARGS__);      \
    default: return cudaErrorInvalidValue;       \
  }

cudaError_t pencil_rows_fwd(const PencilArgs& A, float2* send, const float2* tw, cudaStream_t st) {
  LD_PENCIL_DISPATCH(pencil_passes_fwd, pencil4_fwd, A, send, tw, st)
}
cudaError_t pencil_cols(const PencilArgs& A, float2* buf, const float2* tw, const float* ks, cudaStream_t st) {
  LD_PENCIL_DISPATCH(pencil_passes_cols, pencil4_cols, A, buf, tw, ks, st)
}
cudaError_t pencil_rows_inv(const PencilArgs& A, const float2* recv, float* p, const float2* tw, cudaStream_t st) {
  LD_PENCIL_DISPATCH(pencil_passes_inv, pencil4_inv, A, recv, p, tw, st)
}
cudaError_t pencil_correct(const PencilArgs& A, const float* p, const float* pbelow, const float* pabove,
                           long long pstride, float* Uout, int out_rows, int out_row0, cudaStream_t st) {
  const size_t quads = (size_t)A.B * (A.N / A.P) * (A.N / 4);
  pen_correct<<<(unsigned)((quads + 255) / 256), 256, 0, st>>>(A, p, pbelow, pabove, pstride, Uout, out_rows, out_row0);
  return cudaGetLastError();
}

cudaError_t pencil_set_smem_limits() {
  cudaError_t e = cudaSuccess;
  auto setc = [&](auto kern, int N, int CC) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(sizeof(float2) * ((size_t)CC * (N + 1) + N) + sizeof(float) * N));
  };
  setc(pen_cols<8, 32>, 256, 32);
  setc(pen_cols<16, 16>, 512, 16);
  setc(pen_cols<32, 8>, 1024, 8);
  auto set4 = [&](auto kern, size_t bytes) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  };
  set4(pen_rows_fwd_4s<32>, smem4_bytes<32>(1));
  set4(pen_rows_fwd_4s<64>, smem4_bytes<64>(1));
  set4(pen_rows_inv_4s<32>, smem4_bytes<32>(1));
  set4(pen_rows_inv_4s<64>, smem4_bytes<64>(1));
  set4(pen_cols_4s<32, 2>, smem4_bytes<32>(2));
  set4(pen_cols_r2s<4, 8, 4>, cols_r2s_smem<4, 8>());
  set4(pen_cols_r2s<8, 8, 4>, cols_r2s_smem<8, 8>());
  set4(pen_cols_r2s<16, 8, 4>, cols_r2s_smem<16, 8>());
  set4(pen_cols_r2s<32, 4, 4>, cols_r2s_smem<32, 4>());
  set4(pen_inv_correct_r2<4, R2_CORR_R>, inv_corr_smem<4, R2_CORR_R>());
  set4(pen_inv_correct_r2<8, R2_CORR_R>, inv_corr_smem<8, R2_CORR_R>());
  set4(pen_inv_correct_r2<16, R2_CORR_R>, inv_corr_smem<16, R2_CORR_R>());
  set4(pen_inv_correct_r2<32, R2_CORR_R>, inv_corr_smem<32, R2_CORR_R>());
  set4(pen_cols_4s<64, 2>, smem4_bytes<64>(2));
  set4(pen_cols_4s<32, 4>, smem4_bytes<32>(4));
  set4(pen_cols_4s<64, 4>, smem4_bytes<64>(4));
  set4(pen_cols_4k_hw<1>, cols4k_smem());
  set4(pen_cols_4k_hw<2>, cols4k_smem());
  set4(pen_rows_fwd_4k_hw<1>, cols4k_smem());
  set4(pen_rows_fwd_4k_hw<2>, cols4k_smem());
  set4(pen_rows_inv_4k_hw<1>, cols4k_smem());
  set4(pen_rows_inv_4k_hw<2>, cols4k_smem());
  return e;
}

// kernel launches of launch_projection_pencil (the bench's gpu_launches count): the real-data form with
// the fused inverse + correction pass is 3, the other forms 4
int projection_pencil_launches(int N) {
  static const bool c2c = getenv("LD_PROJ_C2C") != nullptr, unfused = getenv("LD_PROJ_UNFUSED") != nullptr;
  return (!c2c && !unfused && (N == 128 || N == 256 || N == 512 || N == 1024)) ? 3 : 4;
}

// Single-domain projection through the pencil passes (P = 1): spec [B][N][N] complex, p [B][N][N].
cudaError_t launch_projection_pencil(const float* Ustar, float* Uout, float2* spec, float* p, int N, int B, float h,
                                     const float2* tw, const float* ksym2, cudaStream_t st) {
  PencilArgs A;
  A.N = N; A.B = B; A.P = 1; A.rank = 0;
  A.half_inv_h = 0.5f / h;
  A.scale = 1.0f / ((float)N * (float)N);
  A.U = Ustar; A.rows = N; A.row0 = 0;
  A.vbelow = Ustar + (size_t)N * N + (size_t)(N - 1) * N;   // v row N-1 of element 0; stride 2 N^2
  A.vabove = Ustar + (size_t)N * N;                          // v row 0
  A.vstride = 2LL * N * N;
  cudaError_t e;
  // real-data form (two real rows per complex transform, N/2 + 1 column transforms) for N = 256 .. 1024;
  // LD_PROJ_C2C=1 keeps the complex passes (measurement knob)
  static const bool c2c = getenv("LD_PROJ_C2C") != nullptr;
  // the inverse row pass fused with the correction (LD_PROJ_UNFUSED=1 keeps the two passes: measurement)
  static const bool unfused = getenv("LD_PROJ_UNFUSED") != nullptr;
  if (!c2c && (N == 128 || N == 256 || N == 512 || N == 1024)) {
    // N = 256: the half-warp FFT passes (LD_PEN_WARPFFT=1 keeps the 32-lane shuffle-FFT passes)
    static const bool warpfft = getenv("LD_PEN_WARPFFT") != nullptr;
    if (N == 256 && !unfused && !warpfft) return projection_n256(A, spec, tw, ksym2, Uout, st);
    float* uo = unfused ? nullptr : Uout;
    e = N == 128 ? projection_r2<4>(A, spec, p, tw, ksym2, st, uo)
                 : (N == 256 ? projection_r2<8>(A, spec, p, tw, ksym2, st, uo)
                             : (N == 512 ? projection_r2<16>(A, spec, p, tw, ksym2, st, uo)
                                         : projection_r2<32>(A, spec, p, tw, ksym2, st, uo)));
    if (e != cudaSuccess || !unfused) return e;
    return pencil_correct(A, p, p + (size_t)(N - 1) * N, p, (long long)N * N, Uout, N, 0, st);
  }
  if ((e = pencil_rows_fwd(A, spec, tw, st)) != cudaSuccess) return e;
  if ((e = pencil_cols(A, spec, tw, ksym2, st)) != cudaSuccess) return e;
  if ((e = pencil_rows_inv(A, spec, p, tw, st)) != cudaSuccess) return e;
  return pencil_correct(A, p, p + (size_t)(N - 1) * N, p, (long long)N * N, Uout, N, 0, st);
}

}  // namespace ld
