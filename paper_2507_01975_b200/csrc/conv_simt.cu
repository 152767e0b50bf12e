// conv_simt.cu -- fp32-exact 3x3 periodic conv layer (SIMT FFMA), the parity mode
// (LD_CONV_FP32) of SURVEY.md §8a rows a1-a2.
//
//   out[b, y, x, o] = phi( bias[o] + sum_{ky,kx,ci} W[ky*3+kx][ci][o] * in[b, y+ky-1, x+kx-1, ci] )
//
// (cross-correlation with circular padding, PAPER.md:246-250 generalised; R6).  The
// last layer has Pi and w_base folded into W/bias at ld_init (R4), so its outputs are
// the constrained stencils w directly (x-major cell-major [B][N(x)][N(y)][24]) plus e ([B][N][N][2]);
// OUT_PLANAR_ALL writes the first co_real channels planar [B][co_real][N][N] (eval entry points).
//
// Tile: 8x8 cells per CTA, each thread owns 4 consecutive cells in x and 8 output
// channels; the (8+2)^2 halo of a 16-channel input chunk and the matching weight
// chunk are staged in shared memory with periodic wrap on load.
#include "common.cuh"

namespace ld {

constexpr int kTile = 8;        // 8x8 output cells per CTA
constexpr int kHalo = kTile + 2;
constexpr int kCiChunk = 16;

enum OutMode { OUT_NHWC = 0, OUT_STENCIL = 1, OUT_PLANAR_ALL = 2 };

template <int CO_PAD, bool IN_PLANAR>
__global__ void __launch_bounds__(16 * (CO_PAD / 8))
conv3x3_simt_kernel(const float* __restrict__ in, int Ci, int N,
                    const float* __restrict__ Wt,    // [9][Ci][CO_PAD]
                    const float* __restrict__ bias,  // [CO_PAD]
                    int act,                         // -1 none, 0 ReLU, 1 GELU
                    int out_mode, int co_real,
                    float* __restrict__ out0,        // NHWC [B][N][N][CO_PAD] or planar w / R
                    float* __restrict__ out1)        // e cell-major [B][N][N][2] (OUT_STENCIL), may be null
{
  __shared__ float in_s[kCiChunk][kHalo][kHalo + 1];
  __shared__ __align__(16) float w_s[9][kCiChunk][CO_PAD];

  const int b = blockIdx.z;
  const int ty0 = blockIdx.y * kTile, tx0 = blockIdx.x * kTile;
  const int cg = threadIdx.x & 15;            // cell group: row r, 4 cells from x0
  const int og = threadIdx.x >> 4;            // output-channel group of 8
  const int r = cg >> 1, x0 = (cg & 1) * 4;
  const int co0 = og * 8;
  const size_t plane = (size_t)N * N;

  float acc[4][8];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int o = 0; o < 8; ++o) acc[c][o] = 0.f;

  for (int ci0 = 0; ci0 < Ci; ci0 += kCiChunk) {
    const int cc = min(kCiChunk, Ci - ci0);
    // ---- stage the periodic halo tile of this channel chunk
    for (int idx = threadIdx.x; idx < cc * kHalo * kHalo; idx += blockDim.x) {
      int ci, cell;
      if (IN_PLANAR) { ci = idx / (kHalo * kHalo); cell = idx % (kHalo * kHalo); }
      else           { cell = idx / cc; ci = idx % cc; }
      const int hy = cell / kHalo, hx = cell % kHalo;
      const int gy = wrap(ty0 - 1 + hy, N), gx = wrap(tx0 - 1 + hx, N);
      float v;
      if (IN_PLANAR) v = in[((size_t)b * Ci + ci0 + ci) * plane + (size_t)gy * N + gx];
      else           v = in[(((size_t)b * N + gy) * N + gx) * Ci + ci0 + ci];
      in_s[ci][hy][hx] = v;
    }
    for (int idx = threadIdx.x; idx < 9 * cc * CO_PAD; idx += blockDim.x) {
      const int o = idx % CO_PAD, ci = (idx / CO_PAD) % cc, tap = idx / (CO_PAD * cc);
      w_s[tap][ci][o] = Wt[((size_t)tap * Ci + ci0 + ci) * CO_PAD + o];
    }
    __syncthreads();
    for (int ci = 0; ci < cc; ++ci) {
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        float xin[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) xin[q] = in_s[ci][r + ky][x0 + q];
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const float4 wa = *reinterpret_cast<const float4*>(&w_s[ky * 3 + kx][ci][co0]);
          const float4 wb = *reinterpret_cast<const float4*>(&w_s[ky * 3 + kx][ci][co0 + 4]);
          const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int o = 0; o < 8; ++o) acc[c][o] = fmaf(xin[c + kx], wv[o], acc[c][o]);
        }
      }
    }
    __syncthreads();
  }

  // ---- epilogue: bias, activation, store
  const int gy = ty0 + r;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int gx = tx0 + x0 + c;
    float v[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      float t = acc[c][o] + bias[co0 + o];
      if (act == 0) t = fmaxf(t, 0.f);
      else if (act == 1) t = gelu_erf(t);
      v[o] = t;
    }
    if (out_mode == OUT_NHWC) {
      float* dst = out0 + (((size_t)b * N + gy) * N + gx) * CO_PAD + co0;
      *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(dst + 4) = make_float4(v[4], v[5], v[6], v[7]);
    } else if (out_mode == OUT_STENCIL) {
      // x-major cell-major stencils w[b][x][y][24] and TC term e[b][x][y][2] (the flux kernel's layout)
      const size_t cell = ((size_t)b * N + gx) * N + gy;
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int co = co0 + o;
        if (co < 24) out0[cell * 24 + co] = v[o];
        else if (out1 && co < co_real) out1[cell * 2 + (co - 24)] = v[o];
      }
    } else {
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int co = co0 + o;
        if (co < co_real) out0[((size_t)b * co_real + co) * plane + (size_t)gy * N + gx] = v[o];
      }
    }
  }
}

// Host launcher.  co_pad must be 32 or 64.
cudaError_t launch_conv_simt(const float* in, bool in_planar, int Ci, int N, int B,
                             const float* Wt, const float* bias, int co_pad, int act,
                             int out_mode, int co_real, float* out0, float* out1,
                             cudaStream_t st) {
  dim3 grid(N / kTile, N / kTile, B);
  if (co_pad == 64) {
    if (in_planar)
      conv3x3_simt_kernel<64, true><<<grid, 128, 0, st>>>(in, Ci, N, Wt, bias, act, out_mode, co_real, out0, out1);
    else
      conv3x3_simt_kernel<64, false><<<grid, 128, 0, st>>>(in, Ci, N, Wt, bias, act, out_mode, co_real, out0, out1);
  } else if (co_pad == 32) {
    if (in_planar)
      conv3x3_simt_kernel<32, true><<<grid, 64, 0, st>>>(in, Ci, N, Wt, bias, act, out_mode, co_real, out0, out1);
    else
      conv3x3_simt_kernel<32, false><<<grid, 64, 0, st>>>(in, Ci, N, Wt, bias, act, out_mode, co_real, out0, out1);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace ld

// ---------------------------------------------------------------------------
// First layer (Ci = 2: the planar velocity field) -> NHWC activations of type T.
// One thread per (cell, 16-channel group): 18 inputs (L1-cached, shared by neighbours),
// 16 x 18 FMAs, 16 activations written as one contiguous 64-B (fp32) / 32-B (fp16) run.
// ---------------------------------------------------------------------------
#include <cuda_fp16.h>

namespace ld {

constexpr int kFirstCells = 2;   // consecutive cells per thread (register budget: 3 CTAs/SM)

template <typename T, int W>
__global__ void __launch_bounds__(256, 3)
conv_first_kernel(const float* __restrict__ u, int N, int B, const float* __restrict__ Wt /*[9][2][W]*/,
                  const float* __restrict__ bias, int act, T* __restrict__ out) {
  // one thread = kFirstCells consecutive cells in x x 16 output channels: every weight
  // float4 read from shared memory feeds 4 * kFirstCells FMAs.
  constexpr int CC = kFirstCells;
  __shared__ __align__(16) float w_s[9 * 2 * W + W];
  for (int i = threadIdx.x; i < 9 * 2 * W; i += blockDim.x) w_s[i] = Wt[i];
  for (int i = threadIdx.x; i < W; i += blockDim.x) w_s[9 * 2 * W + i] = bias[i];
  __syncthreads();
  constexpr int G = W / 16;                        // channel groups per cell
  const size_t plane = (size_t)N * N;
  const size_t total = (size_t)B * (plane / CC) * G;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    // warp-uniform channel group g (weights become shared-memory broadcasts); the 32 lanes
    // of a warp take 32 consecutive cell groups (coalesced loads of u)
    const int g = (int)((t >> 5) % G);
    const size_t quad = ((t >> 5) / G) * 32 + (t & 31);   // CC-cell group index
    const size_t b = quad / (plane / CC), q = quad - b * (plane / CC);
    const int y = (int)(q / (N / CC)), x0 = (int)(q - (size_t)y * (N / CC)) * CC;
    float xin[2][3][CC + 2];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy) {
        const float* row = u + (b * 2 + c) * plane + (size_t)wrap(y + dy - 1, N) * N;
#pragma unroll
        for (int k = 0; k < CC + 2; ++k) xin[c][dy][k] = __ldg(row + wrap(x0 + k - 1, N));
      }
    float acc[CC][16];
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const float bo = w_s[9 * 2 * W + g * 16 + o];
#pragma unroll
      for (int cc = 0; cc < CC; ++cc) acc[cc][o] = bo;
    }
#pragma unroll
    for (int tap = 0; tap < 9; ++tap)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float4* wp = reinterpret_cast<const float4*>(&w_s[(tap * 2 + c) * W + g * 16]);
#pragma unroll
        for (int o4 = 0; o4 < 4; ++o4) {
          const float4 wv = wp[o4];
          const float ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
#pragma unroll
            for (int cc = 0; cc < CC; ++cc)
              acc[cc][4 * o4 + e] = fmaf(xin[c][tap / 3][cc + tap % 3], ww[e], acc[cc][4 * o4 + e]);
        }
      }
#pragma unroll
    for (int cc = 0; cc < CC; ++cc) {
#pragma unroll
      for (int o = 0; o < 16; ++o)
        acc[cc][o] = act == 1 ? gelu_erf(acc[cc][o]) : (act == 0 ? fmaxf(acc[cc][o], 0.f) : acc[cc][o]);
      T* dst = out + ((b * plane + (size_t)y * N + x0 + cc) * W + g * 16);
      if (sizeof(T) == 4) {
        float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int o = 0; o < 4; ++o)
          d[o] = make_float4(acc[cc][4 * o], acc[cc][4 * o + 1], acc[cc][4 * o + 2], acc[cc][4 * o + 3]);
      } else {
        uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          __half2 h[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) h[e] = __floats2half2_rn(acc[cc][8 * o + 2 * e], acc[cc][8 * o + 2 * e + 1]);
          d[o] = *reinterpret_cast<uint4*>(h);
        }
      }
    }
  }
}

cudaError_t launch_conv_first(const float* u, int N, int B, const float* Wt, const float* bias, int width, int act,
                              int f16, void* out, cudaStream_t st) {
  const size_t total = (size_t)B * N * N / kFirstCells * (width / 16);
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (width == 64) {
    if (f16) conv_first_kernel<__half, 64><<<blocks, 256, 0, st>>>(u, N, B, Wt, bias, act, (__half*)out);
    else conv_first_kernel<float, 64><<<blocks, 256, 0, st>>>(u, N, B, Wt, bias, act, (float*)out);
  } else if (width == 32) {
    if (f16) conv_first_kernel<__half, 32><<<blocks, 256, 0, st>>>(u, N, B, Wt, bias, act, (__half*)out);
    else conv_first_kernel<float, 32><<<blocks, 256, 0, st>>>(u, N, B, Wt, bias, act, (float*)out);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace ld
