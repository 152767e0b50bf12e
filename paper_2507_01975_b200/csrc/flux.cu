// flux.cu -- K2: fused stencil application -> face fluxes -> divergence -> forcing/drag
// -> RK stage combination.
//
// Per cell (i, j) (Eq.4; readings R2, R3, R9, R12):
//   x-face i-1/2 (owned by cell i):  c^x = sum_t wIx[t] c(i-3+t, j),  dc^x = (1/h) sum_t wDx[t] c(i-3+t, j)
//   y-face j-1/2 (owned by cell j):  same with shifts in j and the y stencils
//   F^x_c = gamma u^x c^x - nu dc^x,  F^y_c = gamma v^y c^y - nu dc^y
//   T_c   = -[F^x_c(i+1) - F^x_c(i) + F^y_c(j+1) - F^y_c(j)] / h  (+ f_j - alpha u, - alpha v)
//   out   = a u^n + b X + c dt T + q dt acc (+ e)           (Shu-Osher stage, R13)
//
// Layout: X, u^n, out, acc: planar [B][2][N][N] (y rows, x fastest); stencils w: x-major
// cell-major [B][N(x)][N(y)][24] (channels wIx[6] wDx[6] wIy[6] wDy[6], as the tcgen05 conv
// epilogue writes them: one 96-B run per cell, read as 6 x 16 B); TC term e: [B][N(x)][N(y)][2].
// CTA tile TX x TY cells, one thread per cell.  The stage field with a radius-3 halo (periodic
// wrap) and the stencils of the extra +x / +y face owners are staged once in shared memory;
// every face flux is computed exactly once (conservative) into shared memory.  All global
// loads a thread needs (its stencils, u^n, acc, e) are issued before the first barrier so
// their latencies overlap.
#include <cstdlib>

#include "common.cuh"

namespace ld {


// Tile: TX (x, one lane per column) x TY (y) cells, 256 threads, each thread owns the CPT = TY/8
// cells (tx, ty + 8 j): the per-thread staging and setup are shared by its cells, and all index
// arithmetic is compile-time except the tile origin.
template <int TX, int TY, bool FIXED, bool FNO = false>
__global__ void __launch_bounds__(TX * 8, 2048 / (TX * 8) < 3 ? 2048 / (TX * 8) : 3)
flux_rk_kernel(FluxParams P, StageCoef S, BaseStencil base,
               const float* __restrict__ X, const float* un,
               const float* __restrict__ w, const float* __restrict__ e,
               float* acc, float* out, int write_T, int bulk)
{
  constexpr int NT = TX * 8, CPT = TY / 8;
  constexpr int HX = TX + 6, HY = TY + 6;
  constexpr int WCOL = (TY + 1) * 24;            // floats of one staged stencil column
  extern __shared__ __align__(16) float sm[];
  float* ws = sm;                                // [TX+1][TY+1][24]
  float* us = ws + (TX + 1) * WCOL;              // [2][HY][HX]
  float* Fx = us + 2 * HY * HX;                  // [2][TY][TX+1]
  float* Fy = Fx + 2 * TY * (TX + 1);            // [2][TY+1][TX]

  const int N = P.n, NY = P.ny;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX, y0 = P.y_off + blockIdx.y * TY;   // tile origin in the X / w domain
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const size_t plane = (size_t)N * NY;
  auto wy = [NY](int y) { return y < 0 ? y + NY : (y >= NY ? y - NY : y); };

  // ---- stencils: column cx of the tile (cells y0 .. y0+TY, x0 + cx) is one contiguous
  // (TY+1) x 96-B run of w[b][x][y][24] (split where y0 + TY wraps to 0): thread t copies the
  // 16-B chunks j = t, t + NT, ... of the flattened [TX+1][TY+1][6] chunk grid with cp.async
  // bulk mode: one cp.async.bulk per tile column (its (TY+1) x 96 B are one contiguous run of the
  // x-major stencil layout; two when the +y row wraps), completion on an mbarrier -- 33 copy
  // instructions per tile instead of ~3400 16-B cp.async
  uint64_t* wbar = reinterpret_cast<uint64_t*>(Fy + ((2 * (TY + 1) * TX + 1) & ~1));
  if (!FIXED && bulk) {
    const float* wb = w + (size_t)b * N * NY * 24;
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(wbar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < 32) {
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(wbar);
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((TX + 1) * (TY + 1) * 96)
                     : "memory");
      __syncwarp();
      const int n1 = NY - y0 < TY + 1 ? NY - y0 : TY + 1;   // cells before the periodic wrap in y
      for (int cx = tid; cx < TX + 1; cx += 32) {
        const float* col = wb + (size_t)((x0 + cx) & (N - 1)) * NY * 24;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ws + cx * WCOL);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(col + (size_t)y0 * 24), "r"(n1 * 96), "r"(bar) : "memory");
        if (n1 < TY + 1)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           dst + n1 * 96),
                       "l"(col), "r"((TY + 1 - n1) * 96), "r"(bar) : "memory");
      }
    }
  } else if (!FIXED) {
    constexpr int CH = (TX + 1) * (TY + 1) * 6;
    const float* wb = w + (size_t)b * N * NY * 24;
#pragma unroll 4
    for (int j = tid; j < CH; j += NT) {
      const int cx = j / ((TY + 1) * 6), r = j - cx * ((TY + 1) * 6);
      const int cy = r / 6, q = r - cy * 6;
      const float* src = wb + ((size_t)((x0 + cx) & (N - 1)) * NY + wy(y0 + cy)) * 24 + q * 4;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ws + cx * WCOL + r * 4);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // ---- per-thread loads of the RK combination, issued early
  const int ly0 = blockIdx.y * TY + ty;   // first own row, counted from the first computed row
  float un0[CPT], un1[CPT], ac0[CPT], ac1[CPT], e0[CPT], e1[CPT];
  const bool need_acc = S.q != 0.f || (S.r != 0.f && !S.acc_init);
  const size_t unpl = (size_t)P.un_rows * N, apl = (size_t)P.a_rows * N, opl = (size_t)P.o_rows * N;
  const size_t nbase = (size_t)b * 2 * unpl + (size_t)(P.un_row0 + ly0) * N + x0 + tx;
  const size_t abase = (size_t)b * 2 * apl + (size_t)(P.a_row0 + ly0) * N + x0 + tx;
  const size_t obase = (size_t)b * 2 * opl + (size_t)(P.o_row0 + ly0) * N + x0 + tx;
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    un0[j] = un1[j] = ac0[j] = ac1[j] = e0[j] = e1[j] = 0.f;
    if (!write_T) {
      const size_t o = (size_t)(8 * j) * N;
      if (S.a != 0.f) { un0[j] = un[nbase + o]; un1[j] = un[nbase + o + unpl]; }
      if (need_acc) { ac0[j] = acc[abase + o]; ac1[j] = acc[abase + o + apl]; }
      if (S.add_e) {
        const float2 ee = *reinterpret_cast<const float2*>(e + (((size_t)b * N + x0 + tx) * NY + y0 + ty + 8 * j) * 2);
        e0[j] = ee.x; e1[j] = ee.y;
      }
    }
  }
  // ---- halo tile of the stage field (periodic wrap): rows ty + 8 k, columns tx and tx + TX
  {
    const float* Xb = X + (size_t)b * 2 * plane;
    const int cxa = (x0 - 3 + tx) & (N - 1), cxb = (x0 - 3 + TX + tx) & (N - 1);
#pragma unroll
    for (int k = 0; k < (HY + 7) / 8; ++k) {
      const int ry = ty + 8 * k;
      if (ry < HY) {
        const float* row = Xb + (size_t)wy(y0 - 3 + ry) * N;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          us[(c * HY + ry) * HX + tx] = row[c * plane + cxa];
          if (tx < 6) us[(c * HY + ry) * HX + TX + tx] = row[c * plane + cxb];
        }
      }
    }
  }
  if (!FIXED && bulk) {
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(wbar);
    asm volatile(
        "{\n.reg .pred P1;\nFLX_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@P1 bra FLX_DONE;\nbra FLX_WAIT;\nFLX_DONE:\n}\n" ::"r"(bar)
        : "memory");
  } else if (!FIXED) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();

  // x-face flux of local cell (ly in [0,TY), lx in [0,TX]) with its 6 interp + 6 deriv taps
  auto xface = [&](int ly, int lx) {
    float wv[12];
    if (FIXED) {
#pragma unroll
      for (int t = 0; t < 12; ++t) wv[t] = base.w[t];
    } else {
      const float4* w4 = reinterpret_cast<const float4*>(ws + lx * WCOL + ly * 24);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const float4 v = w4[q];
        wv[4 * q] = v.x; wv[4 * q + 1] = v.y; wv[4 * q + 2] = v.z; wv[4 * q + 3] = v.w;
      }
    }
    const float* u0 = us + (0 * HY + ly + 3) * HX + lx;
    const float* v0 = us + (1 * HY + ly + 3) * HX + lx;
    float uI, uD, vI, vD;
    face_taps2<1>(wv, u0, v0, uI, uD, vI, vD);
    float gu = uD * P.inv_h, gv = vD * P.inv_h;
    if (FNO) {   // NEXT-2 branch at this x-face (channels 0-3)
      const size_t fi = ((size_t)b * 8 * NY + wy(y0 + ly)) * N + ((x0 + lx) & (N - 1));
      const size_t fp = (size_t)NY * N;
      uI += P.fno[fi]; vI += P.fno[fi + fp]; gu += P.fno[fi + 2 * fp]; gv += P.fno[fi + 3 * fp];
    }
    const float adv = P.gamma * uI;
    Fx[(0 * TY + ly) * (TX + 1) + lx] = adv * uI - P.nu * gu;
    Fx[(1 * TY + ly) * (TX + 1) + lx] = adv * vI - P.nu * gv;
  };
  // y-face flux of local cell (ly in [0,TY], lx in [0,TX))
  auto yface = [&](int ly, int lx) {
    float wv[12];
    if (FIXED) {
#pragma unroll
      for (int t = 0; t < 12; ++t) wv[t] = base.w[12 + t];
    } else {
      const float4* w4 = reinterpret_cast<const float4*>(ws + lx * WCOL + ly * 24 + 12);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const float4 v = w4[q];
        wv[4 * q] = v.x; wv[4 * q + 1] = v.y; wv[4 * q + 2] = v.z; wv[4 * q + 3] = v.w;
      }
    }
    const float* u0 = us + (0 * HY + ly) * HX + lx + 3;
    const float* v0 = us + (1 * HY + ly) * HX + lx + 3;
    float uI, uD, vI, vD;
    face_taps2<HX>(wv, u0, v0, uI, uD, vI, vD);
    float gu = uD * P.inv_h, gv = vD * P.inv_h;
    if (FNO) {   // NEXT-2 branch at this y-face (channels 4-7)
      const size_t fp = (size_t)NY * N;
      const size_t fi = ((size_t)b * 8 * NY + wy(y0 + ly)) * N + x0 + lx + 4 * fp;
      uI += P.fno[fi]; vI += P.fno[fi + fp]; gu += P.fno[fi + 2 * fp]; gv += P.fno[fi + 3 * fp];
    }
    const float adv = P.gamma * vI;
    Fy[(0 * (TY + 1) + ly) * TX + lx] = adv * uI - P.nu * gu;
    Fy[(1 * (TY + 1) + ly) * TX + lx] = adv * vI - P.nu * gv;
  };

#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    xface(ty + 8 * j, tx);
    yface(ty + 8 * j, tx);
    if (tx == TX - 1) xface(ty + 8 * j, TX);
  }
  if (ty == 7) yface(TY, tx);
  __syncthreads();

#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int ly = ty + 8 * j;
    float T[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float t = -((Fx[(c * TY + ly) * (TX + 1) + tx + 1] - Fx[(c * TY + ly) * (TX + 1) + tx]) +
                  (Fy[(c * (TY + 1) + ly + 1) * TX + tx] - Fy[(c * (TY + 1) + ly) * TX + tx])) * P.inv_h;
      if (P.forced) {
        if (c == 0) t += P.force_row[P.gy0 + blockIdx.y * TY + ly];
        t -= P.drag * us[(c * HY + ly + 3) * HX + tx + 3];
      }
      T[c] = t;
    }
    const size_t o = (size_t)(8 * j) * N;
    if (write_T) {
      out[obase + o] = T[0];
      out[obase + o + opl] = T[1];
      continue;
    }
    const float unv[2] = {un0[j], un1[j]}, acv[2] = {ac0[j], ac1[j]}, ev[2] = {e0[j], e1[j]};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float v = S.a * unv[c] + S.b * us[(c * HY + ly + 3) * HX + tx + 3] + S.c * P.dt * T[c];
      if (S.q != 0.f) v += S.q * P.dt * acv[c];
      if (S.add_e) v += ev[c];
      if (S.r != 0.f) acc[abase + o + c * apl] = acv[c] + S.r * T[c];
      out[obase + o + c * opl] = v;
    }
  }
}

// Column-mapped K2 (rows % 32 == 0; measurement variant, LD_FLUX_COL=1): a warp is 32 consecutive y cells at one x -- the contiguous
// direction of the stencil layout w[b][x][y][24] -- so every lane loads its own cell's 24 stencil
// weights straight into registers (one contiguous 3-KB run per warp, 96 B in flight per thread, no
// shared-memory staging of w); 8 warps = 8 x columns per CTA.  The stage field's halo tile (38 x 14 x 2
// floats) and the x-face fluxes of the CTA's 9 face columns go through shared memory (7 KB), the +y
// face flux comes from lane + 1 by a shuffle (lane 31 evaluates the face of row y0 + 32 itself).  Every
// face and every cell is evaluated with the same fp32 operations in the same order as flux_rk_kernel
// (and the fused stage kernel), so the results are bitwise identical to them.
template <bool FIXED, bool FNO>
__global__ void __launch_bounds__(256, 4)
flux_col_kernel(FluxParams P, StageCoef S, BaseStencil base, const float* __restrict__ X, const float* un,
                const float* __restrict__ w, const float* __restrict__ e, float* acc, float* out, int write_T) {
  constexpr int TX = 8, TY = 32, HX = TX + 6, HY = TY + 6;
  __shared__ float us[2][HY][HX + 1];
  __shared__ float Fxs[2][TX + 1][TY];
  const int N = P.n, NY = P.ny;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX, y0 = P.y_off + blockIdx.y * TY;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t plane = (size_t)N * NY;
  auto wy = [NY](int y) { return y < 0 ? y + NY : (y >= NY ? y - NY : y); };
  const int x = x0 + wid, ly = blockIdx.y * TY + lane;   // cell column, row counted from the first computed row
  // ---- this cell's stencils (registers), issued first
  float wv[24];
  const size_t wcell = (((size_t)b * N + x) * NY + wy(y0 + lane)) * 24;
  if (FIXED) {
#pragma unroll
    for (int k = 0; k < 24; ++k) wv[k] = base.w[k];
  } else {
    const float4* w4 = reinterpret_cast<const float4*>(w + wcell);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const float4 v = __ldg(w4 + q);
      wv[4 * q] = v.x; wv[4 * q + 1] = v.y; wv[4 * q + 2] = v.z; wv[4 * q + 3] = v.w;
    }
  }
  // ---- RK inputs of this cell
  const bool need_acc = S.q != 0.f || (S.r != 0.f && !S.acc_init);
  const size_t unpl = (size_t)P.un_rows * N, apl = (size_t)P.a_rows * N, opl = (size_t)P.o_rows * N;
  const size_t nidx = (size_t)b * 2 * unpl + (size_t)(P.un_row0 + ly) * N + x;
  const size_t aidx = (size_t)b * 2 * apl + (size_t)(P.a_row0 + ly) * N + x;
  const size_t oidx = (size_t)b * 2 * opl + (size_t)(P.o_row0 + ly) * N + x;
  float unv[2] = {0.f, 0.f}, acv[2] = {0.f, 0.f}, ev[2] = {0.f, 0.f};
  if (!write_T) {
    if (S.a != 0.f) { unv[0] = un[nidx]; unv[1] = un[nidx + unpl]; }
    if (need_acc) { acv[0] = acc[aidx]; acv[1] = acc[aidx + apl]; }
    if (S.add_e) {
      const float2 ee = *reinterpret_cast<const float2*>(e + (((size_t)b * N + x) * NY + y0 + lane) * 2);
      ev[0] = ee.x; ev[1] = ee.y;
    }
  }
  // ---- halo tile of the stage field (periodic wrap)
  {
    const float* Xb = X + (size_t)b * 2 * plane;
    for (int k = threadIdx.x; k < 2 * HY * HX; k += 256) {
      const int c = k / (HY * HX), r = (k / HX) % HY, cx = k % HX;
      us[c][r][cx] = Xb[c * plane + (size_t)wy(y0 - 3 + r) * N + ((x0 - 3 + cx) & (N - 1))];
    }
  }
  __syncthreads();
  // x-face flux through the face owned by local column lx (taps lx .. lx+5 of the halo tile)
  auto xface = [&](const float* wq, int lx, float& Fu, float& Fv) {
    const float* u0 = &us[0][lane + 3][lx];
    const float* v0 = &us[1][lane + 3][lx];
    float uI = 0.f, uD = 0.f, vI = 0.f, vD = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const float uu = u0[t], vv = v0[t];
      uI = fmaf(wq[t], uu, uI); uD = fmaf(wq[6 + t], uu, uD);
      vI = fmaf(wq[t], vv, vI); vD = fmaf(wq[6 + t], vv, vD);
    }
    float gu = uD * P.inv_h, gv = vD * P.inv_h;
    if (FNO) {
      const size_t fi = ((size_t)b * 8 * NY + wy(y0 + lane)) * N + ((x0 + lx) & (N - 1));
      const size_t fp = (size_t)NY * N;
      uI += P.fno[fi]; vI += P.fno[fi + fp]; gu += P.fno[fi + 2 * fp]; gv += P.fno[fi + 3 * fp];
    }
    const float adv = P.gamma * uI;
    Fu = adv * uI - P.nu * gu;
    Fv = adv * vI - P.nu * gv;
  };
  // y-face flux through the face owned by local row lyy of this column (taps lyy .. lyy+5)
  auto yface = [&](const float* wq, int lyy, float& Fu, float& Fv) {
    float uI = 0.f, uD = 0.f, vI = 0.f, vD = 0.f;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const float uu = us[0][lyy + t][wid + 3], vv = us[1][lyy + t][wid + 3];
      uI = fmaf(wq[t], uu, uI); uD = fmaf(wq[6 + t], uu, uD);
      vI = fmaf(wq[t], vv, vI); vD = fmaf(wq[6 + t], vv, vD);
    }
    float gu = uD * P.inv_h, gv = vD * P.inv_h;
    if (FNO) {
      const size_t fp = (size_t)NY * N;
      const size_t fi = ((size_t)b * 8 * NY + wy(y0 + lyy)) * N + x + 4 * fp;
      uI += P.fno[fi]; vI += P.fno[fi + fp]; gu += P.fno[fi + 2 * fp]; gv += P.fno[fi + 3 * fp];
    }
    const float adv = P.gamma * vI;
    Fu = adv * uI - P.nu * gu;
    Fv = adv * vI - P.nu * gv;
  };
  // extra faces (loaded late, only by the threads that need them): warp TX-1 the x-face of column x0 + TX,
  // lane 31 the y-face of row y0 + TY
  float fxu, fxv;
  xface(wv, wid, fxu, fxv);
  Fxs[0][wid][lane] = fxu;
  Fxs[1][wid][lane] = fxv;
  if (wid == TX - 1) {
    float wx2[12];
    if (FIXED) {
#pragma unroll
      for (int k = 0; k < 12; ++k) wx2[k] = base.w[k];
    } else {
      const float4* w4 = reinterpret_cast<const float4*>(w + (((size_t)b * N + ((x0 + TX) & (N - 1))) * NY + wy(y0 + lane)) * 24);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const float4 v = __ldg(w4 + q);
        wx2[4 * q] = v.x; wx2[4 * q + 1] = v.y; wx2[4 * q + 2] = v.z; wx2[4 * q + 3] = v.w;
      }
    }
    float au, av;
    xface(wx2, TX, au, av);
    Fxs[0][TX][lane] = au;
    Fxs[1][TX][lane] = av;
  }
  float fyu, fyv;
  yface(wv + 12, lane, fyu, fyv);
  float nyu = __shfl_down_sync(0xffffffffu, fyu, 1), nyv = __shfl_down_sync(0xffffffffu, fyv, 1);
  if (lane == 31) {
    float wy2[12];
    if (FIXED) {
#pragma unroll
      for (int k = 0; k < 12; ++k) wy2[k] = base.w[12 + k];
    } else {
      const float4* w4 = reinterpret_cast<const float4*>(w + (((size_t)b * N + x) * NY + wy(y0 + TY)) * 24 + 12);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const float4 v = __ldg(w4 + q);
        wy2[4 * q] = v.x; wy2[4 * q + 1] = v.y; wy2[4 * q + 2] = v.z; wy2[4 * q + 3] = v.w;
      }
    }
    yface(wy2, TY, nyu, nyv);
  }
  __syncthreads();
  const float Fy[2] = {fyu, fyv}, Fyn[2] = {nyu, nyv};
  float T[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float t = -((Fxs[c][wid + 1][lane] - Fxs[c][wid][lane]) + (Fyn[c] - Fy[c])) * P.inv_h;
    if (P.forced) {
      if (c == 0) t += P.force_row[P.gy0 + ly];
      t -= P.drag * us[c][lane + 3][wid + 3];
    }
    T[c] = t;
  }
  if (write_T) {
    out[oidx] = T[0];
    out[oidx + opl] = T[1];
    return;
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float v = S.a * unv[c] + S.b * us[c][lane + 3][wid + 3] + S.c * P.dt * T[c];
    if (S.q != 0.f) v += S.q * P.dt * acv[c];
    if (S.add_e) v += ev[c];
    if (S.r != 0.f) acc[aidx + c * apl] = acv[c] + S.r * T[c];
    out[oidx + c * opl] = v;
  }
}

// K2 after the output layer's flux epilogue (conv_xn.cu OUT_FLUX, single domain, N % 32 == 0): the face
// fluxes arrive per cell as F[b][x][y][4] = (F^x_u, F^x_v at i-1/2, F^y_u, F^y_v at j-1/2), so this kernel
// is the divergence, forcing / drag and the Shu-Osher stage only -- per cell-stage it reads F 16 (+ the
// +x / +y neighbours' faces, shared within the tile), U 8, u^n 8 and writes 8 B, instead of K2's 120 B
// (the stencils never reach HBM).  32 x 16 cells per CTA (two per thread: 8 CTAs of 256 threads per SM;
// 32 x 32 with 4 cells per thread needed 62 registers, 4 CTAs per SM: c4 50.5 vs 47.8 us, c3 28.1 vs 26.8);
// the x-major fluxes (and e) are staged in shared
// memory with y along the lanes and read back with x along the lanes, so every global access is
// coalesced.  The same fp32 operations in the same order as flux_rk_kernel.
template <int TYC>
__global__ void __launch_bounds__(256, 8) flux_div_kernel(FluxParams P, StageCoef S, const float* __restrict__ X,
                                                       const float* un, const float4* __restrict__ F,
                                                       const float2* __restrict__ e, float* acc, float* out) {
  constexpr int KC = TYC / 8;      // cells per thread
  __shared__ float4 Fs[33][TYC + 1];   // [x][y], one extra column / row: the +x / +y neighbours' own faces
  __shared__ float2 Es[32][TYC + 1];
  const int N = P.n, b = blockIdx.z, x0 = blockIdx.x * 32, y0 = blockIdx.y * TYC;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const bool need_acc = S.q != 0.f || (S.r != 0.f && !S.acc_init);
  const size_t plane = (size_t)N * N;
  const size_t unpl = (size_t)P.un_rows * N, apl = (size_t)P.a_rows * N, opl = (size_t)P.o_rows * N;
  // every global load of the CTA is issued before the barrier: the fluxes (and e) straight into shared
  // memory by cp.async (no registers held, all in flight together -- the earlier register-staged loop
  // waited out one load latency per iteration), the planar per-cell operands of the thread's cells
  // (x = lane, y = wp + 8 k) into registers
  constexpr int NF = 33 * (TYC + 1), NE = 32 * TYC;
  for (int i = threadIdx.x; i < NF; i += 256) {   // column cx: TYC + 1 consecutive y
    const int cx = i / (TYC + 1), r = i - cx * (TYC + 1);
    const float4* src = F + ((size_t)b * N + ((x0 + cx) & (N - 1))) * N + ((y0 + r) & (N - 1));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(&Fs[cx][r])),
                 "l"(src) : "memory");
  }
  if (S.add_e)
    for (int i = threadIdx.x; i < NE; i += 256) {
      const int cx = i / TYC, r = i - cx * TYC;
      const float2* src = e + ((size_t)b * N + x0 + cx) * N + y0 + r;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(&Es[cx][r])),
                   "l"(src) : "memory");
    }
  asm volatile("cp.async.commit_group;" ::: "memory");
  float xc[KC][2], unv[KC][2], acv[KC][2];
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int gy = y0 + wp + 8 * k, gx = x0 + lane;
    const size_t xi = (size_t)b * 2 * plane + (size_t)gy * N + gx;
    const size_t nbase = (size_t)b * 2 * unpl + (size_t)(P.un_row0 + gy) * N + gx;
    const size_t abase = (size_t)b * 2 * apl + (size_t)(P.a_row0 + gy) * N + gx;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      xc[k][c] = X[xi + c * plane];
      unv[k][c] = S.a != 0.f ? un[nbase + c * unpl] : 0.f;
      acv[k][c] = need_acc ? acc[abase + c * apl] : 0.f;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int ly = wp + 8 * k, gy = y0 + ly, gx = x0 + lane;
    const float4 f = Fs[lane][ly], fxp = Fs[lane + 1][ly], fyp = Fs[lane][ly + 1];
    const float Fx0[2] = {f.x, f.y}, Fx1[2] = {fxp.x, fxp.y}, Fy0[2] = {f.z, f.w}, Fy1[2] = {fyp.z, fyp.w};
    float T[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float t = -((Fx1[c] - Fx0[c]) + (Fy1[c] - Fy0[c])) * P.inv_h;
      if (P.forced) {
        if (c == 0) t += P.force_row[P.gy0 + gy];
        t -= P.drag * xc[k][c];
      }
      T[c] = t;
    }
    const size_t abase = (size_t)b * 2 * apl + (size_t)(P.a_row0 + gy) * N + gx;
    const size_t obase = (size_t)b * 2 * opl + (size_t)(P.o_row0 + gy) * N + gx;
    const float2 ee = S.add_e ? Es[lane][ly] : make_float2(0.f, 0.f);
    const float ev[2] = {ee.x, ee.y};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float v = S.a * unv[k][c] + S.b * xc[k][c] + S.c * P.dt * T[c];
      if (S.q != 0.f) v += S.q * P.dt * acv[k][c];
      if (S.add_e) v += ev[c];
      if (S.r != 0.f) acc[abase + c * apl] = acv[k][c] + S.r * T[c];
      out[obase + c * opl] = v;
    }
  }
}

cudaError_t launch_flux_div(const FluxParams& P, const StageCoef& S, const float* X, const float* un, const float* F,
                            const float* e, float* acc, float* out, cudaStream_t st) {
  if (P.n % 32 != 0 || P.ny != P.n || P.rows != P.n || P.y_off != 0 || P.fno != nullptr) return cudaErrorInvalidValue;
  dim3 grid(P.n / 32, P.n / 16, P.batch);
  flux_div_kernel<16><<<grid, 256, 0, st>>>(P, S, X, un, reinterpret_cast<const float4*>(F),
                                        reinterpret_cast<const float2*>(e), acc, out);
  return cudaGetLastError();
}

template <int TX, int TY>
static size_t flux_smem_bytes() {   // + 16 B: the bulk-copy mbarrier (8-B aligned after Fy)
  return sizeof(float) * ((size_t)(TX + 1) * (TY + 1) * 24 + 2 * (TY + 6) * (TX + 6) + 2 * TY * (TX + 1) +
                          2 * (TY + 1) * TX) + 16;
}

// Dynamic shared-memory limits of every flux_rk_kernel instance, on the CURRENT device (function
// attributes are per device): called by ld_init, errors reported there.
template <int TX, int TY>
static cudaError_t flux_attr_t() {
  const int smem = (int)flux_smem_bytes<TX, TY>();
  cudaError_t e = cudaFuncSetAttribute(flux_rk_kernel<TX, TY, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(flux_rk_kernel<TX, TY, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(flux_rk_kernel<TX, TY, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return e;
}

cudaError_t flux_set_smem_limits() {
  // flux_div_kernel: 13 KB static shared memory per CTA; the maximum carve-out keeps 8 CTAs (64 warps) per
  // SM resident (every thread issues its loads before the barrier)
  cudaError_t e = cudaFuncSetAttribute(flux_div_kernel<16>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) e = flux_attr_t<32, 16>();
  if (e == cudaSuccess) e = flux_attr_t<32, 8>();
  if (e == cudaSuccess) e = flux_attr_t<16, 8>();
  if (e == cudaSuccess) e = flux_attr_t<8, 8>();
  return e;
}

template <int TX, int TY>
static void launch_flux_t(const FluxParams& P, const StageCoef& S, const BaseStencil& bs, const float* X,
                          const float* un, const float* w, const float* e, float* acc, float* out, int write_T,
                          cudaStream_t st) {
  dim3 block(TX, 8), grid(P.n / TX, P.rows / TY, P.batch);
  const size_t smem = flux_smem_bytes<TX, TY>();
  static const int bulk_env = getenv("LD_FLUX_BULK") ? atoi(getenv("LD_FLUX_BULK")) : -1;   // measurement knob
  const int bulk = bulk_env >= 0 ? bulk_env : 0;   // measured slower (c4 151 vs 141 us, c3 80 vs 74): off
  if (w == nullptr)
    flux_rk_kernel<TX, TY, true><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T, 0);
  else if (P.fno != nullptr)
    flux_rk_kernel<TX, TY, false, true><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T, bulk);
  else
    flux_rk_kernel<TX, TY, false><<<grid, block, smem, st>>>(P, S, bs, X, un, w, e, acc, out, write_T, bulk);
}

cudaError_t launch_flux_rk(const FluxParams& P, const StageCoef& S, const float* base24,
                           const float* X, const float* un, const float* w, const float* e,
                           float* acc, float* out, int write_T, cudaStream_t st) {
  BaseStencil bs;
  for (int i = 0; i < 24; ++i) bs.w[i] = base24 ? base24[i] : 0.f;
  // rows per tile: 16 when the computed rows allow it (P.rows is a multiple of 8)
  // (32 x 32 tiles measured slower at c4: 104 KB of smem per CTA leaves 16 warps per SM)
  // column-mapped kernel: measured slower than the staged tile kernel (c4 206 vs 141 us, c3 102 vs 74:
  // the planar u^n / acc / out accesses are strided along a warp), so only with the knob LD_FLUX_COL=1
  static const bool col_env = getenv("LD_FLUX_COL") != nullptr;
  if (col_env && P.n >= 8 && P.rows % 32 == 0) {
    dim3 grid(P.n / 8, P.rows / 32, P.batch);
    if (w == nullptr)
      flux_col_kernel<true, false><<<grid, 256, 0, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
    else if (P.fno != nullptr)
      flux_col_kernel<false, true><<<grid, 256, 0, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
    else
      flux_col_kernel<false, false><<<grid, 256, 0, st>>>(P, S, bs, X, un, w, e, acc, out, write_T);
    return cudaGetLastError();
  }
  static const int ty_env = getenv("LD_FLUX_TY") ? atoi(getenv("LD_FLUX_TY")) : 16;   // measurement knob
  if (P.n >= 32 && P.rows % 16 == 0 && ty_env == 16) launch_flux_t<32, 16>(P, S, bs, X, un, w, e, acc, out, write_T, st);
  else if (P.n >= 32) launch_flux_t<32, 8>(P, S, bs, X, un, w, e, acc, out, write_T, st);
  else if (P.n == 16) launch_flux_t<16, 8>(P, S, bs, X, un, w, e, acc, out, write_T, st);
  else launch_flux_t<8, 8>(P, S, bs, X, un, w, e, acc, out, write_T, st);
  return cudaGetLastError();
}

}  // namespace ld
