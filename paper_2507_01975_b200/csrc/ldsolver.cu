// ldsolver.cu -- host side of the C ABI (include/ldsolver.h): validation, workspace
// layout, weight packing (Pi / w_base folding), RK stage sequencing, CUDA-graph replay.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/ldsolver.h"
#include "common.cuh"

namespace ld {
cudaError_t launch_conv_simt(const float* in, bool in_planar, int Ci, int N, int B, const float* Wt,
                             const float* bias, int co_pad, int act, int out_mode, int co_real, float* out0,
                             float* out1, cudaStream_t st);
cudaError_t launch_flux_rk(const FluxParams& P, const StageCoef& S, const float* base24, const float* X,
                           const float* un, const float* w, const float* e, float* acc, float* out, int write_T,
                           cudaStream_t st);
cudaError_t launch_flux_div(const FluxParams& P, const StageCoef& S, const float* X, const float* un, const float* F,
                            const float* e, float* acc, float* out, cudaStream_t st);
cudaError_t launch_projection(const float* Ustar, float* Uout, float2* spec, float* p, int N, int B, float h,
                              const float2* tw, const float* ksym2, cudaStream_t st);
cudaError_t projection_set_smem_limits();
cudaError_t flux_set_smem_limits();
cudaError_t spectral_set_smem_limits();
size_t spectral_smem_bytes(int N, int K);
size_t spectral_smem_bytes_io(int N, int K, int cin, int cout);
cudaError_t launch_spectral_io(const float* u, float* out, int N, int B, int K, int cin, int cout, int out_mode,
                               const float2* M, const float2* tw, cudaStream_t st);
cudaError_t launch_hist_push(float* hist, const float* u, int B, int kc, size_t field_per_elem, cudaStream_t st);
cudaError_t launch_spectral(const float* u, float* out, int N, int B, int K, const float2* M, const float2* tw,
                            cudaStream_t st);
size_t spectral_big_scratch_bytes(int N, int B, int K, int cin, int cout);
cudaError_t launch_spectral_big(const float* u, float* out, int N, int B, int K, int cin, int cout, int out_mode,
                                const float2* M, const float2* tw, void* scratch, cudaStream_t st);
cudaError_t launch_flux_projection(const FluxParams& P, const StageCoef& S, const float* base24, const float* X,
                                   const float* un, const float* w, const float* e, float* acc, float* Uout,
                                   const float2* tw, const float* ksym2, cudaStream_t st);
bool fused_stage_available(int n);
bool projection_uses_pencil(int N, int B);
int projection_pencil_launches(int N);
bool tc_conv_available();
cudaError_t tc_conv_prepare();
cudaError_t launch_conv_tc_ci(const void* in, int Ci, int N, int Ny, int B, const void* Wtc, const float* bias,
                              int co_pad, int f16, int act, int out_mode, int co_real, void* out0, float* out1,
                              cudaStream_t st, const FluxEpi* fe = nullptr);
size_t tc_weight_bytes(int ci, int co_pad, int f16);
cudaError_t launch_conv_tc_fused1(const float* u, const float* W1, const float* b1, int act1, int N, int Ny, int B,
                                  const void* Wtc, const float* bias, int f16, int act, void* out0, cudaStream_t st);
void tc_pack_weights(const float* Wt /*[9][ci][co_pad]*/, int ci, int co_pad, int f16, uint8_t* dst);
cudaError_t launch_conv_first(const float* u, int N, int B, const float* Wt, const float* bias, int width, int act,
                              int f16, void* out, cudaStream_t st);
cudaError_t launch_nonfinite_check(const float* u, size_t n, int step, int* flag, cudaStream_t st);
cudaError_t launch_downsample(const float* fine, int nf, int f, size_t nplanes, float* coarse, cudaStream_t st);
cudaError_t launch_copy_rows(float* dst, int d_step, int d_off, int d_rows, int d_row0, const float* src, int s_step,
                             int s_off, int s_rows, int s_row0, int nplanes, int count, int N, cudaStream_t st);
cudaError_t pencil_rows_fwd(const PencilArgs& A, float2* send, const float2* tw, cudaStream_t st);
cudaError_t pencil_cols(const PencilArgs& A, float2* buf, const float2* tw, const float* ks, cudaStream_t st);
cudaError_t pencil_rows_inv(const PencilArgs& A, const float2* recv, float* p, const float2* tw, cudaStream_t st);
cudaError_t pencil_correct(const PencilArgs& A, const float* p, const float* pbelow, const float* pabove,
                           long long pstride, float* Uout, int out_rows, int out_row0, cudaStream_t st);
// OUT_NHWC: the tcgen05 conv's blocked layout; OUT_FLUX: the output layer writes face fluxes (conv_xn.cu)
enum { OUT_NHWC = 0, OUT_STENCIL = 1, OUT_PLANAR_ALL = 2, OUT_FLUX = 3 };
// NEXT-4 adjoint pieces (adjoint.cu)
cudaError_t adj_fwd_faces(const float* U, const float* R, const float* base24, int N, int B, float inv_h, float nu,
                          float gamma, float* w_out, float* F4, cudaStream_t st);
cudaError_t adj_extract_e(const float* R, int N, int B, float* E, cudaStream_t st);
cudaError_t adj_fwd_combine(const float* F4, const float* U, const float* un, const float* E, int N, int B, float inv_h,
                            int forced, const float* force_row, float drag, float a, float b, float cdt, float ec,
                            float* Tout, float* Y, cudaStream_t st);
cudaError_t adj_bwd_faces(const float* U, const float* w, const float* Tb, const float* eb, int N, int B, float inv_h,
                          float nu, float gamma, float* Fadj, float* Rb, cudaStream_t st);
cudaError_t adj_bwd_gather(const float* Fadj, const float* w, const float* Tb, int N, int B, int forced, float drag,
                           float* Ub, cudaStream_t st);
cudaError_t adj_act(const float* z, float* y, size_t n, int act, int mode, cudaStream_t st);
cudaError_t adj_lin3(float* out, float a, const float* x, float b, const float* y, float c, const float* z, size_t n,
                     cudaStream_t st);
cudaError_t adj_wgrad(const float* H, bool planar, int ci, const float* G, int co_pad, int N, int B, float* Wb, float* bb,
                      cudaStream_t st);
cudaError_t adj_transpose_w(const float* W, int ci, int co_pad, int cout_pad, float* Wt, cudaStream_t st);
cudaError_t adj_pack_grads(const float* Wb, const float* bb, int ci, int co, int co_pad, float* blob, cudaStream_t st);
cudaError_t launch_flux5x4_rk(const FluxParams& P, const StageCoef& S, const float* w80, const float* X, const float* un,
                              float* acc, float* out, int write_T, cudaStream_t st);
cudaError_t launch_scalar_rk(const FluxParams& P, const StageCoef& S, const float* base24, float D, const float* X,
                             const float* w, const float* sX, const float* sn, float* acc, float* out, cudaStream_t st);
}  // namespace ld

using namespace ld;

static thread_local std::string g_err;

static ld_status fail(ld_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
static ld_status cuda_fail(cudaError_t e, const char* where) {
  return fail(LD_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define LD_CUDA(call, where)                           \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

namespace {

struct Layer {
  int ci, co, co_pad;
  size_t w_off, b_off;      // SIMT layout [9][ci][co_pad] + bias[co_pad] (floats, in workspace)
  bool tc;                  // runs on the tcgen05 kernel
  size_t wtc_off;           // tcgen05 operand layout (bytes into the tc weight region)
  size_t wtc_raw_off;       // last layer only: raw (un-folded) weights for ld_eval_net
};

struct Layout {
  size_t total = 0;
  size_t add(size_t bytes) {
    size_t off = total;
    total += (bytes + 255) & ~(size_t)255;
    return off;
  }
};

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// Per half-plane mode k of O_F (NEXT-2): M(k) = Q R_L(k) ... R_1(k), an 8 x 2 complex matrix,
// composed in fp64 from the fp32 blob (R_1 [nm][C][2][2], R_l [nm][C][C][2], Q [8][C]) and rounded
// once.  faces: rows 0-3 times e^{-i pi kx / n} and rows 4-7 times e^{-i pi ky / n} -- the
// operator evaluated half a cell towards -x / -y, i.e. on the x- / y-faces (reading N2-6).
static size_t sp_param_count_io(int K, int L, int C, int cin, int cout) {
  const size_t nm = (size_t)(K + 1) * (2 * K + 1) - K;
  return nm * ((size_t)C * cin * 2 + (size_t)(L - 1) * C * C * 2) + (size_t)cout * C;
}
static void compose_spectral(const float* params, int K, int L, int C, int n, bool faces, std::vector<float2>& hM,
                             int cin = 2, int cout = 8) {
  const size_t nm = (size_t)(K + 1) * (2 * K + 1) - K;
  hM.assign(nm * cout * cin, make_float2(0.f, 0.f));
  const float* Q = params + nm * ((size_t)C * cin * 2 + (size_t)(L - 1) * C * C * 2);
  std::vector<std::complex<double>> cur, nxt;
  size_t m = 0;
  for (int kx = 0; kx <= K; ++kx)
    for (int ky = -K; ky <= K; ++ky) {
      if (kx == 0 && ky < 0) continue;
      cur.assign((size_t)C * cin, 0.0);   // [C][cin]
      const float* r1 = params + m * C * cin * 2;
      for (int o = 0; o < C; ++o)
        for (int i = 0; i < cin; ++i) cur[o * cin + i] = {r1[(o * cin + i) * 2], r1[(o * cin + i) * 2 + 1]};
      for (int l = 1; l < L; ++l) {
        const float* rl = params + nm * C * cin * 2 + (size_t)(l - 1) * nm * C * C * 2 + m * C * C * 2;
        nxt.assign((size_t)C * cin, 0.0);
        for (int o = 0; o < C; ++o)
          for (int i = 0; i < cin; ++i)
            for (int c = 0; c < C; ++c)
              nxt[o * cin + i] += std::complex<double>(rl[(o * C + c) * 2], rl[(o * C + c) * 2 + 1]) * cur[c * cin + i];
        cur.swap(nxt);
      }
      for (int j = 0; j < cout; ++j) {
        std::complex<double> sh = 1.0;
        if (faces) sh = std::polar(1.0, -M_PI * (j < 4 ? kx : ky) / n);
        for (int i = 0; i < cin; ++i) {
          std::complex<double> v = 0.0;
          for (int c = 0; c < C; ++c) v += (double)Q[j * C + c] * cur[c * cin + i];
          v *= sh;
          hM[(m * cout + j) * cin + i] = make_float2((float)v.real(), (float)v.imag());
        }
      }
      ++m;
    }
}

// O_F / history-TC operators too large for the shared-memory cluster kernel run as three global-memory
// passes (spectral.cu "large-N form") with scratch in the workspace
bool fno_big(const ld_config* c) {
  return c->fno_layers > 0 && (c->n > 128 || spectral_smem_bytes(c->n, c->fno_kmax) > 227 * 1024);
}
bool tch_big(const ld_config* c) {
  return c->tc_mode == 1 &&
         (c->n > 64 || spectral_smem_bytes_io(c->n, c->tc_kmax, 2 * c->tc_interval, 2) > 227 * 1024);
}

ld_status validate(const ld_config* c, const ld_dist* d) {
  if (!c) return fail(LD_ERR_INVALID_ARG, "cfg is NULL");
  if (!is_pow2(c->n)) return fail(LD_ERR_UNSUPPORTED, "n must be a power of two (R22)");
  if (c->n < 8 || c->n > 8192) return fail(LD_ERR_INVALID_ARG, "n must be in [8, 8192]");
  if (c->batch < 1) return fail(LD_ERR_INVALID_ARG, "batch must be >= 1");
  if (!(c->length > 0)) return fail(LD_ERR_INVALID_ARG, "length must be > 0");
  if (c->system != LD_SYSTEM_BURGERS && c->system != LD_SYSTEM_NS)
    return fail(LD_ERR_INVALID_ARG, "system must be 0 (Burgers) or 1 (NS)");
  if (!(c->nu >= 0)) return fail(LD_ERR_INVALID_ARG, "nu must be >= 0");
  if (!(c->dt > 0)) return fail(LD_ERR_INVALID_ARG, "dt must be > 0");
  if (c->rk_order < 2 || c->rk_order > 4) return fail(LD_ERR_INVALID_ARG, "rk_order must be 2, 3 or 4");
  if (c->stencil_mode != LD_STENCIL_LEARNED && c->stencil_mode != LD_STENCIL_FIXED && c->stencil_mode != LD_STENCIL_5X4)
    return fail(LD_ERR_INVALID_ARG, "stencil_mode must be 0, 1 or 2");
  if (c->stencil_mode == LD_STENCIL_5X4) {   // the paper's constant 5x4 face kernels
    if (c->tc_head || c->fno_layers > 0 || c->tc_mode != 0 || c->freeze_stencils != 0 || c->scalar_mode != 0)
      return fail(LD_ERR_UNSUPPORTED, "stencil_mode 2 (5x4 kernels): tc_head, fno, tc_mode, freeze, scalar must be off");
    if (d && (d->mode == 2 || d->mode == 3)) return fail(LD_ERR_UNSUPPORTED, "stencil_mode 2 is single-domain");
  }
  if (c->stencil_mode == LD_STENCIL_LEARNED) {
    if (c->n_layers < 2) return fail(LD_ERR_INVALID_ARG, "n_layers must be >= 2");
    if (c->width != 32 && c->width != 64) return fail(LD_ERR_UNSUPPORTED, "width must be 32 or 64");
    if (c->activation != LD_ACT_RELU && c->activation != LD_ACT_GELU)
      return fail(LD_ERR_INVALID_ARG, "activation must be 0 (ReLU) or 1 (GELU)");
  }
  if (c->tc_head != 0 && c->tc_head != 1) return fail(LD_ERR_INVALID_ARG, "tc_head must be 0 or 1");
  if (c->tc_head && c->stencil_mode == LD_STENCIL_FIXED)
    return fail(LD_ERR_INVALID_ARG, "tc_head needs the learned net (stencil_mode 0)");
  if (c->tc_interval < 1) return fail(LD_ERR_INVALID_ARG, "tc_interval must be >= 1");
  if (c->conv_precision != LD_CONV_FP32 && c->conv_precision != LD_CONV_TF32 && c->conv_precision != LD_CONV_F16 &&
      c->conv_precision != LD_CONV_BF16)
    return fail(LD_ERR_INVALID_ARG, "conv_precision must be 0 (fp32), 1 (tf32), 2 (f16) or 3 (bf16)");
  if (c->check_finite_every < 0) return fail(LD_ERR_INVALID_ARG, "check_finite_every must be >= 0");
  if (c->fno_layers < 0) return fail(LD_ERR_INVALID_ARG, "fno_layers must be >= 0");
  if (c->fno_layers > 0) {   // NEXT-2 frequency-domain branch
    if (c->stencil_mode != LD_STENCIL_LEARNED) return fail(LD_ERR_INVALID_ARG, "the fno branch needs stencil_mode 0");
    if (c->fno_width < 1 || c->fno_kmax < 0 || 2 * c->fno_kmax >= c->n)
      return fail(LD_ERR_INVALID_ARG, "fno: width >= 1 and 0 <= kmax < n/2");

    if (d && (d->mode == 2 || d->mode == 3)) return fail(LD_ERR_UNSUPPORTED, "fno branch is single-domain");
  }
  if (c->system == LD_SYSTEM_NS && c->n > 4096)
    return fail(LD_ERR_UNSUPPORTED, "the FFT projection supports n <= 4096 (pencil / four-step transforms)");
  const bool tc_net = c->conv_precision != LD_CONV_FP32 && c->stencil_mode == LD_STENCIL_LEARNED;
  const int net_rows = (d && (d->mode == 2 || d->mode == 3) && d->world > 0) ? c->n / d->world + 16 : c->n;
  if (tc_net && (double)c->batch * c->n * net_rows > (double)(1u << 28))
    return fail(LD_ERR_UNSUPPORTED, "tcgen05 net: at most 2^28 cells (batch * n^2) per handle (32-bit operand "
                                    "offsets); split the batch over handles or ranks");
  if (c->freeze_stencils != 0 && c->freeze_stencils != 1) return fail(LD_ERR_INVALID_ARG, "freeze_stencils must be 0 or 1");
  if (c->tc_mode != 0 && c->tc_mode != 1) return fail(LD_ERR_INVALID_ARG, "tc_mode must be 0 (net head) or 1 (history)");
  if (c->tc_mode == 1) {   // NEXT-3 history block
    if (c->tc_head) return fail(LD_ERR_INVALID_ARG, "tc_mode 1 replaces the net's TC head: tc_head must be 0");
    if (c->tc_layers < 1 || c->tc_width < 1 || c->tc_kmax < 0 || 2 * c->tc_kmax >= c->n)
      return fail(LD_ERR_INVALID_ARG, "tc history: tc_layers, tc_width >= 1 and 0 <= tc_kmax < n/2");
    if ((size_t)c->n * 2 * c->tc_interval * 8 + (size_t)(2 * c->tc_interval + 2) * (2 * c->tc_kmax + 1) * 8 > 227 * 1024)
      return fail(LD_ERR_UNSUPPORTED, "tc history: the mode pass's n x 2k_c inputs exceed shared memory");
    if (d && (d->mode == 2 || d->mode == 3)) return fail(LD_ERR_UNSUPPORTED, "tc history is single-domain");
  }
  if (c->scalar_mode != 0 && c->scalar_mode != 1) return fail(LD_ERR_INVALID_ARG, "scalar_mode must be 0 or 1");
  if (c->scalar_mode == 1) {   // passive scalar (readings S1-S4)
    if (!(c->scalar_diff >= 0)) return fail(LD_ERR_INVALID_ARG, "scalar_diff must be >= 0");
    if (c->fno_layers > 0 || c->tc_mode != 0 || c->freeze_stencils != 0)
      return fail(LD_ERR_UNSUPPORTED, "scalar_mode needs fno_layers = 0, tc_mode = 0, freeze_stencils = 0");
    if (d && (d->mode == 2 || d->mode == 3)) return fail(LD_ERR_UNSUPPORTED, "scalar_mode is single-domain");
  }
  if (d) {
    if (d->mode < 0 || d->mode > 3) return fail(LD_ERR_INVALID_ARG, "dist.mode must be 0, 1, 2 or 3");
    if (d->world < 1 || d->rank < 0 || d->rank >= d->world) return fail(LD_ERR_INVALID_ARG, "bad rank/world");
    if (d->mode == 2 || d->mode == 3) {
      const int P = d->world, N = c->n;
      if (d->mode == 2 && !d->nccl_comm) return fail(LD_ERR_INVALID_ARG, "slab mode 2 needs an NCCL communicator");
      if (c->stencil_mode == LD_STENCIL_LEARNED && c->conv_precision == LD_CONV_FP32)
        return fail(LD_ERR_UNSUPPORTED, "slab decomposition runs the net on the tcgen05 path (conv_precision 1 or 2)");
      if (c->system == LD_SYSTEM_NS && N < 256)
        return fail(LD_ERR_UNSUPPORTED, "slab decomposition: the distributed FFT needs n >= 256");
      if (N % P != 0 || (N / P) % 8 != 0) return fail(LD_ERR_INVALID_ARG, "slab decomposition needs (n / world) % 8 == 0");
      const int cc = N >= 2048 ? 2 : (N >= 1024 ? 8 : (N >= 512 ? 16 : 32));
      if (c->system == LD_SYSTEM_NS && (N / P) % cc != 0)
        return fail(LD_ERR_INVALID_ARG, "slab decomposition: n / world must be a multiple of the column chunk");
      const int L = c->stencil_mode == LD_STENCIL_LEARNED ? c->n_layers : 0;
      const int hlo = L > 3 ? L : 3, hhi_min = L + 1 > 3 ? L + 1 : 3;
      if (N / P < hlo || N / P < hhi_min + 8)
        return fail(LD_ERR_INVALID_ARG, "slab decomposition: slabs thinner than the stencil / net halo");
    }
  }
  return LD_OK;
}

// slab geometry: halo rows below / above the own rows and the extended height (multiple of 8)
static void slab_geometry(const ld_config* c, int P, int& n, int& m, int& hlo, int& hhi, int& next) {
  n = c->n / P;
  m = c->n / P;
  const int L = c->stencil_mode == LD_STENCIL_LEARNED ? c->n_layers : 0;
  hlo = L > 3 ? L : 3;
  const int hhi_min = L + 1 > 3 ? L + 1 : 3;
  next = (n + hlo + hhi_min + 7) / 8 * 8;
  hhi = next - n - hlo;
}

int n_out_of(const ld_config* c) { return 24 + (c->tc_head ? 2 : 0); }

std::vector<Layer> plan_layers(const ld_config* c) {
  std::vector<Layer> L;
  if (c->stencil_mode != LD_STENCIL_LEARNED) return L;
  for (int l = 0; l < c->n_layers; ++l) {
    Layer y{};
    y.ci = l == 0 ? 2 : c->width;
    y.co = l == c->n_layers - 1 ? n_out_of(c) : c->width;
    y.co_pad = y.co <= 32 ? 32 : 64;
    L.push_back(y);
  }
  return L;
}

bool use_tc(const ld_config* c) { return c->conv_precision != LD_CONV_FP32 && c->stencil_mode == LD_STENCIL_LEARNED; }
// 16-bit operand code of the tcgen05 net: 0 none (fp32 activations, TF32 MMA), 1 fp16, 2 bf16
int use_f16(const ld_config* c) {
  if (c->stencil_mode != LD_STENCIL_LEARNED) return 0;
  return c->conv_precision == LD_CONV_F16 ? 1 : (c->conv_precision == LD_CONV_BF16 ? 2 : 0);
}
size_t act_elem(const ld_config* c) { return use_f16(c) ? 2 : 4; }

}  // namespace

// Slab decomposition: rank r owns rows [r n, (r+1) n) of every field.
struct SlabRank {
  float* Uext;            // [B][2][next][N] stage field + halos (rows [Hlo, Hlo+n) are the own rows)
  void* act[2];           // net activations on the N x next extended slab
  float *w, *e;           // [B][N][next][24], [B][N][next][2]
  float *Upre, *Ust[2], *acc;   // [B][2][n][N]
  float2 *send, *recv;    // [P][B][n][m] spectrum blocks (all-to-all buffers)
  float* p;               // [B][n][N]
  float *hs_lo, *hs_hi, *hr_lo, *hr_hi;   // U halos: own first Hhi / last Hlo rows, received Hlo / Hhi rows
  float *r1s[2], *r1r[2];                 // 1-row halos [B][N]: send (to below, to above), recv (from below, above)
};
struct SlabState {
  int P, n, m, Hlo, Hhi, next;
  int rank0, nloc;        // first local rank, local rank contexts (P virtual, 1 with NCCL)
  bool nccl;
  void* comm;             // ncclComm_t
  std::vector<SlabRank> R;
};

struct ld_handle {
  ld_config cfg;
  int dist_mode;
  SlabState* slab;        // modes 2 / 3
  int N, B, n_out;
  size_t plane, field;               // N*N, B*2*N*N floats
  std::vector<Layer> layers;
  // device pointers (all inside the caller's workspace)
  float *U[2], *Upre, *acc, *e, *w, *p, *ubuf, *wts, *raw_last_w, *raw_last_b;
  void* act[2];                      // activations: NHWC (fp32-exact mode) or the tcgen05 blocked layout [B][K-step][x][y][32 B]
  uint8_t* wtc;                      // tcgen05 weight operands
  float2 *spec, *tw;
  float *ksym2, *force_row;
  int* flag;
  float* fno_out;        // NEXT-2 branch on the faces [B][8][N][N] (fno_layers > 0)
  float2 *fno_M, *fno_tw;
  float* hist;           // NEXT-3 ring of the last k_c step inputs [B][k_c][2][N][N] (tc_mode 1)
  float2 *tc_M, *tc_tw;
  float *sS[2], *s_acc;  // passive scalar stage buffers / RK4 accumulator (scalar_mode 1)
  void* sp_scratch;      // large-N O_F / history-TC scratch
  float base24[24];
  float w5x4[80];        // stencil_mode 2: W_P + Pi W_L [axis][op][5][4] (fp64-constrained at ld_init)
  int64_t step;
  bool tc;
  // CUDA graph cache (per add_e flag) keyed by u pointer and stream
  cudaGraphExec_t gexec[2];
  float* g_u[2];
  bool use_graphs;
  cudaStream_t cap_stream;
  int launches_per_step;
  // pipelined host path (ld_rollout_host): batch-chunk views of this handle (same weights / tables,
  // element-offset buffers, own graphs and streams) so the H2D / D2H copies of one chunk overlap the
  // steps of the others; empty when not applicable
  std::vector<ld_handle*> views;
  std::vector<cudaStream_t> view_streams;
  std::vector<cudaEvent_t> view_events;
  std::vector<cudaEvent_t> view_cdone;   // chunk v's steps done (chunk v + 1's steps wait for it)
  bool is_view;
  // kernel-class timing (ld_set_kernel_timing)
  bool timing;
  std::vector<cudaEvent_t> ev_pool;   // pairs (start, end)
  std::vector<int> ev_cls;            // class of each used pair
  size_t ev_used;
};

// NVTX ranges per kernel class / step (SURVEY.md §5 tracing): visible in nsys / ncu timelines; a
// no-op when no tool is attached.  (Under CUDA-graph replay they mark the capture, not each replay.)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
static const char* kClassNames[8] = {"ld:conv_first", "ld:conv_hidden", "ld:conv_last", "ld:flux_rk",
                                     "ld:projection", "ld:flux_proj", "ld:fno", "ld:scalar"};

static void tbegin(ld_handle* H, cudaStream_t st) {
  nvtxRangePushA("ld:kernel");
  if (!H->timing) return;
  if (2 * (H->ev_used + 1) > H->ev_pool.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    H->ev_pool.push_back(a);
    H->ev_pool.push_back(b);
  }
  cudaEventRecord(H->ev_pool[2 * H->ev_used], st);
}
static void tend(ld_handle* H, int cls, cudaStream_t st) {
  nvtxRangePop();
  nvtxMarkA(kClassNames[cls & 7]);
  if (!H->timing) return;
  cudaEventRecord(H->ev_pool[2 * H->ev_used + 1], st);
  if (H->ev_cls.size() <= H->ev_used) H->ev_cls.resize(H->ev_used + 1);
  H->ev_cls[H->ev_used] = cls;
  H->ev_used += 1;
}

static bool is_slab(const ld_dist* d) { return d && (d->mode == 2 || d->mode == 3); }
static int own_rows(const ld_config* c, const ld_dist* d) { return d && d->mode == 2 ? c->n / d->world : c->n; }

// per-rank slab buffer sizes in bytes, in the order SlabRank lists them
static std::vector<size_t> slab_rank_sizes(const ld_config* c, int P) {
  int n, m, hlo, hhi, next;
  slab_geometry(c, P, n, m, hlo, hhi, next);
  const size_t N = c->n, B = c->batch, own = B * 2 * (size_t)n * N * 4;
  const bool learned = c->stencil_mode == LD_STENCIL_LEARNED;
  const size_t act = learned ? B * (size_t)next * N * c->width * act_elem(c) : 256;
  const bool ns = c->system == LD_SYSTEM_NS;
  return {B * 2 * (size_t)next * N * 4, act, act,
          learned ? B * N * next * 24 * 4 : 256, c->tc_head ? B * N * next * 2 * 4 : 256,
          own, own, own, c->rk_order == 4 ? own : 256,
          ns ? B * (size_t)n * N * 8 : 256, ns ? B * (size_t)n * N * 8 : 256, ns ? B * (size_t)n * N * 4 : 256,
          B * 2 * (size_t)hhi * N * 4, B * 2 * (size_t)hlo * N * 4, B * 2 * (size_t)hlo * N * 4, B * 2 * (size_t)hhi * N * 4,
          B * N * 4, B * N * 4, B * N * 4, B * N * 4};
}

static Layout make_layout(const ld_config* c, const ld_dist* d, std::vector<Layer>& layers, size_t offs[32],
                          std::vector<size_t>* slab_offs = nullptr) {
  Layout L;
  const bool slab = is_slab(d);
  const size_t N = c->n, B = c->batch, plane = N * N, field = B * 2 * plane;
  const size_t sd = slab ? 0 : 1;   // single-domain buffers are unused (256 B) in the slab modes
  const size_t ufield = B * 2 * (size_t)own_rows(c, d) * N;
  int k = 0;
  offs[k++] = L.add(sd * field * 4);  // U0
  offs[k++] = L.add(sd * field * 4);  // U1
  offs[k++] = L.add(sd * field * 4);  // Upre
  offs[k++] = L.add(c->rk_order == 4 ? sd * field * 4 : 256);  // acc
  offs[k++] = L.add((c->tc_head || c->tc_mode == 1) ? sd * field * 4 : 256);   // e (TC head or history block)
  offs[k++] = L.add(c->stencil_mode == LD_STENCIL_LEARNED ? sd * B * 24 * plane * 4 : 256);  // w
  const size_t act = c->stencil_mode == LD_STENCIL_LEARNED ? sd * B * plane * (size_t)c->width * act_elem(c) : 256;
  offs[k++] = L.add(act);  // act0
  offs[k++] = L.add(act);  // act1
  offs[k++] = L.add(c->system == LD_SYSTEM_NS ? sd * B * plane * 4 : 256);               // p
  offs[k++] = L.add(c->system == LD_SYSTEM_NS ? sd * B * N * N * 8 : 256);              // spec (complex rows)
  offs[k++] = L.add(ufield * 4);                                                          // ubuf (host path)
  offs[k++] = L.add((N / 2) * 8);                                                   // tw
  offs[k++] = L.add(N * 4);                                                         // ksym2
  offs[k++] = L.add(N * 4);                                                         // force_row
  offs[k++] = L.add(256);                                                           // flag
  {   // NEXT-2 branch: faces [B][8][N][N], composed per-mode matrices, twiddles
    const bool fo = c->fno_layers > 0;
    const size_t nm = (size_t)(c->fno_kmax + 1) * (2 * c->fno_kmax + 1) - c->fno_kmax;
    offs[k++] = L.add(fo ? B * 8 * plane * 4 : 256);
    offs[k++] = L.add(fo ? nm * 16 * 8 : 256);
    offs[k++] = L.add(fo ? N * 8 : 256);
  }
  {   // NEXT-3 history block: ring [B][k_c][2][N][N], composed per-mode 2 x 2k_c matrices, twiddles
    const bool th = c->tc_mode == 1;
    const size_t kc = c->tc_interval;
    const size_t nm = (size_t)(c->tc_kmax + 1) * (2 * c->tc_kmax + 1) - c->tc_kmax;
    offs[k++] = L.add(th ? B * kc * 2 * plane * 4 : 256);
    offs[k++] = L.add(th ? nm * 2 * 2 * kc * 8 : 256);
    offs[k++] = L.add(th ? N * 8 : 256);
  }
  {   // large-N O_F / history-TC scratch (spectral.cu large-N form)
    size_t sc = 256;
    if (fno_big(c)) sc = std::max(sc, spectral_big_scratch_bytes(c->n, c->batch, c->fno_kmax, 2, 8));
    if (tch_big(c)) sc = std::max(sc, spectral_big_scratch_bytes(c->n, c->batch, c->tc_kmax, 2 * c->tc_interval, 2));
    offs[k++] = L.add(sd * sc + (1 - sd) * 256);
  }
  {   // passive scalar: two stage buffers and the RK4 accumulator, [B][N][N] each
    const size_t sc = c->scalar_mode == 1 ? sd * B * plane * 4 : 256;
    offs[k++] = L.add(sc);
    offs[k++] = L.add(sc);
    offs[k++] = L.add(c->scalar_mode == 1 && c->rk_order == 4 ? sc : 256);
  }
  // weights
  size_t wfl = 0, tcb = 0;
  for (size_t l = 0; l < layers.size(); ++l) {
    Layer& y = layers[l];
    y.w_off = wfl; wfl += (size_t)9 * y.ci * y.co_pad;
    y.b_off = wfl; wfl += y.co_pad;
    y.tc = use_tc(c);   // every layer, the first one with its 2 input channels padded to one K-step
    y.wtc_off = y.wtc_raw_off = 0;
    if (y.tc) {
      y.wtc_off = tcb; tcb += (tc_weight_bytes(y.ci, y.co_pad, use_f16(c)) + 255) & ~(size_t)255;
      if (l + 1 == layers.size()) {
        y.wtc_raw_off = tcb; tcb += (tc_weight_bytes(y.ci, y.co_pad, use_f16(c)) + 255) & ~(size_t)255;
      }
    }
  }
  if (!layers.empty()) { wfl += (size_t)9 * layers.back().ci * layers.back().co_pad + layers.back().co_pad; }
  offs[k++] = L.add(wfl * 4 + 256);  // wts (+ raw last layer)
  offs[k++] = L.add(tcb + 256);      // tcgen05 weight operands
  if (slab) {   // per local rank context: mode 3 emulates all P ranks, mode 2 holds its own
    const int nloc = d->mode == 3 ? d->world : 1;
    const std::vector<size_t> sz = slab_rank_sizes(c, d->world);
    for (int r = 0; r < nloc; ++r)
      for (size_t q : sz) {
        const size_t o = L.add(q);
        if (slab_offs) slab_offs->push_back(o);
      }
  }
  return L;
}

// elements per net sub-batch (run_net_step): the per-layer activations of a chunk fit a budget well
// inside the 126 MB L2 (LD_NET_CHUNK_MB).  Measured slower at c4 / c3 (11.97 vs 10.45 ms per step with
// 64 MB chunks: a 4-element launch has ~30 us of fixed prologue / tail against ~20 us of MMAs), so the
// default budget is 0 = the whole batch per launch; kept as a measurement knob.
static int net_chunk_elems(const ld_config* c, bool tc) {
  static const int budget_mb = getenv("LD_NET_CHUNK_MB") ? atoi(getenv("LD_NET_CHUNK_MB")) : 0;
  if (!tc || budget_mb <= 0 || c->stencil_mode != LD_STENCIL_LEARNED) return c->batch;
  const size_t per_elem = (size_t)c->n * c->n * (size_t)c->width * act_elem(c);
  const size_t fit = ((size_t)budget_mb << 20) / per_elem;
  return fit < 1 ? 1 : (fit < (size_t)c->batch ? (int)fit : c->batch);
}

extern "C" ld_status ld_destroy(ld_handle* H);

// Batch-chunk views for the pipelined host path: C chunks of B / C elements, each a shallow copy of the
// handle whose per-element buffers start at its first element (every buffer a view touches is
// element-major), with its own capture stream, graph cache and copy / compute stream.  Only for the
// plain single-domain step (no slab, O_F branch, history TC or scalar) with B % C == 0, N >= 64.
// stream priority of chunk view v in ld_rollout_host: chunk 0 highest, so the interleaved chunks finish
// one after the other (each chunk's copy-out overlaps the later chunks' kernels) while the lower-priority
// chunks' small kernels still fill the gaps of the higher ones (LD_HOST_NO_PRIO=1: all equal, measurement)
static int view_priority(int v) {
  static const bool off = getenv("LD_HOST_NO_PRIO") != nullptr;
  int least = 0, greatest = 0;
  if (off || cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return 0;
  const int p = greatest + v;   // numerically lower = higher priority
  return p > least ? least : p;
}

static ld_status make_views(ld_handle* H) {
  const ld_config& c = H->cfg;
  // small problems (c1 / c2: launch- and latency-bound) lose more to the extra concurrent launches than
  // they gain from the overlap (c2 e2e 2.2e8 with 4 chunks vs 2.8e8 without): pipeline from 2^21 cells
  if (H->slab || c.fno_layers > 0 || c.tc_mode != 0 || c.scalar_mode != 0 || H->N < 64 ||
      (size_t)H->B * H->plane < ((size_t)1 << 21))
    return LD_OK;
  const int C = H->B % 4 == 0 && H->B >= 8 ? 4 : (H->B % 2 == 0 && H->B >= 4 ? 2 : 1);
  if (C == 1) return LD_OK;
  const int nb = H->B / C;
  const size_t plane = H->plane;
  const bool learned = c.stencil_mode == LD_STENCIL_LEARNED;
  for (int v = 0; v < C; ++v) {
    ld_handle* V = new ld_handle(*H);
    V->views.clear(); V->view_streams.clear(); V->view_events.clear(); V->view_cdone.clear();
    V->is_view = true;
    V->timing = false;
    V->ev_pool.clear(); V->ev_cls.clear(); V->ev_used = 0;
    V->gexec[0] = V->gexec[1] = nullptr;
    V->g_u[0] = V->g_u[1] = nullptr;
    V->cap_stream = nullptr;
    const size_t b0 = (size_t)v * nb;
    V->B = nb;
    V->cfg.batch = nb;
    V->field = (size_t)nb * 2 * plane;
    const size_t f2 = b0 * 2 * plane;
    V->U[0] += f2; V->U[1] += f2; V->Upre += f2; V->ubuf += f2;
    if (c.rk_order == 4) V->acc += f2;
    if (c.tc_head) V->e += f2;
    if (learned) {
      V->w += b0 * 24 * plane;
      const size_t ab = b0 * plane * (size_t)c.width * act_elem(&c);
      V->act[0] = (char*)V->act[0] + ab;
      V->act[1] = (char*)V->act[1] + ab;
    }
    if (c.system == LD_SYSTEM_NS) {
      V->p += b0 * plane;
      V->spec += b0 * plane;
    }
    cudaStream_t vs = nullptr;
    cudaEvent_t ve = nullptr, vc = nullptr;
    if (cudaStreamCreateWithFlags(&V->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithPriority(&vs, cudaStreamNonBlocking, view_priority(v)) != cudaSuccess ||
        cudaEventCreateWithFlags(&ve, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&vc, cudaEventDisableTiming) != cudaSuccess) {
      H->views.push_back(V);
      return fail(LD_ERR_CUDA, "ld_init: chunk view streams");
    }
    H->views.push_back(V);
    H->view_streams.push_back(vs);
    H->view_events.push_back(ve);
    H->view_cdone.push_back(vc);
  }
  return LD_OK;
}

extern "C" {

size_t ld_param_count(const ld_config* c) {
  if (validate(c, nullptr) != LD_OK) return 0;
  size_t n = 0;
  for (auto& y : plan_layers(c)) n += (size_t)y.co * 9 * y.ci + y.co;
  if (c->stencil_mode == LD_STENCIL_5X4) n += 80;   // W_L [2 axes][2 ops][5][4]
  if (c->fno_layers > 0) n += ld_spectral_param_count(c->fno_kmax, c->fno_layers, c->fno_width);
  if (c->tc_mode == 1) n += sp_param_count_io(c->tc_kmax, c->tc_layers, c->tc_width, 2 * c->tc_interval, 2);
  return n;
}

ld_status ld_workspace_bytes(const ld_config* c, const ld_dist* d, size_t* out) {
  ld_status s = validate(c, d);
  if (s != LD_OK) return s;
  if (!out) return fail(LD_ERR_INVALID_ARG, "out_bytes is NULL");
  auto layers = plan_layers(c);
  size_t offs[32];
  *out = make_layout(c, d, layers, offs).total;
  return LD_OK;
}

// NEXT-2 branch tables: the per-mode matrices (with the face shifts) from the blob part after the
// conv parameters, and the twiddles e^{-2 pi i m / n}
static cudaError_t upload_tc_hist(ld_handle* H, const ld_config* c, const float* params) {
  if (c->tc_mode != 1) return cudaSuccess;
  size_t off = 0;
  for (auto& y : plan_layers(c)) off += (size_t)y.co * 9 * y.ci + y.co;
  if (c->fno_layers > 0) off += ld_spectral_param_count(c->fno_kmax, c->fno_layers, c->fno_width);
  std::vector<float2> hM, htw(c->n);
  compose_spectral(params + off, c->tc_kmax, c->tc_layers, c->tc_width, c->n, false, hM, 2 * c->tc_interval, 2);
  for (int m = 0; m < c->n; ++m) {
    const double a = -2.0 * M_PI * m / c->n;
    htw[m] = make_float2((float)cos(a), (float)sin(a));
  }
  cudaError_t e = cudaMemcpy(H->tc_M, hM.data(), hM.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(H->tc_tw, htw.data(), htw.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)   // the ring starts empty (zeros); corrections only read it once full
    e = cudaMemset(H->hist, 0, (size_t)c->batch * c->tc_interval * 2 * H->plane * sizeof(float));
  return e;
}

static cudaError_t upload_fno(ld_handle* H, const ld_config* c, const float* params) {
  if (c->fno_layers <= 0) return cudaSuccess;
  size_t nconv = 0;
  for (auto& y : plan_layers(c)) nconv += (size_t)y.co * 9 * y.ci + y.co;
  std::vector<float2> hM, htw(c->n);
  compose_spectral(params + nconv, c->fno_kmax, c->fno_layers, c->fno_width, c->n, true, hM);
  for (int m = 0; m < c->n; ++m) {
    const double a = -2.0 * M_PI * m / c->n;
    htw[m] = make_float2((float)cos(a), (float)sin(a));
  }
  cudaError_t e = cudaMemcpy(H->fno_M, hM.data(), hM.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(H->fno_tw, htw.data(), htw.size() * sizeof(float2), cudaMemcpyHostToDevice);
  return e;
}

ld_status ld_init(const ld_config* c, const ld_dist* d, const float* params, size_t n_params,
                  const double* base_in, void* ws, size_t ws_bytes, ld_handle** out) {
  ld_status s = validate(c, d);
  if (s != LD_OK) return s;
  if (!out) return fail(LD_ERR_INVALID_ARG, "out is NULL");
  if (!ws) return fail(LD_ERR_INVALID_ARG, "workspace is NULL");
  if (((uintptr_t)ws) & 255) return fail(LD_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  const size_t need_params = ld_param_count(c);
  if (c->stencil_mode == LD_STENCIL_LEARNED || need_params > 0) {
    if (!params) return fail(LD_ERR_INVALID_ARG, "params is NULL in learned mode");
    if (n_params != need_params)
      return fail(LD_ERR_INVALID_ARG, "n_params mismatch: got " + std::to_string(n_params) + ", need " +
                                          std::to_string(need_params));
  }
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    return fail(LD_ERR_CUDA, "no CUDA device available (there is no CPU fallback)");
  if (use_tc(c) && !tc_conv_available())
    return fail(LD_ERR_UNSUPPORTED, "tcgen05 conv not available on this device (needs sm_100a)");

  auto layers = plan_layers(c);
  size_t offs[32];
  std::vector<size_t> soffs;
  Layout L = make_layout(c, d, layers, offs, &soffs);
  if (ws_bytes < L.total) return fail(LD_ERR_INVALID_ARG, "workspace too small: need " + std::to_string(L.total));

  ld_handle* H = new ld_handle();
  H->cfg = *c;
  H->dist_mode = d ? d->mode : 0;
  H->slab = nullptr;
  H->N = c->n; H->B = c->batch; H->n_out = n_out_of(c);
  H->plane = (size_t)c->n * c->n;
  H->field = (size_t)c->batch * 2 * own_rows(c, d) * c->n;   // the caller's field (own slab in mode 2)
  if (is_slab(d)) {
    SlabState* S = new SlabState();
    slab_geometry(c, d->world, S->n, S->m, S->Hlo, S->Hhi, S->next);
    S->P = d->world;
    S->nccl = d->mode == 2;
    S->nloc = S->nccl ? 1 : S->P;
    S->rank0 = S->nccl ? d->rank : 0;
    S->comm = d->nccl_comm;
    char* w8s = (char*)ws;
    size_t q = 0;
    for (int r = 0; r < S->nloc; ++r) {
      SlabRank R;
      auto nx = [&]() { return (void*)(w8s + soffs[q++]); };
      R.Uext = (float*)nx(); R.act[0] = nx(); R.act[1] = nx();
      R.w = (float*)nx(); R.e = (float*)nx();
      R.Upre = (float*)nx(); R.Ust[0] = (float*)nx(); R.Ust[1] = (float*)nx(); R.acc = (float*)nx();
      R.send = (float2*)nx(); R.recv = (float2*)nx(); R.p = (float*)nx();
      R.hs_lo = (float*)nx(); R.hs_hi = (float*)nx(); R.hr_lo = (float*)nx(); R.hr_hi = (float*)nx();
      R.r1s[0] = (float*)nx(); R.r1s[1] = (float*)nx(); R.r1r[0] = (float*)nx(); R.r1r[1] = (float*)nx();
      S->R.push_back(R);
    }
    H->slab = S;
  }
  H->layers = layers;
  H->tc = use_tc(c);
  H->step = 0;
  H->gexec[0] = H->gexec[1] = nullptr;
  H->g_u[0] = H->g_u[1] = nullptr;
  H->timing = false;
  H->ev_used = 0;
  H->use_graphs = getenv("LD_NO_GRAPH") == nullptr && !is_slab(d);   // env knob for measurement runs
  H->cap_stream = nullptr;
  char* w8 = (char*)ws;
  int k = 0;
  H->U[0] = (float*)(w8 + offs[k++]);
  H->U[1] = (float*)(w8 + offs[k++]);
  H->Upre = (float*)(w8 + offs[k++]);
  H->acc = (float*)(w8 + offs[k++]);
  H->e = (float*)(w8 + offs[k++]);
  H->w = (float*)(w8 + offs[k++]);
  H->act[0] = (void*)(w8 + offs[k++]);
  H->act[1] = (void*)(w8 + offs[k++]);
  H->p = (float*)(w8 + offs[k++]);
  H->spec = (float2*)(w8 + offs[k++]);
  H->ubuf = (float*)(w8 + offs[k++]);
  H->tw = (float2*)(w8 + offs[k++]);
  H->ksym2 = (float*)(w8 + offs[k++]);
  H->force_row = (float*)(w8 + offs[k++]);
  H->flag = (int*)(w8 + offs[k++]);
  H->fno_out = (float*)(w8 + offs[k++]);
  H->fno_M = (float2*)(w8 + offs[k++]);
  H->fno_tw = (float2*)(w8 + offs[k++]);
  H->hist = (float*)(w8 + offs[k++]);
  H->tc_M = (float2*)(w8 + offs[k++]);
  H->tc_tw = (float2*)(w8 + offs[k++]);
  H->sp_scratch = (void*)(w8 + offs[k++]);
  H->sS[0] = (float*)(w8 + offs[k++]);
  H->sS[1] = (float*)(w8 + offs[k++]);
  H->s_acc = (float*)(w8 + offs[k++]);
  H->wts = (float*)(w8 + offs[k++]);
  H->wtc = (uint8_t*)(w8 + offs[k++]);

  // ---- base stencils (R5) and the constraint projectors (R4)
  double base[24];
  if (base_in) {
    for (int i = 0; i < 24; ++i) base[i] = base_in[i];
  } else {
    for (int i = 0; i < 24; ++i) base[i] = 0.0;
    for (int ax = 0; ax < 2; ++ax) {
      base[ax * 12 + 0 + 2] = 0.5; base[ax * 12 + 0 + 3] = 0.5;     // interp
      base[ax * 12 + 6 + 2] = -1.0; base[ax * 12 + 6 + 3] = 1.0;    // deriv
    }
  }
  for (int i = 0; i < 24; ++i) H->base24[i] = (float)base[i];
  if (c->stencil_mode == LD_STENCIL_5X4) {
    // W = W_P + Pi W_L (reading F2): W_P linear interpolation / central difference on the face-normal line
    // (tangential row b = 2, normal taps a = 1, 2); Pi projects out span{1} (interp) / span{1, s, t} (deriv),
    // s = a - 3/2, t = b - 2 (mutually orthogonal in R^20)
    for (int ax = 0; ax < 2; ++ax)
      for (int op = 0; op < 2; ++op) {
        double r[20], m = 0, ms = 0, mt = 0, ss = 0, tt = 0;
        for (int q = 0; q < 20; ++q) {
          r[q] = params[(ax * 2 + op) * 20 + q];
          const double sq = (q % 4) - 1.5, tq = (q / 4) - 2.0;
          m += r[q]; ms += sq * r[q]; mt += tq * r[q]; ss += sq * sq; tt += tq * tq;
        }
        for (int q = 0; q < 20; ++q) {
          const double sq = (q % 4) - 1.5, tq = (q / 4) - 2.0;
          double wv = r[q] - m / 20.0;
          if (op == 1) wv -= sq * ms / ss + tq * mt / tt;
          if (q == 2 * 4 + 1) wv += op == 0 ? 0.5 : -1.0;   // W_P
          if (q == 2 * 4 + 2) wv += op == 0 ? 0.5 : 1.0;
          H->w5x4[(ax * 2 + op) * 20 + q] = (float)wv;
        }
      }
  }
  double PI_[6][6], PD_[6][6];
  {
    const double s[6] = {-2.5, -1.5, -0.5, 0.5, 1.5, 2.5};
    double ss = 0;
    for (int t = 0; t < 6; ++t) ss += s[t] * s[t];
    for (int a = 0; a < 6; ++a)
      for (int b2 = 0; b2 < 6; ++b2) {
        PI_[a][b2] = (a == b2 ? 1.0 : 0.0) - 1.0 / 6.0;
        PD_[a][b2] = PI_[a][b2] - s[a] * s[b2] / ss;
      }
  }

  // ---- pack weights: blob W[co][ky][kx][ci], b[co] -> [tap][ci][co_pad], bias[co_pad]
  std::vector<float> hw;
  std::vector<uint8_t> htc;
  {
    size_t total_fl = 0, total_tc = 0;
    for (auto& y : layers) {
      total_fl = std::max(total_fl, y.b_off + y.co_pad);
      if (y.tc) total_tc = std::max(total_tc, std::max(y.wtc_off, y.wtc_raw_off) +
                                                  tc_weight_bytes(y.ci, y.co_pad, use_f16(c)));
    }
    htc.assign(total_tc, 0);
    size_t raw_off = total_fl;
    if (!layers.empty()) total_fl += (size_t)9 * layers.back().ci * layers.back().co_pad + layers.back().co_pad;
    hw.assign(total_fl, 0.f);
    size_t off = 0;
    for (size_t l = 0; l < layers.size(); ++l) {
      const Layer& y = layers[l];
      const bool last = l + 1 == layers.size();
      std::vector<double> W((size_t)y.co * 9 * y.ci), bb(y.co);
      for (size_t i = 0; i < W.size(); ++i) W[i] = params[off + i];
      off += W.size();
      for (int i = 0; i < y.co; ++i) bb[i] = params[off + i];
      off += y.co;
      auto put = [&](size_t base_off, size_t bias_off, const std::vector<double>& Wm, const std::vector<double>& bm) {
        for (int co = 0; co < y.co; ++co)
          for (int tap = 0; tap < 9; ++tap)
            for (int ci = 0; ci < y.ci; ++ci)
              hw[base_off + ((size_t)tap * y.ci + ci) * y.co_pad + co] = (float)Wm[((size_t)co * 9 + tap) * y.ci + ci];
        for (int co = 0; co < y.co; ++co) hw[bias_off + co] = (float)bm[co];
      };
      if (last) {
        // raw copy (for ld_eval_net), then fold Pi and w_base into the output layer (exact: linear)
        put(raw_off, raw_off + (size_t)9 * y.ci * y.co_pad, W, bb);
        std::vector<double> Wf(W), bf(bb);
        for (int blk = 0; blk < 4; ++blk) {
          const double(*Pm)[6] = (blk % 2 == 0) ? PI_ : PD_;
          for (int t = 0; t < 6; ++t) {
            const int o = blk * 6 + t;
            double sb = base[o];
            for (int t2 = 0; t2 < 6; ++t2) sb += Pm[t][t2] * bb[blk * 6 + t2];
            bf[o] = sb;
            for (int r = 0; r < 9 * y.ci; ++r) {
              double sw = 0;
              for (int t2 = 0; t2 < 6; ++t2) sw += Pm[t][t2] * W[(size_t)(blk * 6 + t2) * 9 * y.ci + r];
              Wf[(size_t)o * 9 * y.ci + r] = sw;
            }
          }
        }
        put(y.w_off, y.b_off, Wf, bf);
      } else {
        put(y.w_off, y.b_off, W, bb);
      }
      if (y.tc) {
        tc_pack_weights(&hw[y.w_off], y.ci, y.co_pad, use_f16(c), &htc[y.wtc_off]);
        if (last) tc_pack_weights(&hw[raw_off], y.ci, y.co_pad, use_f16(c), &htc[y.wtc_raw_off]);
      }
    }
    H->raw_last_w = layers.empty() ? nullptr : H->wts + raw_off;
    H->raw_last_b = layers.empty() ? nullptr : H->wts + raw_off + (size_t)9 * layers.back().ci * layers.back().co_pad;
  }

  // ---- FFT tables (fp64 -> fp32) and forcing row table
  const int N = c->n;
  std::vector<float2> tw(N / 2);
  std::vector<float> ks(N), fr(N);
  const double h = c->length / N;
  for (int kk = 0; kk < N / 2; ++kk) {
    const double ang = -2.0 * M_PI * kk / N;
    tw[kk] = make_float2((float)cos(ang), (float)sin(ang));
  }
  for (int m = 0; m < N; ++m) {
    const int km = m < N / 2 ? m : m - N;
    double kh = sin(2.0 * M_PI * km / N) / h;
    if (m == 0 || m == N / 2) kh = 0.0;
    ks[m] = (float)(kh * kh);
    fr[m] = (float)(c->force_amp * sin(c->force_k * (m + 0.5) * h));
  }
  cudaError_t e;
  if ((e = cudaMemcpy(H->tw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(H->ksym2, ks.data(), ks.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(H->force_row, fr.data(), fr.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (!hw.empty() && (e = cudaMemcpy(H->wts, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) ||
      (!htc.empty() && (e = cudaMemcpy(H->wtc, htc.data(), htc.size(), cudaMemcpyHostToDevice)) != cudaSuccess) ||
      (e = projection_set_smem_limits()) != cudaSuccess || (e = flux_set_smem_limits()) != cudaSuccess ||
      (e = spectral_set_smem_limits()) != cudaSuccess || (H->tc && (e = tc_conv_prepare()) != cudaSuccess) ||
      (e = upload_fno(H, c, params)) != cudaSuccess || (e = upload_tc_hist(H, c, params)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&H->cap_stream, cudaStreamNonBlocking)) != cudaSuccess) {
    delete H;
    return cuda_fail(e, "ld_init");
  }
  // launches per step: per stage L convs + flux (+4 projection)
  const int nchunk = is_slab(d) ? 1 : (c->batch + net_chunk_elems(c, H->tc) - 1) / net_chunk_elems(c, H->tc);
  int per_stage = (int)layers.size() * nchunk + 1 + (c->fno_layers > 0 ? 1 : 0) + (c->scalar_mode == 1 ? 1 : 0) +
                  (c->system == LD_SYSTEM_NS ? (fused_stage_available(c->n) && c->stencil_mode != LD_STENCIL_5X4
                                                    ? 0 : (projection_uses_pencil(c->n, c->batch) ? projection_pencil_launches(c->n) : 1)) : 0);
  if (is_slab(d))   // per local rank: 3 halo copies + net + flux (+ 2 halo copies + 4 FFT passes + 2 row copies)
    per_stage = (d->mode == 3 ? d->world : 1) * (3 + (int)layers.size() + 1 + (c->system == LD_SYSTEM_NS ? 8 : 0));
  H->launches_per_step = per_stage * c->rk_order;
  H->is_view = false;
  if (getenv("LD_HOST_NO_PIPELINE") == nullptr) {
    const ld_status vs = make_views(H);
    if (vs != LD_OK) {
      ld_destroy(H);
      return vs;
    }
  }
  *out = H;
  g_err.clear();
  return LD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// stage building blocks
// ---------------------------------------------------------------------------
// Net evaluation.  mode OUT_STENCIL: the step's layout (cell-major w [B][N][N][24], e
// [B][N][N][2]); OUT_PLANAR_ALL: planar [B][co_out][N][N] for the eval entry points, with the
// raw (un-folded) last layer when raw is set.
static cudaError_t run_net_on(ld_handle* H, const float* X, int Ny, void* const act_buf[2], float* w_out, float* e_out,
                              bool raw, int out_mode, int co_out, cudaStream_t st, int Bsub = 0) {
  const ld_config& c = H->cfg;
  const int Bn = Bsub > 0 ? Bsub : H->B;   // elements this call evaluates (a sub-batch of the handle's)
  const int act = c.activation == LD_ACT_GELU ? 1 : 0;
  const int f16 = use_f16(&c);   // 0 TF32, 1 fp16, 2 bf16
  const void* in = X;
  int cur = 0;
  // FUSE1 (conv_xn.cu): the second layer recomputes the first in its producer -- measured 14x slower at
  // c4 (8.6 ms vs 0.26 + 0.62 ms: the producer's uncoalesced field reads and FFMA work starve the MMA,
  // and staging the field would add to the shared-memory traffic that bounds the layer), so only with
  // the measurement knob LD_FUSE1=1 (tcgen05 net, >= 3 layers, width 64, Ny % 128 == 0)
  static const bool want_fuse1 = getenv("LD_FUSE1") != nullptr;
  const bool fuse1 = want_fuse1 && H->tc && H->layers.size() >= 3 && H->layers[0].co == 64 && H->layers[1].ci == 64 &&
                     H->layers[1].co == 64 && Ny % 128 == 0 && H->N % 4 == 0;
  for (size_t l = 0; l < H->layers.size(); ++l) {
    const Layer& y = H->layers[l];
    const bool last = l + 1 == H->layers.size();
    if (fuse1 && l == 0) continue;   // computed inside layer 1's producer
    if (fuse1 && l == 1) {
      const Layer& y0 = H->layers[0];
      tbegin(H, st);
      cudaError_t e = launch_conv_tc_fused1(X, H->wts + y0.w_off, H->wts + y0.b_off, act, H->N, Ny, Bn,
                                            H->wtc + y.wtc_off, H->wts + y.b_off, f16, act, act_buf[cur], st);
      tend(H, 0, st);   // kernel-timing class 0: the fused first + second layer
      if (e != cudaSuccess) return e;
      in = act_buf[cur];
      cur ^= 1;
      continue;
    }
    const float* W = H->wts + y.w_off;
    const float* b = H->wts + y.b_off;
    if (last && raw) { W = H->raw_last_w; b = H->raw_last_b; }
    void* o0 = last ? (void*)w_out : act_buf[cur];
    const int mode = last ? out_mode : OUT_NHWC;
    const int co_real = (last && out_mode == OUT_PLANAR_ALL) ? co_out : y.co;
    // OUT_FLUX: the face fluxes of the stage field X the net reads (the physics as in flux_params)
    const FluxEpi fe{X, c.system == LD_SYSTEM_BURGERS ? 0.5f : 1.0f, (float)c.nu, (float)(H->N / c.length)};
    cudaError_t e;
    tbegin(H, st);
    if (l == 0 && !y.tc)
      e = launch_conv_first(X, H->N, Bn, W, b, y.co, act, f16, o0, st);
    else if (y.tc)
      e = launch_conv_tc_ci(in, y.ci, H->N, Ny, Bn, H->wtc + (last && raw ? y.wtc_raw_off : y.wtc_off), b, y.co_pad,
                            f16, last ? -1 : act, mode, co_real, o0, last ? e_out : nullptr, st,
                            mode == OUT_FLUX ? &fe : nullptr);
    else if (mode == OUT_FLUX)
      e = cudaErrorInvalidValue;   // (use_flux_epi requires the tcgen05 output layer)
    else
      e = launch_conv_simt((const float*)in, false, y.ci, H->N, Bn, W, b, y.co_pad, last ? -1 : act, mode, co_real,
                           (float*)o0, last ? e_out : nullptr, st);
    tend(H, l == 0 ? 0 : (last ? 2 : 1), st);
    if (e != cudaSuccess) return e;
    in = o0;
    cur ^= 1;
  }
  return cudaSuccess;
}

static cudaError_t run_net(ld_handle* H, const float* X, float* w_out, float* e_out, bool raw, int out_mode,
                           int co_out, cudaStream_t st) {
  return run_net_on(H, X, H->N, H->act, w_out, e_out, raw, out_mode, co_out, st);
}

// The step's net in L2-sized sub-batches (tcgen05 path, stencil output): the batch is cut into chunks
// whose per-layer activations (nb N^2 width bytes) fit in a budget well inside the 126 MB L2, and each
// chunk runs all L layers before the next starts, so a layer's output is read back by the next layer
// from L2 instead of HBM (c4: 4 elements = 67 MB per layer).  The stencils / e land at the chunk's
// element offset.  LD_NET_CHUNK_MB sets the budget (0: whole batch).
static cudaError_t run_net_step(ld_handle* H, const float* X, float* w_out, float* e_out, cudaStream_t st,
                                int out_mode = OUT_STENCIL) {
  const int nb = net_chunk_elems(&H->cfg, H->tc);
  if (nb >= H->B) return run_net(H, X, w_out, e_out, false, out_mode, 24, st);
  const int per_cell = out_mode == OUT_FLUX ? 4 : 24;
  for (int b0 = 0; b0 < H->B; b0 += nb) {
    const int n = H->B - b0 < nb ? H->B - b0 : nb;
    const cudaError_t e = run_net_on(H, X + (size_t)b0 * 2 * H->plane, H->N, H->act,
                                     w_out + (size_t)b0 * per_cell * H->plane,
                                     e_out ? e_out + (size_t)b0 * 2 * H->plane : nullptr, false, out_mode, 24, st, n);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

static FluxParams flux_params(const ld_handle* H) {
  const ld_config& c = H->cfg;
  FluxParams P;
  P.n = H->N; P.batch = H->B;
  P.h = (float)(c.length / H->N); P.inv_h = (float)(H->N / c.length);
  P.nu = (float)c.nu;
  P.gamma = c.system == LD_SYSTEM_BURGERS ? 0.5f : 1.0f;
  P.dt = (float)c.dt;
  P.drag = (float)c.drag;
  P.forced = (c.force_amp != 0.0 || c.drag != 0.0) ? 1 : 0;
  P.force_row = H->force_row;
  P.ny = H->N; P.y_off = 0; P.rows = H->N; P.gy0 = 0;   // single domain
  P.o_rows = P.un_rows = P.a_rows = H->N;
  P.o_row0 = P.un_row0 = P.a_row0 = 0;
  P.fno = c.fno_layers > 0 ? H->fno_out : nullptr;
  return P;
}

static void stage_coefs(int rk, int s, StageCoef& S) {
  S = StageCoef{0.f, 0.f, 0.f, 0.f, 0.f, 0, 0};
  if (rk == 2) {
    const float a[2] = {1.f, 0.5f}, b[2] = {0.f, 0.5f}, cc[2] = {1.f, 0.5f};
    S.a = a[s]; S.b = b[s]; S.c = cc[s];
  } else if (rk == 3) {
    const float a[3] = {1.f, 0.75f, 1.f / 3.f}, b[3] = {0.f, 0.25f, 2.f / 3.f}, cc[3] = {1.f, 0.25f, 2.f / 3.f};
    S.a = a[s]; S.b = b[s]; S.c = cc[s];
  } else {
    const float cc[4] = {0.5f, 0.5f, 1.f, 1.f / 6.f}, r[4] = {1.f, 2.f, 2.f, 0.f};
    S.a = 1.f; S.b = 0.f; S.c = cc[s]; S.r = r[s]; S.acc_init = s == 0; S.q = s == 3 ? 1.f / 6.f : 0.f;
  }
}

// The output layer applies the stencils itself (conv_xn.cu OUT_FLUX: face fluxes instead of the 24 stencils
// per cell) and K2 shrinks to flux_div_kernel: tcgen05 output layer, learned per-stage stencils, single
// domain with N % 128 == 0 (the 16 strips of a conv tile are one column segment), no O_F branch (its face
// values enter before the flux product) and no passive scalar (which reads the stencils).  LD_FLUX_EPI=0
// keeps the stencil round trip (measurement knob).
static bool use_flux_epi(const ld_handle* H) {
  static const bool off = getenv("LD_FLUX_EPI") != nullptr && atoi(getenv("LD_FLUX_EPI")) == 0;
  const ld_config& c = H->cfg;
  return !off && H->tc && !H->layers.empty() && H->layers.back().tc && c.stencil_mode == LD_STENCIL_LEARNED &&
         !c.freeze_stencils && c.fno_layers == 0 && H->N >= 128 && H->N % 128 == 0;
}

static cudaError_t enqueue_step(ld_handle* H, float* u, bool add_e, cudaStream_t st, float* s_user = nullptr) {
  NvtxRange step_range("ld:step");
  const ld_config& c = H->cfg;
  const bool learned = c.stencil_mode == LD_STENCIL_LEARNED;
  const bool fepi = learned && s_user == nullptr && use_flux_epi(H);
  const bool ns = c.system == LD_SYSTEM_NS;
  const int p = c.rk_order;
  const FluxParams P = flux_params(H);
  const float* X = u;
  if (c.tc_mode == 1) {   // NEXT-3: push this step's input into the ring; at correction steps
                          // e = history operator of the last k_c inputs (TC layout, added at the last stage)
    cudaError_t e0 = launch_hist_push(H->hist, u, H->B, c.tc_interval, 2 * H->plane, st);
    if (e0 == cudaSuccess && add_e)
      e0 = tch_big(&c) ? launch_spectral_big(H->hist, H->e, H->N, H->B, c.tc_kmax, 2 * c.tc_interval, 2, 1, H->tc_M,
                                             H->tc_tw, H->sp_scratch, st)
                       : launch_spectral_io(H->hist, H->e, H->N, H->B, c.tc_kmax, 2 * c.tc_interval, 2, 1, H->tc_M,
                                            H->tc_tw, st);
    if (e0 != cudaSuccess) return e0;
  }
  for (int s = 0; s < p; ++s) {
    const bool last = s == p - 1;
    cudaError_t e;
    if (learned && (s == 0 || !c.freeze_stencils)) {   // frozen: the first stage's stencils serve every stage
      e = run_net_step(H, X, H->w, (s == 0 && add_e && c.tc_mode == 0) ? H->e : nullptr, st,
                       fepi ? OUT_FLUX : OUT_STENCIL);
      if (e != cudaSuccess) return e;
    }
    if (c.fno_layers > 0) {   // NEXT-2: O_F of the stage field on the faces -> H->fno_out (P.fno)
      tbegin(H, st);
      e = fno_big(&c) ? launch_spectral_big(X, H->fno_out, H->N, H->B, c.fno_kmax, 2, 8, 0, H->fno_M, H->fno_tw,
                                            H->sp_scratch, st)
                      : launch_spectral(X, H->fno_out, H->N, H->B, c.fno_kmax, H->fno_M, H->fno_tw, st);
      tend(H, 6, st);
      if (e != cudaSuccess) return e;
    }
    StageCoef S;
    stage_coefs(p, s, S);
    if (s_user) {   // passive scalar: this stage's velocity X and stencils, before X is overwritten
      const float* sX = s == 0 ? s_user : H->sS[(s - 1) & 1];
      float* sout = last ? s_user : H->sS[s & 1];
      tbegin(H, st);
      e = launch_scalar_rk(P, S, H->base24, (float)c.scalar_diff, X, learned ? H->w : nullptr, sX, s_user, H->s_acc,
                           sout, st);
      tend(H, 7, st);
      if (e != cudaSuccess) return e;
    }
    S.add_e = (last && add_e) ? 1 : 0;
    float* next = last ? u : H->U[s & 1];
    float* dest = ns ? H->Upre : next;
    if (c.stencil_mode == LD_STENCIL_5X4) {   // constant 5x4 face kernels, then the projection
      tbegin(H, st);
      e = launch_flux5x4_rk(P, S, H->w5x4, X, u, H->acc, dest, 0, st);
      tend(H, 3, st);
      if (e == cudaSuccess && ns) {
        tbegin(H, st);
        e = launch_projection(H->Upre, next, H->spec, H->p, H->N, H->B, P.h, H->tw, H->ksym2, st);
        tend(H, 4, st);
      }
      if (e != cudaSuccess) return e;
      X = next;
      continue;
    }
    if (ns && !fepi) {   // fused flux + projection (N <= 64): kernel-timing class 5
      tbegin(H, st);
      e = launch_flux_projection(P, S, H->base24, X, u, learned ? H->w : nullptr, H->e, H->acc, next, H->tw,
                                 H->ksym2, st);
      if (e == cudaSuccess) {
        tend(H, 5, st);
        X = next;
        continue;
      }
      if (e != cudaErrorNotSupported) return e;
      (void)cudaGetLastError();
    }
    tbegin(H, st);
    e = fepi ? launch_flux_div(P, S, X, u, H->w, H->e, H->acc, dest, st)
             : launch_flux_rk(P, S, H->base24, X, u, learned ? H->w : nullptr, H->e, H->acc, dest, 0, st);
    tend(H, 3, st);
    if (e != cudaSuccess) return e;
    if (ns) {
      tbegin(H, st);
      e = launch_projection(H->Upre, next, H->spec, H->p, H->N, H->B, P.h, H->tw, H->ksym2, st);
      tend(H, 4, st);
      if (e != cudaSuccess) return e;
    }
    X = next;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Slab decomposition (BASELINE.json c5a).  Rank r owns rows
// [r n, (r+1) n).  Per RK stage:
//   1. halo exchange of the stage field: Hlo rows from rank r-1, Hhi rows from rank r+1 ->
//      extended slab Uext (N x next rows, next = n + Hlo + Hhi, Hlo >= L, Hhi >= L+1 for an
//      L-layer 3x3 net, both >= 3 for the 6-tap stencils);
//   2. the net runs on Uext as a periodic N x next domain: the wrapped edge rows are wrong but
//      every layer only spreads that by one row, so rows [L, next-L), which contain the own rows
//      and the +y face owner row, are exact;
//   3. the fused stencil / flux / RK kernel computes the own rows from Uext;
//   4. (NS) projection by a distributed FFT: 1-row halo of v, row FFTs of the own rows,
//      all-to-all (P blocks of N/P spectrum positions), column FFTs + Poisson divide + inverse,
//      all-to-all back, inverse row FFTs, 1-row halo of p, U = U* - G_c p.
// Transfers go through slab_exchange: NCCL grouped send/recv between processes (mode 2), or
// device-to-device copies between the P emulated rank contexts of one process (mode 3).  Both
// modes run the same pack / exchange / unpack sequence and the same kernels.
// ---------------------------------------------------------------------------
struct XOp {
  int rank, peer, tag;
  void* buf;
  size_t bytes;
  bool send;
};

// Asynchronous NCCL failures (a peer died, a network / NVLink error) surface through
// ncclCommGetAsyncError, not through the enqueue calls: check after every exchange and every slab step.
static ld_status nccl_async_status(ncclComm_t comm, const char* where) {
  ncclResult_t async = ncclSuccess;
  const ncclResult_t q = ncclCommGetAsyncError(comm, &async);
  if (q != ncclSuccess) return fail(LD_ERR_NCCL, std::string(where) + ": ncclCommGetAsyncError: " + ncclGetErrorString(q));
  if (async != ncclSuccess && async != ncclInProgress)
    return fail(LD_ERR_NCCL, std::string(where) + ": asynchronous NCCL error: " + ncclGetErrorString(async));
  return LD_OK;
}

static ld_status slab_exchange(ld_handle* H, std::vector<XOp>& ops, cudaStream_t st) {
  SlabState* S = H->slab;
  if (!S->nccl) {
    for (const XOp& r : ops) {
      if (r.send) continue;
      bool found = false;
      for (const XOp& q : ops)
        if (q.send && q.rank == r.peer && q.peer == r.rank && q.tag == r.tag) {
          if (q.bytes != r.bytes) return fail(LD_ERR_INVALID_ARG, "slab exchange: size mismatch");
          LD_CUDA(cudaMemcpyAsync(r.buf, q.buf, r.bytes, cudaMemcpyDeviceToDevice, st), "slab exchange");
          found = true;
          break;
        }
      if (!found) return fail(LD_ERR_INVALID_ARG, "slab exchange: unmatched receive");
    }
    return LD_OK;
  }
  // NCCL pairs the k-th send from a to b with the k-th receive at b from a: issue in tag order
  std::stable_sort(ops.begin(), ops.end(), [](const XOp& a, const XOp& b) { return a.tag < b.tag; });
  ncclComm_t comm = (ncclComm_t)S->comm;
  ncclResult_t nr = ncclGroupStart();
  for (const XOp& o : ops) {
    if (nr != ncclSuccess) break;
    if (o.send) nr = ncclSend(o.buf, o.bytes / 4, ncclFloat, o.peer, comm, st);
    else nr = ncclRecv(o.buf, o.bytes / 4, ncclFloat, o.peer, comm, st);
  }
  ncclResult_t ne = ncclGroupEnd();
  if (nr != ncclSuccess || ne != ncclSuccess)
    return fail(LD_ERR_NCCL, std::string("slab exchange: ") + ncclGetErrorString(nr != ncclSuccess ? nr : ne));
  return nccl_async_status(comm, "slab exchange");
}

struct FieldView {
  float* p;
  int rows, row0;
};

static ld_status slab_step(ld_handle* H, float* u, bool add_e, cudaStream_t st) {
  NvtxRange step_range("ld:slab_step");
  SlabState* S = H->slab;
  const ld_config& c = H->cfg;
  const int N = H->N, B = H->B, P = S->P, n = S->n, m = S->m, Hlo = S->Hlo, Hhi = S->Hhi, next = S->next;
  const bool learned = c.stencil_mode == LD_STENCIL_LEARNED, ns = c.system == LD_SYSTEM_NS;
  const int pstages = c.rk_order;
  const size_t rowB = (size_t)B * N * 4;   // one row of every element, one channel
  auto uview = [&](int r) { return S->nccl ? FieldView{u, n, 0} : FieldView{u, N, r * n}; };
  auto wrapr = [P](int r) { return (r % P + P) % P; };
  ld_status ls;
  for (int s = 0; s < pstages; ++s) {
    const bool last = s == pstages - 1;
    // ---- 1. halo exchange of the stage field into Uext
    std::vector<XOp> ops;
    for (int i = 0; i < S->nloc; ++i) {
      SlabRank& R = S->R[i];
      const int r = S->rank0 + i;
      const FieldView X = s == 0 ? uview(r) : FieldView{R.Ust[(s - 1) & 1], n, 0};
      LD_CUDA(launch_copy_rows(R.hs_lo, 1, 0, Hhi, 0, X.p, 1, 0, X.rows, X.row0, 2 * B, Hhi, N, st), "slab pack");
      LD_CUDA(launch_copy_rows(R.hs_hi, 1, 0, Hlo, 0, X.p, 1, 0, X.rows, X.row0 + n - Hlo, 2 * B, Hlo, N, st), "slab pack");
      LD_CUDA(launch_copy_rows(R.Uext, 1, 0, next, Hlo, X.p, 1, 0, X.rows, X.row0, 2 * B, n, N, st), "slab own rows");
      ops.push_back({r, wrapr(r - 1), 0, R.hs_lo, 2 * Hhi * rowB, true});
      ops.push_back({r, wrapr(r + 1), 1, R.hs_hi, 2 * Hlo * rowB, true});
      ops.push_back({r, wrapr(r + 1), 0, R.hr_hi, 2 * Hhi * rowB, false});
      ops.push_back({r, wrapr(r - 1), 1, R.hr_lo, 2 * Hlo * rowB, false});
    }
    if ((ls = slab_exchange(H, ops, st)) != LD_OK) return ls;
    for (int i = 0; i < S->nloc; ++i) {
      SlabRank& R = S->R[i];
      LD_CUDA(launch_copy_rows(R.Uext, 1, 0, next, 0, R.hr_lo, 1, 0, Hlo, 0, 2 * B, Hlo, N, st), "slab unpack");
      LD_CUDA(launch_copy_rows(R.Uext, 1, 0, next, Hlo + n, R.hr_hi, 1, 0, Hhi, 0, 2 * B, Hhi, N, st), "slab unpack");
    }
    // ---- 2. net on the extended slab, 3. stencils / fluxes / RK on the own rows
    StageCoef SC;
    stage_coefs(pstages, s, SC);
    SC.add_e = (last && add_e) ? 1 : 0;
    for (int i = 0; i < S->nloc; ++i) {
      SlabRank& R = S->R[i];
      const int r = S->rank0 + i;
      if (learned) LD_CUDA(run_net_on(H, R.Uext, next, R.act, R.w, (s == 0 && add_e) ? R.e : nullptr, false,
                                      OUT_STENCIL, 24, st), "slab net");
      FluxParams F = flux_params(H);
      F.ny = next; F.y_off = Hlo; F.rows = n; F.gy0 = r * n;
      const FieldView un = uview(r);
      F.un_rows = un.rows; F.un_row0 = un.row0;
      F.a_rows = n; F.a_row0 = 0;
      FieldView out = ns ? FieldView{R.Upre, n, 0} : (last ? uview(r) : FieldView{R.Ust[s & 1], n, 0});
      F.o_rows = out.rows; F.o_row0 = out.row0;
      tbegin(H, st);
      LD_CUDA(launch_flux_rk(F, SC, H->base24, R.Uext, un.p, learned ? R.w : nullptr, R.e, R.acc, out.p, 0, st),
              "slab flux");
      tend(H, 3, st);
    }
    if (!ns) continue;
    // ---- 4. distributed FFT projection
    auto pargs = [&](SlabRank& R, int r) {
      PencilArgs A;
      A.N = N; A.B = B; A.P = P; A.rank = r;
      A.half_inv_h = (float)(0.5 * N / c.length);
      A.scale = 1.0f / ((float)N * (float)N);
      A.U = R.Upre; A.rows = n; A.row0 = 0;
      A.vbelow = R.r1r[0]; A.vabove = R.r1r[1]; A.vstride = N;
      return A;
    };
    tbegin(H, st);   // kernel-timing class 4: the whole distributed projection (exchanges included)
    ops.clear();
    for (int i = 0; i < S->nloc; ++i) {   // v rows 0 and n-1 of U* to the neighbours
      SlabRank& R = S->R[i];
      const int r = S->rank0 + i;
      LD_CUDA(launch_copy_rows(R.r1s[0], 1, 0, 1, 0, R.Upre, 2, 1, n, 0, B, 1, N, st), "slab pack v");
      LD_CUDA(launch_copy_rows(R.r1s[1], 1, 0, 1, 0, R.Upre, 2, 1, n, n - 1, B, 1, N, st), "slab pack v");
      ops.push_back({r, wrapr(r - 1), 2, R.r1s[0], rowB, true});
      ops.push_back({r, wrapr(r + 1), 3, R.r1s[1], rowB, true});
      ops.push_back({r, wrapr(r + 1), 2, R.r1r[1], rowB, false});
      ops.push_back({r, wrapr(r - 1), 3, R.r1r[0], rowB, false});
    }
    if ((ls = slab_exchange(H, ops, st)) != LD_OK) return ls;
    const size_t blk = (size_t)B * n * m * sizeof(float2);
    ops.clear();
    for (int i = 0; i < S->nloc; ++i) {
      SlabRank& R = S->R[i];
      const int r = S->rank0 + i;
      LD_CUDA(pencil_rows_fwd(pargs(R, r), R.send, H->tw, st), "slab rows fwd");
      for (int q = 0; q < P; ++q) {
        ops.push_back({r, q, 10, (char*)R.send + q * blk, blk, true});
        ops.push_back({r, q, 10, (char*)R.recv + q * blk, blk, false});
      }
    }
    if ((ls = slab_exchange(H, ops, st)) != LD_OK) return ls;
    ops.clear();
    for (int i = 0; i < S->nloc; ++i) {
      SlabRank& R = S->R[i];
      const int r = S->rank0 + i;
      LD_CUDA(pencil_cols(pargs(R, r), R.recv, H->tw, H->ksym2, st), "slab cols");
      for (int q = 0; q < P; ++q) {
        ops.push_back({r, q, 11, (char*)R.recv + q * blk, blk, true});
        ops.push_back({r, q, 11, (char*)R.send + q * blk, blk, false});
      }
    }
    if ((ls = slab_exchange(H, ops, st)) != LD_OK) return ls;
    ops.clear();
    for (int i = 0; i < S->nloc; ++i) {
      SlabRank& R = S->R[i];
      const int r = S->rank0 + i;
      LD_CUDA(pencil_rows_inv(pargs(R, r), R.send, R.p, H->tw, st), "slab rows inv");
      LD_CUDA(launch_copy_rows(R.r1s[0], 1, 0, 1, 0, R.p, 1, 0, n, 0, B, 1, N, st), "slab pack p");
      LD_CUDA(launch_copy_rows(R.r1s[1], 1, 0, 1, 0, R.p, 1, 0, n, n - 1, B, 1, N, st), "slab pack p");
      ops.push_back({r, wrapr(r - 1), 4, R.r1s[0], rowB, true});
      ops.push_back({r, wrapr(r + 1), 5, R.r1s[1], rowB, true});
      ops.push_back({r, wrapr(r + 1), 4, R.r1r[1], rowB, false});
      ops.push_back({r, wrapr(r - 1), 5, R.r1r[0], rowB, false});
    }
    if ((ls = slab_exchange(H, ops, st)) != LD_OK) return ls;
    for (int i = 0; i < S->nloc; ++i) {
      SlabRank& R = S->R[i];
      const int r = S->rank0 + i;
      const FieldView out = last ? uview(r) : FieldView{R.Ust[s & 1], n, 0};
      LD_CUDA(pencil_correct(pargs(R, r), R.p, R.r1r[0], R.r1r[1], N, out.p, out.rows, out.row0, st), "slab correct");
    }
    tend(H, 4, st);
  }
  return LD_OK;
}

// One step as a replayed CUDA graph: the ~20-70 launches of a step are captured once per
// (field pointer, add_e) and replayed with a single cudaGraphLaunch (launch-latency bound
// configs c1/c2).  Kernel-timing mode bypasses the graph so every launch gets its events.
static cudaError_t launch_step(ld_handle* H, float* u, bool add_e, cudaStream_t st) {
  if (H->timing || !H->use_graphs) return enqueue_step(H, u, add_e, st);
  const int g = add_e ? 1 : 0;
  if (H->gexec[g] == nullptr || H->g_u[g] != u) {
    if (H->gexec[g]) {
      cudaGraphExecDestroy(H->gexec[g]);
      H->gexec[g] = nullptr;
    }
    cudaStreamCaptureStatus cs;
    cudaError_t e = cudaStreamIsCapturing(st, &cs);
    if (e != cudaSuccess) return e;
    if (cs != cudaStreamCaptureStatusNone) return enqueue_step(H, u, add_e, st);   // caller is capturing
    cudaStream_t cap = H->cap_stream;
    if ((e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return e;
    cudaError_t e2 = enqueue_step(H, u, add_e, cap);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(cap, &graph);
    if (e2 != cudaSuccess) return e2;
    if (e != cudaSuccess) return e;
    e = cudaGraphInstantiate(&H->gexec[g], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return e;
    H->g_u[g] = u;
  }
  return cudaGraphLaunch(H->gexec[g], st);
}

// Slab steps as CUDA graphs too (the ~100 launches, copies and NCCL group calls of a slab step per rank
// replayed with one cudaGraphLaunch; NCCL point-to-point calls are capturable): captured per (field
// pointer, add_e) like launch_step; LD_SLAB_NO_GRAPH=1 launches eagerly.
static ld_status slab_launch(ld_handle* H, float* u, bool add_e, cudaStream_t st) {
  static const bool no_graph = getenv("LD_SLAB_NO_GRAPH") != nullptr;
  if (H->timing || no_graph || getenv("LD_NO_GRAPH") != nullptr) return slab_step(H, u, add_e, st);
  const int g = add_e ? 1 : 0;
  if (H->gexec[g] == nullptr || H->g_u[g] != u) {
    if (H->gexec[g]) {
      cudaGraphExecDestroy(H->gexec[g]);
      H->gexec[g] = nullptr;
    }
    cudaStreamCaptureStatus cs;
    LD_CUDA(cudaStreamIsCapturing(st, &cs), "slab graph");
    if (cs != cudaStreamCaptureStatusNone) return slab_step(H, u, add_e, st);   // caller is capturing
    cudaStream_t cap = H->cap_stream;
    LD_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "slab graph capture");
    const ld_status ls = slab_step(H, u, add_e, cap);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cap, &graph);
    if (ls != LD_OK) {
      if (graph) cudaGraphDestroy(graph);
      return ls;
    }
    LD_CUDA(e, "slab graph capture");
    const cudaError_t ei = cudaGraphInstantiate(&H->gexec[g], graph, 0);
    cudaGraphDestroy(graph);
    LD_CUDA(ei, "slab graph instantiate");
    H->g_u[g] = u;
  }
  LD_CUDA(cudaGraphLaunch(H->gexec[g], st), "slab graph launch");
  if (H->slab->nccl) return nccl_async_status((ncclComm_t)H->slab->comm, "slab step");
  return LD_OK;
}

static ld_status do_steps(ld_handle* H, float* u, int n, float* traj, int save_every, cudaStream_t st,
                          float* s_user = nullptr) {
  const ld_config& c = H->cfg;
  if ((c.scalar_mode == 1) != (s_user != nullptr))
    return fail(LD_ERR_INVALID_ARG, c.scalar_mode == 1 ? "scalar_mode handle: use ld_step_scalar / ld_rollout_scalar"
                                                        : "ld_step_scalar needs a scalar_mode = 1 handle");
  const bool check = c.check_finite_every > 0;
  if (check) LD_CUDA(cudaMemsetAsync(H->flag, 0x7f, sizeof(int), st), "ld_rollout");
  for (int k = 0; k < n; ++k) {
    const bool add_e = (c.tc_head || c.tc_mode == 1) && ((H->step + 1) % c.tc_interval == 0);
    if (H->slab) {
      const ld_status ls = slab_launch(H, u, add_e, st);
      if (ls != LD_OK) return ls;
    } else {
      cudaError_t e = s_user ? enqueue_step(H, u, add_e, st, s_user) : launch_step(H, u, add_e, st);
      if (e != cudaSuccess) return cuda_fail(e, "ld_step");
    }
    H->step += 1;
    if (traj && save_every > 0 && (k + 1) % save_every == 0) {
      float* dst = traj + (size_t)((k + 1) / save_every - 1) * H->field;
      LD_CUDA(cudaMemcpyAsync(dst, u, H->field * 4, cudaMemcpyDeviceToDevice, st), "ld_rollout snapshot");
    }
    if (check && ((k + 1) % c.check_finite_every == 0 || k + 1 == n)) {
      const cudaError_t e = launch_nonfinite_check(u, H->field, (int)(H->step - 1), H->flag, st);
      if (e != cudaSuccess) return cuda_fail(e, "ld_rollout finite check");
    }
  }
  if (check) {
    int bad = 0;
    LD_CUDA(cudaMemcpyAsync(&bad, H->flag, sizeof(int), cudaMemcpyDeviceToHost, st), "ld_rollout");
    LD_CUDA(cudaStreamSynchronize(st), "ld_rollout");
    if (bad != 0x7f7f7f7f)
      return fail(LD_ERR_NONFINITE, "simulation diverged: non-finite field at step " + std::to_string(bad));
  }
  return LD_OK;
}

extern "C" {

ld_status ld_step(ld_handle* H, float* u, void* stream) {
  if (!H || !u) return fail(LD_ERR_INVALID_ARG, "ld_step: NULL handle or field");
  return do_steps(H, u, 1, nullptr, 0, (cudaStream_t)stream);
}

ld_status ld_rollout(ld_handle* H, float* u, int32_t n, float* traj, int32_t save_every, void* stream) {
  if (!H || !u) return fail(LD_ERR_INVALID_ARG, "ld_rollout: NULL handle or field");
  if (n < 0) return fail(LD_ERR_INVALID_ARG, "n_steps must be >= 0");
  if (traj && save_every < 1) return fail(LD_ERR_INVALID_ARG, "save_every must be >= 1 with traj");
  return do_steps(H, u, n, traj, save_every, (cudaStream_t)stream);
}

ld_status ld_step_scalar(ld_handle* H, float* u, float* s, void* stream) {
  if (!H || !u || !s) return fail(LD_ERR_INVALID_ARG, "ld_step_scalar: NULL handle or field");
  return do_steps(H, u, 1, nullptr, 0, (cudaStream_t)stream, s);
}

ld_status ld_rollout_scalar(ld_handle* H, float* u, float* s, int32_t n, void* stream) {
  if (!H || !u || !s) return fail(LD_ERR_INVALID_ARG, "ld_rollout_scalar: NULL handle or field");
  if (n < 0) return fail(LD_ERR_INVALID_ARG, "n_steps must be >= 0");
  return do_steps(H, u, n, nullptr, 0, (cudaStream_t)stream, s);
}

ld_status ld_rollout_host(ld_handle* H, float* u_host, int32_t n, void* stream) {
  if (!H || !u_host) return fail(LD_ERR_INVALID_ARG, "ld_rollout_host: NULL handle or field");
  if (n < 0) return fail(LD_ERR_INVALID_ARG, "n_steps must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  if (!H->views.empty() && H->cfg.check_finite_every == 0) {
    // pipelined: chunk v's copy-in, steps and copy-out on its own stream, so the copies of one chunk
    // overlap the kernels of the others; every chunk starts after the caller's stream and the caller's
    // stream waits for all of them (bitwise the same result as the whole batch: Pin-14).  The chunks'
    // steps interleave on their streams: chaining them (chunk v's first kernel after chunk v - 1's last,
    // LD_HOST_SEQUENTIAL=1) exposes only the last copy-out but measured slower end to end (c4 3.86e8 vs
    // 3.99e8, c3 3.61e8 vs 4.05e8 cell-updates/s): a chunk's small flux / projection kernels no longer
    // overlap the other chunks' convs.
    cudaEvent_t start = H->view_events[0];
    LD_CUDA(cudaEventRecord(start, st), "ld_rollout_host");
    for (size_t v = 0; v < H->views.size(); ++v) LD_CUDA(cudaStreamWaitEvent(H->view_streams[v], start, 0), "ld_rollout_host");
    for (size_t v = 0; v < H->views.size(); ++v) {
      ld_handle* V = H->views[v];
      cudaStream_t vs = H->view_streams[v];
      float* hu = u_host + v * V->field;
      V->step = H->step;
      LD_CUDA(cudaMemcpyAsync(V->ubuf, hu, V->field * 4, cudaMemcpyHostToDevice, vs), "ld_rollout_host H2D");
      static const bool sequential = getenv("LD_HOST_SEQUENTIAL") != nullptr;   // measurement knob
      if (v > 0 && sequential) LD_CUDA(cudaStreamWaitEvent(vs, H->view_cdone[v - 1], 0), "ld_rollout_host");
      const ld_status ls = do_steps(V, V->ubuf, n, nullptr, 0, vs);
      if (ls != LD_OK) return ls;
      LD_CUDA(cudaEventRecord(H->view_cdone[v], vs), "ld_rollout_host");
      LD_CUDA(cudaMemcpyAsync(hu, V->ubuf, V->field * 4, cudaMemcpyDeviceToHost, vs), "ld_rollout_host D2H");
    }
    for (size_t v = 0; v < H->views.size(); ++v) {
      LD_CUDA(cudaEventRecord(H->view_events[v], H->view_streams[v]), "ld_rollout_host");
      LD_CUDA(cudaStreamWaitEvent(st, H->view_events[v], 0), "ld_rollout_host");
    }
    H->step += n;
    LD_CUDA(cudaStreamSynchronize(st), "ld_rollout_host");
    return LD_OK;
  }
  LD_CUDA(cudaMemcpyAsync(H->ubuf, u_host, H->field * 4, cudaMemcpyHostToDevice, st), "ld_rollout_host H2D");
  ld_status s = do_steps(H, H->ubuf, n, nullptr, 0, st);
  if (s != LD_OK) return s;
  LD_CUDA(cudaMemcpyAsync(u_host, H->ubuf, H->field * 4, cudaMemcpyDeviceToHost, st), "ld_rollout_host D2H");
  LD_CUDA(cudaStreamSynchronize(st), "ld_rollout_host");
  return LD_OK;
}

ld_status ld_eval_net(ld_handle* H, const float* U, float* R, void* stream) {
  if (H && H->slab) return fail(LD_ERR_UNSUPPORTED, "component entry points are single-domain (use ld_step in slab modes)");
  if (!H || !U || !R) return fail(LD_ERR_INVALID_ARG, "ld_eval_net: NULL argument");
  if (H->cfg.stencil_mode != LD_STENCIL_LEARNED) return fail(LD_ERR_INVALID_ARG, "no net in fixed mode");
  cudaError_t e = run_net(H, U, R, nullptr, true, OUT_PLANAR_ALL, H->n_out, (cudaStream_t)stream);
  return e == cudaSuccess ? LD_OK : cuda_fail(e, "ld_eval_net");
}

ld_status ld_eval_stencils(ld_handle* H, const float* U, float* w, void* stream) {
  if (H && H->slab) return fail(LD_ERR_UNSUPPORTED, "component entry points are single-domain (use ld_step in slab modes)");
  if (!H || !U || !w) return fail(LD_ERR_INVALID_ARG, "ld_eval_stencils: NULL argument");
  if (H->cfg.stencil_mode != LD_STENCIL_LEARNED) return fail(LD_ERR_INVALID_ARG, "no net in fixed mode");
  cudaError_t e = run_net(H, U, w, nullptr, false, OUT_PLANAR_ALL, 24, (cudaStream_t)stream);
  return e == cudaSuccess ? LD_OK : cuda_fail(e, "ld_eval_stencils");
}

ld_status ld_eval_tendency(ld_handle* H, const float* U, float* T, void* stream) {
  if (H && H->slab) return fail(LD_ERR_UNSUPPORTED, "component entry points are single-domain (use ld_step in slab modes)");
  if (!H || !U || !T) return fail(LD_ERR_INVALID_ARG, "ld_eval_tendency: NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  const bool learned = H->cfg.stencil_mode == LD_STENCIL_LEARNED;
  cudaError_t e = cudaSuccess;
  if (learned) e = run_net(H, U, H->w, nullptr, false, OUT_STENCIL, 24, st);
  if (e == cudaSuccess && H->cfg.fno_layers > 0)
    e = fno_big(&H->cfg) ? launch_spectral_big(U, H->fno_out, H->N, H->B, H->cfg.fno_kmax, 2, 8, 0, H->fno_M,
                                                 H->fno_tw, H->sp_scratch, st)
                         : launch_spectral(U, H->fno_out, H->N, H->B, H->cfg.fno_kmax, H->fno_M, H->fno_tw, st);
  if (e == cudaSuccess) {
    StageCoef S{0.f, 0.f, 0.f, 0.f, 0.f, 0, 0};
    if (H->cfg.stencil_mode == LD_STENCIL_5X4)
      e = launch_flux5x4_rk(flux_params(H), S, H->w5x4, U, U, H->acc, T, 1, st);
    else
      e = launch_flux_rk(flux_params(H), S, H->base24, U, U, learned ? H->w : nullptr, H->e, H->acc, T, 1, st);
  }
  return e == cudaSuccess ? LD_OK : cuda_fail(e, "ld_eval_tendency");
}

ld_status ld_project(ld_handle* H, const float* in, float* out, void* stream) {
  if (H && H->slab) return fail(LD_ERR_UNSUPPORTED, "component entry points are single-domain (use ld_step in slab modes)");
  if (!H || !in || !out) return fail(LD_ERR_INVALID_ARG, "ld_project: NULL argument");
  if (H->cfg.system != LD_SYSTEM_NS)   // Burgers handles have no spectrum / pressure buffers (R9)
    return fail(LD_ERR_INVALID_ARG, "ld_project: the handle's system is Burgers (no projection, R9)");
  cudaError_t e = launch_projection(in, out, H->spec, H->p, H->N, H->B, (float)(H->cfg.length / H->N), H->tw,
                                    H->ksym2, (cudaStream_t)stream);
  return e == cudaSuccess ? LD_OK : cuda_fail(e, "ld_project");
}

ld_status ld_set_graph_replay(ld_handle* H, int32_t enable) {
  if (!H) return fail(LD_ERR_INVALID_ARG, "NULL handle");
  H->use_graphs = enable != 0;
  return LD_OK;
}

ld_status ld_set_kernel_timing(ld_handle* H, int32_t enable) {
  if (!H) return fail(LD_ERR_INVALID_ARG, "NULL handle");
  H->timing = enable != 0;
  return LD_OK;
}

ld_status ld_kernel_times(ld_handle* H, double* ms, int64_t* cnt, int32_t n) {
  if (!H || !ms || !cnt || n < 1) return fail(LD_ERR_INVALID_ARG, "ld_kernel_times: bad argument");
  for (int i = 0; i < n; ++i) { ms[i] = 0.0; cnt[i] = 0; }
  for (size_t k = 0; k < H->ev_used; ++k) {
    LD_CUDA(cudaEventSynchronize(H->ev_pool[2 * k + 1]), "ld_kernel_times");
    float t = 0.f;
    LD_CUDA(cudaEventElapsedTime(&t, H->ev_pool[2 * k], H->ev_pool[2 * k + 1]), "ld_kernel_times");
    const int c = H->ev_cls[k];
    if (c < n) { ms[c] += t; cnt[c] += 1; }
  }
  H->ev_used = 0;
  return LD_OK;
}

ld_status ld_get_step_index(const ld_handle* H, int64_t* out) {
  if (!H || !out) return fail(LD_ERR_INVALID_ARG, "NULL argument");
  *out = H->step;
  return LD_OK;
}

ld_status ld_reset_step_counter(ld_handle* H) {
  if (!H) return fail(LD_ERR_INVALID_ARG, "NULL handle");
  H->step = 0;
  return LD_OK;
}

ld_status ld_launches_per_step(const ld_handle* H, int32_t* out) {
  if (!H || !out) return fail(LD_ERR_INVALID_ARG, "NULL argument");
  *out = H->launches_per_step;
  return LD_OK;
}

ld_status ld_destroy(ld_handle* H) {
  if (!H) return fail(LD_ERR_INVALID_ARG, "NULL handle");
  for (ld_handle* V : H->views) {
    for (int i = 0; i < 2; ++i)
      if (V->gexec[i]) cudaGraphExecDestroy(V->gexec[i]);
    if (V->cap_stream) cudaStreamDestroy(V->cap_stream);
    delete V;
  }
  for (auto vs : H->view_streams) cudaStreamDestroy(vs);
  for (auto ve : H->view_events) cudaEventDestroy(ve);
  for (auto vc : H->view_cdone) cudaEventDestroy(vc);
  if (H->is_view) return LD_OK;
  delete H->slab;
  for (int i = 0; i < 2; ++i)
    if (H->gexec[i]) cudaGraphExecDestroy(H->gexec[i]);
  for (auto ev : H->ev_pool) cudaEventDestroy(ev);
  if (H->cap_stream) cudaStreamDestroy(H->cap_stream);
  delete H;
  return LD_OK;
}

// ---------------------------------------------------------------------------
// NEXT-4: vector-Jacobian product of one step (adjoint.cu).  Mirrors the reverse
// pass of oracle/adjoint_oracle.py; every kernel is fp32 SIMT.
// ---------------------------------------------------------------------------
namespace {
struct VjpWs {
  float *Ust[4], *Ub[4], *Y, *pre, *Tb, *E, *Hb0, *w24, *F4, *Fadj, *R, *Rb, *G[2], *zero;
  std::vector<float*> z, h, Wt, gW, gb;
  size_t total;
};

// Workspace of ld_step_vjp, carved in order from `base` (nullptr: sizes only)
VjpWs vjp_layout(const ld_handle* H, char* base) {
  VjpWs V{};
  Layout L;
  const size_t F = H->field, cells = (size_t)H->B * H->plane;
  auto take = [&](size_t floats) { const size_t o = L.add(floats * 4); return base ? (float*)(base + o) : nullptr; };
  for (int i = 0; i < 4; ++i) V.Ust[i] = take(F);
  for (int i = 0; i < 4; ++i) V.Ub[i] = take(F);
  V.Y = take(F); V.pre = take(F); V.Tb = take(F); V.E = take(F); V.Hb0 = take(F);
  V.w24 = take(cells * 24); V.F4 = take(cells * 4); V.Fadj = take(cells * 8);
  const bool learned = H->cfg.stencil_mode == LD_STENCIL_LEARNED;
  V.R = take(learned ? cells * 32 : 64); V.Rb = take(learned ? cells * 32 : 64);
  const int wmax = learned ? H->cfg.width : 0;
  V.G[0] = take(learned ? cells * wmax : 64); V.G[1] = take(learned ? cells * wmax : 64);
  V.zero = take(64);
  for (size_t l = 0; l < H->layers.size(); ++l) {
    const Layer& y = H->layers[l];
    const bool last = l + 1 == H->layers.size();
    V.z.push_back(last ? nullptr : take(cells * y.co_pad));
    V.h.push_back(last ? nullptr : take(cells * y.co_pad));
    const int cout_pad = l == 0 ? 32 : y.ci;
    V.Wt.push_back(take((size_t)9 * y.co_pad * cout_pad));
    V.gW.push_back(take((size_t)9 * y.ci * y.co_pad));
    V.gb.push_back(take(y.co_pad));
  }
  V.total = L.total;
  return V;
}

// forward net (fp32 SIMT) on the stage field U, keeping z_l, h_l = phi(z_l) and the raw output R
cudaError_t vjp_net_fwd(ld_handle* H, VjpWs& V, const float* U, cudaStream_t st) {
  const ld_config& c = H->cfg;
  const size_t cells = (size_t)H->B * H->plane;
  for (size_t l = 0; l < H->layers.size(); ++l) {
    const Layer& y = H->layers[l];
    const bool last = l + 1 == H->layers.size();
    const float* in = l == 0 ? U : V.h[l - 1];
    const float* W = last ? H->raw_last_w : H->wts + y.w_off;
    const float* b = last ? H->raw_last_b : H->wts + y.b_off;
    float* out = last ? V.R : V.z[l];
    cudaError_t e = launch_conv_simt(in, l == 0, y.ci, H->N, H->B, W, b, y.co_pad, -1, OUT_NHWC, y.co, out, nullptr, st);
    if (e == cudaSuccess && !last) e = adj_act(V.z[l], V.h[l], cells * y.co_pad, c.activation, 0, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// net reverse pass from Rb (cotangent of R): parameter gradients += and Ub += d/dU
cudaError_t vjp_net_bwd(ld_handle* H, VjpWs& V, const float* U, float* Ub, cudaStream_t st) {
  const ld_config& c = H->cfg;
  const size_t cells = (size_t)H->B * H->plane;
  const float* G = V.Rb;
  int ping = 0;
  for (int l = (int)H->layers.size() - 1; l >= 0; --l) {
    const Layer& y = H->layers[l];
    const float* Hin = l == 0 ? U : V.h[l - 1];
    cudaError_t e = adj_wgrad(Hin, l == 0, y.ci, G, y.co_pad, H->N, H->B, V.gW[l], V.gb[l], st);
    if (e != cudaSuccess) return e;
    if (l > 0) {   // H_bar = conv(G, flipped W^T); G_{l-1} = H_bar * phi'(z_{l-1})
      float* Gn = V.G[ping];
      ping ^= 1;
      e = launch_conv_simt(G, false, y.co_pad, H->N, H->B, V.Wt[l], V.zero, y.ci, -1, OUT_NHWC, y.ci, Gn, nullptr, st);
      if (e == cudaSuccess) e = adj_act(V.z[l - 1], Gn, cells * y.ci, c.activation, 1, st);
      if (e != cudaSuccess) return e;
      G = Gn;
    } else {       // d/dU (planar, 2 channels) added to Ub
      e = launch_conv_simt(G, false, y.co_pad, H->N, H->B, V.Wt[0], V.zero, 32, -1, OUT_PLANAR_ALL, 2, V.Hb0, nullptr, st);
      if (e == cudaSuccess) e = adj_lin3(Ub, 1.f, Ub, 1.f, V.Hb0, 0.f, nullptr, H->field, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

struct VjpPhys {
  float inv_h, nu, gamma, drag;
  int forced;
};
VjpPhys vjp_phys(const ld_handle* H) {
  const ld_config& c = H->cfg;
  return VjpPhys{(float)(H->N / c.length), (float)c.nu, c.system == LD_SYSTEM_BURGERS ? 0.5f : 1.0f, (float)c.drag,
                 (c.force_amp != 0.0 || c.drag != 0.0) ? 1 : 0};
}

// Y = a un + b U + cdt T(U) (+ ec E); keeps e of this evaluation in V.E when keep_e
cudaError_t vjp_stage_fwd(ld_handle* H, VjpWs& V, const float* U, const float* un, float a, float b, float cdt, float ec,
                          bool keep_e, float* Y, float* Tout, cudaStream_t st) {
  const bool learned = H->cfg.stencil_mode == LD_STENCIL_LEARNED;
  const VjpPhys ph = vjp_phys(H);
  cudaError_t e = cudaSuccess;
  if (learned) e = vjp_net_fwd(H, V, U, st);
  if (e == cudaSuccess && keep_e && learned && H->cfg.tc_head) e = adj_extract_e(V.R, H->N, H->B, V.E, st);
  if (e == cudaSuccess)
    e = adj_fwd_faces(U, learned ? V.R : nullptr, H->base24, H->N, H->B, ph.inv_h, ph.nu, ph.gamma, V.w24, V.F4, st);
  if (e == cudaSuccess)
    e = adj_fwd_combine(V.F4, U, un, V.E, H->N, H->B, ph.inv_h, ph.forced, H->force_row, ph.drag, a, b, cdt, ec, Tout, Y,
                        st);
  return e;
}

// Ub += (dT/dU)^T Tb at U (and the e path: eb = cotangent of this net's e, or nullptr)
cudaError_t vjp_T(ld_handle* H, VjpWs& V, const float* U, const float* Tb, const float* eb, float* Ub, cudaStream_t st) {
  const bool learned = H->cfg.stencil_mode == LD_STENCIL_LEARNED;
  const VjpPhys ph = vjp_phys(H);
  cudaError_t e = cudaSuccess;
  if (learned) e = vjp_net_fwd(H, V, U, st);
  if (e == cudaSuccess)
    e = adj_fwd_faces(U, learned ? V.R : nullptr, H->base24, H->N, H->B, ph.inv_h, ph.nu, ph.gamma, V.w24, V.F4, st);
  if (e == cudaSuccess)
    e = adj_bwd_faces(U, V.w24, Tb, eb, H->N, H->B, ph.inv_h, ph.nu, ph.gamma, V.Fadj, learned ? V.Rb : nullptr, st);
  if (e == cudaSuccess) e = adj_bwd_gather(V.Fadj, V.w24, Tb, H->N, H->B, ph.forced, ph.drag, Ub, st);
  if (e == cudaSuccess && learned) e = vjp_net_bwd(H, V, U, Ub, st);
  return e;
}

// P (NS) or the identity (Burgers), out of place
cudaError_t vjp_P(ld_handle* H, const float* in, float* out, cudaStream_t st) {
  if (H->cfg.system == LD_SYSTEM_NS)
    return launch_projection(in, out, H->spec, H->p, H->N, H->B, (float)(H->cfg.length / H->N), H->tw, H->ksym2, st);
  return adj_lin3(out, 1.f, in, 0.f, nullptr, 0.f, nullptr, H->field, st);
}
}  // namespace

extern "C" {

ld_status ld_vjp_workspace_bytes(const ld_handle* H, size_t* out) {
  if (!H || !out) return fail(LD_ERR_INVALID_ARG, "ld_vjp_workspace_bytes: NULL argument");
  *out = vjp_layout(H, nullptr).total;
  return LD_OK;
}

ld_status ld_step_vjp(ld_handle* H, const float* u, const float* gout, float* gin, float* gparams, void* ws,
                      size_t ws_bytes, void* stream) {
  if (!H || !u || !gout || !gin || !ws) return fail(LD_ERR_INVALID_ARG, "ld_step_vjp: NULL argument");
  if (H->slab) return fail(LD_ERR_UNSUPPORTED, "ld_step_vjp is single-domain");
  const ld_config& c = H->cfg;
  if (c.fno_layers > 0 || c.tc_mode != 0 || c.freeze_stencils != 0)
    return fail(LD_ERR_UNSUPPORTED, "ld_step_vjp covers the BASELINE step (fno_layers, tc_mode, freeze_stencils = 0)");
  if (c.stencil_mode == LD_STENCIL_LEARNED && c.width != 64 && c.width != 32)
    return fail(LD_ERR_UNSUPPORTED, "ld_step_vjp: width must be 32 or 64");
  if (((uintptr_t)ws) & 255) return fail(LD_ERR_INVALID_ARG, "vjp workspace must be 256-byte aligned");
  VjpWs V = vjp_layout(H, (char*)ws);
  if (ws_bytes < V.total) return fail(LD_ERR_INVALID_ARG, "vjp workspace too small: need " + std::to_string(V.total));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t F = H->field;
  const float dt = (float)c.dt;
  const bool learned = c.stencil_mode == LD_STENCIL_LEARNED;
  const bool add_e = c.tc_head && ((H->step + 1) % c.tc_interval == 0);
#define VJ(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) return cuda_fail(_e, "ld_step_vjp"); } while (0)
  // parameter-gradient accumulators and the backward conv weights (flipped, transposed)
  for (size_t l = 0; l < H->layers.size(); ++l) {
    const Layer& y = H->layers[l];
    const bool last = l + 1 == H->layers.size();
    VJ(cudaMemsetAsync(V.gW[l], 0, (size_t)9 * y.ci * y.co_pad * 4, st));
    VJ(cudaMemsetAsync(V.gb[l], 0, (size_t)y.co_pad * 4, st));
    VJ(adj_transpose_w(last ? H->raw_last_w : H->wts + y.w_off, y.ci, y.co_pad, l == 0 ? 32 : y.ci, V.Wt[l], st));
  }
  VJ(cudaMemsetAsync(V.zero, 0, 256, st));
  VJ(cudaMemsetAsync(V.E, 0, F * 4, st));
  VJ(cudaMemsetAsync(gin, 0, F * 4, st));
  VJ(cudaMemcpyAsync(V.Ust[0], u, F * 4, cudaMemcpyDeviceToDevice, st));
  const float* eb = nullptr;
  if (c.rk_order == 2 || c.rk_order == 3) {
    // Shu-Osher: U_{s+1} = P(a_s u + b_s U_s + c_s dt T(U_s) [+ e at the last stage]), U_0 = u
    const int p = c.rk_order;
    const float A2[2][3] = {{1.f, 0.f, 1.f}, {0.5f, 0.5f, 0.5f}};
    const float A3[3][3] = {{1.f, 0.f, 1.f}, {0.75f, 0.25f, 0.25f}, {1.f / 3.f, 2.f / 3.f, 2.f / 3.f}};
    auto co = [&](int s, int k) { return p == 2 ? A2[s][k] : A3[s][k]; };
    for (int s = 0; s + 1 < p; ++s) {   // forward recompute of the stage fields U_1 .. U_{p-1}
      VJ(vjp_stage_fwd(H, V, V.Ust[s], u, co(s, 0), co(s, 1), co(s, 2) * dt, 0.f, false, V.Y, nullptr, st));
      VJ(vjp_P(H, V.Y, V.Ust[s + 1], st));
    }
    for (int s = 0; s < p; ++s) VJ(cudaMemsetAsync(V.Ub[s], 0, F * 4, st));
    for (int s = p - 1; s >= 0; --s) {
      VJ(vjp_P(H, s == p - 1 ? gout : V.Ub[s + 1], V.pre, st));   // P self-adjoint
      if (s == p - 1 && add_e) {   // e (stage-1 net) enters before the last projection
        VJ(cudaMemcpyAsync(V.E, V.pre, F * 4, cudaMemcpyDeviceToDevice, st));
        eb = V.E;
      }
      VJ(adj_lin3(gin, 1.f, gin, co(s, 0), V.pre, 0.f, nullptr, F, st));
      VJ(adj_lin3(V.Ub[s], 1.f, V.Ub[s], co(s, 1), V.pre, 0.f, nullptr, F, st));
      VJ(adj_lin3(V.Tb, co(s, 2) * dt, V.pre, 0.f, nullptr, 0.f, nullptr, F, st));
      VJ(vjp_T(H, V, V.Ust[s], V.Tb, s == 0 ? eb : nullptr, V.Ub[s], st));
    }
    VJ(adj_lin3(gin, 1.f, gin, 1.f, V.Ub[0], 0.f, nullptr, F, st));
  } else {
    // classical RK4: U2 = P(u + dt/2 K1), U3 = P(u + dt/2 K2), U4 = P(u + dt K3),
    // out = P(u + dt/6 (K1 + 2 K2 + 2 K3 + K4) + e)
    VJ(vjp_stage_fwd(H, V, V.Ust[0], u, 1.f, 0.f, 0.5f * dt, 0.f, false, V.Y, nullptr, st));
    VJ(vjp_P(H, V.Y, V.Ust[1], st));
    VJ(vjp_stage_fwd(H, V, V.Ust[1], u, 1.f, 0.f, 0.5f * dt, 0.f, false, V.Y, nullptr, st));
    VJ(vjp_P(H, V.Y, V.Ust[2], st));
    VJ(vjp_stage_fwd(H, V, V.Ust[2], u, 1.f, 0.f, dt, 0.f, false, V.Y, nullptr, st));
    VJ(vjp_P(H, V.Y, V.Ust[3], st));
    VJ(vjp_P(H, gout, V.pre, st));
    if (add_e) {
      VJ(cudaMemcpyAsync(V.E, V.pre, F * 4, cudaMemcpyDeviceToDevice, st));
      eb = V.E;
    }
    VJ(adj_lin3(gin, 1.f, V.pre, 0.f, nullptr, 0.f, nullptr, F, st));
    // K cotangents: Ub[0..3] <- K1b..K4b = dt/6, dt/3, dt/3, dt/6 times pre
    const float kc[4] = {dt / 6.f, dt / 3.f, dt / 3.f, dt / 6.f};
    for (int k = 0; k < 4; ++k) VJ(adj_lin3(V.Ub[k], kc[k], V.pre, 0.f, nullptr, 0.f, nullptr, F, st));
    const float back[4] = {0.f, 0.5f * dt, 0.5f * dt, dt};   // U_{k+1} = P(u + back[k+1] K_k)
    for (int k = 3; k >= 1; --k) {   // stage k evaluates K_{k+1} = T(U_{k+1})... stored as Ust[k]
      VJ(cudaMemsetAsync(V.Y, 0, F * 4, st));
      VJ(vjp_T(H, V, V.Ust[k], V.Ub[k], nullptr, V.Y, st));       // U_k cotangent
      VJ(vjp_P(H, V.Y, V.Tb, st));                                 // through U_k = P(u + back[k] K_{k-1})
      VJ(adj_lin3(gin, 1.f, gin, 1.f, V.Tb, 0.f, nullptr, F, st));
      VJ(adj_lin3(V.Ub[k - 1], 1.f, V.Ub[k - 1], back[k], V.Tb, 0.f, nullptr, F, st));
    }
    VJ(vjp_T(H, V, V.Ust[0], V.Ub[0], eb, gin, st));
  }
  if (gparams && learned) {   // += into the blob layout W[co][ky][kx][ci], b[co]
    size_t off = 0;
    for (size_t l = 0; l < H->layers.size(); ++l) {
      const Layer& y = H->layers[l];
      VJ(adj_pack_grads(V.gW[l], V.gb[l], y.ci, y.co, y.co_pad, gparams + off, st));
      off += (size_t)y.co * 9 * y.ci + y.co;
    }
  }
#undef VJ
  return LD_OK;
}

// Reverse pass through an n-step rollout from u0 (the paper trains on autoregressive rollouts of k_s
// steps): the forward states u^0 .. u^{n-1} are recomputed into traj_ws ([n][B][2][N][N],
// caller-owned) with the handle's step kernels, then g is carried back step by step with ld_step_vjp
// (TC gating at each step's index, starting from the handle's current index, which is restored).
// gin = (d u^n / d u^0)^T gout; gparams += sum over the steps of the parameter cotangents.
ld_status ld_rollout_vjp(ld_handle* H, const float* u0, int32_t n, const float* gout, float* gin, float* gparams,
                         float* traj_ws, void* ws, size_t ws_bytes, void* stream) {
  if (!H || !u0 || !gout || !gin || (n > 0 && !traj_ws)) return fail(LD_ERR_INVALID_ARG, "ld_rollout_vjp: NULL argument");
  if (n < 0) return fail(LD_ERR_INVALID_ARG, "n_steps must be >= 0");
  if (H->cfg.scalar_mode != 0) return fail(LD_ERR_UNSUPPORTED, "ld_rollout_vjp: scalar handles step with ld_step_scalar");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t F = H->field;
  const int64_t k0 = H->step;
  if (n == 0) {
    LD_CUDA(cudaMemcpyAsync(gin, gout, F * 4, cudaMemcpyDeviceToDevice, st), "ld_rollout_vjp");
    return LD_OK;
  }
  LD_CUDA(cudaMemcpyAsync(traj_ws, u0, F * 4, cudaMemcpyDeviceToDevice, st), "ld_rollout_vjp");
  for (int k = 1; k < n; ++k) {   // u^k = step(u^{k-1})
    LD_CUDA(cudaMemcpyAsync(traj_ws + (size_t)k * F, traj_ws + (size_t)(k - 1) * F, F * 4, cudaMemcpyDeviceToDevice, st),
            "ld_rollout_vjp");
    const ld_status ls = do_steps(H, traj_ws + (size_t)k * F, 1, nullptr, 0, st);
    if (ls != LD_OK) { H->step = k0; return ls; }
  }
  // g_n = gout; g_k = VJP_k(u^k)^T g_{k+1}; the cotangent alternates between gin and the handle's host
  // staging buffer (never read and written in one call)
  float* bufs[2] = {gin, H->ubuf};
  const float* g = gout;
  int cur = 0;
  for (int k = n - 1; k >= 0; --k) {
    H->step = k0 + k;
    if (bufs[cur] == g) cur ^= 1;
    float* dst = bufs[cur];
    const ld_status ls = ld_step_vjp(H, traj_ws + (size_t)k * F, g, dst, gparams, ws, ws_bytes, stream);
    if (ls != LD_OK) { H->step = k0; return ls; }
    g = dst;
    cur ^= 1;
  }
  if (g != gin) LD_CUDA(cudaMemcpyAsync(gin, g, F * 4, cudaMemcpyDeviceToDevice, st), "ld_rollout_vjp");
  H->step = k0;
  return LD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Frequency-domain operator O_F (spectral.cu)
// ---------------------------------------------------------------------------
struct ld_spectral {
  int n, K;
  float2* M;    // [n_modes][8][2] composed per-mode matrices (workspace)
  float2* tw;   // [n] e^{-2 pi i m / n} (workspace)
};

static size_t sp_modes(int K) { return (size_t)(K + 1) * (2 * K + 1) - K; }

size_t ld_spectral_param_count(int32_t k_max, int32_t layers, int32_t width) {
  if (k_max < 0 || layers < 1 || width < 1) return 0;
  return sp_modes(k_max) * ((size_t)width * 2 * 2 + (size_t)(layers - 1) * width * width * 2) + (size_t)8 * width;
}

ld_status ld_spectral_workspace_bytes(int32_t n, int32_t k_max, size_t* out) {
  if (!out) return fail(LD_ERR_INVALID_ARG, "out is NULL");
  if (n < 8 || (n & (n - 1)) || k_max < 0 || 2 * k_max >= n)
    return fail(LD_ERR_INVALID_ARG, "spectral: n must be a power of two >= 8 and 0 <= k_max < n/2");
  *out = ((sp_modes(k_max) * 16 * sizeof(float2) + 255) & ~(size_t)255) + (size_t)n * sizeof(float2);
  return LD_OK;
}

ld_status ld_spectral_create(int32_t n, int32_t k_max, int32_t layers, int32_t width, const float* params,
                             size_t n_params, void* ws, size_t ws_bytes, ld_spectral** out) {
  size_t need = 0;
  ld_status s = ld_spectral_workspace_bytes(n, k_max, &need);
  if (s != LD_OK) return s;
  if (!out || !params || !ws) return fail(LD_ERR_INVALID_ARG, "spectral: NULL argument");
  if (layers < 1 || width < 1) return fail(LD_ERR_INVALID_ARG, "spectral: layers and width must be >= 1");
  if (n_params != ld_spectral_param_count(k_max, layers, width))
    return fail(LD_ERR_INVALID_ARG, "spectral: n_params mismatch, need " +
                                        std::to_string(ld_spectral_param_count(k_max, layers, width)));
  if (ws_bytes < need) return fail(LD_ERR_INVALID_ARG, "spectral: workspace too small, need " + std::to_string(need));
  if (spectral_smem_bytes(n, k_max) > 227 * 1024)
    return fail(LD_ERR_UNSUPPORTED, "spectral: (n, k_max) tables exceed shared memory");
  const size_t nm = sp_modes(k_max);
  std::vector<float2> hM;
  compose_spectral(params, k_max, layers, width, n, false, hM);
  std::vector<float2> htw(n);
  for (int m = 0; m < n; ++m) {
    const double a = -2.0 * M_PI * m / n;
    htw[m] = make_float2((float)cos(a), (float)sin(a));
  }
  {
    const cudaError_t ea = spectral_set_smem_limits();
    if (ea != cudaSuccess) return cuda_fail(ea, "ld_spectral_create");
  }
  ld_spectral* op = new ld_spectral();
  op->n = n; op->K = k_max;
  op->M = (float2*)ws;
  op->tw = (float2*)((char*)ws + ((nm * 16 * sizeof(float2) + 255) & ~(size_t)255));
  cudaError_t e;
  if ((e = cudaMemcpy(op->M, hM.data(), hM.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(op->tw, htw.data(), htw.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess) {
    delete op;
    return cuda_fail(e, "ld_spectral_create");
  }
  *out = op;
  return LD_OK;
}

ld_status ld_spectral_apply(ld_spectral* op, const float* u, int32_t batch, float* out, void* stream) {
  if (!op || !u || !out) return fail(LD_ERR_INVALID_ARG, "ld_spectral_apply: NULL argument");
  if (batch < 1) return fail(LD_ERR_INVALID_ARG, "ld_spectral_apply: batch must be >= 1");
  const cudaError_t e = launch_spectral(u, out, op->n, batch, op->K, op->M, op->tw, (cudaStream_t)stream);
  return e == cudaSuccess ? LD_OK : cuda_fail(e, "ld_spectral_apply");
}

ld_status ld_spectral_destroy(ld_spectral* op) {
  if (!op) return fail(LD_ERR_INVALID_ARG, "NULL operator");
  delete op;
  return LD_OK;
}

ld_status ld_nccl_unique_id(uint8_t* out) {
  if (!out) return fail(LD_ERR_INVALID_ARG, "out is NULL");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(LD_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  memcpy(out, &id, 128);
  return LD_OK;
}

ld_status ld_nccl_comm_init(const uint8_t* id, int32_t world, int32_t rank, void** comm_out) {
  if (!id || !comm_out) return fail(LD_ERR_INVALID_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(LD_ERR_INVALID_ARG, "bad rank/world");
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = ncclCommInitRank(&comm, world, uid, rank);
  if (r != ncclSuccess) return fail(LD_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  *comm_out = comm;
  return LD_OK;
}

ld_status ld_nccl_comm_destroy(void* comm) {
  if (!comm) return fail(LD_ERR_INVALID_ARG, "NULL communicator");
  const ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
  if (r != ncclSuccess) return fail(LD_ERR_NCCL, std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
  return LD_OK;
}

ld_status ld_slab_geometry(const ld_config* cfg, int32_t world, int32_t* out5) {
  ld_status s = validate(cfg, nullptr);   // geometry only: no device-path (FFT size, precision) limits
  if (s != LD_OK) return s;
  if (world < 1 || cfg->n % world != 0 || (cfg->n / world) % 8 != 0)
    return fail(LD_ERR_INVALID_ARG, "slab geometry needs (n / world) % 8 == 0");
  if (!out5) return fail(LD_ERR_INVALID_ARG, "out is NULL");
  int n, m, hlo, hhi, next;
  slab_geometry(cfg, world, n, m, hlo, hhi, next);
  out5[0] = n; out5[1] = m; out5[2] = hlo; out5[3] = hhi; out5[4] = next;
  return LD_OK;
}

ld_status ld_downsample(const float* fine, int32_t n_fine, int32_t batch, int32_t factor, float* coarse,
                        void* stream) {
  if (!fine || !coarse) return fail(LD_ERR_INVALID_ARG, "ld_downsample: NULL field");
  if (batch < 1 || factor < 1 || n_fine < 1 || n_fine % factor != 0)
    return fail(LD_ERR_INVALID_ARG, "ld_downsample: need batch >= 1, factor >= 1, n_fine % factor == 0");
  const cudaError_t e = launch_downsample(fine, n_fine, factor, (size_t)batch * 2, coarse, (cudaStream_t)stream);
  return e == cudaSuccess ? LD_OK : cuda_fail(e, "ld_downsample");
}

const char* ld_last_error(void) { return g_err.c_str(); }

const char* ld_version(void) {
  return "ldsolver-b200 0.1 (sm_100a; kernels: conv_simt, conv_tcgen05_tf32, flux_rk, fft_projection)";
}

}  // extern "C"
