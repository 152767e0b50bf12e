/*
 * ldsolver.h -- C ABI of the B200-native LDSolver coarse-grid rollout step.
 *
 * What one step computes (citations are /root/reference/PAPER.md lines "P:n";
 * readings R1-R23 are restated in DESIGN.md "Readings of the paper"):
 *
 *   for each RK stage s ("FV module ... RK4 sub-step"; R7, R13):
 *     (a) net   R = W_L * phi(... phi(W_1 * U_s + b_1) ...) + b_L, 3x3 periodic conv
 *               (P:246-250 learnable conv, generalised per BASELINE.json north_star; R1, R6)
 *         w = w_base + Pi R   (P:240-244 physics conv as w_base; R4, R5)
 *     (b) faces c^x = sum_t w_I[t] c(i-3+t), dc^x = (1/h) sum_t w_D[t] c(i-3+t), same in y (R2, R3)
 *     (c) F = gamma u_f c_f - nu dc_f, T = -div_h F + f - alpha u (Eq.4; R9, R12)
 *     (e) U_{s+1}^pre = a_s u^n + b_s U_s + c_s dt T (+ e at the last stage; Eq.2; R8)
 *     (d) NS only: U_{s+1} = U^pre - G_c p, p = -(D_c G_c)^+ D_c U^pre by FFT
 *               (Eq.13-15, spectral Poisson P:315; R10)
 *
 * Layout conventions (all device buffers fp32, row-major, caller-owned):
 *   field u : [B][2][N][N]  component 0 = u (x-velocity), 1 = v; index [j][i] = [y][x];
 *             cell centres ((i+1/2)h, (j+1/2)h), h = length/N; periodic in both axes.
 *   params  : host fp32 blob; for each layer l = 1..L: W_l[co][ky][kx][ci] then b_l[co];
 *             widths 2 -> width -> ... -> width -> n_out, n_out = 24 (+2 if tc_head).
 *             Output channel order R[0:6] x-interp, R[6:12] x-deriv, R[12:18] y-interp,
 *             R[18:24] y-deriv, R[24:26] temporal correction e.
 *   base    : host fp64 [2 axes][2 ops][6 taps] (op 0 interp, op 1 deriv), or NULL for
 *             2nd-order central (interp (0,0,1/2,1/2,0,0), deriv (0,0,-1,1,0,0)).
 *
 * Ownership: the caller owns u, traj and the workspace (device memory, e.g. torch
 * tensors).  ld_init copies and re-packs the weights into the workspace (folding Pi
 * and w_base into the last layer) and keeps no host pointer.  Every call enqueues
 * asynchronously on the given stream; results are ready when that stream is.
 * One handle is single-owner (not thread-safe); distinct handles are independent.
 *
 * Errors: every entry point validates its arguments before any device work and
 * returns LD_ERR_INVALID_ARG / LD_ERR_UNSUPPORTED with a message in ld_last_error()
 * (thread-local).  CUDA failures return LD_ERR_CUDA.  With check_finite_every > 0,
 * ld_rollout synchronises the stream once at the end and returns LD_ERR_NONFINITE
 * naming the first checked step whose field held NaN/Inf.  There is no CPU
 * fallback: without a CUDA device every compute call returns LD_ERR_CUDA.
 */
#ifndef LDSOLVER_H
#define LDSOLVER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LD_OK = 0,
  LD_ERR_INVALID_ARG = -1,
  LD_ERR_CUDA = -2,
  LD_ERR_NCCL = -3,
  LD_ERR_OOM = -4,
  LD_ERR_NONFINITE = -5,
  LD_ERR_UNSUPPORTED = -6
} ld_status;

enum { LD_SYSTEM_BURGERS = 0, LD_SYSTEM_NS = 1 };
enum { LD_ACT_RELU = 0, LD_ACT_GELU = 1 };
enum { LD_STENCIL_LEARNED = 0, LD_STENCIL_FIXED = 1, LD_STENCIL_5X4 = 2 };
enum { LD_CONV_FP32 = 0, LD_CONV_TF32 = 1, LD_CONV_F16 = 2, LD_CONV_BF16 = 3 };

typedef struct {
  int32_t n;                  /* N: power of two, 8 <= N <= 8192 (R22)                       */
  int32_t batch;              /* B >= 1: fields per call (local batch in ensemble mode)       */
  double length;              /* domain side L (2*pi for every BASELINE config)               */
  int32_t system;             /* LD_SYSTEM_BURGERS (gamma = 1/2, no projection) or _NS        */
  double nu;                  /* viscosity >= 0 ("nu", "1/Re")                    */
  double dt;                  /* time step > 0, fixed for the rollout (caller's CFL rule R11) */
  int32_t rk_order;           /* 2 Heun, 3 SSP-RK3, 4 classical RK4 (R13)              */
  double force_amp, force_k;  /* f = (force_amp sin(force_k y), 0) at cell centres (R12)      */
  double drag;                /* linear drag alpha: T -= alpha u (both components)            */
  int32_t n_layers;           /* L >= 2 conv layers including the linear output layer (R6)    */
  int32_t width;              /* hidden channels: 32 or 64                                    */
  int32_t activation;         /* LD_ACT_RELU or LD_ACT_GELU (exact erf)                       */
  int32_t tc_head;            /* 1: two extra output channels e added at the last stage (R8)  */
  int32_t tc_interval;        /* k_c >= 1: e is added when (k+1) % k_c == 0, k = step index   */
  int32_t stencil_mode;       /* LD_STENCIL_LEARNED, _FIXED (w = w_base, net skipped), or     *
                               * _5X4: the paper's constant 5x4 face kernels W_P + Pi W_L        *
                               * (params_host = W_L [2 axes][2 ops][5 tangential][4   *
                               * normal], 80 floats; readings F1-F3 in DESIGN.md §8i)            */
  int32_t conv_precision;     /* LD_CONV_FP32 (SIMT fp32, parity), LD_CONV_TF32 (tcgen05      *
                               * kind::tf32 on fp32 activations) or LD_CONV_F16 (tcgen05       *
                               * kind::f16 on fp16 activations, fp32 accumulate; n >= 16) or   *
                               * LD_CONV_BF16 (kind::f16 on bf16 activations / weights)          */
  int32_t check_finite_every; /* 0 = off; else check the field every this many steps          */
  /* Frequency-domain branch O_F of the flux block (Eq. 8; readings
   * N2-1..N2-6 in DESIGN.md §8c): fno_layers = 0 turns it off (every BASELINE config).  With
   * fno_layers >= 1 (single domain, learned stencils; N <= 128 in one shared-memory cluster kernel, larger N
   * as three global-memory passes with scratch in the workspace), each RK stage evaluates O_F on
   * the stage field, placed on the faces by a half-cell spectral shift, and adds its 8 outputs to
   * the face values: interpolated u, v and the derivatives of u, v at the x-face and the y-face.
   * Its parameters (ld_spectral_param_count(fno_kmax, fno_layers, fno_width) floats, layout as
   * for ld_spectral_create) follow the conv parameters in params_host.                         */
  int32_t fno_kmax, fno_layers, fno_width;
  /* Temporal correction (Eq. 2, Eq. 12; reading N3-1..N3-3
   * in DESIGN.md §8d): tc_mode 0 = the net's TC head (tc_head, R8); tc_mode 1 = the history block:
   * the last k_c = tc_interval step inputs (a ring in the workspace) feed an operator of the O_F
   * family (2 k_c input channels, 2 outputs, cell-centred) whose output is the e added at the last
   * stage of every k_c-th step.  Needs tc_head = 0 and a single domain (N <= 64 in shared memory, larger N
   * as global-memory passes); its parameters
   * (modes / layout as ld_spectral_create with 2 k_c inputs and Q [2][tc_width]) follow the conv
   * and fno parameters in params_host. */
  int32_t tc_mode, tc_kmax, tc_layers, tc_width;
  /* 0 (default, reading R7: "the flux block runs inside each RK sub-step"): the net runs
   * on every stage field.  1: the stencils of the step's first stage are reused by the later
   * stages (a cheaper variant, SURVEY.md §8f "per-step frozen stencils"; different results). */
  int32_t freeze_stencils;
  /* Passive scalar (the shear flow's "coupled advection-diffusion equation alongside the
   * NSE"; SURVEY.md §8f lower row; readings S1-S4 in DESIGN.md §8h): scalar_mode 1 advects and diffuses
   * a scalar s with the stage's face velocities and learned stencils, diffusivity scalar_diff >= 0,
   * through the same RK stages (not projected, no forcing / TC).  A scalar handle steps with
   * ld_step_scalar / ld_rollout_scalar (ld_step / ld_rollout return LD_ERR_INVALID_ARG); single domain,
   * fno_layers = 0, tc_mode = 0, freeze_stencils = 0. */
  int32_t scalar_mode;
  double scalar_diff;
} ld_config;

/* Process placement:
 *  mode 0  single GPU, one field [B][2][N][N].
 *  mode 1  ensemble shard: this rank owns its own batch of B fields; no collective on the
 *          data path (PAR-1).
 *  mode 2  slab decomposition over `world` processes (PAR-2/3): rank r owns rows
 *          [r N/world, (r+1) N/world) of every field; u_dev passed to ld_step / ld_rollout is the
 *          rank's slab [B][2][N/world][N].  Halo rows and the all-to-all transposes of the
 *          distributed FFT go through NCCL on `nccl_comm` (an ncclComm_t, e.g. from
 *          ld_nccl_comm_init), enqueued on the caller's stream.
 *  mode 3  the same slab decomposition with all `world` ranks emulated in this process on one
 *          GPU (transfers become device-to-device copies between the rank contexts); u_dev is the
 *          global field [B][2][N][N].  Used to test the decomposition against mode 0 on one GPU.
 * Slab modes need conv_precision 1 or 2 (or stencil_mode FIXED), (N/world) % 8 == 0, slabs at
 * least as thick as the halos (max(L,3) below, max(L+1,3) above for an L-layer net) and, for NS,
 * 256 <= N <= 4096 (the distributed pencil FFT; four-step transforms at N = 2048 / 4096) with N/world a
 * multiple of the column chunk; otherwise LD_ERR_INVALID_ARG / LD_ERR_UNSUPPORTED.  The component entry
 * points (ld_eval_*, ld_project) are single-domain and return LD_ERR_UNSUPPORTED in slab modes. */
typedef struct {
  int32_t mode, rank, world;
  void* nccl_comm;
} ld_dist;

typedef struct ld_handle ld_handle;

/* Number of floats in the packed parameter blob for this config (0 if invalid). */
size_t ld_param_count(const ld_config* cfg);

/* Bytes of device workspace ld_init needs (256-byte aligned start required). */
ld_status ld_workspace_bytes(const ld_config* cfg, const ld_dist* dist, size_t* out_bytes);

/* Create a handle.  params_host: ld_param_count floats (ignored, may be NULL, in
 * LD_STENCIL_FIXED mode).  base_stencils_host: 24 doubles or NULL.  workspace_dev:
 * caller-owned device buffer of >= ld_workspace_bytes.  Uses the current CUDA device. */
ld_status ld_init(const ld_config* cfg, const ld_dist* dist, const float* params_host,
                  size_t n_params, const double* base_stencils_host, void* workspace_dev,
                  size_t workspace_bytes, ld_handle** out);

/* One full time step in place on u_dev ([B][2][N][N] device), then step index += 1. */
ld_status ld_step(ld_handle* h, float* u_dev, void* stream);

/* n_steps >= 0 steps in place.  traj_dev: NULL, or [n_steps/save_every][B][2][N][N]
 * device buffer receiving a snapshot after every save_every-th step (save_every >= 1). */
ld_status ld_rollout(ld_handle* h, float* u_dev, int32_t n_steps, float* traj_dev,
                     int32_t save_every, void* stream);

/* End-to-end entry point: copies u_host ([B][2][N][N], ideally pinned) to the handle's
 * internal device field, runs n_steps steps, copies the result back into u_host, and
 * synchronises the stream before returning. */
ld_status ld_rollout_host(ld_handle* h, float* u_host, int32_t n_steps, void* stream);

/* Coupled (u, s) steps of a scalar_mode = 1 handle: u_dev [B][2][N][N] and s_dev [B][N][N] (device,
 * in place).  One step = ld_step's momentum step plus the scalar through the same stages. */
ld_status ld_step_scalar(ld_handle* h, float* u_dev, float* s_dev, void* stream);
ld_status ld_rollout_scalar(ld_handle* h, float* u_dev, float* s_dev, int32_t n_steps, void* stream);

/* Component entry points (same kernels as the step; used for parity tests).
 *  ld_eval_net      : R_dev [B][n_out][N][N] = raw net output of U_dev (before Pi / base);
 *  ld_eval_stencils : w_dev [B][24][N][N] = constrained stencils w_base + Pi R;
 *  ld_eval_tendency : T_dev [B][2][N][N] = T(U_dev) with the net evaluated on U_dev;
 *  ld_project       : out_dev = P(in_dev) (NS projection; in-place allowed; LD_ERR_INVALID_ARG
 *                     on a Burgers handle, which has no projection buffers). */
ld_status ld_eval_net(ld_handle* h, const float* U_dev, float* R_dev, void* stream);
ld_status ld_eval_stencils(ld_handle* h, const float* U_dev, float* w_dev, void* stream);
ld_status ld_eval_tendency(ld_handle* h, const float* U_dev, float* T_dev, void* stream);
ld_status ld_project(ld_handle* h, const float* in_dev, float* out_dev, void* stream);

/* CUDA-graph replay of whole steps (default on): ld_step / ld_rollout capture one step's
 * launches per (field pointer, TC-add flag) and replay the graph.  0 = launch every kernel
 * individually.  Results are bitwise identical either way. */
ld_status ld_set_graph_replay(ld_handle* h, int32_t enable);

/* Per-kernel-class device timing (bench roofline).  When enabled, every launch of a
 * kernel class is bracketed by CUDA events on the launching stream.  Classes:
 * 0 conv first layer, 1 conv hidden layers, 2 conv output layer, 3 fused flux/RK (K2),
 * 4 projection (K3-K6; in slab modes the whole distributed projection including its
 * exchanges), 5 fused flux + projection stage kernel (NS, N <= 64), 6 the O_F branch
 * (fno_layers > 0), 7 the passive-scalar stage kernel (scalar_mode 1).  ld_kernel_times synchronises, returns the summed milliseconds
 * and launch counts per class since the last call, and resets them; classes >= n_classes
 * are dropped, so size the buffers with LD_N_KERNEL_CLASSES. */
#define LD_N_KERNEL_CLASSES 8
ld_status ld_set_kernel_timing(ld_handle* h, int32_t enable);
ld_status ld_kernel_times(ld_handle* h, double* ms_out, int64_t* count_out, int32_t n_classes);

ld_status ld_get_step_index(const ld_handle* h, int64_t* out);
ld_status ld_reset_step_counter(ld_handle* h);
/* Number of kernel launches one ld_step enqueues (for the bench's gpu_launches count). */
ld_status ld_launches_per_step(const ld_handle* h, int32_t* out);
ld_status ld_destroy(ld_handle* h);

/* Thread-local message describing the last non-OK status ("" if none). */
/* NCCL plumbing for mode 2.  ld_nccl_unique_id: rank 0 creates the 128-byte id (the caller
 * broadcasts it, e.g. with torch.distributed); ld_nccl_comm_init: every rank creates its
 * communicator on the current CUDA device (ncclCommInitRank; collective, blocks until all
 * ranks join); ld_nccl_comm_destroy releases it after the last handle using it is destroyed. */
ld_status ld_nccl_unique_id(uint8_t* out_128_bytes);
ld_status ld_nccl_comm_init(const uint8_t* id_128_bytes, int32_t world, int32_t rank, void** comm_out);
ld_status ld_nccl_comm_destroy(void* comm);
/* Host-only: slab geometry for `world` ranks -> out5 = {rows per rank n, spectrum positions per
 * rank m, halo rows below Hlo, halo rows above Hhi, extended slab height n + Hlo + Hhi}.  Checks
 * only the geometry ((n / world) % 8 == 0), not the device-path limits ld_init enforces. */
ld_status ld_slab_geometry(const ld_config* cfg, int32_t world, int32_t* out5);

/* Block-mean downsampling of fine-grid fields to a coarse grid (the paper
 * builds its coarse training data by downsampling fine-grid DNS, Table S1):
 * coarse_dev [B][2][n/f][n/f] = mean of the f x f fine cells of fine_dev [B][2][n][n]
 * (finite-volume cell averages).  Both device buffers are the caller's; n % f == 0 else
 * LD_ERR_INVALID_ARG.  Asynchronous on `stream`.  Together with stencil_mode FIXED (the
 * physics-only solver, "by activating only the physics-based convolution") this is the
 * fine-grid DNS / data-generation path. */
ld_status ld_downsample(const float* fine_dev, int32_t n_fine, int32_t batch, int32_t factor, float* coarse_dev,
                        void* stream);

/* Frequency-domain operator O_F (Eq. 8, P:252-256:
 * O_F(u) = Q(F^{-1}(R_L . F(u))); readings N2-1..N2-4 in DESIGN.md §8c) as a standalone
 * operator (the same operator runs inside the step when ld_config.fno_layers > 0, N2-5/N2-6).  Modes |kx|, |ky| <= k_max are retained
 * (0 <= k_max < n/2); the L = `layers` per-mode complex maps R_l and the real Q [8][width]
 * come as one fp32 host blob:
 *   R_1 [n_modes][width][2][re,im], R_l (l >= 2) [n_modes][width][width][re,im], Q [8][width],
 * modes in half-plane order (for kx in 0..k_max, ky in -k_max..k_max, skipping kx = 0, ky < 0;
 * n_modes = (k_max+1)(2 k_max+1) - k_max); R(-k) = conj(R(k)) is implied, so the output is real.
 * ld_spectral_create composes Q R_L ... R_1 per mode in fp64 into the caller's workspace
 * (ld_spectral_workspace_bytes) and keeps no host pointers.  ld_spectral_apply: u_dev
 * [batch][2][n][n] -> out_dev [batch][8][n][n] (channels: interp / deriv x x-face / y-face x
 * u / v, cell-centred), asynchronous on `stream`.  Errors: LD_ERR_INVALID_ARG for a bad shape,
 * count or NULL pointer, LD_ERR_UNSUPPORTED when the (n, k_max) tables exceed shared memory. */
typedef struct ld_spectral ld_spectral;
size_t ld_spectral_param_count(int32_t k_max, int32_t layers, int32_t width);
ld_status ld_spectral_workspace_bytes(int32_t n, int32_t k_max, size_t* out_bytes);
ld_status ld_spectral_create(int32_t n, int32_t k_max, int32_t layers, int32_t width, const float* params_host,
                             size_t n_params, void* workspace_dev, size_t workspace_bytes, ld_spectral** out);
ld_status ld_spectral_apply(ld_spectral* op, const float* u_dev, int32_t batch, float* out_dev, void* stream);
ld_status ld_spectral_destroy(ld_spectral* op);

/* Adjoint of one step (the solver is "fully differentiable" and trained by
 * back-propagating the rollout loss).  For the step that ld_step would take
 * from u_dev at the handle's current step index (TC gating, R8; the index is NOT advanced):
 *   gin_dev     [B][2][N][N] = (d u^{n+1} / d u^n)^T gout_dev        (overwritten)
 *   gparams_dev [ld_param_count] += (d u^{n+1} / d theta)^T gout_dev  (accumulated; NULL = skip)
 * in the layout of params_host (W_l[co][ky][kx][ci], b_l[co]; theta = the raw blob, before Pi / w_base).
 * Reverse pass of the discrete step (readings in DESIGN.md §8g): RK stages in reverse, the projection
 * self-adjoint, face stencils / fluxes / divergence / drag adjoints, Pi^T = Pi, the conv net in reverse;
 * e from the stage-1 net.  All fp32 SIMT kernels (the net recomputed in fp32 whatever conv_precision).
 * vjp_ws: caller-owned device scratch of ld_vjp_workspace_bytes(h) bytes (256-byte aligned).  Single
 * domain, fno_layers = 0, tc_mode = 0, freeze_stencils = 0 (else LD_ERR_UNSUPPORTED).  Asynchronous on
 * `stream`; u_dev and gout_dev are not modified. */
ld_status ld_vjp_workspace_bytes(const ld_handle* h, size_t* out_bytes);
/* Reverse pass through an n_steps rollout from u0_dev (training on autoregressive rollouts):
 * gin_dev = (d u^n / d u^0)^T gout_dev, gparams_dev += the sum of the steps' parameter cotangents (NULL =
 * skip).  traj_ws: caller-owned device scratch of n_steps fields [n][B][2][N][N] (the recomputed forward
 * states); vjp_ws as for ld_step_vjp.  Starts at the handle's step index and restores it. */
ld_status ld_rollout_vjp(ld_handle* h, const float* u0_dev, int32_t n_steps, const float* gout_dev, float* gin_dev,
                         float* gparams_dev, float* traj_ws, void* vjp_ws, size_t vjp_ws_bytes, void* stream);
ld_status ld_step_vjp(ld_handle* h, const float* u_dev, const float* gout_dev, float* gin_dev, float* gparams_dev,
                      void* vjp_ws, size_t vjp_ws_bytes, void* stream);

const char* ld_last_error(void);
/* Build identification string (arch, kernels compiled in). */
const char* ld_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LDSOLVER_H */
