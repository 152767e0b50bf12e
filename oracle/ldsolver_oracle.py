"""CPU ORACLE for the LDSolver coarse-grid rollout step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this module.  The product path
(``paper_2507_01975_b200``) never imports it and has no CPU fallback.  This
file shares no code with the CUDA path: it is a plain, slow, fp64 numpy
restatement of the step, written in the order of PAPER.md and of the readings
listed in DESIGN.md ("Readings of the paper", R1-R23 of SURVEY.md §8c).

Citations: ``P:n`` = /root/reference/PAPER.md line n (LaTeX source).

Conventions (SURVEY.md §8 grid conventions): domain [0, L)^2, N x N cells,
h = L/N; cell (i, j) has centre ((i+1/2)h, (j+1/2)h); arrays are indexed
``[..., j, i]`` (y, x); indices are periodic mod N.  Fields are ``[B][2][N][N]``
with component 0 = u (x-velocity), 1 = v (y-velocity).

Pinned by tests/test_oracle_pins.py.  The random-weight
conv net is pinned to its definition (torch conv2d, brute-force loops from the packed
blob); the paper prints no trained weights or worked numeric example to pin it to.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional

import numpy as np

# ----------------------------------------------------------------------------
# Configuration accessors (plain dict or any object with these attributes)
# ----------------------------------------------------------------------------


def _get(cfg, name, default=None):
    if isinstance(cfg, dict):
        return cfg.get(name, default)
    return getattr(cfg, name, default)


# ----------------------------------------------------------------------------
# 1. Network (P:246-250 learnable conv, generalised to a 3x3-conv stencil net
#    by BASELINE.json north_star)
# ----------------------------------------------------------------------------


def unpack_params(params: np.ndarray, n_layers: int, width: int, n_out: int):
    """Split the blob W_l[co][ky][kx][ci], b_l[co] (layer order) into fp64 arrays."""
    chans = [2] + [width] * (n_layers - 1) + [n_out]
    p = np.asarray(params, dtype=np.float64)
    layers = []
    off = 0
    for l in range(n_layers):
        ci, co = chans[l], chans[l + 1]
        nw = co * 9 * ci
        W = p[off:off + nw].reshape(co, 3, 3, ci)
        off += nw
        b = p[off:off + co]
        off += co
        layers.append((W, b))
    if off != p.size:
        raise ValueError(f"param blob has {p.size} floats, expected {off}")
    return layers


def gelu(x):
    """Exact-erf GELU: 1/2 x (1 + erf(x / sqrt 2)) (R6)."""
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def relu(x):
    return np.maximum(x, 0.0)


def conv3x3_periodic(H, W, b):
    """Cross-correlation with circular padding (as PyTorch Conv2d, padding_mode='circular').

    H: [B][N][N][Cin] indexed [b, j, i, c];  W: [Cout][3][3][Cin];  b: [Cout].
    out[b, j, i, o] = b[o] + sum_{ky,kx,c} W[o, ky, kx, c] * H[b, j+ky-1, i+kx-1, c]  (mod N)
    """
    out = np.zeros(H.shape[:3] + (W.shape[0],)) + b
    for ky in range(3):
        for kx in range(3):
            dy, dx = ky - 1, kx - 1
            # shifted[b, j, i, c] = H[b, (j+dy) % N, (i+dx) % N, c]
            shifted = np.roll(H, shift=(-dy, -dx), axis=(1, 2))
            # one [cells x Cin] @ [Cin x Cout] product per tap (2-D, so numpy hands it to BLAS whole)
            out += (shifted.reshape(-1, H.shape[-1]) @ W[:, ky, kx, :].T).reshape(out.shape)
    return out


def net_forward(U, layers, activation: int):
    """R = H_L with H_0 = U and H_l = phi(W_l * H_{l-1} + b_l), phi skipped on the last layer.

    U: [B][2][N][N] -> R: [B][N][N][n_out]
    """
    H = np.moveaxis(np.asarray(U, dtype=np.float64), 1, -1)  # [B][N][N][2]
    phi = gelu if activation == 1 else relu
    for l, (W, b) in enumerate(layers):
        H = conv3x3_periodic(H, W, b)
        if l < len(layers) - 1:
            H = phi(H)
    return H


# ----------------------------------------------------------------------------
# 2. Constraint (R4): w = w_base + Pi R   (P:240-244 physics conv as w_base)
# ----------------------------------------------------------------------------

S_OFFSETS = np.array([-2.5, -1.5, -0.5, 0.5, 1.5, 2.5])  # tap position minus face position


def default_base_stencils():
    """[2 axes][2 ops][6]: op 0 = interp, op 1 = deriv.  2nd-order central (R5)."""
    base = np.zeros((2, 2, 6))
    base[:, 0, 2:4] = 0.5          # linear interpolation  (c_{i-1} + c_i) / 2
    base[:, 1, 2] = -1.0           # central difference    (c_i - c_{i-1}) / h
    base[:, 1, 3] = 1.0
    return base


def projector_interp():
    """Pi_I = I - 1 1^T / 6: keeps sum(w_I) = sum(w_I^base) (= 1, reproduces constants)."""
    return np.eye(6) - np.ones((6, 6)) / 6.0


def projector_deriv():
    """Pi_D = orthogonal projector onto null{1, s}: keeps sum(w_D) = 0 and sum(s w_D) = 1."""
    one = np.ones(6) / math.sqrt(6.0)
    s = S_OFFSETS / np.linalg.norm(S_OFFSETS)
    return np.eye(6) - np.outer(one, one) - np.outer(s, s)


def constrain(R, base=None):
    """R[..., 0:24] -> w[..., 2 axes, 2 ops, 6].

    Channel order (R4): R[0:6] x-interp, R[6:12] x-deriv, R[12:18] y-interp,
    R[18:24] y-deriv.
    """
    if base is None:
        base = default_base_stencils()
    PI, PD = projector_interp(), projector_deriv()
    raw = np.asarray(R, dtype=np.float64)[..., :24].reshape(R.shape[:-1] + (2, 2, 6))
    w = np.empty_like(raw)
    w[..., 0, :] = raw[..., 0, :] @ PI.T
    w[..., 1, :] = raw[..., 1, :] @ PD.T
    return w + base


# ----------------------------------------------------------------------------
# 3.-6. Tendency T(U): faces, fluxes, divergence, source
#   P:201 ("the flux block computes grad u ... at the interfaces, and u_bar"),
#   Eq.4 P:224-227 (face-flux sum), P:189 (Burgers flux u^2/2 - nu grad u, R9),
#   forcing/drag R12.
# ----------------------------------------------------------------------------


def face_values(c, w_axis_op, axis):
    """Apply a 6-tap stencil along `axis` (-1 = x, -2 = y) at the face owned by each cell.

    out[.., j, i] = sum_t w[.., j, i, t] * c[.., (i-3+t)] (x) ; same in j for y.
    The face at i-1/2 (resp. j-1/2) is owned by cell i (resp. j) (R2).
    """
    out = np.zeros_like(c)
    for t in range(6):
        # np.roll by s gives out[k] = in[k - s]; we need in[k - 3 + t] -> s = 3 - t
        out += w_axis_op[..., t] * np.roll(c, shift=3 - t, axis=axis)
    return out


def tendency(U, w, cfg, h, fno=None):
    """T(U) for U: [B][2][N][N], w: [B][N][N][2][2][6] (axis, op, tap).

    fno: None, or the frequency-domain branch on the faces [B][8][N][N] (NEXT-2, reading N2-5:
    O^(m) = O_P + O_L + O_F): channels (interp u, interp v, d/dx u, d/dx v) at the x-face
    and (interp u, interp v, d/dy u, d/dy v) at the y-face, added to the stencil face values
    (derivatives in derivative units, after the 1/h)."""
    nu = float(_get(cfg, "nu"))
    system = int(_get(cfg, "system"))
    gamma = 0.5 if system == 0 else 1.0  # R9 reading (A): F = 1/2 u (x) u - nu grad u
    u, v = U[:, 0], U[:, 1]
    wIx, wDx = w[..., 0, 0, :], w[..., 0, 1, :]
    wIy, wDy = w[..., 1, 0, :], w[..., 1, 1, :]
    # face-normal advecting velocities from the interp stencil (R3)
    ux = face_values(u, wIx, -1)
    vy = face_values(v, wIy, -2)
    if fno is not None:
        ux = ux + fno[:, 0]
        vy = vy + fno[:, 5]
    T = np.empty_like(U)
    for ci, c in enumerate((u, v)):
        cx = face_values(c, wIx, -1)
        dcx = face_values(c, wDx, -1) / h
        cy = face_values(c, wIy, -2)
        dcy = face_values(c, wDy, -2) / h
        if fno is not None:
            cx = cx + fno[:, ci]
            dcx = dcx + fno[:, 2 + ci]
            cy = cy + fno[:, 4 + ci]
            dcy = dcy + fno[:, 6 + ci]
        Fx = gamma * ux * cx - nu * dcx     # flux through x-face i-1/2
        Fy = gamma * vy * cy - nu * dcy     # flux through y-face j-1/2
        # T = -[F(i+1) - F(i) + F(j+1) - F(j)] / h
        T[:, ci] = -((np.roll(Fx, -1, axis=-1) - Fx) + (np.roll(Fy, -1, axis=-2) - Fy)) / h
    amp = float(_get(cfg, "force_amp", 0.0) or 0.0)
    kf = float(_get(cfg, "force_k", 0.0) or 0.0)
    alpha = float(_get(cfg, "drag", 0.0) or 0.0)
    if amp != 0.0 or alpha != 0.0:
        n = U.shape[-1]
        y = (np.arange(n) + 0.5) * h
        T[:, 0] += amp * np.sin(kf * y)[:, None] - alpha * u
        T[:, 1] += -alpha * v
    return T


# ----------------------------------------------------------------------------
# The paper's own constant 5x4 face kernels (O_P + O_L = (W_P + W_L) * u with W in R^{5x4};
# SURVEY.md §8f lower row; readings F1-F3 in DESIGN.md §8i): 4 taps along the face normal (symmetric about
# the face) x 5 across it, one kernel per (axis, op), constant in space.
# ----------------------------------------------------------------------------

def base_5x4():
    """W_P [2 axes][2 ops][5 tangential b][4 normal a]: linear interpolation / central difference on the
    face-normal line (b = 2): taps a = 1, 2 (cells i-1, i around the face i-1/2)."""
    W = np.zeros((2, 2, 5, 4))
    W[:, 0, 2, 1] = W[:, 0, 2, 2] = 0.5
    W[:, 1, 2, 1], W[:, 1, 2, 2] = -1.0, 1.0
    return W


def constrain_5x4(WL):
    """W = W_P + Pi W_L (reading F2, the 2-D analogue of R4): Pi keeps sum(W_I) = 1 (constants
    reproduced), sum(W_D) = 0, sum(s W_D) = 1 and sum(t W_D) = 0 with s = a - 3/2 / t = b - 2 the normal /
    tangential offset of a tap (the derivative exact on every linear field); Pi = orthogonal projector
    onto the complement of span{1} (interp) / span{1, s, t} (deriv) in R^20 (1, s, t mutually orthogonal)."""
    WL = np.asarray(WL, dtype=np.float64).reshape(2, 2, 5, 4)
    one = np.ones(20) / math.sqrt(20.0)
    sv = np.tile(np.arange(4) - 1.5, 5)
    sv = sv / np.linalg.norm(sv)
    tv = np.repeat(np.arange(5) - 2.0, 4)
    tv = tv / np.linalg.norm(tv)
    PI = np.eye(20) - np.outer(one, one)
    PD = PI - np.outer(sv, sv) - np.outer(tv, tv)
    out = base_5x4().copy()
    for ax in range(2):
        out[ax, 0] += (PI @ WL[ax, 0].ravel()).reshape(5, 4)
        out[ax, 1] += (PD @ WL[ax, 1].ravel()).reshape(5, 4)
    return out


def face_values_5x4(c, W, axis):
    """x-face (axis -1) of cell (j, i): sum_{b<5, a<4} W[b, a] c(j - 2 + b, i - 2 + a);
    y-face (axis -2): sum W[b, a] c(j - 2 + a, i - 2 + b)."""
    out = np.zeros_like(c)
    for b in range(5):
        for a in range(4):
            if axis == -1:
                out += W[b, a] * np.roll(c, shift=(2 - b, 2 - a), axis=(-2, -1))
            else:
                out += W[b, a] * np.roll(c, shift=(2 - a, 2 - b), axis=(-2, -1))
    return out


def tendency_5x4(U, W, cfg, h):
    """T(U) with the constant 5x4 face kernels W [2][2][5][4] (flux form, source as tendency())."""
    nu = float(_get(cfg, "nu"))
    gamma = 0.5 if int(_get(cfg, "system")) == 0 else 1.0
    u, v = U[:, 0], U[:, 1]
    ux = face_values_5x4(u, W[0, 0], -1)
    vy = face_values_5x4(v, W[1, 0], -2)
    T = np.empty_like(U)
    for ci, c in enumerate((u, v)):
        Fx = gamma * ux * face_values_5x4(c, W[0, 0], -1) - nu * face_values_5x4(c, W[0, 1], -1) / h
        Fy = gamma * vy * face_values_5x4(c, W[1, 0], -2) - nu * face_values_5x4(c, W[1, 1], -2) / h
        T[:, ci] = -((np.roll(Fx, -1, axis=-1) - Fx) + (np.roll(Fy, -1, axis=-2) - Fy)) / h
    amp = float(_get(cfg, "force_amp", 0.0) or 0.0)
    kf = float(_get(cfg, "force_k", 0.0) or 0.0)
    alpha = float(_get(cfg, "drag", 0.0) or 0.0)
    if amp != 0.0 or alpha != 0.0:
        n = U.shape[-1]
        y = (np.arange(n) + 0.5) * h
        T[:, 0] += amp * np.sin(kf * y)[:, None] - alpha * u
        T[:, 1] += -alpha * v
    return T


def scalar_tendency(U, S, w, D, h):
    """Passive-scalar transport ("a coupled advection-diffusion equation alongside the NSE";
    readings S1-S4): F_s = u_f s_f - D ds_f on each face, with the face-normal velocity
    and the interp / deriv stencils of the momentum flux (shared, R3); T_s = -div_h F_s.
    S: [B][N][N]."""
    u, v = U[:, 0], U[:, 1]
    wIx, wDx = w[..., 0, 0, :], w[..., 0, 1, :]
    wIy, wDy = w[..., 1, 0, :], w[..., 1, 1, :]
    Fx = face_values(u, wIx, -1) * face_values(S, wIx, -1) - D * face_values(S, wDx, -1) / h
    Fy = face_values(v, wIy, -2) * face_values(S, wIy, -2) - D * face_values(S, wDy, -2) / h
    return -((np.roll(Fx, -1, axis=-1) - Fx) + (np.roll(Fy, -1, axis=-2) - Fy)) / h


# ----------------------------------------------------------------------------
# 7. Projection (Eq.13-15; spectral Poisson P:315; R10)
# ----------------------------------------------------------------------------


def div_c(U, h):
    """Centred divergence d = [u(i+1)-u(i-1) + v(j+1)-v(j-1)] / 2h."""
    u, v = U[:, 0], U[:, 1]
    return ((np.roll(u, -1, -1) - np.roll(u, 1, -1)) + (np.roll(v, -1, -2) - np.roll(v, 1, -2))) / (2 * h)


def symbol(n, h):
    """k_hat_m = sin(k_m h)/h, k_m = m (m < N/2) else m - N; exactly 0 at m = 0 and m = N/2 (R10, R23)."""
    m = np.arange(n)
    k = np.where(m < n // 2, m, m - n)
    kh = np.sin(k * 2.0 * math.pi / n) / h
    kh[0] = 0.0
    kh[n // 2] = 0.0
    return kh


def solve_pressure(d, h):
    """p = Re IDFT2( -DFT2(d) / (kx^2 + ky^2) ), p_hat = 0 on the 4 null modes (mx, my in {0, N/2})."""
    n = d.shape[-1]
    kh = symbol(n, h)
    den = kh[None, :] ** 2 + kh[:, None] ** 2     # [my][mx]
    null = np.zeros((n, n), dtype=bool)
    for a in (0, n // 2):
        for b in (0, n // 2):
            null[a, b] = True
    den_safe = np.where(null, 1.0, den)
    dh = np.fft.fft2(d)
    ph = np.where(null, 0.0, -dh / den_safe)
    return np.real(np.fft.ifft2(ph))


def project(U, h):
    """u <- u - G_c p with D_c G_c p = D_c u (p is dt x pressure; dt cancels)."""
    p = solve_pressure(div_c(U, h), h)
    out = np.array(U, dtype=np.float64, copy=True)
    out[:, 0] -= (np.roll(p, -1, -1) - np.roll(p, 1, -1)) / (2 * h)
    out[:, 1] -= (np.roll(p, -1, -2) - np.roll(p, 1, -2)) / (2 * h)
    return out


# ----------------------------------------------------------------------------
# 8. One step: RK with per-stage projection (R7, R8, R13)
# ----------------------------------------------------------------------------


# ----------------------------------------------------------------------------
# Fine -> coarse data path: the paper's coarse training fields are the
# fine-grid DNS "downsampled ... to the desired coarse grid resolutions" (Table S1
# P:563).  Reading: finite-volume cell averages, i.e. the block mean of the f x f fine cells.
# ----------------------------------------------------------------------------


def downsample(u, f: int):
    """coarse[b, c, J, I] = mean_{dj, di < f} fine[b, c, J f + dj, I f + di]."""
    u = np.asarray(u, dtype=np.float64)
    B, C, n, _ = u.shape
    return u.reshape(B, C, n // f, f, n // f, f).mean(axis=(3, 5))


class Oracle:
    """Holds a config, the unpacked net and base stencils; runs steps in fp64."""

    def __init__(self, cfg, params: Optional[np.ndarray] = None, base_stencils=None):
        self.cfg = cfg
        self.n = int(_get(cfg, "n"))
        self.h = float(_get(cfg, "length", 2 * math.pi)) / self.n
        self.dt = float(_get(cfg, "dt"))
        self.system = int(_get(cfg, "system"))
        self.rk = int(_get(cfg, "rk_order"))
        self.tc = int(_get(cfg, "tc_head", 0) or 0)
        self.kc = int(_get(cfg, "tc_interval", 1) or 1)
        self.fixed = int(_get(cfg, "stencil_mode", 0) or 0) == 1
        self.w5x4 = None   # stencil_mode 2: the constrained constant 5x4 kernels
        if int(_get(cfg, "stencil_mode", 0) or 0) == 2:
            self.fixed = True
            self.w5x4 = constrain_5x4(np.zeros(80) if params is None else np.asarray(params, np.float64)[:80])
        self.activation = int(_get(cfg, "activation", 1))
        self.base = default_base_stencils() if base_stencils is None else np.asarray(base_stencils, np.float64).reshape(2, 2, 6)
        self.n_out = 24 + (2 if self.tc else 0)
        self.layers = None
        self.fno = None
        self.tc_hist = None   # NEXT-3 history block: ((R, Q), K)
        self.hist = []        # the last k_c step inputs, oldest first
        fl = int(_get(cfg, "fno_layers", 0) or 0)
        tcm = int(_get(cfg, "tc_mode", 0) or 0)
        p = np.asarray(params) if params is not None else np.zeros(0)
        off = 0
        if not self.fixed:
            L, Wd = int(_get(cfg, "n_layers")), int(_get(cfg, "width"))
            chans = [2] + [Wd] * (L - 1) + [self.n_out]
            nconv = sum(co * 9 * ci + co for ci, co in zip(chans[:-1], chans[1:]))
            self.layers = unpack_params(p[:nconv] if (fl > 0 or tcm == 1) else p, L, Wd, self.n_out)
            off = nconv
            if fl > 0:   # NEXT-2: the spectral blob follows the conv parameters
                from .spectral_oracle import unpack_spectral, _modes
                K, C = int(_get(cfg, "fno_kmax")), int(_get(cfg, "fno_width"))
                nm = len(_modes(K))
                nsp = nm * (C * 2 * 2 + (fl - 1) * C * C * 2) + 8 * C
                self.fno = (unpack_spectral(p[off:off + nsp], K, fl, C), K)
                off += nsp
        if tcm == 1:     # NEXT-3: the history block's blob comes last (2 k_c inputs, 2 outputs)
            from .spectral_oracle import unpack_spectral
            K, Lt, C = int(_get(cfg, "tc_kmax")), int(_get(cfg, "tc_layers")), int(_get(cfg, "tc_width"))
            self.tc_hist = (unpack_spectral(p[off:], K, Lt, C, n_in=2 * self.kc, n_out=2), K)
        self.step_index = 0

    # -- pieces ---------------------------------------------------------------
    def net(self, U):
        return net_forward(U, self.layers, self.activation)

    def stencils(self, U):
        """(w, e): w [B][N][N][2][2][6], e [B][2][N][N] or None."""
        B, n = U.shape[0], self.n
        if self.fixed:
            w = np.broadcast_to(self.base, (B, n, n, 2, 2, 6)).copy()
            return w, None
        R = self.net(U)
        w = constrain(R, self.base)
        e = np.moveaxis(R[..., 24:26], -1, 1) if self.tc else None
        return w, e

    def T(self, U, w_frozen=None):
        if self.w5x4 is not None:
            return tendency_5x4(U, self.w5x4, self.cfg, self.h), None
        w, e = self.stencils(U) if w_frozen is None else (w_frozen, None)
        fo = None
        if self.fno is not None:
            from .spectral_oracle import spectral_faces
            (R, Q), K = self.fno
            fo = spectral_faces(U, R, Q, K)
        return tendency(U, w, self.cfg, self.h, fo), e

    def P(self, U):
        return project(U, self.h) if self.system == 1 else U

    # -- one step ---------------------------------------------------------------
    def step(self, u):
        u = np.asarray(u, dtype=np.float64)
        dt = self.dt
        k = self.step_index
        T1, e = self.T(u)
        if int(_get(self.cfg, "freeze_stencils", 0) or 0) == 1:
            # per-step frozen stencils: every stage uses the stencils of u
            wf, _ = self.stencils(u)
            T = lambda U: (self.T(U, wf)[0], None)
        else:
            T = self.T
        if self.tc_hist is not None:
            # NEXT-3 (Eq. 2 / Eq. 12, readings N3-1..N3-3): the buffer holds the last k_c step inputs
            # u_{k-k_c+1} .. u_k; at steps with (k+1) % k_c == 0 (always with a full buffer) their
            # channel stack goes through the operator and the result is the e of the last stage
            self.hist = (self.hist + [u.copy()])[-self.kc:]
            add_e = (k + 1) % self.kc == 0
            if add_e:
                from .spectral_oracle import spectral_operator
                (R, Q), K = self.tc_hist
                e = spectral_operator(np.concatenate(self.hist, axis=1), R, Q, K)
        else:
            add_e = self.tc and ((k + 1) % self.kc == 0)
        E = e if add_e else 0.0
        if self.rk == 2:   # Heun / SSP-RK2 (R13)
            U1 = self.P(u + dt * T1)
            T2, _ = T(U1)
            out = self.P(0.5 * u + 0.5 * (U1 + dt * T2) + E)
        elif self.rk == 3:  # SSP-RK3, Shu-Osher form (R13)
            U1 = self.P(u + dt * T1)
            T2, _ = T(U1)
            U2 = self.P(0.75 * u + 0.25 * (U1 + dt * T2))
            T3, _ = T(U2)
            out = self.P(u / 3.0 + (2.0 / 3.0) * (U2 + dt * T3) + E)
        elif self.rk == 4:  # classical RK4
            K1 = T1
            U2 = self.P(u + 0.5 * dt * K1)
            K2, _ = T(U2)
            U3 = self.P(u + 0.5 * dt * K2)
            K3, _ = T(U3)
            U4 = self.P(u + dt * K3)
            K4, _ = T(U4)
            out = self.P(u + (dt / 6.0) * (K1 + 2 * K2 + 2 * K3 + K4) + E)
        else:
            raise ValueError(f"rk_order {self.rk}")
        self.step_index += 1
        return out

    def step_scalar(self, u, s):
        """One coupled step of (u, s): the momentum step exactly as step(), and the passive scalar s
        [B][N][N] through the same RK stages (Shu-Osher / RK4 coefficients) with the stage's stencils
        and face velocities; s is not projected and gets no TC term (readings S1-S4)."""
        D = float(_get(self.cfg, "scalar_diff", 0.0) or 0.0)
        u = np.asarray(u, dtype=np.float64)
        s = np.asarray(s, dtype=np.float64)
        dt = self.dt
        k0 = self.step_index
        # stage fields of the momentum step, recomputed here alongside the scalar
        Ts = lambda U, S: scalar_tendency(U, S, self.stencils(U)[0], D, self.h)
        if self.rk in (2, 3):
            coef = {2: [(1.0, 0.0, 1.0), (0.5, 0.5, 0.5)],
                    3: [(1.0, 0.0, 1.0), (0.75, 0.25, 0.25), (1.0 / 3.0, 2.0 / 3.0, 2.0 / 3.0)]}[self.rk]
            U, S = u, s
            Us = [u]
            for a, b, c in coef[:-1]:
                T, _ = self.T(U)
                S = a * s + b * S + c * dt * Ts(U, S)
                U = self.P(a * u + b * U + c * dt * T)
                Us.append(U)
            a, b, c = coef[-1]
            S = a * s + b * S + c * dt * Ts(U, S)
        else:
            U2 = self.P(u + 0.5 * dt * self.T(u)[0])
            U3 = self.P(u + 0.5 * dt * self.T(U2)[0])
            U4 = self.P(u + dt * self.T(U3)[0])
            K1 = Ts(u, s)
            S2 = s + 0.5 * dt * K1
            K2 = Ts(U2, S2)
            S3 = s + 0.5 * dt * K2
            K3 = Ts(U3, S3)
            S4 = s + dt * K3
            K4 = Ts(U4, S4)
            S = s + dt / 6.0 * (K1 + 2 * K2 + 2 * K3 + K4)
        self.step_index = k0
        u_next = self.step(u)
        return u_next, S

    def rollout(self, u, n_steps: int, save_every: int = 0) -> Dict[str, object]:
        """Repeat step() n_steps times; snapshots every save_every."""
        traj: List[np.ndarray] = []
        u = np.asarray(u, dtype=np.float64)
        for s in range(n_steps):
            u = self.step(u)
            if not np.all(np.isfinite(u)):
                raise FloatingPointError(f"non-finite field at step {self.step_index - 1}")
            if save_every and (s + 1) % save_every == 0:
                traj.append(u.copy())
        return {"u": u, "traj": traj}


def step(u, cfg, params=None, base_stencils=None, step_index: int = 0):
    o = Oracle(cfg, params, base_stencils)
    o.step_index = step_index
    return o.step(u)


def rollout(u, cfg, params, n_steps, base_stencils=None):
    return Oracle(cfg, params, base_stencils).rollout(u, n_steps)["u"]
