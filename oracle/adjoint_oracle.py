"""CPU ORACLE of the adjoint (vector-Jacobian product) of one LDSolver step -- TEST INFRASTRUCTURE ONLY.

SURVEY.md §8f NEXT-4: "adjoint step for training (reverse mode through conv, stencils, RK, and P,
which is self-adjoint)".  The paper's solver is "fully differentiable" and is trained by
rolling out autoregressively and back-propagating the MSE loss of Eq. to the net
parameters theta.  This module restates, in fp64 numpy and in the reverse order of
oracle/ldsolver_oracle.py's forward step, the map

    (u^n, g) -> (u_bar = (d u^{n+1} / d u^n)^T g,  theta_bar = (d u^{n+1} / d theta)^T g)

for one step.  Only tests/ import it; the product path never does.  Pinned by
tests/test_adjoint_oracle.py against torch autograd (conv pieces), central finite differences of
the forward oracle in fp64 (dot-product tests for u and theta), and closed forms (symmetric linear
step at u = 0, conservation of the mean, translation equivariance).

Readings: the adjoint of the step as the forward oracle computes it, i.e. of
the discrete scheme (discretise-then-differentiate), with everything that the forward treats as
an input held fixed (dt, nu, forcing, base stencils) and e taken from the stage-1 net (R8).
"""
from __future__ import annotations

import math

import numpy as np

from . import ldsolver_oracle as F


# ----------------------------------------------------------------------------- net pieces

def conv3x3_transpose(G, W):
    """Adjoint of F.conv3x3_periodic in its input: Hbar[b, j, i, c] = sum_{o, ky, kx} W[o, ky, kx, c]
    G[b, j - (ky - 1), i - (kx - 1), o] (the forward reads H at (j + ky - 1, i + kx - 1))."""
    out = np.zeros(G.shape[:3] + (W.shape[-1],))
    for ky in range(3):
        for kx in range(3):
            dy, dx = ky - 1, kx - 1
            shifted = np.roll(G, shift=(dy, dx), axis=(1, 2))   # shifted[j, i] = G[j - dy, i - dx]
            out += (shifted.reshape(-1, G.shape[-1]) @ W[:, ky, kx, :]).reshape(out.shape)
    return out


def conv3x3_wgrad(H, G):
    """d/dW of sum(G * conv(H, W)): Wbar[o, ky, kx, c] = sum_{b, j, i} G[b, j, i, o] H[b, j + ky - 1, i + kx - 1, c]."""
    Co, Ci = G.shape[-1], H.shape[-1]
    Wb = np.zeros((Co, 3, 3, Ci))
    g2 = G.reshape(-1, Co)
    for ky in range(3):
        for kx in range(3):
            shifted = np.roll(H, shift=(-(ky - 1), -(kx - 1)), axis=(1, 2))
            Wb[:, ky, kx, :] = g2.T @ shifted.reshape(-1, Ci)
    return Wb


def gelu_grad(x):
    """d/dx of 1/2 x (1 + erf(x / sqrt 2)) = Phi(x) + x phi(x)."""
    from scipy.special import erf
    return 0.5 * (1.0 + erf(x / math.sqrt(2.0))) + x * np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)


def net_forward_saved(U, layers, activation):
    """Forward net keeping each layer's input H_{l-1} and pre-activation z_l."""
    H = np.moveaxis(np.asarray(U, dtype=np.float64), 1, -1)
    phi = F.gelu if activation == 1 else F.relu
    saved = []
    for l, (W, b) in enumerate(layers):
        z = F.conv3x3_periodic(H, W, b)
        saved.append((H, z))
        H = phi(z) if l < len(layers) - 1 else z
    return H, saved


def net_vjp(saved, layers, activation, Rbar):
    """(Ubar [B][2][N][N], [(Wbar, bbar) per layer]) for the cotangent Rbar [B][N][N][n_out] of R."""
    grads = [None] * len(layers)
    G = Rbar
    for l in range(len(layers) - 1, -1, -1):
        W, b = layers[l]
        Hin, z = saved[l]
        grads[l] = (conv3x3_wgrad(Hin, G), G.sum(axis=(0, 1, 2)))
        Hbar = conv3x3_transpose(G, W)
        if l > 0:
            zprev = saved[l - 1][1]
            dphi = gelu_grad(zprev) if activation == 1 else (zprev > 0).astype(np.float64)
            G = Hbar * dphi
        else:
            G = Hbar
    return np.moveaxis(G, -1, 1), grads


# ----------------------------------------------------------------------------- stencils / fluxes

def face_values_T(gbar, w_axis_op, axis):
    """Adjoint of F.face_values in the field: out = sum_t w[..., t] roll(c, 3 - t) ->
    c_bar = sum_t roll(w[..., t] gbar, -(3 - t))."""
    out = np.zeros_like(gbar)
    for t in range(6):
        out += np.roll(w_axis_op[..., t] * gbar, shift=-(3 - t), axis=axis)
    return out


def face_values_wgrad(gbar, c, axis):
    """d/dw[..., t] of sum(gbar * face_values(c, w)) = gbar * roll(c, 3 - t)."""
    return np.stack([gbar * np.roll(c, shift=3 - t, axis=axis) for t in range(6)], axis=-1)


def tendency_vjp(U, w, cfg, h, Tbar):
    """(Ubar, wbar) of F.tendency (fno = None) for the cotangent Tbar [B][2][N][N]."""
    nu = float(F._get(cfg, "nu"))
    gamma = 0.5 if int(F._get(cfg, "system")) == 0 else 1.0
    u, v = U[:, 0], U[:, 1]
    wIx, wDx, wIy, wDy = w[..., 0, 0, :], w[..., 0, 1, :], w[..., 1, 0, :], w[..., 1, 1, :]
    ux = F.face_values(u, wIx, -1)
    vy = F.face_values(v, wIy, -2)
    Ubar = np.zeros_like(U)
    wbar = np.zeros_like(w)
    uxbar = np.zeros_like(u)
    vybar = np.zeros_like(v)
    for ci, c in enumerate((u, v)):
        cx = F.face_values(c, wIx, -1)
        cy = F.face_values(c, wIy, -2)
        # T = -((roll(Fx, -1, x) - Fx) + (roll(Fy, -1, y) - Fy)) / h
        Fxbar = -(np.roll(Tbar[:, ci], 1, axis=-1) - Tbar[:, ci]) / h
        Fybar = -(np.roll(Tbar[:, ci], 1, axis=-2) - Tbar[:, ci]) / h
        # Fx = gamma ux cx - nu dcx,  dcx = face(c, wDx) / h
        uxbar += gamma * cx * Fxbar
        cxbar = gamma * ux * Fxbar
        dcxbar = -nu * Fxbar / h
        vybar += gamma * cy * Fybar
        cybar = gamma * vy * Fybar
        dcybar = -nu * Fybar / h
        Ubar[:, ci] += (face_values_T(cxbar, wIx, -1) + face_values_T(dcxbar, wDx, -1) +
                        face_values_T(cybar, wIy, -2) + face_values_T(dcybar, wDy, -2))
        wbar[..., 0, 0, :] += face_values_wgrad(cxbar, c, -1)
        wbar[..., 0, 1, :] += face_values_wgrad(dcxbar, c, -1)
        wbar[..., 1, 0, :] += face_values_wgrad(cybar, c, -2)
        wbar[..., 1, 1, :] += face_values_wgrad(dcybar, c, -2)
    Ubar[:, 0] += face_values_T(uxbar, wIx, -1)
    wbar[..., 0, 0, :] += face_values_wgrad(uxbar, u, -1)
    Ubar[:, 1] += face_values_T(vybar, wIy, -2)
    wbar[..., 1, 0, :] += face_values_wgrad(vybar, v, -2)
    alpha = float(F._get(cfg, "drag", 0.0) or 0.0)
    amp = float(F._get(cfg, "force_amp", 0.0) or 0.0)
    if amp != 0.0 or alpha != 0.0:       # T_u += f - alpha u, T_v += -alpha v (f does not depend on U)
        Ubar -= alpha * Tbar
    return Ubar, wbar


def constrain_T(wbar):
    """Adjoint of F.constrain in R (Pi_I, Pi_D symmetric): Rbar[0:24] = Pi wbar per (axis, op)."""
    PI, PD = F.projector_interp(), F.projector_deriv()
    Rb = np.empty(wbar.shape[:-3] + (24,))
    r = Rb.reshape(wbar.shape[:-3] + (2, 2, 6))
    r[..., 0, :] = wbar[..., 0, :] @ PI
    r[..., 1, :] = wbar[..., 1, :] @ PD
    return Rb


# ----------------------------------------------------------------------------- one step

class AdjointOracle(F.Oracle):
    """Forward oracle + the reverse pass of its step (BASELINE step only: no fno / history TC /
    frozen stencils)."""

    def _T_saved(self, U):
        """T(U) and what its VJP needs: (T, e, ctx)."""
        B, n = U.shape[0], self.n
        if self.fixed:
            w = np.broadcast_to(self.base, (B, n, n, 2, 2, 6)).copy()
            return F.tendency(U, w, self.cfg, self.h), None, (U, w, None)
        R, saved = net_forward_saved(U, self.layers, self.activation)
        w = F.constrain(R, self.base)
        e = np.moveaxis(R[..., 24:26], -1, 1) if self.tc else None
        return F.tendency(U, w, self.cfg, self.h), e, (U, w, saved)

    def _T_vjp(self, ctx, Tbar, ebar, grads):
        """Ubar of T (and of e if ebar is given) at ctx; parameter cotangents accumulated in grads."""
        U, w, saved = ctx
        Ubar, wbar = tendency_vjp(U, w, self.cfg, self.h, Tbar)
        if saved is None:
            return Ubar
        Rbar = np.zeros(w.shape[:3] + (self.n_out,))
        Rbar[..., :24] = constrain_T(wbar)
        if ebar is not None:
            Rbar[..., 24:26] = np.moveaxis(ebar, 1, -1)
        Ub, g = net_vjp(saved, self.layers, self.activation, Rbar)
        for l, (Wb, bb) in enumerate(g):
            grads[l][0][...] += Wb
            grads[l][1][...] += bb
        return Ubar + Ub

    def _Pt(self, X):   # P is an orthogonal projector (G_c = -D_c^T): self-adjoint
        return self.P(X)

    def step_vjp(self, u, gbar):
        """(u_bar, theta_bar blob) of one step from u (step index self.step_index, not advanced)."""
        for name in ("fno_layers", "tc_mode", "freeze_stencils"):
            if int(F._get(self.cfg, name, 0) or 0):
                raise ValueError(f"step_vjp covers the BASELINE step ({name} must be 0)")
        u = np.asarray(u, dtype=np.float64)
        g = np.asarray(gbar, dtype=np.float64)
        dt = self.dt
        add_e = bool(self.tc) and ((self.step_index + 1) % self.kc == 0)
        grads = [] if self.fixed else [(np.zeros_like(W), np.zeros_like(b)) for W, b in self.layers]
        ub = np.zeros_like(u)
        if self.rk in (2, 3):
            # Shu-Osher: U_{s+1} = P(a_s u + b_s U_s + c_s dt T(U_s) [+ e at the last stage]), U_0 = u
            coef = {2: [(1.0, 0.0, 1.0), (0.5, 0.5, 0.5)],
                    3: [(1.0, 0.0, 1.0), (0.75, 0.25, 0.25), (1.0 / 3.0, 2.0 / 3.0, 2.0 / 3.0)]}[self.rk]
            Us, ctxs, e1 = [u], [], None
            for s, (a, b, c) in enumerate(coef):
                T, e, ctx = self._T_saved(Us[-1])
                if s == 0:
                    e1 = e
                ctxs.append(ctx)
                if s + 1 < len(coef):
                    Us.append(self.P(a * u + b * Us[-1] + c * dt * T))
            Ub_next = g          # cotangent of U_{s+1} (the step output for the last stage)
            Ubar_stage = [np.zeros_like(u) for _ in coef]
            ebar = None
            for s in range(len(coef) - 1, -1, -1):
                a, b, c = coef[s]
                pre = self._Pt(Ub_next if s == len(coef) - 1 else Ubar_stage[s + 1])
                if s == len(coef) - 1 and add_e:
                    ebar = pre
                ub += a * pre
                Ubar_stage[s] += b * pre
                Ubar_stage[s] += self._T_vjp(ctxs[s], c * dt * pre, ebar if s == 0 else None, grads)
            ub += Ubar_stage[0]
        elif self.rk == 4:
            T1, e1, c1 = self._T_saved(u)
            U2 = self.P(u + 0.5 * dt * T1)
            T2, _, c2 = self._T_saved(U2)
            U3 = self.P(u + 0.5 * dt * T2)
            T3, _, c3 = self._T_saved(U3)
            U4 = self.P(u + dt * T3)
            T4, _, c4 = self._T_saved(U4)
            pre = self._Pt(g)                      # out = P(u + dt/6 (K1 + 2K2 + 2K3 + K4) + E)
            ebar = pre if add_e else None
            ub += pre
            K1b, K2b, K3b, K4b = dt / 6 * pre, dt / 3 * pre, dt / 3 * pre, dt / 6 * pre
            U4b = self._T_vjp(c4, K4b, None, grads)
            p4 = self._Pt(U4b)                     # U4 = P(u + dt K3)
            ub += p4
            K3b = K3b + dt * p4
            U3b = self._T_vjp(c3, K3b, None, grads)
            p3 = self._Pt(U3b)                     # U3 = P(u + dt/2 K2)
            ub += p3
            K2b = K2b + 0.5 * dt * p3
            U2b = self._T_vjp(c2, K2b, None, grads)
            p2 = self._Pt(U2b)                     # U2 = P(u + dt/2 K1)
            ub += p2
            K1b = K1b + 0.5 * dt * p2
            ub += self._T_vjp(c1, K1b, ebar, grads)
        else:
            raise ValueError(self.rk)
        blob = np.concatenate([np.concatenate([Wb.ravel(), bb]) for Wb, bb in grads]) if grads else np.zeros(0)
        return ub, blob


def step_vjp(u, cfg, params, gbar, base_stencils=None, step_index: int = 0):
    o = AdjointOracle(cfg, params, base_stencils)
    o.step_index = step_index
    return o.step_vjp(u, gbar)
