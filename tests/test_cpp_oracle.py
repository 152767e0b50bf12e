"""Pins of the plain C++ CPU oracle (oracle/cpp/ldsolver_oracle.cpp, BASELINE.json north_star's
"plain, slow CPU C++ implementation of the same step in fp64/fp32").

Every check compares it with something other than itself: a library routine (torch conv2d), a
closed form (shear-mode / Taylor-Green decay factors, the Kolmogorov fixed point, the 1-D Burgers
scheme, the pass-through TC net), an invariant (moments of the constrained stencils, zero tendency
of a constant field, mean momentum, divergence after projection, translation equivariance), a
brute-force construction written here (the classical FV right-hand side, the dense bordered 8x8
Poisson solve), and element-wise agreement with the independently written numpy oracle
(oracle/ldsolver_oracle.py; the two share no code).  P:n = PAPER.md line; Rk / Pin-k = SURVEY.md §8c.
"""
import math

import numpy as np
import pytest

import oracle as O
from ldgen import make_ic, make_weights
from ldgen.configs import get_config
from ldgen.ic import make_config_ic
from oracle import cpp_oracle as X
from tests.test_oracle_pins import (TWO_PI, _Rp, _burgers_1d_rhs, _centres, _cfg, _classical_fv_rhs,
                                    _passthrough_tc_params)


def test_builds_and_counts_threads():
    X.build()
    assert X.hardware_threads() >= 1


def test_net_matches_torch_circular_conv2d():
    torch = pytest.importorskip("torch")
    n, L, W = 8, 3, 5
    cfg = _cfg(n=n, stencil_mode=0, n_layers=L, width=W, activation=1, tc_head=1)
    params = make_weights(L, W, 26, seed=3, init="stress")
    u = make_ic("noise", n, 2, seed=1)
    got = X.net_forward(u, cfg, params)
    # torch reference: circular pad + conv2d per layer, exact-erf GELU between layers
    x = torch.from_numpy(u.copy())
    off = 0
    chans = [2, W, W, 26]
    p = torch.from_numpy(params.astype(np.float64))
    for l in range(L):
        ci, co = chans[l], chans[l + 1]
        Wl = p[off:off + co * 9 * ci].reshape(co, 3, 3, ci).permute(0, 3, 1, 2)
        off += co * 9 * ci
        bl = p[off:off + co]
        off += co
        x = torch.nn.functional.conv2d(torch.nn.functional.pad(x, (1, 1, 1, 1), mode="circular"), Wl, bl)
        if l < L - 1:
            x = torch.nn.functional.gelu(x, approximate="none")
    np.testing.assert_allclose(got, np.moveaxis(x.numpy(), 1, -1), rtol=1e-12, atol=1e-12)


def test_relu_net_and_stencil_moments():
    n = 8
    cfg = _cfg(n=n, stencil_mode=0, n_layers=3, width=8, activation=0)
    params = make_weights(3, 8, 24, seed=7, init="stress")
    u = make_ic("noise", n, 1, seed=2)
    w = X.stencils(u, cfg, params).reshape(1, n, n, 2, 2, 6)
    s = np.arange(6) - 2.5
    np.testing.assert_allclose(w[..., 0, :].sum(-1), 1.0, atol=1e-12)        # interp reproduces constants (R4)
    np.testing.assert_allclose(w[..., 1, :].sum(-1), 0.0, atol=1e-12)        # deriv kills constants
    np.testing.assert_allclose((w[..., 1, :] * s).sum(-1), 1.0, atol=1e-12)  # deriv exact on linear data
    # ReLU net: every hidden activation is >= 0 -> the stencils differ from the base (learned path live)
    assert np.abs(w - O.default_base_stencils()).max() > 1e-2


@pytest.mark.parametrize("system", [0, 1])
def test_fixed_mode_equals_classical_fv(system):
    """Pin-1 (brute-force classical 2nd-order FV loops, forcing and drag)."""
    n = 8
    u = make_ic("noise", n, 2, seed=9)
    cfg = _cfg(n=n, system=system, nu=0.03, force_amp=0.7, force_k=2.0, drag=0.2)
    T = X.tendency(u, cfg)
    ref = _classical_fv_rhs(u, 0.03, TWO_PI / n, 0.5 if system == 0 else 1.0, 0.7, 2.0, 0.2)
    np.testing.assert_allclose(T, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("system", [0, 1])
def test_constant_field_zero_tendency_learned(system):
    """Pin-2."""
    n = 16
    cfg = _cfg(n=n, system=system, stencil_mode=0, nu=0.05)
    params = make_weights(3, 8, 24, seed=1, init="stress")
    u = np.ones((1, 2, n, n)) * np.array([0.3, -1.7])[None, :, None, None]
    assert np.abs(X.tendency(u, cfg, params)).max() < 1e-12


@pytest.mark.parametrize("n", [8, 64, 256])
def test_projection_divergence_free_idempotent(n):
    """Pin-4 (|D_c P u| < 1e-10 in fp64, idempotent, mean-preserving, non-expansive)."""
    h = TWO_PI / n
    cfg = _cfg(n=n)
    u = make_ic("noise", n, 2, seed=n)
    pu = X.project(u, cfg)
    d = ((np.roll(pu[:, 0], -1, -1) - np.roll(pu[:, 0], 1, -1)) + (np.roll(pu[:, 1], -1, -2) - np.roll(pu[:, 1], 1, -2))) / (2 * h)
    assert np.abs(d).max() < 1e-10
    np.testing.assert_allclose(X.project(pu, cfg), pu, atol=1e-12)
    np.testing.assert_allclose(pu.mean(axis=(-1, -2)), u.mean(axis=(-1, -2)), atol=1e-14)
    assert np.linalg.norm(pu) <= np.linalg.norm(u) * (1 + 1e-14)


def test_projection_matches_dense_bordered_solve_8x8():
    """Pin-5: P u = u - G_c p with p from Gaussian elimination on [A Z; Z^T 0], A = D_c G_c by loops."""
    n = 8
    h = TWO_PI / n
    idx = lambda j, i: (j % n) * n + (i % n)
    G = np.zeros((2 * n * n, n * n))
    D = np.zeros((n * n, 2 * n * n))
    for j in range(n):
        for i in range(n):
            r = idx(j, i)
            G[r, idx(j, i + 1)] += 1 / (2 * h); G[r, idx(j, i - 1)] -= 1 / (2 * h)
            G[n * n + r, idx(j + 1, i)] += 1 / (2 * h); G[n * n + r, idx(j - 1, i)] -= 1 / (2 * h)
            D[r, idx(j, i + 1)] += 1 / (2 * h); D[r, idx(j, i - 1)] -= 1 / (2 * h)
            D[r, n * n + idx(j + 1, i)] += 1 / (2 * h); D[r, n * n + idx(j - 1, i)] -= 1 / (2 * h)
    A = D @ G
    Z = np.zeros((n * n, 4))
    for j in range(n):
        for i in range(n):
            Z[idx(j, i)] = [1, (-1) ** i, (-1) ** j, (-1) ** (i + j)]
    u = make_ic("noise", n, 1, seed=3)
    K = np.block([[A, Z], [Z.T, np.zeros((4, 4))]])
    p = np.linalg.solve(K, np.concatenate([D @ u.reshape(-1), np.zeros(4)]))[:n * n]
    np.testing.assert_allclose(X.project(u, _cfg(n=n)), (u.reshape(-1) - G @ p).reshape(1, 2, n, n), atol=1e-12)


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("system", [0, 1])
def test_shear_mode_decay_factor(p, system):
    """Pin-7: u = (sin k y, 0) decays by R_p(-nu k_hat^2 dt), k_hat = 2 sin(kh/2)/h."""
    n, k, nu, dt = 32, 3, 0.05, 0.02
    Xc, Y, h = _centres(n)
    u0 = np.stack([np.sin(k * Y), np.zeros_like(Y)])[None]
    u1 = X.step(u0, _cfg(n=n, system=system, rk_order=p, nu=nu, dt=dt))
    kh = 2 * math.sin(k * h / 2) / h
    np.testing.assert_allclose(u1, _Rp(-nu * kh * kh * dt, p) * u0, atol=1e-14)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_taylor_green_one_step_exact(p):
    """Pin-8."""
    n, nu, dt = 32, 0.01, 0.05
    h = TWO_PI / n
    u0 = make_ic("taylor_green", n, 1)
    u1 = X.step(u0, _cfg(n=n, rk_order=p, nu=nu, dt=dt))
    k1 = 2 * math.sin(h / 2) / h
    np.testing.assert_allclose(u1, _Rp(-2 * nu * k1 * k1 * dt, p) * u0, atol=1e-14)


def test_kolmogorov_fixed_point():
    """Pin-9."""
    n, nu, chi, kf, alpha = 64, 1e-3, 1.0, 4, 0.1
    Xc, Y, h = _centres(n)
    kh = 2 * math.sin(kf * h / 2) / h
    A = chi / (nu * kh * kh + alpha)
    u0 = np.stack([A * np.sin(kf * Y), np.zeros_like(Y)])[None]
    cfg = _cfg(n=n, nu=nu, force_amp=chi, force_k=kf, drag=alpha, dt=0.5 * h / A)
    np.testing.assert_allclose(X.rollout(u0, cfg, None, 5), u0, atol=1e-13 * A)


@pytest.mark.parametrize("system", [0, 1])
def test_mean_momentum_conserved_learned(system):
    """Pin-10."""
    n = 16
    cfg = _cfg(n=n, system=system, stencil_mode=0, nu=0.01, dt=0.02, rk_order=3)
    params = make_weights(3, 8, 24, seed=5, init="stress")
    params[-24 * 9 * 8 - 24:] *= 0.05
    u0 = make_ic("fourier", n, 2, seed=1) + np.array([0.2, -0.1])[None, :, None, None]
    u = X.rollout(u0, cfg, params, 10)
    np.testing.assert_allclose(u.sum(axis=(-1, -2)), u0.sum(axis=(-1, -2)), atol=1e-11)


def test_translation_equivariance():
    """Pin-13 (with forcing: the y shift is a multiple of N / k_f)."""
    n = 16
    cfg = _cfg(n=n, system=1, stencil_mode=0, nu=0.01, dt=0.02, force_amp=0.5, force_k=2, drag=0.1, tc_head=1)
    params = make_weights(3, 8, 26, seed=3, init="stress")
    u0 = make_ic("noise", n, 1, seed=2)
    a = X.step(u0, cfg, params)
    b = X.step(np.roll(u0, (n // 2, 5), axis=(-2, -1)), cfg, params)
    np.testing.assert_allclose(np.roll(a, (n // 2, 5), axis=(-2, -1)), b, atol=1e-12)


@pytest.mark.parametrize("rk", [2, 3, 4])
@pytest.mark.parametrize("system", [0, 1])
def test_tc_term_from_stage1_net(rk, system):
    """R8 closed form (see tests/test_oracle_pins.py): e = u^n / 8 added before the last projection,
    and only at steps with (k+1) % k_c == 0."""
    n = 8
    u = make_ic("noise", n, 1, seed=11)
    kw = dict(n=n, system=system, nu=0.05, dt=0.1, rk_order=rk, n_layers=3, width=4, activation=0)
    plain = X.step(u, _cfg(stencil_mode=1, **kw))
    want = 0.125 * (u if system == 0 else X.project(u, _cfg(n=n)))
    cfg2 = _cfg(stencil_mode=0, tc_head=1, tc_interval=2, **kw)
    np.testing.assert_allclose(X.step(u, cfg2, _passthrough_tc_params(), step_index=1) - plain, want, atol=1e-12)
    np.testing.assert_allclose(X.step(u, cfg2, _passthrough_tc_params(), step_index=0), plain, atol=1e-13)


@pytest.mark.parametrize("rk", [2, 3, 4])
def test_burgers_step_is_unprojected_1d_burgers(rk):
    """R9: a compressible u = (f(x), 0) follows the 1-D viscous Burgers FV scheme, unprojected."""
    n, nu, dt = 16, 0.02, 0.05
    h = TWO_PI / n
    x = (np.arange(n) + 0.5) * h
    f = np.sin(x) + 0.3 * np.cos(3 * x) + 0.2
    u = np.zeros((1, 2, n, n))
    u[0, 0] = f[None, :]
    out = X.step(u, _cfg(n=n, system=0, nu=nu, dt=dt, rk_order=rk))
    R = lambda g: _burgers_1d_rhs(g, nu, h)
    if rk == 2:
        g1 = f + dt * R(f)
        ref = 0.5 * f + 0.5 * (g1 + dt * R(g1))
    elif rk == 3:
        g1 = f + dt * R(f)
        g2 = 0.75 * f + 0.25 * (g1 + dt * R(g1))
        ref = f / 3 + 2 / 3 * (g2 + dt * R(g2))
    else:
        k1 = R(f); k2 = R(f + dt / 2 * k1); k3 = R(f + dt / 2 * k2); k4 = R(f + dt * k3)
        ref = f + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    np.testing.assert_allclose(out[0, 0], np.broadcast_to(ref, (n, n)), atol=1e-13)
    assert np.abs(out[0, 1]).max() == 0.0


# ------------------------------------------------------- agreement with the independent numpy oracle

@pytest.mark.parametrize("name,n,B,rk,steps", [("c1", 16, 2, 2, 3), ("c2", 16, 2, 3, 2), ("c3", 16, 2, 3, 3),
                                               ("c4", 32, 1, 3, 2), ("c2", 8, 3, 4, 2)])
def test_agrees_with_numpy_oracle(name, n, B, rk, steps):
    cfg = get_config(name, n=n, batch=B, rk_order=rk, tc_interval=2)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=1, init="stress")
    ref = O.rollout(u0, cfg, params, steps)
    got = X.rollout(u0, cfg, params, steps)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12
    np.testing.assert_allclose(X.stencils(u0, cfg, params).reshape(B, n, n, 2, 2, 6),
                               O.constrain(O.net_forward(u0, O.unpack_params(params, cfg.n_layers, cfg.width,
                                                                              cfg.n_out), cfg.activation)),
                               atol=1e-12)


def test_fp32_variant_and_thread_independence():
    cfg = get_config("c3", n=16, batch=3)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=1, init="stress")
    ref = X.step(u0, cfg, params, threads=1)
    for th in (2, 3, 8):      # element-parallel (B >= threads) and row-parallel (B < threads) forms
        assert np.array_equal(X.step(u0, cfg, params, threads=th), ref)
    f32 = X.step(u0, cfg, params, precision=1)
    err = np.linalg.norm(f32 - ref) / np.linalg.norm(ref)
    assert 1e-9 < err < 1e-5, err        # fp32 arithmetic: a real difference, within the fp32 parity bound


def test_nonfinite_reported_with_step_index():
    cfg = _cfg(n=8, system=0, nu=0.0, dt=1e3, rk_order=2)
    with pytest.raises(FloatingPointError, match="step"):
        X.rollout(make_ic("noise", 8, 1, seed=0) * 10, cfg, None, 200)
