"""Pins of the adjoint (VJP) oracle of one step (oracle/adjoint_oracle.py, SURVEY.md §8f NEXT-4;
PAPER.md P:141 "fully differentiable", training loss P:348-352).

Each check compares it with something other than itself: torch autograd of conv2d (the conv
pieces), central finite differences of the independent forward oracle in fp64 (dot-product tests
<u_bar, du> = d/de <g, step(u + e du)> and the same for theta), and closed forms (at u = 0 with
fixed stencils the step is linear and symmetric, so its VJP is the step itself -- for a shear mode
the factor R_p(z); a uniform cotangent is conserved when the mean momentum is).
"""
import math

import numpy as np
import pytest

import oracle as O
from ldgen import make_ic, make_weights
from ldgen.configs import get_config
from ldgen.ic import make_config_ic
from oracle import adjoint_oracle as A
from tests.test_oracle_pins import TWO_PI, _Rp, _centres, _cfg


def test_conv_transpose_and_wgrad_match_torch_autograd():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    B, N, Ci, Co = 2, 6, 3, 4
    H = rng.standard_normal((B, N, N, Ci))
    W = rng.standard_normal((Co, 3, 3, Ci))
    G = rng.standard_normal((B, N, N, Co))
    x = torch.tensor(np.moveaxis(H, -1, 1), requires_grad=True)
    w = torch.tensor(W.transpose(0, 3, 1, 2).copy(), requires_grad=True)
    y = torch.nn.functional.conv2d(torch.nn.functional.pad(x, (1, 1, 1, 1), mode="circular"), w)
    (y * torch.tensor(np.moveaxis(G, -1, 1))).sum().backward()
    np.testing.assert_allclose(A.conv3x3_transpose(G, W), np.moveaxis(x.grad.numpy(), 1, -1), atol=1e-12)
    np.testing.assert_allclose(A.conv3x3_wgrad(H, G), w.grad.numpy().transpose(0, 2, 3, 1), atol=1e-12)


def test_gelu_grad_matches_torch():
    torch = pytest.importorskip("torch")
    x = torch.linspace(-5, 5, 101, dtype=torch.float64, requires_grad=True)
    torch.nn.functional.gelu(x, approximate="none").sum().backward()
    np.testing.assert_allclose(A.gelu_grad(x.detach().numpy()), x.grad.numpy(), atol=1e-14)


def _fd_dot(cfg, params, u, g, du=None, dp=None, k=0, eps=1e-6):
    """Central difference of <g, step(u + e du, p + e dp)> at e = 0 (fp64 forward oracle)."""
    def f(e):
        uu = u if du is None else u + e * du
        pp = params if dp is None else (params.astype(np.float64) + e * dp)
        o = O.Oracle(cfg, pp)
        o.step_index = k
        return float(np.sum(g * o.step(uu)))
    return (f(eps) - f(-eps)) / (2 * eps)


@pytest.mark.parametrize("name,rk,k", [("c1", 2, 0), ("c2", 3, 0), ("c3", 3, 0), ("c3", 4, 0), ("c4", 3, 0)])
def test_dot_product_state(name, rk, k):
    """<u_bar, du> equals the directional derivative of <g, step(u)> (fp64 central differences)."""
    cfg = get_config(name, n=8, batch=2, rk_order=rk, width=8, tc_interval=1)
    u = make_config_ic(cfg)
    cfg = cfg.with_dt(u)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=2, init="stress").astype(np.float64)
    rng = np.random.default_rng(1)
    g = rng.standard_normal(u.shape)
    du = rng.standard_normal(u.shape)
    ub, _ = A.step_vjp(u, cfg, params, g, step_index=k)
    lhs = float(np.sum(ub * du))
    rhs = _fd_dot(cfg, params, u, g, du=du, k=k)
    assert abs(lhs - rhs) < 1e-7 * max(1.0, abs(rhs)), (lhs, rhs)


@pytest.mark.parametrize("name,rk", [("c2", 3), ("c3", 3), ("c1", 2), ("c3", 4)])
def test_dot_product_params(name, rk):
    """<theta_bar, dtheta> equals the directional derivative of <g, step(u; theta)> (TC head on:
    the e path is included; tc_interval 1 so e is added)."""
    cfg = get_config(name, n=8, batch=2, rk_order=rk, width=8, tc_interval=1)
    u = make_config_ic(cfg)
    cfg = cfg.with_dt(u)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=3, init="stress").astype(np.float64)
    rng = np.random.default_rng(4)
    g = rng.standard_normal(u.shape)
    dp = rng.standard_normal(params.shape)
    _, pb = A.step_vjp(u, cfg, params, g)
    assert pb.shape == params.shape
    lhs = float(np.sum(pb * dp))
    rhs = _fd_dot(cfg, params, u, g, dp=dp)
    assert abs(lhs - rhs) < 1e-7 * max(1.0, abs(rhs)), (lhs, rhs)


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("system", [0, 1])
def test_vjp_at_rest_is_the_linear_step(p, system):
    """At u = 0 with fixed central stencils the step is the linear diffusion step (advection is
    quadratic), a symmetric Fourier multiplier commuting with P: its VJP on the shear mode
    g = (sin k y, 0) is R_p(-nu k_hat^2 dt) g (Pin-7's factor)."""
    n, k, nu, dt = 16, 3, 0.05, 0.02
    Xc, Y, h = _centres(n)
    g = np.stack([np.sin(k * Y), np.zeros_like(Y)])[None]
    ub, _ = A.step_vjp(np.zeros_like(g), _cfg(n=n, system=system, rk_order=p, nu=nu, dt=dt), None, g)
    kh = 2 * math.sin(k * h / 2) / h
    np.testing.assert_allclose(ub, _Rp(-nu * kh * kh * dt, p) * g, atol=1e-14)


@pytest.mark.parametrize("system", [0, 1])
def test_uniform_cotangent_is_conserved(system):
    """sum(u^{n+1}) = sum(u^n) per component for any weights (no forcing / drag / TC; Pin-10), so a
    uniform cotangent is mapped to itself and theta gets no gradient from it."""
    cfg = _cfg(n=8, system=system, stencil_mode=0, nu=0.02, dt=0.05, n_layers=3, width=8)
    params = make_weights(3, 8, 24, seed=5, init="stress").astype(np.float64)
    u = make_ic("noise", 8, 2, seed=3)
    g = np.ones_like(u) * np.array([0.7, -1.3])[None, :, None, None]
    ub, pb = A.step_vjp(u, cfg, params, g)
    np.testing.assert_allclose(ub, g, atol=1e-12)
    assert np.abs(pb).max() < 1e-10


def test_translation_equivariance():
    cfg = _cfg(n=16, system=1, stencil_mode=0, nu=0.01, dt=0.02, tc_head=1, n_layers=3, width=8)
    params = make_weights(3, 8, 26, seed=3, init="stress").astype(np.float64)
    rng = np.random.default_rng(7)
    u = rng.standard_normal((1, 2, 16, 16))
    g = rng.standard_normal((1, 2, 16, 16))
    a, pa = A.step_vjp(u, cfg, params, g)
    s = (3, 5)
    b, pb = A.step_vjp(np.roll(u, s, axis=(-2, -1)), cfg, params, np.roll(g, s, axis=(-2, -1)))
    np.testing.assert_allclose(np.roll(a, s, axis=(-2, -1)), b, atol=1e-11)
    np.testing.assert_allclose(pa, pb, atol=1e-10)


def test_tc_gating_changes_only_at_correction_steps():
    """With k_c = 2, step 0 adds no e: theta_bar of the step equals that of the same net without the
    e channels' contribution; at step 1 the e channels receive P(g)-shaped gradient."""
    cfg = get_config("c3", n=8, batch=1, width=8, tc_interval=2)
    u = make_config_ic(cfg)
    cfg = cfg.with_dt(u)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=1, init="stress").astype(np.float64)
    g = np.random.default_rng(0).standard_normal(u.shape)
    _, p0 = A.step_vjp(u, cfg, params, g, step_index=0)
    _, p1 = A.step_vjp(u, cfg, params, g, step_index=1)
    # the last layer's bias entries of e (channels 24, 25): zero gradient without the correction,
    # sum over cells of P(g) with it (d e / d b_e = 1 everywhere; e enters before the final P)
    nb = p0.size - 26
    assert np.abs(p0[nb + 24:nb + 26]).max() == 0.0
    Pg = O.project(g, cfg.h)
    np.testing.assert_allclose(p1[nb + 24:nb + 26], Pg.sum(axis=(0, 2, 3)), atol=1e-10)
