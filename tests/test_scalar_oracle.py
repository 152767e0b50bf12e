"""Pins of the passive-scalar transport in the oracle (the shear flow "requires solving a
coupled advection-diffusion equation alongside the NSE"; readings S1-S4 in DESIGN.md §8h).

Each pin compares with something other than the oracle's own formula: hand-written classical FV loops,
the closed-form decay of a diffusing Fourier mode under the RK stability polynomial, exact invariants
(uniform scalar in a discretely solenoidal flow, conservation of the scalar mass), one-way coupling and
translation equivariance."""
import math

import numpy as np
import pytest

import oracle as O
from ldgen import make_ic, make_weights
from ldgen.configs import get_config
from ldgen.ic import make_config_ic, make_scalar_ic
from tests.test_oracle_pins import TWO_PI, _Rp, _centres, _cfg


def _fv_scalar_rhs(U, S, D, h):
    """Classical 2nd-order FV scalar tendency, loops: face value (c(i-1) + c(i)) / 2, gradient (c(i) - c(i-1)) / h."""
    B, _, n, _ = U.shape
    T = np.zeros_like(S)
    for b in range(B):
        for j in range(n):
            for i in range(n):
                def fx(ii):
                    uf = 0.5 * (U[b, 0, j, (ii - 1) % n] + U[b, 0, j, ii % n])
                    sf = 0.5 * (S[b, j, (ii - 1) % n] + S[b, j, ii % n])
                    return uf * sf - D * (S[b, j, ii % n] - S[b, j, (ii - 1) % n]) / h

                def fy(jj):
                    vf = 0.5 * (U[b, 1, (jj - 1) % n, i] + U[b, 1, jj % n, i])
                    sf = 0.5 * (S[b, (jj - 1) % n, i] + S[b, jj % n, i])
                    return vf * sf - D * (S[b, jj % n, i] - S[b, (jj - 1) % n, i]) / h
                T[b, j, i] = -(fx(i + 1) - fx(i) + fy(j + 1) - fy(j)) / h
    return T


def test_fixed_stencils_equal_classical_fv():
    n, D = 8, 0.03
    h = TWO_PI / n
    U = make_ic("noise", n, 2, seed=1)
    S = np.random.default_rng(2).standard_normal((2, n, n))
    w = np.broadcast_to(O.default_base_stencils(), (2, n, n, 2, 2, 6))
    np.testing.assert_allclose(O.scalar_tendency(U, S, w, D, h), _fv_scalar_rhs(U, S, D, h), atol=1e-12)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_diffusing_mode_at_rest(p):
    """u = 0: s = sin(k x) decays by R_p(-D k_hat^2 dt), k_hat = 2 sin(kh/2)/h (fixed central stencils)."""
    n, k, D, dt = 32, 3, 0.05, 0.02
    Xc, Y, h = _centres(n)
    s0 = np.sin(k * Xc)[None]
    cfg = _cfg(n=n, rk_order=p, nu=0.01, dt=dt, scalar_diff=D)
    u1, s1 = O.Oracle(cfg).step_scalar(np.zeros((1, 2, n, n)), s0)
    kh = 2 * math.sin(k * h / 2) / h
    np.testing.assert_allclose(s1, _Rp(-D * kh * kh * dt, p) * s0, atol=1e-14)
    assert np.abs(u1).max() == 0.0


def test_uniform_scalar_in_solenoidal_flow_is_steady():
    """Central stencils: the face-velocity divergence equals D_c u, which P makes zero, so a uniform
    scalar has zero tendency at every stage (SPEC.md's "uniform scalar, any solenoidal velocity")."""
    n = 32
    h = TWO_PI / n
    u = O.project(make_ic("spectrum", n, 1, seed=4), h)
    cfg = _cfg(n=n, nu=1e-3, dt=0.5 * h, scalar_diff=0.01)
    _, s1 = O.Oracle(cfg).step_scalar(u, np.full((1, n, n), 0.37))
    np.testing.assert_allclose(s1, 0.37, atol=1e-13)


@pytest.mark.parametrize("rk", [2, 3, 4])
def test_scalar_mass_conserved_learned(rk):
    cfg = get_config("c4", n=16, batch=2, rk_order=rk, scalar_mode=1, scalar_diff=5e-4)
    u = make_config_ic(cfg)
    cfg = cfg.with_dt(u)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=2, init="stress")
    s = make_scalar_ic(16, 2) + np.random.default_rng(3).standard_normal((2, 16, 16)) * 0.1
    o = O.Oracle(cfg, params)
    u1, s1 = o.step_scalar(u, s)
    np.testing.assert_allclose(s1.sum(axis=(-1, -2)), s.sum(axis=(-1, -2)), atol=1e-11)
    assert np.abs(s1 - s).max() > 1e-4                      # it did move
    np.testing.assert_array_equal(u1, O.step(u, cfg, params))   # one-way coupling: momentum unchanged


def test_scalar_translation_equivariance():
    cfg = get_config("c4", n=16, batch=1, scalar_mode=1, scalar_diff=1e-3, dt=0.02)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=2, init="stress")
    rng = np.random.default_rng(5)
    u = rng.standard_normal((1, 2, 16, 16)) * 0.3
    s = rng.standard_normal((1, 16, 16))
    _, a = O.Oracle(cfg, params).step_scalar(u, s)
    sh = (4, 7)
    _, b = O.Oracle(cfg, params).step_scalar(np.roll(u, sh, axis=(-2, -1)), np.roll(s, sh, axis=(-2, -1)))
    np.testing.assert_allclose(np.roll(a, sh, axis=(-2, -1)), b, atol=1e-12)
