"""Pins of the paper's constant 5x4 face kernels in the oracle (O_P^(m) + O_L^(m) =
(W_P + W_L) * u, W in R^{5x4}, "central differencing for derivatives ... linear interpolation", W_L
"initialized with minor random values"; readings F1-F3 in DESIGN.md §8i).  Each pin compares with a
hand-written construction, a closed-form Fourier symbol, exactness on linear data, or an invariant."""
import math

import numpy as np
import pytest

import oracle as O
from ldgen import make_ic
from tests.test_oracle_pins import TWO_PI, _cfg, _classical_fv_rhs


def _wl(seed, scale=0.3):
    return np.random.default_rng(seed).standard_normal(80) * scale


@pytest.mark.parametrize("system", [0, 1])
def test_zero_learned_part_is_classical_fv(system):
    n = 8
    u = make_ic("noise", n, 2, seed=3)
    cfg = _cfg(n=n, system=system, stencil_mode=2, nu=0.03, force_amp=0.7, force_k=2.0, drag=0.2)
    T, _ = O.Oracle(cfg, np.zeros(80, dtype=np.float32)).T(u)
    np.testing.assert_allclose(T, _classical_fv_rhs(u, 0.03, TWO_PI / n, 0.5 if system == 0 else 1.0, 0.7, 2.0, 0.2),
                               atol=1e-12)


def test_fourier_symbol_of_a_face_kernel():
    n, kx, ky = 16, 3, 2
    h = TWO_PI / n
    x = (np.arange(n) + 0.5) * h
    X, Y = np.meshgrid(x, x, indexing="xy")
    W = np.random.default_rng(1).standard_normal((5, 4))
    c = np.exp(1j * (kx * X + ky * Y))
    for axis in (-1, -2):
        got = O.face_values_5x4(c.real, W, axis) + 1j * O.face_values_5x4(c.imag, W, axis)
        if axis == -1:   # taps (j - 2 + b, i - 2 + a)
            sym = sum(W[b, a] * np.exp(1j * (kx * (a - 2) + ky * (b - 2)) * h) for b in range(5) for a in range(4))
        else:            # taps (j - 2 + a, i - 2 + b)
            sym = sum(W[b, a] * np.exp(1j * (ky * (a - 2) + kx * (b - 2)) * h) for b in range(5) for a in range(4))
        np.testing.assert_allclose(got, sym * c, atol=1e-12)


def test_constrained_kernels_exact_on_constants_and_linear_fields():
    """Interp of a constant is the constant; the derivative of any linear field alpha x + beta y at an
    x-face is alpha (y-face: beta) -- checked on a non-periodic 5x4 window, for random W_L."""
    W = O.constrain_5x4(_wl(2))
    h = 0.37
    alpha, beta = 1.3, -0.6
    for ax in range(2):
        A = np.arange(4) - 1.5           # normal offsets of the taps from the face, in cells
        Bt = np.arange(5) - 2.0          # tangential offsets
        normal, tang = (alpha, beta) if ax == 0 else (beta, alpha)
        lin = np.array([[normal * A[a] * h + tang * Bt[b] * h + 0.8 for a in range(4)] for b in range(5)])
        assert abs(np.sum(W[ax, 0]) - 1.0) < 1e-13
        assert abs(np.sum(W[ax, 1] * lin) / h - normal) < 1e-12


@pytest.mark.parametrize("system", [0, 1])
def test_invariants_with_learned_kernels(system):
    n = 16
    cfg = _cfg(n=n, system=system, stencil_mode=2, nu=0.01, dt=0.02)
    p = _wl(4, 0.05).astype(np.float32)
    u0 = make_ic("fourier", n, 2, seed=1) + np.array([0.2, -0.1])[None, :, None, None]
    u = O.rollout(u0, cfg, p, 5)
    np.testing.assert_allclose(u.sum(axis=(-1, -2)), u0.sum(axis=(-1, -2)), atol=1e-11)   # mean momentum
    c = np.ones((1, 2, n, n)) * np.array([0.3, -0.7])[None, :, None, None]
    np.testing.assert_allclose(O.step(c, cfg, p), c, atol=1e-13)                           # constant state
    s = (5, 3)
    a = O.step(u0[:1], cfg, p)
    b = O.step(np.roll(u0[:1], s, axis=(-2, -1)), cfg, p)
    np.testing.assert_allclose(np.roll(a, s, axis=(-2, -1)), b, atol=1e-12)
    assert not np.allclose(a, O.step(u0[:1], cfg, np.zeros(80, dtype=np.float32)))          # W_L acts
