"""Pins of the frequency-domain operator oracle (oracle/spectral_oracle.py; Eq. 8,
P:252-256; readings N2-1..N2-4 in DESIGN.md §8c).

Each check compares against something the mathematics fixes independently of the oracle's
own FFT routine: closed forms for single Fourier modes (including a phase, which fixes the
sign convention of F versus F^{-1} and the conjugate extension), a brute-force O(N^4) DFT
truncation on 8 x 8, exact zero output for modes above K, shift equivariance (the operator
is a per-mode multiplier, so it commutes with periodic translations), linearity and the
composition of layers."""
import numpy as np
import pytest

import oracle as O
from ldgen.spectral import half_plane_modes, make_spectral_params, n_modes


def _diag_params(K, C, value, L=1):
    R = []
    for _ in range(L):
        a = np.zeros((n_modes(K), C, C, 2), dtype=np.float64)
        for c in range(C):
            a[:, c, c, 0] = np.real(value)
            a[:, c, c, 1] = np.imag(value)
        a[half_plane_modes(K).index((0, 0)), :, :, 1] = 0.0
        R.append(a)
    return R


def _mode_field(N, kx, ky, phase=0.0):
    y, x = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    return np.cos(2 * np.pi * (kx * x + ky * y) / N + phase)


def test_zero_input_gives_zero():
    R, Q = make_spectral_params(3, 4, 2)
    assert np.all(O.spectral_operator(np.zeros((1, 2, 16, 16)), R, Q, 3) == 0.0)


@pytest.mark.parametrize("kx,ky", [(1, 0), (0, 2), (2, -3), (3, 3)])
def test_single_mode_scaled_by_two(kx, ky):
    N, K = 16, 3
    u = np.zeros((1, 2, N, N))
    u[0, 0] = _mode_field(N, kx, ky)
    u[0, 1] = 0.5 * _mode_field(N, kx, ky, 0.3)
    Q = np.eye(8, 2)
    out = O.spectral_operator(u, _diag_params(K, 2, 2.0), Q, K)
    assert np.allclose(out[0, 0], 2 * u[0, 0], atol=1e-12)
    assert np.allclose(out[0, 1], 2 * u[0, 1], atol=1e-12)
    assert np.all(np.abs(out[0, 2:]) < 1e-12)


@pytest.mark.parametrize("phi", [0.25, -1.0, np.pi / 2])
def test_phase_rotation_closed_form(phi):
    """R(k) = e^{i phi} on the half plane (e^{-i phi} on its mirror): cos(theta) -> cos(theta + phi)
    for a mode with kx > 0 -- fixes F's sign convention and the conjugate extension."""
    N, K = 16, 4
    u = np.zeros((1, 2, N, N))
    u[0, 0] = _mode_field(N, 2, -1)
    R = _diag_params(K, 2, np.exp(1j * phi))
    out = O.spectral_operator(u, R, np.eye(8, 2), K)
    assert np.allclose(out[0, 0], _mode_field(N, 2, -1, phi), atol=1e-12)


def test_modes_above_K_are_discarded():
    N, K = 16, 3
    u = np.zeros((1, 2, N, N))
    u[0, 0] = _mode_field(N, K + 1, 0) + _mode_field(N, 1, K + 2, 0.7)
    u[0, 1] = _mode_field(N, 0, K + 1)
    R, Q = make_spectral_params(K, 4, 2, seed=3)
    assert np.max(np.abs(O.spectral_operator(u, R, Q, K))) < 1e-12


def test_identity_layer_is_brute_force_truncation():
    """R = I, Q = I: O_F(u) is u with every mode outside |kx|, |ky| <= K removed, here computed
    by explicit O(N^4) DFT sums (no FFT)."""
    N, K = 8, 2
    rng = np.random.default_rng(5)
    u = rng.standard_normal((1, 2, N, N))
    out = O.spectral_operator(u, _diag_params(K, 2, 1.0), np.eye(8, 2), K)
    ref = np.zeros((2, N, N))
    idx = np.arange(N)
    for c in range(2):
        for ky in range(-K, K + 1):
            for kx in range(-K, K + 1):
                coef = sum(u[0, c, y, x] * np.exp(-2j * np.pi * (kx * x + ky * y) / N)
                           for y in range(N) for x in range(N))
                ref[c] += np.real(coef * np.exp(2j * np.pi * (kx * idx[None, :] + ky * idx[:, None]) / N)) / N**2
    assert np.allclose(out[0, :2], ref, atol=1e-12)


def test_shift_equivariance_and_linearity():
    N, K = 16, 4
    rng = np.random.default_rng(9)
    u1, u2 = rng.standard_normal((2, 1, 2, N, N))
    R, Q = make_spectral_params(K, 6, 2, seed=1)
    o1 = O.spectral_operator(u1, R, Q, K)
    sh = np.roll(np.roll(u1, 3, axis=-1), -5, axis=-2)
    assert np.allclose(O.spectral_operator(sh, R, Q, K), np.roll(np.roll(o1, 3, axis=-1), -5, axis=-2), atol=1e-10)
    o2 = O.spectral_operator(u2, R, Q, K)
    assert np.allclose(O.spectral_operator(2 * u1 - 3 * u2, R, Q, K), 2 * o1 - 3 * o2, atol=1e-10)


def test_layers_compose_per_mode():
    """Two layers equal one layer whose per-mode matrix is R2(k) R1(k)."""
    N, K, C = 16, 3, 3
    R, Q = make_spectral_params(K, C, 2, seed=2)
    c1 = R[0][..., 0].astype(np.float64) + 1j * R[0][..., 1]
    c2 = R[1][..., 0].astype(np.float64) + 1j * R[1][..., 1]
    prod = np.einsum("moc,mci->moi", c2, c1)
    Rp = np.stack([prod.real, prod.imag], axis=-1)
    u = np.random.default_rng(4).standard_normal((2, 2, N, N))
    assert np.allclose(O.spectral_operator(u, R, Q, K), O.spectral_operator(u, [Rp], Q, K), atol=1e-10)


def test_K_validation():
    with pytest.raises(ValueError):
        O.spectral_operator(np.zeros((1, 2, 8, 8)), _diag_params(4, 2, 1.0), np.eye(8, 2), 4)


# ---------------------------------------------------------------- NEXT-2b: O_F inside the step

def _fno_cfg(**kw):
    from ldgen.configs import get_config
    base = dict(n=16, batch=2, fno_kmax=4, fno_layers=2, fno_width=3)
    base.update(kw)
    cfg = get_config("c2", **base)
    return cfg.replace(dt=0.01)


def _fno_params(cfg, scale=1.0, seed=0):
    from ldgen import make_weights
    from ldgen.spectral import spectral_blob
    conv = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=seed, init="stress")
    return np.concatenate([conv, spectral_blob(cfg.fno_kmax, cfg.fno_width, cfg.fno_layers, seed=seed + 1,
                                               scale=scale)])


def test_face_shift_closed_form():
    """Identity layers: the x-face channels are the mode at x - h/2, the y-face ones at y - h/2."""
    N, K = 16, 3
    u = np.zeros((1, 2, N, N))
    u[0, 0] = _mode_field(N, 2, 1)
    Q = np.zeros((8, 2))
    Q[0, 0] = Q[4, 0] = 1.0
    out = O.spectral_faces(u, _diag_params(K, 2, 1.0), Q, K)
    y, x = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    assert np.allclose(out[0, 0], np.cos(2 * np.pi * (2 * (x - 0.5) + y) / N), atol=1e-12)
    assert np.allclose(out[0, 4], np.cos(2 * np.pi * (2 * x + (y - 0.5)) / N), atol=1e-12)


def test_step_with_zero_spectral_params_equals_plain_step():
    cfg = _fno_cfg()
    p = _fno_params(cfg, scale=0.0)
    p[-8 * cfg.fno_width:] = 0.0
    u = np.random.default_rng(1).standard_normal((2, 2, 16, 16))
    plain = cfg.replace(fno_layers=0)
    from ldgen import make_weights
    conv = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="stress")
    assert np.array_equal(O.step(u, cfg, p), O.step(u, plain, conv))


def test_step_with_fno_conserves_momentum_and_commutes_with_shifts():
    """Flux form: the face terms telescope, so sum(u), sum(v) are conserved with O_F on (unforced);
    O_F is a per-mode multiplier, so the whole step commutes with periodic translations."""
    cfg = _fno_cfg(system=1)
    p = _fno_params(cfg, scale=0.3)
    u = np.random.default_rng(2).standard_normal((2, 2, 16, 16))
    out = O.step(u, cfg, p)
    assert np.allclose(out.sum(axis=(-2, -1)), u.sum(axis=(-2, -1)), atol=1e-10)
    sh = lambda a: np.roll(np.roll(a, 3, axis=-1), -5, axis=-2)
    assert np.allclose(O.step(sh(u), cfg, p), sh(out), atol=1e-10)
    # and O_F changes the step (the branch is live)
    from ldgen import make_weights
    conv = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="stress")
    assert np.max(np.abs(out - O.step(u, cfg.replace(fno_layers=0), conv))) > 1e-6


# ---------------------------------------------------------------- NEXT-3: history TC block

def _tc_cfg(kc=3, **kw):
    from ldgen.configs import get_config
    base = dict(n=16, batch=2, tc_head=0, tc_mode=1, tc_interval=kc, tc_kmax=4, tc_layers=2, tc_width=4)
    base.update(kw)
    return get_config("c3", **base).replace(dt=0.01)


def _tc_params(cfg, scale=0.3, zero=False):
    from ldgen import make_weights
    from ldgen.spectral import spectral_blob
    conv = make_weights(cfg.n_layers, cfg.width, 24, seed=0, init="stress")
    tc = spectral_blob(cfg.tc_kmax, cfg.tc_width, cfg.tc_layers, seed=2, scale=scale,
                       n_in=2 * cfg.tc_interval, n_out=2)
    return conv, np.concatenate([conv, 0 * tc if zero else tc])


def test_history_tc_only_acts_every_kc_steps():
    """Eq. 2: before the first multiple of k_c the trajectory is the plain FV one; a
    zero operator never changes it."""
    cfg = _tc_cfg(kc=3)
    conv, p = _tc_params(cfg)
    plain = cfg.replace(tc_mode=0)
    u = np.random.default_rng(3).standard_normal((2, 2, 16, 16))
    assert np.array_equal(O.rollout(u, cfg, p, 2), O.rollout(u, plain, conv, 2))
    assert not np.allclose(O.rollout(u, cfg, p, 3), O.rollout(u, plain, conv, 3))
    _, pz = _tc_params(cfg, zero=True)
    assert np.array_equal(O.rollout(u, cfg, pz, 7), O.rollout(u, plain, conv, 7))


def test_history_tc_correction_is_projected_lowpass_of_newest_state():
    """One layer, R = I on the retained modes, Q picking the newest input's (u, v) with weight a:
    e = a * lowpass_K(u_k) and, the projection being linear, u_{k+1} - FV(u_k) = a P(lowpass_K(u_k))
    (the correction enters before the last projection, reading R8 / N3-3)."""
    from ldgen.spectral import half_plane_modes, n_modes
    kc, K, a = 2, 3, 0.7
    cfg = _tc_cfg(kc=kc, tc_kmax=K, tc_layers=1, tc_width=2 * kc)
    conv, _ = _tc_params(cfg)
    C = 2 * kc
    R = np.zeros((n_modes(K), C, C, 2))
    for c in range(C):
        R[:, c, c, 0] = 1.0
    Q = np.zeros((2, C))
    Q[0, C - 2] = Q[1, C - 1] = a
    p = np.concatenate([conv, R.ravel(), Q.ravel()])
    u0 = np.random.default_rng(4).standard_normal((2, 2, 16, 16))
    o = O.Oracle(cfg, p)
    u1 = o.step(u0)                       # k = 0: buffer [u0], no correction (1 % 2 != 0)
    u2 = o.step(u1)                       # k = 1: correction from [u0, u1]
    plain = O.Oracle(cfg.replace(tc_mode=0), conv)
    plain.step_index = 1
    fv = plain.step(u1)
    m = np.fft.fftfreq(16, d=1.0 / 16)
    mask = (np.abs(m)[:, None] <= K) & (np.abs(m)[None, :] <= K)
    low = np.real(np.fft.ifft2(np.fft.fft2(u1, axes=(-2, -1)) * mask, axes=(-2, -1)))
    assert np.allclose(u2 - fv, a * O.project(low, cfg.h), atol=1e-10)
