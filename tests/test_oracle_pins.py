"""Pins of the CPU oracle against things the paper and the mathematics fix.

None of these re-types the oracle's own formula: each compares the oracle with
a closed form, a library routine, an invariant, or a brute-force construction
written independently here.  Citation keys: P:n = PAPER.md line, Rk/Pin-k =
SURVEY.md §8c readings / pins (restated in DESIGN.md).
"""
import math

import numpy as np
import pytest

import oracle as O
from ldgen import make_ic, make_weights
from ldgen.configs import get_config

TWO_PI = 2.0 * math.pi


def _cfg(**kw):
    base = dict(n=16, batch=1, system=1, nu=0.01, dt=0.01, rk_order=3, force_amp=0.0,
                force_k=0.0, drag=0.0, n_layers=3, width=8, activation=1, tc_head=0,
                tc_interval=1, stencil_mode=1, length=TWO_PI)
    base.update(kw)
    return base


def _centres(n):
    h = TWO_PI / n
    x = (np.arange(n) + 0.5) * h
    X, Y = np.meshgrid(x, x, indexing="xy")
    return X, Y, h


# ---------------------------------------------------------------------------
# Net: conv = torch Conv2d cross-correlation with circular padding; GELU = erf GELU
# ---------------------------------------------------------------------------

def test_conv_matches_torch_circular_conv2d():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    B, N, Ci, Co = 2, 7, 3, 5
    H = rng.standard_normal((B, N, N, Ci))
    W = rng.standard_normal((Co, 3, 3, Ci))
    b = rng.standard_normal(Co)
    got = O.conv3x3_periodic(H, W, b)
    x = torch.from_numpy(np.moveaxis(H, -1, 1).copy())
    xp = torch.nn.functional.pad(x, (1, 1, 1, 1), mode="circular")
    ref = torch.nn.functional.conv2d(xp, torch.from_numpy(W.transpose(0, 3, 1, 2).copy()),
                                     torch.from_numpy(b))
    np.testing.assert_allclose(got, np.moveaxis(ref.numpy(), 1, -1), rtol=1e-13, atol=1e-13)


def test_conv_bruteforce_tiny():
    """Direct quadruple loop on a 3x3 grid (brute force on tiny input)."""
    rng = np.random.default_rng(2)
    N, Ci, Co = 3, 2, 2
    H = rng.standard_normal((1, N, N, Ci))
    W = rng.standard_normal((Co, 3, 3, Ci))
    b = rng.standard_normal(Co)
    got = O.conv3x3_periodic(H, W, b)
    for j in range(N):
        for i in range(N):
            for o in range(Co):
                s = b[o]
                for ky in range(3):
                    for kx in range(3):
                        for c in range(Ci):
                            s += W[o, ky, kx, c] * H[0, (j + ky - 1) % N, (i + kx - 1) % N, c]
                assert abs(got[0, j, i, o] - s) < 1e-12


@pytest.mark.parametrize("activation", [0, 1])
def test_net_forward_bruteforce_tiny(activation):
    """The whole net from the packed blob, by explicit loops over the documented blob layout
    (W_l[co][ky][kx][ci] then b_l[co], layer order; include/ldsolver.h) with the activation on
    every layer but the last (math.erf GELU / ReLU) -- pins unpacking, layer order, activation
    placement and the periodic 3x3 taps together."""
    import math
    rng = np.random.default_rng(7)
    N, L, Wd, n_out = 4, 3, 3, 5
    chans = [2] + [Wd] * (L - 1) + [n_out]
    blob = rng.standard_normal(sum(co * 9 * ci + co for ci, co in zip(chans[:-1], chans[1:])))
    U = rng.standard_normal((1, 2, N, N))
    got = O.net_forward(U, O.unpack_params(blob, L, Wd, n_out), activation)
    H = [[[U[0, c, j, i] for c in range(2)] for i in range(N)] for j in range(N)]   # H[j][i][c]
    off = 0
    for l in range(L):
        ci, co = chans[l], chans[l + 1]
        Wb = blob[off:off + co * 9 * ci]
        off += co * 9 * ci
        bb = blob[off:off + co]
        off += co
        out = [[[0.0] * co for _ in range(N)] for _ in range(N)]
        for j in range(N):
            for i in range(N):
                for o in range(co):
                    s = bb[o]
                    for ky in range(3):
                        for kx in range(3):
                            for c in range(ci):
                                s += Wb[((o * 3 + ky) * 3 + kx) * ci + c] * H[(j + ky - 1) % N][(i + kx - 1) % N][c]
                    if l < L - 1:
                        s = 0.5 * s * (1.0 + math.erf(s / math.sqrt(2.0))) if activation == 1 else max(s, 0.0)
                    out[j][i][o] = s
        H = out
    for j in range(N):
        for i in range(N):
            for o in range(n_out):
                assert abs(got[0, j, i, o] - H[j][i][o]) < 1e-12


def test_gelu_exact_erf():
    torch = pytest.importorskip("torch")
    x = np.linspace(-6, 6, 1001)
    ref = torch.nn.functional.gelu(torch.from_numpy(x), approximate="none").numpy()
    np.testing.assert_allclose(O.gelu(x), ref, rtol=1e-14, atol=1e-15)
    assert O.gelu(np.array([0.0]))[0] == 0.0


def test_unpack_rejects_wrong_size():
    blob = make_weights(3, 8, 24)
    with pytest.raises(ValueError):
        O.unpack_params(blob[:-1], 3, 8, 24)


# ---------------------------------------------------------------------------
# Pin-3: constraint projectors (R4)
# ---------------------------------------------------------------------------

def test_constraint_moments_any_R():
    rng = np.random.default_rng(3)
    R = rng.standard_normal((5, 4, 24)) * 3
    w = O.constrain(R)
    s = np.arange(6) - 2.5
    np.testing.assert_allclose(w[..., 0, :].sum(-1), 1.0, atol=1e-13)     # interp reproduces constants
    np.testing.assert_allclose(w[..., 1, :].sum(-1), 0.0, atol=1e-13)     # deriv kills constants
    np.testing.assert_allclose((w[..., 1, :] * s).sum(-1), 1.0, atol=1e-13)  # deriv exact on linear data


def test_constraint_is_nearest_admissible_stencil():
    """base + Pi r = orthogonal projection of base + r onto the affine constraint set (KKT solve)."""
    rng = np.random.default_rng(4)
    r = rng.standard_normal(24)
    w = O.constrain(r[None, :])[0]
    base = O.default_base_stencils()
    s = np.arange(6) - 2.5
    for ax in range(2):
        for op, (A, c) in enumerate([(np.ones((1, 6)), np.array([1.0])),
                                     (np.stack([np.ones(6), s]), np.array([0.0, 1.0]))]):
            target = base[ax, op] + r[ax * 12 + op * 6: ax * 12 + op * 6 + 6]
            m = A.shape[0]
            K = np.block([[np.eye(6), A.T], [A, np.zeros((m, m))]])
            sol = np.linalg.solve(K, np.concatenate([target, c]))
            np.testing.assert_allclose(w[ax, op], sol[:6], atol=1e-12)


def test_deriv_exact_on_linear_nonperiodic_harness():
    """Pin-3: a constrained derivative stencil differentiates linear data exactly for any R."""
    rng = np.random.default_rng(5)
    w = O.constrain(rng.standard_normal((1, 24)))[0]
    h = 0.37
    i = 10
    data = 2.0 + 3.0 * (np.arange(20) + 0.5) * h          # c(x) = 2 + 3x at centres
    for ax in range(2):
        d = sum(w[ax, 1, t] * data[i - 3 + t] for t in range(6)) / h
        c = sum(w[ax, 0, t] * 2.0 for t in range(6))
        assert abs(d - 3.0) < 1e-12 and abs(c - 2.0) < 1e-12


# ---------------------------------------------------------------------------
# Faces: Fourier symbol of a 6-tap face stencil (shift direction, anchoring R2)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("axis", [-1, -2])
def test_face_stencil_fourier_symbol(axis):
    n = 16
    X, Y, h = _centres(n)
    k = 3
    coord = X if axis == -1 else Y
    c = np.exp(1j * k * coord)
    rng = np.random.default_rng(6)
    w = rng.standard_normal(6)
    got = O.face_values(c[None], np.broadcast_to(w, (1, n, n, 6)), axis)[0]
    sym = sum(w[t] * np.exp(1j * k * h * (t - 3)) for t in range(6))
    np.testing.assert_allclose(got, sym * c, atol=1e-12)
    # 2nd-order interp at face i-1/2 of cos(k x) is cos(k (x - h/2)) cos(k h / 2)
    wi = O.default_base_stencils()[0, 0]
    got = O.face_values(np.cos(k * coord)[None], np.broadcast_to(wi, (1, n, n, 6)), axis)[0]
    np.testing.assert_allclose(got, np.cos(k * (coord - h / 2)) * math.cos(k * h / 2), atol=1e-13)


# ---------------------------------------------------------------------------
# Pin-1: fixed 2nd-order stencils == classical 2nd-order FV scheme, brute-force loops
# ---------------------------------------------------------------------------

def _classical_fv_rhs(U, nu, h, gamma, amp=0.0, kf=0.0, alpha=0.0):
    B, _, n, _ = U.shape
    T = np.zeros_like(U)
    for b in range(B):
        for j in range(n):
            for i in range(n):
                def comp(c, jj, ii):
                    return U[b, c, jj % n, ii % n]
                for c in range(2):
                    def Fx(ii):  # flux through x-face ii-1/2
                        uf = 0.5 * (comp(0, j, ii - 1) + comp(0, j, ii))
                        cf = 0.5 * (comp(c, j, ii - 1) + comp(c, j, ii))
                        return gamma * uf * cf - nu * (comp(c, j, ii) - comp(c, j, ii - 1)) / h

                    def Fy(jj):
                        vf = 0.5 * (comp(1, jj - 1, i) + comp(1, jj, i))
                        cf = 0.5 * (comp(c, jj - 1, i) + comp(c, jj, i))
                        return gamma * vf * cf - nu * (comp(c, jj, i) - comp(c, jj - 1, i)) / h
                    T[b, c, j, i] = -(Fx(i + 1) - Fx(i) + Fy(j + 1) - Fy(j)) / h
                y = (j + 0.5) * h
                T[b, 0, j, i] += amp * math.sin(kf * y) - alpha * U[b, 0, j, i]
                T[b, 1, j, i] += -alpha * U[b, 1, j, i]
    return T


@pytest.mark.parametrize("system", [0, 1])
def test_fixed_mode_equals_classical_fv(system):
    n = 8
    cfg = _cfg(n=n, system=system, nu=0.03, force_amp=0.7, force_k=2.0, drag=0.2)
    u = make_ic("noise", n, 2, seed=9)
    o = O.Oracle(cfg)
    T, _ = o.T(u)
    ref = _classical_fv_rhs(u, 0.03, o.h, 0.5 if system == 0 else 1.0, 0.7, 2.0, 0.2)
    np.testing.assert_allclose(T, ref, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------------------
# Pin-2: constant field -> zero tendency for any (random, constrained) stencils
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("system", [0, 1])
def test_constant_field_zero_tendency_learned(system):
    n = 12
    cfg = _cfg(n=n, system=system, stencil_mode=0, nu=0.05)
    params = make_weights(3, 8, 24, seed=1, init="stress")
    u = np.ones((1, 2, n, n)) * np.array([0.3, -1.7])[None, :, None, None]
    o = O.Oracle(cfg, params)
    T, _ = o.T(u)
    assert np.abs(T).max() < 1e-12


# ---------------------------------------------------------------------------
# Pin-4 / Pin-5: projection
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n", [8, 64, 256])
def test_projection_divergence_free_idempotent(n):
    h = TWO_PI / n
    u = make_ic("noise", n, 2, seed=n)
    pu = O.project(u, h)
    assert np.abs(O.div_c(pu, h)).max() < 1e-10
    np.testing.assert_allclose(O.project(pu, h), pu, atol=1e-12)
    np.testing.assert_allclose(pu.mean(axis=(-1, -2)), u.mean(axis=(-1, -2)), atol=1e-14)
    assert np.linalg.norm(pu) <= np.linalg.norm(u) * (1 + 1e-14)
    # a pure discrete gradient is removed entirely
    phi = np.random.default_rng(0).standard_normal((1, n, n))
    g = np.stack([(np.roll(phi, -1, -1) - np.roll(phi, 1, -1)) / (2 * h),
                  (np.roll(phi, -1, -2) - np.roll(phi, 1, -2)) / (2 * h)], axis=1)
    assert np.abs(O.project(g, h)).max() < 1e-10


def test_poisson_matches_dense_bordered_solve_8x8():
    """Pin-5: FFT Poisson == Gaussian elimination on [A Z; Z^T 0], A = D_c G_c built by loops."""
    n = 8
    h = TWO_PI / n
    idx = lambda j, i: (j % n) * n + (i % n)
    G = np.zeros((2 * n * n, n * n))     # p -> (px, py), centred
    D = np.zeros((n * n, 2 * n * n))     # (u, v) -> d, centred
    for j in range(n):
        for i in range(n):
            r = idx(j, i)
            G[r, idx(j, i + 1)] += 1 / (2 * h)
            G[r, idx(j, i - 1)] -= 1 / (2 * h)
            G[n * n + r, idx(j + 1, i)] += 1 / (2 * h)
            G[n * n + r, idx(j - 1, i)] -= 1 / (2 * h)
            D[r, idx(j, i + 1)] += 1 / (2 * h)
            D[r, idx(j, i - 1)] -= 1 / (2 * h)
            D[r, n * n + idx(j + 1, i)] += 1 / (2 * h)
            D[r, n * n + idx(j - 1, i)] -= 1 / (2 * h)
    A = D @ G
    Z = np.zeros((n * n, 4))
    for j in range(n):
        for i in range(n):
            Z[idx(j, i)] = [1, (-1) ** i, (-1) ** j, (-1) ** (i + j)]
    assert np.linalg.matrix_rank(A) == n * n - 4
    u = make_ic("noise", n, 1, seed=3)
    d = D @ u.reshape(-1)
    K = np.block([[A, Z], [Z.T, np.zeros((4, 4))]])
    sol = np.linalg.solve(K, np.concatenate([d, np.zeros(4)]))
    p_dense = sol[:n * n].reshape(n, n)
    p_fft = O.solve_pressure(d.reshape(1, n, n), h)[0]
    np.testing.assert_allclose(p_fft, p_dense, atol=1e-12)
    # and the projection equals u - G p_dense
    proj = (u.reshape(-1) - G @ p_dense.reshape(-1)).reshape(1, 2, n, n)
    np.testing.assert_allclose(O.project(u, h), proj, atol=1e-12)


def test_symbol_nyquist_and_dc_are_zero():
    s = O.symbol(16, TWO_PI / 16)
    assert s[0] == 0.0 and s[8] == 0.0
    np.testing.assert_allclose(s[1], math.sin(TWO_PI / 16) / (TWO_PI / 16))


# ---------------------------------------------------------------------------
# Pin-7 / Pin-7': linear part, RK stability polynomials (R13)
# ---------------------------------------------------------------------------

def _Rp(z, p):
    if p == 2:
        return 1 + z + z * z / 2
    if p == 3:
        return 1 + z + z * z / 2 + z ** 3 / 6
    return 1 + z + z * z / 2 + z ** 3 / 6 + z ** 4 / 24


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("system", [0, 1])
def test_shear_mode_decay_factor(p, system):
    n, k, nu, dt = 32, 3, 0.05, 0.02
    X, Y, h = _centres(n)
    u0 = np.stack([np.sin(k * Y), np.zeros_like(Y)])[None]
    cfg = _cfg(n=n, system=system, rk_order=p, nu=nu, dt=dt)
    u1 = O.step(u0, cfg)
    kh = 2 * math.sin(k * h / 2) / h
    np.testing.assert_allclose(u1, _Rp(-nu * kh * kh * dt, p) * u0, atol=1e-14)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_constant_learned_deriv_stencil_symbol(p):
    """Pin-7': bias-only last layer => constant asymmetric stencils; closed-form growth factor."""
    n, k, nu, dt = 16, 2, 0.04, 0.01
    X, Y, h = _centres(n)
    rng = np.random.default_rng(11)
    params = make_weights(3, 8, 24, seed=2, init="stress")
    layers_sz = [(8 * 9 * 2 + 8), (8 * 9 * 8 + 8)]
    off = sum(layers_sz)
    params[off:off + 24 * 9 * 8] = 0.0                 # W_L = 0 -> R = b_L everywhere
    r = (rng.standard_normal(24) * 0.3).astype(np.float32)
    params[off + 24 * 9 * 8:] = r
    # expected constrained y-deriv stencil: KKT projection of base + r (independent of O.constrain)
    s = np.arange(6) - 2.5
    A = np.stack([np.ones(6), s])
    target = np.array([0, 0, -1, 1, 0, 0.0]) + r[18:24].astype(np.float64)
    K = np.block([[np.eye(6), A.T], [A, np.zeros((2, 2))]])
    wD = np.linalg.solve(K, np.concatenate([target, [0.0, 1.0]]))[:6]
    S = sum(wD[t] * np.exp(1j * k * h * (t - 3)) for t in range(6))
    lam = (nu / h ** 2) * (np.exp(1j * k * h) - 1) * S
    for system in (0, 1):
        cfg = _cfg(n=n, system=system, rk_order=p, nu=nu, dt=dt, stencil_mode=0, n_layers=3, width=8)
        u0 = np.stack([np.cos(k * Y), np.zeros_like(Y)])[None]
        u1 = O.step(u0, cfg, params)
        ref = np.real(_Rp(lam * dt, p) * np.exp(1j * k * Y))
        np.testing.assert_allclose(u1[0, 0], ref, atol=1e-13)
        np.testing.assert_allclose(u1[0, 1], 0.0, atol=1e-13)


# ---------------------------------------------------------------------------
# Pin-8: Taylor-Green
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("p", [2, 3, 4])
def test_taylor_green_one_step_exact(p):
    n, nu, dt = 32, 0.01, 0.05
    h = TWO_PI / n
    u0 = make_ic("taylor_green", n, 1)
    u1 = O.step(u0, _cfg(n=n, rk_order=p, nu=nu, dt=dt))
    k1 = 2 * math.sin(h / 2) / h
    np.testing.assert_allclose(u1, _Rp(-2 * nu * k1 * k1 * dt, p) * u0, atol=1e-14)


def test_taylor_green_converges_to_continuum_second_order():
    """Against exp(-2 nu t) (BASELINE.json north_star's TG check), observed order ~2."""
    nu, T = 0.01, 1.0
    errs = []
    for n in (16, 32, 64):
        h = TWO_PI / n
        steps = int(round(T / (0.5 * h)))
        dt = T / steps
        cfg = _cfg(n=n, nu=nu, dt=dt)
        u0 = make_ic("taylor_green", n, 1)
        u = O.rollout(u0, cfg, None, steps)
        ref = u0 * math.exp(-2 * nu * T)
        errs.append(np.linalg.norm(u - ref) / np.linalg.norm(ref))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert errs[-1] < 1e-4
    for q in orders:
        assert 1.8 < q < 2.2, (errs, orders)


# ---------------------------------------------------------------------------
# Pin-9: Kolmogorov laminar state is an exact discrete fixed point
# ---------------------------------------------------------------------------

def test_kolmogorov_fixed_point():
    n, nu, chi, kf, alpha = 64, 1e-3, 1.0, 4, 0.1
    X, Y, h = _centres(n)
    kh = 2 * math.sin(kf * h / 2) / h
    A = chi / (nu * kh * kh + alpha)
    u0 = np.stack([A * np.sin(kf * Y), np.zeros_like(Y)])[None]
    cfg = _cfg(n=n, nu=nu, force_amp=chi, force_k=kf, drag=alpha, dt=0.5 * h / A)
    u = O.rollout(u0, cfg, None, 5)
    np.testing.assert_allclose(u, u0, atol=1e-13 * A)


# ---------------------------------------------------------------------------
# Pin-10: conservation of mean momentum (no forcing, drag or TC), any weights
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("system", [0, 1])
def test_mean_momentum_conserved_learned(system):
    n = 16
    cfg = _cfg(n=n, system=system, stencil_mode=0, nu=0.01, dt=0.02, rk_order=3)
    params = make_weights(3, 8, 24, seed=5, init="stress")
    params[-24 * 9 * 8 - 24:] *= 0.05
    u0 = make_ic("fourier", n, 2, seed=1) + np.array([0.2, -0.1])[None, :, None, None]
    m0 = u0.sum(axis=(-1, -2))
    u = O.rollout(u0, cfg, params, 10)
    np.testing.assert_allclose(u.sum(axis=(-1, -2)), m0, atol=1e-11)


# ---------------------------------------------------------------------------
# Pin-11: skew-symmetry of advection on divergence-free fields, KE decay
# ---------------------------------------------------------------------------

def test_advection_energy_neutral_and_ke_decay():
    n = 32
    h = TWO_PI / n
    u = O.project(make_ic("spectrum", n, 1, seed=4), h)
    cfg = _cfg(n=n, nu=0.0)
    o = O.Oracle(cfg)
    T, _ = o.T(u)
    PT = O.project(T, h)
    assert abs(np.sum(u * PT)) / np.sum(u * u) < 1e-13
    cfg = _cfg(n=n, nu=1e-3, dt=0.5 * h)
    o = O.Oracle(cfg)
    ke = [np.sum(u * u)]
    for _ in range(30):
        u = o.step(u)
        ke.append(np.sum(u * u))
    assert all(ke[i + 1] <= ke[i] * (1 + 1e-14) for i in range(30))


# ---------------------------------------------------------------------------
# Pin-13: translation equivariance, any weights
# ---------------------------------------------------------------------------

def test_translation_equivariance():
    n = 16
    cfg = _cfg(n=n, system=1, stencil_mode=0, nu=0.01, dt=0.02, force_amp=0.5, force_k=2, drag=0.1,
               tc_head=1)
    params = make_weights(3, 8, 26, seed=3, init="stress")
    u0 = make_ic("noise", n, 1, seed=2)
    sx, sy = 5, n // 2   # sy must be a multiple of N / k_f with forcing
    a = O.step(u0, cfg, params)
    b = O.step(np.roll(u0, (sy, sx), axis=(-2, -1)), cfg, params)
    np.testing.assert_allclose(np.roll(a, (sy, sx), axis=(-2, -1)), b, atol=1e-12)


# ---------------------------------------------------------------------------
# Temporal-correction head gating (Eq.2, R8)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("system", [0, 1])
def test_tc_head_adds_e_every_kc_steps(system):
    n = 8
    params = make_weights(3, 8, 26, seed=4, init="stress")
    off = (8 * 9 * 2 + 8) + (8 * 9 * 8 + 8)
    params[off:off + 26 * 9 * 8] = 0.0
    params[off + 26 * 9 * 8 + 24] = 0.25
    params[off + 26 * 9 * 8 + 25] = -0.5
    cfg = _cfg(n=n, system=system, stencil_mode=0, tc_head=1, tc_interval=2, nu=0.01, dt=0.1)
    o = O.Oracle(cfg, params)
    u = np.zeros((1, 2, n, n))
    u1 = o.step(u)                  # k = 0: (0+1) % 2 != 0 -> no correction
    assert np.abs(u1).max() == 0.0
    u2 = o.step(u1)                 # k = 1: correction e = b_L[24:26] (constant field)
    np.testing.assert_allclose(u2[0, 0], 0.25, atol=1e-15)
    np.testing.assert_allclose(u2[0, 1], -0.5, atol=1e-15)


def test_rollout_zero_and_one_step():
    cfg = get_config("c1", n=16)
    u0 = make_ic("fourier", 16, 1, seed=0)
    cfg = cfg.with_dt(u0)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0)
    o = O.Oracle(cfg, params)
    np.testing.assert_array_equal(o.rollout(u0, 0)["u"], u0)
    np.testing.assert_array_equal(O.rollout(u0, cfg, params, 1), O.step(u0, cfg, params))


def test_nonfinite_reported_with_step_index():
    cfg = _cfg(n=8, system=0, nu=0.0, dt=1e3, rk_order=2)
    u0 = make_ic("noise", 8, 1, seed=0) * 10
    with pytest.raises(FloatingPointError, match="step"):
        O.rollout(u0, cfg, None, 200)


# ---------------------------------------------------------------- NEXT-1: fine -> coarse downsampling

def test_downsample_pins():
    """Block mean (Table S1; reading: finite-volume cell averages) pinned to a
    brute-force loop, to exactness on constant and linear fields, and to conservation of the
    domain mean."""
    rng = np.random.default_rng(3)
    u = rng.standard_normal((2, 2, 8, 8))
    f = 4
    got = O.downsample(u, f)
    brute = np.zeros((2, 2, 2, 2))
    for b in range(2):
        for c in range(2):
            for J in range(2):
                for I in range(2):
                    s = 0.0
                    for dj in range(f):
                        for di in range(f):
                            s += u[b, c, J * f + dj, I * f + di]
                    brute[b, c, J, I] = s / (f * f)
    assert np.allclose(got, brute, rtol=0, atol=1e-14)
    assert np.allclose(O.downsample(np.full((1, 2, 16, 16), 2.5), 8), 2.5)
    # a linear field's block mean is its value at the block centre (cell-average exactness)
    n, f = 32, 4
    h = 2 * np.pi / n
    x = (np.arange(n) + 0.5) * h
    lin = np.broadcast_to(3.0 * x[None, :] - 1.5 * x[:, None], (1, 2, n, n))
    xc = (np.arange(n // f) + 0.5) * h * f
    assert np.allclose(O.downsample(lin, f)[0, 0], 3.0 * xc[None, :] - 1.5 * xc[:, None], atol=1e-12)
    assert abs(O.downsample(u, 2).mean() - u.mean()) < 1e-15


def test_frozen_stencils_variant():
    """Per-step frozen stencils: identical to the per-stage net (R7) when the net's
    output does not depend on the field (zero last layer: w = w_base), different otherwise; the
    frozen step also keeps the invariants (mean momentum, a constant field is a fixed point)."""
    from ldgen import make_weights
    from ldgen.configs import get_config
    cfg = get_config("c2", n=16, batch=2).replace(dt=0.01)
    fz = cfg.replace(freeze_stencils=1)
    u = np.random.default_rng(6).standard_normal((2, 2, 16, 16))
    p0 = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="zero_last")
    assert np.array_equal(O.step(u, fz, p0), O.step(u, cfg, p0))
    p = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="stress")
    out = O.step(u, fz, p)
    assert not np.allclose(out, O.step(u, cfg, p))
    assert np.allclose(out.sum(axis=(-2, -1)), u.sum(axis=(-2, -1)), atol=1e-10)
    c = np.ones((1, 2, 16, 16)) * np.array([0.3, -0.7])[None, :, None, None]
    assert np.allclose(O.step(c, fz, p), c, atol=1e-13)


# ---------------------------------------------------------------------------
# R8: the TC term e comes from the STAGE-1 net evaluation on u^n (Eq.2: the correction
# acts on the step's input fields), not from a later stage's net
# ---------------------------------------------------------------------------

def _passthrough_tc_params(width=4, scale=0.125):
    """3-layer ReLU net whose stencil outputs are zero (w = w_base) and whose TC outputs are
    e = scale * (u, v) of the net's INPUT field: layer 1 splits u, v into ReLU(+-u), ReLU(+-v)
    (centre tap), layer 2 passes them through (non-negative, so ReLU is the identity), and the
    output layer recombines e_u = scale (ReLU(u) - ReLU(-u)) = scale u, same for v."""
    L1 = np.zeros((width, 3, 3, 2)); b1 = np.zeros(width)
    L1[0, 1, 1, 0], L1[1, 1, 1, 0], L1[2, 1, 1, 1], L1[3, 1, 1, 1] = 1.0, -1.0, 1.0, -1.0
    L2 = np.zeros((width, 3, 3, width)); b2 = np.zeros(width)
    for c in range(4):
        L2[c, 1, 1, c] = 1.0
    L3 = np.zeros((26, 3, 3, width)); b3 = np.zeros(26)
    L3[24, 1, 1, 0], L3[24, 1, 1, 1] = scale, -scale
    L3[25, 1, 1, 2], L3[25, 1, 1, 3] = scale, -scale
    return np.concatenate([a.ravel() for a in (L1, b1, L2, b2, L3, b3)]).astype(np.float32)


@pytest.mark.parametrize("rk", [2, 3, 4])
@pytest.mark.parametrize("system", [0, 1])
def test_tc_term_from_stage1_net(rk, system):
    """With w = w_base the learned step equals the classical FV step plus e, and e = u^n / 8:
    Burgers (no projection, R9) adds exactly u^n / 8; NS adds P(u^n / 8) = P(u^n) / 8 (P linear,
    pinned by Pin-4/5).  Taking e from a later stage field would add U_s / 8, which differs from
    u^n / 8 by dt T / 8 = O(1e-2) here."""
    n = 8
    u = make_ic("noise", n, 1, seed=11)
    kw = dict(n=n, system=system, nu=0.05, dt=0.1, rk_order=rk, n_layers=3, width=4, activation=0)
    learned = O.step(u, _cfg(stencil_mode=0, tc_head=1, tc_interval=1, **kw), _passthrough_tc_params())
    plain = O.step(u, _cfg(stencil_mode=1, tc_head=0, **kw))
    want = 0.125 * (u if system == 0 else O.project(u, TWO_PI / n))   # 1/8: exact in the fp32 blob
    np.testing.assert_allclose(learned - plain, want, rtol=0, atol=1e-12)
    # and the alternative reading really is distinguishable at this dt
    o = O.Oracle(_cfg(stencil_mode=1, **kw))
    U1 = o.P(u + 0.1 * o.T(u)[0])
    assert np.abs(0.1 * (U1 - u)).max() > 1e-3


# ---------------------------------------------------------------------------
# R9: Burgers (S = 0) has NO projection: a compressible 1-D Burgers field u = (f(x), 0) stays
# compressible and follows the 1-D viscous Burgers FV scheme F = u^2/2 - nu du/dx step for step
# ---------------------------------------------------------------------------

def _burgers_1d_rhs(f, nu, h):
    """Classical 2nd-order FV tendency of 1-D viscous Burgers, written out by loops:
    face i-1/2 value (f[i-1] + f[i]) / 2, gradient (f[i] - f[i-1]) / h."""
    n = len(f)
    F = np.empty(n)
    for i in range(n):
        fm = f[(i - 1) % n]
        uf = 0.5 * (fm + f[i])
        F[i] = 0.5 * uf * uf - nu * (f[i] - fm) / h
    return np.array([-(F[(i + 1) % n] - F[i]) / h for i in range(n)])


@pytest.mark.parametrize("rk", [2, 3, 4])
def test_burgers_step_is_unprojected_1d_burgers(rk):
    n, nu, dt = 16, 0.02, 0.05
    h = TWO_PI / n
    x = (np.arange(n) + 0.5) * h
    f = np.sin(x) + 0.3 * np.cos(3 * x) + 0.2       # compressible: D_c u = f'(x) != 0
    u = np.zeros((1, 2, n, n))
    u[0, 0] = f[None, :]
    out = O.step(u, _cfg(n=n, system=0, nu=nu, dt=dt, rk_order=rk))
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
    np.testing.assert_allclose(out[0, 0], np.broadcast_to(ref, (n, n)), rtol=0, atol=1e-13)
    assert np.abs(out[0, 1]).max() == 0.0
    assert np.abs(O.div_c(out, h)).max() > 0.1     # a projection would have removed it
