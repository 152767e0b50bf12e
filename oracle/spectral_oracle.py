"""CPU ORACLE for the frequency-domain operator O_F -- TEST INFRASTRUCTURE ONLY.

PAPER.md Eq. 8:  O_F(u) = Q( F^{-1}( R_L . F(u) ) ),  "F and F^{-1} ... the forward
and inverse Fourier transforms", "R_L ... the frequency-space correction layers", "Q ... a
learnable projection mapping spectral features back to physical space"; "decomposes the
flow field into spectral components via F, applies L-layer frequency-space corrections, and
then reconstructs the enhanced features through F^{-1}".  Readings (DESIGN.md §8c,
N2-1..N2-4): F = unnormalised 2-D DFT of each input channel (u, v); only the modes
|kx|, |ky| <= K are kept (SPEC.md "retain lowest k_max modes"); the L layers are per-mode
complex linear maps applied one after another in frequency space (the paper names no
nonlinearity between them); parameters live on the half plane and extend by
R(-k) = conj(R(k)), so F^{-1} (with the 1/N^2 factor) returns a real field; Q is a pointwise
real map C -> 8 applied after F^{-1}.  Written with numpy's FFT, step by step in the paper's
order, in float64.  Shares no code with the CUDA path (fft.cu / spectral.cu).
"""
from __future__ import annotations

import numpy as np


def _modes(K: int):
    return [(kx, ky) for kx in range(K + 1) for ky in range(-K, K + 1) if not (kx == 0 and ky < 0)]


def full_plane(R_half: np.ndarray, K: int, N: int) -> np.ndarray:
    """Half-plane parameters [n_modes][co][ci][2] -> complex [co][ci][N(ky)][N(kx)] on the
    whole DFT grid: retained modes and their conjugate partners, zero elsewhere."""
    co, ci = R_half.shape[1], R_half.shape[2]
    out = np.zeros((co, ci, N, N), dtype=np.complex128)
    Rc = R_half[..., 0].astype(np.float64) + 1j * R_half[..., 1].astype(np.float64)
    for m, (kx, ky) in enumerate(_modes(K)):
        out[:, :, ky % N, kx % N] = Rc[m]
        out[:, :, (-ky) % N, (-kx) % N] = np.conj(Rc[m])
    return out


def spectral_operator(u: np.ndarray, R, Q: np.ndarray, K: int) -> np.ndarray:
    """u [B][c_in][N][N] (y rows, x columns) -> Q(F^-1(R_L..R_1 F(u))) [B][rows of Q][N][N]
    (O_F: c_in = 2, 8 outputs; the history TC block: c_in = 2 k_c, 2 outputs)."""
    u = np.asarray(u, dtype=np.float64)
    B, _, N, _ = u.shape
    if not (0 <= K < N // 2):
        raise ValueError("K must satisfy 0 <= K < N/2")
    uh = np.fft.fft2(u, axes=(-2, -1))                     # F: unnormalised DFT over (y, x)
    h = uh
    for Rl in R:                                           # R_L . : per-mode linear layers
        Rf = full_plane(np.asarray(Rl), K, N)              # zero outside the retained set
        h = np.einsum("oiyx,biyx->boyx", Rf, h)
    hx = np.fft.ifft2(h, axes=(-2, -1))                    # F^{-1} (includes 1/N^2)
    assert np.max(np.abs(hx.imag)) <= 1e-9 * max(1.0, np.max(np.abs(hx.real))), "conjugate symmetry"
    return np.einsum("oc,bcyx->boyx", np.asarray(Q, dtype=np.float64), hx.real)   # Q pointwise


def unpack_spectral(blob, K: int, L: int, C: int, n_in: int = 2, n_out: int = 8):
    """Flat (R_1 .. R_L, Q) blob -> (R list, Q), in the documented layout
    (R_1 [n_modes][C][n_in][2], R_l [n_modes][C][C][2], Q [n_out][C])."""
    nm = len(_modes(K))
    b = np.asarray(blob, dtype=np.float64)
    R, off = [], 0
    for l in range(L):
        cin = n_in if l == 0 else C
        n = nm * C * cin * 2
        R.append(b[off:off + n].reshape(nm, C, cin, 2))
        off += n
    Q = b[off:off + n_out * C].reshape(n_out, C)
    off += n_out * C
    if off != b.size:
        raise ValueError(f"spectral blob has {b.size} floats, expected {off}")
    return R, Q


def half_cell_shift(f: np.ndarray, axis: int) -> np.ndarray:
    """f evaluated half a cell towards -axis (f(x - h/2)), exactly, for a band-limited periodic
    field with no Nyquist content: multiply mode m by e^{-i pi m / N} (reading N2-6)."""
    n = f.shape[axis]
    m = np.fft.fftfreq(n, d=1.0 / n)
    shape = [1] * f.ndim
    shape[axis] = n
    ph = np.exp(-1j * np.pi * m / n).reshape(shape)
    out = np.fft.ifft(np.fft.fft(f, axis=axis) * ph, axis=axis)
    assert np.max(np.abs(out.imag)) <= 1e-9 * max(1.0, np.max(np.abs(out.real)))
    return out.real


def spectral_faces(u, R, Q, K: int) -> np.ndarray:
    """O_F(u) placed on the faces the flux uses (reading N2-6): channels 0-3 (x-face i-1/2) at
    x - h/2, channels 4-7 (y-face j-1/2) at y - h/2.  [B][8][N][N]."""
    o = spectral_operator(u, R, Q, K)
    out = np.empty_like(o)
    out[:, :4] = half_cell_shift(o[:, :4], -1)
    out[:, 4:] = half_cell_shift(o[:, 4:], -2)
    return out
