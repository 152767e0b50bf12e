"""Seeded parameters for the frequency-domain operator O_F (Eq. 8, P:252-256;
SURVEY.md §8f NEXT-2).  Inputs only -- none of the operator's arithmetic lives here.

Retained modes: |kx| <= K and |ky| <= K (K < N/2).  Parameters are stored on the
half plane H (the other half follows by conjugate symmetry, so the operator's output
is real), enumerated in this order -- both sides enumerate it themselves:

    for kx in 0..K:  for ky in -K..K:  skip (kx == 0 and ky < 0)

    n_modes(K) = (K + 1) (2K + 1) - K

Layer l (1..L): R_l[mode][c_out][c_in][re, im] with c_in = 2 (u, v) for l = 1 and C
afterwards, c_out = C.  The imaginary part at k = (0, 0) is zero (a real map there).
Q[8][C] real.  Values: float64 from PCG64 rounded once to float32.
"""
from __future__ import annotations

import numpy as np

N_OUT = 8   # (interp, deriv) x (x-face, y-face) x (u, v)


def n_modes(K: int) -> int:
    return (K + 1) * (2 * K + 1) - K


def half_plane_modes(K: int):
    """The (kx, ky) list in storage order."""
    return [(kx, ky) for kx in range(K + 1) for ky in range(-K, K + 1) if not (kx == 0 and ky < 0)]


def make_spectral_params(K: int, C: int, L: int, seed: int = 0, scale: float = 1.0, n_in: int = 2, n_out: int = N_OUT):
    """Returns (R list of float32 arrays [n_modes][C][c_in][2], Q float32 [n_out][C])."""
    rng = np.random.default_rng(104729 + int(seed))
    R = []
    for l in range(L):
        cin = n_in if l == 0 else C
        a = rng.standard_normal((n_modes(K), C, cin, 2)) * (scale / np.sqrt(cin))
        a[half_plane_modes(K).index((0, 0)), :, :, 1] = 0.0
        R.append(a.astype(np.float32))
    Q = (rng.standard_normal((n_out, C)) / np.sqrt(C)).astype(np.float32)
    return R, Q


def spectral_blob(K: int, C: int, L: int, seed: int = 0, scale: float = 1.0, n_in: int = 2,
                  n_out: int = N_OUT) -> np.ndarray:
    """The flat float32 blob (R_1, ..., R_L, Q) that follows the conv parameters when
    ld_config.fno_layers > 0 (n_in 2, n_out 8) or tc_mode = 1 (n_in 2 k_c, n_out 2)."""
    R, Q = make_spectral_params(K, C, L, seed=seed, scale=scale, n_in=n_in, n_out=n_out)
    return np.concatenate([r.ravel() for r in R] + [Q.ravel()]).astype(np.float32)
