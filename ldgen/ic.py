"""Seeded initial conditions, layout [B][2][N][N] (c=0: u, c=1: v; [j][i] = [y][x]).

Cell centres are x_i = (i + 1/2) h, y_j = (j + 1/2) h on [0, L)^2 (SURVEY.md §8
grid conventions, R12).  Element b of a batch is drawn from its own generator
seeded with ``element_seed(base, b)``, so a shard of a batch is bitwise equal to
the same rows of the full batch (ensemble sharding).

Kinds (BASELINE.json configs):

* ``fourier``  (c1): Euclidean |k| <= 4, k != 0, half-plane modes, independent
  N(0,1) cos and sin coefficients divided by (1 + |k|^2), u and v independent,
  then one common scale so that max(max|u|, max|v|) = 1 (R15, R16).
* ``spectrum`` (c2, c3, c5): random-phase streamfunction with velocity energy
  spectrum E(k) ∝ k^4 exp(-(k/4)^2) used literally (R14), i.e.
  |psi_hat(k)| ∝ sqrt(E(|k|) / (pi |k|)) / |k|; the velocity is taken as the
  centred difference of psi, u = (psi(j+1) - psi(j-1)) / 2h,
  v = -(psi(i+1) - psi(i-1)) / 2h, which is discretely divergence free under
  the centred divergence by construction (this replaces R18's "then P", so the
  generator never calls the method's projection), then normalised to max 1.
* ``shear``    (c4): u = tanh((y - pi/2)/delta) for y <= pi, tanh((3pi/2 - y)/delta)
  for y > pi, delta = pi/15, v = 0.05 sin x; identical for every element (R17).
* ``taylor_green``: u = cos x sin y, v = -sin x cos y (test input).
* ``zero``: all zeros.
"""
from __future__ import annotations

import math
from typing import Iterable, Optional

import numpy as np


def element_seed(base: int, b: int) -> int:
    return int(base) * 1_000_003 + int(b) + 12345


def centres(n: int, length: float = 2.0 * math.pi):
    h = length / n
    x = (np.arange(n) + 0.5) * h
    return x, h


def _fourier(n, length, rng):
    x, h = centres(n, length)
    X, Y = np.meshgrid(x, x, indexing="xy")  # X[j, i] = x_i, Y[j, i] = y_j
    k0 = 2.0 * math.pi / length
    out = np.zeros((2, n, n))
    for c in range(2):
        for kx in range(0, 5):
            for ky in range(-4, 5):
                if kx == 0 and ky <= 0:
                    continue
                if kx * kx + ky * ky > 16:
                    continue
                amp = 1.0 / (1.0 + kx * kx + ky * ky)
                a, b = rng.standard_normal(2) * amp
                ph = k0 * (kx * X + ky * Y)
                out[c] += a * np.cos(ph) + b * np.sin(ph)
    return out


def _spectrum(n, length, rng, k_peak=4.0):
    _, h = centres(n, length)
    k = np.fft.fftfreq(n, d=1.0 / n) * (2.0 * math.pi / length)
    KX, KY = np.meshgrid(k, k, indexing="xy")
    kk = np.sqrt(KX ** 2 + KY ** 2)
    with np.errstate(divide="ignore", invalid="ignore"):
        E = kk ** 4 * np.exp(-(kk / k_peak) ** 2)
        amp = np.where(kk > 0, np.sqrt(E / (math.pi * kk)) / kk, 0.0)
    phase = rng.uniform(0.0, 2.0 * math.pi, size=(n, n))
    psi = np.real(np.fft.ifft2(amp * np.exp(1j * phase))) * n * n
    u = (np.roll(psi, -1, axis=0) - np.roll(psi, 1, axis=0)) / (2.0 * h)
    v = -(np.roll(psi, -1, axis=1) - np.roll(psi, 1, axis=1)) / (2.0 * h)
    return np.stack([u, v])


def _shear(n, length):
    x, _ = centres(n, length)
    X, Y = np.meshgrid(x, x, indexing="xy")
    delta = math.pi / 15.0
    u = np.where(Y <= math.pi, np.tanh((Y - math.pi / 2) / delta),
                 np.tanh((3 * math.pi / 2 - Y) / delta))
    v = 0.05 * np.sin(X)
    return np.stack([u, v])


def _taylor_green(n, length):
    x, _ = centres(n, length)
    X, Y = np.meshgrid(x, x, indexing="xy")
    return np.stack([np.cos(X) * np.sin(Y), -np.sin(X) * np.cos(Y)])


def _normalise(f):
    m = max(np.abs(f[0]).max(), np.abs(f[1]).max())
    return f / m if m > 0 else f


def make_ic(kind: str, n: int, batch: int, seed: int = 0,
            elements: Optional[Iterable[int]] = None,
            length: float = 2.0 * math.pi, dtype=np.float64) -> np.ndarray:
    """Return a [len(elements)][2][n][n] array (elements default to range(batch))."""
    idx = list(range(batch)) if elements is None else list(elements)
    out = np.empty((len(idx), 2, n, n), dtype=dtype)
    for o, b in enumerate(idx):
        rng = np.random.default_rng(element_seed(seed, b))
        if kind == "fourier":
            f = _normalise(_fourier(n, length, rng))
        elif kind == "spectrum":
            f = _normalise(_spectrum(n, length, rng))
        elif kind == "shear":
            f = _shear(n, length)
        elif kind == "taylor_green":
            f = _taylor_green(n, length)
        elif kind == "zero":
            f = np.zeros((2, n, n))
        elif kind == "noise":
            f = rng.standard_normal((2, n, n))
        else:
            raise ValueError(f"unknown IC kind {kind!r}")
        out[o] = f
    return out


def make_scalar_ic(n: int, batch: int, length: float = 2.0 * math.pi, dtype=np.float64) -> np.ndarray:
    """Passive scalar of the shear-flow case ("mixture transport"; SPEC.md: "a passive
    scalar initialized as the layer indicator"): s = 1/2 (tanh((y - pi/2)/delta) - tanh((y - 3pi/2)/delta)),
    delta = pi/15 -- the smoothed indicator of the band between c4's two shear layers, [B][n][n]."""
    x, _ = centres(n, length)
    Y = np.broadcast_to(x[:, None], (n, n))
    delta = math.pi / 15.0
    s = 0.5 * (np.tanh((Y - math.pi / 2) / delta) - np.tanh((Y - 3 * math.pi / 2) / delta))
    return np.broadcast_to(s, (batch, n, n)).astype(dtype).copy()


def make_config_ic(cfg, elements=None, dtype=np.float64) -> np.ndarray:
    return make_ic(cfg.ic, cfg.n, cfg.batch, seed=cfg.seed, elements=elements,
                   length=cfg.length, dtype=dtype)
