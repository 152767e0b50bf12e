"""Seeded random-init weight blob for the 3x3 conv stencil network.

Blob layout (the C-ABI's ``params_host``, include/ldsolver.h): for each layer
l = 1..L in order, ``W_l[co][ky][kx][ci]`` then ``b_l[co]``, fp32.
Channel widths: 2 -> width -> ... -> width -> n_out (n_out = 24, or 26 with the
temporal-correction head).

Init ("initialized with minor random values"):
hidden layers U(+-1/sqrt(fan_in)) for weights and biases, fan_in = 9*C_in; the
last layer U(+-last_scale) with last_scale = 1e-3 by default ("normal"), or
1/sqrt(fan_in) ("stress", used for one-step parity so the learned path
dominates).  Values are drawn in float64 from numpy's PCG64 and rounded once to
float32; both the oracle and the GPU path consume the float32 blob.
"""
from __future__ import annotations

import math
from typing import List, Tuple

import numpy as np


def layer_shapes(n_layers: int, width: int, n_out: int) -> List[Tuple[int, int]]:
    chans = [2] + [width] * (n_layers - 1) + [n_out]
    return [(chans[i], chans[i + 1]) for i in range(n_layers)]


def param_count(n_layers: int, width: int, n_out: int) -> int:
    return sum(co * 9 * ci + co for ci, co in layer_shapes(n_layers, width, n_out))


def make_weights(n_layers: int, width: int, n_out: int, seed: int = 0,
                 init: str = "normal") -> np.ndarray:
    rng = np.random.default_rng(7919 + int(seed))
    parts = []
    shapes = layer_shapes(n_layers, width, n_out)
    for li, (ci, co) in enumerate(shapes):
        fan_in = 9 * ci
        last = li == len(shapes) - 1
        if not last or init == "stress":
            s = 1.0 / math.sqrt(fan_in)
        elif init == "normal":
            s = 1e-3
        elif init == "zero_last":
            s = 0.0
        else:
            raise ValueError(init)
        W = rng.uniform(-1.0, 1.0, size=(co, 3, 3, ci)) * s
        b = rng.uniform(-1.0, 1.0, size=(co,)) * s
        parts += [W.ravel(), b]
    return np.concatenate(parts).astype(np.float32)


def make_config_weights(cfg, seed: int = 0, init: str = "normal") -> np.ndarray:
    return make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=seed, init=init)
