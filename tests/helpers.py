"""Shared test helpers: build a GPU solver and the oracle from one LDConfig."""
import numpy as np

from ldgen import make_weights
from ldgen.ic import make_config_ic


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def setup(cfg, init="normal", seed=0, elements=None):
    u0 = make_config_ic(cfg, elements=elements)
    if cfg.dt is None:
        cfg = cfg.with_dt(u0)
    params = None
    if cfg.stencil_mode == 0:
        params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=seed, init=init)
    return cfg, u0, params


def gpu_solver(cfg, params, base=None, **over):
    from paper_2507_01975_b200 import ldsolver as L
    c = L.make_config(cfg, **over)
    return L.Solver(c, params, base)


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
