"""GPU parity of the paper's constant 5x4 face kernels (stencil_mode 2; readings F1-F3,
DESIGN.md §8i) against the fp64 oracle (tests/test_5x4_oracle.py pins it).  fp32 throughout: 1e-5 one
step, 1e-4 after 20 steps."""
import numpy as np
import pytest

import oracle as O
from ldgen import make_ic
from ldgen.configs import get_config
from tests.helpers import gpu_solver, rel_l2, to_dev

pytestmark = pytest.mark.gpu


def _params(seed=1, scale=0.05):
    return (np.random.default_rng(seed).standard_normal(80) * scale).astype(np.float32)


@pytest.mark.parametrize("name,n,B,rk", [("c2", 64, 2, 3), ("c3", 128, 1, 3), ("c1", 32, 2, 2), ("c2", 32, 2, 4),
                                         ("c2", 256, 1, 3)])
def test_5x4_one_step_and_tendency(name, n, B, rk):
    import torch
    cfg = get_config(name, n=n, batch=B, rk_order=rk, stencil_mode=2, tc_head=0)
    u0 = make_ic(cfg.ic, n, B, seed=2)
    cfg = cfg.with_dt(u0)
    p = _params()
    s = gpu_solver(cfg, p)
    u = to_dev(u0)
    s.ld_step(u)
    assert rel_l2(u.cpu().numpy(), O.step(u0, cfg, p)) < 1e-5
    T = torch.empty_like(u)
    s.ld_eval_tendency(to_dev(u0), T)
    Tref, _ = O.Oracle(cfg, p).T(u0)
    assert rel_l2(T.cpu().numpy(), Tref) < 1e-5


def test_5x4_rollout():
    cfg = get_config("c3", n=64, batch=2, stencil_mode=2, tc_head=0)
    u0 = make_ic("spectrum", 64, 2, seed=3)
    cfg = cfg.with_dt(u0)
    p = _params(2)
    s = gpu_solver(cfg, p)
    u = to_dev(u0)
    s.ld_rollout(u, 20)
    assert rel_l2(u.cpu().numpy(), O.rollout(u0, cfg, p, 20)) < 1e-4
