"""GPU parity of the per-step frozen-stencil variant (ld_config.freeze_stencils = 1; SURVEY.md §8f
lower row): the net runs on the first stage field only, every stage reuses its stencils."""
import numpy as np
import pytest

import oracle as O
from ldgen.configs import get_config
from tests.helpers import gpu_solver, rel_l2, setup, to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n,B,over,tol", [
    ("c2", 64, 2, {}, 1e-5),                      # fused stage
    ("c3", 128, 1, {}, 1e-5),                     # K2 + proj_cluster, TC head
    ("c2", 32, 2, {"rk_order": 4}, 1e-5),
    ("c2", 64, 3, {"conv_precision": 1}, 2e-3),   # tcgen05 TF32 net
])
def test_frozen_step_matches_oracle(name, n, B, over, tol):
    cfg = get_config(name, n=n, batch=B, freeze_stencils=1, **over)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_step(u)
    ref = O.step(u0, cfg, params)
    assert rel_l2(u.cpu().numpy(), ref) < tol


def test_frozen_rollout_parity():
    cfg = get_config("c2", n=32, batch=2, freeze_stencils=1)
    cfg, u0, params = setup(cfg)
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_rollout(u, 50)
    assert rel_l2(u.cpu().numpy(), O.rollout(u0, cfg, params, 50)) < 1e-4
