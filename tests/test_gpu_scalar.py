"""GPU parity of the passive scalar ("mixture transport" of the shear flow; readings S1-S4,
DESIGN.md §8h) against the fp64 oracle (Oracle.step_scalar, pinned in tests/test_scalar_oracle.py).
Tolerances as the momentum step: one step 1e-5 (fp32 net) / 2e-3 (TF32 net); 20-step rollout 1e-4."""
import numpy as np
import pytest

import oracle as O
from ldgen import make_weights
from ldgen.configs import get_config
from ldgen.ic import make_config_ic, make_scalar_ic
from tests.helpers import gpu_solver, rel_l2, to_dev

pytestmark = pytest.mark.gpu


def _setup(n, B, rk, prec, init="stress", D=5e-4):
    cfg = get_config("c4", n=n, batch=B, rk_order=rk, conv_precision=prec, scalar_mode=1, scalar_diff=D)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=1, init=init)
    s0 = make_scalar_ic(n, B) + 0.05 * np.random.default_rng(n).standard_normal((B, n, n))
    return cfg, u0, s0, params


@pytest.mark.parametrize("n,B,rk,prec,tol", [(32, 2, 3, 0, 1e-5), (64, 2, 3, 1, 2e-3), (64, 1, 4, 0, 1e-5),
                                             (128, 1, 2, 1, 2e-3), (256, 1, 3, 0, 1e-5)])
def test_scalar_one_step(n, B, rk, prec, tol):
    cfg, u0, s0, params = _setup(n, B, rk, prec)
    o = O.Oracle(cfg, params)
    uref, sref = o.step_scalar(u0, s0)
    s = gpu_solver(cfg, params)
    u, sd = to_dev(u0), to_dev(s0)
    s.ld_step_scalar(u, sd)
    assert rel_l2(sd.cpu().numpy(), sref) < tol
    assert rel_l2(sd.cpu().numpy() - s0, sref - s0) < 100 * tol     # the increment itself
    assert rel_l2(u.cpu().numpy(), uref) < tol


def test_scalar_rollout_and_mass():
    import torch
    cfg, u0, s0, params = _setup(64, 2, 3, 0, init="normal")
    o = O.Oracle(cfg, params)
    uref, sref = u0, s0
    for _ in range(20):
        uref, sref = o.step_scalar(uref, sref)
    s = gpu_solver(cfg, params)
    u, sd = to_dev(u0), to_dev(s0)
    s.ld_rollout_scalar(u, sd, 20)
    assert rel_l2(sd.cpu().numpy(), sref) < 1e-4
    assert rel_l2(u.cpu().numpy(), uref) < 1e-4
    m0 = s0.sum(axis=(1, 2))
    assert np.allclose(sd.double().sum(dim=(1, 2)).cpu().numpy(), m0, rtol=1e-5)


def test_scalar_handle_rejects_plain_step():
    from paper_2507_01975_b200 import ldsolver as L
    cfg, u0, s0, params = _setup(32, 1, 3, 0)
    s = gpu_solver(cfg, params)
    with pytest.raises(L.LDError):
        s.ld_step(to_dev(u0))
