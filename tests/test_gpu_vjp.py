"""GPU parity of the adjoint step ld_step_vjp against the fp64 adjoint oracle
(oracle/adjoint_oracle.py, itself pinned by finite differences and closed forms).

Tolerances (fp32 SIMT arithmetic throughout): u_bar relative L2 <= 1e-5, as the
forward fp32 step; theta_bar relative L2 <= 1e-4: every weight gradient is a sum over all B N^2 cells
(and 9 taps / stages) of products of fp32 quantities, whose rounding grows like eps32 sqrt(B N^2) ~
3e-5 for B N^2 = 2 x 64^2 relative to the largest terms, and cancellation between cells of opposite
sign lifts the relative error of the sum by the ratio of |terms| to |sum| (measured <= ~10 here).
"""
import numpy as np
import pytest

from ldgen import make_weights
from ldgen.configs import get_config
from ldgen.ic import make_config_ic
from oracle import adjoint_oracle as A
from tests.helpers import gpu_solver, rel_l2, to_dev

pytestmark = pytest.mark.gpu


def _case(name, n, B, rk, k, **over):
    import torch
    cfg = get_config(name, n=n, batch=B, rk_order=rk, conv_precision=0, tc_interval=2, **over)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = None if cfg.stencil_mode else make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=1, init="stress")
    g = np.random.default_rng(n + B + rk).standard_normal(u0.shape)
    ub_ref, pb_ref = A.step_vjp(u0, cfg, None if params is None else params.astype(np.float64), g, step_index=k)
    s = gpu_solver(cfg, params)
    for _ in range(k):          # advance the handle's step index to k (TC gating)
        s.ld_step(to_dev(u0))
    u, gd = to_dev(u0), to_dev(g)
    gin = torch.empty_like(u)
    gp = None if params is None else torch.zeros(params.size, device="cuda")
    s.ld_step_vjp(u, gd, gin, gp)
    torch.cuda.synchronize()
    assert torch.equal(u, to_dev(u0)) and torch.equal(gd, to_dev(g))      # inputs untouched
    return gin.cpu().numpy(), None if gp is None else gp.cpu().numpy(), ub_ref, pb_ref


@pytest.mark.parametrize("name,n,B,rk,k", [
    ("c1", 32, 1, 2, 0),        # Burgers, 3 x 32 ReLU net, RK2
    ("c2", 32, 2, 3, 0),        # NS decaying, 6 x 64 GELU, SSP-RK3
    ("c3", 32, 2, 3, 1),        # forcing + drag + TC head, correction step (k_c = 2, k = 1)
    ("c3", 16, 3, 4, 1),        # classical RK4 with the TC term
    ("c4", 64, 1, 3, 0),        # double shear layer, no correction at this step
    ("c2", 64, 2, 2, 0),
])
def test_vjp_parity(name, n, B, rk, k):
    gin, gp, ub_ref, pb_ref = _case(name, n, B, rk, k)
    assert rel_l2(gin, ub_ref) < 1e-5, rel_l2(gin, ub_ref)
    assert rel_l2(gp, pb_ref) < 1e-4, rel_l2(gp, pb_ref)


@pytest.mark.parametrize("system", [0, 1])
def test_vjp_fixed_stencils(system):
    gin, gp, ub_ref, _ = _case("c2", 32, 2, 3, 0, stencil_mode=1, system=system, tc_head=0)
    assert gp is None
    assert rel_l2(gin, ub_ref) < 1e-5


def test_vjp_independent_of_forward_precision():
    """The VJP recomputes the net in fp32 whatever conv_precision the handle's forward uses."""
    import torch
    cfg = get_config("c2", n=32, batch=2)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=1, init="stress")
    g = to_dev(np.random.default_rng(0).standard_normal(u0.shape))
    outs = []
    for prec in (0, 1):
        s = gpu_solver(cfg.replace(conv_precision=prec), params)
        gin = torch.empty_like(g)
        gp = torch.zeros(params.size, device="cuda")
        s.ld_step_vjp(to_dev(u0), g, gin, gp)
        outs.append((gin, gp))
    assert torch.equal(outs[0][0], outs[1][0])


def test_vjp_gparams_accumulate():
    import torch
    cfg = get_config("c2", n=16, batch=1)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=1, init="stress")
    s = gpu_solver(cfg.replace(conv_precision=0), params)
    g = to_dev(np.random.default_rng(2).standard_normal(u0.shape))
    gin = torch.empty_like(g)
    gp = torch.zeros(params.size, device="cuda")
    s.ld_step_vjp(to_dev(u0), g, gin, gp)
    once = gp.clone()
    s.ld_step_vjp(to_dev(u0), g, gin, gp)
    assert torch.allclose(gp, 2 * once, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("name,n,B,rk,steps", [("c3", 32, 2, 3, 3), ("c1", 32, 1, 2, 4), ("c2", 16, 2, 4, 2)])
def test_rollout_vjp_parity(name, n, B, rk, steps):
    """ld_rollout_vjp (forward states recomputed, step VJPs chained in reverse, TC gating per step) vs the
    oracle's step VJPs composed along the oracle's own rollout."""
    import torch
    import oracle as O
    cfg = get_config(name, n=n, batch=B, rk_order=rk, conv_precision=0, tc_interval=2)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=1, init="stress")
    g = np.random.default_rng(3).standard_normal(u0.shape)
    p64 = params.astype(np.float64)
    o = O.Oracle(cfg, p64)
    states = [u0]
    for _ in range(steps - 1):
        states.append(o.step(states[-1]))
    gk, pb = g, np.zeros(params.size)
    for k in range(steps - 1, -1, -1):
        ub, pk = A.step_vjp(states[k], cfg, p64, gk, step_index=k)
        gk, pb = ub, pb + pk
    s = gpu_solver(cfg, params)
    gin = torch.empty_like(to_dev(u0))
    gp = torch.zeros(params.size, device="cuda")
    s.ld_rollout_vjp(to_dev(u0), steps, to_dev(g), gin, gp)
    torch.cuda.synchronize()
    assert rel_l2(gin.cpu().numpy(), gk) < 1e-5 * steps
    assert rel_l2(gp.cpu().numpy(), pb) < 1e-4 * steps
    assert s.step_index() == 0
