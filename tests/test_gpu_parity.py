"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same
seeded inputs.  Tolerances (BASELINE.json north_star):
relative L2 <= 1e-5 for one step / one component with the fp32 conv, <= 2e-3 with
the TF32 tensor-core conv, <= 1e-3 after a 100-step rollout.
"""
import math

import numpy as np
import pytest

import oracle as O
from ldgen import make_ic, make_weights
from ldgen.configs import get_config
from tests.helpers import gpu_solver, rel_l2, setup, to_dev

pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-5


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------- projection (a6)

@pytest.mark.parametrize("n,B", [(8, 3), (16, 2), (32, 3), (64, 4), (128, 3), (256, 2), (512, 2), (1024, 1),
                                 (2048, 1), (4096, 1)])
def test_projection_parity(n, B):
    torch = _torch()
    cfg = get_config("c2", n=n, batch=B, dt=0.01, stencil_mode=1)
    s = gpu_solver(cfg, None)
    u = make_ic("noise", n, B, seed=n)
    out = torch.empty_like(to_dev(u))
    s.ld_project(to_dev(u), out)
    got = out.cpu().numpy()
    ref = O.project(u, cfg.h)
    assert rel_l2(got, ref) < TOL_FP32
    d = O.div_c(got.astype(np.float64), cfg.h)
    assert np.abs(d).max() < 1e-4 * np.abs(u).max() / cfg.h


@pytest.mark.parametrize("n,B", [(2048, 1), (4096, 2)])
def test_projection_repeatable_four_step(n, B):
    """The four-step projection passes (N >= 2048) give bitwise the same result on every call, each equal to
    the oracle: an intra-CTA race on the shared twiddle tables (fixed in session 6 -- the N = 4096 column pass
    built its W256 table from W4096 entries other warps had not yet written) shows up as call-to-call
    differences on noise input, whose high modes every twiddle touches."""
    torch = _torch()
    cfg = get_config("c2", n=n, batch=B, dt=0.01, stencil_mode=1)
    s = gpu_solver(cfg, None)
    u = make_ic("noise", n, B, seed=n + 1)
    ud = to_dev(u)
    ref = O.project(u, cfg.h)
    first = None
    for _ in range(4):
        out = torch.empty_like(ud)
        s.ld_project(ud, out)
        got = out.cpu().numpy()
        if first is None:
            first = got
            assert rel_l2(got, ref) < TOL_FP32
        else:
            assert np.array_equal(got.view(np.uint32), first.view(np.uint32))


def test_projection_in_place_and_idempotent():
    torch = _torch()
    cfg = get_config("c2", n=64, batch=2, dt=0.01, stencil_mode=1)
    s = gpu_solver(cfg, None)
    u = to_dev(make_ic("spectrum", 64, 2, seed=1))
    once = torch.empty_like(u)
    s.ld_project(u, once)
    twice = once.clone()
    s.ld_project(twice, twice)
    assert rel_l2(twice.cpu().numpy(), once.cpu().numpy()) < 1e-6


# ---------------------------------------------------------------- net (a1, a2)

@pytest.mark.parametrize("name,n,B", [("c1", 32, 1), ("c2", 64, 2), ("c3", 16, 2)])
def test_net_raw_and_stencils_parity(name, n, B):
    torch = _torch()
    cfg = get_config(name, n=n, batch=B)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    U = to_dev(u0)
    R = torch.empty((B, cfg.n_out, n, n), device="cuda")
    s.ld_eval_net(U, R)
    layers = O.unpack_params(params, cfg.n_layers, cfg.width, cfg.n_out)
    Rref = O.net_forward(u0, layers, cfg.activation)            # [B][N][N][n_out]
    assert rel_l2(R.cpu().numpy(), np.moveaxis(Rref, -1, 1)) < TOL_FP32
    w = torch.empty((B, 24, n, n), device="cuda")
    s.ld_eval_stencils(U, w)
    wref = O.constrain(Rref).reshape(B, n, n, 24)
    assert rel_l2(w.cpu().numpy(), np.moveaxis(wref, -1, 1)) < TOL_FP32


# ---------------------------------------------------------------- tendency (a3, a4)

@pytest.mark.parametrize("name,n,B,mode", [("c1", 32, 1, 0), ("c1", 16, 2, 1), ("c2", 64, 2, 0),
                                           ("c3", 32, 2, 0), ("c3", 64, 1, 1)])
def test_tendency_parity(name, n, B, mode):
    torch = _torch()
    cfg = get_config(name, n=n, batch=B, stencil_mode=mode)
    if mode == 1:
        cfg = cfg.replace(tc_head=0)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    T = torch.empty((B, 2, n, n), device="cuda")
    s.ld_eval_tendency(to_dev(u0), T)
    o = O.Oracle(cfg, params)
    Tref, _ = o.T(u0)
    assert rel_l2(T.cpu().numpy(), Tref) < TOL_FP32


# ---------------------------------------------------------------- one step (a1-a7)

ONE_STEP_CASES = [
    ("c1", 32, 1, 2, {}),
    ("c1", 8, 2, 2, {}),                               # smallest grid, ragged tile
    ("c2", 64, 3, 3, {}),
    ("c2", 64, 2, 4, {}),                               # classical RK4 path
    ("c3", 128, 2, 3, {}),                              # forcing + drag + TC head
    ("c4", 64, 2, 3, {}),                               # shear IC + TC (reduced N)
    ("c2", 32, 2, 3, {"stencil_mode": 1}),              # physics-only (fixed stencils)
    ("c1", 16, 2, 2, {"stencil_mode": 1}),
]


@pytest.mark.parametrize("name,n,B,rk,over", ONE_STEP_CASES)
def test_one_step_parity(name, n, B, rk, over):
    cfg = get_config(name, n=n, batch=B, rk_order=rk, **over)
    if over.get("stencil_mode") == 1:
        cfg = cfg.replace(tc_head=0)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_step(u)
    got = u.cpu().numpy()
    ref = O.step(u0, cfg, params)
    assert rel_l2(got, ref) < TOL_FP32, rel_l2(got, ref)
    assert s.step_index() == 1


def test_tc_interval_gating_matches_oracle():
    cfg = get_config("c3", n=32, batch=2, tc_interval=3)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    o = O.Oracle(cfg, params)
    ref = u0
    for k in range(4):
        s.ld_step(u)
        ref = o.step(ref)
        assert rel_l2(u.cpu().numpy(), ref) < 5 * TOL_FP32, k


# ---------------------------------------------------------------- rollouts

@pytest.mark.parametrize("name,n,B,steps", [("c1", 32, 1, 100), ("c2", 64, 2, 100)])
def test_rollout_parity_100_steps(name, n, B, steps):
    cfg = get_config(name, n=n, batch=B)
    cfg, u0, params = setup(cfg, init="normal")
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_rollout(u, steps)
    ref = O.rollout(u0, cfg, params, steps)
    assert rel_l2(u.cpu().numpy(), ref) < 1e-3
    assert s.step_index() == steps


def test_rollout_snapshots_and_zero_steps():
    torch = _torch()
    cfg = get_config("c1", n=16, batch=2)
    cfg, u0, params = setup(cfg)
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_rollout(u, 0)
    assert torch.equal(u, to_dev(u0))
    traj = torch.empty((3, 2, 2, 16, 16), device="cuda")
    s.ld_rollout(u, 6, traj, 2)
    v = to_dev(u0)
    s2 = gpu_solver(cfg, params)
    for k in range(3):
        s2.ld_rollout(v, 2)
        assert torch.equal(traj[k], v)
    assert torch.equal(u, v)


@pytest.mark.parametrize("name,n,B,over", [
    ("c2", 32, 2, {}),
    ("c3", 32, 5, {"tc_interval": 2}),      # odd split (2 + 3), TC gating across calls
    ("c2", 64, 3, {"rk_order": 4}),         # RK4 accumulator halves
    ("c2", 32, 4, {"conv_precision": 1}),   # tcgen05 net on the halves
])
def test_rollout_host_matches_device(name, n, B, over):
    """ld_rollout_host (H2D + steps + D2H) equals ld_rollout on the device bitwise, across calls
    (step counter / TC gating)."""
    torch = _torch()
    cfg = get_config(name, n=n, batch=B, **over)
    cfg, u0, params = setup(cfg)
    a = gpu_solver(cfg, params)
    b = gpu_solver(cfg, params)
    ud = to_dev(u0)
    a.ld_rollout(ud, 3)
    a.ld_rollout(ud, 2)
    uh = torch.from_numpy(u0.astype(np.float32)).pin_memory()
    b.ld_rollout_host(uh, 3)
    b.ld_rollout_host(uh, 2)
    assert torch.equal(ud.cpu(), uh)
    assert b.step_index() == 5


# ---------------------------------------------------------------- invariants on the GPU (T3)

def test_batch_permutation_bitwise_and_determinism():
    torch = _torch()
    cfg = get_config("c2", n=64, batch=4)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    a = to_dev(u0)
    s.ld_step(a)
    perm = [2, 0, 3, 1]
    b = to_dev(u0[perm])
    s2 = gpu_solver(cfg, params)
    s2.ld_step(b)
    assert torch.equal(a[perm], b)
    c = to_dev(u0)
    s3 = gpu_solver(cfg, params)
    s3.ld_step(c)
    assert torch.equal(a, c)


def test_kolmogorov_fixed_point_gpu():
    n = 64
    cfg = get_config("c3", n=n, batch=1, stencil_mode=1, tc_head=0)
    h = cfg.h
    y = (np.arange(n) + 0.5) * h
    kh = 2 * math.sin(4 * h / 2) / h
    A = 1.0 / (cfg.nu * kh * kh + cfg.drag)
    u0 = np.zeros((1, 2, n, n))
    u0[0, 0] = (A * np.sin(4 * y))[:, None]
    cfg = cfg.replace(dt=0.5 * h / A)
    s = gpu_solver(cfg, None)
    u = to_dev(u0)
    s.ld_rollout(u, 20)
    assert rel_l2(u.cpu().numpy(), u0) < 1e-5


def test_constant_field_fixed_point_gpu():
    cfg = get_config("c2", n=32, batch=2)
    cfg, _, params = setup(cfg, init="stress")
    u0 = np.ones((2, 2, 32, 32)) * np.array([0.3, -0.7])[None, :, None, None]
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_rollout(u, 5)
    assert np.abs(u.cpu().numpy() - u0).max() < 1e-6


def test_nonfinite_detected_with_step_index():
    cfg = get_config("c1", n=16, batch=1, stencil_mode=1, nu=0.0, dt=50.0)
    from paper_2507_01975_b200 import ldsolver as L
    s = gpu_solver(cfg, None, check_finite_every=1)
    u = to_dev(make_ic("noise", 16, 1, seed=0) * 10)
    with pytest.raises(L.LDError, match="NONFINITE.*step"):
        s.ld_rollout(u, 50)


def test_graph_replay_bitwise_equals_eager():
    torch = _torch()
    cfg = get_config("c3", n=32, batch=2, tc_interval=2)
    cfg, u0, params = setup(cfg, init="stress")
    a = gpu_solver(cfg, params)
    b = gpu_solver(cfg, params)
    b.set_graph_replay(False)
    ua, ub = to_dev(u0), to_dev(u0)
    a.ld_rollout(ua, 5)
    b.ld_rollout(ub, 5)
    assert torch.equal(ua, ub)
    # a different field pointer re-captures
    uc = to_dev(u0)
    c = gpu_solver(cfg, params)
    c.ld_rollout(uc, 2)
    ud = uc.clone()
    c.ld_rollout(ud, 3)
    assert torch.equal(ud, ua)


@pytest.mark.parametrize("n,f,B", [(64, 4, 3), (256, 16, 2), (1024, 16, 1), (96 * 0 + 128, 1, 1)])
def test_downsample_parity(n, f, B):
    """ld_downsample (NEXT-1 data path) equals the oracle's block mean."""
    torch = _torch()
    from paper_2507_01975_b200 import ldsolver as L
    u = make_ic("noise", n, B, seed=n + f)
    fine = to_dev(u)
    coarse = torch.empty((B, 2, n // f, n // f), device="cuda")
    L.ld_downsample(fine, f, coarse)
    assert rel_l2(coarse.cpu().numpy(), O.downsample(u, f)) < 1e-6


@pytest.mark.parametrize("name,n,B,rk,over", [
    ("c3", 64, 3, 3, {}),                                # forcing + drag + TC term (add_e)
    ("c2", 64, 2, 4, {}),                                # RK4 accumulator
    ("c2", 32, 5, 3, {"stencil_mode": 1, "tc_head": 0}), # fixed stencils, 16 rows per CTA
    ("c2", 64, 2, 3, {"conv_precision": 1}),             # TF32 net
    ("c2", 32, 1, 2, {}),                                # small batch: 4 rows per CTA
])
def test_fused_stage_bitwise_equals_two_kernel_path(name, n, B, rk, over, monkeypatch):
    """N <= 64: the fused flux + projection kernel (fft.cu flux_proj_cluster) runs the same fp32
    operations as flux_rk_kernel followed by proj_cluster, so the step is bitwise identical to
    the two-kernel path (LD_NO_FUSED_STAGE) -- and both match the oracle (test_one_step_parity)."""
    torch = _torch()
    cfg = get_config(name, n=n, batch=B, rk_order=rk, **over)
    cfg, u0, params = setup(cfg, init="stress")
    fused = gpu_solver(cfg, params)
    fused.set_graph_replay(False)
    uf = to_dev(u0)
    fused.ld_rollout(uf, 3)
    monkeypatch.setenv("LD_NO_FUSED_STAGE", "1")
    two = gpu_solver(cfg, params)
    two.set_graph_replay(False)
    ut = to_dev(u0)
    two.ld_rollout(ut, 3)
    assert torch.equal(uf, ut), float((uf - ut).abs().max())
    ref = O.step(O.step(O.step(u0, cfg, params), cfg, params), cfg, params)
    assert rel_l2(uf.cpu().numpy(), ref) < (TOL_FP32 if cfg.conv_precision == 0 else 2e-3)
