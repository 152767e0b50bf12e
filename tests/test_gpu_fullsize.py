"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (the
whole batch in one call), checked on sampled outputs the oracle can compute:

* c2 (64^2, B=32), c3 (128^2, B=128), c4 (256^2, B=64): one full step of the whole batch
  on the GPU; the oracle recomputes sampled batch elements (elements are independent).
* c5b (1024^2, B=64 per GPU) and c5a (4096^2, B=8, single GPU): components on element
  samples -- the net on periodic patches (finite receptive field: a cell at distance >= L
  from the patch edge is exact), the tendency given the GPU's stencils, and the full
  spectral projection of one element -- plus invariants that hold at any size.
"""
import numpy as np
import pytest

import oracle as O
from ldgen.configs import get_config
from tests.helpers import gpu_solver, rel_l2, setup, to_dev

pytestmark = pytest.mark.gpu

TOL = {0: 1e-5, 1: 2e-3, 2: 2e-3}


def _torch():
    import torch
    return torch


@pytest.mark.parametrize("prec", [0, 1, 2])
@pytest.mark.parametrize("name,samples", [("c2", [0, 13, 31]), ("c3", [0, 127]), ("c4", [0])])
def test_full_batch_one_step(name, samples, prec):
    torch = _torch()
    cfg = get_config(name, conv_precision=prec)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_step(u)
    got = u.cpu().numpy()
    assert np.isfinite(got).all()
    ref = O.step(u0[samples], cfg, params)
    err = rel_l2(got[samples], ref)
    assert err < TOL[prec], err
    if name == "c4":   # identical IC for every element (R17): outputs must be bitwise identical
        assert torch.equal(u[0:1].expand_as(u), u)


def _net_patch(u_el, layers, act, cy, cx, half=24):
    """Oracle net on a periodic patch of u_el centred at (cy, cx): returns R at the centre
    (exact because the patch half-width exceeds the net's receptive radius)."""
    n = u_el.shape[-1]
    ys = (np.arange(cy - half, cy + half) % n)
    xs = (np.arange(cx - half, cx + half) % n)
    patch = u_el[:, ys][:, :, xs][None]
    R = O.net_forward(patch, layers, act)
    return R[0, half, half]


@pytest.mark.parametrize("name,B,prec", [("c5b", 64, 2), ("c5b", 64, 1), ("c5a", 8, 2)])
def test_large_components(name, B, prec):
    torch = _torch()
    cfg = get_config(name, batch=B, conv_precision=prec)
    cfg, u0, params = setup(cfg, init="stress", elements=range(B))
    n = cfg.n
    s = gpu_solver(cfg, params)
    U = to_dev(u0)
    # (a) net output at sampled cells of sampled elements (patch oracle)
    R = torch.empty((B, cfg.n_out, n, n), device="cuda")
    s.ld_eval_net(U, R)
    layers = O.unpack_params(params, cfg.n_layers, cfg.width, cfg.n_out)
    rng = np.random.default_rng(5)
    got, ref = [], []
    for b in (0, B - 1):
        for _ in range(6):
            cy, cx = rng.integers(0, n, 2)
            ref.append(_net_patch(u0[b], layers, cfg.activation, int(cy), int(cx)))
            got.append(R[b, :, cy, cx].cpu().numpy())
    assert rel_l2(np.array(got), np.array(ref)) < TOL[prec]
    del R
    # (b) tendency of element 0 given the GPU's own stencils (isolates a3-a4 at full size)
    w = torch.empty((B, 24, n, n), device="cuda")
    s.ld_eval_stencils(U, w)
    T = torch.empty_like(U)
    s.ld_eval_tendency(U, T)
    w0 = w[0].permute(1, 2, 0).cpu().numpy().astype(np.float64).reshape(n, n, 2, 2, 6)[None]
    Tref = O.tendency(u0[:1], w0, cfg, cfg.h)
    # T = -(F(i+1) - F(i))/h: in fp32 the face-flux difference cancels to ~h |dF| while its
    # rounding stays ~eps32 |F|, so the relative error of T alone grows like eps32/h (about
    # 4e-5 at N = 4096).  The step output u + dt T is not affected (dt T << u).
    tol_T = 1e-5 * max(1.0, n / 512)
    assert rel_l2(T[0:1].cpu().numpy(), Tref) < tol_T
    del w, T
    # (c) projection of element 0 (full spectral solve) + invariants on the whole batch
    P = torch.empty_like(U)
    s.ld_project(U, P)
    assert rel_l2(P[0:1].cpu().numpy(), O.project(u0[:1], cfg.h)) < 1e-5
    Pn = P.double()
    div = ((torch.roll(Pn[:, 0], -1, -1) - torch.roll(Pn[:, 0], 1, -1)) +
           (torch.roll(Pn[:, 1], -1, -2) - torch.roll(Pn[:, 1], 1, -2))) / (2 * cfg.h)
    assert float(div.abs().max()) < 1e-4 * float(U.abs().max()) / cfg.h
    assert torch.allclose(Pn.mean(dim=(-1, -2)), U.double().mean(dim=(-1, -2)), atol=1e-6)


def test_c5b_shard_full_step_element0():
    """One full c5b step (1024^2, the bench's per-GPU shard of 64) against the oracle on
    element 0 (about 1 TFLOP of fp64 oracle work)."""
    cfg = get_config("c5b", batch=64, conv_precision=2)
    cfg, u0, params = setup(cfg, init="normal", elements=range(64))
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_step(u)
    ref = O.step(u0[:1], cfg, params)
    assert rel_l2(u[0:1].cpu().numpy(), ref) < 2e-3
