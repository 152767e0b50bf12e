"""Round-2 GPU parity coverage (VERDICT r01 "parity on every config"):

* 100-step TF32 rollouts against the fp64 oracle on the c3 physics (128^2: forcing, drag, TC head)
  and the c4 physics (256^2 double shear layer, TC head) -- Eq. 2 P:203-212 rolled out;
* the c5b per-GPU shard (1024^2, B = 64) one full step in the TF32 headline precision, element 0;
* Pin-14: an ensemble shard of B/P elements gives bitwise the same rows as the
  full-batch step, across the batch-dependent kernel switches (two-CTA conv form when a layer has
  <= 2 tiles per SM, contiguous-tile operand layout for N >= 128, the projection's cluster size,
  the first layer's 4-byte producer path for grids of several tiles per CTA).

Tolerances: BASELINE.json north_star (one step 2e-3 for the TF32 conv, 100 steps 1e-3).
"""
import numpy as np
import pytest

import oracle as O
from ldgen import make_weights
from ldgen.configs import get_config
from ldgen.ic import make_config_ic
from tests.helpers import gpu_solver, rel_l2, setup, to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(1500)
@pytest.mark.parametrize("name,n,B", [("c3", 128, 2), ("c4", 256, 1)])
def test_rollout_100_steps_tf32(name, n, B):
    cfg = get_config(name, n=n, batch=B, conv_precision=1)
    cfg, u0, params = setup(cfg, init="normal")
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_rollout(u, 100)
    ref = O.rollout(u0, cfg, params, 100)
    got = u.cpu().numpy()
    assert np.isfinite(got).all()
    err = rel_l2(got, ref)
    assert err < 1e-3, err
    # the learned part moved the trajectory (not a pure physics rollout) and e was applied
    assert rel_l2(O.rollout(u0, cfg.replace(stencil_mode=1, tc_head=0), None, 100), ref) > 1e-2 * err


@pytest.mark.timeout(1500)
def test_c5b_shard_full_step_element0_tf32():
    cfg = get_config("c5b", batch=64, conv_precision=1)
    cfg, u0, params = setup(cfg, init="normal", elements=range(64))
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_step(u)
    ref = O.step(u0[:1], cfg, params)
    assert rel_l2(u[0:1].cpu().numpy(), ref) < 2e-3


# --------------------------------------------------------------------------- Pin-14

def _shard_vs_full(name, n, B, P, prec, steps=2):
    import torch
    cfg = get_config(name, n=n, batch=B, conv_precision=prec, tc_interval=2)
    full = make_config_ic(cfg, elements=range(B)).astype(np.float32)
    cfg = cfg.with_dt(full)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="stress")
    s = gpu_solver(cfg, params)
    uf = to_dev(full)
    s.ld_rollout(uf, steps)                      # crosses a TC-correction step (k_c = 2)
    b = B // P
    for r in range(P):
        part = make_config_ic(cfg.replace(batch=b), elements=range(r * b, (r + 1) * b)).astype(np.float32)
        assert np.array_equal(part, full[r * b:(r + 1) * b])      # the inputs shard bitwise (ldgen)
        sr = gpu_solver(cfg.replace(batch=b), params)
        us = to_dev(part)
        sr.ld_rollout(us, steps)
        assert torch.equal(us, uf[r * b:(r + 1) * b]), (r, float((us - uf[r * b:(r + 1) * b]).abs().max()))


@pytest.mark.parametrize("n,B,P,prec", [
    (64, 64, 2, 1),     # 512 tiles per layer (one CTA per SM) vs 256 per shard (two-CTA form)
    (64, 32, 4, 1),     # two-CTA form vs 64 tiles
    (64, 64, 2, 2),     # F16 operands
    (128, 16, 2, 1),    # contiguous tiles; projection cluster 8 -> 8 / 4 CTAs per element
    (128, 8, 8, 1),     # one element per rank: first layer without the 4-byte producer path
    (256, 4, 2, 1),     # pencil projection
])
def test_pin14_ensemble_shard_bitwise(n, B, P, prec):
    _shard_vs_full("c3", n, B, P, prec)


# --------------------------------------------------------------------------- pipelined host path

@pytest.mark.parametrize("name,n,B,steps,over", [("c4", 128, 128, 2, {}), ("c2", 256, 32, 1, {}),
                                                 ("c3", 256, 32, 3, {"tc_interval": 2}),
                                                 ("c2", 512, 10, 1, {"rk_order": 4}), ("c1", 512, 8, 2, {})])
def test_host_rollout_chunks_bitwise(name, n, B, steps, over):
    """ld_rollout_host runs B/C-element chunks on their own streams (copies of one chunk overlap the
    kernels of the others); the result must equal the device-resident whole-batch rollout bitwise."""
    import torch
    cfg = get_config(name, n=n, batch=B, conv_precision=1, **over)
    cfg, u0, params = setup(cfg, init="stress")
    a = gpu_solver(cfg, params)
    ud = to_dev(u0)
    a.ld_rollout(ud, steps)
    b = gpu_solver(cfg, params)
    uh = torch.from_numpy(u0.astype(np.float32)).pin_memory()
    b.ld_rollout_host(uh, steps)
    assert torch.equal(uh, ud.cpu())
    assert b.step_index() == steps
    b.ld_rollout_host(uh, 1)          # graphs of the chunk views replayed, TC gating continues
    a.ld_rollout(ud, 1)
    assert torch.equal(uh, ud.cpu())


def test_project_rejects_burgers_handle():
    """a Burgers handle has no spectrum / pressure buffers; ld_project must refuse it (at n = 256,
    where the pencil passes would otherwise write B N^2 complex values past the placeholders)."""
    import torch
    from paper_2507_01975_b200 import ldsolver as L
    cfg = get_config("c1", n=256, batch=2, dt=0.01)
    s = gpu_solver(cfg, make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0))
    u = torch.zeros((2, 2, 256, 256), device="cuda")
    with pytest.raises(L.LDError, match="INVALID_ARG"):
        s.ld_project(u, torch.empty_like(u))


def test_binding_rejects_bad_tensors():
    import torch
    from paper_2507_01975_b200 import ldsolver as L
    cfg = get_config("c2", n=32, batch=2)
    cfg, u0, params = setup(cfg)
    s = gpu_solver(cfg, params)
    for bad in (to_dev(u0).double(), to_dev(u0)[:, :, :, :16], to_dev(u0).transpose(2, 3),
                torch.from_numpy(u0.astype(np.float32))):
        with pytest.raises(L.LDError):
            s.ld_step(bad)
