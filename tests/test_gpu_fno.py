"""GPU parity of the step with the frequency-domain branch O_F on (
PAPER.md Eq. 6-8: O^(m) = O_P + O_L + O_F; readings N2-1..N2-6 in DESIGN.md §8c) against the fp64
oracle: spectral.cu evaluates O_F of each stage field on the faces, K2 / the fused stage kernel
add it to the stencil face values.  Bounds as for the plain step: 1e-5 (fp32-exact net) and 2e-3
(tcgen05 TF32 net) relative L2."""
import numpy as np
import pytest

import oracle as O
from ldgen import make_weights
from ldgen.configs import get_config
from ldgen.spectral import spectral_blob
from tests.helpers import gpu_solver, rel_l2, to_dev
from ldgen.ic import make_config_ic

pytestmark = pytest.mark.gpu


def _setup(name, n, B, K, L, C, scale=0.3, **over):
    cfg = get_config(name, n=n, batch=B, fno_kmax=K, fno_layers=L, fno_width=C, **over)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = np.concatenate([make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="stress"),
                             spectral_blob(K, C, L, seed=1, scale=scale)])
    return cfg, u0, params


@pytest.mark.parametrize("name,n,B,K,L,C,over,tol", [
    ("c2", 32, 2, 5, 2, 4, {}, 1e-5),                       # N = 32 fused stage
    ("c2", 64, 2, 12, 2, 8, {}, 1e-5),                      # SPEC shape, fused stage
    ("c3", 128, 1, 8, 1, 3, {}, 1e-5),                      # K2 + proj_cluster, forcing, TC head
    ("c2", 64, 2, 6, 2, 4, {"rk_order": 4}, 1e-5),          # RK4 accumulator
    ("c1", 32, 2, 4, 1, 2, {}, 1e-5),                       # Burgers (no projection)
    ("c2", 64, 3, 10, 2, 6, {"conv_precision": 1}, 2e-3),   # tcgen05 TF32 net
    ("c4", 256, 1, 12, 2, 8, {}, 1e-5),                     # large-N form (three global passes), c4 grid
    ("c3", 256, 2, 8, 1, 4, {"conv_precision": 1, "scale": 2.0}, 2e-3),   # large-N form, TF32, forcing + TC
    ("c2", 256, 1, 20, 1, 4, {}, 1e-5),                     # large-N, K + 1 > 16: the generic passes
    ("c2", 512, 1, 15, 1, 4, {}, 1e-5),                     # large-N, 64 KB twiddle table (K + 1 = 16)
])
def test_step_with_fno_matches_oracle(name, n, B, K, L, C, over, tol):
    over = dict(over)
    scale = over.pop("scale", 0.3)      # a stronger branch where the TF32 bound would hide a 0.3-scale one
    cfg, u0, params = _setup(name, n, B, K, L, C, scale=scale, **over)
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_step(u)
    ref = O.step(u0, cfg, params)
    plain = O.step(u0, cfg.replace(fno_layers=0), params[:params.size - len(spectral_blob(K, C, L, seed=1, scale=scale))])
    err = rel_l2(u.cpu().numpy(), ref)
    assert err < tol, err
    assert rel_l2(plain, ref) > 10 * tol   # the branch changes the step by far more than the bound


def test_fno_tendency_matches_oracle():
    import torch
    cfg, u0, params = _setup("c3", 64, 2, 8, 2, 4)
    s = gpu_solver(cfg, params)
    T = torch.empty((2, 2, 64, 64), device="cuda")
    s.ld_eval_tendency(to_dev(u0), T)
    o = O.Oracle(cfg, params)
    ref, _ = o.T(np.asarray(u0, dtype=np.float64))
    assert rel_l2(T.cpu().numpy(), ref) < 1e-5


def test_fno_fused_stage_bitwise_equals_two_kernel_path(monkeypatch):
    import torch
    cfg, u0, params = _setup("c2", 64, 2, 12, 2, 8)
    a = gpu_solver(cfg, params)
    a.set_graph_replay(False)
    ua = to_dev(u0)
    a.ld_rollout(ua, 2)
    monkeypatch.setenv("LD_NO_FUSED_STAGE", "1")
    b = gpu_solver(cfg, params)
    b.set_graph_replay(False)
    ub = to_dev(u0)
    b.ld_rollout(ub, 2)
    assert torch.equal(ua, ub)


def test_fno_rollout_parity_20_steps():
    cfg, u0, params = _setup("c2", 32, 2, 5, 2, 4, scale=0.1)
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_rollout(u, 20)
    ref = O.rollout(u0, cfg, params, 20)
    assert rel_l2(u.cpu().numpy(), ref) < 1e-4
