"""GPU parity of the history temporal-correction block (Eq. 2
P:203-212, Eq. 12; readings N3-1..N3-3 in DESIGN.md §8d): the ring of the last k_c step
inputs in the workspace, the O_F-family operator (spectral.cu, 2 k_c inputs, 2 outputs, TC layout)
at every k_c-th step, its output added at the last stage -- against the fp64 oracle over rollouts
that cross several corrections."""
import numpy as np
import pytest

import oracle as O
from ldgen import make_weights
from ldgen.configs import get_config
from ldgen.ic import make_config_ic
from ldgen.spectral import spectral_blob
from tests.helpers import gpu_solver, rel_l2, to_dev

pytestmark = pytest.mark.gpu


def _setup(name, n, B, kc, K, L, C, scale=0.2, **over):
    cfg = get_config(name, n=n, batch=B, tc_head=0, tc_mode=1, tc_interval=kc, tc_kmax=K, tc_layers=L,
                     tc_width=C, **over)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    conv = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="stress") if cfg.stencil_mode == 0 \
        else np.zeros(0, np.float32)
    tc = spectral_blob(K, C, L, seed=2, scale=scale, n_in=2 * kc, n_out=2)
    return cfg, u0, conv, np.concatenate([conv, tc]).astype(np.float32)


@pytest.mark.parametrize("name,n,B,kc,K,L,C,over,steps,tol", [
    ("c3", 32, 2, 4, 6, 2, 8, {}, 9, 1e-4),                          # forced flow (the paper's use)
    ("c3", 64, 2, 3, 12, 1, 6, {}, 7, 1e-4),                         # N = 64, fused stage
    ("c2", 32, 3, 1, 5, 2, 4, {}, 4, 1e-4),                          # k_c = 1: every step
    ("c3", 32, 2, 2, 4, 2, 4, {"stencil_mode": 1}, 5, 1e-4),         # physics-only FV + TC
    ("c3", 64, 2, 4, 10, 2, 8, {"conv_precision": 1}, 9, 2e-3),      # tcgen05 TF32 net
    ("c3", 128, 1, 2, 8, 2, 4, {}, 5, 1e-4),                          # large-N form (global passes)
    ("c4", 256, 1, 3, 12, 1, 4, {"conv_precision": 1}, 4, 2e-3),     # c4 grid, large-N form, TF32 net
    ("c3", 128, 2, 2, 20, 1, 4, {}, 3, 1e-4),                         # large-N, K + 1 > 16: generic passes
])
def test_history_tc_rollout_matches_oracle(name, n, B, kc, K, L, C, over, steps, tol):
    cfg, u0, conv, params = _setup(name, n, B, kc, K, L, C, **over)
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_rollout(u, steps)
    ref = O.rollout(u0, cfg, params, steps)
    err = rel_l2(u.cpu().numpy(), ref)
    assert err < tol, err
    plain = O.rollout(u0, cfg.replace(tc_mode=0), conv if conv.size else None, steps)
    assert rel_l2(plain, ref) > 10 * tol     # the corrections are live


def test_history_tc_graph_and_host_paths_agree():
    import torch
    cfg, u0, conv, params = _setup("c3", 32, 2, 3, 5, 2, 4)
    a = gpu_solver(cfg, params)
    b = gpu_solver(cfg, params)
    b.set_graph_replay(False)
    ua, ub = to_dev(u0), to_dev(u0)
    a.ld_rollout(ua, 4)
    a.ld_rollout(ua, 3)
    b.ld_rollout(ub, 7)
    assert torch.equal(ua, ub)
    c = gpu_solver(cfg, params)
    uh = torch.from_numpy(u0.astype(np.float32)).pin_memory()
    c.ld_rollout_host(uh, 7)
    assert torch.equal(ua.cpu(), uh)
