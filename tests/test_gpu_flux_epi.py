"""The output layer's flux epilogue (conv_xn.cu OUT_FLUX + flux_div_kernel): for N % 128 == 0
on the tcgen05 net the last conv layer applies the stencils to the stage field itself and writes the face
fluxes, so the 24 stencils per cell never reach HBM.  Every face flux and every cell is evaluated with the
same fp32 operations in the same order as the stencil round trip (output layer -> w -> flux_rk_kernel), so
the step must be BITWISE the step with the round trip (LD_FLUX_EPI=0, run in a subprocess because the knob
is read once per process), and within the north_star bounds of the fp64 oracle (Eq. 4 P:224-227,
the RK stage P:201)."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import oracle as O
from ldgen.configs import get_config
from tests.helpers import gpu_solver, rel_l2, setup, to_dev

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from ldgen.configs import get_config
from tests.helpers import gpu_solver, setup, to_dev
name, n, B, steps, prec, rk, out = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6]), int(sys.argv[7]), sys.argv[8]
cfg = get_config(name, n=n, batch=B, conv_precision=prec, rk_order=rk, tc_interval=2)
cfg, u0, params = setup(cfg, init="stress")
s = gpu_solver(cfg, params)
u = to_dev(u0)
s.ld_rollout(u, steps)
np.save(out, u.cpu().numpy())
"""


def _run(name, n, B, steps, prec, rk, epi):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "u.npy")
        env = dict(os.environ, LD_FLUX_EPI=str(epi))
        subprocess.run([sys.executable, "-c", _CHILD, ROOT, name, str(n), str(B), str(steps), str(prec), str(rk), out],
                       check=True, env=env, timeout=600)
        return np.load(out)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name,n,B,steps,prec,rk", [
    ("c3", 128, 4, 3, 1, 3),     # forcing + drag + TC head (e through the epilogue), k_c = 2 correction step
    ("c4", 256, 2, 2, 1, 3),     # the bench workload's physics
    ("c2", 128, 3, 2, 2, 4),     # F16 operands, classical RK4 (acc)
    ("c1", 128, 2, 2, 3, 2),     # Burgers (gamma = 1/2, no projection), BF16, width-32 ReLU net
    ("c3", 128, 20, 1, 1, 3),    # more than two tiles per SM: the one-CTA-per-SM form
])
def test_flux_epilogue_bitwise_equals_stencil_round_trip(name, n, B, steps, prec, rk):
    a = _run(name, n, B, steps, prec, rk, 1)
    b = _run(name, n, B, steps, prec, rk, 0)
    assert np.array_equal(a, b), float(np.abs(a - b).max())


@pytest.mark.parametrize("name,n,B", [("c4", 256, 1), ("c3", 128, 2)])
def test_flux_epilogue_step_matches_oracle(name, n, B):
    cfg = get_config(name, n=n, batch=B, conv_precision=1)
    cfg, u0, params = setup(cfg, init="normal")
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_step(u)
    assert rel_l2(u.cpu().numpy(), O.step(u0, cfg, params)) < 2e-3
