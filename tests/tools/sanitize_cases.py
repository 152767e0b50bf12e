"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
python tests/tools/sanitize_cases.py  (run under `compute-sanitizer --tool <t> --error-exitcode 9`)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from ldgen import make_weights  # noqa: E402
from ldgen.configs import get_config  # noqa: E402
from ldgen.ic import make_scalar_ic  # noqa: E402
from paper_2507_01975_b200 import ldsolver as L  # noqa: E402
from tests.helpers import gpu_solver, setup, to_dev  # noqa: E402


def run(name, **over):
    cfg = get_config(name, **over)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_rollout(u, 2)
    torch.cuda.synchronize()
    print("ok", name, over, flush=True)
    return cfg, u0, params


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "step"):
    run("c1", n=32, batch=1, conv_precision=0)                 # SIMT conv, K2, Burgers
    run("c1", n=32, batch=1, conv_precision=1)                 # tcgen05 conv (TF32)
    run("c2", n=64, batch=2, conv_precision=1)                 # two-CTA conv form, fused flux + projection cluster
    run("c3", n=128, batch=1, conv_precision=2)                # F16 conv, contiguous tiles, proj_cluster
    run("c4", n=256, batch=1, conv_precision=1)                # pencil projection
    run("c2", n=32, batch=2, stencil_mode=2, tc_head=0)       # 5x4 kernels
if which in ("all", "slab"):
    cfg = get_config("c3", n=256, batch=1, conv_precision=1)
    cfg, u0, params = setup(cfg, init="stress")
    s = L.Solver(L.make_config(cfg), params, dist=L.ld_dist(mode=3, rank=0, world=2, nccl_comm=None))
    u = to_dev(u0)
    s.ld_step(u)
    torch.cuda.synchronize()
    print("ok slab mode 3", flush=True)
if which in ("all", "extra"):
    cfg = get_config("c4", n=32, batch=1, scalar_mode=1, scalar_diff=1e-3, conv_precision=1)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    s.ld_step_scalar(to_dev(u0), to_dev(make_scalar_ic(32, 1)))
    cfg = get_config("c3", n=32, batch=1, conv_precision=0)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    g = to_dev(np.ones_like(u0))
    gin = torch.empty_like(g)
    gp = torch.zeros(params.size, device="cuda")
    s.ld_step_vjp(to_dev(u0), g, gin, gp)
    torch.cuda.synchronize()
    print("ok scalar + vjp", flush=True)
