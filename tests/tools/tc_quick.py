"""Quick on-GPU check of the tcgen05 conv against the fp32 SIMT path (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from ldgen.configs import get_config
from tests.helpers import gpu_solver, setup, to_dev

for name, n, B in [("c2", 64, 2), ("c1", 32, 1), ("c3", 128, 3)]:
    cfg = get_config(name, n=n, batch=B, conv_precision=1)
    cfg, u0, params = setup(cfg, init="stress")
    a = gpu_solver(cfg, params)
    b = gpu_solver(cfg.replace(conv_precision=0), params)
    U = to_dev(u0)
    wa = torch.empty((B, 24, n, n), device="cuda"); wb = torch.empty_like(wa)
    a.ld_eval_stencils(U, wa); b.ld_eval_stencils(U, wb)
    torch.cuda.synchronize()
    d = (wa - wb)
    print(name, "relL2 tf32 vs fp32 stencils:", float(d.norm() / wb.norm()), "maxabs", float(d.abs().max()),
          "finite", bool(torch.isfinite(wa).all()))
    if float(d.norm() / wb.norm()) > 1e-2:
        bad = (d.abs() > 1e-2 * wb.abs().max()).nonzero()[:10]
        print("  first bad idx (b,c,y,x):", bad.tolist())
