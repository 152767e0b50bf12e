"""Quick on-GPU check of the tcgen05 conv paths against the oracle (debug aid): prints the
relative L2 error of the raw net output R and of one step for each conv precision."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import oracle as O
from ldgen.configs import get_config
from tests.helpers import gpu_solver, rel_l2, setup, to_dev

for name, n, B in [("c2", 64, 2), ("c1", 32, 1), ("c3", 128, 2)]:
    cfg0 = get_config(name, n=n, batch=B)
    cfg0, u0, params = setup(cfg0, init="stress")
    layers = O.unpack_params(params, cfg0.n_layers, cfg0.width, cfg0.n_out)
    Rref = np.moveaxis(O.net_forward(u0, layers, cfg0.activation), -1, 1)
    uref = O.step(u0, cfg0, params)
    for prec in (0, 1, 2):
        cfg = cfg0.replace(conv_precision=prec)
        s = gpu_solver(cfg, params)
        U = to_dev(u0)
        R = torch.empty((B, cfg.n_out, n, n), device="cuda")
        s.ld_eval_net(U, R)
        u = to_dev(u0)
        s.ld_step(u)
        torch.cuda.synchronize()
        print(f"{name} N={n} prec={prec}: relL2 R={rel_l2(R.cpu().numpy(), Rref):.3e} "
              f"step={rel_l2(u.cpu().numpy(), uref):.3e}", flush=True)
