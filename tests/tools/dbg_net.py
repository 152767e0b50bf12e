import numpy as np, torch
import oracle as O
from ldgen.configs import get_config
from tests.helpers import gpu_solver, rel_l2, setup, to_dev
for name,n,B,prec,L in [("c1",32,2,1,2),("c1",32,2,1,3),("c2",64,2,1,2),("c2",64,2,1,3),("c1",64,1,1,2),("c1",32,1,1,2)]:
    cfg = get_config(name, n=n, batch=B, conv_precision=prec, n_layers=L)
    cfg, u0, params = setup(cfg, init="stress")
    s = gpu_solver(cfg, params)
    U = to_dev(u0)
    layers = O.unpack_params(params, cfg.n_layers, cfg.width, cfg.n_out)
    Rref = np.moveaxis(O.net_forward(u0, layers, cfg.activation), -1, 1)
    R = torch.empty((B, cfg.n_out, n, n), device="cuda")
    s.ld_eval_net(U, R)
    R = R.cpu().numpy()
    d = np.abs(R - Rref).max(axis=1)
    print(name, n, B, "L", L, "relL2 %.3e" % rel_l2(R, Rref), "bad cells (err>1e-2*max):", int((d > 1e-2*np.abs(Rref).max()).sum()), "of", d.size)
    for b in range(B):
        bx = np.where(d[b].max(axis=0) > 1e-2*np.abs(Rref).max())[0]; by = np.where(d[b].max(axis=1) > 1e-2*np.abs(Rref).max())[0]
        print("   b", b, "bad x", bx[:20], "bad y", by[:40])
