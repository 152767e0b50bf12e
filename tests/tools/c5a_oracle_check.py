"""c5a (4096^2) one full TF32 step of batch element 0 on the GPU vs the plain C++ oracle (fp64, all host
threads; ~16.5 TFLOP of CPU work, several minutes on 16 cores).  SURVEY.md §8d: "c5a GPU-single is compared
to O1 for 1 step on element 0".  Prints one JSON line; also run by tests/test_gpu_c5a_oracle.py when
LD_SLOW_TESTS=1."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main(prec=1):
    import torch
    from ldgen.configs import get_config
    from oracle import cpp_oracle as X
    from tests.helpers import gpu_solver, rel_l2, setup, to_dev
    cfg = get_config("c5a", batch=1, conv_precision=prec)
    cfg, u0, params = setup(cfg, init="normal", elements=[0])
    s = gpu_solver(cfg, params)
    u = to_dev(u0)
    s.ld_step(u)
    torch.cuda.synchronize()
    got = u.cpu().numpy()
    del u, s
    t0 = time.time()
    ref = X.step(u0, cfg, params)
    el = time.time() - t0
    err = rel_l2(got, ref)
    inc = rel_l2(got - u0, ref - u0)
    out = {"check": "c5a element 0, one step, GPU (conv_precision %d) vs C++ oracle fp64" % prec, "rel_l2": err,
           "rel_l2_increment": inc, "oracle_seconds": el, "oracle_threads": X.hardware_threads(), "tol": 2e-3}
    print(json.dumps(out))
    return out


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
