"""B200 version of the paper's Table 4 comparison, SURVEY.md §8f NEXT-1:
fine-grid DNS (the physics-only solver: stencil_mode FIXED) vs the LDSolver coarse step,
both through the public API, as GPU seconds per simulated physical second; plus the cost of the
block-mean downsampling that turns DNS fields into coarse training data (ld_downsample).
Context only: the paper's numbers are an A100 running RK4 + FNO branches.

python tests/tools/dns_table.py [--steps K] > profiles/...json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from ldgen import make_weights  # noqa: E402
from ldgen.configs import get_config  # noqa: E402
from ldgen.ic import make_config_ic  # noqa: E402
from paper_2507_01975_b200 import ldsolver as L  # noqa: E402

PAPER_A100 = {  # PAPER.md P:517-518, seconds of GPU time per physical second
    "decaying": {"dns": 29.2402, "ldsolver": 2.3773, "dns_grid": "1024^2", "coarse_grid": "64^2"},
    "forced": {"dns": 32.8061, "ldsolver": 3.8036, "dns_grid": "1024^2", "coarse_grid": "64^2"},
}


def time_steps(solver, u, steps, warmup=3):
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        solver.ld_step(u, st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        solver.ld_step(u, st)
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps   # ms per step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    out = {"what": "GPU seconds per physical second (lower is better), one B200, fp32 / TF32 conv", "rows": []}
    for name, cname in (("decaying", "c2"), ("forced", "c3")):
        for batch in (1, 32):
            # fine-grid DNS: fixed 2nd-order central stencils, 1024^2, RK3 + projection
            dns_cfg = get_config(cname, n=1024, batch=batch, stencil_mode=1, tc_head=0)
            u0 = make_config_ic(dns_cfg)
            dns_cfg = dns_cfg.with_dt(u0)
            dns = L.Solver(L.make_config(dns_cfg), None)
            ud = torch.from_numpy(u0.astype(np.float32)).cuda()
            ms_dns = time_steps(dns, ud, a.steps)
            coarse = torch.empty((batch, 2, 64, 64), device="cuda")
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            L.ld_downsample(ud, 16, coarse)
            ev1.record()
            torch.cuda.synchronize()
            ms_ds = ev0.elapsed_time(ev1)
            del dns, ud
            # LDSolver coarse step: the config's net on 64^2
            cfg = get_config(cname, n=64, batch=batch, conv_precision=1)
            uc = make_config_ic(cfg)
            cfg = cfg.with_dt(uc)
            params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="normal")
            lds = L.Solver(L.make_config(cfg), params)
            u = torch.from_numpy(uc.astype(np.float32)).cuda()
            ms_ld = time_steps(lds, u, a.steps)
            row = {"flow": name, "batch": batch,
                   "dns": {"grid": "1024^2", "dt": dns_cfg.dt, "ms_per_step": ms_dns,
                           "s_per_physical_s_per_traj": ms_dns / 1e3 / dns_cfg.dt / batch,
                           "cell_updates_per_s": batch * 1024 * 1024 / (ms_dns / 1e3)},
                   "ldsolver": {"grid": "64^2", "dt": cfg.dt, "ms_per_step": ms_ld,
                                "s_per_physical_s_per_traj": ms_ld / 1e3 / cfg.dt / batch,
                                "cell_updates_per_s": batch * 64 * 64 / (ms_ld / 1e3)},
                   "downsample_1024_to_64_ms": ms_ds,
                   "paper_a100": PAPER_A100[name]}
            row["speedup_ldsolver_vs_dns"] = (row["dns"]["s_per_physical_s_per_traj"] /
                                              row["ldsolver"]["s_per_physical_s_per_traj"])
            out["rows"].append(row)
            print(f"{name:9s} B={batch:3d}  DNS 1024^2 {row['dns']['s_per_physical_s_per_traj']:.4f} s/s  "
                  f"LDSolver 64^2 {row['ldsolver']['s_per_physical_s_per_traj']:.5f} s/s  "
                  f"speed-up {row['speedup_ldsolver_vs_dns']:.1f}x  (paper A100: "
                  f"{PAPER_A100[name]['dns'] / PAPER_A100[name]['ldsolver']:.1f}x)", file=sys.stderr)
            del lds, u
    print(json.dumps(out))


if __name__ == "__main__":
    main()
