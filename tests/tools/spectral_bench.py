"""Time ld_spectral_apply (NEXT-2 operator O_F) at a given shape with CUDA events.

python tests/tools/spectral_bench.py [--n 64 --batch 32 --k 12 --layers 2 --width 8 --reps 200]
Prints one JSON line: us per apply, algorithmic FLOP (truncated-DFT form, no recomputation),
achieved TFLOP/s against the FP32 ALU peak (148 SM x 128 lanes x 2 x sm_max_mhz)."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--k", type=int, default=12)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--width", type=int, default=8)
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    import torch
    from ldgen.spectral import make_spectral_params, n_modes
    from paper_2507_01975_b200 import ldsolver as L
    R, Q = make_spectral_params(a.k, a.width, a.layers)
    op = L.SpectralOp(a.n, a.k, a.layers, a.width, L.SpectralOp.pack(R, Q))
    u = torch.randn(a.batch, 2, a.n, a.n, device="cuda")
    out = torch.empty(a.batch, 8, a.n, a.n, device="cuda")
    for _ in range(10):
        op.apply(u, out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        op.apply(u, out)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / a.reps
    N, K = a.n, a.k
    KX, KY = K + 1, 2 * K + 1
    fma = 4 * N * N * KX + 8 * N * KX * KY + 64 * n_modes(K) + 32 * N * KX * KY + 16 * N * N * K
    flop = 2.0 * fma * a.batch
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "..", "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    ach = flop / (us * 1e-6) / 1e12
    print(json.dumps({"op": "ld_spectral_apply", "n": N, "batch": a.batch, "k_max": K, "layers": a.layers,
                      "width": a.width, "us_per_apply": us, "algorithmic_flop": flop,
                      "roofline": {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                                   "frac": ach / peak},
                      "bytes": 4.0 * a.batch * N * N * (2 + 8)}))


if __name__ == "__main__":
    main()
