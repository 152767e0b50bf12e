"""The measurement knobs that switch a kernel form are bitwise neutral (round 2, session 5).

Each case runs the same seeded problem in two fresh processes -- once with the default kernels, once with
an environment knob selecting the older form (the knobs are read once per process) -- and compares the
outputs bit for bit:

* LD_PROJ_UNFUSED=1: the inverse row pass and the correction as two kernels (p through HBM) instead of
  the fused pen_inv_correct_r2 (p on chip) -- projection (Eq.13-15) and a full c4-shape step;
* LD_PEN_COLS_OLD=1: the column pass with per-row 8-B stores instead of the staged, coalesced form;
* LD_PEN4_CC2=1: the four-step column pass with 2 instead of 4 columns per CTA (N = 2048);
* LD_HOST_SEQUENTIAL=1: ld_rollout_host's batch chunks chained instead of interleaved on their streams;
* LD_XN_GATHER_Y=1: the TF32 first layer's 4-byte operand gather with one row per lane (32 rows per warp
  instruction) instead of the x-fastest item order (the same values land in the same stage slots);
* LD_XN_NO_CT_OUT=1: the output layer (flux epilogue) with 16 ten-row strips per operand stage instead of the
  contiguous 130-row column form (the same MMAs on the same operands).

The arithmetic is the same operations in the same order in both forms, so any difference is a bug.  (At
N = 256 the projection runs the half-warp FFT passes by default; the projection knobs are compared on the
32-lane shuffle-FFT passes, LD_PEN_WARPFFT=1, and the two FFT forms against each other to rounding.)
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from ldgen.configs import get_config
from tests.helpers import setup, gpu_solver, to_dev
what, n, B, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
cfg = get_config("c4", n=n, batch=B, conv_precision=1)
cfg, u0, params = setup(cfg, init="stress", elements=range(B))
s = gpu_solver(cfg, params)
u = to_dev(u0)
if what == "project":
    o = torch.empty_like(u)
    s.ld_project(u, o)
    res = o
elif what == "step":
    s.ld_rollout(u, 2)
    res = u
else:  # host rollout (pinned host buffer, pipelined chunks)
    h = torch.from_numpy(np.ascontiguousarray(u0, dtype=np.float32)).pin_memory()
    s.ld_rollout_host(h, 2)
    res = h
torch.cuda.synchronize()
np.save(out, res.cpu().numpy())
'''


def _run(tmp_path, what, n, B, env_extra, tag):
    path = tmp_path / f"{what}_{tag}.npy"
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), what, str(n), str(B), str(path)],
                       env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


W = {"LD_PEN_WARPFFT": "1"}   # N = 256 on the 32-lane shuffle-FFT passes (the knobs below select among those)


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("what,n,B,knob,base", [
    ("project", 256, 3, "LD_PROJ_UNFUSED", W),
    ("project", 128, 2, "LD_PROJ_UNFUSED", {}),
    ("project", 1024, 1, "LD_PROJ_UNFUSED", {}),
    ("step", 256, 2, "LD_PROJ_UNFUSED", W),
    ("project", 256, 3, "LD_PEN_COLS_OLD", W),
    ("project", 512, 1, "LD_PEN_COLS_OLD", {}),
    ("project", 2048, 1, "LD_PEN4_CC2", {}),
    ("host", 256, 32, "LD_HOST_SEQUENTIAL", {}),
    ("step", 256, 4, "LD_XN_GATHER_Y", {}),
    ("step", 256, 2, "LD_XN_NO_CT_OUT", {}),
])
def test_knob_bitwise(tmp_path, what, n, B, knob, base):
    a = _run(tmp_path, what, n, B, dict(base), "default")
    b = _run(tmp_path, what, n, B, {**base, knob: "1"}, "knob")
    assert np.isfinite(a).all()
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), float(np.abs(a - b).max())


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("what,B", [("project", 3), ("step", 2)])
def test_n256_halfwarp_fft_matches_warp_fft(tmp_path, what, B):
    """The N = 256 half-warp FFT passes (16 x 16 four-step, fft256.cuh) against the 32-lane shuffle-FFT
    passes: a different summation order, so agreement to fp32 rounding of the transform, not bitwise."""
    a = _run(tmp_path, what, 256, B, {}, "halfwarp")
    b = _run(tmp_path, what, 256, B, dict(W), "warp")
    assert np.isfinite(a).all()
    err = float(np.linalg.norm((a - b).astype(np.float64)) / np.linalg.norm(b.astype(np.float64)))
    assert err < 1e-5, err


@pytest.mark.timeout(1200)
def test_n4096_halfwarp_passes_match_shuffle_form(tmp_path):
    """The N = 4096 row and column passes on half-warp FFTs (16 x 256 four-step) against the 64 x 64 shuffle-FFT block
    transform (LD_PEN4_OLD=1): agreement to fp32 rounding of the transforms."""
    a = _run(tmp_path, "project", 4096, 1, {}, "halfwarp")
    b = _run(tmp_path, "project", 4096, 1, {"LD_PEN4_OLD": "1"}, "old")
    assert np.isfinite(a).all()
    err = float(np.linalg.norm((a - b).astype(np.float64)) / np.linalg.norm(b.astype(np.float64)))
    assert err < 1e-5, err
