"""GPU parity of the frequency-domain operator O_F (spectral.cu via ld_spectral_apply) against
the fp64 oracle (oracle/spectral_oracle.py; Eq. 8).

The kernel evaluates truncated DFT sums in fp32 with the layers composed per mode on the host
(fp64, rounded once); the oracle runs numpy FFTs layer by layer in fp64.  Bound: relative L2
<= 1e-5 (fp32 sums of N terms, twice each way), per batch element and channel group."""
import numpy as np
import pytest

import oracle as O
from ldgen.spectral import make_spectral_params

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _run(n, K, Lr, Cw, B, seed=0):
    import torch
    from paper_2507_01975_b200 import ldsolver as L
    R, Q = make_spectral_params(K, Cw, Lr, seed=seed)
    op = L.SpectralOp(n, K, Lr, Cw, L.SpectralOp.pack(R, Q))
    u = np.random.default_rng(seed + 11).standard_normal((B, 2, n, n)).astype(np.float32)
    ud = torch.from_numpy(u).cuda()
    out = torch.full((B, 8, n, n), float("nan"), device="cuda")
    op.apply(ud, out)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), O.spectral_operator(u, R, Q, K), op, ud


@pytest.mark.parametrize("n,K,Lr,Cw,B", [
    (64, 12, 2, 8, 3),      # the SPEC default shape (k_max 12 on 64^2, width 8, two layers)
    (32, 5, 1, 4, 2),
    (16, 0, 1, 1, 1),       # only the mean mode
    (16, 7, 3, 3, 2),       # K = N/2 - 1: every mode but the Nyquist lines
    (128, 12, 2, 6, 2),
    (8, 3, 1, 2, 5),
    (64, 12, 2, 8, 64),     # 4 output channels per CTA
    (32, 6, 1, 3, 300),     # 8 output channels per CTA
])
def test_spectral_parity(n, K, Lr, Cw, B):
    got, ref, _, _ = _run(n, K, Lr, Cw, B)
    assert np.all(np.isfinite(got))
    for b in range(B):
        err = np.linalg.norm(got[b] - ref[b]) / max(np.linalg.norm(ref[b]), 1e-300)
        assert err < TOL, (b, err)


def test_spectral_batch_elements_independent_and_deterministic():
    import torch
    got, _, op, ud = _run(32, 6, 2, 5, 4, seed=2)
    perm = [2, 0, 3, 1]
    out2 = torch.empty((4, 8, 32, 32), device="cuda")
    op.apply(ud[perm].contiguous(), out2)
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy(), got[perm].astype(np.float32))
