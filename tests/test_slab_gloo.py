"""World-size-2 (and 4) gloo model of the slab decomposition on CPU.

Each process owns rows [r n, (r+1) n) of every field and runs the decomposed step in fp64 with
the oracle's own pieces (oracle.net_forward / constrain / tendency for the local arithmetic),
exchanging data with real point-to-point messages: the stage-field halo (Hlo rows from rank r-1,
Hhi rows from rank r+1, the geometry taken from libldsolver's host-only ld_slab_geometry), the
1-row v and p halos of the projection and the two block transposes of the distributed FFT.
The gathered result must equal the oracle's single-domain step -- so the halo depths, the
extended-slab ("periodic in the slab, edges discarded") net, the own-row flux and the
rows / transpose / columns / transpose / rows FFT decomposition that the CUDA slab modes
implement are checked with real multi-process exchanges.  (The CUDA kernels themselves are
checked against single-domain runs on the GPU: tests/test_gpu_slab.py.)"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from ldgen import make_weights
from ldgen.configs import get_config
from ldgen.ic import make_config_ic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _xchg(sends, recvs):
    """sends / recvs: lists of (peer, tag, ndarray).  Returns the received arrays."""
    reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(a)), peer, tag=tag) for peer, tag, a in sends]
    out = []
    for peer, tag, shape in recvs:
        t = torch.empty(shape, dtype=torch.float64)
        dist.recv(t, peer, tag=tag)
        out.append(t.numpy())
    for r in reqs:
        r.wait()
    return out


def _slab_stage_T(X_own, cfg, layers, geo, r, P, h):
    """Tendency of the own rows (+ the TC term of the own rows) via the extended slab."""
    n, m, hlo, hhi, nxt = geo
    lo, hi = _xchg([((r - 1) % P, 0, X_own[:, :, :hhi]), ((r + 1) % P, 1, X_own[:, :, n - hlo:])],
                   [((r + 1) % P, 0, X_own[:, :, :hhi].shape), ((r - 1) % P, 1, X_own[:, :, n - hlo:].shape)])
    Uext = np.concatenate([hi, X_own, lo], axis=2)        # rows: Hlo from r-1, own, Hhi from r+1
    assert Uext.shape[2] == nxt
    R = O.net_forward(Uext, layers, cfg.activation)       # periodic on the slab: edge rows discarded
    w = O.constrain(R)
    unforced = cfg.replace(force_amp=0.0, drag=0.0)
    T = O.tendency(Uext, w, unforced, h)[:, :, hlo:hlo + n]
    if cfg.force_amp or cfg.drag:
        y = (np.arange(r * n, (r + 1) * n) + 0.5) * h
        T[:, 0] += cfg.force_amp * np.sin(cfg.force_k * y)[:, None] - cfg.drag * X_own[:, 0]
        T[:, 1] += -cfg.drag * X_own[:, 1]
    e = np.moveaxis(R[..., 24:26], -1, 1)[:, :, hlo:hlo + n] if cfg.tc_head else None
    return T, e


def _slab_project(U_own, geo, r, P, N, h):
    n, m = geo[0], geo[1]
    B = U_own.shape[0]
    vb, va = _xchg([((r - 1) % P, 2, U_own[:, 1, 0]), ((r + 1) % P, 3, U_own[:, 1, n - 1])],
                   [((r - 1) % P, 3, (B, N)), ((r + 1) % P, 2, (B, N))])
    u, v = U_own[:, 0], U_own[:, 1]
    vup = np.concatenate([v[:, 1:], va[:, None]], axis=1)
    vdn = np.concatenate([vb[:, None], v[:, :-1]], axis=1)
    d = ((np.roll(u, -1, -1) - np.roll(u, 1, -1)) + (vup - vdn)) / (2 * h)
    D = np.fft.fft(d, axis=-1)                                            # rows (own y), all kx
    blocks = [np.ascontiguousarray(D[:, :, q * m:(q + 1) * m]) for q in range(P)]
    recv = [blocks[r]] + _xchg([(q, 10, np.stack([blocks[q].real, blocks[q].imag])) for q in range(P) if q != r],
                               [(q, 10, (2, B, n, m)) for q in range(P) if q != r])
    recv = [recv[0]] + [a[0] + 1j * a[1] for a in recv[1:]]
    order = [r] + [q for q in range(P) if q != r]
    cols = np.concatenate([recv[order.index(q)] for q in range(P)], axis=1)   # [B][N (all y)][m]
    kh = O.symbol(N, h)
    Dh = np.fft.fft(cols, axis=1)
    kx = np.arange(r * m, (r + 1) * m)
    den = kh[None, :, None] ** 2 + kh[kx][None, None, :] ** 2
    null = np.zeros_like(den, dtype=bool)
    for a in (0, N // 2):
        for c in (0, N // 2):
            if r * m <= c < (r + 1) * m:
                null[:, a, c - r * m] = True
    ph = np.where(null, 0.0, -Dh / np.where(null, 1.0, den))
    pc = np.fft.ifft(ph, axis=1)                                          # back to y, my kx block
    back = [pc[:, q * n:(q + 1) * n] for q in range(P)]
    got = [back[r]] + _xchg([(q, 11, np.stack([back[q].real, back[q].imag])) for q in range(P) if q != r],
                            [(q, 11, (2, B, n, m)) for q in range(P) if q != r])
    got = [got[0]] + [a[0] + 1j * a[1] for a in got[1:]]
    rows = np.concatenate([got[order.index(q)] for q in range(P)], axis=-1)   # [B][n][N] all kx
    p = np.real(np.fft.ifft(rows, axis=-1))
    pb, pa = _xchg([((r - 1) % P, 4, p[:, 0]), ((r + 1) % P, 5, p[:, n - 1])],
                   [((r - 1) % P, 5, (B, N)), ((r + 1) % P, 4, (B, N))])
    pup = np.concatenate([p[:, 1:], pa[:, None]], axis=1)
    pdn = np.concatenate([pb[:, None], p[:, :-1]], axis=1)
    out = U_own.copy()
    out[:, 0] -= (np.roll(p, -1, -1) - np.roll(p, 1, -1)) / (2 * h)
    out[:, 1] -= (pup - pdn) / (2 * h)
    return out


def _worker(rank, world, port, name, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01975_b200 import ldsolver as L
    cfg = get_config(name, n=n, batch=2, conv_precision=1)
    u0 = make_config_ic(cfg)
    cfg = cfg.with_dt(u0)
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="stress")
    geo = L.slab_geometry(L.make_config(cfg), world)
    nrow = geo[0]
    layers = O.unpack_params(params, cfg.n_layers, cfg.width, cfg.n_out)
    h = cfg.length / n
    un = u0[:, :, rank * nrow:(rank + 1) * nrow].astype(np.float64)
    # SSP-RK3 with per-stage projection and the TC term at the last stage (oracle §8c(c1) step 8)
    T1, e = _slab_stage_T(un, cfg, layers, geo, rank, world, h)
    U1 = _slab_project(un + cfg.dt * T1, geo, rank, world, n, h)
    T2, _ = _slab_stage_T(U1, cfg, layers, geo, rank, world, h)
    U2 = _slab_project(0.75 * un + 0.25 * (U1 + cfg.dt * T2), geo, rank, world, n, h)
    T3, _ = _slab_stage_T(U2, cfg, layers, geo, rank, world, h)
    pre = un / 3 + 2.0 / 3 * (U2 + cfg.dt * T3) + (e if cfg.tc_head else 0.0)
    U3 = _slab_project(pre, geo, rank, world, n, h)
    parts = [torch.empty_like(torch.from_numpy(U3)) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(U3)))
    if rank == 0:
        full = np.concatenate([p.numpy() for p in parts], axis=2)
        ref = O.step(u0, cfg, params)
        out.put(float(np.linalg.norm(full - ref) / np.linalg.norm(ref)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,name,n", [(2, "c3", 64), (4, "c3", 64)])
def test_slab_decomposition_gloo_matches_oracle(world, name, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    err, t0 = None, time.time()
    while err is None and time.time() - t0 < 500:
        try:
            err = q.get(timeout=2)
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert err is not None and err < 1e-12, err
