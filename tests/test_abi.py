"""CPU-side checks of the C-ABI library: it loads, exports every symbol the header
declares, sizes params/workspace like the generators, and validates arguments
before touching a device (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

from ldgen import param_count
from ldgen.configs import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2507_01975_b200 import build, ldsolver
    build.build()
    return ldsolver


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "ldsolver.h")).read()
    names = set(re.findall(r"\b(ld_[a-z_]+)\s*\(", hdr))
    assert "ld_init" in names and "ld_step" in names and "ld_rollout" in names
    lib = L.lib()
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert set(L.EXPORTS) >= names


@pytest.mark.parametrize("name", list(CONFIGS))
def test_param_count_matches_generator(L, name):
    cfg = CONFIGS[name].replace(dt=0.01)
    c = L.make_config(cfg)
    assert L.param_count(c) == param_count(cfg.n_layers, cfg.width, cfg.n_out)
    assert L.workspace_bytes(c) > 0


@pytest.mark.parametrize("field,value,status", [
    ("n", 48, "LD_ERR_UNSUPPORTED"), ("n", 4, "LD_ERR_INVALID_ARG"), ("dt", 0.0, "LD_ERR_INVALID_ARG"),
    ("rk_order", 5, "LD_ERR_INVALID_ARG"), ("batch", 0, "LD_ERR_INVALID_ARG"), ("width", 48, "LD_ERR_UNSUPPORTED"),
    ("tc_interval", 0, "LD_ERR_INVALID_ARG"), ("nu", -1.0, "LD_ERR_INVALID_ARG")])
def test_validation_before_device_work(L, field, value, status):
    cfg = CONFIGS["c2"].replace(dt=0.01)
    c = L.make_config(cfg, **{field: value})
    with pytest.raises(L.LDError, match=status):
        L.workspace_bytes(c)


def test_init_rejects_param_mismatch_and_has_no_cpu_fallback(L):
    cfg = CONFIGS["c1"].replace(dt=0.01)
    c = L.make_config(cfg)
    h = C.c_void_p()
    nb = L.workspace_bytes(c)
    st = L.lib().ld_init(C.byref(c), None, None, 0, None, 256, nb, C.byref(h))
    assert st == -1 and b"params" in L.lib().ld_last_error()
    import numpy as np
    p = np.zeros(L.param_count(c) + 1, np.float32)
    st = L.lib().ld_init(C.byref(c), None, p.ctypes.data, p.size, None, 256, nb, C.byref(h))
    assert st == -1 and b"n_params mismatch" in L.lib().ld_last_error()
    import torch
    if not torch.cuda.is_available():
        p = np.zeros(L.param_count(c), np.float32)
        st = L.lib().ld_init(C.byref(c), None, p.ctypes.data, p.size, None, 256, nb, C.byref(h))
        assert st == -2 and b"no CUDA device" in L.lib().ld_last_error()


def test_slab_mode_2_needs_a_communicator(L):
    cfg = CONFIGS["c2"].replace(dt=0.01, n=256, conv_precision=1)
    c = L.make_config(cfg)
    d = L.ld_dist(mode=2, rank=0, world=8, nccl_comm=None)
    with pytest.raises(L.LDError, match="INVALID_ARG"):
        L.workspace_bytes(c, d)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2507_01975_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"import\s+(\w+)|from\s+(\w+)", src).__str__(), f


# ---------------------------------------------------------------- slab decomposition (host logic)

@pytest.mark.parametrize("name,n,P", [("c3", 256, 2), ("c3", 512, 8), ("c1", 256, 4), ("c2", 1024, 8)])
def test_slab_geometry_covers_the_stencil_and_net_halos(L, name, n, P):
    cfg = CONFIGS[name].replace(dt=0.01, n=n, conv_precision=1)
    c = L.make_config(cfg)
    rows, m, hlo, hhi, nxt = L.slab_geometry(c, P)
    layers = cfg.n_layers
    assert rows == n // P and m == n // P
    assert hlo >= max(layers, 3) and hhi >= max(layers + 1, 3)      # net receptive field + 6-tap stencils
    assert nxt == rows + hlo + hhi and nxt % 8 == 0                   # tcgen05 strips are 8 rows
    assert hlo <= rows and hhi <= rows                                # halos come from one neighbour


@pytest.mark.parametrize("over,status", [
    (dict(n=256, conv_precision=0), "LD_ERR_UNSUPPORTED"),   # fp32-exact net not on the slab path
    (dict(n=128), "LD_ERR_UNSUPPORTED"),                     # NS distributed FFT needs n >= 256
    (dict(n=256), None)])
def test_slab_validation(L, over, status):
    cfg = CONFIGS["c3"].replace(dt=0.01, conv_precision=1).replace(**over)
    c = L.make_config(cfg)
    d = L.ld_dist(mode=3, rank=0, world=4, nccl_comm=None)
    if status is None:
        assert L.workspace_bytes(c, d) > L.workspace_bytes(c) // 4
    else:
        with pytest.raises(L.LDError, match=status):
            L.workspace_bytes(c, d)
    d2 = L.ld_dist(mode=2, rank=0, world=4, nccl_comm=None)   # mode 2 needs a communicator
    with pytest.raises(L.LDError):
        L.workspace_bytes(c, d2)


def test_spectral_counts_and_validation(L):
    """ld_spectral_*: parameter count matches the generator; shape checks before device work."""
    import numpy as np
    from ldgen.spectral import make_spectral_params
    for K, Lr, Cw in [(0, 1, 1), (3, 2, 4), (12, 2, 8)]:
        R, Q = make_spectral_params(K, Cw, Lr)
        blob = L.SpectralOp.pack(R, Q)
        assert L.lib().ld_spectral_param_count(K, Lr, Cw) == blob.size
    nb = C.c_size_t()
    assert L.lib().ld_spectral_workspace_bytes(64, 12, C.byref(nb)) == 0 and nb.value > 0
    for n, k in [(48, 4), (64, 32), (4, 1), (64, -1)]:
        assert L.lib().ld_spectral_workspace_bytes(n, k, C.byref(nb)) == -1
    h = C.c_void_p()
    p = np.zeros(10, np.float32)
    st = L.lib().ld_spectral_create(64, 3, 1, 2, p.ctypes.data_as(C.c_void_p), p.size, None, 0, C.byref(h))
    assert st == -1


def test_fno_config_counts_and_validation(L):
    """fno_* fields: the spectral blob is appended to the conv parameters; the branch is
    single-domain, learned-stencil only, 0 <= kmax < n/2; n > 128 takes the large-N (global-pass) form."""
    from ldgen.spectral import spectral_blob
    cfg = CONFIGS["c2"].replace(dt=0.01, fno_kmax=12, fno_layers=2, fno_width=8)
    c = L.make_config(cfg)
    assert L.param_count(c) == param_count(cfg.n_layers, cfg.width, cfg.n_out) + spectral_blob(12, 8, 2).size
    assert L.workspace_bytes(c) > L.workspace_bytes(L.make_config(cfg.replace(fno_layers=0)))
    for over, status in [({"fno_kmax": 32}, "LD_ERR_INVALID_ARG"), ({"fno_width": 0}, "LD_ERR_INVALID_ARG"),
                         ({"stencil_mode": 2, "tc_head": 0}, "LD_ERR_UNSUPPORTED"),
                         ({"stencil_mode": 1, "tc_head": 0}, "LD_ERR_INVALID_ARG"),
                         ({"fno_layers": -1}, "LD_ERR_INVALID_ARG")]:
        with pytest.raises(L.LDError, match=status):
            L.workspace_bytes(L.make_config(cfg.replace(**over)))
    big = L.workspace_bytes(L.make_config(cfg.replace(n=256)))       # large-N form: accepted, with scratch
    assert big > L.workspace_bytes(L.make_config(cfg.replace(n=256, fno_layers=0)))


def test_tc_history_config_counts_and_validation(L):
    from ldgen.spectral import spectral_blob
    cfg = CONFIGS["c3"].replace(dt=0.01, n=64, tc_head=0, tc_mode=1, tc_interval=4, tc_kmax=10, tc_layers=2,
                                tc_width=8)
    c = L.make_config(cfg)
    assert L.param_count(c) == param_count(cfg.n_layers, cfg.width, 24) + spectral_blob(10, 8, 2, n_in=8, n_out=2).size
    for over, status in [({"tc_head": 1}, "LD_ERR_INVALID_ARG"), ({"stencil_mode": 2}, "LD_ERR_UNSUPPORTED"),
                         ({"tc_layers": 0}, "LD_ERR_INVALID_ARG"), ({"tc_mode": 2}, "LD_ERR_INVALID_ARG")]:
        with pytest.raises(L.LDError, match=status):
            L.workspace_bytes(L.make_config(cfg.replace(**over)))
    assert L.workspace_bytes(L.make_config(cfg.replace(n=256))) > 0     # large-N form (global passes)


def test_size_limits_rejected_before_device_work(L):
    """NS projection up to n = 4096; the tcgen05 net's 32-bit operand offsets cap a handle at 2^28
    cells (batch * n^2); both are refused with LD_ERR_UNSUPPORTED instead of failing later."""
    cfg = CONFIGS["c5a"].replace(dt=0.01)
    with pytest.raises(L.LDError, match="LD_ERR_UNSUPPORTED"):
        L.workspace_bytes(L.make_config(cfg, n=8192, batch=1))
    with pytest.raises(L.LDError, match="LD_ERR_UNSUPPORTED"):
        L.workspace_bytes(L.make_config(cfg, n=4096, batch=17, conv_precision=1))
    assert L.workspace_bytes(L.make_config(cfg, n=4096, batch=16, conv_precision=1)) > 0
    assert L.workspace_bytes(L.make_config(cfg, n=8192, batch=1, system=0)) > 0   # Burgers: no projection
