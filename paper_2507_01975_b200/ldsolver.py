"""Thin ctypes binding of include/ldsolver.h (argument marshalling only).

Every step of the path runs in libldsolver.so's CUDA kernels; this module only
converts Python/torch objects into the C ABI's plain pointers and sizes.  There
is no CPU fallback: if the library or a CUDA device is missing, calls raise.
PyTorch is used for device memory (the workspace and fields) and streams.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# LDSOLVER_LIB: another build of the same library (A/B measurement of kernel variants)
LIB_PATH = os.environ.get("LDSOLVER_LIB") or os.path.join(HERE, "libldsolver.so")

LD_OK = 0
STATUS_NAMES = {0: "LD_OK", -1: "LD_ERR_INVALID_ARG", -2: "LD_ERR_CUDA", -3: "LD_ERR_NCCL",
                -4: "LD_ERR_OOM", -5: "LD_ERR_NONFINITE", -6: "LD_ERR_UNSUPPORTED"}


class ld_config(C.Structure):
    _fields_ = [("n", C.c_int32), ("batch", C.c_int32), ("length", C.c_double), ("system", C.c_int32),
                ("nu", C.c_double), ("dt", C.c_double), ("rk_order", C.c_int32),
                ("force_amp", C.c_double), ("force_k", C.c_double), ("drag", C.c_double),
                ("n_layers", C.c_int32), ("width", C.c_int32), ("activation", C.c_int32),
                ("tc_head", C.c_int32), ("tc_interval", C.c_int32), ("stencil_mode", C.c_int32),
                ("conv_precision", C.c_int32), ("check_finite_every", C.c_int32),
                ("fno_kmax", C.c_int32), ("fno_layers", C.c_int32), ("fno_width", C.c_int32),
                ("tc_mode", C.c_int32), ("tc_kmax", C.c_int32), ("tc_layers", C.c_int32), ("tc_width", C.c_int32),
                ("freeze_stencils", C.c_int32), ("scalar_mode", C.c_int32), ("scalar_diff", C.c_double)]


class ld_dist(C.Structure):
    _fields_ = [("mode", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("nccl_comm", C.c_void_p)]


class LDError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None

EXPORTS = {
    "ld_param_count": (C.c_size_t, [C.POINTER(ld_config)]),
    "ld_workspace_bytes": (C.c_int, [C.POINTER(ld_config), C.POINTER(ld_dist), C.POINTER(C.c_size_t)]),
    "ld_init": (C.c_int, [C.POINTER(ld_config), C.POINTER(ld_dist), C.c_void_p, C.c_size_t, C.c_void_p,
                          C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "ld_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ld_rollout": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "ld_rollout_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "ld_step_scalar": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ld_rollout_scalar": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "ld_eval_net": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ld_eval_stencils": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ld_eval_tendency": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ld_project": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ld_set_graph_replay": (C.c_int, [C.c_void_p, C.c_int32]),
    "ld_set_kernel_timing": (C.c_int, [C.c_void_p, C.c_int32]),
    "ld_kernel_times": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32]),
    "ld_get_step_index": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "ld_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "ld_nccl_comm_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "ld_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
    "ld_slab_geometry": (C.c_int, [C.POINTER(ld_config), C.c_int32, C.POINTER(C.c_int32)]),
    "ld_downsample": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "ld_reset_step_counter": (C.c_int, [C.c_void_p]),
    "ld_launches_per_step": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "ld_destroy": (C.c_int, [C.c_void_p]),
    "ld_spectral_param_count": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
    "ld_spectral_workspace_bytes": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]),
    "ld_spectral_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t,
                                     C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "ld_spectral_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "ld_spectral_destroy": (C.c_int, [C.c_void_p]),
    "ld_vjp_workspace_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "ld_step_vjp": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                              C.c_void_p]),
    "ld_rollout_vjp": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_size_t, C.c_void_p]),
    "ld_last_error": (C.c_char_p, []),
    "ld_version": (C.c_char_p, []),
}


def lib():
    """Load libldsolver.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != LD_OK:
        raise LDError(status, lib().ld_last_error().decode())


def make_config(cfg, **overrides) -> ld_config:
    """Build an ld_config from an ldgen.LDConfig-like object (attribute names match)."""
    c = ld_config()
    src = dict(n=cfg.n, batch=cfg.batch, length=cfg.length, system=cfg.system, nu=cfg.nu, dt=cfg.dt,
               rk_order=cfg.rk_order, force_amp=cfg.force_amp, force_k=cfg.force_k, drag=cfg.drag,
               n_layers=cfg.n_layers, width=cfg.width, activation=cfg.activation, tc_head=cfg.tc_head,
               tc_interval=cfg.tc_interval, stencil_mode=cfg.stencil_mode,
               conv_precision=cfg.conv_precision, check_finite_every=0,
               fno_kmax=getattr(cfg, "fno_kmax", 0), fno_layers=getattr(cfg, "fno_layers", 0),
               fno_width=getattr(cfg, "fno_width", 0), tc_mode=getattr(cfg, "tc_mode", 0),
               tc_kmax=getattr(cfg, "tc_kmax", 0), tc_layers=getattr(cfg, "tc_layers", 0),
               tc_width=getattr(cfg, "tc_width", 0), freeze_stencils=getattr(cfg, "freeze_stencils", 0),
               scalar_mode=getattr(cfg, "scalar_mode", 0), scalar_diff=getattr(cfg, "scalar_diff", 0.0))
    src.update(overrides)
    for k, v in src.items():
        setattr(c, k, v)
    return c


def param_count(c: ld_config) -> int:
    return int(lib().ld_param_count(C.byref(c)))


def workspace_bytes(c: ld_config, dist: Optional[ld_dist] = None) -> int:
    out = C.c_size_t()
    _check(lib().ld_workspace_bytes(C.byref(c), C.byref(dist) if dist else None, C.byref(out)))
    return out.value


def slab_geometry(c: ld_config, world: int):
    """(n, m, Hlo, Hhi, next) of the slab decomposition over `world` ranks (host-only)."""
    out = (C.c_int32 * 5)()
    _check(lib().ld_slab_geometry(C.byref(c), int(world), out))
    return tuple(int(v) for v in out)


def ld_downsample(fine, factor: int, coarse, stream=None):
    """coarse [B][2][n/f][n/f] = f x f block means of fine [B][2][n][n] (device tensors)."""
    B, _, n, _ = fine.shape
    _check(lib().ld_downsample(_ptr(fine), int(n), int(B), int(factor), _ptr(coarse), _stream(stream)))


class SpectralOp:
    """Frequency-domain operator O_F (include/ldsolver.h ld_spectral_*): marshalling only."""

    def __init__(self, n: int, k_max: int, layers: int, width: int, params, device=None):
        import numpy as np
        import torch
        self.n, self.k_max = int(n), int(k_max)
        blob = np.ascontiguousarray(params, dtype=np.float32).ravel()
        need = int(lib().ld_spectral_param_count(self.k_max, int(layers), int(width)))
        if blob.size != need:
            raise LDError(-1, f"spectral params: got {blob.size}, need {need}")
        nb = C.c_size_t()
        _check(lib().ld_spectral_workspace_bytes(self.n, self.k_max, C.byref(nb)))
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.workspace = torch.empty(nb.value + 256, dtype=torch.uint8, device=self.device)
        h = C.c_void_p()
        _check(lib().ld_spectral_create(self.n, self.k_max, int(layers), int(width),
                                        blob.ctypes.data_as(C.c_void_p), blob.size, _ptr(self.workspace),
                                        nb.value, C.byref(h)))
        self.handle = h

    @staticmethod
    def pack(R, Q):
        """Flat blob from ldgen.spectral.make_spectral_params output (R list, Q)."""
        import numpy as np
        return np.concatenate([np.asarray(r, dtype=np.float32).ravel() for r in R] +
                              [np.asarray(Q, dtype=np.float32).ravel()])

    def apply(self, u, out, stream=None):
        _check(lib().ld_spectral_apply(self.handle, _ptr(u), int(u.shape[0]), _ptr(out), _stream(stream)))

    def close(self):
        if getattr(self, "handle", None):
            lib().ld_spectral_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().ld_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm_init(uid: bytes, world: int, rank: int) -> int:
    """NCCL communicator for slab mode 2 on the current CUDA device (collective)."""
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    comm = C.c_void_p()
    _check(lib().ld_nccl_comm_init(buf, int(world), int(rank), C.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm: int):
    _check(lib().ld_nccl_comm_destroy(C.c_void_p(comm)))


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def _stream(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Solver:
    """One ld_handle plus its torch-owned device workspace."""

    def __init__(self, c: ld_config, params: Optional[np.ndarray] = None, base_stencils=None,
                 dist: Optional[ld_dist] = None, device=None):
        import torch
        self.cfg = c
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        nbytes = workspace_bytes(c, dist)
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base_ptr = self.workspace.data_ptr()
        aligned = (base_ptr + 255) & ~255
        p = None if params is None else np.ascontiguousarray(params, dtype=np.float32)
        b = None if base_stencils is None else np.ascontiguousarray(base_stencils, dtype=np.float64).ravel()
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib().ld_init(C.byref(c), C.byref(dist) if dist else None,
                                 None if p is None else p.ctypes.data, 0 if p is None else p.size,
                                 None if b is None else b.ctypes.data, aligned, nbytes, C.byref(h)))
        self.handle = h
        self.dist = dist

    # -- argument checks (the C ABI takes raw pointers: reject what would be read as garbage) --
    def _rows(self) -> int:
        d = self.dist
        return self.cfg.n // d.world if (d is not None and d.mode == 2) else self.cfg.n

    def _check_field(self, t, channels: int = 2, what: str = "field", host: bool = False):
        """t must be a contiguous float32 tensor [B][channels][rows][N] on this solver's device
        (host memory for the host entry point)."""
        import torch
        if not isinstance(t, torch.Tensor):
            raise LDError(-1, f"{what}: expected a torch.Tensor")
        if t.dtype != torch.float32:
            raise LDError(-1, f"{what}: dtype {t.dtype}, need torch.float32")
        if not t.is_contiguous():
            raise LDError(-1, f"{what}: must be contiguous")
        if host:
            if t.is_cuda:
                raise LDError(-1, f"{what}: the host entry point needs a host (ideally pinned) tensor")
        elif not t.is_cuda or t.device != self.device:
            raise LDError(-1, f"{what}: must live on {self.device}, got {t.device}")
        want = (self.cfg.batch, channels, self._rows(), self.cfg.n)
        if tuple(t.shape) != want:
            raise LDError(-1, f"{what}: shape {tuple(t.shape)}, need {want}")

    # -- API mirrors the C names ------------------------------------------------
    def ld_step(self, u, stream=None):
        self._check_field(u, what="u")
        _check(lib().ld_step(self.handle, _ptr(u), _stream(stream)))

    def ld_rollout(self, u, n_steps: int, traj=None, save_every: int = 0, stream=None):
        self._check_field(u, what="u")
        if traj is not None:
            import torch
            nsnap = int(n_steps) // max(int(save_every), 1)
            if (traj.dtype != torch.float32 or not traj.is_contiguous() or traj.device != self.device
                    or traj.numel() < nsnap * u.numel()):
                raise LDError(-1, f"traj: need a contiguous float32 tensor on {self.device} with >= "
                                  f"{nsnap} snapshots of {tuple(u.shape)}")
        _check(lib().ld_rollout(self.handle, _ptr(u), int(n_steps), _ptr(traj), int(save_every), _stream(stream)))

    def _check_scalar(self, s):
        import torch
        want = (self.cfg.batch, self._rows(), self.cfg.n)
        if (not isinstance(s, torch.Tensor) or s.dtype != torch.float32 or not s.is_contiguous()
                or s.device != self.device or tuple(s.shape) != want):
            raise LDError(-1, f"s: need a contiguous float32 tensor {want} on {self.device}")

    def ld_step_scalar(self, u, s, stream=None):
        self._check_field(u, what="u")
        self._check_scalar(s)
        _check(lib().ld_step_scalar(self.handle, _ptr(u), _ptr(s), _stream(stream)))

    def ld_rollout_scalar(self, u, s, n_steps: int, stream=None):
        self._check_field(u, what="u")
        self._check_scalar(s)
        _check(lib().ld_rollout_scalar(self.handle, _ptr(u), _ptr(s), int(n_steps), _stream(stream)))

    def ld_rollout_host(self, u_host, n_steps: int, stream=None):
        self._check_field(u_host, what="u_host", host=True)
        _check(lib().ld_rollout_host(self.handle, u_host.data_ptr(), int(n_steps), _stream(stream)))

    def ld_eval_net(self, U, R, stream=None):
        self._check_field(U, what="U")
        self._check_field(R, channels=24 + (2 if self.cfg.tc_head else 0), what="R")
        _check(lib().ld_eval_net(self.handle, _ptr(U), _ptr(R), _stream(stream)))

    def ld_eval_stencils(self, U, w, stream=None):
        self._check_field(U, what="U")
        self._check_field(w, channels=24, what="w")
        _check(lib().ld_eval_stencils(self.handle, _ptr(U), _ptr(w), _stream(stream)))

    def ld_eval_tendency(self, U, T, stream=None):
        self._check_field(U, what="U")
        self._check_field(T, what="T")
        _check(lib().ld_eval_tendency(self.handle, _ptr(U), _ptr(T), _stream(stream)))

    def ld_project(self, inp, out, stream=None):
        self._check_field(inp, what="in")
        self._check_field(out, what="out")
        _check(lib().ld_project(self.handle, _ptr(inp), _ptr(out), _stream(stream)))

    def ld_step_vjp(self, u, gout, gin, gparams=None, stream=None):
        """gin = (d step / d u)^T gout; gparams += (d step / d theta)^T gout (NEXT-4).  The VJP scratch
        workspace is allocated once (torch) and reused."""
        import torch
        for t, nm in ((u, "u"), (gout, "gout"), (gin, "gin")):
            self._check_field(t, what=nm)
        if gparams is not None and (gparams.dtype != torch.float32 or not gparams.is_contiguous()
                                    or gparams.device != self.device or gparams.numel() != param_count(self.cfg)):
            raise LDError(-1, f"gparams: need a contiguous float32 tensor of {param_count(self.cfg)} on {self.device}")
        if getattr(self, "_vjp_ws", None) is None:
            nb = C.c_size_t()
            _check(lib().ld_vjp_workspace_bytes(self.handle, C.byref(nb)))
            self._vjp_ws = torch.empty(nb.value + 256, dtype=torch.uint8, device=self.device)
            self._vjp_bytes = nb.value
        base = (self._vjp_ws.data_ptr() + 255) & ~255
        _check(lib().ld_step_vjp(self.handle, _ptr(u), _ptr(gout), _ptr(gin), _ptr(gparams), base, self._vjp_bytes,
                                 _stream(stream)))

    def ld_rollout_vjp(self, u0, n_steps: int, gout, gin, gparams=None, stream=None):
        """gin = (d u^n / d u^0)^T gout through an n-step rollout; gparams += its parameter cotangent."""
        import torch
        for t, nm in ((u0, "u0"), (gout, "gout"), (gin, "gin")):
            self._check_field(t, what=nm)
        if gparams is not None and (gparams.dtype != torch.float32 or not gparams.is_contiguous()
                                    or gparams.device != self.device or gparams.numel() != param_count(self.cfg)):
            raise LDError(-1, f"gparams: need a contiguous float32 tensor of {param_count(self.cfg)} on {self.device}")
        if getattr(self, "_vjp_ws", None) is None:
            nb = C.c_size_t()
            _check(lib().ld_vjp_workspace_bytes(self.handle, C.byref(nb)))
            self._vjp_ws = torch.empty(nb.value + 256, dtype=torch.uint8, device=self.device)
            self._vjp_bytes = nb.value
        traj = torch.empty((max(int(n_steps), 1),) + tuple(u0.shape), dtype=torch.float32, device=self.device)
        base = (self._vjp_ws.data_ptr() + 255) & ~255
        _check(lib().ld_rollout_vjp(self.handle, _ptr(u0), int(n_steps), _ptr(gout), _ptr(gin), _ptr(gparams),
                                    _ptr(traj), base, self._vjp_bytes, _stream(stream)))

    KERNEL_CLASSES = ("conv_first", "conv_hidden", "conv_last", "flux_rk", "projection", "flux_proj", "fno", "scalar")

    def set_graph_replay(self, enable: bool):
        _check(lib().ld_set_graph_replay(self.handle, 1 if enable else 0))

    def set_kernel_timing(self, enable: bool):
        _check(lib().ld_set_kernel_timing(self.handle, 1 if enable else 0))

    def kernel_times(self):
        """{class: (total_ms, launches)} since the last call (synchronises)."""
        n = len(self.KERNEL_CLASSES)
        ms = (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        _check(lib().ld_kernel_times(self.handle, ms, cnt, n))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(self.KERNEL_CLASSES)}

    def step_index(self) -> int:
        v = C.c_int64()
        _check(lib().ld_get_step_index(self.handle, C.byref(v)))
        return v.value

    def reset_step_counter(self):
        _check(lib().ld_reset_step_counter(self.handle))

    def launches_per_step(self) -> int:
        v = C.c_int32()
        _check(lib().ld_launches_per_step(self.handle, C.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "handle", None):
            lib().ld_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
