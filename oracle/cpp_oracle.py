"""ctypes wrapper of the plain C++ CPU oracle (oracle/cpp/ldsolver_oracle.cpp) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may use
this module.  The library is built in-tree (``build()``; g++ -O2, no -ffast-math, -pthread) by
``__graft_entry__.build()``; it shares no code with the CUDA path (paper_2507_01975_b200).

API (fp64 numpy in / out, fields [B][2][N][N]; cfg = an ldgen.LDConfig or a dict with its fields):
  step(u, cfg, params, base=None, step_index=0, threads=0, precision=0)   one step (R8 gating by step_index)
  rollout(u, cfg, params, n_steps, ...)                                   n steps (FloatingPointError on NaN/Inf)
  net_forward(u, cfg, params)  -> R [B][N][N][n_out]
  stencils(u, cfg, params, base=None) -> w [B][N][N][24]
  tendency(u, cfg, params, base=None) -> T [B][2][N][N]
  project(u, cfg)  -> P(u)
  hardware_threads() -> threads the library uses by default
precision 1 runs the same code in fp32 (a diagnostic variant; inputs / outputs stay fp64).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cpp", "ldsolver_oracle.cpp")
LIB = os.path.join(HERE, "cpp", "libldoracle.so")
FLAGS = ["-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-fno-fast-math"]


class ora_config(C.Structure):
    _fields_ = [("n", C.c_int32), ("batch", C.c_int32), ("length", C.c_double), ("system", C.c_int32),
                ("nu", C.c_double), ("dt", C.c_double), ("rk_order", C.c_int32),
                ("force_amp", C.c_double), ("force_k", C.c_double), ("drag", C.c_double),
                ("n_layers", C.c_int32), ("width", C.c_int32), ("activation", C.c_int32),
                ("tc_head", C.c_int32), ("tc_interval", C.c_int32), ("stencil_mode", C.c_int32)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["g++", *FLAGS, "-o", LIB + ".tmp", SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("C++ oracle build failed:\n" + r.stdout + r.stderr)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        L.ora_rollout.argtypes = [C.POINTER(ora_config), C.c_void_p, C.c_size_t, C.c_void_p, dp, C.c_int64,
                                  C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]
        L.ora_net.argtypes = [C.POINTER(ora_config), C.c_void_p, C.c_size_t, dp, dp, C.c_int32]
        L.ora_stencils.argtypes = [C.POINTER(ora_config), C.c_void_p, C.c_size_t, C.c_void_p, dp, dp, C.c_int32]
        L.ora_tendency.argtypes = [C.POINTER(ora_config), C.c_void_p, C.c_size_t, C.c_void_p, dp, dp, C.c_int32]
        L.ora_project.argtypes = [C.POINTER(ora_config), dp, C.c_int32]
        L.ora_param_count.argtypes = [C.POINTER(ora_config)]
        L.ora_param_count.restype = C.c_size_t
        L.ora_last_error.restype = C.c_char_p
        for f in ("ora_rollout", "ora_net", "ora_stencils", "ora_tendency", "ora_project", "ora_hardware_threads"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _get(cfg, name, default=None):
    if isinstance(cfg, dict):
        return cfg.get(name, default)
    return getattr(cfg, name, default)


def _cfg(cfg, batch):
    c = ora_config()
    c.n = int(_get(cfg, "n"))
    c.batch = int(batch)
    c.length = float(_get(cfg, "length", 2 * math.pi))
    c.system = int(_get(cfg, "system"))
    c.nu = float(_get(cfg, "nu"))
    c.dt = float(_get(cfg, "dt", 0.0) or 0.0)
    c.rk_order = int(_get(cfg, "rk_order", 3))
    c.force_amp = float(_get(cfg, "force_amp", 0.0) or 0.0)
    c.force_k = float(_get(cfg, "force_k", 0.0) or 0.0)
    c.drag = float(_get(cfg, "drag", 0.0) or 0.0)
    c.n_layers = int(_get(cfg, "n_layers", 2) or 2)
    c.width = int(_get(cfg, "width", 1) or 1)
    c.activation = int(_get(cfg, "activation", 1))
    c.tc_head = int(_get(cfg, "tc_head", 0) or 0)
    c.tc_interval = int(_get(cfg, "tc_interval", 1) or 1)
    c.stencil_mode = int(_get(cfg, "stencil_mode", 0) or 0)
    for unsupported in ("fno_layers", "tc_mode", "freeze_stencils"):
        if int(_get(cfg, unsupported, 0) or 0) != 0:
            raise ValueError(f"the C++ oracle covers the BASELINE step only ({unsupported} must be 0)")
    return c


def _params(params):
    if params is None:
        return None, 0, None
    p = np.ascontiguousarray(params, dtype=np.float32).ravel()
    return p.ctypes.data_as(C.c_void_p), p.size, p


def _base(base):
    if base is None:
        return None, None
    b = np.ascontiguousarray(base, dtype=np.float64).ravel()
    assert b.size == 24
    return b.ctypes.data_as(C.c_void_p), b


def _err(rc):
    if rc != 0:
        raise ValueError(lib().ora_last_error().decode())


def hardware_threads() -> int:
    return int(lib().ora_hardware_threads())


def rollout(u, cfg, params, n_steps: int, base=None, step_index: int = 0, threads: int = 0, precision: int = 0):
    x = np.array(u, dtype=np.float64, copy=True, order="C")
    c = _cfg(cfg, x.shape[0])
    pp, npar, keep = _params(params)
    bp, keepb = _base(base)
    bad = C.c_int64(-1)
    rc = lib().ora_rollout(C.byref(c), pp, npar, bp, x.ctypes.data_as(C.POINTER(C.c_double)), int(step_index),
                           int(n_steps), int(threads), int(precision), C.byref(bad))
    if rc == -5:
        raise FloatingPointError(f"non-finite field at step {bad.value}")
    _err(rc)
    return x


def step(u, cfg, params=None, base=None, step_index: int = 0, threads: int = 0, precision: int = 0):
    return rollout(u, cfg, params, 1, base, step_index, threads, precision)


def net_forward(u, cfg, params, threads: int = 0):
    x = np.ascontiguousarray(u, dtype=np.float64)
    c = _cfg(cfg, x.shape[0])
    n_out = 24 + (2 if c.tc_head else 0)
    out = np.zeros((x.shape[0], c.n, c.n, n_out))
    pp, npar, keep = _params(params)
    _err(lib().ora_net(C.byref(c), pp, npar, x.ctypes.data_as(C.POINTER(C.c_double)),
                       out.ctypes.data_as(C.POINTER(C.c_double)), int(threads)))
    return out


def stencils(u, cfg, params, base=None, threads: int = 0):
    x = np.ascontiguousarray(u, dtype=np.float64)
    c = _cfg(cfg, x.shape[0])
    out = np.zeros((x.shape[0], c.n, c.n, 24))
    pp, npar, keep = _params(params)
    bp, keepb = _base(base)
    _err(lib().ora_stencils(C.byref(c), pp, npar, bp, x.ctypes.data_as(C.POINTER(C.c_double)),
                            out.ctypes.data_as(C.POINTER(C.c_double)), int(threads)))
    return out


def tendency(u, cfg, params=None, base=None, threads: int = 0):
    x = np.ascontiguousarray(u, dtype=np.float64)
    c = _cfg(cfg, x.shape[0])
    out = np.zeros_like(x)
    pp, npar, keep = _params(params)
    bp, keepb = _base(base)
    _err(lib().ora_tendency(C.byref(c), pp, npar, bp, x.ctypes.data_as(C.POINTER(C.c_double)),
                            out.ctypes.data_as(C.POINTER(C.c_double)), int(threads)))
    return out


def project(u, cfg, threads: int = 0):
    x = np.array(u, dtype=np.float64, copy=True, order="C")
    c = _cfg(cfg, x.shape[0])
    _err(lib().ora_project(C.byref(c), x.ctypes.data_as(C.POINTER(C.c_double)), int(threads)))
    return x
