"""BASELINE.json configs c1..c5 as plain parameter records (inputs only).

Every field mirrors a field of ``ld_config`` in include/ldsolver.h.  The dt rule
is the caller-side choice recorded as SURVEY.md §8c R11 (BASELINE.json c1:
"dt from CFL 0.5"; the other configs are silent):

    dt = 0.5 * h / u_ref
    c1      : u_ref = max|u0| + max|v0|              (2-D CFL)
    c2, c4  : u_ref = 1                               (IC normalised to max 1)
    c3, c5  : u_ref = max(1, chi / (nu k_f^2 + alpha)) (laminar Kolmogorov amplitude)
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

SYSTEM_BURGERS = 0
SYSTEM_NS = 1
ACT_RELU = 0
ACT_GELU = 1
STENCIL_LEARNED = 0
STENCIL_FIXED = 1
CONV_FP32 = 0
CONV_TF32 = 1


@dataclasses.dataclass
class LDConfig:
    name: str
    n: int
    batch: int
    system: int
    nu: float
    rk_order: int
    steps: int
    ic: str
    n_layers: int
    width: int
    activation: int
    tc_head: int = 0
    tc_interval: int = 1
    force_amp: float = 0.0
    force_k: float = 0.0
    drag: float = 0.0
    stencil_mode: int = STENCIL_LEARNED
    conv_precision: int = CONV_FP32
    length: float = 2.0 * math.pi
    dt: Optional[float] = None  # filled by with_dt()
    seed: int = 0
    fno_kmax: int = 0           # frequency-domain branch O_F (NEXT-2); fno_layers = 0: off
    fno_layers: int = 0
    fno_width: int = 0
    tc_mode: int = 0            # 0: TC head of the net; 1: history block over tc_interval inputs (NEXT-3)
    tc_kmax: int = 0
    tc_layers: int = 0
    tc_width: int = 0
    freeze_stencils: int = 0    # 1: the net runs once per step, its stencils reused by every stage
    scalar_mode: int = 0        # 1: a passive scalar advected-diffused with the flow (NS only)
    scalar_diff: float = 0.0    # its diffusivity D

    @property
    def h(self) -> float:
        return self.length / self.n

    @property
    def n_out(self) -> int:
        """Output channels of the last conv layer: 24 stencil + 2 TC (R3)."""
        return 24 + (2 if self.tc_head else 0)

    def u_ref(self, u0: np.ndarray) -> float:
        if self.name.startswith("c1") or self.ic == "fourier":
            return float(np.abs(u0[:, 0]).max() + np.abs(u0[:, 1]).max())
        if self.force_amp != 0.0:
            lam = self.force_amp / (self.nu * self.force_k ** 2 + self.drag)
            return max(1.0, lam)
        return 1.0

    def with_dt(self, u0: np.ndarray) -> "LDConfig":
        return dataclasses.replace(self, dt=0.5 * self.h / self.u_ref(u0))

    def replace(self, **kw) -> "LDConfig":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: 2-D viscous Burgers, 32^2, B=1, RK2, 3x32 ReLU net.
    "c1": LDConfig("c1", n=32, batch=1, system=SYSTEM_BURGERS, nu=0.01, rk_order=2,
                   steps=100, ic="fourier", n_layers=3, width=32, activation=ACT_RELU),
    # configs[1]: decaying NS, 64^2, B=32, RK3 + FFT projection, 6x64 GELU net.
    "c2": LDConfig("c2", n=64, batch=32, system=SYSTEM_NS, nu=1e-3, rk_order=3,
                   steps=1000, ic="spectrum", n_layers=6, width=64, activation=ACT_GELU),
    # configs[2]: Kolmogorov forced flow, 128^2, B=128, f=(sin 4y,0), drag 0.1, + TC head.
    "c3": LDConfig("c3", n=128, batch=128, system=SYSTEM_NS, nu=1e-3, rk_order=3,
                   steps=2000, ic="spectrum", n_layers=6, width=64, activation=ACT_GELU,
                   tc_head=1, force_amp=1.0, force_k=4.0, drag=0.1),
    # configs[3]: double shear layer, 256^2, B=64, full step with TC.
    "c4": LDConfig("c4", n=256, batch=64, system=SYSTEM_NS, nu=5e-4, rk_order=3,
                   steps=1000, ic="shear", n_layers=6, width=64, activation=ACT_GELU,
                   tc_head=1),
    # configs[4] (slab form): 4096^2, B=8, nu=1e-4, Kolmogorov forcing as c3.
    "c5a": LDConfig("c5a", n=4096, batch=8, system=SYSTEM_NS, nu=1e-4, rk_order=3,
                    steps=200, ic="spectrum", n_layers=6, width=64, activation=ACT_GELU,
                    tc_head=1, force_amp=1.0, force_k=4.0, drag=0.1),
    # configs[4] (ensemble form): 1024^2, B=512 sharded over ranks with no communication.
    "c5b": LDConfig("c5b", n=1024, batch=512, system=SYSTEM_NS, nu=1e-4, rk_order=3,
                    steps=200, ic="spectrum", n_layers=6, width=64, activation=ACT_GELU,
                    tc_head=1, force_amp=1.0, force_k=4.0, drag=0.1),
}


def get_config(name: str, **overrides) -> LDConfig:
    return dataclasses.replace(CONFIGS[name], **overrides)
