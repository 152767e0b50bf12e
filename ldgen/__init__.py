"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NONE of the method's arithmetic (no stencils, fluxes,
projection, RK or network evaluation).  It only produces inputs:

* ``configs``  -- the BASELINE.json configs c1..c5 as plain parameter records,
                  including the caller-side dt rule (the
                  C-ABI takes dt as an input, "δt").
* ``ic``       -- seeded initial velocity fields.
* ``weights``  -- seeded random-init weight blobs for the 3x3 conv net
                  ("minor random values").

Both sides receive the same arrays; neither side's arithmetic lives here.
"""
from .configs import CONFIGS, LDConfig, get_config  # noqa: F401
from .ic import make_ic  # noqa: F401
from .weights import make_weights, param_count, layer_shapes  # noqa: F401
