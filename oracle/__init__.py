"""CPU oracle (fp64 numpy) for the LDSolver rollout step.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product
package paper_2507_01975_b200, which shares no code with it.
"""
from .ldsolver_oracle import (  # noqa: F401
    Oracle, step, rollout, project, div_c, solve_pressure, symbol, tendency,
    constrain, net_forward, conv3x3_periodic, unpack_params, gelu, relu,
    default_base_stencils, projector_interp, projector_deriv, face_values, S_OFFSETS, downsample,
    scalar_tendency, base_5x4, constrain_5x4, face_values_5x4, tendency_5x4,
)
from .spectral_oracle import spectral_operator, full_plane, spectral_faces, unpack_spectral, half_cell_shift  # noqa: F401,E402
