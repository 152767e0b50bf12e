"""B200-native LDSolver coarse-grid rollout step (arXiv 2507.01975).

The compute path is libldsolver.so (hand-written sm_100a CUDA behind the C ABI in
include/ldsolver.h); ``ldsolver`` is its thin ctypes binding.  Nothing in this
package imports the CPU oracle, and there is no CPU fallback.
"""
__version__ = "0.1.0"
