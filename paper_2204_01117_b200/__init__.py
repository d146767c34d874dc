"""citywind on the B200: the per-time-step RANS solver of UrbanFlow
(arXiv 2204.01117) as hand-written sm_100a CUDA kernels behind the
reference's Python step / simulate / optimize API.

Modules mirror the reference package ``citywind``:
  grid, geometry, linalg, solver, scenario, optimize, io
plus ``scenes`` (synthetic workload generators) and the native layer
(``_native``: ctypes binding of include/citywind_b200.h; ``build``).
"""
__version__ = "0.1.0"

from .errors import (ClassificationError, MeshError, ProjectionError, ScenarioError,  # noqa: F401
                     SingularSystemError)
from .grid import CellLabel, FlowState, GridSpec, PorosityField  # noqa: F401
