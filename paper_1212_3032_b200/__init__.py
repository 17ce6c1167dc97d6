"""B200-native (sm_100a, FP64) per-frequency solve of the exponentially
windowed elastodynamic BEM of arXiv 1212.3032 — a drop-in for the hot path
of the CPU reference ``ewbem`` 0.1.0.

Host API mirrors the reference names (Assembler, apply_bcs, gmres,
block_diag_precond, sem_initial_guess, run_sweep, ...); the compute runs in
``libewbem_b200.so`` (C ABI: ``include/ewbem_b200.h``).  Importing the
package is cheap; compute calls raise ``NativeUnavailable`` without the
library or a CUDA device (no CPU fallback).
"""

__version__ = "0.1.0"

from ._lib import NativeUnavailable  # noqa: F401
from .assembly import (  # noqa: F401
    DIRICHLET, NEUMANN, Assembler, BoundaryConditionError, BoundaryConditionSet, DenseSystem,
    apply_bcs, assemble_tu, scatter_solution,
)
from .driver import SweepError, SweepResult, emit_outputs, run_sweep  # noqa: F401
from .linsolve import (  # noqa: F401
    SolutionHistory, SolveStats, block_diag_precond, gmres, sem_initial_guess,
)
from .material import Material, wave_speeds, wavenumbers  # noqa: F401
from .matfree import MatrixFreeOperator  # noqa: F401
from .quadrature import QuadratureSet  # noqa: F401
from .spec import Probe, SweepSpec  # noqa: F401
from .surface import SurfaceMesh  # noqa: F401
from .transform import (  # noqa: F401
    Spectrum, SpectrumSymmetryError, TimeSignal, conjugate_fill, eta_from_kappa,
    forward_mft, frequency_grid, inverse_mft, window_weights,
)
