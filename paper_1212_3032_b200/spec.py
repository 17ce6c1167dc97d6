"""Sweep description consumed by ``run_sweep`` / ``DeviceSweep``.

``run_sweep`` is duck-typed on the reference's ``SweepConfig``
(``config.py:58-108``): a reference config object, built by the reference's
own ``parse_config`` or library API, runs unchanged.  ``SweepSpec`` and
``Probe`` are the minimal stand-ins used where the reference does not exist
(the GPU box: tests, benchmark, ``workloads.py``).  The ``.cfg`` parser and
the CLI stay with the reference (out of scope).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

from .transform import WINDOW_KINDS


@dataclass(frozen=True)
class Probe:
    """A monitored DOF: displacement or traction of one element component."""

    name: str
    element: int
    component: int
    quantity: str            # "displacement" | "traction"

    @property
    def dof(self) -> int:
        return 3 * self.element + self.component


@dataclass
class SweepSpec:
    """Same field names and defaults as the reference's SweepConfig."""

    mesh: object
    material: object
    bcs: object
    signals: list
    signal_names: list
    probes: list
    period: float
    n_omega: int
    kappa: float = 4.0
    window: str = "hanning"
    sem_enabled: bool = True
    sem_depth: int = 4
    tol: float = 1e-5
    restart: int = 60
    maxiter: int = 1000
    output_dir: Path = Path("out")
    figures: bool = True
    workers: int = 1
    allow_floating: bool = False
    raw: list = field(default_factory=list)

    def __post_init__(self):
        # what the device path relies on; the reference's own object carries
        # the full validation of a user configuration
        if not (self.period > 0 and self.n_omega >= 4 and self.n_omega % 2 == 0):
            raise ValueError("need period > 0 and an even n_omega >= 4")
        if self.window not in WINDOW_KINDS or not 0 < self.tol < 1 or self.sem_depth < 1:
            raise ValueError("bad window, tol or sem_depth")
        if any(not 0 <= p.dof < self.mesh.n_dofs for p in self.probes):
            raise ValueError("probe outside the mesh")
        self.bcs.validate(allow_floating=self.allow_floating)
