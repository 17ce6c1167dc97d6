"""Dense collocation assembly on the B200 (mirror of reference ``assembly.py``).

``Assembler(mesh, material)`` creates a device context (``ewb_ctx_create``):
geometry upload, exact GPU tier classification, near grading, self rules
and the static row-sum pass — the reference's ``__init__`` +
``_prepare_geometry`` + ``static_offdiag_rowsums`` (assembly.py:112-216).

Per frequency there are two entry points:

* ``assemble_tu(omega)`` -> (T, U) dense complex128 (N,N) CUDA tensors —
  the reference seam ``assembly.py:219`` (use ``.cpu().numpy()`` for host
  arrays, or ``host=True``);
* ``assemble_system(omega, bcs, prescribed)`` -> :class:`DenseSystem` — the
  fused kernel path used by the sweep: assembly + ``apply_bcs`` + the 3x3
  block-diagonal preconditioner, never materialising T or U.

Everything numeric runs in ``libewbem_b200.so``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass

import numpy as np

from . import _lib
from .material import Material
from .surface import corner_arrays
from .quadrature import QuadratureSet, device_rule_tables, gauss_legendre_tables

log = logging.getLogger(__name__)

NEUMANN = 0    # traction prescribed, displacement unknown   (assembly.py:32)
DIRICHLET = 1  # displacement prescribed, traction unknown   (assembly.py:33)


class BoundaryConditionError(ValueError):
    """Inconsistent or incomplete boundary-condition specification."""


@dataclass
class BoundaryConditionSet:
    """Per-element, per-component BC kinds and signal indices (assembly.py:41-83)."""

    kind: np.ndarray          # (n_elements, 3) uint8
    signal_index: np.ndarray  # (n_elements, 3) int32

    @classmethod
    def traction_free(cls, n_elements: int) -> "BoundaryConditionSet":
        return cls(kind=np.zeros((n_elements, 3), dtype=np.uint8),
                   signal_index=np.zeros((n_elements, 3), dtype=np.int32))

    def set_region(self, mesh, region_tag: int, components, kind: int,
                   signal_index: int) -> None:
        elements = np.flatnonzero(mesh.region_tag == region_tag)
        if elements.size == 0:
            raise BoundaryConditionError(f"region tag {region_tag} matches no elements")
        for c in components:
            self.kind[elements, c] = kind
            self.signal_index[elements, c] = signal_index

    def validate(self, allow_floating: bool = False) -> None:
        if not allow_floating and not (self.kind == DIRICHLET).any():
            raise BoundaryConditionError(
                "no Dirichlet DOF anywhere: the solid is free-floating "
                "(set allow_floating to override)")

    def flat_kind(self) -> np.ndarray:
        return self.kind.reshape(-1)

    def flat_signal(self) -> np.ndarray:
        return self.signal_index.reshape(-1)


@dataclass
class DenseSystem:
    """A a = b at one frequency; arrays are CUDA tensors (assembly.py:87-100).

    ``pinv`` holds the inverse 3x3 diagonal blocks of A (the reference's
    block_diag_precond factorisation) when the fused path produced it.
    """

    A: object
    b: object
    unknown_kind: np.ndarray
    pinv: object = None

    @property
    def n(self) -> int:
        return int(self.b.shape[0])


def _torch():
    import torch

    return torch


def _as_device(a, dtype):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


class Assembler:
    """Device-resident per-mesh context + per-frequency assembly (assembly.py:103-254)."""

    def __init__(self, mesh, material: Material,
                 quadrature: QuadratureSet | None = None, exterior: bool = False):
        """``exterior=True`` (not a reference mode; parity unpinned) puts +I on
        every dynamic T diagonal block: c + PV int T = I for an unbounded
        medium instead of the reference's interior identity."""
        lib = _lib.require_cuda()
        self.mesh = mesh
        self.material = material
        self.quad = quadrature or QuadratureSet.default()
        if self.quad != QuadratureSet.default():
            raise NotImplementedError("only the default quadrature ladder is compiled in")
        v0, v1, v2 = corner_arrays(mesh)
        corners = np.ascontiguousarray(np.stack([v0, v1, v2], axis=1))  # (n_e, 3, 3)
        rules, off, q = device_rule_tables()
        gl8, gl16 = gauss_legendre_tables(self.quad.duffy_radial, self.quad.duffy_angular)
        host = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (mesh.centroids, mesh.normals, mesh.areas, mesh.diameters, corners,
                 gl8, gl16, rules)]
        self._keep = host + [off, q]
        out = ctypes.c_void_p()
        _lib.check(lib.ewb_ctx_create(
            host[0].ctypes.data, host[1].ctypes.data, host[2].ctypes.data, host[3].ctypes.data,
            host[4].ctypes.data, mesh.n_elements, material.lam, material.mu, material.rho,
            host[5].ctypes.data, host[6].ctypes.data, host[7].ctypes.data, off.ctypes.data,
            q.ctypes.data, _lib.stream_handle(), ctypes.byref(out)), "ewb_ctx_create")
        self._ctx = out
        self._lib = lib
        self._static_tu = None
        self.exterior = bool(exterior)
        if self.exterior:
            _lib.check(lib.ewb_ctx_set_exterior(self._ctx, 1, _lib.stream_handle()))

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.ewb_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ctx(self):
        return self._ctx

    @property
    def n(self) -> int:
        return self.mesh.n_dofs

    def pair_counts(self) -> dict:
        """Element-pair census by tier (for the algorithmic work count)."""
        c = (ctypes.c_int64 * 8)()
        _lib.check(self._lib.ewb_ctx_counts(self._ctx, c))
        return dict(n_elements=c[0], far=c[1], mid=c[2], near=c[3],
                    near_levels={1: c[4], 2: c[5], 3: c[6], 4: c[7]})

    def pair_lists(self) -> dict:
        """The near / mid pair tables as host CSR arrays (rows sorted): near_ptr,
        near_j, near_lvl, mid_ptr, mid_j (assembly.py:132-161's buckets)."""
        pc = self.pair_counts()
        n = pc["n_elements"]
        out = dict(near_ptr=np.empty(n + 1, np.int32), near_j=np.empty(pc["near"], np.int32),
                   near_lvl=np.empty(pc["near"], np.int32), mid_ptr=np.empty(n + 1, np.int32),
                   mid_j=np.empty(pc["mid"], np.int32))
        _lib.check(self._lib.ewb_ctx_pair_lists(
            self._ctx, *[out[k].ctypes.data for k in ("near_ptr", "near_j", "near_lvl",
                                                      "mid_ptr", "mid_j")],
            _lib.stream_handle()), "ewb_ctx_pair_lists")
        return out

    def point_evals(self) -> int:
        """Quadrature-point evaluations per dense assembly."""
        pc = self.pair_counts()
        nl = pc["near_levels"]
        return (3 * pc["far"] + 7 * pc["mid"] + 28 * nl[1] + 112 * nl[2] + 448 * nl[3]
                + 1792 * nl[4] + 384 * pc["n_elements"])

    # ------------------------------------------------------------------
    def static_offdiag_rowsums(self, host: bool = True):
        torch = _torch()
        out = torch.empty((self.mesh.n_elements, 3, 3), dtype=torch.float64, device="cuda")
        _lib.check(self._lib.ewb_static_rowsums(self._ctx, _lib.ptr(out), _lib.stream_handle()))
        return out.cpu().numpy() if host else out

    def assemble_static_tu(self, host: bool = False):
        """Static (Kelvin) T, U with the rigid-body diagonal (assembly.py:184-216)."""
        torch = _torch()
        if self._static_tu is None:
            n = self.n
            t = torch.empty((n, n), dtype=torch.float64, device="cuda")
            u = torch.empty((n, n), dtype=torch.float64, device="cuda")
            _lib.check(self._lib.ewb_static_tu(self._ctx, _lib.ptr(t), _lib.ptr(u),
                                               _lib.stream_handle()), "ewb_static_tu")
            self._check_flags()
            self._static_tu = (t, u)
        t, u = self._static_tu
        return (t.cpu().numpy(), u.cpu().numpy()) if host else (t, u)

    def _check_flags(self, omega=None):
        nf, sg = ctypes.c_int32(), ctypes.c_int32()
        _lib.check(self._lib.ewb_ctx_flags(self._ctx, ctypes.byref(nf), ctypes.byref(sg),
                                           _lib.stream_handle()))
        if nf.value:
            raise FloatingPointError(f"non-finite entries assembled at omega = {omega}")
        return sg.value

    def assemble_tu(self, omega: complex, host: bool = False, out=None):
        """Dense T and U at complex omega, free term absorbed (assembly.py:219-254)."""
        torch = _torch()
        omega = complex(omega)
        if omega == 0:
            ts, us = self.assemble_static_tu()
            t, u = ts.to(torch.complex128), us.to(torch.complex128)
        else:
            n = self.n
            if out is not None:
                t, u = out
            else:
                t = torch.empty((n, n), dtype=torch.complex128, device="cuda")
                u = torch.empty((n, n), dtype=torch.complex128, device="cuda")
            _lib.check(self._lib.ewb_assemble_tu(self._ctx, omega.real, omega.imag, _lib.ptr(t),
                                                 _lib.ptr(u), _lib.stream_handle()),
                       "ewb_assemble_tu")
            self._check_flags(omega)
        return (t.cpu().numpy(), u.cpu().numpy()) if host else (t, u)

    def assemble_system(self, omega: complex, bcs: BoundaryConditionSet, prescribed,
                        out: DenseSystem | None = None, check: bool = True) -> DenseSystem:
        """Fused assemble_tu + apply_bcs + block preconditioner, on the device."""
        torch = _torch()
        omega = complex(omega)
        kinds = np.ascontiguousarray(bcs.flat_kind(), dtype=np.uint8)
        n = self.n
        p = _as_device(prescribed, torch.complex128)
        if p.shape != (n,):
            raise ValueError("prescribed spectrum has wrong length")
        if omega == 0:
            t, u = self.assemble_tu(0.0)
            return apply_bcs(t, u, bcs, p)
        if out is None:
            out = DenseSystem(A=torch.empty((n, n), dtype=torch.complex128, device="cuda"),
                              b=torch.empty(n, dtype=torch.complex128, device="cuda"),
                              unknown_kind=kinds.copy(),
                              pinv=torch.empty((n // 3, 3, 3), dtype=torch.complex128,
                                               device="cuda"))
        kd = getattr(out, "_kinds_dev", None)
        if kd is None or not np.array_equal(getattr(out, "_kinds_host", None), kinds):
            kd = torch.from_numpy(kinds).cuda()
            out._kinds_dev, out._kinds_host = kd, kinds
        _lib.check(self._lib.ewb_assemble_system(
            self._ctx, omega.real, omega.imag, _lib.ptr(kd), _lib.ptr(p), _lib.ptr(out.A),
            _lib.ptr(out.b), _lib.ptr(out.pinv), _lib.stream_handle()), "ewb_assemble_system")
        if check:
            singular = self._check_flags(omega)
            if singular:
                log.warning("%d singular 3x3 diagonal blocks; identity fallback", singular)
        return out

    MAX_BATCH = 32   # EWB_MAX_BATCH

    def assemble_system_multi(self, omegas, bcs: BoundaryConditionSet, prescribed,
                              out: "SystemBatch | None" = None, flags=None,
                              check: bool = True) -> "SystemBatch":
        """``assemble_system`` for nf <= 32 frequencies of one sweep in one pass
        over the element pairs (ewb_assemble_system_multi).

        ``prescribed`` is (nf, N).  Member f equals ``assemble_system(omegas[f])``
        to <= 1e-13 of max|A|: pair geometry and the damping factors are shared
        and, for an equispaced batch (omega_k = k dw - i eta), the phase
        factors are stepped instead of re-evaluated.  ``flags`` (optional
        (nf, 4) int32 CUDA tensor, zeroed by the caller) receives the
        per-member fault words; with ``check`` they are read back and raised on.
        """
        torch = _torch()
        om = np.asarray([complex(w) for w in omegas], dtype=complex)
        nf = len(om)
        if not 1 <= nf <= self.MAX_BATCH:
            raise ValueError(f"batch of {nf} frequencies (1..{self.MAX_BATCH})")
        if np.any(om == 0):
            raise ValueError("omega == 0 takes the static path (assemble_system)")
        kinds = np.ascontiguousarray(bcs.flat_kind(), dtype=np.uint8)
        n = self.n
        p = _as_device(prescribed, torch.complex128)
        if tuple(p.shape) != (nf, n):
            raise ValueError("prescribed spectra must be (nf, N)")
        if out is None or out.A.shape[0] < nf:
            out = SystemBatch.allocate(nf, n)
        kd = getattr(out, "_kinds_dev", None)
        if kd is None or not np.array_equal(getattr(out, "_kinds_host", None), kinds):
            kd = torch.from_numpy(kinds).cuda()
            out._kinds_dev, out._kinds_host = kd, kinds
        own_flags = flags is None
        if own_flags:
            flags = torch.zeros((nf, 4), dtype=torch.int32, device="cuda")
        ore = np.ascontiguousarray(om.real)
        oim = np.ascontiguousarray(om.imag)
        _lib.check(self._lib.ewb_assemble_system_multi(
            self._ctx, nf, ore.ctypes.data, oim.ctypes.data, _lib.ptr(kd), _lib.ptr(p),
            _lib.ptr(out.A), _lib.ptr(out.b), _lib.ptr(out.pinv), _lib.ptr(flags),
            _lib.stream_handle()), "ewb_assemble_system_multi")
        out.nf = nf
        out.unknown_kind = kinds.copy()
        if check:
            fl = flags.cpu().numpy()
            for f in range(nf):
                if fl[f, 0]:
                    raise FloatingPointError(f"non-finite entries assembled at omega = {om[f]}")
                if fl[f, 1]:
                    log.warning("%d singular 3x3 diagonal blocks; identity fallback", fl[f, 1])
        return out


@dataclass
class SystemBatch:
    """nf dense systems of one sweep, stacked: A (nf,N,N), b (nf,N), pinv (nf,n_e,3,3)."""

    A: object
    b: object
    pinv: object
    unknown_kind: np.ndarray | None = None
    nf: int = 0

    @classmethod
    def allocate(cls, nf: int, n: int) -> "SystemBatch":
        torch = _torch()
        return cls(A=torch.empty((nf, n, n), dtype=torch.complex128, device="cuda"),
                   b=torch.empty((nf, n), dtype=torch.complex128, device="cuda"),
                   pinv=torch.empty((nf, n // 3, 3, 3), dtype=torch.complex128, device="cuda"))

    def member(self, f: int) -> DenseSystem:
        if not 0 <= f < self.nf:
            raise IndexError(f)
        return DenseSystem(A=self.A[f], b=self.b[f], unknown_kind=self.unknown_kind,
                           pinv=self.pinv[f])


def assemble_tu(mesh, material: Material, omega: complex,
                quadrature: QuadratureSet | None = None):
    return Assembler(mesh, material, quadrature).assemble_tu(omega)


def apply_bcs(t_mat, u_mat, bcs: BoundaryConditionSet, prescribed) -> DenseSystem:
    """Column swap into A and b (assembly.py:263-297), on the device."""
    torch = _torch()
    lib = _lib.require_cuda()
    kinds = np.ascontiguousarray(bcs.flat_kind(), dtype=np.uint8)
    n = len(kinds)
    t = _as_device(t_mat, torch.complex128)
    u = _as_device(u_mat, torch.complex128)
    if tuple(t.shape) != (n, n) or tuple(u.shape) != (n, n):
        raise ValueError("matrix/BC size mismatch")
    if isinstance(prescribed, np.ndarray) or not hasattr(prescribed, "device"):
        pr = np.asarray(prescribed, dtype=complex)
        if pr.shape != (n,):
            raise ValueError("prescribed spectrum has wrong length")
        if not np.isfinite(pr).all():
            raise ValueError("unresolved (non-finite) prescribed boundary value")
    p = _as_device(prescribed, torch.complex128)
    if tuple(p.shape) != (n,):
        raise ValueError("prescribed spectrum has wrong length")
    if not bool(torch.isfinite(torch.view_as_real(p)).all()):
        raise ValueError("unresolved (non-finite) prescribed boundary value")
    kd = torch.from_numpy(kinds).cuda()
    a = torch.empty((n, n), dtype=torch.complex128, device="cuda")
    b = torch.empty(n, dtype=torch.complex128, device="cuda")
    _lib.check(lib.ewb_apply_bcs(_lib.ptr(t), _lib.ptr(u), _lib.ptr(kd), _lib.ptr(p), n,
                                 _lib.ptr(a), _lib.ptr(b), _lib.stream_handle()), "ewb_apply_bcs")
    return DenseSystem(A=a, b=b, unknown_kind=kinds.copy())


def scatter_solution(system: DenseSystem, a, prescribed):
    """(u, t) full DOF vectors (assembly.py:300-305); device tensors in, device out."""
    torch = _torch()
    a = _as_device(a, torch.complex128)
    p = _as_device(prescribed, torch.complex128)
    neu = torch.from_numpy(np.asarray(system.unknown_kind) == NEUMANN).cuda()
    return torch.where(neu, a, p), torch.where(~neu, a, p)
