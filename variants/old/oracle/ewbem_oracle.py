"""CPU oracle for the per-frequency BEM solve — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference
arm may import it.  The product path (``paper_1212_3032_b200``) never
imports anything under ``oracle/`` and fails loudly without its CUDA
library.

It is a numpy restatement of the reference ``ewbem`` 0.1.0 hot path
(``/root/reference/pkg/src/ewbem``), written from the published
algorithm and organised differently from the reference; every function
cites the reference lines it follows.  The third-party arithmetic is the
same as the reference's: numpy (complex ufuncs, BLAS ``matmul``, LAPACK
``inv``/``qr``/``solve``, pocketfft ``fft``), pinned as numpy 2.3.5 /
OpenBLAS 0.3.30 in the survey container.

Parity pinning: ``tests/golden/make_golden.py`` imports the live
reference in the build container and writes fixtures (assembled T/U,
tier tables, rule tables, GMRES/SEM/transform vectors, sweep iteration
counts and histories).  ``tests/test_oracle_golden.py`` checks this
oracle against every fixture, and against the live reference whenever
``/root/reference`` is importable.

Structure (reference file:line in brackets):
  Medium ............ material constants, wavenumbers   [material.py:11-94]
  element_geometry .. centroids/normals/areas/diam.      [mesh.py:88-106]
  rules ............. gauss3/7, subdivided, Duffy self   [quadrature.py:63-185]
  tiers ............. classify + near grading            [quadrature.py:223-235,
                                                          assembly.py:132-161,
                                                          mesh.py:165-204]
  radial scalars .... closed / 24-term series / static   [kernels.py:56-152]
  contract .......... weighted U/T block contraction     [kernels.py:292-357]
  DenseOracle ....... geometry prep, static pass, T/U    [assembly.py:103-254]
  apply_bcs ......... column swap into A, b              [assembly.py:263-305]
  gmres / precond / sem                                  [linsolve.py:51-242]
  spectral pipeline . eta, grid, forward, fill, inverse  [transform.py:113-211]
  sweep ............. the frequency loop                 [driver.py:92-176]
"""

from __future__ import annotations

import math
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np

FOUR_PI = 4.0 * math.pi
NEUMANN, DIRICHLET = 0, 1


# ----------------------------------------------------------------------
# material                                         [material.py:11-94]
# ----------------------------------------------------------------------
@dataclass(frozen=True)
class Medium:
    lam: float
    mu: float
    rho: float

    @classmethod
    def young_poisson(cls, E, nu, rho):           # [material.py:44-55]
        mu = E / (2.0 * (1.0 + nu))
        lam = 0.0 if nu == 0.0 else E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
        return cls(lam, mu, float(rho))

    @property
    def c_s(self):                                 # [material.py:68-70]
        return float(np.sqrt(self.mu / self.rho))

    @property
    def c_p(self):                                 # [material.py:72-75]
        return float(np.sqrt((self.lam + 2.0 * self.mu) / self.rho))

    def wavenumbers(self, omega):                  # [material.py:83-94]
        omega = complex(omega)
        if omega.imag > 1e-12 * max(1.0, abs(omega)):
            raise ValueError(f"frequency {omega} has positive imaginary part")
        return omega / self.c_s, omega / self.c_p


# ----------------------------------------------------------------------
# element geometry                                 [mesh.py:88-106]
# ----------------------------------------------------------------------
def element_geometry(vertices, triangles):
    v = np.asarray(vertices, dtype=np.float64)
    t = np.asarray(triangles, dtype=np.int64)
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    n = np.cross(b - a, c - a)
    n2 = np.linalg.norm(n, axis=1)
    edges = np.stack([np.linalg.norm(b - a, axis=1), np.linalg.norm(c - b, axis=1),
                      np.linalg.norm(a - c, axis=1)], axis=1)
    return dict(centroids=(a + b + c) / 3.0, normals=n / n2[:, None],
                areas=0.5 * n2, diameters=edges.max(axis=1),
                corners=np.stack([a, b, c], axis=1))


# ----------------------------------------------------------------------
# quadrature rules                                 [quadrature.py:37-185]
# A rule is (bary (Q,3), weights (Q,)) on the reference triangle.
# ----------------------------------------------------------------------
def rule_g3():                                     # [quadrature.py:63-72]
    hi, lo = 2 / 3, 1 / 6
    bary = np.array([[hi, lo, lo], [lo, hi, lo], [lo, lo, hi]])
    return bary, np.full(3, 1 / 3)


def rule_g7():                                     # [quadrature.py:75-88]
    r15 = np.sqrt(15.0)
    pa, pb = (6.0 + r15) / 21.0, (6.0 - r15) / 21.0
    wa, wb = (155.0 + r15) / 1200.0, (155.0 - r15) / 1200.0
    bary, wts = [[1 / 3, 1 / 3, 1 / 3]], [9.0 / 40.0]
    for p, w in ((pa, wa), (pb, wb)):
        q = 1 - 2 * p
        bary += [[p, p, q], [p, q, p], [q, p, p]]
        wts += [w, w, w]
    return np.array(bary), np.array(wts)


def rule_refine(rule, levels):                     # [quadrature.py:110-132]
    """Base rule replicated on the 4**levels congruent midpoint children."""
    bary, wts = rule
    patches = [np.eye(3)]
    for _ in range(levels):
        nxt = []
        for p in patches:
            m01, m12, m20 = (p[0] + p[1]) / 2, (p[1] + p[2]) / 2, (p[2] + p[0]) / 2
            nxt += [np.array([p[0], m01, m20]), np.array([m01, p[1], m12]),
                    np.array([m20, m12, p[2]]), np.array([m01, m12, m20])]
        patches = nxt
    share = 1.0 / len(patches)
    return (np.concatenate([bary @ p for p in patches]),
            np.concatenate([wts * share for _ in patches]))


def self_points(verts, n_radial=8, n_angular=16):  # [quadrature.py:135-185]
    """Duffy/asinh rule centred on the centroid: (Q,3) points, (Q,) weights."""
    verts = np.asarray(verts, dtype=float)
    ctr = verts.mean(axis=0)
    xr, wr = np.polynomial.legendre.leggauss(n_radial)
    s = 0.5 * (xr + 1.0)
    ws = 0.5 * wr
    xa, wa = np.polynomial.legendre.leggauss(n_angular)
    out_p, out_w = [], []
    for k in range(3):
        a = verts[k] - ctr
        b = verts[(k + 1) % 3] - ctr
        e1 = a / np.linalg.norm(a)
        nz = np.cross(a, b)
        nz /= np.linalg.norm(nz)
        e2 = np.cross(nz, e1)
        a2 = np.array([a @ e1, a @ e2])
        b2 = np.array([b @ e1, b @ e2])
        t1 = np.arctan2(a2[1], a2[0])
        t2 = np.arctan2(b2[1], b2[0])
        if t2 <= t1:
            t2 += 2.0 * np.pi
        ed = b2 - a2
        foot = a2 + (-(a2 @ ed) / (ed @ ed)) * ed
        h = np.linalg.norm(foot)
        tf = np.arctan2(foot[1], foot[0])
        u_lo = np.arcsinh(np.tan(t1 - tf))
        u_hi = np.arcsinh(np.tan(t2 - tf))
        u = 0.5 * (u_hi - u_lo) * xa + 0.5 * (u_hi + u_lo)
        wu = 0.5 * (u_hi - u_lo) * wa
        theta = tf + np.arctan(np.sinh(u))
        ray = h * np.cosh(u)
        w2 = ws[:, None] * (wu / np.cosh(u))[None, :] * s[:, None] * (ray ** 2)[None, :]
        dirs = np.stack([np.cos(theta), np.sin(theta)], axis=1)
        p2 = s[:, None, None] * ray[None, :, None] * dirs[None, :, :]
        p3 = ctr + p2[..., 0:1] * e1 + p2[..., 1:2] * e2
        out_p.append(p3.reshape(-1, 3))
        out_w.append(w2.ravel())
    return np.concatenate(out_p), np.concatenate(out_w)


# ----------------------------------------------------------------------
# tiers and near grading      [quadrature.py:206-235, assembly.py:132-161]
# ----------------------------------------------------------------------
FAR_RATIO, NEAR_RATIO = 4.0, 1.5
NEAR_GRADING = (0.60, 0.30, 0.15)


def tier_table(centroids, diameters):
    """uint8 (n_e, n_e): 0 far, 1 mid, 2 near; ratio normalised by the COLUMN."""
    gap = np.linalg.norm(centroids[:, None, :] - centroids[None, :, :], axis=-1)
    ratio = gap / diameters[None, :]
    tier = np.zeros(ratio.shape, dtype=np.uint8)
    tier[ratio < FAR_RATIO] = 1
    tier[ratio < NEAR_RATIO] = 2
    return tier


def tiers_for_rows(centroids, diameters, rows, cols=None):
    cols = np.arange(len(centroids)) if cols is None else cols
    gap = np.linalg.norm(centroids[rows][:, None, :] - centroids[cols][None, :, :], axis=-1)
    ratio = gap / diameters[cols][None, :]
    tier = np.zeros(ratio.shape, dtype=np.uint8)
    tier[ratio < FAR_RATIO] = 1
    tier[ratio < NEAR_RATIO] = 2
    return tier


def surface_distance(points, verts):               # [mesh.py:165-204]
    """Distance from points (M,3) to the triangle ``verts`` (3,3)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    p0, p1, p2 = np.asarray(verts, dtype=float)
    u, v = p1 - p0, p2 - p0
    rel = pts - p0
    uu, uv, vv = u @ u, u @ v, v @ v
    ru, rv = rel @ u, rel @ v
    det = uu * vv - uv * uv
    s = np.clip((vv * ru - uv * rv) / det, 0.0, 1.0)
    t = np.clip((uu * rv - uv * ru) / det, 0.0, 1.0)
    over = s + t > 1.0
    if over.any():
        excess = (s[over] + t[over] - 1.0) / 2.0
        s[over] = np.clip(s[over] - excess, 0.0, 1.0)
        t[over] = np.clip(t[over] - excess, 0.0, 1.0)
    best = np.linalg.norm(pts - (p0 + s[:, None] * u + t[:, None] * v), axis=1)
    for a, b in ((p0, p1), (p1, p2), (p2, p0)):
        seg = b - a
        f = np.clip(((pts - a) @ seg) / (seg @ seg), 0.0, 1.0)
        best = np.minimum(best, np.linalg.norm(pts - (a + f[:, None] * seg), axis=1))
    return best


def near_level(sep_ratio):                         # [quadrature.py:230-235]
    lvl = np.ones(np.shape(sep_ratio), dtype=np.int64)
    for thr in NEAR_GRADING:
        lvl[sep_ratio < thr] += 1
    return lvl


# ----------------------------------------------------------------------
# radial scalars                                   [kernels.py:36-152]
# ----------------------------------------------------------------------
SERIES_SWITCH = 0.35
SERIES_TERMS = 24


def _series_tables():                              # [kernels.py:40-53]
    n = np.arange(SERIES_TERMS)
    inv = np.array([1.0 / math.factorial(k) for k in range(SERIES_TERMS + 2)])
    rot = (-1j) ** n
    c_phi_s = rot * (inv[n] - inv[n + 1] + inv[n + 2])
    c_phi_p = -rot * (inv[n + 1] - inv[n + 2])
    c_psi = rot * (inv[n] - 3.0 * inv[n + 1] + 3.0 * inv[n + 2])
    return c_phi_s, c_phi_p, c_psi


C_PHI_S, C_PHI_P, C_PSI = _series_tables()


def _closed(zs, zp, g2):                           # [kernels.py:102-119]
    es, ep = np.exp(-1j * zs), np.exp(-1j * zp)
    qs, qp = 1.0 / zs, 1.0 / zp
    qs2, qp2 = qs * qs, qp * qp
    f0 = es * (1.0 - 1j * qs - qs2) - g2 * ep * (-1j * qp - qp2)
    f1 = es * (1.0 - 3j * qs - 3.0 * qs2) - g2 * ep * (1.0 - 3j * qp - 3.0 * qp2)
    f2 = es * (-1j * zs - 2.0 + 3j * qs + 3.0 * qs2) - g2 * ep * (-1.0 + 3j * qp + 3.0 * qp2)
    f3 = es * (-1j * zs - 4.0 + 9j * qs + 9.0 * qs2) - g2 * ep * (
        -1j * zp - 4.0 + 9j * qp + 9.0 * qp2)
    return f0, f1, f2, f3


def _series(zs, zp, g2):                           # [kernels.py:122-138]
    acc = [np.zeros(zs.shape, dtype=complex) for _ in range(4)]
    ps = np.ones(zs.shape, dtype=complex)
    pp = np.ones(zs.shape, dtype=complex)
    for n in range(SERIES_TERMS):
        t_phi = C_PHI_S[n] * ps - g2 * C_PHI_P[n] * pp
        t_psi = C_PSI[n] * (ps - g2 * pp)
        acc[0] += t_phi
        acc[1] += t_psi
        acc[2] += (n - 1) * t_phi
        acc[3] += (n - 1) * t_psi
        ps *= zs
        pp *= zp
    return tuple(acc)


def radial_scalars(r, ks, kp):                     # [kernels.py:56-99]
    """(phi, psi, dphi/dr, dpsi/dr) at distances r for wavenumbers ks, kp."""
    r = np.asarray(r, dtype=float)
    if np.any(r <= 0.0):
        raise ValueError("radial_scalars requires r > 0")
    ks, kp = complex(ks), complex(kp)
    g2 = (kp / ks) ** 2
    zs, zp = ks * r, kp * r
    ser = np.abs(zs) < SERIES_SWITCH
    nser = int(ser.sum())
    if nser == 0:
        f = _closed(zs, zp, g2)
    elif nser == ser.size:
        f = _series(zs, zp, g2)
    else:
        f = [np.empty(r.shape, dtype=complex) for _ in range(4)]
        cl = ~ser
        for dst, val in zip(f, _closed(zs[cl], zp[cl], g2)):
            dst[cl] = val
        for dst, val in zip(f, _series(zs[ser], zp[ser], g2)):
            dst[ser] = val
    ir = 1.0 / r
    ir2 = ir * ir
    return f[0] * ir, f[1] * ir, f[2] * ir2, f[3] * ir2


def static_scalars(r, med: Medium):                # [kernels.py:141-152]
    r = np.asarray(r, dtype=float)
    g2 = med.mu / (med.lam + 2.0 * med.mu)
    ir = 1.0 / r
    return (0.5 * (1.0 + g2) * ir, 0.5 * (g2 - 1.0) * ir,
            -0.5 * (1.0 + g2) * ir ** 2, 0.5 * (1.0 - g2) * ir ** 2)


# ----------------------------------------------------------------------
# pair geometry and weighted contraction          [kernels.py:292-357]
# ----------------------------------------------------------------------
def pair_geom(x, y, normal):                       # [kernels.py:196-203,292-298]
    """x (M,3) collocation, y (Q,3) field points -> r (M,Q), d (M,Q,3), d.n."""
    diff = np.asarray(y, dtype=float)[None, :, :] - np.asarray(x, dtype=float)[:, None, :]
    r = np.linalg.norm(diff, axis=-1)
    if np.any(r <= 0.0):
        raise ValueError("coincident source and field points")
    d = diff / r[..., None]
    return r, d, d @ np.asarray(normal, dtype=float)


def contract(f, r, d, dn, w, normal, med: Medium):  # [kernels.py:327-357]
    """Sum_q w_q U(x_m, y_q), Sum_q w_q T(x_m, y_q) -> two (M,3,3) arrays."""
    phi, psi, dphi, dpsi = f
    ratio = (med.lam + 2.0 * med.mu) / med.mu
    ir = 1.0 / r
    psr = psi * ir
    a = dphi - psr
    b = 2.0 * (2.0 * psr - dpsi)
    c = ratio * (dphi - dpsi - 2.0 * psr) - 2.0 * (dphi - dpsi - psr)
    wq = w[None, :]
    dt = d.astype(complex if np.iscomplexobj(phi) else float)
    eye = np.arange(3)
    # displacement kernel: (phi delta_ij - psi d_i d_j) / (4 pi mu)
    u_blk = -np.matmul(((psi * wq)[..., None] * d).swapaxes(-2, -1), dt)
    u_blk[:, eye, eye] += (phi * wq).sum(axis=1)[:, None]
    u_blk /= FOUR_PI * med.mu
    # traction kernel: a(delta dn + n_i d_j) + b dn d_i d_j + c d_i n_j
    aw = a * wq
    t_blk = np.matmul(((b * wq * dn)[..., None] * d).swapaxes(-2, -1), dt)
    va = np.matmul(aw[:, None, :], dt)[:, 0, :]
    vc = np.matmul((c * wq)[:, None, :], dt)[:, 0, :]
    t_blk += normal[None, :, None] * va[:, None, :]
    t_blk += vc[:, :, None] * normal[None, None, :]
    t_blk[:, eye, eye] += (aw * dn).sum(axis=1)[:, None]
    t_blk /= FOUR_PI
    return u_blk, t_blk


def blocks_dynamic(r, d, dn, w, normal, med, omega):   # [kernels.py:301-317]
    ks, kp = med.wavenumbers(omega)
    return contract(radial_scalars(r, ks, kp), r, d, dn, w, np.asarray(normal, float), med)


def blocks_static(r, d, dn, w, normal, med):           # [kernels.py:320-324]
    return contract(static_scalars(r, med), r, d, dn, w, np.asarray(normal, float), med)


# ----------------------------------------------------------------------
# dense assembly                                   [assembly.py:103-254]
# ----------------------------------------------------------------------
class DenseOracle:
    """Per-mesh pair data + per-frequency dense (T, U); reference Assembler."""

    def __init__(self, vertices, triangles, med: Medium, n_radial=8, n_angular=16):
        self.g = element_geometry(vertices, triangles)
        self.med = med
        self.n_e = len(triangles)
        self.n_radial, self.n_angular = n_radial, n_angular
        self._build()
        self._rowsums = None
        self._static = None

    def _build(self):                              # [assembly.py:122-171]
        g = self.g
        tier = tier_table(g["centroids"], g["diameters"])
        self.tiers = tier
        far, mid = rule_g3(), rule_g7()
        near_cache = {}
        xc = g["centroids"]
        self.cols, self.selfs = [], []
        self.near_levels = {}
        for j in range(self.n_e):
            vj = g["corners"][j]
            groups = []
            for tid, rule in ((0, far), (1, mid)):
                rows = np.flatnonzero(tier[:, j] == tid)
                rows = rows[rows != j]
                if rows.size:
                    groups.append((rows, rule))
            nr = np.flatnonzero(tier[:, j] == 2)
            nr = nr[nr != j]
            if nr.size:
                lv = near_level(surface_distance(xc[nr], vj) / g["diameters"][j])
                for i, l in zip(nr, lv):
                    self.near_levels[(int(i), j)] = int(l)
                for l in np.unique(lv):
                    if l not in near_cache:
                        near_cache[l] = rule_refine(rule_g7(), int(l))
                    groups.append((nr[lv == l], near_cache[l]))
            data = []
            for rows, (bary, wts) in groups:
                r, d, dn = pair_geom(xc[rows], bary @ vj, g["normals"][j])
                data.append((rows, wts * g["areas"][j], r, d, dn))
            self.cols.append(data)
            ys, ws = self_points(vj, self.n_radial, self.n_angular)
            r, d, dn = pair_geom(xc[j][None, :], ys, g["normals"][j])
            self.selfs.append((ws, r, d, dn))

    def _static_pass(self):                        # [assembly.py:193-216]
        n_e, g = self.n_e, self.g
        tm = np.zeros((n_e, 3, n_e, 3))
        um = np.zeros((n_e, 3, n_e, 3))
        for j in range(n_e):
            for rows, w, r, d, dn in self.cols[j]:
                ub, tb = blocks_static(r, d, dn, w, g["normals"][j], self.med)
                um[rows, :, j, :] = ub
                tm[rows, :, j, :] = tb
        self._rowsums = tm.sum(axis=2)
        for e in range(n_e):
            tm[e, :, e, :] = -self._rowsums[e]
            w, r, d, dn = self.selfs[e]
            um[e, :, e, :] = blocks_static(r, d, dn, w, g["normals"][e], self.med)[0][0]
        n = 3 * n_e
        self._static = (tm.reshape(n, n), um.reshape(n, n))

    def rowsums(self):
        if self._rowsums is None:
            self._static_pass()
        return self._rowsums

    def static_tu(self):
        if self._static is None:
            self._static_pass()
        return self._static

    def tu(self, omega):                           # [assembly.py:219-254]
        if omega == 0:
            ts, us = self.static_tu()
            return ts.astype(complex), us.astype(complex)
        n_e, g, med = self.n_e, self.g, self.med
        rs = self.rowsums()
        tm = np.zeros((n_e, 3, n_e, 3), dtype=complex)
        um = np.zeros((n_e, 3, n_e, 3), dtype=complex)
        for j in range(n_e):
            nj = g["normals"][j]
            for rows, w, r, d, dn in self.cols[j]:
                ub, tb = blocks_dynamic(r, d, dn, w, nj, med, omega)
                um[rows, :, j, :] = ub
                tm[rows, :, j, :] = tb
            w, r, d, dn = self.selfs[j]
            ud, td = blocks_dynamic(r, d, dn, w, nj, med, omega)
            _, ts = blocks_static(r, d, dn, w, nj, med)
            um[j, :, j, :] = ud[0]
            tm[j, :, j, :] = -rs[j] + (td[0] - ts[0])
        n = 3 * n_e
        t_out, u_out = tm.reshape(n, n), um.reshape(n, n)
        if not (np.isfinite(t_out).all() and np.isfinite(u_out).all()):
            raise FloatingPointError(f"non-finite entries assembled at omega = {omega}")
        return t_out, u_out


def sampled_row_operator(vertices, triangles, med, rows, omega, vectors_t, vectors_u,
                         n_radial=8, n_angular=16, col_block=2048):
    """Rows ``rows`` of T @ vt and U @ vu for meshes too large to assemble.

    Follows the same ladder as DenseOracle (assembly.py:122-171, 193-246)
    restricted to the sampled collocation rows, streaming over columns so
    nothing of size n_e^2 is stored.  ``vectors_*`` are (N, K) complex.
    Returns (Tv (3*len(rows), K), Uv (3*len(rows), K), rowsums (len(rows),3,3)).
    """
    g = element_geometry(vertices, triangles)
    rows = np.asarray(rows, dtype=np.int64)
    n_e = len(triangles)
    xc = g["centroids"]
    vt = np.asarray(vectors_t, dtype=complex).reshape(n_e, 3, -1)
    vu = np.asarray(vectors_u, dtype=complex).reshape(n_e, 3, -1)
    K = vt.shape[2]
    tv = np.zeros((len(rows), 3, K), dtype=complex)
    uv = np.zeros((len(rows), 3, K), dtype=complex)
    rsum = np.zeros((len(rows), 3, 3))
    far, mid = rule_g3(), rule_g7()
    near_cache = {}
    pos = {int(r): k for k, r in enumerate(rows)}
    diag_dyn = {}
    for j0 in range(0, n_e, col_block):
        js = np.arange(j0, min(n_e, j0 + col_block))
        tier = tiers_for_rows(xc, g["diameters"], rows, js)
        for jj, j in enumerate(js):
            vj = g["corners"][j]
            nj = g["normals"][j]
            groups = []
            for tid, rule in ((0, far), (1, mid)):
                sel = np.flatnonzero((tier[:, jj] == tid) & (rows != j))
                if sel.size:
                    groups.append((sel, rule))
            sel = np.flatnonzero((tier[:, jj] == 2) & (rows != j))
            if sel.size:
                lv = near_level(surface_distance(xc[rows[sel]], vj) / g["diameters"][j])
                for l in np.unique(lv):
                    if l not in near_cache:
                        near_cache[l] = rule_refine(rule_g7(), int(l))
                    groups.append((sel[lv == l], near_cache[l]))
            for sel, (bary, wts) in groups:
                r, d, dn = pair_geom(xc[rows[sel]], bary @ vj, nj)
                w = wts * g["areas"][j]
                ub, tb = blocks_dynamic(r, d, dn, w, nj, med, omega)
                _, tsb = blocks_static(r, d, dn, w, nj, med)
                rsum[sel] += tsb
                tv[sel] += np.einsum("mab,bk->mak", tb, vt[j])
                uv[sel] += np.einsum("mab,bk->mak", ub, vu[j])
            if int(j) in pos:
                ys, ws = self_points(vj, n_radial, n_angular)
                r, d, dn = pair_geom(xc[j][None, :], ys, nj)
                ud, td = blocks_dynamic(r, d, dn, ws, nj, med, omega)
                _, ts = blocks_static(r, d, dn, ws, nj, med)
                diag_dyn[int(j)] = (ud[0], td[0] - ts[0])
    for k, i in enumerate(rows):
        ud, tdiff = diag_dyn[int(i)]
        tdiag = -rsum[k] + tdiff
        tv[k] += tdiag @ vt[i]
        uv[k] += ud @ vu[i]
    return tv.reshape(-1, K), uv.reshape(-1, K), rsum


def column_sample_seconds(vertices, triangles, med, cols, omega, n_radial=8, n_angular=16):
    """CPU seconds the reference algorithm spends on the columns ``cols``.

    Runs, for the sampled columns only, exactly the per-column work of
    DenseOracle: bucket/pair-geometry prep (assembly.py:142-171), the static
    integrals (assembly.py:197-203) and one dynamic assembly at ``omega``
    (assembly.py:233-246).  Used by bench.py to extrapolate a full-sweep CPU
    time (per-column cost x n_e) without holding the O(n_e^2) pair data.
    Returns dict(prep=, static=, dynamic=) seconds for the sample.
    """
    g = element_geometry(vertices, triangles)
    xc = g["centroids"]
    far, mid = rule_g3(), rule_g7()
    near_cache = {}
    t0 = time.perf_counter()
    tier = tiers_for_rows(xc, g["diameters"], np.arange(len(triangles)), np.asarray(cols))
    data = []
    for jj, j in enumerate(cols):
        vj = g["corners"][j]
        groups = []
        for tid, rule in ((0, far), (1, mid)):
            rows = np.flatnonzero(tier[:, jj] == tid)
            rows = rows[rows != j]
            if rows.size:
                groups.append((rows, rule))
        nr = np.flatnonzero(tier[:, jj] == 2)
        nr = nr[nr != j]
        if nr.size:
            lv = near_level(surface_distance(xc[nr], vj) / g["diameters"][j])
            for l in np.unique(lv):
                if l not in near_cache:
                    near_cache[l] = rule_refine(rule_g7(), int(l))
                groups.append((nr[lv == l], near_cache[l]))
        buckets = []
        for rows, (bary, wts) in groups:
            r, d, dn = pair_geom(xc[rows], bary @ vj, g["normals"][j])
            buckets.append((rows, wts * g["areas"][j], r, d, dn))
        ys, ws = self_points(vj, n_radial, n_angular)
        r, d, dn = pair_geom(xc[j][None, :], ys, g["normals"][j])
        data.append((j, buckets, (ws, r, d, dn)))
    t1 = time.perf_counter()
    for j, buckets, _ in data:
        for rows, w, r, d, dn in buckets:
            blocks_static(r, d, dn, w, g["normals"][j], med)
    t2 = time.perf_counter()
    for j, buckets, (ws, r, d, dn) in data:
        nj = g["normals"][j]
        for rows, w, rr, dd, ddn in buckets:
            blocks_dynamic(rr, dd, ddn, w, nj, med, omega)
        blocks_dynamic(r, d, dn, ws, nj, med, omega)
        blocks_static(r, d, dn, ws, nj, med)
    t3 = time.perf_counter()
    return dict(prep=t1 - t0, static=t2 - t1, dynamic=t3 - t2)


# ----------------------------------------------------------------------
# boundary conditions                              [assembly.py:263-305]
# ----------------------------------------------------------------------
def apply_bcs(t_mat, u_mat, kinds, prescribed):
    kinds = np.asarray(kinds).reshape(-1)
    n = len(kinds)
    if t_mat.shape != (n, n) or u_mat.shape != (n, n):
        raise ValueError("matrix/BC size mismatch")
    p = np.asarray(prescribed, dtype=complex)
    if p.shape != (n,):
        raise ValueError("prescribed spectrum has wrong length")
    if not np.isfinite(p).all():
        raise ValueError("unresolved (non-finite) prescribed boundary value")
    dmask = kinds == DIRICHLET
    nmask = ~dmask
    a = np.empty((n, n), dtype=complex)
    a[:, nmask] = t_mat[:, nmask]
    a[:, dmask] = -u_mat[:, dmask]
    b = u_mat[:, nmask] @ p[nmask]
    b -= t_mat[:, dmask] @ p[dmask]
    return a, b


def scatter_solution(kinds, a, prescribed):
    kinds = np.asarray(kinds).reshape(-1)
    return (np.where(kinds == NEUMANN, a, prescribed),
            np.where(kinds == DIRICHLET, a, prescribed))


# ----------------------------------------------------------------------
# linear solvers                                   [linsolve.py:51-242]
# ----------------------------------------------------------------------
@dataclass
class Stats:
    k: int = -1
    omega: complex = 0.0
    iterations: int = 0
    init_residual: float = 0.0
    final_residual: float = 0.0
    seconds: float = 0.0
    converged: bool = True
    residual_history: list = field(default_factory=list, repr=False)


class History:                                     # [linsolve.py:51-70]
    def __init__(self, capacity):
        if capacity < 1:
            raise ValueError("history capacity must be >= 1")
        self.q = deque(maxlen=capacity)

    def push(self, x):
        self.q.appendleft(np.array(x, dtype=complex, copy=True))

    def __len__(self):
        return len(self.q)

    def matrix(self):
        if not self.q:
            raise ValueError("empty solution history")
        return np.stack(list(self.q), axis=1)


def _operator(a):                                  # [linsolve.py:73-77]
    if callable(a):
        return a
    m = np.asarray(a)
    return lambda v: m @ v


def block_precond(a_mat):                          # [linsolve.py:80-104]
    n = a_mat.shape[0]
    if a_mat.shape != (n, n) or n % 3:
        raise ValueError("matrix must be square with size divisible by 3")
    nb = n // 3
    inv = np.empty((nb, 3, 3), dtype=complex)
    for i in range(nb):
        blk = a_mat[3 * i:3 * i + 3, 3 * i:3 * i + 3]
        try:
            inv[i] = np.linalg.inv(blk)
        except np.linalg.LinAlgError:
            inv[i] = np.eye(3)
    return (lambda v: np.einsum("bij,bj->bi", inv, v.reshape(nb, 3)).reshape(n)), inv


def gmres(apply_a, b, x0=None, tol=1e-5, restart=60, maxiter=1000, precond=None):
    """Right-preconditioned restarted GMRES, MGS + complex Givens [linsolve.py:107-210]."""
    t0 = time.perf_counter()
    mv = _operator(apply_a)
    pc = precond if precond is not None else (lambda v: v)
    b = np.asarray(b, dtype=complex)
    n = b.shape[0]
    if not 0.0 < tol < 1.0:
        raise ValueError(f"tol must be in (0, 1), got {tol}")
    nb = np.linalg.norm(b)
    st = Stats()
    if nb == 0.0:
        st.seconds = time.perf_counter() - t0
        return np.zeros(n, dtype=complex), st
    x = np.zeros(n, dtype=complex) if x0 is None else np.array(x0, dtype=complex, copy=True)
    r = b - mv(x) if x.any() else b.copy()
    res = np.linalg.norm(r) / nb
    st.init_residual = res
    st.residual_history.append(res)
    its = 0
    while res > tol and its < maxiter:
        m = min(restart, maxiter - its)
        V = np.empty((m + 1, n), dtype=complex)
        H = np.zeros((m + 1, m), dtype=complex)
        cs = np.zeros(m, dtype=complex)
        sn = np.zeros(m, dtype=complex)
        beta = np.linalg.norm(r)
        V[0] = r / beta
        g = np.zeros(m + 1, dtype=complex)
        g[0] = beta
        used = 0
        for j in range(m):
            w = mv(pc(V[j]))
            for i in range(j + 1):
                H[i, j] = np.vdot(V[i], w)
                w -= H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] > 0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                top = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + np.conj(cs[i]) * H[i + 1, j]
                H[i, j] = top
            den = np.sqrt(abs(H[j, j]) ** 2 + abs(H[j + 1, j]) ** 2)
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            elif H[j, j] == 0.0:
                cs[j], sn[j] = 0.0, 1.0
            else:
                cs[j] = abs(H[j, j]) / den
                sn[j] = (H[j, j] / abs(H[j, j])) * np.conj(H[j + 1, j]) / den
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            used = j + 1
            est = abs(g[j + 1]) / nb
            st.residual_history.append(est)
            if est <= tol:
                break
        y = np.zeros(used, dtype=complex)
        for i in range(used - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:used] @ y[i + 1:used]) / H[i, i]
        x = x + pc(V[:used].T @ y)
        r = b - mv(x)
        res = np.linalg.norm(r) / nb
    st.iterations = its
    st.final_residual = res
    st.converged = res <= tol
    st.seconds = time.perf_counter() - t0
    return x, st


def sem_guess(history: History, apply_a, b, rank_tol=1e-10):   # [linsolve.py:213-242]
    mv = _operator(apply_a)
    X = history.matrix()
    Y = np.stack([mv(X[:, i]) for i in range(X.shape[1])], axis=1)
    keep = np.arange(X.shape[1])
    for _ in range(2):
        q, rr = np.linalg.qr(Y[:, keep])
        dg = np.abs(np.diag(rr))
        good = dg >= rank_tol * dg.max() if dg.max() > 0 else dg > 0
        if good.all():
            s = np.linalg.solve(rr, q.conj().T @ b)
            return (X[:, keep] @ s).astype(complex)
        keep = keep[good]
        if keep.size == 0:
            break
    return X[:, 0].copy()


# ----------------------------------------------------------------------
# spectral pipeline                                [transform.py:113-211]
# ----------------------------------------------------------------------
def eta_from_kappa(kappa, period):
    return kappa * math.log(10.0) / period


def frequency_grid(period, n_omega, eta):
    dw = 2.0 * math.pi / period
    return np.arange(n_omega // 2 + 1) * dw - 1j * eta


def forward_spectrum(samples, period, eta):        # [transform.py:122-134]
    n = len(samples)
    dt = period / n
    return np.fft.fft(np.asarray(samples, float) * np.exp(-eta * dt * np.arange(n))) / n


def conjugate_fill(half):                          # [transform.py:137-154]
    half = np.asarray(half, dtype=complex)
    nh = half.size
    n = 2 * (nh - 1)
    full = np.empty(n, dtype=complex)
    full[:nh] = half
    full[0] = half[0].real
    full[nh - 1] = half[nh - 1].real
    full[nh:] = np.conj(full[1:n - nh + 1][::-1])
    return full


def window(kind, n):                               # [transform.py:157-176]
    if kind == "rectangular":
        return np.ones(n)
    ph = 2.0 * math.pi * np.arange(n) / n
    if kind == "hanning":
        return 0.5 * (1.0 + np.cos(ph))
    if kind == "blackman":
        return 0.42 + 0.5 * np.cos(ph) + 0.08 * np.cos(2.0 * ph)
    raise ValueError(kind)


def inverse_transform(full, kind, eta, period):    # [transform.py:179-203]
    """Returns (real samples, imaginary-residue ratio)."""
    n = len(full)
    sig = np.fft.ifft(full * window(kind, n)) * n
    scale = np.abs(sig).max()
    residue = np.abs(sig.imag).max() / scale if scale > 0 else 0.0
    dt = period / n
    return sig.real * np.exp(eta * dt * np.arange(n)), residue


# ----------------------------------------------------------------------
# the sweep                                        [driver.py:92-176]
# ----------------------------------------------------------------------
def sweep(vertices, triangles, med, kinds, dof_signal, signal_samples, probes,
          period, n_omega, kappa, window_kind="hanning", sem_depth=4, sem=True,
          tol=1e-5, restart=60, maxiter=1000):
    """Sequential sweep as run_sweep with workers=1.

    ``signal_samples`` (n_signals, n_omega) time samples; ``dof_signal``
    (N,) signal index per DOF; ``probes`` list of (name, dof, quantity).
    Returns (times, histories dict, stats list, half spectra dict).
    """
    eta = eta_from_kappa(kappa, period)
    om = frequency_grid(period, n_omega, eta)
    nf = len(om)
    spectra = np.stack([forward_spectrum(s, period, eta)[:nf] for s in signal_samples])
    asm = DenseOracle(vertices, triangles, med)
    asm.rowsums()
    hist = History(sem_depth) if sem else None
    probe_half = np.empty((len(probes), nf), dtype=complex)
    stats = []
    kinds = np.asarray(kinds).reshape(-1)
    for k in range(nf):
        tm, um = asm.tu(om[k])
        p = spectra[np.asarray(dof_signal), k]
        a_mat, b = apply_bcs(tm, um, kinds, p)
        x0 = sem_guess(hist, a_mat, b) if hist is not None and len(hist) else None
        pc, _ = block_precond(a_mat)
        a, st = gmres(a_mat, b, x0=x0, tol=tol, restart=restart, maxiter=maxiter, precond=pc)
        st.k, st.omega = k, om[k]
        stats.append(st)
        u, t = scatter_solution(kinds, a, p)
        for i, (_, dof, q) in enumerate(probes):
            probe_half[i, k] = u[dof] if q == "displacement" else t[dof]
        if hist is not None:
            hist.push(a)
    failed = [s.k for s in stats if not s.converged]
    times = np.arange(n_omega) * (period / n_omega)
    hists, halves = {}, {}
    for i, (name, _, _) in enumerate(probes):
        halves[name] = probe_half[i].copy()
        series, _ = inverse_transform(conjugate_fill(probe_half[i]), window_kind, eta, period)
        hists[name] = np.full_like(series, np.nan) if failed else series
    return times, hists, stats, halves
