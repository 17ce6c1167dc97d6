"""Quadrature rule tables uploaded to the device context.

Tables only — rule *generation* is host setup ("table
generation can stay on host"); every integration runs on the GPU.  The
barycentric points and weights are built with the same formulas as the
reference (``quadrature.py:63-132``) so they agree bit-for-bit (checked in
``tests/test_host.py::test_device_rule_tables_bitwise`` against the golden fixtures).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class TriangleRule:
    name: str
    points: np.ndarray   # (Q, 3) barycentric
    weights: np.ndarray  # (Q,) summing to 1
    degree: int

    @property
    def n_points(self) -> int:
        return len(self.weights)

    def mapped(self, verts: np.ndarray) -> np.ndarray:
        return self.points @ verts


def gauss3() -> TriangleRule:
    a, b = 2 / 3, 1 / 6
    pts = np.array([[a, b, b], [b, a, b], [b, b, a]])
    return TriangleRule("gauss3", pts, np.full(3, 1 / 3), degree=2)


def gauss7() -> TriangleRule:
    r = np.sqrt(15.0)
    p1, p2 = (6.0 + r) / 21.0, (6.0 - r) / 21.0
    w1, w2 = (155.0 + r) / 1200.0, (155.0 - r) / 1200.0
    pts, wts = [[1 / 3, 1 / 3, 1 / 3]], [9.0 / 40.0]
    for v, w in ((p1, w1), (p2, w2)):
        o = 1 - 2 * v
        pts += [[v, v, o], [v, o, v], [o, v, v]]
        wts += [w] * 3
    return TriangleRule("gauss7", np.array(pts), np.array(wts), degree=5)


def subdivided(rule: TriangleRule, levels: int = 1) -> TriangleRule:
    """The base rule on each of the 4**levels congruent midpoint children."""
    kids = [np.eye(3)]
    for _ in range(levels):
        nxt = []
        for t in kids:
            a, b, c = (t[0] + t[1]) / 2, (t[1] + t[2]) / 2, (t[2] + t[0]) / 2
            nxt += [np.array([t[0], a, c]), np.array([a, t[1], b]),
                    np.array([c, b, t[2]]), np.array([a, b, c])]
        kids = nxt
    frac = 1.0 / len(kids)
    return TriangleRule(f"{rule.name}-sub{levels}",
                        np.concatenate([rule.points @ t for t in kids]),
                        np.concatenate([rule.weights * frac for _ in kids]),
                        degree=rule.degree)


@dataclass(frozen=True)
class QuadratureSet:
    """The reference's default ladder (``quadrature.py:189-214``).

    far d >= 4: gauss3; mid 1.5 <= d < 4: gauss7; near d < 1.5: gauss7 on
    1..4 midpoint subdivisions graded by separation/diameter < 0.60, 0.30,
    0.15; self: 3 x 8 x 16 Duffy/asinh.  Only this ladder is compiled into
    the device kernels.
    """

    far_threshold: float = 4.0
    near_threshold: float = 1.5
    near_grading: tuple = (0.60, 0.30, 0.15)
    duffy_radial: int = 8
    duffy_angular: int = 16

    @classmethod
    def default(cls) -> "QuadratureSet":
        return cls()

    def classify(self, d: np.ndarray) -> np.ndarray:
        out = np.zeros(np.shape(d), dtype=np.uint8)
        out[d < self.far_threshold] = 1
        out[d < self.near_threshold] = 2
        return out

    def near_level(self, s: np.ndarray) -> np.ndarray:
        lvl = np.ones(np.shape(s), dtype=np.int64)
        for thr in self.near_grading:
            lvl[s < thr] += 1
        return lvl


def device_rule_tables():
    """(rules flat float64, offsets int32[7], Q int32[7]) for ewb_ctx_create.

    Order: gauss3, gauss7, gauss7-sub1..sub4; each table is bary (Q,3)
    followed by weights (Q,).
    """
    rules = [gauss3(), gauss7()] + [subdivided(gauss7(), L) for L in range(1, 5)]
    flat, off, q = [], [], []
    pos = 0
    for r in rules:
        off.append(pos)
        q.append(r.n_points)
        flat.append(np.ascontiguousarray(r.points, dtype=np.float64).ravel())
        flat.append(np.ascontiguousarray(r.weights, dtype=np.float64))
        pos += 4 * r.n_points
    off.append(pos)
    q.append(0)
    return (np.concatenate(flat), np.array(off, dtype=np.int32), np.array(q, dtype=np.int32))


def gauss_legendre_tables(n_radial=8, n_angular=16):
    xr, wr = np.polynomial.legendre.leggauss(n_radial)
    xa, wa = np.polynomial.legendre.leggauss(n_angular)
    return (np.concatenate([xr, wr]).astype(np.float64),
            np.concatenate([xa, wa]).astype(np.float64))
