"""Boundary densities rho_in, rho_f as coarse cell averages (input generation).

PAPER.md P:174-187 defines rho^0 and rho^{K+1} as cell averages of rho_in and
rho_f.  SURVEY §8(c) A21 fixes how the harness computes them so that both
implementations receive identical bytes: a fixed degree-5 7-point triangle
rule (Dunavant), then a scaling to unit discrete mass  sum_j |c_j| rho_j = 1
(|Omega| = 1), applied to both ends.
"""
from __future__ import annotations

import numpy as np

from .mesh import triangle_areas

_S15 = np.sqrt(15.0)
# Degree-5 7-point rule on the reference triangle (barycentric coords, weights sum 1).
_B1 = (6.0 - _S15) / 21.0
_B2 = (6.0 + _S15) / 21.0
_W1 = (155.0 - _S15) / 1200.0
_W2 = (155.0 + _S15) / 1200.0
QUAD_BARY = np.array([
    [1 / 3, 1 / 3, 1 / 3],
    [1 - 2 * _B1, _B1, _B1], [_B1, 1 - 2 * _B1, _B1], [_B1, _B1, 1 - 2 * _B1],
    [1 - 2 * _B2, _B2, _B2], [_B2, 1 - 2 * _B2, _B2], [_B2, _B2, 1 - 2 * _B2],
])
QUAD_W = np.array([9 / 40, _W1, _W1, _W1, _W2, _W2, _W2])


def cell_average(f, verts, tris):
    """(1/|T|) * integral_T f  for every triangle, with the 7-point rule."""
    p = np.asarray(verts)[np.asarray(tris)]            # (nt, 3, 2)
    x = np.einsum("qk,tkd->tqd", QUAD_BARY, p)         # (nt, 7, 2)
    vals = f(x[..., 0], x[..., 1])
    return vals @ QUAD_W


def gaussian(x0, y0, sigma, weight=1.0):
    def f(x, y):
        return weight * np.exp(-((x - x0) ** 2 + (y - y0) ** 2) / (2.0 * sigma ** 2))
    return f


def cos2_bump(x0, y0, radius):
    """cos^2(pi r / (2 radius)) for r < radius, 0 elsewhere (compact support)."""
    def f(x, y):
        r = np.sqrt((x - x0) ** 2 + (y - y0) ** 2)
        return np.where(r < radius, np.cos(np.pi * r / (2.0 * radius)) ** 2, 0.0)
    return f


def mixture(fs, floor=0.0):
    def f(x, y):
        out = np.full(np.broadcast(x, y).shape, floor, dtype=np.float64)
        for g in fs:
            out = out + g(x, y)
        return out
    return f


def normalise_mass(rho, verts, tris, mass=1.0):
    area = triangle_areas(verts, tris)
    return rho * (mass / float(area @ rho))
