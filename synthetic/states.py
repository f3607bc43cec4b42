"""Seeded synthetic IPM states for single-solve parity (input generation).

`initial_state` is the A19 starting point: rho^k uniform with the
boundary mass, s = mu0 / rho, phi = 0.  `random_state` perturbs it smoothly so a
Newton system has nonzero grad(phi) and a nonuniform rho; every random number
is drawn here with numpy PCG64 and passed to both implementations as data.
"""
from __future__ import annotations

import numpy as np

from .mesh import triangle_areas


def initial_state(prob, mu0: float = 1.0):
    nbar, K = prob.nbar, prob.K
    area = triangle_areas(prob.verts, prob.tris)
    mass = float(area @ prob.rho_in)
    rho = np.full(nbar * K, mass / float(area.sum()))
    s = mu0 / rho
    phi = np.zeros(3 * nbar * (K + 1))
    return phi, rho, s


def random_state(prob, seed: int = 0, mu: float = 1e-2, phi_amp: float = 0.3,
                 rho_amp: float = 0.5):
    """A smooth, strictly positive, mass-conserving state with s = mu/rho * (1+noise).

    phi: a smooth travelling wave sampled at the fine-cell *coarse centroids*
    (each coarse triangle's 3 kites get the same base value plus small seeded
    noise); rho: the linear-in-time interpolation of rho_in/rho_f times a seeded
    smooth modulation, then rescaled per slice to the boundary mass.
    """
    rng = np.random.default_rng(seed)
    nbar, K = prob.nbar, prob.K
    v, t = prob.verts, prob.tris
    area = triangle_areas(v, t)
    cen = v[t].mean(axis=1)                      # (nbar, 2)
    a = rng.uniform(0.5, 1.5, size=4)
    ph = rng.uniform(0, 2 * np.pi, size=3)
    phi = np.empty((K + 1, nbar, 3))
    for k in range(K + 1):
        tk = (k + 0.5) / (K + 1)
        base = phi_amp * (a[0] * (cen[:, 0] - 0.5) * np.cos(ph[0] + tk)
                          + a[1] * (cen[:, 1] - 0.5) * np.sin(ph[1] + 2 * tk)
                          + 0.2 * a[2] * np.sin(2 * np.pi * cen[:, 0] + ph[2]) * tk)
        phi[k] = base[:, None] + 0.01 * phi_amp * rng.standard_normal((nbar, 3))
    mass = float(area @ prob.rho_in)
    rho = np.empty((K, nbar))
    for k in range(1, K + 1):
        tk = k / (K + 1)
        r = (1 - tk) * prob.rho_in + tk * prob.rho_f
        mod = 1.0 + rho_amp * 0.5 * (1 + np.sin(3 * cen[:, 0] + 2 * cen[:, 1] + a[3] * k))
        r = np.maximum(r, 1e-3 * r.max()) * mod
        rho[k - 1] = r * (mass / float(area @ r))
    rho = rho.reshape(-1)
    s = (mu / rho) * (1.0 + 0.3 * rng.uniform(-1, 1, size=rho.shape))
    return phi.reshape(-1), rho, s
