"""Dense direct solve of the Newton system (3.1) for tiny instances.

The Jacobian is singular with kernel <(1;0;0)> (Remark 3.1); the
system is consistent when the slice masses are equal (Remark 2.2).  We take the
least-squares (minimum-norm) solution and fix the gauge as A11: δφ^1 has zero
c-weighted mean (the same constant is removed from every φ slice, which is the
kernel direction).  Used only as a pin for the iterative path.
"""
from __future__ import annotations

import numpy as np

from .ops import Discretisation


def direct_newton(d: Discretisation, phi, rho, s, mu):
    J = d.jacobian(phi, rho, s).toarray()
    f, g, h, _ = d.newton_rhs(phi, rho, s, mu)
    rhs = np.concatenate([f, g, h])
    sol, *_ = np.linalg.lstsq(J, rhs, rcond=None)
    n, m = d.n, d.m
    dphi = sol[:n].reshape(d.K + 1, d.N)
    dphi = dphi - (dphi[0] @ d.M) / d.area
    return dphi.reshape(-1), sol[n:n + m], sol[n + m:], J, rhs
