"""Direct solve of the Newton system (3.1) for tiny instances.

The Jacobian is singular with kernel <(1;0;0)> (Remark 3.1), and its left
kernel is (1;0;0) too (the φ rows sum to zero over all slices: 1ᵀA = 0 and Bᵀ's time part
telescopes); the system is consistent when the slice masses are equal (Remark 2.2).  We
take the minimum-norm solution -- the one orthogonal to the kernel -- from the bordered
system [[J, v], [vᵀ, 0]] (x; λ) = (rhs; 0), v = (1;0;0), which is nonsingular because
vᵀv ≠ 0 (kernel not orthogonal to the border, border not in the range of J); for a
consistent right-hand side λ = 0 and x = the least-squares minimum-norm solution.  Then
the gauge is fixed as A11: δφ^1 has zero c-weighted mean (the same constant is removed
from every φ slice, the kernel direction).  Used only as a pin for the iterative path.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .ops import Discretisation


def direct_newton(d: Discretisation, phi, rho, s, mu):
    J = d.jacobian(phi, rho, s).tocsr()
    f, g, h, _ = d.newton_rhs(phi, rho, s, mu)
    rhs = np.concatenate([f, g, h])
    n, m = d.n, d.m
    v = np.r_[np.ones(n), np.zeros(2 * m)]
    Jb = sp.bmat([[J, sp.csr_matrix(v[:, None])], [sp.csr_matrix(v[None, :]), None]], format="csc")
    sol = spla.spsolve(Jb, np.r_[rhs, 0.0])[:-1]
    dphi = sol[:n].reshape(d.K + 1, d.N)
    dphi = dphi - (dphi[0] @ d.M) / d.area
    return dphi.reshape(-1), sol[n:n + m], sol[n + m:], J, rhs
