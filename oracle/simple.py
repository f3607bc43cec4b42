"""NEXT row (f) rank 1: the SIMPLE preconditioner (§5.3) on the
reduced saddle-point system (eq:saddle-point), and its recovery.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Saddle-point system, δs eliminated by δs = ρ^{-1}(h - s δρ):
    J = [[A, B^T], [B, -C]],  rhs (f; g̃),  C = M̄ diag(s/ρ) (A7),  g̃ = g - M̄ h/ρ.
SIMPLE (eq:sca-precs):
    P^{-1} = [[I, -Ã^{-1} B^T], [0, I]] · diag(Ã^{-1}, S̃^{-1}) · [[I, 0], [-B Ã^{-1}, I]]
    Ã = diag(A),  S̃ = -(C + B Ã^{-1} B^T)                          (A31)
so on (r1; r2):
    z1 = Ã^{-1} r1;  z2 = S̃^{-1}(r2 - B z1);  x1 = z1 - Ã^{-1} B^T z2 = Ã^{-1}(r1 - B^T z2).
S̃ z2 = c is solved as Ŝ z2 = -c with Ŝ = -S̃ = C + B Ã^{-1} B^T (SPD, block tridiagonal in
time, "formed explicitly"), by the inner solver of the T system: GMRES(restart_T)
right-preconditioned by one AMG V-cycle (mode T, l1-Jacobi, aggregation across time slices
as AGMG's, dense coarsest <= coarse_max_S = 256 rows), relative eps_in = 1e-1,
cap maxit_inner (A32).  Outer: FGMRES(restart)
on J, stopping at eps_out ||(f;g;h)||.  Recovery: δφ = x1, δρ = x2, δs = ρ^{-1}(h - s δρ).

Pins (tests/test_oracle_simple.py): with an exact Ŝ solve, P^{-1} inverts
J̃ = [[diag(A), B^T], [B, -C]] exactly (the block factorisation multiplies out to J̃);
Ŝ is symmetric positive definite; the SIMPLE direction equals the dense direct solve of
(3.1) (oracle/direct.py) up to the kernel <(1;0;0)> of Remark 3.1; the converged SIMPLE
and BB directions agree.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import amg
from .bb import SolverOpts
from .krylov import fgmres
from .ops import Discretisation


def S_hat(d: Discretisation, phi, rho, s):
    """Ŝ = C + B diag(A)^{-1} B^T  (= -S̃, P:994-998 with A31)."""
    A = d.A(rho)
    B = d.B(phi)
    C = d.C_diag(rho, s)
    return (sp.diags(C) + B @ sp.diags(1.0 / A.diagonal()) @ B.T).tocsr()


class SimpleSolver:
    """Per-Newton-step setup + FGMRES solve on (eq:saddle-point) + recovery."""

    def __init__(self, disc: Discretisation, phi, rho, s, mu, opts: SolverOpts | None = None):
        self.d = d = disc
        self.o = o = opts or SolverOpts()
        self.phi, self.rho, self.s, self.mu = (np.asarray(phi, float), np.asarray(rho, float),
                                               np.asarray(s, float), float(mu))
        self.f, self.g, self.h, self.gt = d.newton_rhs(phi, rho, s, mu)
        self.scale = float(np.sqrt(self.f @ self.f + self.g @ self.g + self.h @ self.h))
        self.rhs = np.concatenate([self.f, self.gt])
        assert d.recon == "arith", "SIMPLE: arithmetic reconstruction only (the harmonic R_H is built for BB)"
        self.A = d.A(rho)
        self.B = d.B(phi)
        self.BT = self.B.T.tocsr()
        self.C = d.C_diag(rho, s)
        self.dA = self.A.diagonal()
        self.S = S_hat(d, phi, rho, s)
        self.inner_its = 0
        if o.exact_inner:
            self.Sinv = np.linalg.inv(self.S.toarray())
        else:
            # A32: one "slice" -- AMG(Ŝ) aggregates across time as well (at φ = 0, B is the
            # pure time difference and Ŝ has no in-slice couplings at all)
            self.amgS = amg.setup(self.S, np.zeros(d.m, dtype=np.int64), "T", o.omega_T, o.coarse_max_S)

    def matvec(self, v):
        """J v = (A x + B^T y; B x - C y)."""
        n = self.d.n
        x, y = v[:n], v[n:]
        return np.concatenate([self.A @ x + self.BT @ y, self.B @ x - self.C * y])

    def apply(self, r):
        """P^{-1} r, eq:sca-precs."""
        o = self.o
        n = self.d.n
        r1, r2 = r[:n], r[n:]
        z1 = r1 / self.dA
        c = self.B @ z1 - r2                       # = -(r2 - B z1)
        if o.exact_inner:
            z2 = self.Sinv @ c
        else:
            z2, its, _, _ = fgmres(lambda v: self.S @ v, lambda v: amg.vcycle(self.amgS, v),
                                   c, float(np.linalg.norm(c)), o.eps_T, o.restart_T, o.maxit_inner)
            self.inner_its += its
        x1 = (r1 - self.BT @ z2) / self.dA
        return np.concatenate([x1, z2])

    def solve(self):
        o = self.o
        sol, its, conv, res = fgmres(self.matvec, self.apply, self.rhs, self.scale,
                                     o.eps_out, o.restart, o.maxit)
        self.stats = dict(outer_its=its, converged=bool(conv), rel_res=res / self.scale,
                          inner_T_its=self.inner_its, inner_A_its_max=0, inner_A_its_total=0)
        self.sol = sol
        return self.recover(sol)

    def recover(self, sol):
        n = self.d.n
        dphi = sol[:n].copy()
        drho = sol[n:].copy()
        ds = (self.h - self.s * drho) / self.rho
        return dphi, drho, ds
