"""NEXT row (f) rank 2: the HSS preconditioner (§5.1) on the reduced
saddle-point system, and its recovery.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

System.  The skew form (eq:saddle-point-skew) of the saddle-point system
(eq:saddle-point; δs eliminated by P:506):
    J_skew = [[A, B^T], [-B, C]],  rhs (f; -g̃),  C = M̄ diag(s/ρ) (A7).
J_skew = S J with S = diag(I, -I) and J = [[A, B^T], [B, -C]], so FGMRES on J with the
right preconditioner M^{-1}_skew S produces the same iterates and residual norms (S is an
isometry) -- the outer solve is SIMPLE's (A33): FGMRES(restart) on J, rhs (f; g̃), stop at
eps_out ||(f;g;h)||; recovery δφ = x1, δρ = x2, δs.  (A36)

Diagonal scaling ("we apply this preconditioner after scaling the linear system
in eq:saddle-point-skew by its diagonal"): D = diag(diag(A), C) (both positive),
    Ĵ = D^{-1/2} J_skew D^{-1/2} = [[Â, B̂^T], [-B̂, I]],  Â = D_A^{-1/2} A D_A^{-1/2},
    B̂ = D_C^{-1/2} B D_A^{-1/2}.
HSS (eq:prec-hss, eq:hss-hk), factors in the paper's reversed order:
    P^{-1} = H_α^{-1} K_α^{-1},  H_α = blkdiag(Â + αI, I + αI),  K_α = [[αI, B̂^T], [-B̂, αI]],
so M^{-1}_skew = D^{-1/2} H_α^{-1} K_α^{-1} D^{-1/2} (the HSS preconditioner of Ĵ carried back
to J_skew: J_skew M^{-1}_skew = D^{1/2} Ĵ P^{-1} D^{-1/2}, similar to Ĵ P^{-1}).
K_α^{-1} by its dual Schur complement (eq:solve-K, "turned out to be more
efficient"): for K_α (u; v) = (a; b):
    (αI + B̂B̂^T/α) v = b + B̂ a/α,   u = (a - B̂^T v)/α.
H_α^{-1}: the K+1 shifted Laplacian systems (Â_k + αI) x^k = u^k (eq:solve-laplacians,
P:690-694) and the diagonal (1+α)^{-1}.
Inner solves (AGMG, α = 0.5, ε_in = 1e-1): per-slice PCG + one V-cycle of
AMG(Â + αI) (I3, mode "As": per-slice aggregation, damped Jacobi, nonsingular per-slice
coarsest) to relative ε_in; (αI + B̂B̂^T/α) -- SPD, block tridiagonal in time like SIMPLE's
Ŝ -- by GMRES(restart_T) + one V-cycle of AMG (mode T, aggregation across time as
A32), relative ε_in; caps maxit_inner.  (A37)

Pins (tests/test_oracle_hss.py): the HSS splitting H_α + K_α = Ĵ + 2αI (Bai-Golub-Ng);
with exact inner solves the apply equals D^{-1/2}(K_α H_α)^{-1} D^{-1/2} S (the Schur route
is the inverse of K_α); the spectrum of 2α (K_α H_α)^{-1} Ĵ lies in the disk |λ - 1| <= 1
(HSS contraction: Ĵ's Hermitian part blkdiag(Â, I) is PSD); the HSS direction equals the
dense direct solve of (3.1).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import amg
from .bb import SolverOpts
from .krylov import fgmres, pcg_slices
from .ops import Discretisation


class HssSolver:
    """Per-Newton-step setup + FGMRES solve on (eq:saddle-point) with HSS + recovery."""

    def __init__(self, disc: Discretisation, phi, rho, s, mu, opts: SolverOpts | None = None):
        self.d = d = disc
        self.o = o = opts or SolverOpts()
        self.phi, self.rho, self.s, self.mu = (np.asarray(phi, float), np.asarray(rho, float),
                                               np.asarray(s, float), float(mu))
        self.f, self.g, self.h, self.gt = d.newton_rhs(phi, rho, s, mu)
        self.scale = float(np.sqrt(self.f @ self.f + self.g @ self.g + self.h @ self.h))
        self.rhs = np.concatenate([self.f, self.gt])
        assert d.recon == "arith", "HSS: arithmetic reconstruction only (the harmonic R_H is built for BB)"
        self.A = d.A(rho)
        self.B = d.B(phi)
        self.BT = self.B.T.tocsr()
        self.C = d.C_diag(rho, s)
        al = self.alpha = o.alpha_hss
        self.sA = 1.0 / np.sqrt(self.A.diagonal())          # D_A^{-1/2}
        self.sC = 1.0 / np.sqrt(self.C)                     # D_C^{-1/2}
        DA, DC = sp.diags(self.sA), sp.diags(self.sC)
        self.Ah = (DA @ self.A @ DA).tocsr()                # Â
        self.Bh = (DC @ self.B @ DA).tocsr()                # B̂
        self.BhT = self.Bh.T.tocsr()
        self.H1 = (self.Ah + al * sp.identity(d.n)).tocsr()                 # Â + αI
        self.SK = (al * sp.identity(d.m) + (self.Bh @ self.BhT) / al).tocsr()   # αI + B̂B̂ᵀ/α
        self.inner_T_its = 0
        self.inner_A_its = []
        if o.exact_inner:
            self.H1inv = np.linalg.inv(self.H1.toarray())
            self.SKinv = np.linalg.inv(self.SK.toarray())
        else:
            slA = np.repeat(np.arange(d.K + 1), d.N)
            self.amgH = amg.setup(self.H1, slA, "As", o.omega_A, o.coarse_max_A)
            self.amgK = amg.setup(self.SK, np.zeros(d.m, dtype=np.int64), "T", o.omega_T, o.coarse_max_S)

    def matvec(self, v):
        """J v = (A x + B^T y; B x - C y)."""
        n = self.d.n
        x, y = v[:n], v[n:]
        return np.concatenate([self.A @ x + self.BT @ y, self.B @ x - self.C * y])

    def apply(self, r):
        """M^{-1}_skew S r = D^{-1/2} H_α^{-1} K_α^{-1} D^{-1/2} (r1; -r2)."""
        o, d, al = self.o, self.d, self.alpha
        n = d.n
        a = self.sA * r[:n]                                  # D^{-1/2} S r
        b = -self.sC * r[n:]
        c = b + (self.Bh @ a) / al                           # K_α^{-1} (dual Schur, eq:solve-K)
        if o.exact_inner:
            v = self.SKinv @ c
        else:
            v, its, _, _ = fgmres(lambda x: self.SK @ x, lambda x: amg.vcycle(self.amgK, x),
                                  c, float(np.linalg.norm(c)), o.eps_in_hss, o.restart_T, o.maxit_inner)
            self.inner_T_its += its
        u = (a - self.BhT @ v) / al
        if o.exact_inner:                                    # H_α^{-1} (eq:solve-laplacians)
            x = self.H1inv @ u
        else:
            x, its = pcg_slices(lambda z: self.H1 @ z, lambda z: amg.vcycle(self.amgH, z), u, d.K + 1,
                                o.eps_in_hss, o.maxit_inner)
            self.inner_A_its.append(its)
        y = v / (1.0 + al)
        return np.concatenate([self.sA * x, self.sC * y])   # D^{-1/2}

    def solve(self):
        o = self.o
        sol, its, conv, res = fgmres(self.matvec, self.apply, self.rhs, self.scale,
                                     o.eps_out, o.restart, o.maxit)
        self.stats = dict(outer_its=its, converged=bool(conv), rel_res=res / self.scale,
                          inner_T_its=self.inner_T_its,
                          inner_A_its_max=int(max((a.max() for a in self.inner_A_its), default=0)),
                          inner_A_its_total=int(sum(a.sum() for a in self.inner_A_its)))
        self.sol = sol
        return self.recover(sol)

    def recover(self, sol):
        n = self.d.n
        dphi = sol[:n].copy()
        drho = sol[n:].copy()
        ds = (self.h - self.s * drho) / self.rho
        return dphi, drho, ds
