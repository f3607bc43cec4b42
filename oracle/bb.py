"""I2 + a6: the BB-preconditioner (§4.5) and recovery.

Projected system (4.17), P:1424-1448:
    J_P = [[A, B^T P^T], [P B, -P C P^T]],  rhs (f; P g̃).
Ideal block-triangular preconditioner (4.18)-(4.20), with the Schur
complement replaced through the approximate commutation (4.22), and
solved as (4.26).  BB apply on (r1; r2):
  (i)   T z = -r2  by GMRES(10) + one AMG(T) V-cycle, relative eps_T (1e-1)
        (A43: the target is max(eps_T ||r2||, 1e-12 ||r||), rounding-level r2 is not solved)
  (ii)  y = P^T (M̄^{-1} Ã z)
  (iii) b = r1 - B^T P^T y;  b^k -= mean(b^k)            (compatibility)
  (iv)  A_k x^k = b^k by PCG + AMG(A_k) V-cycle, relative eps_A (A14: 1e-3), x^k -= mean
Recovery (a6): δρ := P^T y (A30); δφ̃^k -= c^T δφ̃^k/|Ω| (A11);
  δλ = Ē(g̃ - B δφ̃ + C δρ)/|Ω|;
  δφ^k = δφ̃^k + Σ_{i=1}^{k-1} Δt δλ^i  (4.15 with A10);  δs = ρ^{-1}(h - s δρ).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import amg
from .krylov import fgmres, pcg_slices
from .ops import Discretisation


T_NOISE = 1e-12      # A43: delta of the T-solve's stopping rule (relative to ||(r1; r2)||)


@dataclass
class SolverOpts:
    eps_out: float = 1e-10        # A16
    eps_T: float = 1e-1
    eps_A: float = 1e-3           # A14 (paper: 5e-2 with AGMG)
    restart: int = 30             # A15
    maxit: int = 400
    restart_T: int = 10
    maxit_inner: int = 50
    omega_A: float = 2.0 / 3.0
    omega_T: float = 1.0          # I3: l1-Jacobi for AMG(T) (D = row sums of |T|)
    coarse_max_A: int = 64        # rows per slice
    coarse_max_T: int = 1024      # rows in total
    exact_inner: bool = False     # pin mode: exact T solve + exact A_k^+ (no AMG)
    precond: str = "bb"           # "bb" (§4.5), "simple" (§5.3, NEXT f1) or "hss" (§5.1, NEXT f2)
    coarse_max_S: int = 256       # AMG(Ŝ) coarsest rows (SIMPLE, A32; also HSS's K-solve)
    alpha_hss: float = 0.5        # HSS relaxation parameter α
    eps_in_hss: float = 1e-1      # HSS inner tolerance ε_in


class BBSolver:
    """Per-Newton-step setup (a1, a3) + solve (a2, a4, a5) + recovery (a6)."""

    def __init__(self, disc: Discretisation, phi, rho, s, mu, opts: SolverOpts | None = None):
        self.d = d = disc
        self.o = o = opts or SolverOpts()
        self.phi, self.rho, self.s, self.mu = (np.asarray(phi, float), np.asarray(rho, float),
                                               np.asarray(s, float), float(mu))
        # a1: residuals / right-hand sides
        self.f, self.g, self.h, self.gt = d.newton_rhs(phi, rho, s, mu)
        self.scale = float(np.sqrt(self.f @ self.f + self.g @ self.g + self.h @ self.h))
        self.rhs = np.concatenate([self.f, d.P(self.gt)])
        # a2 operators
        self.JP, self.A, self.B, self.BT, self.C = d.make_JP(phi, rho, s)
        # a3: BB setup
        self.Atilde = d.Atilde(rho)
        self.T = d.T_matrix(phi, rho, s)
        self.Mbar_t = np.tile(d.Mbar, d.K)
        self.inner_T_its = 0
        self.inner_A_its = []
        if o.exact_inner:
            self.Tinv = np.linalg.inv(self.T.toarray())
            self.Apinv = [np.linalg.pinv(Ak.toarray()) for Ak in d.A_blocks(rho)]
        else:
            slA = np.repeat(np.arange(d.K + 1), d.N)
            slT = np.repeat(amg.time_blocks(d.K), d.nbar)          # A42: time blocks
            self.amgA = amg.setup(self.A, slA, "A", o.omega_A, o.coarse_max_A)
            self.amgT = amg.setup(self.T, slT, "T", o.omega_T, o.coarse_max_T)

    # ---------------------------------------------------------------- a4
    def apply(self, r):
        d, o = self.d, self.o
        n = d.n
        r1, r2 = r[:n], r[n:]
        if o.exact_inner:
            z = self.Tinv @ (-r2)
        else:
            # A43: stop at max(eps_T ||r2||, delta ||r||) -- an r2 at rounding level of r
            # (P g~ at the A19 point is zero in exact arithmetic) is not solved to eps_T relative
            nr2 = float(np.linalg.norm(r2))
            scale = max(nr2, T_NOISE / o.eps_T * float(np.linalg.norm(r)))
            z, itT, _, _ = fgmres(lambda v: self.T @ v, lambda v: amg.vcycle(self.amgT, v),
                                  -r2, scale, o.eps_T, o.restart_T, o.maxit_inner)
            self.inner_T_its += itT
        y = d.PT((self.Atilde @ z) / self.Mbar_t)
        b = (r1 - self.BT @ d.PT(y)).reshape(d.K + 1, d.N)
        b = b - b.mean(axis=1, keepdims=True)
        if o.exact_inner:
            x = np.stack([self.Apinv[k] @ b[k] for k in range(d.K + 1)])
        else:
            x, its = pcg_slices(lambda v: self.A @ v, lambda v: amg.vcycle(self.amgA, v),
                                b.reshape(-1), d.K + 1, o.eps_A, o.maxit_inner)
            self.inner_A_its.append(its)
            x = x.reshape(d.K + 1, d.N)
        x = x - x.mean(axis=1, keepdims=True)
        return np.concatenate([x.reshape(-1), y])

    # ---------------------------------------------------------------- a5 + a6
    def solve(self):
        o = self.o
        sol, its, conv, res = fgmres(self.JP, self.apply, self.rhs, self.scale,
                                     o.eps_out, o.restart, o.maxit)
        self.stats = dict(outer_its=its, converged=bool(conv), rel_res=res / self.scale,
                          inner_T_its=self.inner_T_its,
                          inner_A_its_max=int(max((a.max() for a in self.inner_A_its), default=0)),
                          inner_A_its_total=int(sum(a.sum() for a in self.inner_A_its)))
        self.sol = sol
        return self.recover(sol)

    def solve_rhs(self, f, g, h):
        """solve(rhs) -> direction for the Newton system (3.1) of this state with a
        caller-given right-hand side (f; g; h), solvable iff Σ_k 1ᵀf^k = 0 (the left kernel of
        J is (1;0;0), Remark 3.1).  (4.17) needs 1ᵀf^k = 0 slice by slice (A30), so the mass
        part of δρ is taken first: summing the k-th φ row of (3.1),
            1ᵀ(A_kδφ^k + (Bᵀδρ)^k) = c̄ᵀ(δρ^{k-1} - δρ^k)/Δt = 1ᵀf^k   (1ᵀA_k = 0, D6),
        fixes the slice masses m_k = c̄ᵀδρ^k = m_{k-1} - Δt 1ᵀf^k (m_0 = 0);  with
        δρ₀^k = (m_k/|Ω|)·1 the remainder δρ' = δρ - δρ₀ solves (3.1) with
        (f - Bᵀδρ₀; g; h - s⊙δρ₀), whose φ rows have zero slice sums, by the BB solve
        (4.17) + recovery; then δρ = δρ' + δρ₀.  Stop at ε‖(f;g;h)‖."""
        d = self.d
        K = d.K
        f = np.asarray(f, float)
        g = np.asarray(g, float)
        h = np.asarray(h, float)
        Sf = f.reshape(K + 1, d.N).sum(axis=1)
        mk = -d.dt * np.cumsum(Sf)[:K]                                    # m_1 .. m_K
        drho0 = np.repeat(mk / d.area, d.nbar)
        self.f = f - self.BT @ drho0
        self.g = g - d.W(self.phi, self.rho) @ drho0 if d.recon == "harm" else g     # W δρ₀ (f4)
        self.h = h - self.s * drho0
        self.gt = self.g - np.tile(d.Mbar, K) * self.h / self.rho         # g̃
        self.scale = float(np.sqrt(f @ f + g @ g + h @ h))
        self.rhs = np.concatenate([self.f, d.P(self.gt)])
        self.inner_T_its = 0
        self.inner_A_its = []
        dphi, drho, ds = self.solve()
        return dphi, drho + drho0, ds

    def recover(self, sol):
        d = self.d
        K, N, n = d.K, d.N, d.n
        dphit = sol[:n].reshape(K + 1, N).copy()
        drho = d.PT(sol[n:])                                             # A30
        dphit = dphit - (dphit @ d.M)[:, None] / d.area                  # A11
        dphit = dphit.reshape(-1)
        Cd = self.C @ drho if d.recon == "harm" else self.C * drho        # C_H δρ (Remark 3.3)
        q = (self.gt - self.B @ dphit + Cd).reshape(K, d.nbar)
        dlam = q.sum(axis=1) / d.area
        shift = np.concatenate([[0.0], np.cumsum(d.dt * dlam)])          # Σ_{i<k} Δt δλ^i (A10)
        dphi = (dphit.reshape(K + 1, N) + shift[:, None]).reshape(-1)
        ds = (self.h - self.s * drho) / self.rho
        return dphi, drho, ds
