"""D2-D12: discrete operators, residuals, Newton blocks and BB operators.

Everything is assembled literally from the paper's block formulas with
scipy.sparse (the library primitive for sparse products); vectors are
slice-concatenated as in P:160-173:  phi = (phi^1; ...; phi^{K+1}) (N each),
rho, s = (rho^1; ...; rho^K) (N̄ each).  rho^0 = rho_in, rho^{K+1} = rho_f.

Readings (restated in DESIGN.md §2):
  A4  Delta t = 1/(K+1), K+1 phi slices
  A5  time term of F_rho and B is Π^T M (not M̄ Π^T as printed P:257-260)
  A6  F_phi has K+1 slices; F_rho, F_s have K
  A7  C = +M̄ diag(s/rho), saddle (2,2) block = -C
  A8  B̃ = -M Π D_t^T + G_f D_x Π H^T  (D10)
  A9  BB Schur solve  T z = -r2,  y = P^T M̄^{-1} Ã z
  Ã_k = +Ē_c diag(|ē| R̄ rho^k / |w̄|) Ē_c^T  (PSD; "discretizes -Delta_rho")

NEXT row f4, the harmonic reconstruction (recon="harm", Remark 3.3 P:587-589;
readings A39-A41 in DESIGN.md §2): the weighted HARMONIC mean of the lifted coarse
densities on every fine edge, ρ̃_σ = R_H(ρ̄)_σ = 1/(λ_σ/ρ̄_{par L} + (1-λ_σ)/ρ̄_{par R}) (same
weights A3; type-a edges, one parent, give ρ̄ itself).  The discrete problem keeps its
Lagrangian form -- F_φ, F_ρ are the derivatives of the same kinetic term
Σ_k ½ Σ_σ |w||e| ρ̃^k_σ (∇φ^k)_σ² -- so R_E is replaced by R_H in A_k and by its Jacobian
J_H(ρ̄^k) = ∂R_H/∂ρ̄ wherever the arithmetic formulas use the (constant) R_E: F_ρ's
¼ J_Hᵀ D (g)² terms, B and Bᵀ.  F_ρ now depends on ρ: the Newton system's (2,2) block is
W = ∂F_ρ/∂ρ (block tridiagonal in time, NSD: R_H is concave), and after δs is eliminated the
saddle-point (2,2) block is -(C - W) = -C_H, "no longer diagonal" (Remark 3.3).  The BB
preconditioner uses diag(C_H) in T ("replacing C with its diagonal", Remark 3.3), the coarse
harmonic R̄_H in Ã and the fine Jacobian J_{H,f}(Πρ̄^k)ᵀD in B̃.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .mesh import TwoLevelMesh, build_two_level


class Discretisation:
    """Two-level TPFA + staggered time grid."""

    def __init__(self, verts, tris, K: int, rho_in, rho_f, validate=True, recon: str = "arith"):
        assert recon in ("arith", "harm")
        self.recon = recon
        g: TwoLevelMesh = build_two_level(verts, tris, validate=validate)
        self.g = g
        self.K = int(K)
        self.dt = 1.0 / (K + 1)                       # A4
        self.nbar, self.N, self.NE = g.nbar, g.N, g.NE
        self.n = self.N * (K + 1)
        self.m = self.nbar * K
        self.area = g.area                            # |Ω|
        self.rho0 = np.asarray(rho_in, dtype=np.float64)
        self.rhoK1 = np.asarray(rho_f, dtype=np.float64)
        N, NE, nbar = g.N, g.NE, g.nbar
        cols = np.arange(NE)
        # E[i,k] = +1 if cell i is the left side of edge k, -1 if right
        self.E = sp.csr_matrix((np.r_[np.ones(NE), -np.ones(NE)],
                                (np.r_[g.e_L, g.e_R], np.r_[cols, cols])), shape=(N, NE))
        self.grad = sp.diags(1.0 / g.w_len) @ self.E.T
        self.div = -(self.E @ sp.diags(g.e_len))
        # injection Π
        self.Pi = sp.csr_matrix((np.ones(N), (np.arange(N), g.parent)), shape=(N, nbar))
        self.M = g.c                                   # diag(|c|)
        self.Mbar = g.cbar                             # diag(|c̄|)
        # arithmetic reconstruction, A3 weights
        self.Rf = sp.csr_matrix((np.r_[g.lam, 1.0 - g.lam], (np.r_[cols, cols], np.r_[g.e_L, g.e_R])),
                                shape=(NE, N))
        self.RE = (self.Rf @ self.Pi).tocsr()
        we = g.w_len * g.e_len
        self.DR = (self.RE.T @ sp.diags(we)).tocsr()
        self.DRf = (self.Rf.T @ sp.diags(we)).tocsr()  # D3 (used by B̃, A8)
        # coarse operators for Ã
        cb = np.arange(g.NEbar)
        self.Ec = sp.csr_matrix((np.r_[np.ones(g.NEbar), -np.ones(g.NEbar)],
                                 (np.r_[g.ebar_L, g.ebar_R], np.r_[cb, cb])), shape=(nbar, g.NEbar))
        self.Rbar = sp.csr_matrix((np.r_[g.lam_bar, 1.0 - g.lam_bar],
                                   (np.r_[cb, cb], np.r_[g.ebar_L, g.ebar_R])), shape=(g.NEbar, nbar))
        self.PiT_M = (self.Pi.T @ sp.diags(self.M)).tocsr()   # Π^T M  (A5)
        self.M_Pi = (sp.diags(self.M) @ self.Pi).tocsr()      # M Π

    # ------------------------------------------------------------------ slices
    def phi_slices(self, phi):
        return np.asarray(phi).reshape(self.K + 1, self.N)

    def rho_slices(self, rho):
        """rho^0 .. rho^{K+1} (boundary data at both ends)."""
        r = np.asarray(rho).reshape(self.K, self.nbar)
        return np.vstack([self.rho0[None], r, self.rhoK1[None]])

    # ---------------------------------------------------- reconstructions
    def recon_edges(self, rbar):
        """ρ̃ = R(ρ̄) on the fine edges: arithmetic R_E ρ̄ (A3) or harmonic R_H(ρ̄) (f4)."""
        if self.recon == "arith":
            return self.RE @ rbar
        g = self.g
        a, b = rbar[g.parent[g.e_L]], rbar[g.parent[g.e_R]]
        return 1.0 / (g.lam / a + (1.0 - g.lam) / b)

    def recon_jac(self, rbar):
        """J = ∂R/∂ρ̄ (N_E x N̄): R_E itself (arithmetic) or, harmonic,
        ∂ρ̃_σ/∂ρ̄_{par L} = λ ρ̃²/a², ∂ρ̃_σ/∂ρ̄_{par R} = (1-λ) ρ̃²/b² (summed on type-a edges)."""
        if self.recon == "arith":
            return self.RE
        g = self.g
        a, b = rbar[g.parent[g.e_L]], rbar[g.parent[g.e_R]]
        rt = 1.0 / (g.lam / a + (1.0 - g.lam) / b)
        cols = np.arange(g.NE)
        return sp.csr_matrix((np.r_[g.lam * rt ** 2 / a ** 2, (1.0 - g.lam) * rt ** 2 / b ** 2],
                              (np.r_[cols, cols], np.r_[g.parent[g.e_L], g.parent[g.e_R]])), shape=(g.NE, self.nbar))

    def recon_jac_fine(self, rbar):
        """The fine-level Jacobian J_f (N_E x N) at the lifted values Πρ̄ (so J = J_f Π): R_f
        (arithmetic) or the harmonic mean's derivatives w.r.t. the two fine cells (B̃, A41)."""
        if self.recon == "arith":
            return self.Rf
        g = self.g
        a, b = rbar[g.parent[g.e_L]], rbar[g.parent[g.e_R]]
        rt = 1.0 / (g.lam / a + (1.0 - g.lam) / b)
        cols = np.arange(g.NE)
        return sp.csr_matrix((np.r_[g.lam * rt ** 2 / a ** 2, (1.0 - g.lam) * rt ** 2 / b ** 2],
                              (np.r_[cols, cols], np.r_[g.e_L, g.e_R])), shape=(g.NE, self.N))

    def recon_hess(self, rbar, wts):
        """Σ_σ wts_σ ∇²R_σ(ρ̄) (N̄ x N̄): 0 (arithmetic); harmonic, with f = ρ̃, a, b the parents:
        ∂²f/∂a² = 2λf²a⁻³(λf/a - 1), ∂²f/∂a∂b = 2λ(1-λ)f³a⁻²b⁻², ∂²f/∂b² = 2(1-λ)f²b⁻³((1-λ)f/b - 1)."""
        if self.recon == "arith":
            return sp.csr_matrix((self.nbar, self.nbar))
        g = self.g
        lam = g.lam
        pL, pR = g.parent[g.e_L], g.parent[g.e_R]
        a, b = rbar[pL], rbar[pR]
        f = 1.0 / (lam / a + (1.0 - lam) / b)
        haa = 2 * lam * f ** 2 / a ** 3 * (lam * f / a - 1.0)
        hbb = 2 * (1 - lam) * f ** 2 / b ** 3 * ((1 - lam) * f / b - 1.0)
        hab = 2 * lam * (1 - lam) * f ** 3 / (a ** 2 * b ** 2)
        return sp.csr_matrix((np.r_[wts * haa, wts * hbb, wts * hab, wts * hab],
                              (np.r_[pL, pR, pL, pR], np.r_[pL, pR, pR, pL])), shape=(self.nbar, self.nbar))

    # ------------------------------------------------------------- A_k
    def rho_bar(self, rho):
        """ρ̄^k = (ρ^k + ρ^{k-1})/2, k = 1..K+1 -> (K+1, N̄)."""
        R = self.rho_slices(rho)
        return np.stack([0.5 * (R[k] + R[k - 1]) for k in range(1, self.K + 2)])

    def rho_tilde(self, rho):
        """ρ̃^k = R((ρ^k + ρ^{k-1})/2), k = 1..K+1 -> (K+1, N_E)."""
        return np.stack([self.recon_edges(rb) for rb in self.rho_bar(rho)])

    def A_blocks(self, rho):
        """A_k = -div diag(ρ̃^k) grad, k = 1..K+1."""
        rt = self.rho_tilde(rho)
        return [(-(self.div @ sp.diags(rt[k]) @ self.grad)).tocsr() for k in range(self.K + 1)]

    def A(self, rho):
        return sp.block_diag(self.A_blocks(rho), format="csr")

    # --------------------------------------------------- residuals (2.5)-(2.7)
    def residual(self, phi, rho, s, mu):
        K, dt = self.K, self.dt
        P = self.phi_slices(phi)
        R = self.rho_slices(rho)
        S = np.asarray(s).reshape(K, self.nbar)
        Ak = self.A_blocks(rho)
        F_phi = np.stack([-self.M_Pi @ ((R[k] - R[k - 1]) / dt) + Ak[k - 1] @ P[k - 1]
                          for k in range(1, K + 2)])                      # (2.5), A6
        gr = [self.grad @ P[k] for k in range(K + 1)]
        we = self.g.w_len * self.g.e_len
        Jk = [self.recon_jac(rb) for rb in self.rho_bar(rho)]             # J(ρ̄^k), k = 1..K+1
        F_rho = np.stack([self.PiT_M @ ((P[k] - P[k - 1]) / dt)          # A5: Π^T M
                          + 0.25 * (Jk[k - 1].T @ (we * gr[k - 1] ** 2) + Jk[k].T @ (we * gr[k] ** 2))
                          + self.Mbar * S[k - 1]
                          for k in range(1, K + 1)])                      # (2.6); = ¼DR(...) for R_E
        F_s = (np.asarray(rho) * np.asarray(s) - mu)                      # (2.7)
        return F_phi.reshape(-1), F_rho.reshape(-1), F_s

    # ------------------------------------------------------ B, B^T
    def grad_phi(self, phi):
        P = self.phi_slices(phi)
        return np.stack([self.grad @ P[k] for k in range(self.K + 1)])   # g^k, (K+1, N_E)

    def B(self, phi, rho=None):
        """B = Π^T M D_t (A5) + H 𝒢 𝒟_x,  m x n, block bidiagonal; 𝒢_k = J(ρ̄^k)ᵀ D diag(g^k)
        (= DR diag(g^k) for the arithmetic R_E, which needs no ρ)."""
        K, dt = self.K, self.dt
        g = self.grad_phi(phi)
        if self.recon == "arith":
            DRk = [self.DR] * (K + 1)
        else:
            we = sp.diags(self.g.w_len * self.g.e_len)
            DRk = [(self.recon_jac(rb).T @ we).tocsr() for rb in self.rho_bar(rho)]
        blocks = [[None] * (K + 1) for _ in range(K)]
        for k in range(1, K + 1):                 # row slice k, column slices k (phi^k) and k+1
            Gk = DRk[k - 1] @ sp.diags(g[k - 1]) @ self.grad
            Gk1 = DRk[k] @ sp.diags(g[k]) @ self.grad
            blocks[k - 1][k - 1] = (-self.PiT_M / dt + 0.5 * Gk)
            blocks[k - 1][k] = (self.PiT_M / dt + 0.5 * Gk1)
        return sp.bmat(blocks, format="csr")

    def C_diag(self, rho, s):
        """C = M̄ diag(s/ρ)  (A7)."""
        return np.tile(self.Mbar, self.K) * np.asarray(s) / np.asarray(rho)

    def W(self, phi, rho):
        """W = ∂F_ρ/∂ρ (m x m), zero for R_E; harmonic: from ¼ J(ρ̄^k)ᵀD(g^k)² with
        ∂ρ̄^k/∂ρ^k = ∂ρ̄^k/∂ρ^{k-1} = ½:  W = Σ_{k=1}^{K+1} ⅛ (u_k u_kᵀ) ⊗ H_k,
        H_k = Σ_σ D_σ (g^k_σ)² ∇²R_σ(ρ̄^k), u_k = e_k + e_{k-1} (boundary slices dropped)."""
        K = self.K
        g = self.grad_phi(phi)
        we = self.g.w_len * self.g.e_len
        rbar = self.rho_bar(rho)
        blocks = [[None] * K for _ in range(K)]
        for k in range(1, K + 2):                  # φ slice k couples ρ^{k-1}, ρ^k
            Hk = 0.125 * self.recon_hess(rbar[k - 1], we * g[k - 1] ** 2)
            idx = [j - 1 for j in (k - 1, k) if 1 <= j <= K]
            for a in idx:
                for b in idx:
                    blocks[a][b] = Hk if blocks[a][b] is None else blocks[a][b] + Hk
        for a in range(K):
            if blocks[a][a] is None:
                blocks[a][a] = sp.csr_matrix((self.nbar, self.nbar))
        return sp.bmat(blocks, format="csr")

    def C_H(self, phi, rho, s):
        """The reduced (2,2) block: C_H = C - W (= C for R_E; Remark 3.3)."""
        C = sp.diags(self.C_diag(rho, s))
        return (C - self.W(phi, rho)).tocsr() if self.recon == "harm" else C.tocsr()

    # -------------------------------------------------- projector P
    def P(self, y):
        """(P y)^k = y^k - c̄ (1^T y^k) / |Ω|."""
        Y = np.asarray(y).reshape(self.K, self.nbar)
        return (Y - self.Mbar[None, :] * Y.sum(1, keepdims=True) / self.area).reshape(-1)

    def PT(self, y):
        """(P^T y)^k = y^k - 1 (c̄^T y^k) / |Ω|  (zero-mean projector)."""
        Y = np.asarray(y).reshape(self.K, self.nbar)
        return (Y - (Y @ self.Mbar)[:, None] / self.area).reshape(-1)

    # ------------------------------------------------ Newton system (3.1)/(3.2)
    def newton_rhs(self, phi, rho, s, mu):
        F_phi, F_rho, F_s = self.residual(phi, rho, s, mu)
        f, g, h = -F_phi, -F_rho, -F_s
        gt = g - np.tile(self.Mbar, self.K) * h / np.asarray(rho)          # g̃
        return f, g, h, gt

    def jacobian(self, phi, rho, s):
        """Full 3x3 block Jacobian (3.1) as a sparse matrix ((2,2) block W, zero for R_E)."""
        A = self.A(rho)
        B = self.B(phi, rho)
        Mb = sp.diags(np.tile(self.Mbar, self.K))
        return sp.bmat([[A, B.T, None],
                        [B, self.W(phi, rho) if self.recon == "harm" else None, Mb],
                        [None, sp.diags(np.asarray(s)), sp.diags(np.asarray(rho))]], format="csr")

    # ------------------------------------------ projected system (4.17) matvec
    def make_JP(self, phi, rho, s):
        """J_P of (4.17); C is the reduced (2,2) block C_H = C - W (a matrix for R_H)."""
        A = self.A(rho)
        B = self.B(phi, rho)
        BT = B.T.tocsr()
        C = self.C_H(phi, rho, s) if self.recon == "harm" else self.C_diag(rho, s)
        n = self.n

        def JP(v):
            x, y = v[:n], v[n:]
            yp = self.PT(y)
            return np.concatenate([A @ x + BT @ yp, self.P(B @ x - C * yp if self.recon == "arith"
                                                            else B @ x - C @ yp)])
        return JP, A, B, BT, C

    # ----------------------------------------------------- BB operators (4.22)
    def Atilde_blocks(self, rho):
        """Ã_k = Ē_c diag(|ē| R̄ρ^k / |w̄|) Ē_c^T, k = 1..K."""
        g = self.g
        R = np.asarray(rho).reshape(self.K, self.nbar)
        out = []
        for k in range(self.K):
            if self.recon == "harm":              # the coarse harmonic mean (A40)
                rb = 1.0 / (g.lam_bar / R[k][g.ebar_L] + (1.0 - g.lam_bar) / R[k][g.ebar_R])
            else:
                rb = self.Rbar @ R[k]
            om = g.ebar_len * rb / g.wbar_len
            out.append((self.Ec @ sp.diags(om) @ self.Ec.T).tocsr())
        return out

    def Atilde(self, rho):
        return sp.block_diag(self.Atilde_blocks(rho), format="csr")

    def Btilde(self, phi, rho=None):
        """B̃ (n x m), D10 / A8:
        (B̃z)^k = MΠ(z^k - z^{k-1})/Δt + ½ DR_f diag(g^k) grad Π (z^{k-1} + z^k),
        k = 1..K+1, z^0 = z^{K+1} = 0;  harmonic: DR_f -> J_f(Πρ̄^k)ᵀ D (A41)."""
        K, dt = self.K, self.dt
        g = self.grad_phi(phi)
        if self.recon == "harm":
            we = sp.diags(self.g.w_len * self.g.e_len)
            DRfk = [(self.recon_jac_fine(rb).T @ we).tocsr() for rb in self.rho_bar(rho)]
        else:
            DRfk = [self.DRf] * (K + 1)
        blocks = [[None] * K for _ in range(K + 1)]
        for k in range(1, K + 2):                 # row slice k; column slices k-1, k of z
            Sk = 0.5 * (DRfk[k - 1] @ sp.diags(g[k - 1]) @ self.grad @ self.Pi)
            if k <= K:
                blocks[k - 1][k - 1] = self.M_Pi / dt + Sk
            if k >= 2:
                blocks[k - 1][k - 2] = -self.M_Pi / dt + Sk
        return sp.bmat(blocks, format="csr")

    def T_matrix(self, phi, rho, s):
        """T = C M̄^{-1} Ã - B M^{-1} B̃  (4.26; C M̄^{-1} = diag(s/ρ)); harmonic: C -> diag(C_H)
        (Remark 3.3)."""
        At = self.Atilde(rho)
        B = self.B(phi, rho)
        Bt = self.Btilde(phi, rho)
        Minv = sp.diags(1.0 / np.tile(self.M, self.K + 1))
        if self.recon == "harm":
            sr = self.C_H(phi, rho, s).diagonal() / np.tile(self.Mbar, self.K)
        else:
            sr = np.asarray(s) / np.asarray(rho)
        return (sp.diags(sr) @ At - B @ (Minv @ Bt)).tocsr()

    # ------------------------------------------------------ kinetic energy D12
    def kinetic_energy(self, phi, rho):
        """KE = Σ_{k=1}^{K+1} Δt ½ φ^k^T A_k φ^k (discrete (1.1))."""
        P = self.phi_slices(phi)
        Ak = self.A_blocks(rho)
        return float(sum(self.dt * 0.5 * P[k] @ (Ak[k] @ P[k]) for k in range(self.K + 1)))

    def slice_mass(self, rho):
        return np.asarray(rho).reshape(self.K, self.nbar) @ self.Mbar
