"""Pins of the harmonic reconstruction (NEXT row f4, Remark 3.3 P:587-589;
DESIGN.md A39-A41) in oracle/ops.py + oracle/bb.py -- against what the mathematics fixes."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.bb import BBSolver, SolverOpts
from oracle.ops import Discretisation
from synthetic import make_problem, random_state


def _disc(name, recon="harm"):
    p = make_problem(name)
    return p, Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f, recon=recon)


def test_harmonic_mean_properties():
    """R_H is the weighted harmonic mean: R_H <= R_E (AM-HM), equality for a constant ρ̄ and on
    every type-a edge (both cells in one triangle); 1-homogeneous; between the two values."""
    p, d = _disc("T1")
    _, da = _disc("T1", "arith")
    g = d.g
    rb = np.random.default_rng(0).uniform(0.1, 3.0, d.nbar)
    h, a = d.recon_edges(rb), da.recon_edges(rb)
    assert np.all(h <= a * (1 + 1e-15))
    assert np.allclose(h[g.e_type == 0], rb[g.parent[g.e_L[g.e_type == 0]]], rtol=1e-15)
    lo = np.minimum(rb[g.parent[g.e_L]], rb[g.parent[g.e_R]])
    hi = np.maximum(rb[g.parent[g.e_L]], rb[g.parent[g.e_R]])
    assert np.all(h >= lo * (1 - 1e-15)) and np.all(h <= hi * (1 + 1e-15))
    assert np.allclose(d.recon_edges(np.full(d.nbar, 2.5)), 2.5, rtol=1e-15)
    assert np.allclose(d.recon_edges(3.0 * rb), 3.0 * h, rtol=1e-14)


def test_harmonic_jacobian_and_hessian_by_differences():
    """J = ∂R_H/∂ρ̄ and Σ wts ∇²R_H against central differences of R_H itself."""
    p, d = _disc("T1")
    rng = np.random.default_rng(1)
    rb = rng.uniform(0.2, 2.0, d.nbar)
    v = rng.standard_normal(d.nbar)
    eps = 1e-6
    fd = (d.recon_edges(rb + eps * v) - d.recon_edges(rb - eps * v)) / (2 * eps)
    assert np.allclose(d.recon_jac(rb) @ v, fd, rtol=1e-7, atol=1e-9)
    wts = rng.uniform(0.5, 1.5, d.g.NE)
    fd2 = (d.recon_jac(rb + eps * v).T @ wts - d.recon_jac(rb - eps * v).T @ wts) / (2 * eps)
    H = d.recon_hess(rb, wts)
    assert np.allclose(H @ v, fd2, rtol=1e-6, atol=1e-8)
    assert abs(H - H.T).max() < 1e-12 * abs(H).max()
    assert np.linalg.eigvalsh(H.toarray()).max() <= 1e-12 * abs(H).max()      # concave: NSD
    # the fine Jacobian lifts: J = J_f Π
    assert abs(d.recon_jac(rb) - d.recon_jac_fine(rb) @ d.Pi).max() < 1e-14 * abs(d.recon_jac(rb)).max()


def test_harmonic_jacobian_finite_difference():
    """(3.1) with R_H -- A_k(R_H), F_ρ with J_Hᵀ, B, Bᵀ with J_H and the new (2,2) block W --
    is the Jacobian of the residuals (2.5)-(2.7) built on R_H."""
    p, d = _disc("T1")
    phi, rho, s = random_state(p, seed=3, mu=0.05)
    n, m = d.n, d.m
    J = d.jacobian(phi, rho, s)
    x0 = np.concatenate([phi, rho, s])

    def F(x):
        return np.concatenate(d.residual(x[:n], x[n:n + m], x[n + m:], 0.05))
    rng = np.random.default_rng(0)
    for _ in range(3):
        v = rng.standard_normal(x0.size)
        eps = 1e-5
        fd = (F(x0 + eps * v) - F(x0 - eps * v)) / (2 * eps)
        assert np.linalg.norm(fd - J @ v) <= 1e-8 * np.linalg.norm(J @ v)
    # the Jacobian is symmetric in its (φ, ρ) block (a Hessian of the Lagrangian)
    Jr = J[:n + m, :n + m]
    assert abs(Jr - Jr.T).max() <= 1e-12 * abs(Jr).max()


def test_harmonic_W_nsd_and_C_H():
    """W ⪯ 0 (R_H concave) so C_H = C - W ⪰ C ≻ 0: the reduced (2,2) block is symmetric positive
    definite and no longer diagonal (Remark 3.3)."""
    p, d = _disc("T1")
    phi, rho, s = random_state(p, seed=4, mu=0.05)
    W = d.W(phi, rho).toarray()
    assert np.abs(W).max() > 0 and np.linalg.eigvalsh(0.5 * (W + W.T)).max() <= 1e-12 * np.abs(W).max()
    CH = d.C_H(phi, rho, s).toarray()
    assert np.count_nonzero(CH - np.diag(np.diag(CH))) > 0
    assert np.linalg.eigvalsh(CH).min() >= d.C_diag(rho, s).min() * (1 - 1e-12)


@pytest.mark.parametrize("name", ["T0", "T1"])
def test_harmonic_bb_solve_matches_direct(name):
    """The BB-preconditioned FGMRES direction with R_H (J_P with C_H, T with diag(C_H), Ã with
    R̄_H, B̃ with J_f; recovery with C_H) equals the dense least-squares solve of (3.1)."""
    p, d = _disc(name)
    phi, rho, s = random_state(p, seed=7, mu=0.05)
    S = BBSolver(d, phi, rho, s, 0.05, SolverOpts(eps_out=1e-12))
    dphi, drho, ds = S.solve()
    assert S.stats["converged"]
    J = d.jacobian(phi, rho, s).toarray()
    f, g, h, _ = d.newton_rhs(phi, rho, s, 0.05)
    rhs = np.concatenate([f, g, h])
    ref, *_ = np.linalg.lstsq(J, rhs, rcond=None)
    n, m = d.n, d.m
    rp = ref[:n].reshape(d.K + 1, d.N)
    rp = (rp - (rp[0] @ d.M) / d.area).reshape(-1)
    for a, b in ((dphi, rp), (drho, ref[n:n + m]), (ds, ref[n + m:])):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)


def test_harmonic_equals_arithmetic_for_uniform_density():
    """At a slice-uniform ρ (the A19 initial point) R_H = R_E on every edge, W = 0 (the Hessian
    terms vanish only through (∇φ)² = 0 at φ = 0), so every operator coincides."""
    p, dh = _disc("T1")
    _, da = _disc("T1", "arith")
    from synthetic import initial_state
    phi, rho, s = initial_state(p, 1.0)
    Th, Ta = dh.T_matrix(phi, rho, s), da.T_matrix(phi, rho, s)
    # only the two slices touching ρ_in / ρ_f are non-uniform: compare the interior rows
    nb = dh.nbar
    rows = slice(nb, (dh.K - 1) * nb)
    assert abs(dh.W(phi, rho)).max() == 0.0
    assert abs(dh.A_blocks(rho)[2] - da.A_blocks(rho)[2]).max() <= 1e-14 * abs(da.A_blocks(rho)[2]).max()
    assert abs((Th - Ta)[rows]).max() <= 1e-12 * abs(Ta).max()


def test_harmonic_ipm_kinetic_energy_translation():
    """Test case 2 (translation of a compact bump, OT cost ½|t|²·mass = 0.16): the IPM
    with R_H converges on every system and its kinetic energy approaches the closed form under
    joint (h, Δt) refinement, the gap to the arithmetic run shrinking with it (the two
    reconstructions are consistent to first order; measured 0.250/0.217 at (L, K) = (1, 4),
    0.194/0.178 at (2, 8))."""
    from oracle.ipm import IpmOpts, ipm_run
    from synthetic import initial_state
    kes = {}
    for L, K in ((1, 4), (2, 8)):
        for recon in ("arith", "harm"):
            p = make_problem("T2b", L=L, K=K)
            d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f, recon=recon)
            phi, rho, s = initial_state(p, 1.0)
            r = ipm_run(d, phi, rho, s, IpmOpts(mu_min=1e-3), SolverOpts(eps_out=1e-8))
            assert all(rec["converged"] for rec in r.log)
            kes[(L, recon)] = r.kinetic_energy
    eh = [kes[(L, "harm")] - 0.16 for L in (1, 2)]
    gap = [kes[(L, "harm")] - kes[(L, "arith")] for L in (1, 2)]
    assert 0 < eh[1] < 0.8 * eh[0], kes                  # converging from above
    assert 0 < gap[1] < 0.6 * gap[0], kes                # R_H >= ... -> R_E: the gap closes


def test_harmonic_solve_rhs_matches_direct():
    """solve(rhs) with R_H: the slice-mass step now also carries W δρ₀ into g (the (2,2) block
    acts on it); the result is the dense least-squares solve of (3.1) with the caller's (f;g;h),
    on a state of the harmonic IPM trajectory (mu = 2^-4)."""
    from oracle.ipm import IpmOpts, ipm_run
    from synthetic import initial_state
    p, d = _disc("T1")
    phi, rho, s = initial_state(p, 1.0)
    r = ipm_run(d, phi, rho, s, IpmOpts(mu_min=2.0 ** -4), SolverOpts())
    phi, rho, s = r.phi, r.rho, r.s
    rng = np.random.default_rng(5)
    f = rng.standard_normal(d.n)
    f -= f.mean()
    g, h = rng.standard_normal(d.m), rng.standard_normal(d.m)
    S = BBSolver(d, phi, rho, s, 2.0 ** -5, SolverOpts(eps_out=1e-12))
    dphi, drho, ds = S.solve_rhs(f, g, h)
    assert S.stats["converged"], S.stats
    J = d.jacobian(phi, rho, s).toarray()
    rhs = np.concatenate([f, g, h])
    ref, *_ = np.linalg.lstsq(J, rhs, rcond=None)
    n, m = d.n, d.m
    rp = ref[:n].reshape(d.K + 1, d.N)
    rp = (rp - (rp[0] @ d.M) / d.area).reshape(-1)
    for a, b in ((dphi, rp), (drho, ref[n:n + m]), (ds, ref[n + m:])):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)
