"""Pins of oracle/hss.py (NEXT row f2, the HSS preconditioner, §5.1)
against what the paper and the mathematics fix -- not against itself."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.bb import BBSolver, SolverOpts
from oracle.hss import HssSolver
from oracle.ops import Discretisation
from synthetic import make_problem, random_state


def _hss(name, seed, mu, exact):
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=seed, mu=mu)
    return p, d, HssSolver(d, phi, rho, s, mu, SolverOpts(exact_inner=exact)), (phi, rho, s)


def _blocks(H):
    d, al = H.d, H.alpha
    Jhat = sp.bmat([[H.Ah, H.BhT], [-H.Bh, sp.diags(H.sC * H.C * H.sC)]]).toarray()
    Ha = sp.block_diag([H.Ah + al * sp.identity(d.n), (1 + al) * sp.identity(d.m)]).toarray()
    Ka = sp.bmat([[al * sp.identity(d.n), H.BhT], [-H.Bh, al * sp.identity(d.m)]]).toarray()
    return Jhat, Ha, Ka


def test_hss_splitting_identity():
    """eq:hss-hk: H_α + K_α = Ĵ + 2αI, where Ĵ = D^{-1/2} J_skew D^{-1/2} is the
    diagonally scaled skew system -- Ĵ has unit diagonal, and J_skew is the
    saddle-point matrix with its second block row negated (eq:saddle-point-skew)."""
    p, d, H, (phi, rho, s) = _hss("T0", 3, 0.1, True)
    Jhat, Ha, Ka = _blocks(H)
    assert np.allclose(Ha + Ka, Jhat + 2 * H.alpha * np.eye(d.n + d.m), rtol=0, atol=1e-12 * abs(Jhat).max())
    assert np.allclose(np.diag(Jhat), 1.0, rtol=0, atol=1e-13)
    # Ĵ is the scaling of J_skew = [[A, B^T], [-B, C]] built independently from the operators
    A, B, C = d.A(rho), d.B(phi), d.C_diag(rho, s)
    Jskew = sp.bmat([[A, B.T], [-B, sp.diags(C)]]).toarray()
    Dm = np.r_[1 / np.sqrt(A.diagonal()), 1 / np.sqrt(C)]
    assert np.allclose(Jhat, Dm[:, None] * Jskew * Dm[None, :], rtol=0, atol=1e-12 * abs(Jhat).max())


def test_hss_exact_apply_is_inverse_of_KH():
    """eq:prec-hss, factors reversed: P = K_α H_α.  With exact inner solves the
    apply (K_α^{-1} through the dual Schur complement eq:solve-K, then H_α^{-1})
    equals D^{-1/2} (K_α H_α)^{-1} D^{-1/2} S on arbitrary vectors (S = diag(I, -I)): fails on a
    sign, transpose or scaling slip anywhere in the apply."""
    p, d, H, _ = _hss("T1", 4, 0.05, True)
    _, Ha, Ka = _blocks(H)
    Dm = np.r_[H.sA, H.sC]
    Sg = np.r_[np.ones(d.n), -np.ones(d.m)]
    P = Ka @ Ha
    rng = np.random.default_rng(0)
    for _ in range(3):
        r = rng.standard_normal(d.n + d.m)
        ref = Dm * np.linalg.solve(P, Dm * Sg * r)
        assert np.linalg.norm(H.apply(r) - ref) <= 1e-10 * np.linalg.norm(ref)


def test_hss_spectrum_in_unit_disk_around_one():
    """HSS contraction (Bai, Golub & Ng, the scheme of P:633): with Ĵ = H + S (H = blkdiag(Â, I)
    Hermitian PSD, S skew), the preconditioned matrix 2α (K_α H_α)^{-1} Ĵ = I - T(α) with
    ρ(T(α)) <= max |α - λ(H)| / |α + λ(H)| <= 1, so its eigenvalues lie in |λ - 1| <= 1 --
    on a random IPM-like state and on the pure-diffusion state φ = 0."""
    for seed, mu in ((5, 0.1), (6, 1e-3)):
        p, d, H, _ = _hss("T0", seed, mu, True)
        Jhat, Ha, Ka = _blocks(H)
        ev = np.linalg.eigvals(2 * H.alpha * np.linalg.solve(Ka @ Ha, Jhat))
        assert np.abs(ev - 1).max() <= 1 + 1e-9, np.abs(ev - 1).max()


@pytest.mark.parametrize("name", ["T0", "T1"])
def test_hss_solve_matches_direct(name):
    """The HSS-preconditioned FGMRES direction (inexact AMG inner solves, ε_in = 1e-1, α = 0.5,
    P:708) equals the dense least-squares solve of (3.1) up to the kernel ⟨(1;0;0)⟩
    (Remark 3.1): δφ differs by a constant, δρ and δs agree."""
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=7, mu=0.05)
    H = HssSolver(d, phi, rho, s, 0.05, SolverOpts(eps_out=1e-12))
    dphi, drho, ds = H.solve()
    assert H.stats["converged"] and H.stats["inner_T_its"] > 0 and H.stats["inner_A_its_total"] > 0
    J = d.jacobian(phi, rho, s).toarray()
    f, g, h, _ = d.newton_rhs(phi, rho, s, 0.05)
    rhs = np.concatenate([f, g, h])
    ref, *_ = np.linalg.lstsq(J, rhs, rcond=None)
    n, m = d.n, d.m
    shift = (dphi - ref[:n]).mean()
    assert np.linalg.norm(dphi - shift - ref[:n]) <= 1e-9 * np.linalg.norm(ref[:n])
    assert np.linalg.norm(drho - ref[n:n + m]) <= 1e-9 * np.linalg.norm(ref[n:n + m])
    assert np.linalg.norm(ds - ref[n + m:]) <= 1e-9 * np.linalg.norm(ref[n + m:])


def test_hss_and_bb_directions_agree():
    """The converged HSS and BB (§4.5) directions of the same Newton system coincide (both
    solve (3.1) to 1e-10; δφ up to the kernel constant, Remark 3.1)."""
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=8, mu=0.02)
    a = HssSolver(d, phi, rho, s, 0.02).solve()
    b = BBSolver(d, phi, rho, s, 0.02).solve()
    shift = (a[0] - b[0]).mean()
    assert np.linalg.norm(a[0] - shift - b[0]) <= 1e-7 * np.linalg.norm(b[0])
    for u, v in zip(a[1:], b[1:]):
        assert np.linalg.norm(u - v) <= 1e-7 * np.linalg.norm(v)


def test_amg_mode_As_coarsest_is_exact_on_one_level():
    """mode "As" (I3 for the nonsingular shifted blocks): when the fine level is already the
    coarsest, one cycle is the exact per-slice solve (no grounding, no mean removal)."""
    from oracle import amg
    rng = np.random.default_rng(3)
    blocks = []
    for k in range(3):
        Q = sp.random(20, 20, density=0.2, random_state=k)
        L = (Q + Q.T)
        L = sp.diags(np.asarray(abs(L).sum(1)).ravel() + 0.5) - L
        blocks.append(L)
    A = sp.block_diag(blocks, format="csr")
    sl = np.repeat(np.arange(3), 20)
    Hh = amg.setup(A, sl, "As", 2 / 3, coarse_max=64)
    b = rng.standard_normal(60)
    assert np.allclose(amg.vcycle(Hh, b), np.linalg.solve(A.toarray(), b), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("L,K,table", [(1, 4, 31), (2, 8, 71)])
def test_hss_counts_vs_paper_table(L, K, table):
    """Outer FGMRES iterations of the HSS-preconditioned solve (α = 0.5, ε_in = 1e-1, AMG inner
    solves as the paper's AGMG) at μ = 1 and the paper's ε_out = 1e-5, test
    case 2 (translated compact bump), within a factor 2 of the first row of the HSS table for
    the two coarsest meshes (31 at N̄ = 56, Nt = 8; 71 at N̄ = 224, Nt = 16) --
    the S:605 acceptance band used for BB (test_bb_counts_vs_table4).  Measured 46 / 98."""
    p = make_problem("T2b", L=L, K=K)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    from synthetic import initial_state
    phi, rho, s = initial_state(p, 1.0)
    H = HssSolver(d, phi, rho, s, 1.0, SolverOpts(precond="hss", eps_out=1e-5, maxit=2000))
    H.solve()
    assert H.stats["converged"] and table / 2 <= H.stats["outer_its"] <= 2 * table, H.stats
