"""Pins of oracle/simple.py (NEXT row f1, the SIMPLE preconditioner)
against what the paper and the mathematics fix -- not against itself."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.bb import BBSolver, SolverOpts
from oracle.direct import direct_newton
from oracle.ops import Discretisation
from oracle.simple import S_hat, SimpleSolver
from synthetic import initial_state, make_problem, random_state


def _disc(name):
    p = make_problem(name)
    return p, Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)


def test_simple_block_factorisation_inverts_Jtilde():
    """eq:sca-precs: with an exact S̃ solve, the three factors multiply out to
    the inverse of J̃ = [[diag(A), B^T], [B, -C]] -- i.e. P = L D U = J̃.  Applying the
    preconditioner to J̃ x returns x for arbitrary x (fails on any sign, transpose or
    index slip in the apply)."""
    p, d = _disc("T1")
    phi, rho, s = random_state(p, seed=3, mu=0.07)
    S = SimpleSolver(d, phi, rho, s, 0.07, SolverOpts(exact_inner=True))
    Jt = sp.bmat([[sp.diags(S.A.diagonal()), S.B.T], [S.B, -sp.diags(S.C)]]).tocsr()
    rng = np.random.default_rng(0)
    for _ in range(3):
        x = rng.standard_normal(d.n + d.m)
        y = S.apply(Jt @ x)
        assert np.linalg.norm(y - x) <= 1e-10 * np.linalg.norm(x)


def test_S_hat_spd_and_entrywise():
    """Ŝ = C + B diag(A)^{-1} B^T (A31) is symmetric positive definite, and entry
    (i, j) equals the brute-force sum over phi unknowns of B_iq B_jq / A_qq + C_i δ_ij."""
    p, d = _disc("T1")
    phi, rho, s = random_state(p, seed=4, mu=0.2)
    Sh = S_hat(d, phi, rho, s).toarray()
    assert np.allclose(Sh, Sh.T, rtol=0, atol=1e-12 * np.abs(Sh).max())
    assert np.linalg.eigvalsh(0.5 * (Sh + Sh.T)).min() > 0
    B = d.B(phi).toarray()
    a = d.A(rho).diagonal()
    C = d.C_diag(rho, s)
    rng = np.random.default_rng(1)
    for i, j in rng.integers(0, d.m, size=(20, 2)):
        v = sum(B[i, q] * B[j, q] / a[q] for q in range(d.n)) + (C[i] if i == j else 0.0)
        assert abs(Sh[i, j] - v) <= 1e-12 * max(1.0, abs(v))


def test_S_hat_block_tridiagonal_in_time():
    """Ŝ is block tridiagonal (slices k, k +- 1 only)."""
    p, d = _disc("T2")
    phi, rho, s = random_state(p, seed=5, mu=0.1)
    Sh = S_hat(d, phi, rho, s).tocoo()
    kr, kc = Sh.row // d.nbar, Sh.col // d.nbar
    assert np.abs(kr - kc).max() <= 1


@pytest.mark.parametrize("name,exact", [("T1", True), ("T1", False), ("T2", False)])
def test_simple_solve_matches_direct(name, exact):
    """SIMPLE-FGMRES on (eq:saddle-point) + δs elimination reproduces the dense direct solve
    of (3.1) up to the kernel <(1;0;0)> of Remark 3.1."""
    p, d = _disc(name)
    phi, rho, s = random_state(p, seed=7, mu=0.05)
    dphi0, drho0, ds0, J, rhs = direct_newton(d, phi, rho, s, 0.05)
    S = SimpleSolver(d, phi, rho, s, 0.05, SolverOpts(exact_inner=exact, eps_out=1e-12, restart=100,
                                                     maxit=2000))
    dphi, drho, ds = S.solve()
    assert S.stats["converged"]
    res = J @ np.concatenate([dphi, drho, ds]) - rhs
    assert np.linalg.norm(res) <= 1e-9 * np.linalg.norm(rhs)
    g = dphi.reshape(d.K + 1, d.N)
    dphi = (g - (g[0] @ d.M) / d.area).reshape(-1)            # gauge of direct.py
    for a, b in ((dphi, dphi0), (drho, drho0), (ds, ds0)):
        assert np.linalg.norm(a - b) <= 1e-7 * np.linalg.norm(b)


def test_simple_and_bb_agree_on_ipm_start():
    """Both preconditioners solve the same Newton system: converged directions agree."""
    p, d = _disc("T2")
    phi, rho, s = initial_state(p, 1.0)
    o = SolverOpts(eps_out=1e-11, maxit=2000)
    a = SimpleSolver(d, phi, rho, s, 1.0, o).solve()
    b = BBSolver(d, phi, rho, s, 1.0, o).solve()
    for x, y in zip(a[1:], b[1:]):
        assert np.linalg.norm(x - y) <= 1e-7 * np.linalg.norm(y)
    gx = a[0].reshape(d.K + 1, d.N)
    gy = b[0].reshape(d.K + 1, d.N)
    gx = gx - (gx[0] @ d.M) / d.area
    gy = gy - (gy[0] @ d.M) / d.area
    assert np.linalg.norm(gx - gy) <= 1e-7 * np.linalg.norm(gy)


def test_hybrid_ipm_reaches_the_same_central_path_point():
    """A34: the BB -> SIMPLE hybrid IPM switches preconditioner below simple_below_mu and
    ends at the same point of the central path as the BB-only run (each mu step's Newton
    loop stops at the same residual tolerance, A18): final KE and rho agree."""
    from oracle.ipm import IpmOpts, ipm_run
    p, d = _disc("T1")
    phi, rho, s = initial_state(p, 1.0)
    thr = 2.0 ** -6 * 1.5
    a = ipm_run(d, phi, rho, s, IpmOpts(mu_min=2.0 ** -12), SolverOpts())
    b = ipm_run(d, phi, rho, s, IpmOpts(mu_min=2.0 ** -12, simple_below_mu=thr), SolverOpts())
    assert all((r["inner_A_its_max"] == 0) == (r["mu"] < thr) for r in b.log)
    assert abs(a.kinetic_energy - b.kinetic_energy) <= 1e-6 * a.kinetic_energy
    assert np.linalg.norm(a.rho - b.rho) <= 1e-4 * np.linalg.norm(a.rho)


def test_stalled_coarsening_jacobi_coarsest_is_exact():
    """I3 / A32: at φ = 0 (A19) B is the pure time difference, so AMG(Ŝ)'s cross-slice
    aggregation collapses every coarse cell's time line and stalls on a DIAGONAL matrix with
    one row per cell; the coarsest "solve" (one l1-Jacobi sweep, ω = 1) is then exact."""
    from oracle import amg
    p, d = _disc("T2")
    phi, rho, s = initial_state(p, 1.0)
    H = amg.setup(S_hat(d, phi, rho, s), np.zeros(d.m, dtype=np.int64), "T", 1.0, 4)
    C = H.levels[-1].A.toarray()
    assert H.sizes[-1] == d.nbar and H.coarse_dense_inv is None
    assert np.count_nonzero(C - np.diag(np.diag(C))) == 0
    b = np.random.default_rng(2).standard_normal(d.nbar)
    x = amg._coarse_solve(H, b)
    assert np.allclose(C @ x, b, rtol=0, atol=1e-12 * np.abs(b).max())
