"""Pins for oracle I1-I6 and a6: Krylov drivers, AMG, BB preconditioner, recovery."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import amg
from oracle.bb import BBSolver, SolverOpts
from oracle.direct import direct_newton
from oracle.krylov import fgmres, pcg_slices
from oracle.ops import Discretisation
from synthetic import initial_state, make_problem, random_state


# ------------------------------------------------------------------ Krylov
def test_fgmres_identity_and_exact_preconditioner():
    """A = I -> 1 iteration; exact inverse as preconditioner -> 1 iteration."""
    rng = np.random.default_rng(0)
    b = rng.standard_normal(50)
    x, its, conv, _ = fgmres(lambda v: v, lambda v: v, b, np.linalg.norm(b), 1e-12, 30, 400)
    assert its == 1 and conv and np.allclose(x, b)
    A = rng.standard_normal((50, 50)) + 10 * np.eye(50)
    Ai = np.linalg.inv(A)
    x, its, conv, _ = fgmres(lambda v: A @ v, lambda v: Ai @ v, b, np.linalg.norm(b), 1e-12, 30, 400)
    assert its == 1 and np.allclose(A @ x, b, atol=1e-10)


def test_fgmres_restart_and_cap():
    """Unpreconditioned nonsymmetric system: converges with restarts; true residual
    <= tol*scale; the cap is honoured and reported (P:1770 '400 limit')."""
    rng = np.random.default_rng(1)
    n = 200
    A = sp.diags([-1.0, 2.5, -1.3], [-1, 0, 1], shape=(n, n)).tocsr()
    b = rng.standard_normal(n)
    x, its, conv, _ = fgmres(lambda v: A @ v, lambda v: v, b, np.linalg.norm(b), 1e-10, 10, 2000)
    assert conv and np.linalg.norm(b - A @ x) <= 1.01e-10 * np.linalg.norm(b) * 10
    x, its, conv, _ = fgmres(lambda v: A @ v, lambda v: v, b, np.linalg.norm(b), 1e-14, 5, 7)
    assert its == 7 and not conv


def test_pcg_slices_matches_direct():
    """Per-slice PCG on independent SPD blocks = K separate CG runs (I4)."""
    rng = np.random.default_rng(2)
    blocks = []
    for k in range(3):
        Q = rng.standard_normal((20, 20))
        blocks.append(Q @ Q.T + (k + 1) * np.eye(20))
    A = sp.block_diag(blocks, format="csr")
    b = rng.standard_normal(60)
    x, its = pcg_slices(lambda v: A @ v, lambda v: v, b, 3, 1e-12, 200)
    assert np.allclose(x, np.linalg.solve(A.toarray(), b), rtol=1e-8)
    assert its.shape == (3,) and np.all(its > 0)
    # freezing: slice with b = 0 does no work
    b2 = b.copy()
    b2[20:40] = 0
    x2, its2 = pcg_slices(lambda v: A @ v, lambda v: v, b2, 3, 1e-12, 200)
    assert its2[1] == 0 and np.all(x2[20:40] == 0)


# --------------------------------------------------------------------- AMG
def _lap1d(n):
    return sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(n, n)).tocsr()


def test_matching_and_galerkin():
    """I3: pairs are mutual and within a slice; every coupled row
    ends in an aggregate of >= 2 rows (attach step); coarse = P^T A P (brute
    force dense); tie-breaking and the attach rule on hand-worked cases."""
    A = sp.block_diag([_lap1d(37), _lap1d(23)], format="csr")
    sl = np.r_[np.zeros(37, int), np.ones(23, int)]
    agg, nc, slc = amg.match(A, sl)
    sizes = np.bincount(agg)
    assert np.all(sizes >= 2) and np.all(sizes <= 4)
    for c in range(nc):
        mem = np.nonzero(agg == c)[0]
        assert len(set(sl[mem])) == 1
        assert np.all(np.diff(mem) == 1)          # 1-D: aggregates are contiguous runs
    H = amg.setup(A, sl, "A", 2 / 3, coarse_max=4)
    P = np.zeros((60, H.levels[0].nc))
    P[np.arange(60), H.levels[0].agg] = 1
    assert np.allclose(H.levels[1].A.toarray(), P.T @ A.toarray() @ P, atol=1e-14)
    # uniform weights: near-ties go to the lowest prio(j) (hash, then index).
    # 1-D, 5 rows, prio order 0 < 3 < 1 < 2 < 4: round 1: 0 -> 1, 1 -> 0 (mutual),
    # 2 -> 3 (prio 3 < 1), 3 -> 2 (prio 2 < 4) (mutual), 4 -> 3; row 4 is left free
    # and joins the pair of its only matched neighbour 3 -> aggregates {0,1},{2,3,4}
    hp = [int(v) >> 32 for v in amg.prio(np.arange(5))]
    assert sorted(range(5), key=lambda j: hp[j]) == [0, 3, 1, 2, 4]
    agg5, nc5, _ = amg.match(_lap1d(5), np.zeros(5, int))
    assert list(agg5) == [0, 0, 1, 1, 1] and nc5 == 2
    # a decoupled row (zero off-diagonals) stays a singleton
    D = sp.block_diag([_lap1d(4), sp.csr_matrix([[1.0]])], format="csr")
    aggD, ncD, _ = amg.match(D, np.zeros(5, int))
    assert list(aggD) == [0, 0, 1, 1, 2] and ncD == 3


def test_vcycle_symmetric_and_convergent():
    """Mode A on a block of weighted Laplacians A_k: the V(1,1) operator is
    symmetric on consistent vectors (CG is legitimate), and PCG reaches
    1e-8 in few iterations."""
    p = make_problem("C1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    _, rho, _ = random_state(p, seed=1)
    A = d.A(rho)
    sl = np.repeat(np.arange(d.K + 1), d.N)
    H = amg.setup(A, sl, "A", 2 / 3, 64)
    assert len(H.levels) >= 3 and max(np.bincount(H.levels[-1].slice_of_row)) <= 64
    rng = np.random.default_rng(3)

    def consistent(v):
        V = v.reshape(d.K + 1, d.N)
        return (V - V.mean(1, keepdims=True)).reshape(-1)
    u, v = consistent(rng.standard_normal(d.n)), consistent(rng.standard_normal(d.n))
    Mu, Mv = consistent(amg.vcycle(H, u)), consistent(amg.vcycle(H, v))
    assert abs(Mu @ v - u @ Mv) < 1e-10 * abs(Mu @ v)
    x, its = pcg_slices(lambda q: A @ q, lambda q: amg.vcycle(H, q), u, d.K + 1, 1e-8, 100)
    assert its.max() < 60
    r = (u - A @ x).reshape(d.K + 1, d.N)
    assert np.all(np.linalg.norm(r, axis=1) <= 1e-8 * np.linalg.norm(u.reshape(d.K + 1, d.N), axis=1))
    # coarsening: >= 2.5x per level on the fine levels (two pairwise passes)
    sz = H.sizes
    assert sz[0] / sz[1] > 2.5 and sz[1] / sz[2] > 2.5


def test_time_blocks_bound_the_T_aggregates(monkeypatch):
    """A42: AMG(T) groups T's rows in time blocks (oracle/amg.py::time_blocks); the build uses
    single-slice blocks (TIME_BLOCK = 1, I3's rule).  With blocks of 2 slices (the machinery
    the GPU shares through bbot_time_blocks) every aggregate on every level lies in one block
    and aggregates do span the slices of a block; with the default every aggregate lies in
    one slice."""
    assert amg.TIME_BLOCK == 1 and list(amg.time_blocks(8)) == list(range(8))
    p = make_problem("T1", L=1, K=16)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    T = d.T_matrix(phi, rho, s)
    for B in (2, 1):
        monkeypatch.setattr(amg, "TIME_BLOCK", B)
        blk = amg.time_blocks(d.K)
        assert list(blk) == [k // B for k in range(16)]
        slT = np.repeat(np.arange(d.K), d.nbar)
        H = amg.setup(T, np.repeat(blk, d.nbar), "T", 1.0, 64)
        spans = False
        member_slice = slT.copy()
        member_block = np.repeat(blk, d.nbar)
        for lv in H.levels[:-1]:
            for c in range(lv.nc):
                mem = np.nonzero(lv.agg == c)[0]
                assert len(set(member_block[mem])) == 1
                spans |= len(set(member_slice[mem])) > 1
            first = np.full(lv.nc, -1)
            for i in range(len(lv.agg) - 1, -1, -1):
                first[lv.agg[i]] = i
            member_block = member_block[first]
            member_slice = member_slice[first]
        assert spans == (B > 1)


# ----------------------------------------------------------- BB / recovery
def test_ideal_preconditioner_two_iterations():
    """(4.18) with the exact projected Schur complement S = -P(C + B A^+ B^T)P^T
    and exact A^+ makes FGMRES converge in 2 iterations."""
    p = make_problem("T0")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=2, mu=0.1)
    S0 = BBSolver(d, phi, rho, s, 0.1, SolverOpts(exact_inner=True))
    A = S0.A.toarray()
    Ap = np.linalg.pinv(A)
    B = S0.B.toarray()
    Pm = np.stack([d.P(e) for e in np.eye(d.m)], 1)
    S = -Pm @ (np.diag(S0.C) + B @ Ap @ B.T) @ Pm.T
    Sp = np.linalg.pinv(S)
    n = d.n

    def U_inv(r):
        y = Pm.T @ (Sp @ r[n:])
        x = Ap @ (r[:n] - B.T @ (Pm.T @ y))
        return np.concatenate([x, y])
    _, its, conv, _ = fgmres(S0.JP, U_inv, S0.rhs, S0.scale, 1e-10, 30, 400)
    assert conv and its == 2


@pytest.mark.parametrize("name,exact", [("T1", True), ("T1", False), ("T2b", False)])
def test_bb_solve_matches_direct(name, exact):
    """BB-FGMRES (4.17) + recovery (a6) reproduces the dense direct solution of
    (3.1) (north star: Krylov vs dense direct on tiny instances)."""
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=7, mu=0.05)
    dphi0, drho0, ds0, J, rhs = direct_newton(d, phi, rho, s, 0.05)
    # restart 100: the T2b random state (vanishing rho_in) stagnates FGMRES(30)
    S = BBSolver(d, phi, rho, s, 0.05, SolverOpts(exact_inner=exact, eps_out=1e-12, restart=100))
    dphi, drho, ds = S.solve()
    assert S.stats["converged"]
    for a, b in ((dphi, dphi0), (drho, drho0), (ds, ds0)):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)
    # the recovered direction satisfies (3.1) (A10, A30)
    res = J @ np.concatenate([dphi, drho, ds]) - rhs
    assert np.linalg.norm(res) <= 1e-9 * np.linalg.norm(rhs)


def test_recovery_residual_equals_projected_residual():
    """A16: after recovery, ||res(3.2)|| = ||res(4.17)|| for an approximate solution."""
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=8, mu=0.05)
    S = BBSolver(d, phi, rho, s, 0.05, SolverOpts(exact_inner=True, eps_out=1e-3))
    dphi, drho, ds = S.solve()
    r417 = S.JP(S.sol) - S.rhs
    J32 = sp.bmat([[S.A, S.B.T], [S.B, -sp.diags(S.C)]]).tocsr()
    r32 = J32 @ np.concatenate([dphi, drho]) - np.concatenate([S.f, S.gt])
    assert abs(np.linalg.norm(r32) / np.linalg.norm(r417) - 1) < 1e-6


@pytest.mark.parametrize("L,K,table", [(1, 4, 6), (2, 8, 8)])
def test_bb_counts_vs_table4(L, K, table):
    """Outer FGMRES iterations at mu = 1 with exact inner solves within a factor 2
    of Table 4's first row (6 and 8 at eps_out = 1e-5), test case 2
    (translated compact bump).  S:605 acceptance band."""
    p = make_problem("T2b", L=L, K=K)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    S = BBSolver(d, phi, rho, s, 1.0, SolverOpts(exact_inner=True, eps_out=1e-5))
    S.solve()
    assert table / 2 <= S.stats["outer_its"] <= 2 * table


@pytest.mark.slow
def test_T_smoother_contracts_on_ipm_path():
    """I3 reading: AMG(T) smooths with l1-Jacobi, x += omega D^-1 (b - T x) with
    D_ii = sum_j |T_ij| and omega = 1 (SolverOpts().omega_T).  Plain damped Jacobi
    (D = diag T, SURVEY's omega = 0.7) breaks along the IPM path: the spectrum of
    diag(T)^-1 T grows past 2/0.7 (T2 at mu = 2^-13: 2.41; C1 at 1.2e-4: 3.09) and on
    C2 at mu = 0.25 diag(T) even has negative entries.  With the l1 diagonal every
    eigenvalue of D^-1 T satisfies |1 - omega lambda| < 1 (Gershgorin gives |lambda| <=
    1; here Re lambda > 0), at mu = 1 and deep in the path."""
    from threadpoolctl import threadpool_limits
    from oracle.ipm import IpmOpts, ipm_run
    from oracle.ops import Discretisation
    from synthetic import initial_state, make_problem
    p = make_problem("T2")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    om = SolverOpts().omega_T
    T0 = d.T_matrix(phi, rho, s).toarray()
    with threadpool_limits(1):
        r = ipm_run(d, phi, rho, s, IpmOpts(mu_min=2.0 ** -13), SolverOpts())
    T = d.T_matrix(r.phi, r.rho, r.s).toarray()
    ev_jac = np.linalg.eigvals(T / np.diag(T)[:, None])
    assert ev_jac.real.max() > 2.0                              # diag-Jacobi's spectrum has grown
    for M in (T0, T):
        H = amg.setup(__import__("scipy.sparse", fromlist=["csr_matrix"]).csr_matrix(M),
                      np.repeat(np.arange(d.K), d.nbar), "T", om, 1024)
        assert np.allclose(H.levels[0].dinv, 1.0 / np.abs(M).sum(1))   # the oracle uses the l1 diagonal
        ev = np.linalg.eigvals(M / np.abs(M).sum(1)[:, None])
        assert ev.real.min() > 0 and np.abs(1.0 - om * ev).max() < 1.0


def _seeded_rhs(d, seed):
    """(f; g; h) in the range of (3.1): Σ_all f = 0 (left kernel (1;0;0), Remark 3.1), but
    nonzero slice sums 1ᵀf^k, so the slice-mass step of solve_rhs is exercised."""
    rng = np.random.default_rng(seed)
    f = rng.standard_normal(d.n)
    f -= f.mean()
    return f, rng.standard_normal(d.m), rng.standard_normal(d.m)


@pytest.mark.parametrize("name", ["T0", "T1"])
def test_solve_rhs_matches_direct(name):
    """solve(rhs) (north star) with a caller-given (f; g; h): the BB-FGMRES
    solve + slice-mass step + recovery reproduces the dense least-squares solve of (3.1)
     in the A11 gauge, and the (3.1) residual is at the FGMRES tolerance."""
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=21, mu=0.05)
    f, g, h = _seeded_rhs(d, 5)
    assert np.abs(f.reshape(d.K + 1, d.N).sum(1)).max() > 1e-3
    S = BBSolver(d, phi, rho, s, 0.05, SolverOpts(eps_out=1e-12))
    dphi, drho, ds = S.solve_rhs(f, g, h)
    assert S.stats["converged"]
    J = d.jacobian(phi, rho, s).toarray()
    rhs = np.concatenate([f, g, h])
    ref, *_ = np.linalg.lstsq(J, rhs, rcond=None)
    n, m = d.n, d.m
    rp = ref[:n].reshape(d.K + 1, d.N)
    rp = (rp - (rp[0] @ d.M) / d.area).reshape(-1)
    for a, b in ((dphi, rp), (drho, ref[n:n + m]), (ds, ref[n + m:])):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)
    res = J @ np.concatenate([dphi, drho, ds]) - rhs
    assert np.linalg.norm(res) <= 1e-9 * np.linalg.norm(rhs)


def test_solve_rhs_newton_rhs_is_plain_solve():
    """With (f; g; h) = -F (the Newton right-hand side of a renormalised state) the slice
    masses m_k are 0 and solve_rhs is the plain Newton solve."""
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=22, mu=0.05)
    S1 = BBSolver(d, phi, rho, s, 0.05)
    a = S1.solve()
    S2 = BBSolver(d, phi, rho, s, 0.05)
    b = S2.solve_rhs(S2.f, S2.g, S2.h)
    for u, v in zip(a, b):
        assert np.allclose(u, v, rtol=0, atol=1e-13 * max(1.0, abs(v).max()))


def test_direct_newton_is_the_least_squares_min_norm_solution():
    """oracle/direct.py (the pin of every Krylov direction): its bordered sparse solve
    [[J, v], [vᵀ, 0]] with the kernel v = (1;0;0) of Remark 3.1 equals the dense
    least-squares minimum-norm solution of (3.1) (then the A11 gauge)."""
    for name in ("T0", "T1"):
        p = make_problem(name)
        d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
        phi, rho, s = random_state(p, seed=7, mu=0.05)
        dphi, drho, ds, J, rhs = direct_newton(d, phi, rho, s, 0.05)
        ref, *_ = np.linalg.lstsq(J.toarray(), rhs, rcond=None)
        n, m = d.n, d.m
        rp = ref[:n].reshape(d.K + 1, d.N)
        rp = (rp - (rp[0] @ d.M) / d.area).reshape(-1)
        for a, b in ((dphi, rp), (drho, ref[n:n + m]), (ds, ref[n + m:])):
            assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)


def test_T_solve_noise_floor():
    """A43: the T-solve of a BB apply stops at max(eps_T ||r2||, 1e-12 ||r||).  At the A19
    point P g~ is zero in exact arithmetic (g~ is proportional to c̄ per slice); rounding-level
    perturbations of r2 then cost no T iterations and leave z unchanged to rounding, while an
    r2 well above the floor is solved to eps_T relative as before."""
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    S = BBSolver(d, phi, rho, s, 1.0)
    r = S.rhs / np.linalg.norm(S.rhs)
    assert np.linalg.norm(r[d.n:]) <= 1e-14          # P g~ = 0 up to rounding
    rng = np.random.default_rng(0)
    z0 = S.apply(r)
    t0 = S.inner_T_its
    rn = r.copy()
    rn[d.n:] += d.P(rng.standard_normal(d.m)) * 1e-15 / np.sqrt(d.m)
    z1 = S.apply(rn)
    assert S.inner_T_its == t0                       # noise: no T iterations
    assert np.linalg.norm(z1 - z0) <= 1e-10 * np.linalg.norm(z0)
    rs = r.copy()
    rs[d.n:] += d.P(rng.standard_normal(d.m)) * 1e-6
    S.apply(rs)
    assert S.inner_T_its > t0                        # a real r2 is solved
