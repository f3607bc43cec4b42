"""GPU parity of NEXT row f4 -- the harmonic reconstruction (Remark 3.3;
DESIGN.md A39-A41) with the BB preconditioner -- against oracle/ops.py (recon="harm").
Tolerances as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

from threadpoolctl import threadpool_limits           # noqa: E402

from oracle import amg as oamg                        # noqa: E402
from oracle.bb import BBSolver, SolverOpts            # noqa: E402
from oracle.ops import Discretisation                 # noqa: E402
from synthetic import initial_state, make_problem, random_state   # noqa: E402


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2209_00315_b200 as pb
    return pb


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _setup(name, seed=3, mu=1e-2):
    pb = _gpu()
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f, recon="harm")
    phi, rho, s = random_state(p, seed=seed, mu=mu)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, opts=pb.default_solver_opts(recon=1))
    ctx.set_state(phi, rho, s, mu)
    return pb, p, d, ctx, (phi, rho, s, mu)


@pytest.mark.parametrize("name", ["T1", "C1", "T2b"])
def test_harmonic_operators_parity(name):
    """Residuals (2.5)-(2.7) on R_H, the kinetic energy, T (diag(C_H), R̄_H, J_f) entrywise and
    J_P x with the C_H = C - W block: relative 1e-12."""
    pb, p, d, ctx, (phi, rho, s, mu) = _setup(name)
    Fp, Fr, Fs, nrm = ctx.residual()
    op, orr, os_ = d.residual(phi, rho, s, mu)
    assert _rel(Fp, op) < 1e-12 and _rel(Fr, orr) < 1e-12 and _rel(Fs, os_) < 1e-12
    assert abs(ctx.kinetic_energy() - d.kinetic_energy(phi, rho)) <= 1e-12 * d.kinetic_energy(phi, rho)
    ctx.assemble()
    rp, ci, cv = ctx.get_T()
    Tg = sp.csr_matrix((cv, ci, rp), shape=(d.m, d.m))
    To = d.T_matrix(phi, rho, s)
    assert abs(Tg - To).max() <= 1e-12 * abs(To).max()
    JP, *_ = d.make_JP(phi, rho, s)
    x = np.random.default_rng(11).standard_normal(d.n + d.m)
    assert _rel(ctx.jp_matvec(x), JP(x)) < 1e-12


@pytest.mark.parametrize("name", ["T1", "C1"])
def test_harmonic_amg_and_bb_apply_parity(name):
    pb, p, d, ctx, (phi, rho, s, mu) = _setup(name)
    ctx.assemble()
    S = BBSolver(d, phi, rho, s, mu, SolverOpts())
    for which, H in ((0, S.amgA), (1, S.amgT)):
        sizes = ctx.amg_info(which)
        assert sizes == H.sizes, (which, sizes, H.sizes)
        for lvl in range(len(sizes) - 1):
            assert np.array_equal(ctx.amg_agg(which, lvl), H.levels[lvl].agg), (which, lvl)
    r = np.random.default_rng(9).standard_normal(d.n + d.m)
    r[d.n:] = d.P(r[d.n:])
    zg, itT, itA = ctx.bb_apply(r)
    zo = S.apply(r)
    assert itT == S.inner_T_its and itA == int(S.inner_A_its[-1].max())
    assert _rel(zg, zo) < 1e-8


def _ipm_state(name, mu_target):
    from oracle.ipm import IpmOpts, ipm_run
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f, recon="harm")
    phi, rho, s = initial_state(p, 1.0)
    if mu_target < 1.0:
        with threadpool_limits(1):
            r = ipm_run(d, phi, rho, s, IpmOpts(mu_min=mu_target), SolverOpts())
        phi, rho, s = r.phi, r.rho, r.s
    return p, d, phi, rho, s


@pytest.mark.parametrize("name,mu", [("T1", 2.0 ** -6), ("T2", 2.0 ** -4), ("C1", 2.0 ** -3)])
def test_harmonic_newton_direction_parity(name, mu):
    """North star on the harmonic problem: the Newton direction of the next IPM system (the
    oracle's own harmonic trajectory) to 1e-8 per block, outer counts +-1."""
    pb = _gpu()
    p, d, phi, rho, s = _ipm_state(name, mu)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, opts=pb.default_solver_opts(recon=1))
    ctx.set_state(phi, rho, s, mu / 2)
    ctx.assemble()
    dphi, drho, ds, st = ctx.solve()
    S = BBSolver(d, phi, rho, s, mu / 2, SolverOpts())
    o = S.solve()
    assert S.stats["converged"] and st["converged"] == 1
    assert abs(st["outer_its"] - S.stats["outer_its"]) <= 1, (st, S.stats)
    for a, b in zip((dphi, drho, ds), o):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b), np.linalg.norm(a - b) / np.linalg.norm(b)


def test_harmonic_ipm_parity_T1():
    """The full IPM (mu 1 -> 2^-12) with R_H on both sides: outer counts +-1 per system, final
    kinetic energy to 1e-6 (north star)."""
    from oracle.ipm import IpmOpts, ipm_run
    pb = _gpu()
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f, recon="harm")
    phi, rho, s = initial_state(p, 1.0)
    with threadpool_limits(1):
        res = ipm_run(d, phi, rho, s, IpmOpts(mu_min=2.0 ** -12), SolverOpts())
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, opts=pb.default_solver_opts(recon=1))
    ctx.set_state(phi, rho, s, 1.0)
    st, log = ctx.ipm_run(pb.default_ipm_opts(mu_min=2.0 ** -12))
    assert st["n_systems"] == len(res.log)
    for g, o in zip(log, res.log):
        assert abs(g["outer_its"] - o["outer_its"]) <= 1, (g, o)
    assert abs(st["kinetic_energy"] - res.kinetic_energy) <= 1e-6 * abs(res.kinetic_energy)


def test_harmonic_solve_rhs_parity():
    """solve(rhs) with R_H (slice-mass step with W δρ₀) against the oracle."""
    pb = _gpu()
    p, d, phi, rho, s = _ipm_state("T1", 2.0 ** -6)
    rng = np.random.default_rng(17)
    f = rng.standard_normal(d.n)
    f -= f.mean()
    g, h = rng.standard_normal(d.m), rng.standard_normal(d.m)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, opts=pb.default_solver_opts(recon=1))
    ctx.set_state(phi, rho, s, 2.0 ** -7)
    ctx.assemble()
    out = ctx.solve_rhs(f, g, h)
    S = BBSolver(d, phi, rho, s, 2.0 ** -7, SolverOpts())
    o = S.solve_rhs(f, g, h)
    assert abs(out[3]["outer_its"] - S.stats["outer_its"]) <= 1
    for a, b in zip(out[:3], o):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)
