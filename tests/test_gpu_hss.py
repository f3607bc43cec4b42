"""GPU parity of NEXT row f2 -- the HSS preconditioner (§5.1) on the
saddle-point system, diagonally scaled -- against oracle/hss.py.
Tolerances as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

from oracle import amg as oamg                        # noqa: E402
from oracle.bb import SolverOpts                      # noqa: E402
from oracle.hss import HssSolver                      # noqa: E402
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


def _ctx(name, state="random", mu=1e-2, seed=3, eps_out=1e-10):
    pb = _gpu()
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=seed, mu=mu) if state == "random" else initial_state(p, mu)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, opts=pb.default_solver_opts(precond=2, eps_out=eps_out))
    ctx.set_state(phi, rho, s, mu)
    return pb, p, d, ctx, (phi, rho, s, mu)


@pytest.mark.parametrize("name", ["T1", "C1", "T2b"])
def test_SK_and_J_parity(name):
    """S_K = alpha I + B^ B^T / alpha (eq:solve-K, scaled) entrywise; J x (eq:saddle-point)."""
    pb, p, d, ctx, (phi, rho, s, mu) = _ctx(name)
    ctx.assemble()
    rp, ci, cv = ctx.get_T()
    Sg = sp.csr_matrix((cv, ci, rp), shape=(d.m, d.m))
    H = HssSolver(d, phi, rho, s, mu, SolverOpts(precond="hss"))
    assert abs(Sg - H.SK).max() <= 1e-12 * abs(H.SK).max()
    x = np.random.default_rng(11).standard_normal(d.n + d.m)
    assert _rel(ctx.jp_matvec(x), H.matvec(x)) < 1e-12


@pytest.mark.parametrize("name", ["T1", "C1"])
def test_hss_amg_and_apply_parity(name):
    """AMG(A^ + alpha I) (mode As) and AMG(S_K): identical aggregates on every level, V-cycles
    to 1e-10 / 2e-9; one HSS apply to 1e-8 with identical inner counts."""
    pb, p, d, ctx, (phi, rho, s, mu) = _ctx(name)
    ctx.assemble()
    H = HssSolver(d, phi, rho, s, mu, SolverOpts(precond="hss"))
    for which, Hh, tol in ((0, H.amgH, 1e-10), (1, H.amgK, 2e-9)):
        sizes = ctx.amg_info(which)
        assert sizes == Hh.sizes, (which, sizes, Hh.sizes)
        for lvl in range(len(sizes) - 1):
            assert np.array_equal(ctx.amg_agg(which, lvl), Hh.levels[lvl].agg), (which, lvl)
        b = np.random.default_rng(5 + which).standard_normal(sizes[0])
        assert _rel(ctx.amg_vcycle(which, b), oamg.vcycle(Hh, b)) < tol, which
    r = np.random.default_rng(9).standard_normal(d.n + d.m)
    zg, itK, itH = ctx.bb_apply(r)
    zo = H.apply(r)
    assert itK == H.inner_T_its and itH == int(H.inner_A_its[-1].max()), (itK, itH, H.inner_T_its)
    assert _rel(zg, zo) < 1e-8


def _ipm_state(name, mu_target):
    from oracle.ipm import IpmOpts, ipm_run
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    if mu_target < 1.0:
        r = ipm_run(d, phi, rho, s, IpmOpts(mu_min=mu_target), SolverOpts())
        phi, rho, s = r.phi, r.rho, r.s
    return p, d, phi, rho, s


# HSS needs many more outer iterations than BB (22-264 on average at eps_out = 1e-5,
# growing with refinement); at C1 mu = 1 eps_out = 1e-10 is not reached within 400 on either
# side, so that case runs at the paper's own eps_out = 1e-5
@pytest.mark.parametrize("name,mu,eps", [("T1", 1.0, 1e-10), ("T1", 2.0 ** -6, 1e-10), ("T2", 2.0 ** -4, 1e-10),
                                         ("C1", 1.0, 1e-5), ("C1", 2.0 ** -3, 1e-10)])
def test_hss_direction_parity(name, mu, eps):
    """Newton direction through HSS-FGMRES + δs elimination on IPM states (the next system,
    mu/2): relative 1e-8 per block, outer counts +-1 (north star)."""
    pb = _gpu()
    p, d, phi, rho, s = _ipm_state(name, mu)
    mu_sys = mu / 2 if mu < 1.0 else 1.0
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, opts=pb.default_solver_opts(precond=2, eps_out=eps))
    ctx.set_state(phi, rho, s, mu_sys)
    ctx.assemble()
    dphi, drho, ds, st = ctx.solve()
    H = HssSolver(d, phi, rho, s, mu_sys, SolverOpts(precond="hss", eps_out=eps))
    ophi, orho, os_ = H.solve()
    print(name, mu_sys, "outer gpu/oracle", st["outer_its"], H.stats["outer_its"], "inner K/H",
          st["inner_T_its"], H.stats["inner_T_its"], st["inner_A_its_max"], H.stats["inner_A_its_max"])
    assert H.stats["converged"] and st["converged"] == 1, (st, H.stats)
    assert abs(st["outer_its"] - H.stats["outer_its"]) <= 1, (st, H.stats)
    for a, b in ((dphi, ophi), (drho, orho), (ds, os_)):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b), np.linalg.norm(a - b) / np.linalg.norm(b)


def test_hss_graph_and_eager_identical():
    """The captured CUDA-graph HSS solve and the eager issue are bitwise identical."""
    pb = _gpu()
    p, d, phi, rho, s = _ipm_state("T2", 2.0 ** -3)
    out = []
    for graph in (True, False):
        ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, opts=pb.default_solver_opts(precond=2))
        ctx.set_exec_mode(graph)
        ctx.set_state(phi, rho, s, 2.0 ** -4)
        ctx.assemble()
        out.append(ctx.solve())
    for a, b in zip(out[0][:3], out[1][:3]):
        assert np.array_equal(a, b)
    assert out[0][3]["outer_its"] == out[1][3]["outer_its"]
