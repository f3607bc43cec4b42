"""GPU edge cases and large-size checks (through the C-ABI):
  * the degenerate sizes the method has: one interior density level (K = 1), the
    8-triangle base mesh (L = 0), a coarsest AMG level that is level 0;
  * input errors: obtuse / clockwise meshes (BBOT_E_GEOMETRY), negative densities
    (BBOT_E_INPUT), non-positive state (BBOT_E_STATE), call order (BBOT_E_ORDER),
    option ranges (BBOT_E_INPUT);
  * host (numpy) and device (torch) buffers give identical results;
  * at C3 size (8.5 M unknowns, K = 64) -- too large for the oracle's FGMRES in a
    test -- the recovered GPU direction is checked with the ORACLE's own Jacobian
    (3.1): ||J d - (f;g;h)|| <= eps-level x ||(f;g;h)|| (a property that holds at
    any size: A16, the (4.17) residual equals the (3.2) residual after recovery).
Oracle imports are test infrastructure."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from threadpoolctl import threadpool_limits                      # noqa: E402

from oracle.bb import BBSolver, SolverOpts                       # noqa: E402
from oracle.ops import Discretisation                            # noqa: E402
from synthetic import initial_state, make_problem, random_state  # noqa: E402


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2209_00315_b200 as pb
    return pb


@pytest.mark.parametrize("name,L,K", [("T0", 0, 1), ("T0", 0, 2), ("T1", 1, 1)])
def test_degenerate_sizes_direction_parity(name, L, K):
    pb = _gpu()
    p = make_problem(name, L=L, K=K)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=7, mu=0.1)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(phi, rho, s, 0.1)
    ctx.assemble()
    assert ctx.amg_info(1) == [d.m]           # T fits the dense coarsest: level 0 is coarsest
    dphi, drho, ds, st = ctx.solve()
    with threadpool_limits(1):
        S = BBSolver(d, phi, rho, s, 0.1, SolverOpts())
        ophi, orho, os_ = S.solve()
    assert st["converged"] == 1 and abs(st["outer_its"] - S.stats["outer_its"]) <= 1
    for a, b in ((dphi, ophi), (drho, orho), (ds, os_)):
        assert np.linalg.norm(a - b) <= 1e-8 * max(np.linalg.norm(b), 1e-300)


def test_input_errors():
    pb = _gpu()
    p = make_problem("T0")
    # an obtuse triangle: move an interior vertex far off -> geometry rejected
    v = p.verts.copy()
    v[6] = [0.05, 0.5]
    with pytest.raises(pb.BbotError) as e:
        pb.Context(v, p.tris, p.K, p.rho_in, p.rho_f)
    assert e.value.status == 2
    # clockwise triangles
    with pytest.raises(pb.BbotError) as e:
        pb.Context(p.verts, p.tris[:, ::-1].copy(), p.K, p.rho_in, p.rho_f)
    assert e.value.status == 2
    bad = p.rho_in.copy()
    bad[0] = -1.0
    with pytest.raises(pb.BbotError) as e:
        pb.Context(p.verts, p.tris, p.K, bad, p.rho_f)
    assert e.value.status == 1
    with pytest.raises(pb.BbotError) as e:
        pb.Context(p.verts, p.tris, 0, p.rho_in, p.rho_f)
    assert e.value.status == 1
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    with pytest.raises(pb.BbotError) as e:
        ctx.set_opts(pb.default_solver_opts(restart=64))       # > 32: not supported
    assert e.value.status == 1
    with pytest.raises(pb.BbotError) as e:
        ctx.newton_update(0.95)                                 # no direction yet
    assert e.value.status == 9
    phi, rho, s = initial_state(p, 1.0)
    s[0] = 0.0
    with pytest.raises(pb.BbotError) as e:
        ctx.set_state(phi, rho, s, 1.0)
    assert e.value.status == 3


def test_host_and_device_buffers_identical():
    import torch
    pb = _gpu()
    p = make_problem("C1")
    phi, rho, s = random_state(p, seed=11, mu=1e-2)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(phi, rho, s, 1e-2)
    ctx.assemble()
    h = ctx.solve()
    dev = [torch.tensor(x, device="cuda") for x in (phi, rho, s)]
    ctx.set_state(*dev, 1e-2)
    ctx.assemble()
    out = [torch.empty(ctx.n, dtype=torch.float64, device="cuda"),
           torch.empty(ctx.m, dtype=torch.float64, device="cuda"),
           torch.empty(ctx.m, dtype=torch.float64, device="cuda")]
    g = ctx.solve(*out)
    for a, b in zip(h[:3], g[:3]):
        assert np.array_equal(a, b.cpu().numpy())
    assert h[3]["outer_its"] == g[3]["outer_its"]


def test_C3_direction_satisfies_newton_system():
    """BASELINE configs[2] size (C3: 32768 cells, K = 64, 8.5 M unknowns, compact
    cos^2 bumps with vanishing regions): the GPU direction of the first IPM system,
    checked against the ORACLE's Jacobian (3.1) and right-hand side."""
    import scipy.sparse as sp  # noqa: F401
    pb = _gpu()
    p = make_problem("C3")
    phi, rho, s = initial_state(p, 1.0)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(phi, rho, s, 1.0)
    ctx.assemble()
    dphi, drho, ds, st = ctx.solve()
    assert st["converged"] == 1
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    J = d.jacobian(phi, rho, s)
    f, g, h, _ = d.newton_rhs(phi, rho, s, 1.0)
    rhs = np.concatenate([f, g, h])
    res = J @ np.concatenate([dphi, drho, ds]) - rhs
    # FGMRES stops at 1e-10 on (4.17); the (3.1) residual after recovery is the same
    # quantity (A16) up to rounding in the recovery
    assert np.linalg.norm(res) <= 1e-8 * np.linalg.norm(rhs), np.linalg.norm(res) / np.linalg.norm(rhs)
    # kernel of J (Remark 3.1): the gauge fixes delta phi^1 to zero c-weighted mean (A11)
    assert abs(d.M @ dphi[:d.N]) <= 1e-10 * np.abs(dphi).max() * d.M.sum()
    # north star counts: the oracle's own solve of this system (scripts/oracle_counts.py, oracle
    # only, ~15 min on one core; tests/golden/oracle_counts.json)
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_counts.json")))
    o = gold.get("C3/init/mu=1")
    if o is not None:
        assert o["converged"] and abs(st["outer_its"] - o["outer_its"]) <= 1, (st, o)




def test_C4_first_system_counts_match_oracle():
    """The bench headline system (BASELINE configs[3], C4: 131 072 cells, K = 128, 67.5 M
    unknowns): the GPU's first IPM Newton solve converges with the oracle's own outer count
    +-1 (tests/golden/oracle_counts.json: scripts/oracle_counts.py, oracle only, 7094 s and
    ~30 GB on one core) and the same inner T-GMRES count within the +-1 outer slack."""
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_counts.json")))
    o = gold.get("C4/init/mu=1")
    if o is None:
        pytest.skip("C4 oracle counts not generated")
    pb = _gpu()
    p = make_problem("C4")
    phi, rho, s = initial_state(p, 1.0)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(phi, rho, s, 1.0)
    ctx.assemble()
    st = ctx.solve_stats_only()
    print("C4 gpu", {k: st[k] for k in ("outer_its", "inner_T_its", "inner_A_its_max", "rel_res")}, "oracle", o)
    assert o["converged"] and st["converged"] == 1
    assert abs(st["outer_its"] - o["outer_its"]) <= 1, (st, o)
    assert abs(st["inner_T_its"] - o["inner_T_its"]) <= 50, (st, o)
    if st["outer_its"] == o["outer_its"]:
        # same iterate on both sides: the FGMRES residual estimate and the per-slice PCG work agree
        # (measured: counts 28 / 553 on both sides, PCG slice-iterations 123 213 vs 123 193,
        # relative residuals 5.46331e-11 vs 5.46332e-11)
        assert abs(st["rel_res"] - o["rel_res"]) <= 1e-3 * o["rel_res"], (st["rel_res"], o["rel_res"])
        assert abs(st["inner_A_its_total"] - o["inner_A_its_total"]) <= 0.01 * o["inner_A_its_total"], (st, o)
