"""Pins for oracle a7: IPM continuation, renormalisation, kinetic energy."""
import numpy as np
import pytest

from oracle.bb import SolverOpts
from oracle.ipm import IpmOpts, ipm_run, mu_schedule, renormalise, step_length
from oracle.ops import Discretisation
from synthetic import initial_state, make_problem


def test_mu_schedule():
    """A17: mu_j = 2^-j, j = 0..26; the last one 1.49e-8 >= 1e-8."""
    mus = mu_schedule(IpmOpts())
    assert len(mus) == 27 and mus[0] == 1.0 and abs(mus[-1] - 2.0 ** -26) < 1e-20
    assert all(abs(b / a - 0.5) < 1e-15 for a, b in zip(mus, mus[1:]))


def test_step_length_examples():
    """δ >= 0 -> α = 1;  ρ = (1,1), δρ = (-2, 1), τ = 0.95 -> α = 0.475."""
    one = np.ones(2)
    assert step_length(one, one, one, one, 0.95) == 1.0
    assert abs(step_length(one, one, np.array([-2.0, 1.0]), one, 0.95) - 0.475) < 1e-15


def test_renormalise():
    """Remark 3.2: after renormalisation every slice has the boundary mass."""
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    rho = np.random.default_rng(0).uniform(0.5, 2.0, d.m)
    r = renormalise(d, rho)
    assert np.allclose(d.slice_mass(r), d.Mbar @ d.rho0, rtol=1e-14)


@pytest.fixture(scope="module")
def ipm_t1():
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    masses, gaps = [], []

    def cb(rec):
        pass
    res = ipm_run(d, phi, rho, s, IpmOpts(mu_min=2.0 ** -10), SolverOpts(eps_out=1e-10), cb)
    return d, res


def test_ipm_invariants(ipm_t1):
    """Mass conserved to 1e-13 (Remark 2.2/3.2); ρ, s > 0; the final iterate is
    near the central path: Σ c̄ ρ s ≈ μ |Ω| K (F_s = 0 gives it exactly)."""
    d, res = ipm_t1
    assert np.allclose(d.slice_mass(res.rho), d.Mbar @ d.rho0, rtol=1e-13)
    assert res.rho.min() > 0 and res.s.min() > 0
    gap = np.tile(d.Mbar, d.K) @ (res.rho * res.s)
    assert abs(gap / (res.mu * d.area * d.K) - 1) < 1e-2
    # Newton converges: each mu needs few steps, the final residual meets A18
    per_mu = {}
    for r in res.log:
        per_mu[r["mu"]] = per_mu.get(r["mu"], 0) + 1
    assert len(per_mu) == 11 and max(per_mu.values()) <= 8


def test_ipm_gap_halves(ipm_t1):
    """The duality gap Σ c̄ ρ s follows μ: it halves per IP step (A17)."""
    d, res = ipm_t1
    # rerun 3 IP steps and record the gap at the end of each
    p = make_problem("T1")
    phi, rho, s = initial_state(p, 1.0)
    gaps = []
    for j in range(1, 4):
        r = ipm_run(d, phi, rho, s, IpmOpts(mu_min=2.0 ** -j), SolverOpts())
        gaps.append(np.tile(d.Mbar, d.K) @ (r.rho * r.s))
    assert all(abs(b / a - 0.5) < 0.05 for a, b in zip(gaps, gaps[1:]))


def test_kinetic_energy_translation_closed_form():
    """Test case 2: a translated density; the OT cost is ½|t|²·mass
     = ½·0.32 = 0.16 for t = (0.4, 0.4).  The discrete KE (D12)
    approaches it under joint (h, Δt) refinement."""
    kes = []
    for L, K in [(1, 4), (2, 8)]:
        p = make_problem("T2b", L=L, K=K)
        d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
        phi, rho, s = initial_state(p, 1.0)
        r = ipm_run(d, phi, rho, s, IpmOpts(mu_min=1e-3), SolverOpts(eps_out=1e-8))
        kes.append(r.kinetic_energy)
    err = [abs(k - 0.16) for k in kes]
    assert err[1] < err[0] and err[1] < 0.15 * 0.16 * 1.5, kes


def compression_cost(radius, theta):
    """Closed-form OT cost of test case 3: the optimal map of a density
    onto its dilation x -> c + theta (x - c) is that dilation, so the cost is
    ((1 - theta)^2 / 2) E|x - c|^2 under the unit-mass rho_in.  For the cos^2 bump of
    radius r0 (u = r / r0):  E|x - c|^2 = r0^2 * int_0^1 cos^2(pi u/2) u^3 du /
    int_0^1 cos^2(pi u/2) u du = r0^2 (1/8 - 3/(2 pi^2) + 6/pi^4) / (1/4 - 1/pi^2)."""
    pi = np.pi
    e2 = radius ** 2 * (1 / 8 - 3 / (2 * pi ** 2) + 6 / pi ** 4) / (1 / 4 - 1 / pi ** 2)
    return 0.5 * (1 - theta) ** 2 * e2


def test_compression_cost_closed_form_by_quadrature():
    """The closed form above against a direct 2-D quadrature of the bump's second moment."""
    from synthetic.densities import cos2_bump
    f = cos2_bump(0.5, 0.5, 0.35)
    x = (np.arange(4000) + 0.5) / 4000
    X, Y = np.meshgrid(x, x)
    w = f(X, Y)
    e2 = float((w * ((X - 0.5) ** 2 + (Y - 0.5) ** 2)).sum() / w.sum())
    assert abs(0.5 * 0.25 * e2 - compression_cost(0.35, 0.5)) < 1e-6 * compression_cost(0.35, 0.5)


def test_kinetic_energy_compression_closed_form():
    """Test case 3, compression: the discrete KE (D12) at the end of
    the IPM approaches the closed-form cost under joint (h, Δt) refinement (measured: +60 %
    at L=1/K=4, +34 % at L=2/K=8, +24 % at L=3/K=8 -- the compressed target is 2-4 coarse
    cells across; the paper reports this case as the hardest)."""
    exact = compression_cost(0.35, 0.5)
    kes = []
    for L, K in [(1, 4), (2, 8)]:
        p = make_problem("T2c", L=L, K=K)
        d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
        phi, rho, s = initial_state(p, 1.0)
        r = ipm_run(d, phi, rho, s, IpmOpts(mu_min=1e-3), SolverOpts(eps_out=1e-8))
        kes.append(r.kinetic_energy)
    err = [k / exact - 1 for k in kes]
    assert 0 < err[1] < err[0] and err[1] < 0.4, (kes, exact)


def test_inner_tolerance_tightens_below_mu_tight(monkeypatch):
    """A14': the BB apply's A_k solves use eps_A while mu >= mu_tight and
    min(eps_A, eps_A_tight) below it."""
    import oracle.ipm as ipm_mod
    from oracle.bb import SolverOpts
    from oracle.ipm import IpmOpts, ipm_run
    from oracle.ops import Discretisation
    from synthetic import initial_state, make_problem
    seen = []
    real = ipm_mod.newton_step

    def spy(d, phi, rho, s, mu, opts, tau, keep=None):
        seen.append((mu, opts.eps_A))
        return real(d, phi, rho, s, mu, opts, tau, keep)
    monkeypatch.setattr(ipm_mod, "newton_step", spy)
    p = make_problem("T0")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    ipm_run(d, phi, rho, s, IpmOpts(max_mu_steps=4), SolverOpts())
    o, io = SolverOpts(), IpmOpts()
    assert {m for m, _ in seen} == {1.0, 0.5, 0.25, 0.125}
    for mu, eps in seen:
        assert eps == (o.eps_A if mu >= io.mu_tight else min(o.eps_A, io.eps_A_tight))
