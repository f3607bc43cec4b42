"""a7: interior-point continuation with inexact Newton steps.

PAPER.md P:59, P:192 (log-barrier, mu -> 0), P:552-569 (inexact Newton),
P:571-584 (Remark 3.2: renormalise rho after each Newton update).
Readings: A17 mu_j = mu0 * 0.5^j down to >= mu_min;
A18 at least one Newton step per mu, stop when ||F(x;mu)|| <= max(1e-2 mu, 1e-11)
* ||F(x_init; mu0)||, cap newton_max; A19 initial point; A20 fraction-to-boundary
0.95 on rho and s, no line search; A14': the A_k solves of the BB apply tighten from
eps_A (1e-3) to eps_A_tight (1e-5) once mu < mu_tight (0.3) -- the Newton systems'
conditioning grows as mu -> 0 and the outer FGMRES needs a more accurate
preconditioner (C2 at mu = 0.25: 400-cap at 1e-3, 74 iterations at 1e-5).
A34: the mu-switched BB -> SIMPLE hybrid ("SIMPLE ... becomes
faster in the last IP iterations"): SIMPLE (oracle/simple.py) once mu < simple_below_mu.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .bb import BBSolver, SolverOpts
from .hss import HssSolver
from .simple import SimpleSolver
from .ops import Discretisation


@dataclass
class IpmOpts:
    mu0: float = 1.0
    mu_factor: float = 0.5
    mu_min: float = 1e-8
    newton_rel_tol: float = 1e-2
    newton_abs_floor: float = 1e-11
    frac_to_boundary: float = 0.95
    newton_max: int = 30
    max_mu_steps: int | None = None     # truncate the schedule (tests)
    mu_tight: float = 0.3               # A14': below this mu the A_k solves tighten ...
    eps_A_tight: float = 1e-5           # ... to this relative tolerance
    simple_below_mu: float = 0.0        # A34: SIMPLE instead of BB once mu < this (0 = never)


def step_length(rho, s, drho, ds, tau):
    """alpha = min(1, tau * min_{d_i<0} (-x_i/d_i)) over rho and s (A20)."""
    a = 1.0
    for x, dx in ((rho, drho), (s, ds)):
        neg = dx < 0
        if neg.any():
            a = min(a, tau * float(np.min(-x[neg] / dx[neg])))
    return a


def renormalise(d: Discretisation, rho):
    """ρ^k *= (c̄^T ρ^0)/(c̄^T ρ^k)  (Remark 3.2)."""
    R = np.asarray(rho).reshape(d.K, d.nbar)
    target = float(d.Mbar @ d.rho0)
    return (R * (target / (R @ d.Mbar))[:, None]).reshape(-1)


def res_norm(d, phi, rho, s, mu):
    a, b, c = d.residual(phi, rho, s, mu)
    return float(np.sqrt(a @ a + b @ b + c @ c))


def newton_step(d: Discretisation, phi, rho, s, mu, opts: SolverOpts, tau: float, keep=None):
    S = {"simple": SimpleSolver, "hss": HssSolver}.get(opts.precond, BBSolver)(d, phi, rho, s, mu, opts)
    dphi, drho, ds = S.solve()
    if keep is not None:            # test hook: the system solved and its direction
        keep.update(state=(phi, rho, s), mu=mu, opts=opts, direction=(dphi, drho, ds))
    alpha = step_length(rho, s, drho, ds, tau)
    phi = phi + alpha * dphi
    rho = renormalise(d, rho + alpha * drho)
    s = s + alpha * ds
    return phi, rho, s, alpha, S.stats


def mu_schedule(o: IpmOpts):
    mus = []
    mu = o.mu0
    j = 0
    while mu >= o.mu_min * (1 - 1e-12):
        mus.append(mu)
        j += 1
        mu = o.mu0 * o.mu_factor ** j
    if o.max_mu_steps is not None:
        mus = mus[:o.max_mu_steps]
    return mus


@dataclass
class IpmResult:
    phi: np.ndarray
    rho: np.ndarray
    s: np.ndarray
    mu: float
    kinetic_energy: float
    log: list = field(default_factory=list)


def ipm_run(d: Discretisation, phi, rho, s, ipm: IpmOpts | None = None,
            opts: SolverOpts | None = None, callback=None, keep_systems: bool = False) -> IpmResult:
    """keep_systems: every log record also carries the Newton system it solved
    ("system": dict(state=(phi, rho, s), mu, opts, direction)) -- test infrastructure
    for per-system parity along the oracle's own trajectory."""
    ipm = ipm or IpmOpts()
    opts = opts or SolverOpts()
    F0 = res_norm(d, phi, rho, s, ipm.mu0)
    log = []
    mu = ipm.mu0
    for mu in mu_schedule(ipm):
        tol = max(ipm.newton_rel_tol * mu, ipm.newton_abs_floor) * F0
        for it in range(ipm.newton_max):
            o_mu = opts if mu >= ipm.mu_tight else replace(opts, eps_A=min(opts.eps_A, ipm.eps_A_tight))
            if mu < ipm.simple_below_mu:
                o_mu = replace(o_mu, precond="simple")
            keep = {} if keep_systems else None
            phi, rho, s, alpha, st = newton_step(d, phi, rho, s, mu, o_mu, ipm.frac_to_boundary, keep)
            r = res_norm(d, phi, rho, s, mu)
            rec = dict(mu=mu, newton=it, alpha=alpha, res=r, **st)
            if keep_systems:
                rec["system"] = keep
            log.append(rec)
            if callback:
                callback(rec)
            if r <= tol:
                break
    ke = d.kinetic_energy(phi, rho)
    return IpmResult(phi=phi, rho=rho, s=s, mu=mu, kinetic_energy=ke, log=log)
