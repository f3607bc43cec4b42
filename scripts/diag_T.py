#!/usr/bin/env python
"""Diagnostic: AMG(T) and the inner T-GMRES of one BB apply, GPU vs oracle, on a config's
first Newton system (A19 point, mu = 1): hierarchy sizes, aggregates per level, one
V-cycle, inner T / A counts of a BB apply on seeded right-hand sides.

    python scripts/diag_T.py C2
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(name):
    import torch
    torch.cuda.set_device(0)
    import paper_2209_00315_b200 as pb
    from oracle import amg as oamg
    from oracle.bb import BBSolver, SolverOpts
    from oracle.ops import Discretisation
    from synthetic import initial_state, make_problem
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(phi, rho, s, 1.0)
    ctx.assemble()
    S = BBSolver(d, phi, rho, s, 1.0, SolverOpts())
    sizes = ctx.amg_info(1)
    print("T sizes gpu", sizes, "oracle", S.amgT.sizes)
    for lvl in range(min(len(sizes), len(S.amgT.sizes)) - 1):
        print("  level", lvl, "aggregates equal", np.array_equal(ctx.amg_agg(1, lvl), S.amgT.levels[lvl].agg))
    b = np.random.default_rng(5).standard_normal(sizes[0])
    xg, xo = ctx.amg_vcycle(1, b), oamg.vcycle(S.amgT, b)
    print("V-cycle rel", float(np.max(np.abs(xg - xo)) / np.max(np.abs(xo))))
    for seed in range(4):
        r = np.random.default_rng(seed).standard_normal(d.n + d.m)
        r[d.n:] = d.P(r[d.n:])
        S.inner_T_its = 0
        zg, itT, itA = ctx.bb_apply(r)
        zo = S.apply(r)
        print("apply seed", seed, "T its gpu", itT, "oracle", S.inner_T_its, "A max gpu", itA,
              "oracle", int(S.inner_A_its[-1].max()), "rel", float(np.max(np.abs(zg - zo)) / np.max(np.abs(zo))))

    # restarted T-GMRES(10): a tight inner tolerance forces restarts
    o = pb.default_solver_opts(eps_T=1e-4)
    ctx.set_opts(o)
    ctx.assemble()
    S2 = BBSolver(d, phi, rho, s, 1.0, SolverOpts(eps_T=1e-4))
    for seed in range(2):
        r = np.random.default_rng(seed).standard_normal(d.n + d.m)
        r[d.n:] = d.P(r[d.n:])
        S2.inner_T_its = 0
        zg, itT, itA = ctx.bb_apply(r)
        zo = S2.apply(r)
        print("eps_T=1e-4 apply seed", seed, "T its gpu", itT, "oracle", S2.inner_T_its,
              "rel", float(np.max(np.abs(zg - zo)) / np.max(np.abs(zo))))
    ctx.set_opts(pb.default_solver_opts())
    ctx.assemble()
    dphi, drho, ds, st = ctx.solve()
    S.inner_T_its = 0
    S.inner_A_its = []
    S.solve()
    print("solve gpu", {k: st[k] for k in ("outer_its", "inner_T_its", "inner_A_its_max", "inner_A_its_total")},
          "oracle", S.stats)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2")
