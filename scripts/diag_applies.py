#!/usr/bin/env python
"""Diagnostic: the BB applies of the oracle's own FGMRES solve (first Newton system of a
config, A19 point), re-applied on the GPU one by one: inner T / A counts per apply."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(name):
    import torch
    torch.cuda.set_device(0)
    import paper_2209_00315_b200 as pb
    from oracle.bb import BBSolver
    from oracle.ops import Discretisation
    from synthetic import initial_state, make_problem
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    S = BBSolver(d, phi, rho, s, 1.0)
    recs = []
    orig = S.apply

    def rec_apply(r):
        t0 = S.inner_T_its
        z = orig(r)
        recs.append((r.copy(), S.inner_T_its - t0, int(S.inner_A_its[-1].max())))
        return z
    S.apply = rec_apply
    S.solve()
    print("oracle", S.stats, flush=True)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(phi, rho, s, 1.0)
    ctx.assemble()
    tg = to = 0
    for i, (r, itT, itA) in enumerate(recs):
        zg, gT, gA = ctx.bb_apply(r)
        tg += gT
        to += itT
        print(f"apply {i:2d}: T gpu {gT:3d} oracle {itT:3d}   A max gpu {gA:3d} oracle {itA:3d}", flush=True)
    print("total T gpu", tg, "oracle", to)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2")
