#!/usr/bin/env python
"""One BB apply (a4) on a config's first Newton system with a seeded random right-hand side
(every time slice active in the per-slice PCG: full launches), bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off` (after a warm-up apply):

    BBOT_EAGER=1 ncu --profile-from-start off --kernel-name-base demangled -k regex:LapView \\
        --launch-count 6 --set full -o out python scripts/profile_apply.py --config C4
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    a = ap.parse_args()
    import torch
    import paper_2209_00315_b200 as pb
    from synthetic import initial_state, make_problem
    torch.cuda.set_device(0)
    p = make_problem(a.config)
    phi, rho, s = initial_state(p, 1.0)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(phi, rho, s, 1.0)
    ctx.assemble()
    r = np.random.default_rng(0).standard_normal(ctx.n + ctx.m)
    ctx.bb_apply(r)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    z, itT, itA = ctx.bb_apply(r)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("T its", itT, "A max", itA)


if __name__ == "__main__":
    main()
