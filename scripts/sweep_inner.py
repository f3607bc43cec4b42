#!/usr/bin/env python
"""GPU-only exploration (not a parity or bench artefact): how the inner A_k tolerance eps_A
and the AMG(A) Jacobi weight move the cost of one Newton solve on a config's first system
(A19 point) -- outer / T / PCG counts and device time per solve.

    python scripts/sweep_inner.py --config C4 --eps 1e-3,3e-3,1e-2 --omega 0.6667
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--eps", default="1e-3,3e-3,1e-2,5e-2")
    ap.add_argument("--omega", default="0.6666666666666666")
    ap.add_argument("--newton", type=int, default=0, help="GPU Newton steps at mu=1 before the measured system")
    a = ap.parse_args()
    import torch
    import paper_2209_00315_b200 as pb
    from synthetic import initial_state, make_problem
    torch.cuda.set_device(0)
    p = make_problem(a.config)
    phi, rho, s = initial_state(p, 1.0)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(phi, rho, s, 1.0)
    for _ in range(a.newton):
        ctx.assemble()
        ctx.solve()
        ctx.newton_update(0.95)
    st0 = ctx.get_state()
    for om in [float(x) for x in a.omega.split(",")]:
        for eps in [float(x) for x in a.eps.split(",")]:
            ctx.set_opts(pb.default_solver_opts(eps_A=eps, omega_A=om))
            ctx.set_state(*st0[:3], 1.0)
            ctx.assemble()
            torch.cuda.synchronize()
            t = time.perf_counter()
            _, _, _, st = ctx.solve()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            print(f"{a.config} newton={a.newton} omega_A={om:.4f} eps_A={eps:.0e}: outer {st['outer_its']} "
                  f"T {st['inner_T_its']} A_total {st['inner_A_its_total']} A_max {st['inner_A_its_max']} "
                  f"conv {st['converged']} rel {st['rel_res']:.2e}  {dt * 1e3:.0f} ms", flush=True)


if __name__ == "__main__":
    main()
