#!/usr/bin/env python
"""Full interior-point run of a config on the GPU (A17-A20: mu 1 -> 2^-26), printing
one line per Newton system and a JSON summary -- the configs' own protocol.

    python scripts/ipm_run.py --config C2
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--mu-min", type=float, default=1e-8)
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--simple-below", type=float, default=0.0,
                    help="A34 hybrid: SIMPLE preconditioner for mu below this (0 = BB throughout)")
    a = ap.parse_args()
    import torch
    import paper_2209_00315_b200 as pb
    from synthetic import initial_state, make_problem
    torch.cuda.set_device(0)
    p = make_problem(a.config)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(*initial_state(p, 1.0), 1.0)

    def cb(r):
        if not a.quiet:
            print(f"{'S' if r['mu'] < a.simple_below else 'B'} mu={r['mu']:.3e} newton={r['newton']} outer={r['outer_its']} conv={r['converged']} "
                  f"T={r['inner_T_its']} Amax={r['inner_A_its_max']} res={r['res']:.3e} alpha={r['alpha']:.3f} "
                  f"setup={r['t_setup_ms']:.0f}ms krylov={r['t_krylov_ms']:.0f}ms", flush=True)
    t = time.time()
    st, log = ctx.ipm_run(pb.default_ipm_opts(mu_min=a.mu_min, simple_below_mu=a.simple_below),
                            callback=cb)
    wall = time.time() - t
    print(json.dumps({"config": a.config, "mu_min": a.mu_min, "n_systems": st["n_systems"],
                      "n_converged": st["n_systems"] - st["n_unconverged"], "total_outer": st["total_outer"],
                      "n_unconverged": st["n_unconverged"],
                      "final_mu": st["final_mu"],
                      "kinetic_energy": st["kinetic_energy"], "wall_s": round(wall, 2),
                      "solves_per_s": st["n_systems"] / wall}))


if __name__ == "__main__":
    main()
