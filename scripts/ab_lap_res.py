#!/usr/bin/env python
"""A/B of the residual-based AMG(A) post sweeps (BBOT_LAP_RES, BBOT_SELL_RES; csrc/amg.cu
k_up_dot_res / k_up_res) on one context: every variant
solves the same Newton system eagerly (the env is read at every launch); directions must be
compared bitwise with the first run (the residual-based sweeps differ at rounding level); per-kernel device time from the library's
per-launch CUDA events.

    python scripts/ab_lap_res.py --config C4
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (BBOT_LAP_RES, BBOT_SELL_RES, BBOT_LAP_RDINV)
VARIANTS = [("1", "1", "0"), ("1", "1", "1"), ("1", "1", "0"), ("1", "1", "1")]


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
    ctx.set_exec_mode(False)
    ref = None
    for sb, mb, rd in VARIANTS:
        os.environ.update(BBOT_LAP_RES=sb, BBOT_SELL_RES=mb, BBOT_LAP_RDINV=rd)
        ctx.set_state(phi, rho, s, 1.0)
        ctx.assemble()
        torch.cuda.synchronize()
        ctx.prof_start()
        t = time.perf_counter()
        dphi, drho, ds, st = ctx.solve()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        prof = ctx.prof_stop()
        if ref is None:
            ref = (dphi, drho, ds)
        same = all(np.array_equal(u, v) for u, v in zip(ref, (dphi, drho, ds)))
        top = {k: v for k, v in prof.items() if any(x in k for x in ("k_up_dot", "k_pcg_pq", "k_down", "k_pcg_xr"))
               or "Sell" in k or "k_restrict" in k or "k_tailA" in k}
        tot = sum(v[1] for v in prof.values())
        print(f"LAP_RES={sb} SELL_RES={mb} RDINV={rd}: solve {dt * 1e3:.0f} ms (kernels {tot:.0f} ms) outer {st['outer_its']} "
              f"bitwise={same}", flush=True)
        for k, (n, ms) in sorted(top.items(), key=lambda kv: -kv[1][1]):
            print(f"    {k[:60]:60s} {n:6d} {ms:9.1f} ms", flush=True)


if __name__ == "__main__":
    main()
