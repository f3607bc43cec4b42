#!/usr/bin/env python
"""A/B of the slice-batched level-0 AMG(A) pre-smoothing (BBOT_LAP_SB = 1 | 2) on one
context: every variant solves the same Newton system eagerly (the env is read at every
launch); directions must be bitwise equal to the unbatched run; per-kernel device time from
the library's per-launch CUDA events.

    python scripts/ab_lap_sb.py --config C4
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (BBOT_LAP_SB, _MINB, _EXPL): the round-2 sweep (profiles/r2z_ab_lap_sb_*.log) also batched
# k_up_dot / k_pcg_pq and tried 4-8 CTAs per SM and all-loads-first kernels; only k_down_sb
# <2 slices, 6 CTAs/SM> was kept, so only BBOT_LAP_SB is read now
VARIANTS = [("1", "8", "0"), ("2", "6", "0"), ("1", "8", "0")]


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
    for sb, mb, ex in VARIANTS:
        os.environ.update(BBOT_LAP_SB=sb, BBOT_LAP_SB_MINB=mb, BBOT_LAP_SB_EXPL=ex)
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
               and "Sell" not in k}
        tot = sum(v[1] for v in prof.values())
        print(f"SB={sb} MINB={mb} EXPL={ex}: solve {dt * 1e3:.0f} ms (kernels {tot:.0f} ms) outer {st['outer_its']} "
              f"bitwise={same}", flush=True)
        for k, (n, ms) in sorted(top.items(), key=lambda kv: -kv[1][1]):
            print(f"    {k[:60]:60s} {n:6d} {ms:9.1f} ms", flush=True)


if __name__ == "__main__":
    main()
