"""Exploratory timing of one Newton system on a config (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00315_b200 as pb
from synthetic import make_problem, initial_state, random_state

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
state = sys.argv[2] if len(sys.argv) > 2 else "init"
p = make_problem(name)
if state == "init":
    phi, rho, s = initial_state(p, 1.0); mu = 1.0
else:
    phi, rho, s = random_state(p, seed=3, mu=1e-2); mu = 1e-2
t = time.time()
ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
ctx.set_state(phi, rho, s, mu)
print(f"{name}: nbar={p.nbar} K={p.K} n+m={ctx.n + ctx.m} create {time.time()-t:.2f}s", flush=True)
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    ctx.assemble()
    torch.cuda.synchronize(); ta = time.time() - t
    t = time.time()
    dphi, drho, ds, st = ctx.solve()
    torch.cuda.synchronize(); tsol = time.time() - t
    print(f"rep{rep}: assemble+setup {ta*1e3:.1f} ms, solve {tsol*1e3:.1f} ms, stats {st}", flush=True)
    print("  AMG A levels", ctx.amg_info(0), " T levels", ctx.amg_info(1), flush=True)
    print("  launches", ctx.launch_count(), flush=True)
