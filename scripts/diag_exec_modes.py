import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
torch.cuda.set_device(0)
import paper_2209_00315_b200 as pb
from synthetic import initial_state, make_problem
for name in sys.argv[1:]:
    p = make_problem(name)
    phi, rho, s = initial_state(p, 1.0)
    for mode in (True, False):
        ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
        ctx.set_exec_mode(mode)
        ctx.set_state(phi, rho, s, 1.0)
        ctx.assemble()
        dphi, drho, ds, st = ctx.solve()
        print(name, "graph" if mode else "eager", {k: st[k] for k in ("outer_its", "inner_T_its", "inner_A_its_max", "inner_A_its_total")}, flush=True)
