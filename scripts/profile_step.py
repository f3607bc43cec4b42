#!/usr/bin/env python
"""One bench step (assemble + BB-FGMRES solve + update) bracketed by
cudaProfilerStart/Stop, for `ncu --profile-from-start off`:

    python scripts/profile_step.py --config C2            # plain run (must exit 0 first)
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python scripts/profile_step.py --config C2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--warm", type=int, default=1)
    ap.add_argument("--precond", type=int, default=0, help="0 = BB, 1 = SIMPLE (NEXT f1)")
    a = ap.parse_args()
    import torch
    import paper_2209_00315_b200 as pb
    from synthetic import initial_state, make_problem
    torch.cuda.set_device(0)
    p = make_problem(a.config)
    phi, rho, s = initial_state(p, 1.0)
    stream = torch.cuda.current_stream()
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, stream=stream.cuda_stream,
                     opts=pb.default_solver_opts(precond=a.precond))
    dev = [torch.tensor(x, device="cuda") for x in (phi, rho, s)]

    def step():
        ctx.set_state(*dev, 1.0)
        ctx.assemble()
        st = ctx.solve_stats_only()
        ctx.newton_update(0.95)
        return st

    for _ in range(a.warm):
        step()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    torch.cuda.profiler.start()
    st = step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print({k: st[k] for k in ("outer_its", "inner_T_its", "inner_A_its_max", "converged", "t_assemble_ms",
                              "t_setup_ms", "t_krylov_ms")}, "launches:", ctx.launch_count() - l0)


if __name__ == "__main__":
    main()
