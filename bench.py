#!/usr/bin/env python
"""bench.py -- Newton-system solves/s of the BB-preconditioned IPM solver on B200.

One *step* = one pass of the whole hot path on one Newton
system: restore the state (device copy), assemble (residual/RHS, edge weights,
C, T, AMG(A), AMG(T) setup), FGMRES on (4.17) with the BB preconditioner,
recovery of (dphi, drho, ds), step length + update + renormalisation.

Workload (default): BASELINE.json configs[1] = C2 (64x64-grid-sized acute mesh,
8192 triangles, Nt = K = 32, seeded jitter), the first Newton system of the IPM
(A19 initial point, mu = 1), eps_out = 1e-10.  Inputs are synthetic
(synthetic/), fp64 throughout.

    python bench.py [--gpus N --steps K --warmup W --config C2 --impl bbot|reference]

N > 1 (torchrun): the ranks solve the SAME Newton system together (strong
scaling): each rank owns a time slab of the K+1 potential slices, runs the per-
slice A_k solves of every BB apply on its slab only and exchanges the results
with NCCL inside the apply; the rest is redundant per rank.  The
max-over-ranks device time is the job's time.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
COUNTS_FILE = os.path.join(ROOT, "tests", "golden", "oracle_counts.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bbot", choices=["bbot", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--scale-config", default="C4", help="HBM-bound size reported beside the headline ('' = none)")
    ap.add_argument("--ipm-config", default="C1", help="config whose full IPM run is reported ('' = none)")
    ap.add_argument("--profile-out", default=None, help="write the per-kernel table (json) here")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def max_over_ranks(t, dist=None, device=None):
    """The job's time = the slowest rank's device time (contract: max over ranks)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(t)
    import torch
    tt = torch.tensor([float(t)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def hbm_peak():
    try:
        return float(json.load(open(PEAKS_FILE))["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


def byte_models(ctx, nnzT):
    """Algorithmic (compulsory) bytes per launch of the main kernels.
    fp64 = 8 B, int32 = 4 B; geometry tables shared by all time slices count once.
    A_k is read in cell-ELL form (Aoff [K+1][4][N] = 32 B per row, neighbour table
    [4][N] int32 once); T level 0 as slice-shared ELL (values 8 B per stored entry,
    column pattern [W][nbar] int32 once)."""
    n, m, N, K, nbar = ctx.n, ctx.m, ctx.N, ctx.K, ctx.nbar
    W = ctx.T_width
    A_sizes, T_sizes = ctx.amg_info(0), ctx.amg_info(1)
    nc1A = A_sizes[1] if len(A_sizes) > 1 else 0
    nc1T = T_sizes[1] if len(T_sizes) > 1 else 0
    lapA = 32 * n + 16 * N                  # Aoff + neighbour table
    tT = 8 * nnzT + 4 * W * nbar            # T values + shared column pattern
    return {
        # per-slice PCG (I4): p = z + beta p, q = A z + beta q, p.q  (read z p q, write p q)
        "void bbot::k_pcg_pq<bbot::LapView>": 40 * n + lapA,
        "bbot::k_pcg_xr": 48 * n,                      # x += a p, r -= a q, r.r  (read x r p q, write x r)
        "bbot::k_pcg_rz": 16 * n,
        # level-0 V-cycle sweeps of AMG(A): k_down reads b dinv, writes x r; k_up_dot reads b x
        # dinv agg(4 B) and the level-1 correction, writes z (r.z fused)
        "void bbot::k_down<bbot::LapView>": 32 * n + lapA,
        "void bbot::k_up_dot<bbot::LapView>": 36 * n + 8 * nc1A + lapA,
        "void bbot::k_up<bbot::LapView>": 36 * n + 8 * nc1A + lapA,
        "void bbot::k_spmv<bbot::LapView>": 16 * n + lapA,
        "void bbot::k_spmv<bbot::SliceEllView>": tT + 16 * m,
        "void bbot::k_down<bbot::SliceEllView>": tT + 32 * m,
        "void bbot::k_up<bbot::SliceEllView>": tT + 36 * m + 8 * nc1T,
    }


def _match_model(name, models):
    for k in models:
        if name == k or name.startswith(k + "("):
            return k
    return None


def oracle_sample(config, n_outer_sample=3):
    """Bounded oracle sample on this host: assembly + AMG setups + n_outer_sample
    FGMRES iterations of the same Newton system, single core.  Returns
    (seconds_setup, seconds_per_outer)."""
    from threadpoolctl import threadpool_limits

    from oracle.bb import BBSolver, SolverOpts
    from oracle.ops import Discretisation
    from synthetic import initial_state, make_problem
    p = make_problem(config)
    phi, rho, s = initial_state(p, 1.0)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
        S = BBSolver(d, phi, rho, s, 1.0, SolverOpts(maxit=n_outer_sample))
        t1 = time.perf_counter()
        S.solve()
        t2 = time.perf_counter()
    return t1 - t0, (t2 - t1) / max(1, S.stats["outer_its"])


def oracle_outer_count(config):
    try:
        return int(json.load(open(COUNTS_FILE))[f"{config}/init/mu=1"]["outer_its"])
    except Exception:
        return None


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    n_outer = oracle_outer_count(args.config)
    if n_outer is None:
        print(json.dumps({"impl": "reference", "unavailable": f"no oracle outer count for {args.config}"}))
        return
    for _ in range(args.warmup):
        oracle_sample(args.config)
    vals = []
    t_all = 0.0
    for _ in range(args.steps):
        ts, to = oracle_sample(args.config)
        t_solve = ts + n_outer * to
        vals.append(1.0 / t_solve)
        t_all += t_solve
    value = args.steps / t_all
    sample = (f"per step: oracle assembly + AMG setups + 3 FGMRES iterations of the {args.config} mu=1 system, "
              f"1 core, extrapolated to the oracle's own {n_outer} outer iterations")
    line = {"impl": "reference", "metric": "newton_solves_per_s", "value": value, "unit": "solves/s",
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} first IPM Newton system (mu=1), eps_out=1e-10"},
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def roofline_of(ctx, prof_table, config):
    """Roofline object for the dominant kernel with a byte model, from one eagerly
    issued step's per-launch CUDA-event table."""
    nnzT, _ = ctx.T_nnz()
    models = byte_models(ctx, nnzT)
    total_ms = sum(v[1] for v in prof_table.values())
    ranked = sorted(prof_table.items(), key=lambda kv: -kv[1][1])
    dom = next(((k, v) for k, v in ranked if _match_model(k, models)), None)
    peak, peak_kind = hbm_peak()
    roof = None
    if dom is not None:
        name, (cnt, ms) = dom
        avg_s = ms / cnt / 1e3
        model = models[_match_model(name, models)]
        ach = model / avg_s / 1e9
        traffic = None       # DRAM bytes per launch from the committed ncu --set full capture
        try:
            summ = json.load(open(NCU_SUMMARY))["dram_bytes_per_launch"][config]
            short = _match_model(name, models).replace("bbot::", "").replace("void ", "")
            traffic = next((v for k, v in summ.items() if k.replace("void ", "") == short), None)
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": name, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "peak_source": peak_kind,
                "algorithmic_bytes_per_launch": model, "avg_launch_us": round(avg_s * 1e6, 2),
                "launches_per_step": cnt, "share_of_step": round(ms / total_ms, 4),
                "top_kernel": ranked[0][0], "top_kernel_share": round(ranked[0][1][1] / total_ms, 4)}
    return roof, ranked, total_ms, models


def scale_point(pb, config, dev, stream, steps=2, precond=0):
    """The same step on the largest single-GPU config (C4: 67.5 M unknowns, vectors of
    0.4-0.5 GB, HBM-bound) -- reported beside the headline line, not instead of it.
    precond=1: the same measurement for the SIMPLE preconditioner (NEXT f1)."""
    import torch
    from synthetic import initial_state, make_problem
    p = make_problem(config)
    phi, rho, s = initial_state(p, 1.0)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, stream=stream.cuda_stream,
                     opts=pb.default_solver_opts(precond=precond))
    xs = [torch.tensor(x, device=dev) for x in (phi, rho, s)]
    last = {}

    def step():
        ctx.set_state(*xs, 1.0)
        ctx.assemble()
        last["st"] = ctx.solve_stats_only()
        ctx.newton_update(0.95)

    step()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = e0.elapsed_time(e1) / 1e3 / steps
    ctx.prof_start()
    step()
    roof, _, _, _ = roofline_of(ctx, ctx.prof_stop(), config + ("-SIMPLE" if precond == 1 else ""))
    st = last["st"]
    pre = "SIMPLE" if precond == 1 else "BB"
    out = {"workload": f"{config}: first IPM Newton system (A19 point, mu=1), {pre}, eps_out=1e-10", "nbar": ctx.nbar,
           "K": ctx.K, "n_plus_m": ctx.n + ctx.m, "value": 1.0 / t, "unit": "solves/s", "ms_per_step": 1e3 * t,
           "unknowns_per_s": (ctx.n + ctx.m) / t, "steps": steps, "warmup": 1,
           "solve": {k: st[k] for k in ("outer_its", "inner_T_its", "inner_A_its_max", "inner_A_its_total",
                                        "converged", "rel_res")},
           "timing": {k: round(st[k], 3) for k in ("t_assemble_ms", "t_setup_ms", "t_krylov_ms")},
           "ms_per_outer": round(st["t_krylov_ms"] / max(1, st["outer_its"]), 4),
           "roofline": roof}
    ctx.close()
    return out


def ipm_protocol(pb, config, dev, simple_below_mu=0.0):
    """BASELINE configs[0]'s own protocol on the GPU: the full interior-point run (A17-A20,
    mu 1 -> 2^-26) -- every Newton system of the trajectory, not just the first.
    simple_below_mu > 0: the BB -> SIMPLE hybrid (A34, NEXT f1)."""
    import torch
    from synthetic import initial_state, make_problem
    p = make_problem(config)
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ctx.set_state(*initial_state(p, 1.0), 1.0)
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    st, log = ctx.ipm_run(pb.default_ipm_opts(simple_below_mu=simple_below_mu))
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t
    ctx.close()
    pre = f", SIMPLE below mu={simple_below_mu:g}" if simple_below_mu > 0 else ", BB"
    return {"workload": f"{config}: full IPM, mu 1 -> 2^-26 (A17-A20){pre}, eps_out=1e-10", "n_systems": st["n_systems"],
            "total_outer": st["total_outer"], "n_capped": st["n_unconverged"], "final_mu": st["final_mu"],
            "kinetic_energy": st["kinetic_energy"], "wall_s": round(wall, 3),
            "solves_per_s": st["n_systems"] / wall, "timing": "host wall clock around bbot_ipm_run"}


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if (args.impl == "bbot" and torch.cuda.is_available()) else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend)
    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    import numpy as np

    import paper_2209_00315_b200 as pb
    from synthetic import initial_state, make_problem

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    p = make_problem(args.config)
    phi_h, rho_h, s_h = initial_state(p, 1.0)
    mu = 1.0
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, stream=stream.cuda_stream)
    if world > 1:                                        # time slabs over NCCL (the uid travels via torch.distributed)
        obj = [pb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.set_dist(rank, world, obj[0])
    phi_d = torch.tensor(phi_h, device=dev)
    rho_d = torch.tensor(rho_h, device=dev)
    s_d = torch.tensor(s_h, device=dev)
    last = {}

    def step():
        ctx.set_state(phi_d, rho_d, s_d, mu)            # device -> device restore of the input state
        ctx.assemble()                                   # a1 + a3
        last["st"] = ctx.solve_stats_only()              # a2 + a4 + a5 + a6 (direction stays in HBM)
        last["alpha"] = ctx.newton_update(0.95)          # a7

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    clk = ClockSampler(local_rank)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    clocks = clk.stop()
    t = max_over_ranks(e0.elapsed_time(e1) / 1e3, dist, dev)
    value = args.steps / t                               # one system per step for the whole job
    st = last["st"]

    # ---- end to end through the C-ABI with host buffers (H2D of the state, D2H of the new state)
    phi_o, rho_o, s_o = np.empty_like(phi_h), np.empty_like(rho_h), np.empty_like(s_h)

    def step_e2e():
        ctx.set_state(phi_h, rho_h, s_h, mu)
        ctx.assemble()
        ctx.solve_stats_only()
        ctx.newton_update(0.95)
        ctx.get_state(phi_o, rho_o, s_o)

    step_e2e()
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step_e2e()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    te = max_over_ranks(e0.elapsed_time(e1) / 1e3, dist, dev)
    io_bytes = 8 * (ctx.n + 2 * ctx.m)

    # ---- per-kernel shares: one extra step of the same system issued eagerly (the
    # per-launch profiler brackets every kernel with CUDA events on the launching
    # stream).  The eager issue runs exactly the kernels the graph replays
    # (bitwise-identical results), so its launch count is the step's launch count.
    roof = None
    prof_table = None
    launches = None
    if not args.no_profile:
        l0 = ctx.launch_count()
        ctx.prof_start()
        step()
        prof_table = ctx.prof_stop()
        launches = ctx.launch_count() - l0
        roof, ranked, total_ms, models = roofline_of(ctx, prof_table, args.config)
        if args.profile_out and rank == 0:
            json.dump({"config": args.config, "kernels": {k: {"launches": v[0], "ms": v[1]} for k, v in ranked},
                       "total_ms": total_ms, "models": models}, open(args.profile_out, "w"), indent=1)

    scale = None
    if rank == 0 and world == 1 and args.scale_config and args.scale_config != args.config and not args.no_profile:
        try:
            scale = scale_point(pb, args.scale_config, dev, stream)
        except Exception as ex:                          # the headline line must still print
            scale = {"error": str(ex)[:200]}

    simple = None      # NEXT f1: the SIMPLE preconditioner on the headline config
    if rank == 0 and world == 1 and not args.no_profile:
        try:
            simple = scale_point(pb, args.config, dev, stream, precond=1)
        except Exception as ex:
            simple = {"error": str(ex)[:200]}

    protocol = hybrid = None
    if rank == 0 and world == 1 and args.ipm_config and not args.no_profile:
        try:
            protocol = ipm_protocol(pb, args.ipm_config, dev)
        except Exception as ex:
            protocol = {"error": str(ex)[:200]}
        try:
            hybrid = ipm_protocol(pb, args.ipm_config, dev, simple_below_mu=0.1)
        except Exception as ex:
            hybrid = {"error": str(ex)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_outer = oracle_outer_count(args.config)
        if n_outer is not None:
            ts, to = oracle_sample(args.config)
            cpu = {"value": 1.0 / (ts + n_outer * to), "unit": "solves/s", "cores": 1, "kind": "oracle",
                   "sample": (f"oracle assembly + AMG setups + 3 FGMRES iterations of the same {args.config} mu=1 "
                              f"system on 1 host core ({ts:.1f} s setup, {to:.2f} s/outer), extrapolated to the "
                              f"oracle's own {n_outer} outer iterations (tests/golden/oracle_counts.json)")}

    if rank == 0:
        line = {
            "metric": "newton_solves_per_s", "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: first IPM Newton system (A19 point, mu=1), eps_out=1e-10",
                       "nbar": ctx.nbar, "K": ctx.K, "n_plus_m": ctx.n + ctx.m, "T_width": ctx.T_width,
                       "parallelism": (f"time slabs x{world} (A_k solves partitioned, NCCL exchange)"
                                       if world > 1 else "1 GPU"),
                       "l2": "no flush; per-step working set (FGMRES basis 61 x (n+m) x 8 B) exceeds the 126 MB L2"},
            "unknowns_per_s": value * (ctx.n + ctx.m),
            "solve": {k: st[k] for k in ("outer_its", "inner_T_its", "inner_A_its_max", "inner_A_its_total", "converged", "rel_res",
                                         "amg_levels_A", "amg_levels_T")},
            "e2e": {"value": args.steps / te, "unit": "solves/s", "h2d_bytes_per_step": io_bytes,
                    "d2h_bytes_per_step": io_bytes},
            "gpu_launches": int(launches) if launches is not None else None,
            "timing": {k: round(st[k], 3) for k in ("t_assemble_ms", "t_setup_ms", "t_krylov_ms", "t_graph_ms")},
            "roofline": roof,
            "hbm_scale_point": scale,
            "simple_point": simple,
            "ipm_protocol": protocol,
            "ipm_protocol_hybrid": hybrid,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
