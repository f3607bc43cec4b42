#!/usr/bin/env python
"""bench.py -- Newton-system solves/s of the BB-preconditioned IPM solver on B200.

One *step* = one pass of the whole hot path on one Newton
system: restore the state (device copy), assemble (residual/RHS, edge weights,
C, T, AMG(A), AMG(T) setup), FGMRES on (4.17) with the BB preconditioner,
recovery of (dphi, drho, ds), step length + update + renormalisation.

Workload (default): BASELINE.json configs[3] = C4, the largest configuration that
fits one GPU (BASELINE.json names no config for its metric; 256x256-grid-sized acute
mesh, 131 072 triangles, Nt = K = 128, 67.5 M unknowns, 45 GB resident), the first
Newton system of the IPM (A19 initial point, mu = 1), eps_out = 1e-10.  Inputs are
synthetic (synthetic/), fp64 throughout.  Side objects in the same line: the C2 system
(configs[1]), the SIMPLE preconditioner on it, and configs[0]'s own protocol (the full
C1 IPM, BB and BB -> SIMPLE hybrid).

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
import re
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
    ap.add_argument("--config", default="C4")
    ap.add_argument("--side-config", default="C2", help="smaller config reported beside the headline ('' = none)")
    ap.add_argument("--e2e-steps", type=int, default=5, help="timed steps of the end-to-end (host buffers) leg")
    ap.add_argument("--oracle-config", default="C2",
                    help="largest config whose oracle solve is bounded (C4's oracle: ~400 s setup, 27 GB)")
    ap.add_argument("--oracle-worker", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
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
                 "-lms", "500"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def _arnoldi_mean_j(its, restart):
    """mean Arnoldi index j over `its` iterations of GMRES(restart) cycles."""
    if its <= 0:
        return 0.0
    return sum(i % restart for i in range(its)) / its


class ByteModel:
    """Algorithmic (compulsory) HBM bytes per launch of every hot kernel.
    fp64 = 8 B, int32 = 4 B; geometry tables shared by all time slices count once.
    A_k is read in cell-ELL form (Aoff [K+1][4][N] = 32 B per row + the neighbour table
    [4][N] int32 once); T level 0 as slice-shared ELL (8 B per stored value + the column
    pattern [W][nbar] int32 once); coarse AMG levels as SELL-32 (12 B per stored entry).
    Multigrid kernels run on every level with a different grid: a launch is mapped to its
    level by its CTA count (nblocks(rows, 256)).  Krylov kernels: CGS2 over j+1 basis
    vectors, j = the mean Arnoldi index of this solve's own iteration counts.
    The per-slice PCG and every AMG(A) kernel skip the rows of converged time slices, so
    their bytes per launch are the full-launch bytes times the mean fraction of active
    slices, act = (slice-iterations of the solve) / (PCG launches x (K+1))."""

    def __init__(self, ctx, st, opts=None, pcg_launches=None):
        self.n, self.m, self.N, self.K, self.nbar = ctx.n, ctx.m, ctx.N, ctx.K, ctx.nbar
        self.NE = ctx.NE
        nnzT, W = ctx.T_nnz()
        self.tT = 8 * nnzT + 4 * W * self.nbar
        self.lapA = 32 * self.n + 16 * self.N
        self.levA, self.tailA = ctx.amg_levels(0)
        self.levT, self.tailT = ctx.amg_levels(1)
        r_out = opts.restart if opts is not None else 30
        r_T = opts.restart_T if opts is not None else 10
        self.its_O = max(1, st["outer_its"])
        self.its_T = st["inner_T_its"]
        self.jO = _arnoldi_mean_j(self.its_O, r_out)
        self.jT = _arnoldi_mean_j(max(1, round(self.its_T / self.its_O)), r_T)
        self.act = 1.0
        if pcg_launches:
            self.act = min(1.0, st["inner_A_its_total"] / (pcg_launches * (self.K + 1)))

    @staticmethod
    def _base(name):
        """Kernel name without arguments; the slice-batched level-0 kernels (k_*_sb / _sbx<NS, MINB>,
        NS slices per block) move the bytes of the kernel they batch."""
        base = name.split("(")[0].replace("void ", "").replace("bbot::", "")
        if base.startswith("k_down_sb<") and base.replace(" ", "").endswith((",false>", ",0>")):
            return "k_down_nx<LapView>"              # pre-sweep that does not write x (BBOT_LAP_RES)
        if base.startswith("k_up_dot_res"):           # <true>: 1/diag recomputed from the slots (no dinv read)
            return "k_up_dot_res<LapView,nodinv>" if base.replace(" ", "").endswith(("<true>", "<1>")) \
                else "k_up_dot_res<LapView>"
        m = re.match(r"(k_pcg_pq|k_down|k_up_dot)_sbx?<", base)
        return f"{m.group(1)}<LapView>" if m else base

    def bytes(self, name, grid):
        b = self._bytes(name, grid)
        if b is None:
            return None
        base = self._base(name)
        a_side = base.startswith(("k_pcg_", "k_tailA")) or "<LapView" in base
        if base in ("k_down<SellView>", "k_up<SellView>", "k_restrict", "k_resid_sk<SellView>", "k_jacobi_sk",
                    "k_down_nx<SellView>", "k_up_res<SellView>"):
            lv = self._level(grid, by="nc" if base == "k_restrict" else "n")
            a_side = lv is not None and lv[0] == "A"
        return b * self.act if a_side else b

    def _level(self, grid, by="n"):
        """(hierarchy, level, (n, nnz, nc)) whose row (or coarse-row) count gives `grid` CTAs."""
        for H, levels in (("A", self.levA), ("T", self.levT)):
            for l, (n, nnz, nc) in enumerate(levels):
                rows = n if by == "n" else nc
                if rows > 0 and (rows + 255) // 256 == grid:
                    return H, l, (n, nnz, nc)
        return None

    def _tail(self, levels, tail, nslices):
        if tail <= 0:
            return None
        b = 0
        for n, nnz, nc in levels[tail:]:
            b += 12 * max(nnz, 0) + 40 * n + 8 * nc
        return b

    def _bytes(self, name, grid):
        n, m, N, K, NE = self.n, self.m, self.N, self.K, self.NE
        nm = n + m
        base = self._base(name)
        if base == "k_pcg_pq<LapView>":
            return 40 * n + self.lapA                 # read z p q, write p q (+ A in cell-ELL)
        if base == "k_pcg_xr":
            return 48 * n                             # read x r p q, write x r
        if base == "k_pcg_rz":
            return 16 * n
        if base == "k_down<LapView>":
            return 32 * n + self.lapA                 # read b dinv, write x r
        if base == "k_down_nx<LapView>":
            return 24 * n + self.lapA                 # read b dinv, write r (x = om D^-1 b is recomputed)
        if base == "k_up_dot_res<LapView,nodinv>":
            return 28 * n + 8 * self.levA[0][2] + self.lapA      # read b r agg(4) xc, write z
        if base in ("k_up_dot<LapView>", "k_up<LapView>", "k_up_dot_res<LapView>"):   # _res: r instead of x
            nc1 = self.levA[0][2]
            return 36 * n + 8 * nc1 + self.lapA       # read b x dinv agg(4) xc, write z
        if base == "k_spmv<LapView>":
            return 16 * n + self.lapA
        if base == "k_spmv<SliceEllView>":
            return self.tT + 16 * m
        if base == "k_resid<SliceEllView>":
            return self.tT + 24 * m                   # read b x, write r
        if base == "k_post<SliceEllView>":
            return self.tT + 32 * m                   # read b xt dinv, write out
        if base in ("k_down<SellView>", "k_up<SellView>", "k_down_nx<SellView>", "k_up_res<SellView>"):
            lv = self._level(grid)
            if lv is None:
                return None
            _, _, (nl, nnz, nc) = lv
            if base.startswith("k_down"):
                return 12 * nnz + (24 if "_nx" in base else 32) * nl
            return 12 * nnz + 36 * nl + 8 * nc
        if base == "k_restrict":
            lv = self._level(grid, by="nc")
            if lv is None:
                return None
            _, _, (nl, nnz, nc) = lv
            return 12 * nl + 16 * nc                  # read r via midx(4), mptr; write b_c
        if base == "k_prolong":
            lv = self._level(grid)
            if lv is None:
                return None
            _, _, (nl, nnz, nc) = lv
            return 20 * nl + 8 * nc
        if base in ("k_post<SellView>", "k_resid_sk<SellView>"):
            lv = self._level(grid)
            if lv is None:
                return None
            _, _, (nl, nnz, nc) = lv
            return 12 * nnz + (32 * nl if base.startswith("k_post") else 24 * nl)
        if base == "k_jacobi_sk":
            lv = self._level(grid)
            return 24 * lv[2][0] if lv else None
        if base == "k_jacobi0":
            lv = self._level(grid)
            return 24 * lv[2][0] if lv else None
        if base == "k_tailA":
            return self._tail(self.levA, self.tailA, K + 1)     # one visit per level: a lower bound
        if base == "k_tailT":
            return self._tail(self.levT, self.tailT, K)
        if base.startswith("k_gm_dots<true, 12>") or base.startswith("k_gm_dots<1, 12>"):
            return 8 * m * (self.jT + 4)              # read V[0..j] w zout, write Z[j]
        if base.startswith("k_gm_dots"):
            return 8 * nm * (self.jO + 4)
        if base.startswith("k_gm_orth_dots<12>"):
            return 8 * m * (self.jT + 3)
        if base.startswith("k_gm_orth_dots"):
            return 8 * nm * (self.jO + 3)
        if base.startswith("k_gm_orth<12>"):         # T-GMRES: read V[0..j] w, write w
            return 8 * m * (self.jT + 3)
        if base.startswith("k_gm_orth<"):            # outer FGMRES
            return 8 * nm * (self.jO + 3)
        if base == "k_gm_scale":                     # both GMRES: read w, write V[j+1] vin (launch-weighted)
            wT, wO = self.its_T, self.its_O
            return (wT * 24 * m + wO * 24 * nm) / max(1, wT + wO)
        if base == "k_jp_y1":
            return 48 * n + 16 * N + 8 * (K + 1) * NE + 16 * m
        if base == "k_neg_norm":
            return 16 * m
        return None


def roofline_of(ctx, st, prof_grid, opts=None):
    """Roofline of the TOP kernel by device time, from one eagerly issued step's per-launch
    CUDA-event table (kernel, grid) -> (launches, ms): achieved = algorithmic bytes of its
    launches / their measured time."""
    pcg = sum(c for (nm, _g), (c, _ms) in prof_grid.items() if "k_pcg_pq" in nm)
    bm = ByteModel(ctx, st, opts, pcg_launches=pcg)
    per = {}
    for (name, grid), (cnt, ms) in prof_grid.items():
        e = per.setdefault(name, {"launches": 0, "ms": 0.0, "bytes": 0.0, "full": 0.0, "modeled": True})
        e["launches"] += cnt
        e["ms"] += ms
        b = bm.bytes(name, grid)
        if b is None:
            e["modeled"] = False
        else:
            e["bytes"] += b * cnt
            e["full"] += bm._bytes(name, grid) * cnt
    total_ms = sum(e["ms"] for e in per.values())
    ranked = sorted(per.items(), key=lambda kv: -kv[1]["ms"])
    peak, peak_kind = hbm_peak()
    rows = []
    for name, e in ranked[:25]:
        ach = e["bytes"] / (e["ms"] / 1e3) / 1e9 if e["modeled"] and e["ms"] > 0 else None
        rows.append({"kernel": name.split("(")[0], "launches": e["launches"], "ms": round(e["ms"], 3),
                     "share": round(e["ms"] / total_ms, 4),
                     "GBps": round(ach, 1) if ach is not None else None,
                     "frac": round(ach / peak, 4) if ach is not None else None,
                     "bytes_per_launch": (e["bytes"] / e["launches"]) if e["modeled"] else None,
                     "full_launch_bytes": (e["full"] / e["launches"]) if e["modeled"] else None})
    top = rows[0]
    roof = {"bound": "hbm", "kernel": top["kernel"], "achieved": top["GBps"], "peak": peak, "unit": "GB/s",
            "frac": top["frac"], "traffic": None, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst copy)",
            "algorithmic_bytes_per_launch": top["bytes_per_launch"],
            "algorithmic_bytes_full_launch": top["full_launch_bytes"],
            "active_slice_fraction": round(bm.act, 4),
            "avg_launch_us": round(1e3 * top["ms"] / top["launches"], 2), "launches_per_step": top["launches"],
            "share_of_step": top["share"]}
    # bytes-weighted achieved bandwidth of every modeled kernel (the step's HBM efficiency)
    mod = [e for e in per.values() if e["modeled"]]
    if mod:
        bsum, tsum = sum(e["bytes"] for e in mod), sum(e["ms"] for e in mod)
        roof["modeled_share_of_step"] = round(tsum / total_ms, 4)
        roof["modeled_kernels_GBps"] = round(bsum / (tsum / 1e3) / 1e9, 1)
        roof["modeled_kernels_frac"] = round(bsum / (tsum / 1e3) / 1e9 / peak, 4)
    return roof, rows, total_ms


def ncu_traffic(config, kernel):
    """DRAM bytes per launch (ncu --set full dram__bytes_read.sum + write.sum) of `kernel`
    on `config`, from profiles/ncu_summary.json (captured with the code of the round it
    names); None if that kernel was not captured."""
    try:
        summ = json.load(open(NCU_SUMMARY))
        per = summ["dram_bytes_per_launch"][config]
        norm = lambda t: (t.replace("void ", "").replace("bbot::", "").replace("true", "1")
                          .replace("false", "0").replace(" ", ""))      # ncu prints bool template args as 0/1
        short = norm(kernel)
        for k, v in per.items():
            if norm(k) == short:
                return v, summ.get("round", {}).get(f"{config}/{k}", "r1")
    except Exception:
        pass
    return None, None


def solve_point(pb, config, dev, stream, steps=3, warmup=1, precond=0, state=None):
    """One Newton system of `config` timed step by step (restore, assemble, solve, update)
    with its own per-kernel roofline -- side objects of the headline line."""
    import torch
    from synthetic import initial_state, make_problem
    p = make_problem(config)
    phi, rho, s = initial_state(p, 1.0) if state is None else state
    ctx = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, stream=stream.cuda_stream,
                     opts=pb.default_solver_opts(precond=precond))
    xs = [torch.tensor(x, device=dev) for x in (phi, rho, s)]
    last = {}

    def step():
        ctx.set_state(*xs, 1.0)
        ctx.assemble()
        last["st"] = ctx.solve_stats_only()
        ctx.newton_update(0.95)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = e0.elapsed_time(e1) / 1e3 / steps
    st = last["st"]
    ctx.prof_start()
    step()
    roof, rows, _ = roofline_of(ctx, st, ctx.prof_stop(by_grid=True), pb.default_solver_opts(precond=precond))
    pre = "SIMPLE" if precond == 1 else "BB"
    conv = bool(st["converged"])
    out = {"workload": f"{config}: first IPM Newton system (A19 point, mu=1), {pre}, eps_out=1e-10", "nbar": ctx.nbar,
           "K": ctx.K, "n_plus_m": ctx.n + ctx.m, "ms_per_step": 1e3 * t, "steps": steps, "warmup": warmup,
           "solve": {k: st[k] for k in ("outer_its", "inner_T_its", "inner_A_its_max", "inner_A_its_total",
                                        "converged", "rel_res")},
           "timing": {k: round(st[k], 3) for k in ("t_assemble_ms", "t_setup_ms", "t_krylov_ms")},
           "ms_per_outer": round(st["t_krylov_ms"] / max(1, st["outer_its"]), 4),
           "roofline": roof, "kernels": rows[:8]}
    if conv:
        out.update({"value": 1.0 / t, "unit": "solves/s", "unknowns_per_s": (ctx.n + ctx.m) / t})
    else:   # a capped solve is not a solve at fixed tolerance: no solves/s
        out.update({"value": None, "unit": "solves/s", "capped": True,
                    "note": f"ran to the FGMRES cap (rel. residual {st['rel_res']:.2e}); time per capped step only"})
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
    conv = [r for r in log if r["converged"]]
    return {"workload": f"{config}: full IPM, mu 1 -> 2^-26 (A17-A20){pre}, eps_out=1e-10", "n_systems": st["n_systems"],
            "n_converged": len(conv), "n_capped": st["n_unconverged"], "total_outer": st["total_outer"],
            "final_mu": st["final_mu"], "kinetic_energy": st["kinetic_energy"], "wall_s": round(wall, 3),
            "systems_per_s": st["n_systems"] / wall,
            "note": "host wall clock around bbot_ipm_run; capped systems (FGMRES 400-cap, the paper's dagger) "
                    "are counted as systems, not as solves at fixed tolerance"}


# ----------------------------------------------------------------------------- oracle (CPU baseline)
def oracle_worker(config):
    """Runs in a subprocess pinned to one thread: the oracle's FULL solve of the config's
    first Newton system (setup + BB-FGMRES to eps_out = 1e-10 + recovery), measured."""
    from threadpoolctl import threadpool_limits

    from oracle.bb import BBSolver, SolverOpts
    from oracle.ops import Discretisation
    from synthetic import initial_state, make_problem
    p = make_problem(config)
    phi, rho, s = initial_state(p, 1.0)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
        S = BBSolver(d, phi, rho, s, 1.0, SolverOpts())
        t1 = time.perf_counter()
        S.solve()
        t2 = time.perf_counter()
    print(json.dumps({"config": config, "n_plus_m": d.n + d.m, "setup_s": t1 - t0, "solve_s": t2 - t1,
                      "total_s": t2 - t0, "outer_its": S.stats["outer_its"], "converged": S.stats["converged"]}))


def start_oracle(config):
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               CUDA_VISIBLE_DEVICES="")
    return subprocess.Popen([sys.executable, os.path.abspath(__file__), "--oracle-worker", config],
                            stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, env=env)


def oracle_result(proc, timeout=900):
    try:
        out, _ = proc.communicate(timeout=timeout)
        return json.loads(out.strip().splitlines()[-1])
    except Exception:
        proc.kill()
        return None


def cpu_baseline_from(orc, head_unknowns):
    """The oracle's measured rate (full solve of a bounded config on one core) in the
    headline's unit: unknowns per second of Newton solve at fixed tolerance, divided by the
    headline's n+m.  The oracle's per-unknown cost GROWS with size (more outer iterations
    and AMG levels), so this overstates the oracle at C4 -- a conservative baseline."""
    if orc is None:
        return None
    ups = orc["n_plus_m"] / orc["total_s"]
    full = None
    try:      # the oracle's own full C4 solve (scripts/oracle_counts.py, offline, one core): context
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_counts.json"))).get("C4/init/mu=1")
        if g:
            full = {"seconds_1core": g["seconds_1core"], "solves_per_s": 1.0 / g["seconds_1core"],
                    "outer_its": g["outer_its"], "inner_T_its": g["inner_T_its"],
                    "source": "tests/golden/oracle_counts.json (the oracle's whole C4 step: setup + BB-FGMRES to 1e-10, run offline on one core)"}
    except Exception:
        pass
    return {"value": ups / head_unknowns, "unit": "solves/s", "cores": 1, "kind": "oracle",
            "oracle_full_C4_solve": full,
            "sample": (f"the oracle's full solve of the {orc['config']} mu=1 Newton system (setup {orc['setup_s']:.1f} s "
                       f"+ BB-FGMRES {orc['solve_s']:.1f} s, {orc['outer_its']} outer iterations, eps_out=1e-10) "
                       f"on 1 host core, run concurrently with the GPU legs = {ups:.0f} unknowns/s, divided by the "
                       f"headline's n+m (the oracle cannot set up C4 in a bounded sample: ~400 s and 27 GB)"),
            "measured": orc, "unknowns_per_s": ups}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the oracle (the paper ships no code: MATLAB + AGMG).  Each step is
    the oracle's FULL solve of the C1 mu=1 Newton system on one core (~1 s, measured), its
    unknowns/s then divided by the headline config's n+m (the oracle cannot run C4 in a
    bounded step)."""
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits

    from oracle.bb import BBSolver, SolverOpts
    from oracle.ops import Discretisation
    from synthetic import initial_state, make_problem
    sample_cfg = "C1"
    p = make_problem(sample_cfg)
    phi, rho, s = initial_state(p, 1.0)
    head = make_problem(args.config)
    head_unk = head.n + head.m

    def one():
        with threadpool_limits(1):
            t0 = time.perf_counter()
            d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
            S = BBSolver(d, phi, rho, s, 1.0, SolverOpts())
            S.solve()
            return time.perf_counter() - t0, d.n + d.m, S.stats["outer_its"]

    for _ in range(args.warmup):
        one()
    ts = []
    for _ in range(args.steps):
        t, unk, its = one()
        ts.append(t)
    tot = sum(ts)
    ups = unk * args.steps / tot
    value = ups / head_unk
    sample = (f"per step: the oracle's full solve (setup + BB-FGMRES to 1e-10 + recovery, {its} outer iterations) of the "
              f"{sample_cfg} mu=1 Newton system ({unk} unknowns) on 1 core = {ups:.0f} unknowns/s; value = that / "
              f"{args.config}'s n+m ({head_unk})")
    line = {"impl": "reference", "metric": "newton_solves_per_s", "value": value, "unit": "solves/s",
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} first IPM Newton system (mu=1), eps_out=1e-10 (oracle sampled on "
                                   f"{sample_cfg})"},
            "unknowns_per_s": ups,
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.oracle_worker:
        oracle_worker(args.oracle_worker)
        return
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

    # the CPU baseline (the oracle's full solve of a bounded config on one host core) runs
    # in a subprocess concurrently with the GPU legs
    orc_proc = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        orc_proc = start_oracle(args.oracle_config)

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

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        step_e2e()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    te = max_over_ranks(e0.elapsed_time(e1) / 1e3, dist, dev)
    io_bytes = 8 * (ctx.n + 2 * ctx.m)

    # ---- per-kernel shares: one extra step of the same system issued eagerly (the
    # per-launch profiler brackets every kernel with CUDA events on the launching
    # stream).  The eager issue runs exactly the kernels the graph replays
    # (bitwise-identical results), so its launch count is the step's launch count.
    # ---- device memory of this context (the library's private pool; nothing else allocated from
    # it yet): the FGMRES basis, divided by P under time slabs, and the rest (replicated)
    mem = None
    try:
        used, peak = ctx.mem_usage()
        r_out = 30
        basis = (2 * r_out + 1) * (ctx.n + ctx.m) * 8 / world
        mem = {"used_gb": round(used / 1e9, 3), "peak_gb": round(peak / 1e9, 3),
               "fgmres_basis_gb": round(basis / 1e9, 3),
               "other_gb": round((peak - basis) / 1e9, 3),
               "note": "pool high-water mark after assemble + solve; the FGMRES(30) basis (61 vectors of "
                       "n+m doubles) is slab-local (divided by P), the rest is replicated on every rank"}
    except Exception as ex:
        mem = {"error": str(ex)[:120]}
    roof = None
    kernels = None
    launches = None
    if not args.no_profile:
        l0 = ctx.launch_count()
        ctx.prof_start()
        step()
        prof = ctx.prof_stop(by_grid=True)
        launches = ctx.launch_count() - l0
        roof, kernels, total_ms = roofline_of(ctx, last["st"], prof)
        traffic, rnd = ncu_traffic(args.config, roof["kernel"])
        if traffic is not None and roof["algorithmic_bytes_full_launch"]:
            # ncu captures a launch with every time slice active: compare with the full-launch model
            roof["traffic"] = traffic
            roof["traffic_source"] = (f"profiles/ncu_summary.json ({args.config}, ncu --set full, {rnd} code, "
                                      f"a launch with every slice active)")
            roof["traffic_over_algorithmic"] = round(traffic / roof["algorithmic_bytes_full_launch"], 3)
        if args.profile_out and rank == 0:
            json.dump({"config": args.config, "kernels": kernels, "total_ms": total_ms},
                      open(args.profile_out, "w"), indent=1)

    side = simple = None
    if rank == 0 and world == 1 and args.side_config and not args.no_profile:
        try:
            side = solve_point(pb, args.side_config, dev, stream, steps=5, warmup=2)
        except Exception as ex:                          # the headline line must still print
            side = {"error": str(ex)[:200]}
        try:
            simple = solve_point(pb, args.side_config, dev, stream, steps=3, warmup=1, precond=1)
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

    cpu = cpu_baseline_from(oracle_result(orc_proc), ctx.n + ctx.m) if orc_proc is not None else None

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
                       "l2": "no flush; inputs larger than L2 (per-step working set: FGMRES basis 61 x (n+m) x 8 B)"},
            "unknowns_per_s": value * (ctx.n + ctx.m),
            "solve": {k: st[k] for k in ("outer_its", "inner_T_its", "inner_A_its_max", "inner_A_its_total", "converged",
                                         "rel_res", "amg_levels_A", "amg_levels_T")},
            "e2e": {"value": e2e_steps / te, "unit": "solves/s", "h2d_bytes_per_step": io_bytes,
                    "d2h_bytes_per_step": io_bytes, "steps": e2e_steps},
            "gpu_launches": int(launches) if launches is not None else None,
            "memory": mem,
            "timing": {k: round(st[k], 3) for k in ("t_assemble_ms", "t_setup_ms", "t_krylov_ms", "t_graph_ms")},
            "ms_per_outer": round(st["t_krylov_ms"] / max(1, st["outer_its"]), 3),
            "roofline": roof,
            "kernels": kernels[:12] if kernels else None,
            "side_point": side,
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
