"""Write tests/golden/ipm_<CFG>.json: the ORACLE's full IPM run (A17-A20, mu 1 ->
2^-26 ~ 1.49e-8) on a config -- per-system outer counts / convergence flags /
residuals after each update and the final kinetic energy (D12).  Calls only oracle/
and synthetic/, single BLAS thread (fixed summation order).  The GPU test
tests/test_gpu_parity.py::test_ipm_parity_C1_full compares the CUDA path to it (the
oracle needs ~10 min on one core for C1, too long to re-run inside the GPU suite).

    python scripts/oracle_ipm_golden.py C1
    python scripts/oracle_ipm_golden.py C2 0.0078125     # mu 1 -> 2^-7 only (-> ipm_C2_mu7.json)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from threadpoolctl import threadpool_limits  # noqa: E402

from oracle.bb import SolverOpts  # noqa: E402
from oracle.ipm import IpmOpts, ipm_run  # noqa: E402
from oracle.ops import Discretisation  # noqa: E402
from synthetic import initial_state, make_problem  # noqa: E402


def main(name, mu_min=None):
    p = make_problem(name)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = initial_state(p, 1.0)
    t0 = time.time()
    log = []

    def cb(r):
        log.append({k: (float(v) if isinstance(v, float) else (bool(v) if k == "converged" else v))
                    for k, v in r.items() if k in ("mu", "newton", "alpha", "res", "outer_its", "converged",
                                                    "inner_T_its", "rel_res")})
        print(log[-1], f"{time.time() - t0:.0f}s", flush=True)

    with threadpool_limits(1):
        opts = IpmOpts() if mu_min is None else IpmOpts(mu_min=mu_min)
        res = ipm_run(d, phi, rho, s, opts, SolverOpts(), callback=cb)
    out = {"config": name, "mu_min": mu_min, "kinetic_energy": res.kinetic_energy, "final_mu": res.mu,
           "n_systems": len(log),
           "seconds_1core": round(time.time() - t0, 1), "opts": SolverOpts().__dict__, "systems": log,
           "note": "oracle full IPM (A17-A20), written by scripts/oracle_ipm_golden.py (oracle/ only)"}
    tag = "" if mu_min is None else f"_mu{round(-__import__('math').log2(mu_min))}"
    path = os.environ.get("ORACLE_IPM_OUT") or os.path.join(ROOT, "tests", "golden", f"ipm_{name}{tag}.json")
    json.dump(out, open(path, "w"), indent=0)
    print("wrote", path, "KE", res.kinetic_energy)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C1", float(sys.argv[2]) if len(sys.argv) > 2 else None)
