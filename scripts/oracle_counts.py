"""Write tests/golden/oracle_counts.json: the oracle's own FGMRES outer-iteration and
inner counts on the first IPM Newton system (A19 point, mu = 1) of the configs (calls only
oracle/ and synthetic/, one core).  The GPU parity tests hold the CUDA path to these counts
(+-1 outer) on the configs too large to re-run the oracle inside a test (C2: ~1 min, C3:
~15 min, C4: hours on one core).  ORACLE_COUNTS_OUT=<file>: write there instead (parallel
runs, merged afterwards)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from threadpoolctl import threadpool_limits  # noqa: E402

from oracle.bb import BBSolver, SolverOpts  # noqa: E402
from oracle.ops import Discretisation  # noqa: E402
from synthetic import initial_state, make_problem  # noqa: E402

OUT = os.environ.get("ORACLE_COUNTS_OUT") or os.path.join(ROOT, "tests", "golden", "oracle_counts.json")


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        p = make_problem(name)
        d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
        phi, rho, s = initial_state(p, 1.0)
        t = time.time()
        with threadpool_limits(1):
            S = BBSolver(d, phi, rho, s, 1.0, SolverOpts())
            S.solve()
        key = f"{name}/init/mu=1"
        data[key] = dict(outer_its=S.stats["outer_its"], inner_T_its=S.stats["inner_T_its"],
                         inner_A_its_max=S.stats["inner_A_its_max"], inner_A_its_total=S.stats["inner_A_its_total"],
                         converged=S.stats["converged"], rel_res=float(S.stats["rel_res"]),
                         seconds_1core=round(time.time() - t, 1))
        print(key, data[key], flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2"])
