"""The C-ABI library loads and exports every symbol include/bbot.h declares
(no compute calls: this runs without a GPU)."""
import os
import re

import pytest


def _declared(root):
    src = open(os.path.join(root, "include", "bbot.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bbot_[a-z_]+)\s*\(", src)) - {"bbot_ipm_cb"})


def test_library_exports_all_declared_symbols(root):
    import paper_2209_00315_b200 as pb
    names = _declared(root)
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(pb.lib, n)]
    assert not missing, missing
    # the binding wraps every declared call
    assert set(names) <= set(pb.EXPORTED)


def test_default_options_match_design():
    import paper_2209_00315_b200 as pb
    o = pb.default_solver_opts()
    assert (o.eps_out, o.eps_T, o.eps_A, o.restart, o.maxit) == (1e-10, 1e-1, 1e-3, 30, 400)
    assert (o.restart_T, o.maxit_inner, o.coarse_max_A, o.coarse_max_T) == (10, 50, 64, 1024)
    i = pb.default_ipm_opts()
    assert (i.mu0, i.mu_factor, i.mu_min, i.frac_to_boundary, i.newton_max) == (1.0, 0.5, 1e-8, 0.95, 30)


def test_oracle_defaults_agree_with_library():
    """Same algorithmic constants on both sides (they share no code)."""
    import paper_2209_00315_b200 as pb
    from oracle.bb import SolverOpts
    o, s = pb.default_solver_opts(), SolverOpts()
    for f in ("eps_out", "eps_T", "eps_A", "restart", "maxit", "restart_T", "maxit_inner",
              "omega_A", "omega_T", "coarse_max_A", "coarse_max_T", "coarse_max_S"):
        assert getattr(o, f) == getattr(s, f), f
    assert o.precond == 0 and s.precond == "bb"


def test_oracle_ipm_defaults_agree_with_library():
    """IPM constants (A17-A20, A14') on both sides."""
    import paper_2209_00315_b200 as pb
    from oracle.ipm import IpmOpts
    o, s = pb.default_ipm_opts(), IpmOpts()
    for f in ("mu0", "mu_factor", "mu_min", "newton_rel_tol", "newton_abs_floor", "frac_to_boundary", "newton_max",
              "mu_tight", "eps_A_tight", "simple_below_mu"):
        assert getattr(o, f) == getattr(s, f), f


def test_no_oracle_import_in_product(root):
    """The product package never imports the oracle."""
    pkg = os.path.join(root, "paper_2209_00315_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
