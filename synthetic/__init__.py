"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NONE of the method's arithmetic (no TPFA geometry, no
operators, no solver): it only produces the *problem statement* the paper's
C-ABI takes -- a coarse triangulation (vertices + CCW triangles), the number of
interior density levels K, and the boundary densities rho_in / rho_f as coarse
cell averages.  Every recipe is stated in DESIGN.md §3.

  mesh.py       acute 8-triangle base of [0,1]^2 + midpoint 4-split refinement
                (SURVEY §8(c) A1), seeded vertex jitter (A25)
  densities.py  Gaussian / cos^2-bump / mixture densities, cell-averaged with
                a fixed degree-5 7-point rule and scaled to unit mass (A21)
  configs.py    BASELINE.json configs C1-C5 + small test instances
  states.py     seeded synthetic states (phi, rho, s) for single-solve parity
"""
from .mesh import base_mesh, refine, build_mesh, jitter_mesh, triangle_areas
from .densities import cell_average, gaussian, cos2_bump, mixture, normalise_mass
from .configs import CONFIGS, make_problem, Problem
from .states import random_state, initial_state

__all__ = [
    "base_mesh", "refine", "build_mesh", "jitter_mesh", "triangle_areas",
    "cell_average", "gaussian", "cos2_bump", "mixture", "normalise_mass",
    "CONFIGS", "make_problem", "Problem", "random_state", "initial_state",
]
