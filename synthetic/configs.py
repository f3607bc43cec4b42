"""The BASELINE.json configs C1-C5 plus small test instances.

Each config is a recipe for the problem statement only: mesh (A1 base refined L
times, optional A25 jitter), K interior density levels (Delta t = 1/(K+1),
PAPER.md P:158), and the two boundary densities (A21).  Nothing here touches
the discretisation or the solver.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .densities import cell_average, cos2_bump, gaussian, mixture, normalise_mass
from .mesh import build_mesh, jitter_mesh


@dataclass
class Problem:
    name: str
    L: int
    K: int
    verts: np.ndarray      # (nv, 2) float64
    tris: np.ndarray       # (nt, 3) int32, CCW
    rho_in: np.ndarray     # (nt,) float64 coarse cell averages, unit mass
    rho_f: np.ndarray      # (nt,) float64
    protocol: str = ""
    info: dict = field(default_factory=dict)

    @property
    def nbar(self) -> int:
        return int(self.tris.shape[0])

    @property
    def n(self) -> int:          # phi unknowns  N (K+1), N = 3 Nbar
        return 3 * self.nbar * (self.K + 1)

    @property
    def m(self) -> int:          # rho unknowns  Nbar K
        return self.nbar * self.K


def _gauss_pair(c0, c1, sigma, floor):
    return (mixture([gaussian(*c0, sigma)], floor), mixture([gaussian(*c1, sigma)], floor))


def _random_mixture(seed, ncomp, sigma_range=None, sigma_fixed=None, floor=0.0):
    rng = np.random.default_rng(seed)
    comps, desc = [], []
    for _ in range(ncomp):
        cx = rng.uniform(0.2, 0.8)
        cy = rng.uniform(0.2, 0.8)
        sg = rng.uniform(*sigma_range) if sigma_fixed is None else sigma_fixed
        w = rng.uniform(0.5, 1.5)
        comps.append(gaussian(cx, cy, sg, w))
        desc.append((cx, cy, sg, w))
    return mixture(comps, floor), desc


# name -> (L, K, jitter, density recipe, protocol)
CONFIGS = {
    # tiny instances for the oracle pins and quick parity (not BASELINE configs)
    "T0": dict(L=0, K=2, dens=("gauss", (0.3, 0.3), (0.7, 0.7), 0.1, 1e-3), protocol="unit"),
    "T1": dict(L=1, K=4, dens=("gauss", (0.3, 0.3), (0.7, 0.7), 0.1, 1e-3), protocol="unit"),
    "T2": dict(L=2, K=8, dens=("gauss", (0.3, 0.3), (0.7, 0.7), 0.1, 1e-3), protocol="unit"),
    "T2b": dict(L=2, K=8, dens=("bump", (0.3, 0.3), (0.7, 0.7), 0.2), protocol="unit"),
    # test case 3, compression: not a BASELINE config
    "T2c": dict(L=2, K=8, dens=("compress", (0.5, 0.5), 0.35, 0.5), protocol="unit"),
    "C1c": dict(L=3, K=8, dens=("compress", (0.5, 0.5), 0.35, 0.5), protocol="compression workload"),
    # BASELINE.json configs[0..4]
    "C1": dict(L=3, K=8, dens=("gauss", (0.3, 0.3), (0.7, 0.7), 0.1, 1e-3),
               protocol="full IPM, mu 1 -> 1e-8 by 0.5"),
    "C2": dict(L=5, K=32, jitter=True, dens=("gauss", (0.25, 0.5), (0.75, 0.5), 0.08, 1e-4),
               protocol="full IPM"),
    "C3": dict(L=6, K=64, dens=("bump", (0.3, 0.3), (0.7, 0.7), 0.2),
               protocol="single solve at mu=2^-20 + full IPM"),
    "C4": dict(L=7, K=128, dens=("mix", 40, 41), protocol="full IPM at P=1,2,4,8"),
    "C5": dict(L=8, K=256, dens=("c5",), protocol="20 solves mu 1e-2 -> 1e-8"),
}


def make_problem(name: str, L: int | None = None, K: int | None = None) -> Problem:
    """Build config `name`; L/K may be overridden (same density recipe)."""
    cfg = CONFIGS[name]
    L = cfg["L"] if L is None else L
    K = cfg["K"] if K is None else K
    verts, tris = build_mesh(L)
    info = {}
    if cfg.get("jitter"):
        h = 1.0 / (2 ** (L + 1))           # median edge length of the A1 hierarchy (A1)
        verts, st = jitter_mesh(verts, tris, h=h, amp=0.2, seed=2)
        info["jitter"] = st
    d = cfg["dens"]
    if d[0] == "gauss":
        _, c0, c1, sigma, floor = d
        fin, ffi = _gauss_pair(c0, c1, sigma, floor)
    elif d[0] == "bump":
        _, c0, c1, radius = d
        fin, ffi = cos2_bump(*c0, radius), cos2_bump(*c1, radius)
    elif d[0] == "compress":
        # test case 3 (NEXT f3): a cos^2 bump compressed about its centre by the
        # dilation x -> c + theta (x - c); the target theta^-2 b(|x - c| / theta) is the same
        # bump with radius theta * r0 (unit mass after normalisation)
        _, c, radius, theta = d
        fin, ffi = cos2_bump(*c, radius), cos2_bump(*c, theta * radius)
        info["compression"] = dict(centre=c, radius=radius, theta=theta)
    elif d[0] == "mix":
        fin, din = _random_mixture(d[1], 3, sigma_range=(0.05, 0.15), floor=1e-4)
        ffi, dfi = _random_mixture(d[2], 3, sigma_range=(0.05, 0.15), floor=1e-4)
        info["mixtures"] = (din, dfi)
    elif d[0] == "c5":
        def fin(x, y):
            return np.ones_like(x)
        ffi, dfi = _random_mixture(50, 4, sigma_fixed=0.05, floor=1e-5)
        info["mixtures"] = (None, dfi)
    else:
        raise ValueError(d)
    rho_in = normalise_mass(cell_average(fin, verts, tris), verts, tris)
    rho_f = normalise_mass(cell_average(ffi, verts, tris), verts, tris)
    return Problem(name=name, L=L, K=K, verts=np.ascontiguousarray(verts),
                   tris=np.ascontiguousarray(tris.astype(np.int32)),
                   rho_in=rho_in, rho_f=rho_f, protocol=cfg["protocol"], info=info)
