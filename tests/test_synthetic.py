"""The seeded input generators (synthetic/): counts, seeds, quadrature, masses."""
import numpy as np
import pytest

from synthetic import CONFIGS, build_mesh, cell_average, make_problem, triangle_areas
from synthetic.densities import QUAD_BARY, QUAD_W


def test_quadrature_degree5_exact():
    """The 7-point rule integrates all monomials x^a y^b, a+b <= 5 exactly on the
    reference triangle: ∫ x^a y^b = a! b! / (a+b+2)!."""
    from math import factorial
    v = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    pts = QUAD_BARY @ v
    assert abs(QUAD_W.sum() - 1.0) < 1e-15
    for a in range(6):
        for b in range(6 - a):
            q = 0.5 * (QUAD_W @ (pts[:, 0] ** a * pts[:, 1] ** b))
            ex = factorial(a) * factorial(b) / factorial(a + b + 2)
            assert abs(q - ex) < 1e-15


@pytest.mark.parametrize("name,nbar,K", [("C1", 512, 8), ("C2", 8192, 32), ("C3", 32768, 64)])
def test_config_sizes(name, nbar, K):
    p = make_problem(name)
    assert p.nbar == nbar and p.K == K
    area = triangle_areas(p.verts, p.tris)
    assert abs(area @ p.rho_in - 1) < 1e-13 and abs(area @ p.rho_f - 1) < 1e-13
    assert p.rho_in.min() >= 0 and p.rho_f.min() >= 0
    if name == "C3":
        assert (p.rho_in == 0).sum() > 0          # compact support (A26)


def test_jitter_is_seeded_and_valid():
    a, b = make_problem("C2"), make_problem("C2")
    assert np.array_equal(a.verts, b.verts)
    st = a.info["jitter"]
    assert 0.4 < st["moved"] / st["interior"] < 0.7
    assert triangle_areas(a.verts, a.tris).min() > 0


def test_mixture_seeds_c4():
    (din, dfi) = make_problem("T1").info.get("mixtures", (None, None))
    assert din is None
    v, t = build_mesh(1)
    f = lambda x, y: np.ones_like(x)
    assert np.allclose(cell_average(f, v, t), 1.0)
    assert set(CONFIGS) >= {"C1", "C2", "C3", "C4", "C5"}
