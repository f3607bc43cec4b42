"""Pins for oracle D1-D2 (two-level TPFA geometry).

Every check compares against something other than the oracle's own formula:
exact rational arithmetic, counting identities stated in the paper, or
invariants of the construction.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp

from oracle.mesh import GeometryError, build_two_level
from oracle.ops import Discretisation
from synthetic import base_mesh, build_mesh, make_problem

pytestmark = pytest.mark.filterwarnings("ignore")


def _cc_exact(a, b, c):
    """Circumcentre by Cramer's rule on 2(b-a).x = |b|^2-|a|^2, 2(c-a).x = |c|^2-|a|^2."""
    a, b, c = ([Fraction(v).limit_denominator(1 << 20) for v in p] for p in (a, b, c))
    a11, a12, r1 = 2 * (b[0] - a[0]), 2 * (b[1] - a[1]), b[0] ** 2 + b[1] ** 2 - a[0] ** 2 - a[1] ** 2
    a21, a22, r2 = 2 * (c[0] - a[0]), 2 * (c[1] - a[1]), c[0] ** 2 + c[1] ** 2 - a[0] ** 2 - a[1] ** 2
    det = a11 * a22 - a12 * a21
    return ((r1 * a22 - a12 * r2) / det, (a11 * r2 - r1 * a21) / det)


def test_base_mesh_circumcentres_exact():
    v, t = base_mesh()
    g = build_two_level(v, t)
    # hand-derived: triangle (A,E,P): x = 1/4 (bisector of AE), y = 1/48
    assert _cc_exact(v[0], v[4], v[6]) == (Fraction(1, 4), Fraction(1, 48))
    for i, tri in enumerate(t):
        ex = _cc_exact(*v[tri])
        assert abs(g.cc[i, 0] - float(ex[0])) < 1e-15 and abs(g.cc[i, 1] - float(ex[1])) < 1e-15


@pytest.mark.parametrize("L", [0, 1, 2, 3])
def test_counting_identities(L):
    """N = 3 N̄ and N_E = 2 N̄_E + 3 N̄; N̄_E = 12*4^L - 3*2^L for the A1 base."""
    v, t = build_mesh(L)
    g = build_two_level(v, t)
    assert g.N == 3 * g.nbar
    assert g.NE == 2 * g.NEbar + 3 * g.nbar
    assert g.nbar == 8 * 4 ** L
    assert g.NEbar == 12 * 4 ** L - 3 * 2 ** L
    # all internal edges: every coarse cell has <= 3 neighbours, boundary cells fewer
    deg = np.bincount(np.r_[g.ebar_L, g.ebar_R], minlength=g.nbar)
    assert deg.max() == 3 and deg.sum() == 2 * g.NEbar


@pytest.mark.parametrize("name", ["T1", "C1", "C2"])
def test_areas_and_admissibility(name):
    p = make_problem(name)
    g = build_two_level(p.verts, p.tris)        # validates acuteness + orthogonality
    assert abs(g.cbar.sum() - 1.0) < 1e-13 and abs(g.c.sum() - 1.0) < 1e-13
    # the 3 kites partition their triangle
    assert np.allclose(g.c.reshape(-1, 3).sum(1), g.cbar, rtol=1e-10, atol=0)
    assert g.w_len.min() > 0 and g.e_len.min() > 0
    assert np.all((g.lam > 0) & (g.lam < 1)) and np.all((g.lam_bar > 0) & (g.lam_bar < 1))
    # type-a edges: λ = 1/2 (anchors symmetric about the bisector), |w| = half the coarse edge
    a = g.e_type == 0
    assert np.allclose(g.lam[a], 0.5, atol=1e-12)
    # type-b half edges: |e| = |ē|/2 and |w| = |w̄|/2
    b = np.nonzero(g.e_type == 1)[0]
    nb = b.size // 2
    assert np.allclose(g.e_len[b[:nb]], g.ebar_len / 2, rtol=1e-13)
    assert np.allclose(g.w_len[b[:nb]], g.wbar_len / 2, rtol=1e-12)
    assert np.allclose(g.lam[b[:nb]], g.lam_bar, rtol=1e-10)


def test_rejects_right_triangles():
    """Right triangles give coincident circumcentres, |w| = 0."""
    v = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float)
    t = np.array([[0, 1, 2], [0, 2, 3]])
    with pytest.raises(GeometryError):
        build_two_level(v, t)


def test_adjoint_and_conservation():
    """div = -grad^T diag(|w||e|) entrywise; 1^T div = 0; Π rows/cols."""
    p = make_problem("C1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    D = d.div + d.grad.T @ sp.diags(d.g.w_len * d.g.e_len)
    assert abs(D).max() < 1e-15
    assert abs(np.ones(d.N) @ d.div).max() < 1e-15
    assert np.all(np.asarray(d.Pi.sum(1)).ravel() == 1) and np.all(np.asarray(d.Pi.sum(0)).ravel() == 3)
    assert np.allclose(d.Pi.T @ d.M, d.Mbar, rtol=1e-14)
    # R_E reproduces constants
    assert np.allclose(d.RE @ np.ones(d.nbar), 1.0, atol=1e-15)
