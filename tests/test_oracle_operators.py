"""Pins for oracle D4-D11: residuals, Jacobian, projector, BB operators."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.ops import Discretisation
from synthetic import initial_state, make_problem, random_state


@pytest.fixture(scope="module")
def small():
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=3, mu=0.05)
    return p, d, phi, rho, s


def test_A_blocks_laplacian(small):
    """A_k symmetric, A_k 1 = 0, PSD."""
    _, d, phi, rho, s = small
    for Ak in d.A_blocks(rho):
        assert abs(Ak - Ak.T).max() < 1e-15
        assert abs(Ak @ np.ones(d.N)).max() < 1e-13
        ev = np.linalg.eigvalsh(Ak.toarray())
        assert ev.min() > -1e-12 * ev.max()
        assert np.sum(ev < 1e-10 * ev.max()) == 1      # kernel = constants only


def test_remark_2_2_mass(small):
    """1^T F_φ^k = -c̄^T(ρ^k - ρ^{k-1})/Δt (Remark 2.2)."""
    _, d, phi, rho, s = small
    rho = rho * (1 + 0.1 * np.sin(np.arange(rho.size)))      # break mass equality on purpose
    F_phi, _, _ = d.residual(phi, rho, s, 0.05)
    R = d.rho_slices(rho)
    Fp = F_phi.reshape(d.K + 1, d.N)
    for k in range(1, d.K + 2):
        assert abs(Fp[k - 1].sum() + d.Mbar @ (R[k] - R[k - 1]) / d.dt) < 1e-12


def test_residual_closed_forms(small):
    """constant-in-time ρ with slice-constant φ -> F_φ = 0;
    φ = 0 -> F_ρ = M̄ s;  F_s = ρ s - μ."""
    p, d, phi, rho, s = small
    r0 = np.full(d.nbar, 1.0)
    d2 = Discretisation(p.verts, p.tris, p.K, r0, r0)
    rho_c = np.tile(r0, d.K)
    phi_c = np.repeat(np.linspace(0, 1, d.K + 1), d.N)
    F_phi, _, _ = d2.residual(phi_c, rho_c, s, 0.1)
    assert abs(F_phi).max() < 1e-14
    _, F_rho, F_s = d.residual(np.zeros(d.n), rho, s, 0.3)
    assert np.allclose(F_rho, np.tile(d.Mbar, d.K) * s, rtol=1e-14)
    assert np.allclose(F_s, rho * s - 0.3, rtol=0, atol=1e-15)


def test_jacobian_finite_difference(small):
    """The block matrix (3.1) is the Jacobian of (F_φ;F_ρ;F_s) -- only with A5."""
    _, d, phi, rho, s = small
    n, m = d.n, d.m
    J = d.jacobian(phi, rho, s)
    x0 = np.concatenate([phi, rho, s])

    def F(x):
        return np.concatenate(d.residual(x[:n], x[n:n + m], x[n + m:], 0.05))
    rng = np.random.default_rng(0)
    for _ in range(3):
        v = rng.standard_normal(x0.size)
        eps = 1e-5
        fd = (F(x0 + eps * v) - F(x0 - eps * v)) / (2 * eps)
        assert np.linalg.norm(fd - J @ v) <= 1e-8 * np.linalg.norm(J @ v)


def test_jacobian_kernel_and_shift(small):
    """J (1;0;0) = 0 (Remark 3.1);  B L δλ = M̄ Ē^T δλ for slice constants with
    c_{k+1} - c_k = Δt λ^k (the shift structure of (4.13), A5)."""
    _, d, phi, rho, s = small
    n, m = d.n, d.m
    J = d.jacobian(phi, rho, s)
    assert abs(J @ np.r_[np.ones(n), np.zeros(2 * m)]).max() < 1e-12
    lam = np.random.default_rng(1).standard_normal(d.K)
    c = np.concatenate([[0.0], np.cumsum(d.dt * lam)])
    x = np.repeat(c, d.N)
    B = d.B(phi)
    assert np.allclose(B @ x, (d.Mbar[None, :] * lam[:, None]).reshape(-1), rtol=1e-12, atol=1e-13)
    assert abs(d.A(rho) @ x).max() < 1e-12


def test_projector_identities(small):
    """P^2 = P; Ē M̄ Ē^T = |Ω| I; c̄^T (P^T y)^k = 0; 1^T (B^T P^T y)^k = 0."""
    _, d, phi, rho, s = small
    y = np.random.default_rng(2).standard_normal(d.m)
    assert np.allclose(d.P(d.P(y)), d.P(y), atol=1e-15)
    assert np.allclose(d.PT(d.PT(y)), d.PT(y), atol=1e-15)
    assert abs(d.Mbar.sum() - d.area) < 1e-15 and abs(d.area - 1.0) < 1e-13
    assert abs(d.PT(y).reshape(d.K, d.nbar) @ d.Mbar).max() < 1e-14
    assert abs(d.P(y).reshape(d.K, d.nbar).sum(1)).max() < 1e-14
    BT = d.B(phi).T
    assert abs((BT @ d.PT(y)).reshape(d.K + 1, d.N).sum(1)).max() < 1e-12


def test_JP_kernel_dimension():
    """dim ker J_P = 2K+1 (A30): per-slice constants in δφ̃ (K+1) and in δρ (K)."""
    p = make_problem("T0")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    phi, rho, s = random_state(p, seed=4, mu=0.1)
    JP, *_ = d.make_JP(phi, rho, s)
    M = np.stack([JP(e) for e in np.eye(d.n + d.m)], axis=1)
    sv = np.linalg.svd(M, compute_uv=False)
    assert np.sum(sv < 1e-10 * sv[0]) == 2 * d.K + 1


def test_T_at_zero_potential_is_time_laplacian():
    """φ = 0: 𝒢 = 0, so T = diag(s/ρ)Ã + M̄ D_t D_t^T with the Dirichlet time
    Laplacian (D10 identity: -B M^{-1} B̃ ⊇ D_t M̄ D_t^T)."""
    p = make_problem("T1")
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    _, rho, s = random_state(p, seed=5, mu=0.1)
    T = d.T_matrix(np.zeros(d.n), rho, s).toarray()
    Lt = (2 * np.eye(d.K) - np.eye(d.K, k=1) - np.eye(d.K, k=-1)) / d.dt ** 2
    expect = np.diag(s / rho) @ d.Atilde(rho).toarray() + np.kron(Lt, np.diag(d.Mbar))
    assert np.allclose(T, expect, rtol=1e-12, atol=1e-12 * abs(expect).max())


def test_B_and_Btilde_consistency():
    """B ~ M̄(∂t + ∇φ·∇) on the φ-grid -> ρ-grid and B̃ ~ M(∂t + ∇φ·∇)
    on the ρ-grid -> φ-grid (reading A8): for a linear φ = a·x and a
    smooth Z(t,x), the discrete images converge at first order to the
    continuum ones (errors halve under joint h, Δt refinement).  A wrong sign
    or a wrong time orientation of either operator makes the error O(1)."""
    a = np.array([0.3, 0.2])

    def Z(t, x, y):
        return np.sin(np.pi * t) * np.cos(np.pi * x) * np.cos(np.pi * y)

    def LZ(t, x, y):       # ∂t Z + a·∇Z
        return (np.pi * np.cos(np.pi * t) * np.cos(np.pi * x) * np.cos(np.pi * y)
                - a[0] * np.pi * np.sin(np.pi * t) * np.sin(np.pi * x) * np.cos(np.pi * y)
                - a[1] * np.pi * np.sin(np.pi * t) * np.cos(np.pi * x) * np.sin(np.pi * y))
    eB, eBt = [], []
    for L, K in [(2, 4), (3, 8), (4, 16)]:
        p = make_problem("T1", L=L, K=K)
        d = Discretisation(p.verts, p.tris, K, np.ones(8 * 4 ** L), np.ones(8 * 4 ** L))
        xf, cc = d.g.x, d.g.cc
        phi = np.tile(a[0] * xf[:, 0] + a[1] * xf[:, 1], K + 1)
        tk = np.arange(1, K + 1) / (K + 1)               # ρ times t^k
        th = (np.arange(1, K + 2) - 0.5) / (K + 1)       # φ times (t^{k-1}+t^k)/2
        z = np.concatenate([Z(t, cc[:, 0], cc[:, 1]) for t in tk])
        agg = lambda v: (v.reshape(K + 1, -1) @ d.Pi).reshape(-1)   # sum kites per triangle
        ex = np.concatenate([LZ(t, xf[:, 0], xf[:, 1]) * d.M for t in th])
        eBt.append(np.linalg.norm(agg(d.Btilde(phi) @ z) - agg(ex)) / np.linalg.norm(agg(ex)))
        x = np.concatenate([Z(t, xf[:, 0], xf[:, 1]) for t in th])
        ex2 = np.concatenate([LZ(t, cc[:, 0], cc[:, 1]) * d.Mbar for t in tk])
        eB.append(np.linalg.norm(d.B(phi) @ x - ex2) / np.linalg.norm(ex2))
    for e in (eB, eBt):
        assert e[0] < 0.15 and e[1] < 0.6 * e[0] and e[2] < 0.6 * e[1], (eB, eBt)


# --------------------------------------------------------------------------- Ã, R̄, DR pins
def _jittered_disc(L=2, K=2, seed=7):
    """A jittered A1 mesh (A25 recipe, another seed): λ̄, λ ≠ ½ on almost every edge, so a
    swapped or rescaled reconstruction weight cannot pass by symmetry."""
    from synthetic import build_mesh, jitter_mesh
    v, t = build_mesh(L)
    v, _ = jitter_mesh(v, t, h=1.0 / 2 ** (L + 1), amp=0.2, seed=seed)
    nb = t.shape[0]
    return Discretisation(v, t, K, np.ones(nb), np.ones(nb))


def _interior_triangles(g):
    """Coarse cells whose three edges are all internal (boundary edges are dropped)."""
    cnt = np.bincount(np.r_[g.ebar_L, g.ebar_R], minlength=g.nbar)
    return np.nonzero(cnt == 3)[0]


def test_Atilde_interior_cell_identity():
    """Ã_k = Ē_c diag(|ē| R̄ρ^k/|w̄|) Ē_cᵀ "discretizes -∇·(ρ∇)":
    for u = a·x sampled at the circumcentres and ρ = e_i (one coarse cell),
        uᵀ Ã(e_i) u = Σ_{ē ⊂ ∂i} |ē| (R̄e_i)_ē (a·n_ē)² |w̄_ē| = Σ_ē |ē| d(cc_i, ē) (a·n_ē)² = |c̄_i| |a|²
    exactly, because (R̄e_i)_ē = d(cc_i, ē)/|w̄| (A3 on the coarse mesh) and, by the divergence
    theorem with the circumcentre's perpendicular feet at the edge midpoints,
    Σ_ē |ē| d(cc_i, ē) n nᵀ = |c̄_i| I for every triangle with three internal edges.
    A swapped λ̄ (1 - λ̄), or Ã scaled by any factor, breaks it."""
    d = _jittered_disc()
    g = d.g
    lam = g.lam_bar
    assert np.abs(lam - 0.5).max() > 0.05            # the mesh really is asymmetric
    rng = np.random.default_rng(11)
    inner = _interior_triangles(g)
    assert inner.size > g.nbar // 2
    for a in (np.array([1.0, 0.0]), np.array([0.0, 1.0]), rng.standard_normal(2)):
        u = g.cc @ a
        for i in inner:
            rho = np.zeros(d.K * d.nbar)
            rho[i] = 1.0                              # slice 1 = e_i
            At = d.Atilde_blocks(rho)[0]
            val = u @ (At @ u)
            assert abs(val - g.cbar[i] * (a @ a)) <= 1e-12 * g.cbar[i] * (a @ a), (i, val)


def test_Atilde_symmetric_zero_rowsum_psd():
    """Ã_k = Ãᵀ_k, Ã_k 1 = 0 and PSD (a weighted graph Laplacian)."""
    d = _jittered_disc()
    rho = np.random.default_rng(3).uniform(0.1, 2.0, d.K * d.nbar)
    for At in d.Atilde_blocks(rho):
        assert abs(At - At.T).max() < 1e-15
        assert abs(At @ np.ones(d.nbar)).max() < 1e-13 * abs(At).max()
        ev = np.linalg.eigvalsh(At.toarray())
        assert ev.min() > -1e-12 * ev.max()


def test_DR_interior_cell_identity():
    """The fine reconstruction (A3: λ_σ = d(x_L,σ)/|w|): for φ = a·x sampled at the
    fine cell points, (DR (grad φ)²)_i = Σ_σ R_E[σ,i] |w_σ||e_σ| (a·n_σ)² = Σ_{kites f ⊂ i}
    Σ_{σ ∋ f} |e_σ| d(x_f, σ) (a·n_σ)² = |c̄_i| |a|²  for coarse cells with three internal
    edges (each kite is cyclic with its anchor (v+cc)/2 as circumcentre, A2, so the same
    divergence-theorem identity holds kite by kite).  This pins λ, R_E and DR (a swapped λ,
    a dropped |w| or |e|, or a factor fails it); it is the consistency DR(∇φ)² ≈ |c̄||∇φ|²
    behind the kinetic energy (1.1)."""
    d = _jittered_disc()
    g = d.g
    assert np.abs(g.lam[g.e_type == 1] - 0.5).max() > 0.05
    inner = _interior_triangles(g)
    rng = np.random.default_rng(12)
    for a in (np.array([1.0, 0.0]), np.array([0.0, 1.0]), rng.standard_normal(2)):
        phi = g.x @ a
        gp = d.grad @ phi
        val = d.DR @ (gp ** 2)
        assert np.allclose(val[inner], g.cbar[inner] * (a @ a), rtol=1e-12, atol=0)
        # and the same identity through the kinetic energy D12 for a slice-constant-in-time
        # linear φ with ρ ≡ 1 on the interior cells: KE-per-slice = ½ Σ_i ρ_i |c̄_i| |a|²


def test_Atilde_reading_is_psd_sign():
    """Sign reading (DESIGN §2 A35): the printed 'div · diag · grad' of P:1619-1623 is read as
    +Ē_c diag(·) Ē_cᵀ, i.e. Ã discretises -∇·(ρ∇) (P:1617 'discretizes -Δρ'), PSD: for a
    nonconstant u, uᵀÃu > 0 -- with the other sign the BB Schur approximation T has negative
    diagonal entries (the time Laplacian part is PSD, test_T_at_zero_potential_is_time_laplacian)."""
    d = _jittered_disc()
    rho = np.ones(d.K * d.nbar)
    u = d.g.cc[:, 0]
    assert u @ (d.Atilde_blocks(rho)[0] @ u) > 0.1 * d.area
