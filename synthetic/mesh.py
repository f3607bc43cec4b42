"""Coarse triangulations of the unit square (input generation only).

The paper needs a Delaunay triangulation with only acute angles
and uses a hierarchy of meshes, "each mesh is a refinement of the other"
(P:621).  The FVCA files it used are not available; SURVEY §8(c) A1 fixes the
stand-in: an all-acute 8-triangle base of [0,1]^2 refined L times by the
midpoint 4-split, giving exactly 8*4^L triangles (the configs' 2*N^2 counts).

Numbering is hierarchical: the 4 children of triangle t are 4t..4t+3, so cells
that are close in index are close in space (good gather locality on the GPU).
"""
from __future__ import annotations

import numpy as np

# corners A,B,C,D plus E,G (edge midpoints) and P,Q (interior).
_BASE_VERTS = np.array([
    [0.0, 0.0],        # 0 A
    [1.0, 0.0],        # 1 B
    [1.0, 1.0],        # 2 C
    [0.0, 1.0],        # 3 D
    [0.5, 0.0],        # 4 E
    [0.5, 1.0],        # 5 G
    [7.0 / 16.0, 3.0 / 16.0],  # 6 P
    [9.0 / 16.0, 3.0 / 16.0],  # 7 Q
])
# (A,E,P) (E,Q,P) (E,B,Q) (B,C,Q) (C,G,Q) (Q,G,P) (P,G,D) (D,A,P); all CCW.
_BASE_TRIS = np.array([
    [0, 4, 6], [4, 7, 6], [4, 1, 7], [1, 2, 7],
    [2, 5, 7], [7, 5, 6], [6, 5, 3], [3, 0, 6],
], dtype=np.int64)


def base_mesh():
    """The acute 8-triangle base mesh (vertices float64 (8,2), tris int64 (8,3))."""
    return _BASE_VERTS.copy(), _BASE_TRIS.copy()


def refine(verts: np.ndarray, tris: np.ndarray):
    """Midpoint 4-split of every triangle (children similar to the parent).

    Child order for parent (a,b,c) with midpoints ab, bc, ca:
      4t+0 = (a, ab, ca), 4t+1 = (ab, b, bc), 4t+2 = (ca, bc, c), 4t+3 = (ab, bc, ca).
    CCW orientation is preserved.  Shared edges get a single midpoint vertex.
    """
    verts = np.asarray(verts, dtype=np.float64)
    tris = np.asarray(tris, dtype=np.int64)
    nv = verts.shape[0]
    e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]], axis=0)
    key = np.sort(e, axis=1)
    uniq, inv = np.unique(key, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    mids = 0.5 * (verts[uniq[:, 0]] + verts[uniq[:, 1]])
    nt = tris.shape[0]
    m_ab = nv + inv[0:nt]
    m_bc = nv + inv[nt:2 * nt]
    m_ca = nv + inv[2 * nt:3 * nt]
    a, b, c = tris[:, 0], tris[:, 1], tris[:, 2]
    ch = np.stack([
        np.stack([a, m_ab, m_ca], 1),
        np.stack([m_ab, b, m_bc], 1),
        np.stack([m_ca, m_bc, c], 1),
        np.stack([m_ab, m_bc, m_ca], 1),
    ], axis=1).reshape(-1, 3)
    return np.concatenate([verts, mids], axis=0), ch


def build_mesh(L: int):
    """Base mesh refined L times: 8*4^L triangles."""
    v, t = base_mesh()
    for _ in range(L):
        v, t = refine(v, t)
    return v, t


def triangle_areas(verts, tris):
    p = verts[tris]
    d1 = p[:, 1] - p[:, 0]
    d2 = p[:, 2] - p[:, 0]
    return 0.5 * (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0])


def _max_angle_deg(p):
    """Largest interior angle of triangles p (..., 3, 2), in degrees."""
    out = np.zeros(p.shape[:-2])
    for i in range(3):
        u = p[..., (i + 1) % 3, :] - p[..., i, :]
        w = p[..., (i + 2) % 3, :] - p[..., i, :]
        cos = (u * w).sum(-1) / np.sqrt((u * u).sum(-1) * (w * w).sum(-1))
        out = np.maximum(out, np.degrees(np.arccos(np.clip(cos, -1.0, 1.0))))
    return out


def jitter_mesh(verts, tris, h: float, amp: float = 0.2, seed: int = 2,
                tries: int = 8, max_angle: float = 89.5):
    """Seeded jitter of interior vertices.

    Interior vertices in increasing index order; each draws up to `tries`
    displacements U(-amp*h, amp*h)^2 from numpy.random.default_rng(seed) and
    keeps the first one for which every incident triangle stays positively
    oriented with max angle < `max_angle` degrees; otherwise it stays put.
    Returns (new_verts, stats).
    """
    verts = np.array(verts, dtype=np.float64, copy=True)
    tris = np.asarray(tris, dtype=np.int64)
    rng = np.random.default_rng(seed)
    nv = verts.shape[0]
    eps = 1e-12
    interior = ((verts[:, 0] > eps) & (verts[:, 0] < 1 - eps) &
                (verts[:, 1] > eps) & (verts[:, 1] < 1 - eps))
    # vertex -> incident triangles
    order = np.argsort(tris.reshape(-1), kind="stable")
    vt_ptr = np.searchsorted(tris.reshape(-1)[order], np.arange(nv + 1))
    vt_tri = order // 3
    moved = 0
    disp = []
    for v in range(nv):
        if not interior[v]:
            continue
        inc = tris[vt_tri[vt_ptr[v]:vt_ptr[v + 1]]]
        for _ in range(tries):
            d = rng.uniform(-amp * h, amp * h, size=2)
            old = verts[v].copy()
            verts[v] = old + d
            p = verts[inc]
            area = triangle_areas(verts, inc)
            if np.all(area > 0) and np.all(_max_angle_deg(p) < max_angle):
                moved += 1
                disp.append(np.abs(d).max() / h)
                break
            verts[v] = old
    stats = {"interior": int(interior.sum()), "moved": moved,
             "mean_disp_inf_over_h": float(np.mean(disp)) if disp else 0.0}
    return verts, stats
