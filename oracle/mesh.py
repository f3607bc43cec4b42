"""D1-D2: two-level TPFA finite-volume geometry (§2.1).

Coarse mesh T̄: acute triangles, rho lives on them.  Fine mesh T: each
triangle split into 3 kites "joining the edges midpoints to the triangle's
circumcenter", phi lives on them.  Boundary edges are dropped,
so N = 3 N̄ and N_E = 2 N̄_E + 3 N̄.

Readings: A2 fine cell point = (v + cc)/2; A3 lambda_sigma =
d(x_L, sigma) / (d(x_L, sigma) + d(x_R, sigma)); orientation: L = lower index.
Fine cell index 3t + s for the kite at local vertex s of triangle t.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def circumcentre(a, b, c):
    """Circumcentre of triangles with vertices a, b, c (arrays (...,2))."""
    bx, by = b[..., 0] - a[..., 0], b[..., 1] - a[..., 1]
    cx, cy = c[..., 0] - a[..., 0], c[..., 1] - a[..., 1]
    d = 2.0 * (bx * cy - by * cx)
    b2 = bx * bx + by * by
    c2 = cx * cx + cy * cy
    ux = (cy * b2 - by * c2) / d
    uy = (bx * c2 - cx * b2) / d
    return np.stack([a[..., 0] + ux, a[..., 1] + uy], axis=-1)


def polygon_area(p):
    """Shoelace area of CCW polygons p (..., k, 2)."""
    x, y = p[..., 0], p[..., 1]
    return 0.5 * (x * np.roll(y, -1, axis=-1) - np.roll(x, -1, axis=-1) * y).sum(-1)


def dist_to_line(p, a, b):
    """Distance of points p to the lines through a, b."""
    d = b - a
    cr = d[..., 0] * (p[..., 1] - a[..., 1]) - d[..., 1] * (p[..., 0] - a[..., 0])
    return np.abs(cr) / np.hypot(d[..., 0], d[..., 1])


def max_angle_deg(p):
    out = np.zeros(p.shape[:-2])
    for i in range(3):
        u = p[..., (i + 1) % 3, :] - p[..., i, :]
        w = p[..., (i + 2) % 3, :] - p[..., i, :]
        cos = (u * w).sum(-1) / np.sqrt((u * u).sum(-1) * (w * w).sum(-1))
        out = np.maximum(out, np.degrees(np.arccos(np.clip(cos, -1.0, 1.0))))
    return out


class GeometryError(ValueError):
    pass


@dataclass
class TwoLevelMesh:
    # coarse (T̄)
    nbar: int
    cbar: np.ndarray        # |c̄| areas (N̄,)
    cc: np.ndarray          # circumcentres (N̄,2)
    ebar_L: np.ndarray      # internal coarse edges: left/right cell (N̄_E,)
    ebar_R: np.ndarray
    ebar_len: np.ndarray    # |ē|
    wbar_len: np.ndarray    # |w̄| = |cc_L - cc_R|
    lam_bar: np.ndarray     # λ̄ (weight of the L cell)
    # fine (T)
    N: int
    c: np.ndarray           # |c| kite areas (N,)
    x: np.ndarray           # cell points (N,2)
    parent: np.ndarray      # Π: fine cell -> coarse cell (N,)
    e_L: np.ndarray         # internal fine edges (N_E,)
    e_R: np.ndarray
    e_len: np.ndarray       # |e|
    w_len: np.ndarray       # |w|
    lam: np.ndarray         # λ (weight of the L cell)
    e_type: np.ndarray      # 0 = midpoint-circumcentre segment, 1 = half coarse edge

    @property
    def NE(self):
        return int(self.e_L.shape[0])

    @property
    def NEbar(self):
        return int(self.ebar_L.shape[0])

    @property
    def area(self):          # |Ω|
        return float(self.cbar.sum())


def build_two_level(verts, tris, validate: bool = True, orth_tol: float = 1e-10) -> TwoLevelMesh:
    verts = np.asarray(verts, dtype=np.float64)
    tris = np.asarray(tris, dtype=np.int64)
    nbar = tris.shape[0]
    p = verts[tris]                                   # (N̄,3,2)
    a, b, cpt = p[:, 0], p[:, 1], p[:, 2]
    cbar = polygon_area(p)
    if validate:
        if np.any(cbar <= 0):
            raise GeometryError("non-CCW or degenerate triangle")
        if np.any(max_angle_deg(p) >= 90.0):
            raise GeometryError("non-acute triangle (P:99 requires acute angles)")
    cc = circumcentre(a, b, cpt)

    # ---- coarse internal edges (boundary edges dropped)
    loc = np.array([[0, 1], [1, 2], [2, 0]])
    ev = tris[:, loc].reshape(-1, 2)                  # (3N̄,2) local edge (s, s+1)
    et = np.repeat(np.arange(nbar), 3)
    es = np.tile(np.arange(3), nbar)
    key = np.sort(ev, axis=1)
    order = np.lexsort((et, key[:, 1], key[:, 0]))
    ks = key[order]
    same = np.all(ks[1:] == ks[:-1], axis=1)
    i0 = np.nonzero(same)[0]
    j0, j1 = order[i0], order[i0 + 1]                  # two half-edges of each internal edge
    tA, tB = et[j0], et[j1]
    swap = tA > tB
    tL = np.where(swap, tB, tA)
    tR = np.where(swap, tA, tB)
    va = ks[i0, 0]
    vb = ks[i0, 1]
    ebar_len = np.hypot(*(verts[va] - verts[vb]).T)
    wbar_len = np.hypot(*(cc[tL] - cc[tR]).T)
    dL = dist_to_line(cc[tL], verts[va], verts[vb])
    dR = dist_to_line(cc[tR], verts[va], verts[vb])
    lam_bar = dL / (dL + dR)

    # ---- fine kites: cell 3t+s at vertex s
    N = 3 * nbar
    mids = 0.5 * (p + np.roll(p, -1, axis=1))         # mids[:, s] = mid(v_s, v_{s+1})
    kites = np.stack([p, mids, np.repeat(cc[:, None, :], 3, axis=1), np.roll(mids, 1, axis=1)], axis=2)
    c = polygon_area(kites).reshape(-1)                # (N,)
    x = (0.5 * (p + cc[:, None, :])).reshape(-1, 2)     # A2
    parent = np.repeat(np.arange(nbar), 3)

    # type a: between kites s and s+1 of the same triangle, segment mid(v_s,v_{s+1}) - cc
    fa1 = (3 * np.arange(nbar)[:, None] + np.arange(3)[None, :]).reshape(-1)
    fa2 = (3 * np.arange(nbar)[:, None] + (np.arange(3)[None, :] + 1) % 3).reshape(-1)
    segA0 = mids.reshape(-1, 2)
    segA1 = np.repeat(cc, 3, axis=0)

    # type b: two half coarse edges per internal coarse edge, at va and at vb
    def slot(t, v):
        return np.argmax(tris[t] == v[:, None], axis=1)
    mid_ab = 0.5 * (verts[va] + verts[vb])
    fb1 = np.concatenate([3 * tL + slot(tL, va), 3 * tL + slot(tL, vb)])
    fb2 = np.concatenate([3 * tR + slot(tR, va), 3 * tR + slot(tR, vb)])
    segB0 = np.concatenate([verts[va], verts[vb]])
    segB1 = np.concatenate([mid_ab, mid_ab])

    f1 = np.concatenate([fa1, fb1])
    f2 = np.concatenate([fa2, fb2])
    s0 = np.concatenate([segA0, segB0])
    s1 = np.concatenate([segA1, segB1])
    e_type = np.concatenate([np.zeros(fa1.size, np.int8), np.ones(fb1.size, np.int8)])
    e_L = np.minimum(f1, f2)
    e_R = np.maximum(f1, f2)
    e_len = np.hypot(*(s0 - s1).T)
    w_len = np.hypot(*(x[e_L] - x[e_R]).T)
    dL = dist_to_line(x[e_L], s0, s1)
    dR = dist_to_line(x[e_R], s0, s1)
    lam = dL / (dL + dR)

    if validate:
        for (XL, XR, S0, S1, wl, name) in (
                (cc[tL], cc[tR], verts[va], verts[vb], wbar_len, "coarse"),
                (x[e_L], x[e_R], s0, s1, w_len, "fine")):
            d = S1 - S0
            orth = np.abs(((XL - XR) * d).sum(-1)) / (wl * np.hypot(*d.T))
            if np.any(wl <= 1e-12) or np.any(orth > orth_tol):
                raise GeometryError(f"{name} mesh not TPFA-admissible (|w|>0, orthogonality)")
    return TwoLevelMesh(nbar=nbar, cbar=cbar, cc=cc, ebar_L=tL, ebar_R=tR, ebar_len=ebar_len,
                        wbar_len=wbar_len, lam_bar=lam_bar, N=N, c=c, x=x, parent=parent,
                        e_L=e_L, e_R=e_R, e_len=e_len, w_len=w_len, lam=lam, e_type=e_type)
