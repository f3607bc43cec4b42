"""I3: pairwise-aggregation algebraic multigrid -- the role of AGMG.

PARITY UNPINNED by the paper: AGMG's internals are not in PAPER.md (it is an
external library).  This is the build's own, deterministic
algorithm (DESIGN.md §2 "I3"); the CUDA path implements the
same definition, and only this oracle pins it (plus the generic AMG sanity
pins in tests: Galerkin identity, symmetry of the V-cycle, convergence).

Definition (both sides):
  * rows are grouped in slices (time levels) -- for AMG(T) in time BLOCKS of consecutive
    slices (time_blocks below, A42); couplings across slices (blocks) are never
    used for aggregation (block-diagonal A_k: none exist; T: within a time block only).
  * strength s_ij = (|a_ij| + |a_ji|)/2, j != i, same slice (symmetrised so that
    mutual-maximum matching always progresses on nonsymmetric T).
  * pairwise matching, 16 synchronous rounds: every free row i with
    M_i = max_j s_ij (over free j) > 1e-10 |a_ii| proposes
    p(i) = argmin_prio{ j free : s_ij >= (1 - tau) M_i }   (tau = 1e-8; prio(j) =
    (lowbias32 hash of j, j): near-ties are broken by a fixed pseudo-random
    priority so that uniform-weight graphs match in parallel, not along chains);
    i and j pair iff p(i) = j and p(j) = i.
  * attach: a row still free with M'_i = max_j s_ij over MATCHED j > 1e-10 |a_ii|
    joins the pair of t(i) = argmin_prio{ j matched : s_ij >= (1 - tau) M'_i }; other
    leftovers are singletons.  (Without it, maximal matchings on the dense coarse
    graphs leave most rows single and coarsening stalls: C3/C4 coarsest blocks of
    100-400 rows per slice.)
  * coarse numbering: aggregates ordered by their smallest member (a pair's
    leader is its smaller row; attached rows take their pair's index).
  * two matching passes per level (pass 2 on the Galerkin matrix of pass 1);
    prolongation piecewise constant; coarse matrix Galerkin  A_c = P^T A P.
  * stop: mode "A": max rows per slice <= coarse_max (64); mode "T": total rows
    <= coarse_max (1024); or no coarsening (n_c > 0.9 n); or max_levels.
  * smoother: damped Jacobi (omega), V(1,1) from a zero initial guess.
  * coarsest: mode "A": per slice, grounded at the slice's first row, then the
    slice mean removed;  mode "T": dense solve;  mode "As" (the shifted, nonsingular
    per-slice blocks A_k + alpha I of the HSS preconditioner, NEXT f2): everything as
    mode "A" except that the per-slice coarsest block is inverted as it is (no grounding,
    no mean removal).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

TAU = 1e-8
DECOUPLED = 1e-10
KC_ROWS = 4096      # mode A: K-cycle on coarse levels with <= KC_ROWS rows per slice ...
KC_MIN_LEVELS = 7   # ... in hierarchies of >= KC_MIN_LEVELS levels.  Plain aggregation
#                    V-cycles lose level independence: per-slice PCG to 1e-3 needs 29 its on
#                    C2 (5 levels) but 64 on C4 (8 levels); the K-cycle on the coarse levels
#                    brings C4 back to ~31, while on the shallow C2 it only costs
_M32 = np.uint64(0xFFFFFFFF)


TIME_BLOCK = 1   # A42: slices per AMG(T) aggregation block (1 = I3's within-slice rule)


def time_blocks(K: int) -> np.ndarray:
    """A42: the aggregation unit of AMG(T), blocks of TIME_BLOCK consecutive density slices
    (the last block taking the remainder); aggregates never span two blocks.  T couples
    consecutive slices (the time Laplacian in -B M^-1 B~, A8), which single-slice aggregates
    never coarsen; blocks of max(1, K/8) slices were measured (A42): 2-3x fewer
    T-GMRES iterations at the A19 point and on some IPM iterates, 2x MORE on others (C2 at
    mu = 1 after five Newton steps: 606 -> 1296; the C3 IPM stalled 30x earlier in mu), so
    the build keeps within-slice aggregation (B = 1).  Returns the block of each slice (K,)."""
    B = TIME_BLOCK
    nb = max(1, K // B)
    return np.minimum(np.arange(K) // B, nb - 1)


def prio(j):
    """Tie-break priority of row j among near-equal strengths: a fixed 32-bit
    integer hash (lowbias32), then the index.  Lowest priority wins.  (An index
    tie-break makes uniform-weight graphs match sequentially, one pair per round
    along a chain, so 16 rounds leave most rows unmatched.)"""
    x = np.asarray(j, dtype=np.uint64) & _M32
    x = x ^ (x >> np.uint64(16))
    x = (x * np.uint64(0x7FEB352D)) & _M32
    x = x ^ (x >> np.uint64(15))
    x = (x * np.uint64(0x846CA68B)) & _M32
    x = x ^ (x >> np.uint64(16))
    return (x << np.uint64(32)) | (np.asarray(j, dtype=np.uint64) & _M32)


def _row_of_nnz(A: sp.csr_matrix):
    return np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))


def match(A: sp.csr_matrix, slice_of_row: np.ndarray, rounds: int = 16):
    """Pairwise matching; returns (agg (n,) coarse index, nc, slice_of_coarse)."""
    n = A.shape[0]
    A = A.tocsr()
    diag = np.abs(A.diagonal())
    # symmetrised within-slice strength S = (|A| + |A|^T)/2 restricted to i != j, same slice
    rows = _row_of_nnz(A)
    keep = (A.indices != rows) & (slice_of_row[A.indices] == slice_of_row[rows])
    S = sp.csr_matrix((np.abs(A.data[keep]), (rows[keep], A.indices[keep])), shape=A.shape)
    S = ((S + S.T) * 0.5).tocsr()
    S.sort_indices()
    rows = _row_of_nnz(S)
    cols = S.indices
    s = S.data
    coupled = np.ones(cols.size, dtype=bool)
    pc = prio(cols)
    partner = np.full(n, -1, dtype=np.int64)
    free = np.ones(n, dtype=bool)
    for _ in range(rounds):
        ok = coupled & free[rows] & free[cols]
        sv = np.where(ok, s, -np.inf)
        Mrow = np.full(n, -np.inf)
        np.maximum.at(Mrow, rows, sv)
        has = free & (Mrow > DECOUPLED * diag)
        cand = ok & has[rows] & (s >= (1.0 - TAU) * Mrow[rows])
        best = np.full(n, np.iinfo(np.uint64).max, dtype=np.uint64)
        np.minimum.at(best, rows[cand], pc[cand])
        prop = np.where(has, (best & _M32).astype(np.int64), -1)
        i = np.nonzero(prop >= 0)[0]
        mutual = i[prop[prop[i]] == i]
        partner[mutual] = prop[mutual]
        free[mutual] = False
    # attach step: a row left unmatched joins the pair of its strongest MATCHED
    # neighbour (near-ties -> lower index), so every coupled row ends in an
    # aggregate of >= 2 rows and coarsening cannot stall on dense coarse graphs
    idx = np.arange(n)
    pair_leader = np.where(partner >= 0, np.minimum(idx, partner), idx)
    okm = free[rows] & (partner[cols] >= 0)
    sv = np.where(okm, s, -np.inf)
    Mm = np.full(n, -np.inf)
    np.maximum.at(Mm, rows, sv)
    hasm = free & (Mm > DECOUPLED * diag)
    cand = okm & hasm[rows] & (s >= (1.0 - TAU) * Mm[rows])
    tb = np.full(n, np.iinfo(np.uint64).max, dtype=np.uint64)
    np.minimum.at(tb, rows[cand], pc[cand])
    tgt = (tb & _M32).astype(np.int64)
    leader = pair_leader.copy()
    att = np.nonzero(hasm)[0]
    leader[att] = pair_leader[tgt[att]]
    is_leader = leader == idx
    cidx = np.cumsum(is_leader) - 1
    agg = cidx[leader]
    nc = int(is_leader.sum())
    return agg, nc, slice_of_row[is_leader]


def galerkin(A: sp.csr_matrix, agg: np.ndarray, nc: int) -> sp.csr_matrix:
    n = A.shape[0]
    P = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, nc))
    Ac = (P.T @ A @ P).tocsr()
    Ac.sum_duplicates()
    Ac.sort_indices()
    return Ac


@dataclass
class Level:
    A: sp.csr_matrix
    slice_of_row: np.ndarray
    dinv: np.ndarray
    agg: np.ndarray | None = None      # fine row -> coarse row (None at the coarsest)
    nc: int = 0


@dataclass
class Hierarchy:
    levels: list
    mode: str
    omega: float
    coarse_inv: list = field(default_factory=list)   # mode A: per slice (rows, inv of grounded block)
    coarse_dense_inv: np.ndarray | None = None        # mode T
    nslices: int = 0
    kcycle: list = field(default_factory=list)       # level l: coarse correction INTO l by the K-cycle

    @property
    def sizes(self):
        return [lv.A.shape[0] for lv in self.levels]


def _slice_sizes(slice_of_row, nslices):
    return np.bincount(slice_of_row, minlength=nslices)


def setup(A: sp.csr_matrix, slice_of_row: np.ndarray, mode: str, omega: float,
          coarse_max: int, max_levels: int = 25) -> Hierarchy:
    A = A.tocsr()
    nslices = int(slice_of_row.max()) + 1 if slice_of_row.size else 0
    levels = []
    cur, cur_slice = A, np.asarray(slice_of_row, dtype=np.int64)
    while True:
        n = cur.shape[0]
        dg = (np.asarray(abs(cur).sum(axis=1)).ravel() if mode == "T" else cur.diagonal())
        perslice = mode in ("A", "As")
        lv = Level(A=cur, slice_of_row=cur_slice, dinv=1.0 / dg)
        levels.append(lv)
        small = (_slice_sizes(cur_slice, nslices).max() <= coarse_max) if perslice else (n <= coarse_max)
        if small or len(levels) >= max_levels:
            break
        agg1, nc1, sl1 = match(cur, cur_slice)
        A1 = galerkin(cur, agg1, nc1)
        agg2, nc2, sl2 = match(A1, sl1)
        if nc2 > 0.9 * n:
            break
        lv.agg = agg2[agg1]
        lv.nc = nc2
        cur = galerkin(A1, agg2, nc2)
        cur_slice = sl2
    H = Hierarchy(levels=levels, mode=mode, omega=omega, nslices=nslices)
    L = len(levels)
    H.kcycle = [mode in ("A", "As") and L >= KC_MIN_LEVELS and 0 < l < L - 1 and
                _slice_sizes(levels[l].slice_of_row, nslices).max() <= KC_ROWS for l in range(L)]
    Ac = levels[-1].A.toarray() if (mode in ("A", "As") or levels[-1].A.shape[0] <= coarse_max) else None
    if mode == "A":
        sl = levels[-1].slice_of_row
        for k in range(nslices):
            rows = np.nonzero(sl == k)[0]
            blk = Ac[np.ix_(rows, rows)]
            inv = np.linalg.inv(blk[1:, 1:]) if rows.size > 1 else np.zeros((0, 0))
            H.coarse_inv.append((rows, inv))
    elif mode == "As":
        sl = levels[-1].slice_of_row
        for k in range(nslices):
            rows = np.nonzero(sl == k)[0]
            H.coarse_inv.append((rows, np.linalg.inv(Ac[np.ix_(rows, rows)])))
    elif Ac is not None:
        H.coarse_dense_inv = np.linalg.inv(Ac)
    # else: coarsening stalled above coarse_max (decoupled rows: e.g. AMG(Ŝ) at φ = 0 collapses
    # every cell's time line and leaves a diagonal matrix); the coarsest "solve" is then one
    # l1-Jacobi sweep from zero -- exact for a diagonal matrix (I3, A32)
    return H


def _coarse_solve(H: Hierarchy, b):
    if H.mode == "T":
        if H.coarse_dense_inv is None:                     # stalled coarsening (setup)
            return H.omega * H.levels[-1].dinv * b
        return H.coarse_dense_inv @ b
    x = np.zeros_like(b)
    if H.mode == "As":                          # nonsingular blocks: plain per-slice solve
        for rows, inv in H.coarse_inv:
            x[rows] = inv @ b[rows]
        return x
    for rows, inv in H.coarse_inv:
        if rows.size == 0:
            continue
        xs = np.zeros(rows.size)
        xs[1:] = inv @ b[rows[1:]]          # grounded at the slice's first row
        x[rows] = xs - xs.mean()            # then the slice mean removed
    return x


def _sdot(H, level, u, v):
    """per-slice dot products at a level"""
    return np.bincount(H.levels[level].slice_of_row, weights=u * v, minlength=H.nslices)


def _safe_div(a, b):
    return np.where(b != 0, a / np.where(b != 0, b, 1.0), 0.0)


def kstep(H: Hierarchy, rc, level: int):
    """K-cycle coarse correction at `level` (Notay & Vassilevski's K-cycle, the
    acceleration AGMG uses): two flexible-CG steps on A_level e = rc, per time
    slice, preconditioned by the cycle of `level`, always two steps (no branch):
        c1 = cyc(rc), v1 = A c1, rho1 = c1.v1, a1 = c1.rc, r2 = rc - (a1/rho1) v1
        c2 = cyc(r2), v2 = A c2, g = c2.v1, beta = c2.v2, a2 = c2.r2,
        rho2 = beta - g^2/rho1
        e = (a1/rho1 - g a2/(rho1 rho2)) c1 + (a2/rho2) c2
    (x/0 -> 0 on slices with a zero denominator)."""
    A = H.levels[level].A
    sl = H.levels[level].slice_of_row
    c1 = vcycle(H, rc, level)
    v1 = A @ c1
    rho1 = _sdot(H, level, c1, v1)
    a1 = _sdot(H, level, c1, rc)
    f1 = _safe_div(a1, rho1)
    r2 = rc - f1[sl] * v1
    c2 = vcycle(H, r2, level)
    g = _sdot(H, level, c2, v1)
    a2 = _sdot(H, level, c2, r2)
    v2 = A @ c2
    beta = _sdot(H, level, c2, v2)
    rho2 = beta - g * _safe_div(g, rho1)
    g2 = _safe_div(a2, rho2)
    return (f1 - g * _safe_div(g2, rho1))[sl] * c1 + g2[sl] * c2


def vcycle(H: Hierarchy, b, level: int = 0):
    """One V(1,1) cycle with damped Jacobi from a zero initial guess; in mode A the
    coarse correction into a level with <= KC_ROWS rows per slice (not the
    coarsest) is a K-cycle step (kstep) instead of a single recursive cycle."""
    if level == len(H.levels) - 1:
        return _coarse_solve(H, b)
    lv = H.levels[level]
    w = H.omega
    x = w * lv.dinv * b                                  # pre-smooth from x = 0
    r = b - lv.A @ x
    bc = np.bincount(lv.agg, weights=r, minlength=lv.nc)  # restriction P^T r
    if H.kcycle and H.kcycle[level + 1]:
        xc = kstep(H, bc, level + 1)
    else:
        xc = vcycle(H, bc, level + 1)
    x = x + xc[lv.agg]                                   # prolongation
    x = x + w * lv.dinv * (b - lv.A @ x)                 # post-smooth
    return x
