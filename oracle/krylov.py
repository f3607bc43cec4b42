"""I1, I4, I5: Krylov solvers ("applied as right preconditioners
within a FGMRES cycle" [Saad 1993]; cap 400).

fgmres   right-preconditioned flexible GMRES(restart); classical Gram-Schmidt
         with one re-orthogonalisation (CGS2); Givens rotations; stops when the
         Arnoldi residual |g_{j+1}| <= tol * scale (scale = ||(f;g;h)|| for the
         outer solve; = ||b|| for the inner T solve).  x0 = 0; after a
         restart the true residual b - A x restarts the cycle.  Used for the
         outer solve (I1, FGMRES(30), cap 400) and the inner T solve (I5,
         GMRES(10) right-preconditioned by one V-cycle, relative 1e-1, cap 50).
pcg_slices  I4: independent preconditioned CG per time slice (the K+1 blocks
         A_k), x0 = 0, stop per slice at ||r^k|| <= tol ||b^k||, cap 50;
         a converged slice is frozen.  Written batched (per-slice scalars) --
         mathematically K+1 separate PCG runs.
"""
from __future__ import annotations

import numpy as np

TINY = 1e-300


def fgmres(matvec, precond, b, scale, tol, restart, maxit):
    """Returns (x, its, converged, res_estimate)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    target = tol * scale
    r = b.copy()
    beta = np.linalg.norm(r)
    its = 0
    if beta <= target:
        return x, 0, True, beta
    res = beta
    converged = False
    while True:
        V = np.zeros((restart + 1, b.size))
        Z = np.zeros((restart, b.size))
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        V[0] = r / beta
        jj = 0
        breakdown = False
        for j in range(restart):
            Z[j] = precond(V[j])
            w = matvec(Z[j])
            its += 1
            h = V[:j + 1] @ w                      # CGS2
            w = w - V[:j + 1].T @ h
            h2 = V[:j + 1] @ w
            w = w - V[:j + 1].T @ h2
            h = h + h2
            hn = np.linalg.norm(w)
            H[:j + 1, j] = h
            H[j + 1, j] = hn
            for i in range(j):                     # previous Givens rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            res = abs(g[j + 1])
            jj = j + 1
            if hn <= TINY:
                breakdown = True
            else:
                V[j + 1] = w / hn
            if res <= target or its >= maxit or breakdown:
                break
        y = np.zeros(jj)
        for i in range(jj - 1, -1, -1):             # back substitution
            y[i] = (g[i] - H[i, i + 1:jj] @ y[i + 1:jj]) / H[i, i]
        x = x + Z[:jj].T @ y
        if res <= target or breakdown:
            converged = True
            break
        if its >= maxit:
            break
        r = b - matvec(x)
        beta = np.linalg.norm(r)
        res = beta
        if beta <= target:
            converged = True
            break
    return x, its, converged, res


def pcg_slices(matvec, precond, b, nslices, tol, maxit):
    """Per-slice PCG.  Returns (x, its_per_slice)."""
    b = np.asarray(b, dtype=np.float64)
    L = b.size // nslices

    def sdot(u, v):
        return (u * v).reshape(nslices, L).sum(1)

    def expand(a):
        return np.repeat(a, L)

    x = np.zeros_like(b)
    r = b.copy()
    bn = np.sqrt(sdot(b, b))
    active = bn > 0
    its = np.zeros(nslices, dtype=np.int64)
    if not active.any():
        return x, its
    z = precond(r)
    p = z.copy()
    rz = sdot(r, z)
    for _ in range(maxit):
        q = matvec(p)
        pq = sdot(p, q)
        bad = active & ~(pq > 0)
        active = active & ~bad
        alpha = np.where(active, rz / np.where(pq > 0, pq, 1.0), 0.0)
        x = x + expand(alpha) * p
        r = r - expand(alpha) * q
        its += active
        rn = np.sqrt(sdot(r, r))
        active = active & (rn > tol * bn)
        if not active.any():
            break
        z = precond(r)
        rz_new = sdot(r, z)
        beta = np.where(active, rz_new / np.where(rz != 0, rz, 1.0), 0.0)
        p = z + expand(beta) * p
        rz = np.where(active, rz_new, rz)
    return x, its
