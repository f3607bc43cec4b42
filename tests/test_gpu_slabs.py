"""Time-slab decomposition on ONE GPU: P contexts of this
process, each owning a slab of the time slices, exchange halos and per-slice reduction
totals by device-to-device copies (the virtual backend of the exchange layer; the NCCL
backend issues the same exchanges between processes).  Each rank's calls run in its own
host thread, concurrently.  The decomposed J_P, BB apply and whole Newton solve must equal
the single-GPU results BITWISE (every reduction is an in-order sum of per-slice totals whose
block partition depends only on the slice length) -- on every rank."""
import itertools
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle.ops import Discretisation                # noqa: E402
from synthetic import initial_state, make_problem, random_state   # noqa: E402

_group = itertools.count(1000)


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2209_00315_b200 as pb
    return pb


def _ranks(pb, p, P, opts=None):
    import torch
    grp = next(_group)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, stream=st.cuda_stream, opts=opts) for st in streams]
    for r, c in enumerate(ctxs):
        c.set_dist_virtual(r, P, grp)
    return ctxs, streams


def _parallel(ctxs, fn):
    out = [None] * len(ctxs)
    err = []

    def run(r):
        try:
            out[r] = fn(r, ctxs[r])
        except Exception as ex:                     # surfaced after join
            err.append((r, ex))
    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "virtual ranks did not finish"
    assert not err, err
    return out


def _state(name, kind, mu):
    p = make_problem(name)
    if kind == "init":
        phi, rho, s = initial_state(p, mu)
    else:
        phi, rho, s = random_state(p, seed=5, mu=mu)
    return p, phi, rho, s


@pytest.mark.parametrize("P", [2, 3])
def test_slab_jp_and_bb_apply_bitwise(P):
    """J_P x (4.17) and one BB apply (4.18)-(4.20) with the decomposed T-solve and A_k solves:
    every rank's result (allgathered) equals the single-GPU one bitwise; inner T counts equal."""
    pb = _gpu()
    p, phi, rho, s = _state("C1", "random", 1e-2)
    d = Discretisation(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    x = np.random.default_rng(11).standard_normal(p.n + p.m)
    r = np.random.default_rng(9).standard_normal(p.n + p.m)
    r[p.n:] = d.P(r[p.n:])
    ref = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ref.set_state(phi, rho, s, 1e-2)
    ref.assemble()
    y1 = ref.jp_matvec(x)
    z1, itT, _ = ref.bb_apply(r)
    ctxs, _ = _ranks(pb, p, P)

    def work(rank, c):
        c.set_state(phi, rho, s, 1e-2)
        c.assemble()
        return c.jp_matvec(x), c.bb_apply(r)
    for rank, (y, (z, t, _)) in enumerate(_parallel(ctxs, work)):
        assert np.array_equal(y, y1), (rank, np.abs(y - y1).max())
        assert t == itT, (rank, t, itT)
        assert np.array_equal(z, z1), (rank, np.abs(z - z1).max())


@pytest.mark.parametrize("name,kind,mu,P", [("C1", "init", 1.0, 3), ("C1", "random", 1e-2, 2),
                                            ("T2", "random", 5e-2, 4), ("C2", "init", 1.0, 4),
                                            ("C2", "init", 1.0, 3), ("T0", "init", 1.0, 2)])
def test_slab_newton_solve_bitwise(name, kind, mu, P):
    """The whole Newton solve (FGMRES on (4.17) with the BB preconditioner, recovery a6) on P
    virtual ranks: the direction on every rank equals the single-GPU direction bitwise, with the
    same outer and inner T counts; the replicated Newton update then keeps every rank's state
    identical to the single-GPU one."""
    pb = _gpu()
    p, phi, rho, s = _state(name, kind, mu)
    ref = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    ref.set_state(phi, rho, s, mu)
    ref.assemble()
    dphi, drho, ds, st = ref.solve()
    a1 = ref.newton_update(0.95)
    s1 = ref.get_state()
    ctxs, _ = _ranks(pb, p, P)

    def work(rank, c):
        c.set_state(phi, rho, s, mu)
        c.assemble()
        out = c.solve()
        a = c.newton_update(0.95)
        return out, a, c.get_state(), c.slab()
    res = _parallel(ctxs, work)
    slabs = []
    for rank, ((gphi, grho, gds, gst), a, state, slab) in enumerate(res):
        slabs.append(slab)
        for u, v in ((gphi, dphi), (grho, drho), (gds, ds)):
            assert np.array_equal(u, v), (rank, np.abs(u - v).max())
        assert gst["outer_its"] == st["outer_its"] and gst["inner_T_its"] == st["inner_T_its"], (gst, st)
        assert gst["converged"] == st["converged"]
        assert a == a1
        for u, v in zip(state[:3], s1[:3]):
            assert np.array_equal(u, v)
    B, nb = pb.time_blocks(p.K)        # slabs: whole AMG(T) time blocks (A42)
    starts = [B * (r * nb // P) for r in range(P)] + [p.K + 1]
    assert slabs == [(starts[r], starts[r + 1]) for r in range(P)]


def test_slab_newton_solve_bitwise_harmonic():
    """The decomposed solve with the harmonic reconstruction (NEXT f4: the W block couples
    neighbouring density slices in J_P and the recovery -- two-sided halos): bitwise equal to
    one GPU on P = 3 virtual ranks."""
    pb = _gpu()
    p, phi, rho, s = _state("C1", "random", 1e-2)
    opts = pb.default_solver_opts(recon=1)
    ref = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f, opts=opts)
    ref.set_state(phi, rho, s, 1e-2)
    ref.assemble()
    dphi, drho, ds, st = ref.solve()
    ctxs, _ = _ranks(pb, p, 3, opts=pb.default_solver_opts(recon=1))

    def work(rank, c):
        c.set_state(phi, rho, s, 1e-2)
        c.assemble()
        return c.solve()
    for rank, (gphi, grho, gds, gst) in enumerate(_parallel(ctxs, work)):
        for u, v in ((gphi, dphi), (grho, drho), (gds, ds)):
            assert np.array_equal(u, v), (rank, np.abs(u - v).max())
        assert gst["outer_its"] == st["outer_its"]


def test_slab_rejects_too_many_ranks():
    """P <= nb (every rank owns >= 1 AMG(T) time block, A42): T0 (K = 2, two single-slice
    blocks) cannot take P = 3."""
    pb = _gpu()
    p = make_problem("T0")
    c = pb.Context(p.verts, p.tris, p.K, p.rho_in, p.rho_f)
    with pytest.raises(pb.BbotError):
        c.set_dist_virtual(0, 3, 99)
