"""The exchange plan of the time-slab decomposition (comm.cuh) across real
processes on CPU: world_size 2 and 3 over gloo (127.0.0.1).  Every rank asks libbbot.so for
its owned slices (bbot_slab_plan -- the rule the NCCL and virtual backends use, no GPU
needed), then runs the halo exchange with the NCCL backend's pairing (send the first owned
slice left / receive slice lo-1; send the last owned slice right / receive slice hi) and the
allgather as one broadcast per owner -- on layouts with unequal slice lengths (the AMG(T)
coarse levels) and S = K or K+1 slices.  Checks: the slices are owned exactly once, every
rank owns >= 1 slice when P <= nb (the AMG(T) time blocks, A42), slab boundaries fall on
block boundaries, the halos hold the neighbours' values, the allgather reproduces the global
vector on every rank."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layouts(K):
    rng = np.random.default_rng(K)
    out = []
    for S in (K, K + 1):
        lens = rng.integers(1, 7, size=S)
        out.append(np.r_[0, np.cumsum(lens)])
    return out


def _worker(rank, world, port, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_2209_00315_b200 as pb
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = []
    try:
        _exchange(rank, world, K, dist, torch, pb, res)
    except Exception as ex:                 # report instead of leaving the parent waiting
        q.put((rank, repr(ex)))
        dist.destroy_process_group()
        return
    dist.destroy_process_group()
    q.put((rank, res))


def _exchange(rank, world, K, dist, torch, pb, res):
    if True:
        for off in _layouts(K):
            S = len(off) - 1
            glob = np.arange(off[-1], dtype=np.float64) * 1.5 + 7.0
            plan = [pb.slab_plan(K + 1, world, r, S) for r in range(world)]
            lo, hi = plan[rank]
            buf = torch.full((off[-1],), float("nan"), dtype=torch.float64)
            buf[off[lo]:off[hi]] = torch.from_numpy(glob[off[lo]:off[hi]])
            reqs = []
            if rank > 0 and lo > 0 and hi > lo:
                reqs.append(dist.isend(buf[off[lo]:off[lo + 1]].clone(), rank - 1))
                reqs.append(dist.irecv(buf[off[lo - 1]:off[lo]], rank - 1))
            nlo, nhi = plan[rank + 1] if rank + 1 < world else (S, S)
            if rank + 1 < world and hi < S and nhi > nlo:
                reqs.append(dist.isend(buf[off[hi - 1]:off[hi]].clone(), rank + 1))
                reqs.append(dist.irecv(buf[off[hi]:off[hi + 1]], rank + 1))
            for r_ in reqs:
                r_.wait()
            ok_halo = True
            if lo > 0:
                ok_halo &= bool(np.array_equal(buf[off[lo - 1]:off[lo]].numpy(), glob[off[lo - 1]:off[lo]]))
            if hi < S:
                ok_halo &= bool(np.array_equal(buf[off[hi]:off[hi + 1]].numpy(), glob[off[hi]:off[hi + 1]]))
            for qr in range(world):                    # allgather: one broadcast per owner
                a, b = plan[qr]
                if b > a:
                    part = buf[off[a]:off[b]].clone()
                    dist.broadcast(part, src=qr)
                    buf[off[a]:off[b]] = part
            res.append((S, plan, ok_halo, bool(np.array_equal(buf.numpy(), glob))))


@pytest.mark.parametrize("world,K", [(2, 4), (3, 8), (3, 5), (3, 32)])
def test_slab_exchange_gloo(world, K):
    sys.path.insert(0, ROOT)
    import paper_2209_00315_b200 as pb
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, K, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in out.items():
        assert not isinstance(res, str), res
        for S, plan, ok_halo, ok_all in res:
            owned = [s for a, b in plan for s in range(a, b)]
            assert owned == list(range(S))                 # every slice exactly once, in order
            assert all(b > a for a, b in plan)             # P <= nb: nobody idle
            B, nb = pb.time_blocks(K)
            assert all(a % B == 0 for a, _ in plan)        # slabs are unions of time blocks
            assert ok_halo and ok_all, (rank, S)


@pytest.mark.parametrize("K", [1, 2, 4, 5, 8, 12, 32, 64, 128, 256])
def test_time_blocks_rule_matches_oracle(K):
    """A42: the GPU library's time blocks (bbot_time_blocks) and the oracle's
    (oracle/amg.py::time_blocks) are the same partition of the K density slices, and for
    P = 1..min(8, nb) every slab boundary of bbot_slab_plan is a block boundary."""
    sys.path.insert(0, ROOT)
    import paper_2209_00315_b200 as pb
    from oracle.amg import time_blocks
    B, nb = pb.time_blocks(K)
    blk = time_blocks(K)
    assert blk.max() + 1 == nb and np.array_equal(blk, np.minimum(np.arange(K) // B, nb - 1))
    for P in range(1, min(8, nb) + 1):
        plan = [pb.slab_plan(K + 1, P, r, K) for r in range(P)]
        assert [s for a, b in plan for s in range(a, b)] == list(range(K))
        assert all(b > a for a, b in plan)
        starts = {0} | {int(k) for k in np.nonzero(np.diff(blk))[0] + 1}
        assert all(a in starts for a, _ in plan)
