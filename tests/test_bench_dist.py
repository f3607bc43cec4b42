"""The N > 1 plumbing of bench.py on CPU (gloo, world_size 2, 127.0.0.1): every
rank's device time is reduced with MAX (the contract's max over ranks) and the
reference arm prints only on rank 0.  The GPU arm itself needs CUDA."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q.put((rank, bench.max_over_ranks(1.0 + rank * 0.5, dist)))
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert out == {0: 1.5, 1: 1.5}


@pytest.mark.slow
def test_reference_arm_rank0_only():
    """torchrun --nproc-per-node 2 bench.py --impl reference: one JSON line (rank 0)."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0 and j["cpu_baseline"]["cores"] == 1


def test_byte_model_covers_the_level0_kernel_variants():
    """bench.ByteModel (host logic): every name the level-0 AMG(A) kernels are launched under
    maps to a byte model, the residual-based variants to the smaller ones (DESIGN.md §5:
    k_down_sb<2,false> writes no x: 24n instead of 32n vector bytes; k_up_dot_res<true> reads
    neither x nor dinv: 28n instead of 36n), and ncu's 0/1 spelling of bool template
    arguments finds the same ncu_summary.json entry as the runtime's true/false."""
    sys.path.insert(0, ROOT)
    import bench

    class Ctx:
        n, m, N, K, nbar, NE = 129 * 3000, 128 * 1000, 3000, 128, 1000, 6000

        def T_nnz(self):
            return 27 * self.m, 10

        def amg_levels(self, which):
            return [(self.n, 5 * self.n, self.n // 4), (self.n // 4, 2 * self.n, 0)], 0

    st = {"outer_its": 28, "inner_T_its": 553, "inner_A_its_total": 100}
    bm = bench.ByteModel(Ctx(), st)
    n, lap = Ctx.n, 32 * Ctx.n + 16 * Ctx.N
    nc1 = Ctx.n // 4
    cases = {
        "void bbot::k_down_sb<2, true>(bbot::LapView, double const*)": 32 * n + lap,
        "void bbot::k_down_sb<2, false>(bbot::LapView, double const*)": 24 * n + lap,
        "void bbot::k_up_dot<bbot::LapView>(bbot::LapView)": 36 * n + 8 * nc1 + lap,
        "void bbot::k_up_dot_res<false>(bbot::LapView)": 36 * n + 8 * nc1 + lap,
        "void bbot::k_up_dot_res<true>(bbot::LapView)": 28 * n + 8 * nc1 + lap,
        "void bbot::k_pcg_pq<bbot::LapView>(bbot::LapView, long long)": 40 * n + lap,
    }
    for name, want in cases.items():
        assert bm._bytes(name, 0) == want, name
    g1 = (Ctx.n // 4 + 255) // 256
    assert bm._bytes("void bbot::k_down_nx<bbot::SellView>(x)", g1) == 12 * 2 * n + 24 * (n // 4)
    assert bm._bytes("void bbot::k_down<bbot::SellView>(x)", g1) == 12 * 2 * n + 32 * (n // 4)
    assert bm._bytes("void bbot::k_up_res<bbot::SellView>(x)", g1) == 12 * 2 * n + 36 * (n // 4)
    a, _ = bench.ncu_traffic("C4", "void bbot::k_up_dot_res<true>")
    b, _ = bench.ncu_traffic("C4", "void k_up_dot_res<1>")
    assert a is not None and a == b
