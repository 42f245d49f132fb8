"""Multi-rank (row-slab sharded) path on CPU: world_size 2 over gloo.

The collective logic of paper_2602_20870_b200.dist (row plan, all_reduce of the loss and the
2L+1 partials, all_gather of Y's rows) runs for real across two processes; each rank's local
work is a CPU stand-in (`OracleRows`, test-only) computing exactly what the CUDA shard computes
for its rows. The combined result must equal the unsharded oracle. The CUDA shard kernels
themselves are checked on the GPU in test_gpu_dist.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import prep
from paper_2602_20870_b200 import dist as fgd


def test_plan_rows_covers_tiles():
    for n, w in ((1, 1), (31, 2), (64, 2), (100, 3), (8192, 8), (1000, 7), (70, 4)):
        plan = fgd.plan_rows(n, w)
        assert len(plan) == w and plan[0][0] == 0 and plan[-1][1] == n
        for (a0, a1), (b0, b1) in zip(plan, plan[1:]):
            assert a1 == b0
        for r0, r1 in plan:
            assert r0 % 32 == 0 and (r1 % 32 == 0 or r1 == n) and r0 <= r1
    assert fgd.plan_rows(8192, 8) == [(1024 * g, 1024 * (g + 1)) for g in range(8)]


class OracleRows(fgd.RankCompute):
    """CPU stand-in for CudaShard: the same per-rank partials, from the dense oracle."""

    def __init__(self, f, l, r0, r1):
        self.n, self.l, self.r0, self.r1 = f.shape[0], l, r0, r1
        self.cache = O.PowerCache(f, l)

    def mse_partial(self, alphas, x, xc_rows, want_y=False):
        n, b = x.shape
        loss, s, ys = [], [], []
        for a in alphas:
            q = O.fgfrft_matrix(self.cache, float(a))[self.r0:self.r1]
            y = q @ x
            r = y - xc_rows
            loss.append(float(np.vdot(r, r).real))
            g = np.zeros((n, b), dtype=complex)
            g[self.r0:self.r1] = 2.0 * r / (n * b)
            s.append(O.power_dots(self.cache, g @ x.conj().T))  # rows outside R contribute zero
            ys.append(y)
        return torch.tensor(loss, dtype=torch.float64), torch.from_numpy(np.array(s)), ys

    def apply_rows(self, alphas, x):
        out = [(O.fgfrft_matrix(self.cache, float(a))[self.r0:self.r1] @ x).T for a in alphas]
        return torch.from_numpy(np.ascontiguousarray(np.array(out)))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f = prep.random_unitary(70, 12)
        l = 6
        rng = np.random.default_rng(3)
        x = rng.standard_normal((70, 5)) + 1j * rng.standard_normal((70, 5))
        xc = x + 0.1 * rng.standard_normal((70, 5))
        plan = fgd.plan_rows(70, world)
        r0, r1 = plan[rank]
        sh = fgd.ShardedFGFRFT(OracleRows(f, l, r0, r1), 70, l)
        alphas = [0.37, 1.4, -0.6]
        loss, dl = sh.mse_step(alphas, x, xc[r0:r1])
        y = sh.apply(alphas, x, plan)
        q.put((rank, loss, dl, y))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_step_over_gloo_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f = prep.random_unitary(70, 12)
    cache = O.PowerCache(f, 6)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((70, 5)) + 1j * rng.standard_normal((70, 5))
    xc = x + 0.1 * rng.standard_normal((70, 5))
    for rank, loss, dl, y in res:
        for i, a in enumerate([0.37, 1.4, -0.6]):
            lr, dr, yr = O.dlda_mse(cache, a, x, xc)
            assert loss[i] == pytest.approx(lr, rel=1e-12)
            assert dl[i] == pytest.approx(dr, rel=1e-9, abs=1e-13)
            assert np.allclose(y[i], yr, rtol=0, atol=1e-12)
