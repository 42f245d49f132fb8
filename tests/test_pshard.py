"""Pair-sharded MSE step on CPU (not gpu): the library's band plan (fgfrft_pshard_plan, a host
function) and the decomposition each rank computes, with the collectives run for real over gloo
at world sizes 2 and 3.

Each rank takes Q(a) and dQ/da from the oracle (transform.hpp:111-136 restated), forms its partial
products exactly as the CUDA pair shard does (rectangles A and B of its tile band:
paper_2602_20870_b200.pshard.decomposed_partial), reduce-scatters [Y; dY] by signal-column chunks
(the signal count padded to a multiple of the world size, as the library pads it), takes the loss
and Re<Y - Xc, dY> over its columns and all-reduces them. The result must equal the unsharded
oracle (learn.hpp:88-92 form). The CUDA pair shards themselves are checked in
tests/test_gpu_pshard.py.
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
from paper_2602_20870_b200 import pshard as ps


@pytest.mark.parametrize("n", [1, 40, 64, 1000, 4096, 8192])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_band_plan_balances_pairs(n, world):
    b = ps.pair_plan(n, world)
    nt = -(-n // 32)
    npairs = nt * (nt + 1) // 2
    assert b[0] == 0 and b[-1] == nt and len(b) == world + 1
    assert all(x <= y for x, y in zip(b, b[1:]))
    counts = [ps.pairs_before(b[g + 1], nt) - ps.pairs_before(b[g], nt) for g in range(world)]
    assert sum(counts) == npairs
    if nt >= 4 * world:  # bands are whole tile rows: balanced to within one row of pairs
        assert max(counts) - npairs / world <= nt


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7])
def test_decomposition_sums_to_the_product(world):
    rng = np.random.default_rng(world)
    n, b = 200, 9
    q = rng.standard_normal((n, n))
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    tot = sum(ps.decomposed_partial(q, x, n, world, g) for g in range(world))
    assert np.allclose(tot, q @ x, rtol=1e-13, atol=1e-12)
    # each rank's partial is zero above its band
    for g in range(world):
        r0, _ = ps.rank_rows(n, world, g)
        assert not np.any(ps.decomposed_partial(q, x, n, world, g)[:r0])


def _worker(rank, world, port, qout):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, l, b = 96, 8, 10
        f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 4)))
        cache = O.PowerCache(f, l)
        rng = np.random.default_rng(3)
        x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
        xc = x + 0.1 * rng.standard_normal((n, b))
        out = []
        bpad = -(-b // world) * world
        cb = bpad // world
        for a in (0.37, -1.2):
            q = O.fgfrft_matrix(cache, a)
            dq = O.fgfrft_grad(cache, a)
            blocks = []
            for m in (q, dq):
                part = np.zeros((n, bpad), dtype=complex)
                part[:, :b] = ps.decomposed_partial(m, x, n, world, rank)
                # column-major n x bpad -> contiguous column chunks: the reduce-scatter's layout
                blocks.append(torch.from_numpy(np.ascontiguousarray(part.T)).view(torch.float64).reshape(-1))
            recv = []
            for t in blocks:
                r = torch.empty(t.numel() // world, dtype=torch.float64)
                dist.reduce_scatter_tensor(r, t)
                recv.append(r.view(torch.complex128).reshape(cb, n).numpy().T)
            j0 = rank * cb
            valid = max(0, min(cb, b - j0))
            y, dy = recv[0][:, :valid], recv[1][:, :valid]
            res = y - xc[:, j0:j0 + valid]
            s = torch.tensor([np.vdot(res, res).real, np.sum(np.conj(res) * dy).real], dtype=torch.float64)
            dist.all_reduce(s)
            out.append((float(s[0]) / (n * b), 2.0 * float(s[1]) / (n * b)))
        qout.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_pair_sharded_mse_step_over_gloo(world):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    qout = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, qout)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(qout.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, l, b = 96, 8, 10
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 4)))
    cache = O.PowerCache(f, l)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    for i, a in enumerate((0.37, -1.2)):
        lr, dr, _ = O.dlda_mse(cache, a, x, xc)
        for r in range(world):
            loss, dl = res[r][i]
            assert abs(loss - lr) <= 1e-12 * lr
            assert abs(dl - dr) <= 1e-11 * max(1.0, abs(dr))
