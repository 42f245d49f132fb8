"""Row-slab shard kernels on one GPU: two shards of the same F (ranks emulated SEQUENTIALLY in
one process -- no kernel waits on another) must combine to the unsharded results: summed
partials = full loss / s_k, concatenated rows = full F^a and F^a X."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2602_20870_b200 as fg
import prep
from paper_2602_20870_b200 import dist as fgd

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("kind", ["haar", "graph"])
@pytest.mark.parametrize("n,l,world,n_alpha,b", [(100, 7, 2, 3, 9), (256, 32, 3, 5, 9), (64, 4, 2, 1, 9),
                                                 (96, 6, 4, 2, 9), (512, 8, 2, 2, 40)])
def test_shards_combine_to_unsharded(n, l, world, n_alpha, b, kind):
    """kind = graph: a real orthogonal F (graph GFT) -> real panels and real shard kernels; with
    n >= 512 and 2b >= 64 the shard GEMMs run on the INT8 engine."""
    if kind == "haar":
        f = prep.random_unitary(n, 40 + n)
    else:
        f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 40 + n)))
    o = O.PowerCache(f, l)
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    alphas = list(np.linspace(-0.8, 1.9, n_alpha))
    plan = fgd.plan_rows(n, world)
    loss = np.zeros(n_alpha)
    s = np.zeros((n_alpha, 2 * l + 1))
    dl_direct = np.zeros(n_alpha)  # fgfrft_shard_mse_dlda_partial_dev (dQ rows for <= 2 orders)
    y_rows, q_rows = [], []
    for r0, r1 in plan:
        if r1 == r0:
            continue
        sh = fgd.CudaShard(f, l, r0, r1)
        lp, sp, _ = sh.mse_partial(alphas, x, xc[r0:r1])
        loss += lp.cpu().numpy()
        s += sp.cpu().numpy()
        packed = sh.mse_dlda_partial(alphas, x, xc[r0:r1]).cpu().numpy()
        assert np.allclose(packed[:n_alpha], lp.cpu().numpy(), rtol=1e-13, atol=0)
        dl_direct += packed[n_alpha:]
        y_rows.append(sh.apply_rows(alphas, x).cpu().numpy().transpose(0, 2, 1))
        q_rows.append(sh.synthesize_rows(alphas).cpu().numpy().transpose(0, 2, 1))
        sh.close()
    y = np.concatenate(y_rows, axis=1)
    q = np.concatenate(q_rows, axis=1)
    for i, a in enumerate(alphas):
        qr = O.fgfrft_matrix(o, a)
        assert rel(q[i], qr) <= 1e-12
        assert rel(y[i], qr @ x) <= 1e-12
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert loss[i] / (n * b) == pytest.approx(lr, rel=1e-12)
        _, dc = O.sinc_coeffs(a, l)
        s_ref = O.power_dots(o, (2.0 * (qr @ x - xc) / (n * b)) @ x.conj().T)
        assert np.abs(s[i] - s_ref).max() <= 1e-10 * np.abs(s_ref).sum()
        assert abs(float(np.dot(dc, s[i])) - dr) <= 1e-10 * np.sum(np.abs(dc * s_ref))
        assert abs(dl_direct[i] - dr) <= 1e-10 * np.sum(np.abs(dc * s_ref))


def test_shard_validation():
    f = prep.random_unitary(64, 1)
    with pytest.raises(fg.ParameterError):
        fgd.CudaShard(f, 3, 10, 40)      # not tile aligned
    with pytest.raises(fg.CapacityError):
        fgd.CudaShard(f, 3, 0, 32, memory_budget=1024)
    sh = fgd.CudaShard(f, 3, 32, 64)
    h = sh._h
    with pytest.raises(fg.ParameterError):  # a shard is not a full cache handle
        fg._check(fg.lib().fgfrft_cache_power(h, 1, np.zeros((64, 64), complex).ctypes.data))
    sh.close()


def test_sharded_step_wrapper_single_rank():
    """ShardedFGFRFT with world 1 (no process group): same numbers as the unsharded mse_step."""
    cfg = prep.config1()
    sh = fgd.CudaShard(cfg.f, cfg.l, 0, cfg.n)
    w = fgd.ShardedFGFRFT(sh, cfg.n, cfg.l)
    xc = cfg.x + 0.05
    loss, dl = w.mse_step(cfg.alphas, cfg.x, xc)
    g = fg.PowerCache(cfg.f, cfg.l)
    g.set_engine(fg.ENGINE_DMMA)  # the shards run the DMMA kernels: compare like with like
    l2, d2, _ = fg.mse_step(g, cfg.alphas, cfg.x, xc)
    assert loss[0] == pytest.approx(l2[0], rel=1e-12)
    assert dl[0] == pytest.approx(d2[0], rel=1e-9, abs=1e-14)
    y = w.apply(cfg.alphas, cfg.x)
    assert rel(y[0], fg.apply_series(g, cfg.alphas, cfg.x)[0]) <= 1e-13


@pytest.mark.parametrize("kind,n,b,world", [("graph", 512, 40, 2), ("graph", 300, 9, 3), ("haar", 200, 9, 2),
                                            ("graph", 1024, 64, 4)])
def test_fused_gather_epilogue_writes_every_buffer(kind, n, b, world):
    """fgfrft_shard_apply_gather_dev with the other 'ranks' buffers as peers (here local device
    buffers standing in for NVLink mappings): after every shard's call, every buffer holds the
    full Y. graph + n >= 512 + 2b >= 64 exercises the INT8 epilogue path, the rest the DMMA GEMM
    + P2P push kernel."""
    import torch
    f = prep.random_unitary(n, 5) if kind == "haar" else prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.05, 6)))
    l = 6
    o = O.PowerCache(f, l)
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    alphas = [0.3, 1.7, -0.45]
    bufs = [torch.full((len(alphas), b, n), float("nan"), dtype=torch.complex128, device="cuda") for _ in range(world)]
    for rank, (r0, r1) in enumerate(fgd.plan_rows(n, world)):
        if r1 == r0:
            continue
        sh = fgd.CudaShard(f, l, r0, r1)
        peers = [bufs[q].data_ptr() for q in range(world) if q != rank]
        sh.apply_gather(alphas, x, bufs[rank], peers)
        torch.cuda.synchronize()
        sh.close()
    for q in range(world):
        y = bufs[q].cpu().numpy().transpose(0, 2, 1)
        for i, a in enumerate(alphas):
            assert rel(y[i], O.fgfrft_matrix(o, a) @ x) <= 1e-12


def test_apply_fused_single_rank():
    cfg = prep.config1()
    sh = fgd.CudaShard(cfg.f, cfg.l, 0, cfg.n)
    w = fgd.ShardedFGFRFT(sh, cfg.n, cfg.l)
    y = w.apply_fused(cfg.alphas, cfg.x).cpu().numpy().transpose(0, 2, 1)
    assert rel(y[0], w.apply(cfg.alphas, cfg.x)[0]) <= 1e-14


def _ipc_worker(rank, world, port, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2602_20870_b200.dist as fgd_
    import prep as prep_
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # host collectives: handles, barrier
    try:
        n, l, b = 512, 6, 40
        f = prep_.gft_from_shift(prep_.laplacian(prep_.er_graph(n, 0.05, 6)))
        r0, r1 = fgd_.plan_rows(n, world)[rank]
        sh = fgd_.CudaShard(f, l, r0, r1, device=0)
        w = fgd_.ShardedFGFRFT(sh, n, l)
        rng = np.random.default_rng(n)
        x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
        y = w.apply_fused([0.3, 1.7], x).cpu().numpy()
        y2 = w.apply_fused([0.9, -0.4], x)  # cached IPC mappings, different orders
        y3 = w.apply_fused([0.3, 1.7], x)   # the first result is not aliased by later calls
        q.put((rank, y, y2.cpu().numpy(), y3.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_apply_fused_two_processes_ipc():
    """Two ranks (processes) on the one GPU, gloo for the host collectives: the fused-gather apply
    exchanges CUDA IPC handles, each rank's GEMM epilogue writes its rows into both Y buffers, and
    both ranks end with the full Y. No kernel waits on the other rank (host barrier only)."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, y, y2, y3 = q.get(timeout=300)
        out[rank] = ((y, [0.3, 1.7]), (y2, [0.9, -0.4]), (y3, [0.3, 1.7]))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, l = 512, 6
    f = prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.05, 6)))
    o = O.PowerCache(f, l)
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, 40)) + 1j * rng.standard_normal((n, 40))
    for rank in (0, 1):
        for y, alphas in out[rank]:
            yy = y.transpose(0, 2, 1)
            for i, a in enumerate(alphas):
                assert rel(yy[i], O.fgfrft_matrix(o, a) @ x) <= 1e-12
