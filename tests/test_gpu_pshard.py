"""GPU parity of the pair shards (csrc/capi_pshard.cu) on one B200.

* World G > 1 is emulated sequentially in one process: G local shards (no communicator; no kernel
  waits on another rank), their partial products summed on the host must equal the full
  Y = F^a X and dY = dF^a/da X of the oracle (transform.hpp:111-148), and the loss / dL/da
  formed from the sums must equal the oracle's (learn.hpp:88-92 form).
* The collective path runs for real through the library's NCCL communicator at world 1
  (ncclCommInitRank on the one GPU): reduce-scatter + all-reduce + broadcast calls included.
"""
import numpy as np
import pytest

import oracle as O
import paper_2602_20870_b200 as fg
import prep
from paper_2602_20870_b200 import pshard as ps

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _graph_f(n, seed):
    rng = prep.Rng(seed)
    pts = rng.uniforms(2 * n).reshape(n, 2)
    return prep.gft_from_shift(prep.laplacian(prep.knn_graph(pts, 8)))


@pytest.fixture(scope="module")
def problem():
    import torch
    n, l, b = 640, 12, 40
    f = _graph_f(n, 19)
    rng = np.random.default_rng(8)
    x = rng.standard_normal((n, b)) + 1j * rng.standard_normal((n, b))
    xc = x + 0.1 * rng.standard_normal((n, b))
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    xcd = torch.from_numpy(np.ascontiguousarray(xc.T)).cuda()
    return f, l, x, xc, xd, xcd, O.PowerCache(f, l)


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_local_shards_partials_sum_to_the_full_products(problem, world):
    f, l, x, xc, xd, xcd, o = problem
    n, b = x.shape
    alphas = [0.37, -0.8]
    tot = None
    for g in range(world):
        sh = ps.PairShard(f, l, world=world, rank=g)
        part = sh.partial(alphas, xd, with_dq=True).cpu().numpy()  # [2A, b, n]
        r0 = sh.info()["row_begin"]
        assert not np.any(part[:, :, :r0])  # nothing above the rank's band
        tot = part if tot is None else tot + part
        sh.close()
    for i, a in enumerate(alphas):
        y = tot[i].T
        dy = tot[len(alphas) + i].T
        assert rel(y, O.fgfrft_matrix(o, a) @ x) <= 1e-10
        assert rel(dy, O.fgfrft_grad(o, a) @ x) <= 1e-10
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        res = y - xc
        assert abs(np.vdot(res, res).real / (n * b) - lr) <= 1e-10 * lr
        assert abs(2.0 * np.sum(np.conj(res) * dy).real / (n * b) - dr) <= 1e-9 * max(1.0, abs(dr))


def test_shard_bands_store_a_share_of_the_cache(problem):
    f, l, *_ = problem
    n = f.shape[0]
    nt = -(-n // 32)
    sizes = []
    for g in range(4):
        sh = ps.PairShard(f, l, world=4, rank=g)
        info = sh.info()
        sizes.append(info["pair_end"] - info["pair_begin"])
        assert info["device_bytes"] >= (info["pair_end"] - info["pair_begin"]) * l * 2 * 5120
        sh.close()
    assert sum(sizes) == nt * (nt + 1) // 2
    assert max(sizes) - min(sizes) <= nt


def test_nccl_world1_step_apply_and_host_step(problem):
    f, l, x, xc, xd, xcd, o = problem
    comm = ps.Comm(ps.Comm.unique_id(), 1, 0, 0)
    sh = ps.PairShard(f, l, comm=comm)
    alphas = [0.61, 1.4]
    lo, dl = sh.mse_step_dev(alphas, xd, xcd)
    lo, dl = lo.cpu().numpy(), dl.cpu().numpy()
    lh, dh = sh.mse_step(alphas, x, xc)
    for i, a in enumerate(alphas):
        lr, dr, _ = O.dlda_mse(o, a, x, xc)
        assert abs(lo[i] - lr) <= 1e-10 * lr and abs(lh[i] - lr) <= 1e-10 * lr
        assert abs(dl[i] - dr) <= 1e-9 * max(1.0, abs(dr)) and abs(dh[i] - dr) <= 1e-9 * max(1.0, abs(dr))
    y = sh.apply_dev([0.3, 0.9, -0.2, 1.1], xd).cpu().numpy()
    yi = sh.apply_dev([0.3], xd, inverse=True).cpu().numpy()
    for i, a in enumerate([0.3, 0.9, -0.2, 1.1]):
        assert rel(y[i].T, O.fgfrft_matrix(o, a) @ x) <= 1e-10
    assert rel(yi[0].T, O.fgfrft_matrix(o, 0.3).conj().T @ x) <= 1e-10
    sh.close()
    comm.close()


def test_pair_shard_errors(problem):
    f, l, *_ = problem
    n = f.shape[0]
    with pytest.raises(fg.CapacityError):
        ps.PairShard(f, l, memory_budget=1 << 20, world=2, rank=0)
    with pytest.raises(fg.ParameterError):
        ps.PairShard(prep.random_unitary(64, 1), 4, world=1, rank=0)  # complex F: row shards instead
    with pytest.raises(fg.ParameterError):
        ps.PairShard(f, l, world=2, rank=2)
    sh = ps.PairShard(f, l, world=2, rank=1)
    import torch
    xd = torch.zeros((4, n), dtype=torch.complex128, device="cuda")
    with pytest.raises(fg.ParameterError):  # a local shard of a world > 1 has no communicator
        sh.mse_step_dev([0.5], xd, xd)
    sh.close()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_reduce_scatter_epilogue(problem, world):
    """The fused reduce-scatter's data path, emulated on one GPU: every "rank" GEMM stores its tiles
    into the receive slot it owns in each owner's buffer (here all local memory; on a node, peer
    buffers mapped over NVLink); the owners' slot sums are the column chunks of the full products."""
    import torch
    f, l, x, xc, xd, xcd, o = problem
    n, b = x.shape
    cb = -(-b // world)
    rows = 2  # [Y; dY] of one order
    slot = rows * cb * n  # complex elements of one source rank's slot
    rbs = [torch.zeros(world * slot, dtype=torch.complex128, device="cuda") for _ in range(world)]
    for g in range(world):
        sh = ps.PairShard(f, l, world=world, rank=g)
        sh.partial_scatter([0.37], xd, [rb.data_ptr() + g * slot * 16 for rb in rbs])
        sh.close()
    torch.cuda.synchronize()
    y = np.zeros((n, world * cb), dtype=complex)
    dy = np.zeros_like(y)
    for h in range(world):
        tot = rbs[h].view(world, rows, cb, n).sum(dim=0).cpu().numpy()  # [rows][col][row]
        y[:, h * cb:(h + 1) * cb] = tot[0].T
        dy[:, h * cb:(h + 1) * cb] = tot[1].T
    assert not np.any(y[:, b:]) and not np.any(dy[:, b:])  # padding columns never written
    assert rel(y[:, :b], O.fgfrft_matrix(o, 0.37) @ x) <= 1e-10
    assert rel(dy[:, :b], O.fgfrft_grad(o, 0.37) @ x) <= 1e-10
