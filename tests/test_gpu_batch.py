"""Config-5 kernel (batches of small graphs, complex64) against the fp64 oracle per graph:
within 1e-4 (north star complex64 bar) for F^alpha X and dL/dalpha, all heads and graphs."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2602_20870_b200 as fg
import prep

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("kind", ["graph", "unitary"])
@pytest.mark.parametrize("graphs,n,l,heads,ch", [(24, 64, 16, 4, 64), (9, 40, 5, 2, 17), (5, 64, 16, 1, 64),
                                                 (3, 33, 30, 3, 8)])
def test_graph_batch_forward_and_gradient(graphs, n, l, heads, ch, kind):
    """kind graph: every F real (ER graph GFTs) -> real float slabs and the real kernels; unitary:
    complex F (Haar) -> complex64 slabs."""
    if kind == "graph":
        fs = np.stack([prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 100 + g))) for g in range(graphs)])
    else:
        fs = np.stack([prep.random_unitary(n, 200 + g) for g in range(graphs)])
    rng = np.random.default_rng(graphs)
    alphas = rng.uniform(0.5, 1.5, (graphs, heads))
    x = (rng.standard_normal((graphs, n, ch)) + 1j * rng.standard_normal((graphs, n, ch))).astype(np.complex64)
    gc = (rng.standard_normal((graphs, heads, n, ch)) + 1j * rng.standard_normal((graphs, heads, n, ch))) \
        .astype(np.complex64)
    batch = fg.GraphBatch(fs, l)
    a_d = torch.from_numpy(alphas).cuda()
    x_d = torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 1))).cuda()           # [G, C, n]
    g_d = torch.from_numpy(np.ascontiguousarray(gc.transpose(0, 1, 3, 2))).cuda()       # [G, H, C, n]
    y = batch.forward(a_d, x_d).cpu().numpy().transpose(0, 1, 3, 2)                    # [G, H, n, C]
    dl = batch.dlda(a_d, g_d, x_d).cpu().numpy()
    for gi in range(graphs):
        cache = O.PowerCache(fs[gi], l)
        xg = x[gi].astype(np.complex128)
        for h in range(heads):
            q = O.fgfrft_matrix(cache, alphas[gi, h])
            assert rel(y[gi, h], q @ xg) <= 1e-4
            gg = gc[gi, h].astype(np.complex128)
            s_ref = O.power_dots(cache, gg @ xg.conj().T)
            _, dc = O.sinc_coeffs(alphas[gi, h], l)
            assert abs(dl[gi, h] - float(np.dot(dc, s_ref))) <= 1e-4 * float(np.sum(np.abs(dc * s_ref)))
    batch.close()


def test_graph_batch_validation():
    fs = np.stack([np.eye(8, dtype=complex)] * 2)
    with pytest.raises(fg.ParameterError):
        fg.GraphBatch(np.stack([np.eye(70, dtype=complex)]), 4)
    b = fg.GraphBatch(fs, 4)
    a = torch.zeros((2, 5), dtype=torch.float64, device="cuda")
    x = torch.zeros((2, 3, 8), dtype=torch.complex64, device="cuda")
    with pytest.raises(fg.ParameterError):
        b.forward(a, x)  # 5 heads
    y = b.forward(a[:, :2].contiguous(), x)
    assert y.shape == (2, 2, 3, 8)
    b.close()


@pytest.mark.parametrize("graphs,heads", [(400, 4), (161, 3), (150, 1)])
def test_graph_batch_persistent_tensor_core_kernels(graphs, heads):
    """The config-5 shape (real F, n = 64, 64 channels) runs the persistent tcgen05 kernels: more
    graphs than SMs, so every CTA walks several graphs through one power / signal ring; checked on a
    sample that covers the first, the wrap-around and the last graphs of the persistent loop."""
    n, l, ch = 64, 16, 64
    fs = np.stack([prep.gft_from_shift(prep.laplacian(prep.er_graph(n, 0.1, 500 + g))) for g in range(graphs)])
    rng = np.random.default_rng(graphs + heads)
    alphas = rng.uniform(0.5, 1.5, (graphs, heads))
    x = (rng.standard_normal((graphs, n, ch)) + 1j * rng.standard_normal((graphs, n, ch))).astype(np.complex64)
    gc = (rng.standard_normal((graphs, heads, n, ch)) + 1j * rng.standard_normal((graphs, heads, n, ch))) \
        .astype(np.complex64)
    batch = fg.GraphBatch(fs, l)
    a_d = torch.from_numpy(alphas).cuda()
    x_d = torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 1))).cuda()
    g_d = torch.from_numpy(np.ascontiguousarray(gc.transpose(0, 1, 3, 2))).cuda()
    y = batch.forward(a_d, x_d).cpu().numpy().transpose(0, 1, 3, 2)
    dl = batch.dlda(a_d, g_d, x_d).cpu().numpy()
    sample = sorted({0, 1, 147, 148, 149, graphs // 2, graphs - 2, graphs - 1} & set(range(graphs)))
    for gi in sample:
        cache = O.PowerCache(fs[gi], l)
        xg = x[gi].astype(np.complex128)
        for h in range(heads):
            q = O.fgfrft_matrix(cache, alphas[gi, h])
            assert rel(y[gi, h], q @ xg) <= 1e-4, (gi, h)
            gg = gc[gi, h].astype(np.complex128)
            s_ref = O.power_dots(cache, gg @ xg.conj().T)
            _, dc = O.sinc_coeffs(alphas[gi, h], l)
            assert abs(dl[gi, h] - float(np.dot(dc, s_ref))) <= 1e-4 * float(np.sum(np.abs(dc * s_ref))), (gi, h)
    batch.close()


def test_config5_full_size_sampled():
    """BASELINE config 5 at full size (4096 ER(64, 0.1) graphs, L = 16, 4 heads per graph with orders
    in [0.5, 1.5], 64 complex64 channels -- prep.config5), on the persistent tcgen05 kernels: F^a X
    and dL/da of 24 sampled graphs (first, last, across the persistent loop) against the fp64
    oracle within 1e-4 (north-star complex64 bar)."""
    fs, orders, feats, l = prep.config5()
    graphs, n, ch = feats.shape
    heads = orders.shape[1]
    rng = np.random.default_rng(55)
    gc = (rng.standard_normal((graphs, heads, n, ch)) + 1j * rng.standard_normal((graphs, heads, n, ch))) \
        .astype(np.complex64)
    batch = fg.GraphBatch(fs, l)
    a_d = torch.from_numpy(orders).cuda()
    x_d = torch.from_numpy(np.ascontiguousarray(feats.transpose(0, 2, 1)).astype(np.complex64)).cuda()
    g_d = torch.from_numpy(np.ascontiguousarray(gc.transpose(0, 1, 3, 2))).cuda()
    y = batch.forward(a_d, x_d).cpu().numpy().transpose(0, 1, 3, 2)
    dl = batch.dlda(a_d, g_d, x_d).cpu().numpy()
    sample = sorted(set([0, 1, 147, 148, 2047, 4094, 4095] + list(rng.choice(graphs, 17, replace=False))))
    for gi in sample:
        cache = O.PowerCache(fs[gi], l)
        xg = feats[gi].astype(np.complex64).astype(np.complex128)
        for h in range(heads):
            q = O.fgfrft_matrix(cache, orders[gi, h])
            assert rel(y[gi, h], q @ xg) <= 1e-4, (gi, h)
            gg = gc[gi, h].astype(np.complex128)
            s_ref = O.power_dots(cache, gg @ xg.conj().T)
            _, dc = O.sinc_coeffs(orders[gi, h], l)
            assert abs(dl[gi, h] - float(np.dot(dc, s_ref))) <= 1e-4 * float(np.sum(np.abs(dc * s_ref))), (gi, h)
    batch.close()
