"""Small instances of every kernel family of libfgfrft_b200.so, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

  compute-sanitizer --tool racecheck python tools/sanitize_probe.py

Complex F (DMMA GEMMs, exact synthesis, power dots), real F (doubling build, packed step:
psynth + Ozaki slicing + tcgen05 GEMM + fused loss; node-interpolated sweep; power route with
the DMMA combination; fused small-batch apply), the INT8 DGEMM with 7 digits, pair shards, graph
batches (config-5 kernels), the denoise engine, the spectrum / exact operator / cascade, and the
cache file round trip. Results are checked loosely (the parity tests are elsewhere); the point is
the sanitizer's verdict on every launch.
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402
from paper_2602_20870_b200 import pshard as ps  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    # complex F: DMMA cache build, exact synthesis, DMMA apply, dL/da, MSE step
    fz = prep.random_unitary(96, 3)
    cz = fg.PowerCache(fz, 6)
    x = rng.standard_normal((96, 5)) + 1j * rng.standard_normal((96, 5))
    fg.synthesize(cz, [0.3, -1.1])
    fg.apply_series(cz, [0.3], x, inverse=True)
    fg.mse_step(cz, [0.3, 0.7], x, x + 0.1)
    # real F: doubling build, packed step, node sweep, power route, fused apply
    fr = prep.gft_from_shift(prep.laplacian(prep.grid_graph(16, 32)))
    cr = fg.PowerCache(fr, 8, memory_budget=1 << 30)
    xr = rng.standard_normal((512, 40)) + 1j * rng.standard_normal((512, 40))
    fg.mse_step(cr, [0.41], xr, xr + 0.1, want_y=True)            # packed route
    fg.apply_series(cr, [0.2, 0.9], xr)                            # packed apply, 2 orders
    fg.mse_step(cr, list(np.linspace(0.0, 2.0, 16)), xr, xr + 0.1)  # node route
    fg.mse_step(cr, list(np.linspace(0.5, 0.51, 16)), xr, xr + 0.1)  # power route (narrow)
    fg.apply_series(cr, [0.6], xr[:, :4])                          # fused small-batch apply
    fg.synthesize(cr, [0.25])
    # INT8 DGEMM, 7 digits
    a = torch.randn(256, 256, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    fg._check(fg.lib().fgfrft_dgemm_int8_dev(0, 0, 256, 256, 256, a.data_ptr(), 256, a.data_ptr(), 256,
                                             c.data_ptr(), 256, 7, None))
    # pair shards (local, world 2)
    xd = torch.from_numpy(np.ascontiguousarray(xr.T)).cuda()
    for g in range(2):
        sh = ps.PairShard(fr, 8, world=2, rank=g)
        sh.partial([0.3], xd)
        sh.close()
    # graph batches (config-5 kernels), small
    fs = np.stack([prep.gft_from_shift(prep.laplacian(prep.er_graph(16, 0.3, s))) for s in range(8)])
    batch = fg.GraphBatch(fs, 4)
    al = torch.rand(8, 4, dtype=torch.float64, device="cuda")
    xb = torch.randn(8, 16, 16, dtype=torch.complex64, device="cuda")
    batch.forward(al, xb)
    batch.dlda(al, torch.randn(8, 4, 16, 16, dtype=torch.complex64, device="cuda"), xb)
    # denoise (fast engine) and the spectrum / exact operator / cascade
    dn = fg.DenoiseProblem(cr, xr.real[:, :8], xr.real[:, :8] + 0.1)
    dn.eval(0.5, np.ones(512))
    sp = fg.eigendecompose_unitary(fz)
    fg.exact_gfrft(sp, 0.3)
    cas = fg.CascadeProblem(fz, depth=2, target_order=1.2, truncation=6, eig=sp)
    cas.eval([0.5, 0.6])
    # cache file round trip (device checksum)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "c.bin")
        cz.save(p)
        fg.PowerCache.load(p)
    torch.cuda.synchronize()
    print("sanitize probe ok, launches", fg.launch_count())


if __name__ == "__main__":
    main()
