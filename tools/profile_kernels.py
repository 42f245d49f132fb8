"""One invocation of each hot kernel on config-2 / config-1 shapes, for ncu captures:
  ncu --set full --clock-control none --import-source on -o prof python tools/profile_kernels.py
Kernels: ozgemm_kernel (power products), combine_y_kernel (orders), rsynth_pairs_kernel (one
order, HBM-bound synthesis), rsynth_sweep_kernel (64 orders), rapply_fused_kernel (C1 fused apply),
rgemm_kernel / oz (synthesis route for one order of a large batch)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402


def main():
    cfg = prep.config2()
    n, b = cfg.x.shape
    A = len(cfg.alphas)
    cache = fg.PowerCache(cfg.f, cfg.l, memory_budget=8 << 30)
    cache.prepare()
    L = fg.lib()
    al = np.ascontiguousarray(cfg.alphas, dtype=np.float64)
    x = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda()
    xc = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).cuda()
    loss = torch.empty(A, dtype=torch.float64, device="cuda")
    dl = torch.empty(A, dtype=torch.float64, device="cuda")
    q = torch.empty((A, n, n), dtype=torch.complex128, device="cuda")
    for _ in range(2):  # warm (first call builds workspaces)
        fg._check(L.fgfrft_mse_step_dev(cache.handle, al.ctypes.data, A, x.data_ptr(), xc.data_ptr(), b, None,
                                        loss.data_ptr(), dl.data_ptr()))
    torch.cuda.synchronize()
    # the profiled calls
    fg._check(L.fgfrft_mse_step_dev(cache.handle, al.ctypes.data, A, x.data_ptr(), xc.data_ptr(), b, None,
                                    loss.data_ptr(), dl.data_ptr()))
    one = al[23:24].copy()
    fg._check(L.fgfrft_synthesize_dev(cache.handle, one.ctypes.data, 1, 0, 0, q.data_ptr()))
    fg._check(L.fgfrft_synthesize_dev(cache.handle, al.ctypes.data, A, 0, 0, q.data_ptr()))
    torch.cuda.synchronize()
    c1 = prep.config1()
    g1 = fg.PowerCache(c1.f, c1.l)
    y1 = fg.apply_series(g1, c1.alphas, c1.x)
    torch.cuda.synchronize()
    print("profile driver ok", float(loss[0]), float(np.abs(y1).max()))


if __name__ == "__main__":
    main()
