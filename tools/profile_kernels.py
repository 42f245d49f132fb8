"""Launch each hot-path kernel a few times on the config-2 cache, for ncu captures.

  python tools/profile_kernels.py            # plain run (must exit 0 before ncu is used)
  ncu --set full -k regex:'synth|zgemm|power_dots' ... python tools/profile_kernels.py
Config 2's F is real, so the real-F kernels run: rsynth_pairs (one order), rsynth_sweep
(64-order sweep), rgemm<0,1,1> (Q X, 64 orders batched), rgemm<2,2,0> (Re G X^H), rdots_mma.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402  (device buffers)

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402


def main():
    cfg = prep.config2()
    n, b = cfg.x.shape
    A = len(cfg.alphas)
    cache = fg.PowerCache(cfg.f, cfg.l, memory_budget=8 << 30)
    L = fg.lib()
    al = np.ascontiguousarray(cfg.alphas)
    q = torch.empty((A, n, n), dtype=torch.complex128, device="cuda")
    x = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda()
    xc = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).cuda()
    loss = torch.empty(A, dtype=torch.float64, device="cuda")
    dl = torch.empty(A, dtype=torch.float64, device="cuda")
    one = al[23:24].copy()
    for _ in range(2):
        fg._check(L.fgfrft_synthesize_dev(cache.handle, one.ctypes.data, 1, 0, 0, q.data_ptr()))
        fg._check(L.fgfrft_synthesize_dev(cache.handle, al.ctypes.data, A, 0, 0, q.data_ptr()))
        fg._check(L.fgfrft_mse_step_dev(cache.handle, al.ctypes.data, A, x.data_ptr(), xc.data_ptr(), b, None,
                                        loss.data_ptr(), dl.data_ptr()))
    torch.cuda.synchronize()
    print("profile driver ok", float(loss[0]), float(dl[0]))


if __name__ == "__main__":
    main()
