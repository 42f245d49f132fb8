"""Diagnostic: the config-2 sweep step timed alone, then after a config-3 cache has run steps in
the same process (bench.py's order), then after that cache is closed."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402

stream = torch.cuda.Stream()


def c2(tag):
    fg.profile_enable(True)
    fg.profile_read(reset=True)
    r = bench.c2_sweep(fg, torch, stream, 0)
    prof = {k: round(v[0], 4) for k, v in fg.profile_read(reset=True).items() if v[1]}
    fg.profile_enable(False)
    print(json.dumps({tag: r["ms_per_step"], "route": r["route"], "classes_total_ms": prof}), flush=True)


c2("c2_first")
cfg = prep.config3(seed=1)
cache = fg.PowerCache(cfg.f, cfg.l, memory_budget=24 << 30)
cache.set_stream(stream.cuda_stream)
cache.prepare()
L_ = fg.lib()
xd = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda()
xcd = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).cuda()
lo = torch.empty(1, dtype=torch.float64, device="cuda")
dl = torch.empty(1, dtype=torch.float64, device="cuda")
al = np.array([0.37])
with torch.cuda.stream(stream):
    for i in range(5):
        fg._check(L_.fgfrft_mse_step_dev(cache.handle, al.ctypes.data, 1, xd.data_ptr(), xcd.data_ptr(), cfg.b, None,
                                         lo.data_ptr(), dl.data_ptr()))
torch.cuda.synchronize()
c2("c2_after_c3")
xh = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).pin_memory()
xch = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).pin_memory()
lh, dh = np.empty(1), np.empty(1)
for i in range(5):
    fg._check(L_.fgfrft_mse_step(cache.handle, al.ctypes.data, 1, xh.data_ptr(), xch.data_ptr(), cfg.b, None,
                                 lh.ctypes.data, dh.ctypes.data))
torch.cuda.synchronize()
c2("c2_after_c3_e2e")
cache.close()
c2("c2_after_close")
