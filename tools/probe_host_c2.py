"""Diagnostic: host-side duration of the config-2 sweep API call (alternating vs fixed orders),
device time per step, with and without an unrelated config-3 cache alive in the process."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402

stream = torch.cuda.Stream()
L_ = fg.lib()
cfg = prep.config2(seed=1)
n, b = cfg.x.shape
A = len(cfg.alphas)
cache = fg.PowerCache(cfg.f, cfg.l, memory_budget=8 << 30)
cache.set_stream(stream.cuda_stream)
cache.prepare()
xd = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda()
xcd = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).cuda()
lo = torch.empty(A, dtype=torch.float64, device="cuda")
dl = torch.empty(A, dtype=torch.float64, device="cuda")


def run(tag, al, reps=40):
    al = [np.ascontiguousarray(a) for a in al]
    for i in range(3):
        fg._check(L_.fgfrft_mse_step_dev(cache.handle, al[i & 1].ctypes.data, A, xd.data_ptr(), xcd.data_ptr(), b,
                                         None, lo.data_ptr(), dl.data_ptr()))
    torch.cuda.synchronize()
    hs = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(reps):
        t = time.perf_counter()
        fg._check(L_.fgfrft_mse_step_dev(cache.handle, al[i & 1].ctypes.data, A, xd.data_ptr(), xcd.data_ptr(), b,
                                         None, lo.data_ptr(), dl.data_ptr()))
        hs.append((time.perf_counter() - t) * 1e3)
    e1.record(stream)
    e1.synchronize()
    hs = np.array(hs)
    print(json.dumps({"tag": tag, "dev_ms": e0.elapsed_time(e1) / reps, "host_ms_median": float(np.median(hs)),
                      "host_ms_max": float(hs.max()), "host_ms_p90": float(np.percentile(hs, 90))}), flush=True)


alt = [cfg.alphas, cfg.alphas + 1e-9]
run("alt", alt)
run("fixed", [cfg.alphas, cfg.alphas])
big = [torch.empty(1 << 30, dtype=torch.float64, device="cuda") for _ in range(2)]  # 16 GB resident
run("alt_with_16GB_alive", alt)
del big
torch.cuda.synchronize()
run("alt_again", alt)
