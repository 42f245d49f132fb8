"""Regression probe: config-3 device / e2e steps and the config-2 sweep, each with the library's
per-class profile (diagnostic tool, not a bench line).  python tools/probe_regress.py c3|c2"""
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


def timed(stream, fn, reps=10, warm=3):
    with torch.cuda.stream(stream):
        for i in range(warm):
            fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(stream)
    with torch.cuda.stream(stream):
        for i in range(reps):
            fn(i)
    e1.record(stream)
    e1.synchronize()
    wall = (time.perf_counter() - t) / reps * 1e3
    dev = e0.elapsed_time(e1) / reps
    fg.profile_enable(True)
    fg.profile_read(reset=True)
    with torch.cuda.stream(stream):
        for i in range(reps):
            fn(i)
    torch.cuda.synchronize()
    tr = fg.profile_trace() if os.environ.get("PROBE_TRACE") else []
    prof = {k: round(v[0] / reps, 4) for k, v in fg.profile_read(reset=True).items() if v[1]}
    fg.profile_enable(False)
    out = {"dev_ms": dev, "wall_ms": wall, "classes": prof}
    if tr:  # the last step's launches: (class, start, end) in ms from the step's first launch
        per = len(tr) // reps
        t0 = tr[-per][1]
        out["trace"] = [(c, round(a - t0, 4), round(b - t0, 4)) for c, a, b in tr[-per:]]
    return out


def main():
    which = sys.argv[1]
    L_ = fg.lib()
    stream = torch.cuda.Stream()
    if which == "c3":
        cfg = prep.config3()
        n, b = cfg.n, cfg.b
        cache = fg.PowerCache(cfg.f, cfg.l, memory_budget=200 << 30)
        cache.set_stream(stream.cuda_stream)
        al = [np.array([0.37]), np.array([0.63])]
        xh = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).pin_memory()
        xch = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).pin_memory()
        xd, xcd = xh.cuda(), xch.cuda()
        lo = torch.empty(1, dtype=torch.float64, device="cuda")
        dl = torch.empty(1, dtype=torch.float64, device="cuda")
        lh, dh = np.empty(1), np.empty(1)

        def dev(i):
            fg._check(L_.fgfrft_mse_step_dev(cache.handle, al[i & 1].ctypes.data, 1, xd.data_ptr(), xcd.data_ptr(), b,
                                             None, lo.data_ptr(), dl.data_ptr()))

        def e2e(i):
            fg._check(L_.fgfrft_mse_step(cache.handle, al[i & 1].ctypes.data, 1, xh.data_ptr(), xch.data_ptr(), b,
                                         None, lh.ctypes.data, dh.ctypes.data))
        for ds in os.environ.get("PROBE_DS", "1,0").split(","):
            os.environ["FGFRFT_DSYNTH"] = ds
            print(json.dumps({"c3": "dev", "dsynth": ds, **timed(stream, dev), "route": cache.route_info()[0]}), flush=True)
            print(json.dumps({"c3": "e2e", "dsynth": ds, **timed(stream, e2e), "route": cache.route_info()[0]}), flush=True)
    else:
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
        sets = {"alt": [cfg.alphas, cfg.alphas + 1e-9], "fixed": [cfg.alphas, cfg.alphas],
                "interior": [np.linspace(0.01, 1.99, A), np.linspace(0.01, 1.99, A) + 1e-9]}
        for name, al in sets.items():
            al = [np.ascontiguousarray(a) for a in al]

            def step(i):
                fg._check(L_.fgfrft_mse_step_dev(cache.handle, al[i & 1].ctypes.data, A, xd.data_ptr(), xcd.data_ptr(),
                                                 b, None, lo.data_ptr(), dl.data_ptr()))
            print(json.dumps({"c2": name, **timed(stream, step), "route": cache.route_info()}), flush=True)


if __name__ == "__main__":
    main()
