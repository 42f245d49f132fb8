"""Config-3 step probe: forward F^a X + MSE + dL/da (one order, alternating between two orders
every call) through fgfrft_mse_step_dev, CUDA events on the library stream, plus the library's
per-kernel-class breakdown. Used for ncu launch lists of the headline step.

  python tools/c3_step.py [--steps 10] [--warmup 3] [--config 3|4] [--c64]
"""
import argparse
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="3")
    ap.add_argument("--c64", action="store_true")
    ap.add_argument("--pshard", action="store_true", help="the pair-shard step at world 1 (NCCL communicator)")
    ap.add_argument("--sweep", default="", help="env settings to time in turn, e.g. "
                    "'FGFRFT_PIPE_SHELLS=1;FGFRFT_PIPE_SHELLS=4&FGFRFT_PIPE_GEMM_CTAS=100'")
    ap.add_argument("--trace", action="store_true", help="print the last step's launch timeline (sweep mode)")
    ap.add_argument("--window", default="", help="declare an order window 'lo,hi' (node-operator route)")
    args = ap.parse_args()
    t0 = time.perf_counter()
    cfg = prep.config3() if args.config == "3" else prep.config4()
    prep_s = time.perf_counter() - t0
    n, b, L = cfg.n, cfg.b, cfg.l
    dtype = 1 if args.c64 else 0
    ct = torch.complex64 if args.c64 else torch.complex128
    stream = torch.cuda.Stream()
    t0 = time.perf_counter()
    lib = fg.lib()
    if args.pshard:
        from paper_2602_20870_b200 import pshard as ps
        comm = ps.Comm(ps.Comm.unique_id(), 1, 0, 0)
        cache = ps.PairShard(cfg.f, L, memory_budget=120 << 30, comm=comm)
        step_fn = lib.fgfrft_pshard_mse_step_dev
    else:
        cache = fg.PowerCache(cfg.f, L, memory_budget=200 << 30, dtype=dtype)
        step_fn = None
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    cache.set_stream(stream.cuda_stream)
    if args.window and not args.pshard:
        t1 = time.perf_counter()
        print(json.dumps({"window": args.window, "nodes": cache.set_order_window(*map(float, args.window.split(","))),
                          "window_build_s": time.perf_counter() - t1}), flush=True)
    al = [np.array([0.37]), np.array([0.63])]
    x = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda().to(ct)
    xc = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).cuda().to(ct)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    dl = torch.empty(1, dtype=torch.float64, device="cuda")

    def step(i):
        if step_fn is not None:
            fg._check(step_fn(cache.handle, al[i & 1].ctypes.data, 1, x.data_ptr(), xc.data_ptr(), b, loss.data_ptr(),
                              dl.data_ptr()))
            return
        fg._check(lib.fgfrft_mse_step_dev(cache.handle, al[i & 1].ctypes.data, 1, x.data_ptr(), xc.data_ptr(), b,
                                          None, loss.data_ptr(), dl.data_ptr()))

    if args.sweep:
        for setting in args.sweep.split(";"):
            for kv in filter(None, setting.split("&")):
                k, v = kv.split("=")
                if v:
                    os.environ[k] = v
                else:
                    os.environ.pop(k, None)
            with torch.cuda.stream(stream):
                for i in range(args.warmup):
                    step(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(args.steps):
                step(i)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            fg.profile_enable(True)
            fg.profile_read(reset=True)
            with torch.cuda.stream(stream):
                for i in range(args.steps):
                    step(i)
            torch.cuda.synchronize()
            tr = fg.profile_trace()
            per = len(tr) // args.steps
            trace = [(c, round(a, 3), round(b, 3)) for c, a, b in tr[-per:]]
            t00 = trace[0][1] if trace else 0.0
            trace = [(c, round(a - t00, 3), round(b - t00, 3)) for c, a, b in trace]
            prof = {k: round(v[0] / args.steps, 4) for k, v in fg.profile_read(reset=True).items() if v[1]}
            fg.profile_enable(False)
            if args.trace:
                print(json.dumps({"setting": setting, "trace": trace}), flush=True)
            print(json.dumps({"setting": setting, "ms_per_step": ms, "classes": prof,
                              "route": cache.route_info()[0] if not args.pshard else None,
                              "loss": float(loss[0]), "dlda": float(dl[0])}), flush=True)
        return
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = fg.launch_count()
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = (fg.launch_count() - l0) / args.steps
    fg.profile_enable(True)
    fg.profile_read(reset=True)
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            step(i)
    torch.cuda.synchronize()
    prof = {k: [v[0] / args.steps, v[1] / args.steps] for k, v in fg.profile_read(reset=True).items() if v[1]}
    fg.profile_enable(False)
    print(json.dumps({"config": "C" + args.config, "c64": args.c64, "pshard": args.pshard, "n": n, "l": L, "b": b,
                      "route": cache.route_info() if not args.pshard else None, "ms_per_step": ms,
                      "signal_nodes_per_s": n * b / (ms * 1e-3), "launches_per_step": launches,
                      "prep_s": prep_s, "build_s": build_s, "classes_ms_per_step": prof,
                      "loss": float(loss[0]), "dlda": float(dl[0])}), flush=True)


if __name__ == "__main__":
    main()
