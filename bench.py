#!/usr/bin/env python
"""FGFRFT hot-path benchmark (BASELINE.json metric) on B200.

Headline workload: BASELINE config 3 (configs[2], the largest configuration that fits one GPU):
64x64 4-neighbour grid graph (N = 4096, F = transpose of the Laplacian eigenvectors, real
orthogonal), L = 64 (64 cached powers: 8.6 GB as real doubles, > L2), B = 1024 noisy piecewise-
smooth images, complex128. One STEP = Y = F^a X, the MSE loss against the clean images and
dL/da for one order; the order alternates between 0.37 and 0.63 every step (nothing is reused
across steps except the power cache, which the reference also builds once: transform.hpp:43-59).
`value` = whole-job signal-nodes/s = N * B / step time with inputs resident in HBM (CUDA events on
the library stream); `e2e` = the same step through the C ABI `fgfrft_mse_step` with pinned host
buffers (H2D of X and Xc, D2H of loss and dL/da inside the timed region).

Extra objects: `roofline` (dominant kernel of the step, algorithmic bytes / flops per launch over
its CUDA-event time, ncu DRAM traffic of the same kernel from profiles/), `synthesis` (F^a
synthesis GB/s vs HBM peak, the metric's first half), `cache_build`, `cpu_baseline` (oracle port on
all host cores, bounded sample) + `cpu_baseline_single_thread`, `clocks`, `gpu_launches`,
`parity_check` (the timed step's loss and dL/da against the oracle), `c2_sweep` (config 2's
64-order sweep step, kept as a secondary line).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-cpu-baseline]
Under torchrun (N > 1) the step is row-sharded over the N GPUs (strong scaling on the same
config-3 problem): see DESIGN.md section 6.
"""
import argparse
import csv
import json
import os
import platform
import re
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "F^α synthesis GB/s vs HBM peak; F^α·X signal-nodes/s (complex128)"
UNIT = "signal-nodes/s"
ALPHAS = (0.37, 0.63)   # the step's order alternates between these
WORKLOAD = ("BASELINE config 3 (configs[2]): 64x64 4-neighbour grid graph (N=4096), L=64, B=1024 noisy "
            "piecewise-smooth images, complex128; step = forward F^a X + MSE loss + dL/da for one order "
            "(alternating 0.37 / 0.63)")


def _peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm, src = float(mp["hbm_gbs"]), "MEASURED_PEAKS.json:hbm_gbs (measured copy)"
    except Exception:
        hbm, src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    fp64 = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")))
    i8 = json.load(open(os.path.join(ROOT, "profiles", "r01_int8_peak.json")))
    return {"hbm_gbs": hbm, "hbm_src": src, "fp64_tflops": float(fp64["dmma_m8n8k4_tflops"]),
            "fp64_src": "profiles/r01_fp64_peaks.json:dmma_m8n8k4_tflops (measured DMMA microbenchmark; "
                        "MEASURED_PEAKS.json has no FP64 figure)",
            "int8_tops": float(i8["cublas_int8_8192_tops"]),
            "int8_src": "profiles/r01_int8_peak.json:cublas_int8_8192_tops (measured cuBLAS int8 GEMM 8192^3 on "
                        "this pool, tools/peaks/int8_peak.cu; nominal dense 4500)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        loaded = [r for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        sm = [float(r[1]) for r in loaded]
        mx = [float(r[2]) for r in loaded]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm),
                "power_w_max": max((float(r[3]) for r in loaded if r[3].replace(".", "").isdigit()), default=None)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    """The host CPU as lscpu names it (model, sockets x cores x threads, max MHz), /proc/cpuinfo otherwise."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {k.strip(): v.strip() for k, v in (ln.split(":", 1) for ln in out.splitlines() if ":" in ln)}
        return (f"{kv.get('Model name', '?')}; {kv.get('Socket(s)', '?')} socket x {kv.get('Core(s) per socket', '?')} "
                f"cores x {kv.get('Thread(s) per core', '?')} threads = {kv.get('CPU(s)', '?')} CPUs; "
                f"max MHz {kv.get('CPU max MHz', 'n/a')}; flags avx512f={'avx512f' in kv.get('Flags', '')}")
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def ncu_summary(name_regex: str, files=("r02e_ncu_c3_summary.csv", "r02d_ncu_c3_summary.csv", "r02c_ncu_c3_summary.csv", "r02b_ncu_c3_summary.csv", "r02_ncu_c3_summary.csv",
                                         "r02_ncu_c3_gemm_summary.csv")):
    """The committed ncu --set full summary row (profiles/<file>) of the kernel whose name matches
    `name_regex`: {"traffic": dram read + write bytes per launch, "duration_us", "file"} or None."""
    rx = re.compile(name_regex)
    for name in files:
        path = os.path.join(ROOT, "profiles", name)
        if not os.path.exists(path):
            continue
        with open(path) as fh:
            for r in csv.DictReader(fh):
                if rx.search(r["kernel"]):
                    return {"traffic": float(r["dram_read_bytes"]) + float(r["dram_write_bytes"]),
                            "duration_us": float(r["duration_us"]), "file": "profiles/" + name,
                            "kernel": r["kernel"][:120]}
    return None


def workload_config(n, b, l, real, ws):
    return {"workload": WORKLOAD, "n": n, "l": l, "b": b, "orders_per_step": 1, "alphas": list(ALPHAS),
            "cache_bytes": l * n * n * (8 if real else 16), "real_f": real,
            "l2": "inputs larger than L2 (8.6 GB power cache streamed every step; X, Xc, Y 67 MB each)",
            "parallelism": (f"row shards x{ws} (strong scaling: one config-3 problem split by output rows)"
                            if ws > 1 else "single GPU")}


def oracle_step(O, cache, x, xc, alpha, cores):
    """The reference's CPU path for one step (transform.hpp:111-148 + learn.hpp:88-92 form):
    fgfrft_matrix, apply_forward (OpenBLAS zgemm standing in for Eigen), MSE loss, fgfrft_grad,
    dL/da = Re<G, dQ X>."""
    n, b = x.shape
    q = O.fgfrft_matrix(cache, alpha, nthreads=cores)
    y = q @ x
    r = y - xc
    loss = float(np.vdot(r, r).real) / (n * b)
    g = 2.0 * r / (n * b)
    dq = O.fgfrft_grad(cache, alpha, nthreads=cores)
    dl = float(np.sum(np.conj(g) * (dq @ x)).real)
    return loss, dl


def oracle_cache(O, cfg):
    # real-arithmetic recursion (F is real orthogonal): a quarter of the zgemm flops, same products
    # to rounding; slabs stored as complex128 exactly like the reference (transform.hpp:57-58)
    return O.PowerCache(cfg.f, cfg.l, memory_budget=1 << 40, real_recursion=True)


def run_reference(args, ws, rank):
    """--impl reference: the reference's CPU path (oracle port of transform.hpp; the reference
    itself cannot be built here -- Eigen3 absent) on all host threads, on this arm's workload."""
    if rank != 0:
        return
    import oracle as O
    import prep
    from threadpoolctl import threadpool_limits
    cfg = prep.config3(seed=1)
    cores = os.cpu_count() or 1
    n, b = cfg.x.shape
    with threadpool_limits(cores):
        cache = oracle_cache(O, cfg)
        for i in range(args.warmup):
            oracle_step(O, cache, cfg.x, cfg.x_clean, ALPHAS[i & 1], cores)
        t0 = time.perf_counter()
        for i in range(args.steps):
            oracle_step(O, cache, cfg.x, cfg.x_clean, ALPHAS[i & 1], cores)
        dt = (time.perf_counter() - t0) / args.steps
    value = n * b / dt
    real = bool(np.all(cfg.f.imag == 0))
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "c128", "data": "synthetic",
           "config": workload_config(n, b, cfg.l, real, ws),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(), "kind": "port",
                            "sample": "the full config-3 step per timed step (one order): fgfrft_matrix + apply "
                                      "(OpenBLAS zgemm) + MSE + fgfrft_grad + Re<G, dQ X>, oracle restatement of "
                                      "transform.hpp:21-148; reference C++ unbuildable (no Eigen3)"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline(O, cache, cfg, cores, budget_s):
    """The oracle step timed on this host (bounded: whole steps until budget_s has elapsed)."""
    from threadpoolctl import threadpool_limits
    n, b = cfg.x.shape
    with threadpool_limits(cores):
        done, t0 = 0, time.perf_counter()
        while True:
            oracle_step(O, cache, cfg.x, cfg.x_clean, ALPHAS[done & 1], cores)
            done += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
    return {"value": n * b * done / dt, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(), "kind": "port",
            "sample": f"{done} whole config-3 steps ({dt:.1f} s): oracle fgfrft_matrix + OpenBLAS zgemm apply + "
                      "MSE + fgfrft_grad + Re<G, dQ X>; reference C++ unbuildable here (Eigen3 absent)"}


def timed_events(stream, fn, reps, warm=2):
    import torch
    with torch.cuda.stream(stream):
        for i in range(warm):
            fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    with torch.cuda.stream(stream):
        for i in range(reps):
            fn(i)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def c2_sweep(fg, torch, stream, dev):
    """Config 2's 64-order sweep step (secondary line; the round-1 headline workload)."""
    import prep
    cfg = prep.config2(seed=1)
    n, b = cfg.x.shape
    A = len(cfg.alphas)
    cache = fg.PowerCache(cfg.f, cfg.l, memory_budget=8 << 30, device=dev)
    cache.set_stream(stream.cuda_stream)
    cache.prepare()
    L_ = fg.lib()
    al = [np.ascontiguousarray(cfg.alphas), np.ascontiguousarray(cfg.alphas + 1e-9)]
    xd = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).to(f"cuda:{dev}")
    xcd = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).to(f"cuda:{dev}")
    lo = torch.empty(A, dtype=torch.float64, device=f"cuda:{dev}")
    dl = torch.empty(A, dtype=torch.float64, device=f"cuda:{dev}")

    def step(i):
        fg._check(L_.fgfrft_mse_step_dev(cache.handle, al[i & 1].ctypes.data, A, xd.data_ptr(), xcd.data_ptr(), b,
                                         None, lo.data_ptr(), dl.data_ptr()))

    ms = timed_events(stream, step, 10, warm=3)
    route, nodes = cache.route_info()
    cache.close()
    return {"workload": "BASELINE config 2: N=1024 k-NN graph, L=64, B=256, 64 orders on [0,2] per step "
                        "(orders change every step)", "ms_per_step": ms, "value": n * b * A / (ms * 1e-3),
            "unit": UNIT, "route": {0: "synthesis", 1: "power products", 2: "node interpolation"}.get(route, str(route)),
            "nodes": nodes}


def run_sharded(args, ws, rank, local):
    """--gpus N > 1 (torchrun): the config-3 step on N pair shards (strong scaling). The library owns
    the NCCL communicator (fgfrft_comm_*); torch.distributed (gloo, host tensors) is used only to hand
    out its 128-byte id, for barriers and for the max over ranks of the device-timed step."""
    import torch
    import torch.distributed as dist

    import paper_2602_20870_b200 as fg
    import prep
    from paper_2602_20870_b200 import pshard as ps

    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531"), ("RANK", str(rank)),
                 ("WORLD_SIZE", str(ws))):
        os.environ.setdefault(k, v)
    dist.init_process_group("gloo")
    peaks = _peaks()
    uid = [ps.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = ps.Comm(uid[0], ws, rank, local)
    cfg = prep.config3(seed=1)
    n, b = cfg.x.shape
    L = cfg.l
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    # F from rank 0 only: the library broadcasts it over the communicator (the build's one collective)
    sh = ps.PairShard(cfg.f if rank == 0 else None, L, memory_budget=64 << 30, comm=comm, n=n)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    stream = torch.cuda.Stream()
    sh.set_stream(stream.cuda_stream)
    xd = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).to(dev)
    xcd = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).to(dev)
    L_ = fg.lib()
    al = [np.array([a]) for a in ALPHAS]
    lo = torch.empty(2, dtype=torch.float64, device=dev)
    dl = torch.empty(2, dtype=torch.float64, device=dev)

    def step(i):
        fg._check(L_.fgfrft_pshard_mse_step_dev(sh.handle, al[i & 1].ctypes.data, 1, xd.data_ptr(), xcd.data_ptr(),
                                                b, lo[i & 1:].data_ptr(), dl[i & 1:].data_ptr()))

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    l0 = fg.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    e1.synchronize()
    launches = fg.launch_count() - l0
    clk = clocks.stop() if rank == 0 else None
    torch.cuda.synchronize()
    dist.barrier()
    ms_t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64)
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t[0])
    res = (lo.cpu().numpy().copy(), dl.cpu().numpy().copy())
    # per-rank synthesis class (CUDA events on the stream the kernels run on), separate pass
    fg.profile_enable(True)
    fg.profile_read(reset=True)
    for i in range(args.steps):
        step(i)
    torch.cuda.synchronize()
    prof = fg.profile_read(reset=True)
    fg.profile_enable(False)
    info = sh.info()
    syn_ms, syn_n = prof["synthesis"]
    local_pairs = info["pair_end"] - info["pair_begin"]
    syn_bytes = local_pairs * L * 2 * (32 * 32 * 5 + 8)
    syn_gbs = syn_bytes * syn_n / (syn_ms * 1e-3) / 1e9 if syn_ms else None
    # e2e: host buffers through the C ABI (H2D of X, Xc inside the timed region)
    xh = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).pin_memory()  # column-major n x b, pinned
    xch = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).pin_memory()
    lh, dh = np.empty(1), np.empty(1)

    def step_e2e(i):
        fg._check(L_.fgfrft_pshard_mse_step(sh.handle, al[i & 1].ctypes.data, 1, xh.data_ptr(), xch.data_ptr(), b,
                                            lh.ctypes.data, dh.ctypes.data))

    for i in range(2):
        step_e2e(i)
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        step_e2e(i)
    e2e_t = torch.tensor([(time.perf_counter() - t0) / args.steps * 1e3], dtype=torch.float64)
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_t[0])
    rows = torch.tensor([syn_gbs or 0.0, float(local_pairs)], dtype=torch.float64)
    allrows = [torch.zeros_like(rows) for _ in range(ws)]
    dist.all_gather(allrows, rows)
    check = None
    if rank == 0:  # the unsharded single-GPU step on the same inputs
        cache = fg.PowerCache(cfg.f, L, memory_budget=64 << 30, device=local)
        check = []
        for i, a in enumerate(ALPHAS):
            l1, d1, _ = fg.mse_step(cache, [a], cfg.x, cfg.x_clean)
            check.append({"alpha": a, "loss": float(res[0][i]), "loss_unsharded": float(l1[0]),
                          "loss_rel_diff": abs(float(res[0][i]) - float(l1[0])) / abs(float(l1[0])),
                          "dlda": float(res[1][i]), "dlda_unsharded": float(d1[0]),
                          "dlda_rel_diff": abs(float(res[1][i]) - float(d1[0])) / max(abs(float(d1[0])), 1e-300)})
        cache.close()
        out = {
            "metric": METRIC, "value": n * b / (ms * 1e-3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded generators, prep/)",
            "config": workload_config(n, b, L, True, ws),
            "roofline": {"bound": "hbm", "kernel": "psynth_pairs_kernel<2> on each rank's pair band",
                         "achieved": syn_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": syn_gbs / peaks["hbm_gbs"] if syn_gbs else None, "traffic": None,
                         "algorithmic": "rank 0: its pairs x L x 2 tiles x (5 KB + 8 B scale) read",
                         "per_rank_gbs": [float(r[0]) for r in allrows],
                         "per_rank_pairs": [int(r[1]) for r in allrows], "peak_source": peaks["hbm_src"]},
            "collectives": "per step: ncclReduceScatter of [Y; dY] (2 x N x B complex128, by signal-column chunks) "
                           "+ ncclAllReduce of 2 doubles; build: ncclBroadcast of F",
            "cache_build": {"seconds": build_s, "note": "per-rank panel recursion + packing of its pairs"},
            "e2e": {"value": n * b / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 2 * n * b * 16, "d2h_bytes_per_step": 16,
                    "note": "fgfrft_pshard_mse_step with host X, Xc on every rank; max over ranks of wall time"},
            "gpu_launches": launches, "clocks": clk, "parity_check": check,
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    sh.close()
    comm.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="the pair-sharded path even at N = 1 (validation)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = _dist()

    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if ws > 1 or args.sharded:
        run_sharded(args, ws, rank, local)
        return

    import torch
    import paper_2602_20870_b200 as fg
    import prep

    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    peaks = _peaks()
    cfg = prep.config3(seed=1)
    n, b = cfg.x.shape
    L = cfg.l
    stream = torch.cuda.Stream()

    # ---- K1: power cache built on device, outside the timed region (as transform.hpp:43-59)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    # budget: the reference count L N^2 16 B (17.2 GB) + the packed slabs (5.4 GB) the step route uses
    # + the order window's node operators (2.5 GB, secondary line)
    cache = fg.PowerCache(cfg.f, L, memory_budget=32 << 30, device=local)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    real = cache.is_real()
    cache.set_stream(stream.cuda_stream)
    t0 = time.perf_counter()
    cache.prepare()  # lazily built device structures (packed slabs / digit slices), once per cache
    torch.cuda.synchronize()
    prepare_s = time.perf_counter() - t0

    xd = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).to(dev)      # column-major n x b
    xcd = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).to(dev)
    loss_d = torch.empty(2, dtype=torch.float64, device=dev)
    dlda_d = torch.empty(2, dtype=torch.float64, device=dev)
    al = [np.array([a]) for a in ALPHAS]
    L_ = fg.lib()

    def step_dev(i):
        fg._check(L_.fgfrft_mse_step_dev(cache.handle, al[i & 1].ctypes.data, 1, xd.data_ptr(), xcd.data_ptr(), b,
                                         None, loss_d[i & 1:].data_ptr(), dlda_d[i & 1:].data_ptr()))

    # ---- value: device-resident step, CUDA events on the library stream
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step_dev(i)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = fg.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for i in range(args.steps):
        step_dev(i)
    ev1.record(stream)
    ev1.synchronize()
    launches = fg.launch_count() - launches0
    clk = clocks.stop()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    value = n * b / (ms * 1e-3)
    step_out = (loss_d.cpu().numpy().copy(), dlda_d.cpu().numpy().copy())

    # per-kernel-class device time (CUDA events recorded by the library around each launch class on
    # the stream the kernels run on) from a separate pass of the same K steps, so that the event
    # records stay out of the timed region
    fg.profile_enable(True)
    fg.profile_read(reset=True)
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            step_dev(i)
    torch.cuda.synchronize()
    prof = fg.profile_read(reset=True)
    fg.profile_enable(False)
    tot = sum(v[0] for v in prof.values()) or 1.0
    classes = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps,
                   "share": v[0] / tot} for k, v in prof.items() if v[1]}

    # ---- roofline of the dominant kernel class.
    # synthesis (HBM): Q(a) and dQ/da from ONE pass over the stored powers. achieved / frac count the
    #   SURVEY 8(d) K2 bytes, (S*e + A*16)*N^2 with S = L slabs of e = 8 B (real F) and A = 2 outputs.
    #   On the packed route (route 3) the stored powers are the packed slabs: 5 B per element (40-bit
    #   fixed point + one scale per 32x32 tile and power), pair-major, the diagonal tiles twice; the
    #   bytes the kernel physically moves (packed slabs + scales read, Q and dQ written as real
    #   doubles) are `physical_*`, and ncu's DRAM bytes are `traffic`.
    # int8_gemm (tensor): [Y; dY] = [Q; dQ] X, 2 * (2N) * (2B) * N FP64-equivalent flops per step
    #   (real F x complex X), S(S+1)/2 int8 digit GEMMs of that size (Ozaki, S base-254 digits).
    route, _nodes = cache.route_info()
    S = int(L_.fgfrft_step_int8_digits() if route in (3, 4) else L_.fgfrft_int8_digits())
    products = S * (S + 1) // 2
    e = 8 if real else 16
    nt = -(-n // 32)
    npairs = nt * (nt + 1) // 2
    packed_bytes = npairs * L * 2 * 32 * 32 * 5 + npairs * L * 2 * 8
    # route 4: the digit cache -- npairs * 1024 element-pair rows x 2 pad64(L) powers x 5 digits,
    # + one int32 exponent per row
    dk_rows, dk_kp = npairs * 1024, 2 * (-(-L // 64) * 64)
    digit_bytes = dk_rows * dk_kp * 5 + dk_rows * 4
    # SURVEY 8(d) K2 algorithmic bytes: (S*e + A*16)*N^2 -- S = L stored slabs of e bytes per element,
    # A = 2 outputs (Q, dQ/da) counted at 16 B (the VERDICT r01 formula)
    fp64_bytes = (L * e + 2 * 16) * n * n
    # route 3 on whole 128-row tiles (one order): psynth writes [Q; dQ]'s S Ozaki digits directly
    # (packed.cu SD > 0) instead of FP64 Q, dQ
    emit = route == 3 and n % 128 == 0 and os.environ.get("FGFRFT_PSYNTH_DIGITS", "1") != "0"
    out_bytes = 2 * S * n * n if emit else 2 * 8 * n * n
    syn_bytes = {3: packed_bytes + out_bytes, 4: digit_bytes + 2 * 8 * n * n}.get(route, fp64_bytes)
    dom = max(classes, key=lambda k: classes[k]["ms_per_step"])
    syn = classes.get("synthesis")
    roof = None
    if syn:
        per_launch_ms = syn["ms_per_step"] / syn["launches_per_step"]
        ach = syn_bytes / syn["launches_per_step"] / (per_launch_ms * 1e-3) / 1e9
        fp64_ach = fp64_bytes / syn["launches_per_step"] / (per_launch_ms * 1e-3) / 1e9
        nc = ncu_summary({3: (rf"psynth_pairs_kernel<2, 2, 10, {S}>" if emit else r"psynth_pairs_kernel<2, 2, 10(, 0)?>"),
                          4: r"dsynth_kernel"}.get(route, r"rsynth_pairs"))
        roof = {"bound": "hbm",
                "kernel": {3: (f"psynth_pairs_kernel<2,2,10,{S}> (packed slabs -> the {S} Ozaki digits of Q and dQ/da, "
                               f"one pass, TMA ring)" if emit else
                               "psynth_pairs_kernel<2> (packed slabs -> Q and dQ/da, one pass, TMA ring)"),
                           4: ("dsynth_kernel<2,4> (digit cache -> Q and dQ/da on the INT8 tensor cores: TMA ring, "
                               "2 MMA-issuing warps, TMEM accumulators, mirror pairs per row)")}.get(
                               route, "rsynth_pairs_kernel (FP64 slabs -> Q and dQ/da)"),
                "achieved": fp64_ach, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": fp64_ach / peaks["hbm_gbs"],
                "algorithmic_bytes_per_launch": fp64_bytes / syn["launches_per_step"],
                "algorithmic": (f"SURVEY 8(d) K2: (S*e + A*16)*N^2 with S = L = {L} stored slabs, e = {e} B (real F "
                                f"stored as real doubles), A = 2 outputs (Q, dQ/da) = {fp64_bytes:.4g} B. frac > 1: "
                                f"the kernel streams a 40-bit fixed-point copy of the slabs (5 B per element), see "
                                f"physical_*"),
                "traffic": nc["traffic"] if nc else None,
                "traffic_source": (f"{nc['file']}: dram__bytes_read.sum + dram__bytes_write.sum of "
                                   f"'{nc['kernel'][:60]}' (ncu --set full, one launch)") if nc else None,
                "physical_bytes_per_launch": syn_bytes / syn["launches_per_step"],
                "physical_gbs": ach, "physical_frac": ach / peaks["hbm_gbs"],
                "physical": {3: (f"packed slabs {packed_bytes:.4g} B (npairs*L*2 tiles*5 KB + scales; 5 B per "
                                    f"element, diagonal tiles twice) read + " +
                                    (f"the {S} digits of Q, dQ 2*{S}*N^2 B written" if emit else
                                     "Q, dQ 2*N^2*8 B written") + f" = {syn_bytes:.4g} B"),
                                4: (f"digit cache {digit_bytes:.4g} B (npairs*1024 element-pair rows x {dk_kp} powers "
                                    f"(P_k(e) | P_k(e')) x 5 digits + 4 B exponent per row; 5 B per element and "
                                    f"power, diagonal tiles twice) read + Q, dQ 2*N^2*8 B written = {syn_bytes:.4g} B")
                                }.get(route, f"SURVEY 8(d): (S*e + A*e)*N^2, S = L = {L}, e = {e}, A = 2 = "
                                             f"{syn_bytes:.4g} B"),
                "peak_source": peaks["hbm_src"], "share_of_step": syn["share"],
                "ms_per_launch": per_launch_ms}
    i8 = classes.get("int8_gemm")
    gemm = None
    if i8:
        fp = 2.0 * 2 * n * (2 * b) * n  # [Q; dQ] (2N rows, real) x X (2B real columns), K = N
        tops = fp * products / (i8["ms_per_step"] * 1e-3) / 1e12
        nc = ncu_summary(rf"ozgemm_kernel<{S}")
        gemm = {"bound": "tensor", "kernel": f"ozgemm_kernel<{S},1,2> (tcgen05.mma kind::i8, TMEM accumulators)",
                "achieved": tops, "peak": peaks["int8_tops"], "unit": "TOPS", "frac": tops / peaks["int8_tops"],
                "fp64_equivalent_tflops": fp / (i8["ms_per_step"] * 1e-3) / 1e12,
                "dmma_peak_tflops": peaks["fp64_tflops"],
                "algorithmic": f"2*(2N)*(2B)*N = {fp:.4g} FP64-equivalent flops x {products} int8 digit GEMMs",
                "traffic": nc["traffic"] if nc else None, "peak_source": peaks["int8_src"],
                "share_of_step": i8["share"]}
    if roof is None or (gemm and dom == "int8_gemm"):
        roof, gemm = gemm, roof
    if roof is not None:
        roof["other_kernel"] = gemm
        roof["dominant_class"] = dom
    route_desc = {"route": {0: "synthesis (exact FP64 slabs)", 1: "power products", 2: "node interpolation",
                            3: "packed: Q, dQ/da from the packed slabs + one Ozaki GEMM [Y; dY] = [Q; dQ] X",
                            4: ("packed step, tensor-core synthesis: Q, dQ/da from the digit cache on tcgen05 (kind::i8) "
                                "+ one Ozaki GEMM [Y; dY] = [Q; dQ] X")}.get(route),
                  "int8_digits": S}

    # ---- synthesis GB/s (metric's first half): one order, complex128 output (fgfrft_matrix)
    qbuf = torch.empty((1, n, n), dtype=torch.complex128, device=dev)

    def synth(i):
        fg._check(L_.fgfrft_synthesize_dev(cache.handle, al[i & 1].ctypes.data, 1, 0, 0, qbuf.data_ptr()))

    t_syn = timed_events(stream, synth, 10, warm=3)
    nbytes = (L * e + 16.0) * n * n
    synthesis = {"unit": "GB/s", "orders": 1, "ms": t_syn, "gbs": nbytes / (t_syn * 1e-3) / 1e9,
                 "frac_hbm": nbytes / (t_syn * 1e-3) / 1e9 / peaks["hbm_gbs"], "algorithmic_bytes": nbytes,
                 "peak_hbm_gbs": peaks["hbm_gbs"], "peak_source": peaks["hbm_src"],
                 "layout": "S = L stored slabs, F^-k read as transposed tiles of F^k; real F stored as real "
                           "doubles (8 B/element); output complex128 (fgfrft_matrix, bit-exact to the oracle)"}
    del qbuf

    # ---- e2e: the C ABI call with pinned host buffers (H2D X, Xc + D2H loss, dL/da every step)
    xh = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).pin_memory()
    xch = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).pin_memory()
    lh = np.empty(1)
    dh = np.empty(1)

    def step_e2e(i):
        fg._check(L_.fgfrft_mse_step(cache.handle, al[i & 1].ctypes.data, 1, xh.data_ptr(), xch.data_ptr(), b,
                                     None, lh.ctypes.data, dh.ctypes.data))

    for i in range(args.warmup):
        step_e2e(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # three groups of K steps, the median group reported and all listed: the host link of this pool's
    # boxes runs 41-55 GB/s from one moment to the next (freshly pinned buffers, the first group, are the
    # usual slow one), and this number is the link's
    e2e_groups = []
    for _ in range(3):
        e0.record(stream)
        t_wall = time.perf_counter()
        for i in range(args.steps):
            step_e2e(i)
        e1.record(stream)
        e1.synchronize()
        t_wall = (time.perf_counter() - t_wall) / args.steps
        e2e_groups.append((max(e0.elapsed_time(e1) / args.steps, t_wall * 1e3), e0.elapsed_time(e1) / args.steps,
                           t_wall))
    e2e_ms, e2e_dev_ms, t_wall = sorted(e2e_groups)[1]
    # the link floor of the e2e number: the same 2 N B complex128 bytes as one plain pinned H2D copy
    # each (no kernels), median of 5 -- e2e / this = how close the step sits to the host link
    h2d_dst = torch.empty(2 * n * b * 16, dtype=torch.uint8, device=f"cuda:{local}")
    h2d_ms = []
    for _ in range(5):
        with torch.cuda.stream(stream):
            e0.record(stream)
            h2d_dst[: n * b * 16].copy_(xh.view(torch.uint8).reshape(-1), non_blocking=True)
            h2d_dst[n * b * 16:].copy_(xch.view(torch.uint8).reshape(-1), non_blocking=True)
            e1.record(stream)
        e1.synchronize()
        h2d_ms.append(e0.elapsed_time(e1))
    h2d_ms = float(np.median(h2d_ms))
    del h2d_dst

    extras = {}
    win_out = None
    if not args.no_extras:
        try:
            extras["c2_sweep"] = c2_sweep(fg, torch, stream, local)
        except Exception as ex:  # secondary line only
            extras["c2_sweep"] = {"error": str(ex)}
        # the same step with an order window declared (fgfrft_cache_set_order_window [0, 2]): Q, dQ/da
        # interpolated from r exact node operators (built once, like the power cache) instead of the
        # 64 packed powers -- a secondary line; the headline stays on the reference's series route
        try:
            t0 = time.perf_counter()
            nodes = cache.set_order_window(0.0, 2.0)
            win_build_s = time.perf_counter() - t0
            loss_w = torch.empty(2, dtype=torch.float64, device=dev)
            dlda_w = torch.empty(2, dtype=torch.float64, device=dev)

            def step_win(i):
                fg._check(L_.fgfrft_mse_step_dev(cache.handle, al[i & 1].ctypes.data, 1, xd.data_ptr(), xcd.data_ptr(),
                                                 b, None, loss_w[i & 1:].data_ptr(), dlda_w[i & 1:].data_ptr()))

            ms_w = timed_events(stream, step_win, args.steps, warm=args.warmup)
            route_w = cache.route_info()
            fg.profile_enable(True)
            fg.profile_read(reset=True)
            with torch.cuda.stream(stream):
                for i in range(args.steps):
                    step_win(i)
            torch.cuda.synchronize()
            prof_w = fg.profile_read(reset=True)
            fg.profile_enable(False)
            win_out = (loss_w.cpu().numpy().copy(), dlda_w.cpu().numpy().copy())
            for i in range(args.warmup):
                step_e2e(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            t_w = time.perf_counter()
            for i in range(args.steps):
                step_e2e(i)
            e1.record(stream)
            e1.synchronize()
            e2e_w = max(e0.elapsed_time(e1) / args.steps, (time.perf_counter() - t_w) / args.steps * 1e3)
            syn_w = prof_w.get("synthesis", (0.0, 0))
            syn_ms = syn_w[0] / args.steps if syn_w[1] else None
            wbytes = nodes * n * n * 8 + 2 * n * n * 8
            extras["order_window_step"] = {
                "workload": "config 3 step as the headline, order window [0, 2] declared",
                "route": {"route": route_w[0], "nodes": route_w[1]}, "window_build_s": win_build_s,
                "ms_per_step": ms_w, "value": n * b / (ms_w * 1e-3), "unit": UNIT,
                "e2e": {"value": n * b / (e2e_w * 1e-3), "unit": UNIT, "ms_per_step": e2e_w},
                "kernel_classes_ms_per_step": {k: v[0] / args.steps for k, v in prof_w.items() if v[1]},
                "synthesis_roofline": ({"kernel": "window_synth_kernel<2> (node operators -> Q, dQ/da + row maxima)",
                                        "algorithmic_bytes": wbytes, "achieved_gbs": wbytes / (syn_ms * 1e-3) / 1e9,
                                        "peak": peaks["hbm_gbs"],
                                        "frac": wbytes / (syn_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                        "algorithmic": f"{nodes} node operators x N^2 x 8 B read + Q, dQ 2 N^2 x 8 B "
                                                       f"written"} if syn_ms else None)}
            cache.set_order_window(0.0, 0.0)
        except Exception as ex:  # secondary line only
            extras["order_window_step"] = {"error": str(ex)}

    # ---- parity of the timed step against the oracle (rank 0; the oracle cache is reused by the CPU
    # baseline below). After every GPU timing: the oracle's BLAS threads keep spinning for a while
    # after their work and would steal the launching thread's core from the e2e / sweep timings.
    import oracle as O
    from threadpoolctl import threadpool_limits
    cores = os.cpu_count() or 1
    with threadpool_limits(cores):
        t0 = time.perf_counter()
        ocache = oracle_cache(O, cfg)
        ocache_s = time.perf_counter() - t0
        check = []
        for i, a in enumerate(ALPHAS):
            lr, dr = oracle_step(O, ocache, cfg.x, cfg.x_clean, a, cores)
            if win_out is not None:
                extras["order_window_step"].setdefault("parity_check", []).append(
                    {"alpha": a, "loss_rel_err": abs(float(win_out[0][i]) - lr) / abs(lr),
                     "dlda_rel_err": abs(float(win_out[1][i]) - dr) / max(abs(dr), 1e-300)})
            check.append({"alpha": a, "loss": float(step_out[0][i]), "loss_ref": lr,
                          "loss_rel_err": abs(float(step_out[0][i]) - lr) / abs(lr),
                          "dlda": float(step_out[1][i]), "dlda_ref": dr,
                          "dlda_rel_err": abs(float(step_out[1][i]) - dr) / max(abs(dr), 1e-300)})

    cpu = cpu1 = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(O, ocache, cfg, cores, 15.0)
        cpu1 = cpu_baseline(O, ocache, cfg, 1, 10.0)  # the reference's single-threaded configuration
        cpu["oracle_cache_build_s"] = ocache_s
    del ocache

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded generators, prep/)",
        "config": workload_config(n, b, L, real, ws),
        "roofline": roof,
        "kernel_classes": classes,
        "route": route_desc,
        "synthesis": synthesis,
        "cache_build": {"seconds": build_s, "prepare_seconds": prepare_s,
                        "note": "host wall clock incl. H2D of F and the orthogonality check; prepare = the "
                                "lazily built step structures, once per cache"},
        "e2e": {"value": n * b / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                "device_ms": e2e_dev_ms, "wall_ms": t_wall * 1e3,
                "h2d_bytes_per_step": 2 * n * b * 16, "d2h_bytes_per_step": 2 * 8,
                "groups_ms_per_step": [g[0] for g in e2e_groups],
                "h2d_copy_only_ms": h2d_ms, "h2d_copy_only_gbs": 2 * n * b * 16 / (h2d_ms * 1e-3) / 1e9,
                "note": "h2d_copy_only = the step's X + Xc bytes as plain pinned H2D copies on the same stream "
                        "(the host link's floor for this e2e; it varies box to box)"},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk,
        "parity_check": check,
        "cpu_baseline": cpu,
        "cpu_baseline_single_thread": cpu1,
        **extras,
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
