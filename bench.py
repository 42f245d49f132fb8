#!/usr/bin/env python
"""FGFRFT hot-path benchmark (BASELINE.json metric) on B200.

Workload (BASELINE config 2, configs[1]): N=1024 Gaussian-weighted k-NN sensor graph, L=64
(cache = 64 complex128 powers, 1.07 GB > L2), B=256 noisy bandlimited signals, 64 orders
swept over [0, 2]. One STEP = for every order: Y = F^alpha X, the MSE loss against the clean
signals and dL/dalpha. With a real F (every BASELINE config) the library runs the power-product
route: Z_k = F^k X for k = +-1..+-L in ONE INT8 tensor-core GEMM (Ozaki scheme) over the stacked
cache, then per order Y = sum_k c_k Z_k, the loss and s_k = Re<G, Z_k> on DMMA
(dmma_engine_ms_per_step: the same step on the FP64-tensor-core synthesis route).
`value` is whole-job signal-nodes/s = N * B * A * ranks / step time, inputs resident in HBM;
`e2e` is the same step through the C ABI with pinned host buffers (H2D of X, Xc and D2H of the
per-order losses and gradients inside the timed region).

Extra objects: `roofline` for the dominant kernel (the INT8 Ozaki GEMM, or the DMMA GEMM),
`synthesis` (F^alpha synthesis GB/s vs HBM peak, the metric's first half, 64-order sweep and
single order), `cache_build` (K1 TFLOP/s), `cpu_baseline` (the oracle on this host, bounded
sample; `cpu_baseline_single_thread` the same at 1 thread, the reference's own configuration),
`clocks` (nvidia-smi during the timed region), `gpu_launches`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun (N > 1) every rank runs an independent replica of the workload (different
signal seed; the path shards by independent problems, no data-path collective): weak scaling.
"""
import argparse
import json
import os
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


def _peaks():
    hbm, src = None, None
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
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _config(rank: int):
    import prep
    cfg = prep.config2(seed=1)  # graph / F identical on every rank
    if rank:
        # independent replica: same graph, signals from a rank-derived stream
        rng = prep.Rng(prep.Rng.derive(1, 100 + rank))
        n, b = cfg.x.shape
        coef = np.zeros((n, b))
        coef[:50, :] = rng.gaussians(50 * b).reshape(b, 50).T
        clean = cfg.f.conj().T @ coef.astype(np.complex128)
        cfg.x = np.asfortranarray(clean + 0.1 * rng.gaussians(n * b).reshape(b, n).T)
        cfg.x_clean = np.asfortranarray(clean)
    return cfg


def ncu_traffic(kernel_prefix: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel from the committed ncu
    --set full summaries (newest first: profiles/r01_ncu_node_summary.csv, r01_ncu_final_summary.csv),
    or None."""
    import csv
    for name in ("r01_ncu_node_summary.csv", "r01_ncu_final_summary.csv"):
        try:
            rows = list(csv.reader(open(os.path.join(ROOT, "profiles", name))))
            h, u = rows[0], rows[1]
            ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            for r in rows[2:]:
                if r[ki].startswith(kernel_prefix):
                    return float(r[ri]) * scale[u[ri]] + float(r[wi]) * scale[u[wi]]
        except Exception:
            continue
    return None


def workload_config(cfg, ws):
    """The `config` object of both arms (ours and --impl reference): the same workload."""
    n, b = cfg.x.shape
    real = bool(np.all(cfg.f.imag == 0))
    return {"workload": "BASELINE config 2 (configs[1]): N=1024 Gaussian k-NN sensor graph, L=64, "
                        "B=256 noisy bandlimited signals, 64 orders linspace(0,2); step = forward "
                        "F^a X + MSE loss + dL/da for every order",
            "n": n, "l": cfg.l, "b": b, "orders": len(cfg.alphas),
            "cache_bytes": cfg.l * n * n * (8 if real else 16), "real_f": real,
            "l2": "inputs larger than L2 (0.54 GB real cache + 0.8 GB INT8 digits streamed every step)",
            "parallelism": f"replicas x{ws} (independent problems per rank)"}


def run_reference(args, ws, rank):
    """--impl reference: the reference's CPU path (oracle port; the reference itself cannot be
    built here -- Eigen3 absent) on all host threads, each step a bounded sample of the workload."""
    if rank != 0:
        return
    import oracle as O
    from threadpoolctl import threadpool_limits
    cfg = _config(0)
    cores = os.cpu_count() or 1
    n, b = cfg.x.shape
    sample = [float(a) for a in cfg.alphas[:: max(1, len(cfg.alphas) // 2)][:2]]
    with threadpool_limits(cores):
        cache = O.PowerCache(cfg.f, cfg.l)

        def step():
            for a in sample:
                q = O.fgfrft_matrix(cache, a, nthreads=cores)
                y = q @ cfg.x
                r = y - cfg.x_clean
                g = 2.0 * r / (n * b)
                dq = O.fgfrft_grad(cache, a, nthreads=cores)
                _ = float(np.sum(np.conj(g) * (dq @ cfg.x)).real)

        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        dt = (time.perf_counter() - t0) / args.steps
    value = n * b * len(sample) / dt
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "c128", "data": "synthetic",
           "config": workload_config(cfg, ws),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                            "sample": f"{len(sample)} of 64 orders per step (alphas {sample}): fgfrft_matrix + "
                                      "apply (OpenBLAS zgemm) + fgfrft_grad + <G, dQ X>, oracle restatement of "
                                      "transform.hpp; reference C++ unbuildable (no Eigen3)"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline(cfg, budget_s=20.0, cores=None):
    """Oracle port on this host, bounded sample (rank 0, N=1 only). cores=None: all host cores;
    cores=1: the reference's single-threaded configuration (proj/README.md:47-48)."""
    import oracle as O
    from threadpoolctl import threadpool_limits
    cores = cores or os.cpu_count() or 1
    n, b = cfg.x.shape
    with threadpool_limits(cores):
        cache = O.PowerCache(cfg.f, cfg.l)
        done, t0 = 0, time.perf_counter()
        for a in cfg.alphas:
            q = O.fgfrft_matrix(cache, float(a), nthreads=cores)
            y = q @ cfg.x
            g = 2.0 * (y - cfg.x_clean) / (n * b)
            dq = O.fgfrft_grad(cache, float(a), nthreads=cores)
            _ = float(np.sum(np.conj(g) * (dq @ cfg.x)).real)
            done += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
    return {"value": n * b * done / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"first {done} of 64 orders of the config-2 sweep (~{dt:.1f} s): oracle fgfrft_matrix + "
                      "OpenBLAS apply + fgfrft_grad + <G, dQ X>; reference C++ unbuildable here (Eigen3 absent)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    ws, rank, local = _dist()

    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import torch
    import paper_2602_20870_b200 as fg

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = _peaks()
    cfg = _config(rank)
    n, b = cfg.x.shape
    A, L = len(cfg.alphas), cfg.l
    alphas = np.ascontiguousarray(cfg.alphas, dtype=np.float64)
    stream = torch.cuda.Stream()

    # ---- K1: power cache built on device (DMMA GEMM chain), timed with events on the default stream
    torch.cuda.synchronize()
    fg.profile_enable(True)
    fg.profile_read(reset=True)
    t0 = time.perf_counter()
    cache = fg.PowerCache(cfg.f, L, memory_budget=8 << 30, device=local)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    build_gemm_ms = fg.profile_read(reset=True)["dmma_zgemm"][0]
    fg.profile_enable(False)
    # (L-1) products F^a F^b: 2 n^3 flops real (graph GFT), 8 n^3 complex
    build_flops = (L - 1) * (2.0 if cache.is_real() else 8.0) * n ** 3
    cache.set_stream(stream.cuda_stream)
    # INT8 digit slices of the stacked cache for the power-product route (built once per cache,
    # like the cache itself; outside the timed region)
    t0 = time.perf_counter()
    cache.prepare()
    slices_s = time.perf_counter() - t0

    xd = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).to(f"cuda:{local}")      # column-major n x b
    xcd = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).to(f"cuda:{local}")
    loss_d = torch.empty(A, dtype=torch.float64, device=f"cuda:{local}")
    dlda_d = torch.empty(A, dtype=torch.float64, device=f"cuda:{local}")
    L_ = fg.lib()

    def step_dev():
        fg._check(L_.fgfrft_mse_step_dev(cache.handle, alphas.ctypes.data, A, xd.data_ptr(), xcd.data_ptr(), b,
                                         None, loss_d.data_ptr(), dlda_d.data_ptr()))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- value: device-resident step, CUDA events on the library stream
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step_dev()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = fg.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step_dev()
    ev1.record(stream)
    ev1.synchronize()
    launches = fg.launch_count() - launches0
    clk = clocks.stop()
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    # per-kernel-class device time (CUDA events around each class inside the library) from a
    # separate pass of the same K steps, so the event records stay out of the timed region
    fg.profile_enable(True)
    fg.profile_read(reset=True)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            step_dev()
    torch.cuda.synchronize()
    prof = fg.profile_read(reset=True)
    fg.profile_enable(False)
    value = n * b * A * ws / (ms * 1e-3)

    # loss / gradient sanity against the oracle on one order (rank 0, cheap)
    check = None
    if rank == 0:
        import oracle as O
        ocache = O.PowerCache(cfg.f, L)
        i = 23
        lr, dr, _ = O.dlda_mse(ocache, float(alphas[i]), cfg.x, cfg.x_clean)
        check = {"alpha": float(alphas[i]), "loss_rel_err": abs(float(loss_d[i]) - lr) / abs(lr),
                 "dlda_abs_err": abs(float(dlda_d[i]) - dr), "dlda_ref": dr}
        del ocache

    # ---- dominant kernel roofline.
    # Power-product route (real F, INT8 engine): ozgemm_kernel computes Z = [P_1..P_L; P_1^T..P_L^T] X,
    #   2 * (2L n) * 2B * n FP64-equivalent flops per step (real x complex: 2B real columns), as
    #   S(S+1)/2 int8 digit-product GEMMs (Ozaki, S base-254 digits). combine_kernel: 2 DMMA GEMMs
    #   of 2 * A * (2L+1) * 2nB flops each.
    # Synthesis route (DMMA engine): the DMMA GEMMs Q X and G X^H, 4 n^2 B flops each (real F).
    real = cache.is_real()
    tot_prof = sum(v[0] for v in prof.values())
    shares = {k: (v[0] / tot_prof if tot_prof else None) for k, v in prof.items()}
    i8_ms, i8_n = prof["int8_gemm"]
    route, nodes = cache.route_info()
    power_route = i8_n > 0
    if power_route and route == 2:
        # Node route. Two INT8 Ozaki GEMMs (S(S+1)/2 digit products each):
        #  * node operators W_j = Q(a_j), j < r: n^2 element rows of the sliced cache (K = 2L terms)
        #    x r node coefficient rows. A skinny GEMM (r <= 48 output columns): bound by streaming
        #    the S-digit element-row slices (S * n^2 * 2L bytes) and writing W (r n^2 doubles);
        #  * node products Z'_j = W_j X (r n x 2B x n): tensor-bound.
        # node_combine: Y rows (2 A r 2nB DMMA flops) + the node Gram [Z'; Xc][Z'; Xc]^T.
        S = int(L_.fgfrft_int8_digits())
        products = S * (S + 1) // 2
        r = nodes
        nodeop_ms, nodeop_n = prof["node_operators"]
        fp_basis = 2.0 * n * n * r * (2 * L)
        fp_prod = 2.0 * (r * n) * (2 * b) * n
        basis_bytes = float(S * n * n * 2 * L + r * n * n * 8)
        basis_cache_bytes = float((L if real else 2 * L) * n * n * (8 if real else 16) + r * n * n * 8)
        prod_tops = fp_prod * products * args.steps / (i8_ms * 1e-3) / 1e12
        basis_gbs = basis_bytes * args.steps / (nodeop_ms * 1e-3) / 1e9
        cb_ms, cb_n = prof["combine"]
        cb_flops = 2.0 * A * r * 2 * n * b + 2.0 * (r + 1) * (r + 2) / 2 * 2 * n * b
        traffic = ncu_traffic("void ozgemm_kernel<6, 0, 1>")
        hbm_peak = peaks["hbm_gbs"]
        roof = {"bound": "hbm",
                "kernel": f"ozgemm_kernel<{S},0,1> (node operators: tcgen05.mma kind::i8 over the element-row "
                          f"digit slices of the cache, r = {r} output columns)",
                "achieved": basis_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": basis_gbs / hbm_peak,
                "traffic": traffic,
                "traffic_note": "DRAM read + write per launch of the node-operator GEMM (ncu --set full capture)",
                "peak_source": peaks["hbm_src"],
                "algorithmic": (f"per launch: S*N^2*2L digit bytes of the element-row slices read + r*N^2*8 "
                                f"bytes of W written = {basis_bytes:.4g} B ({basis_cache_bytes:.4g} B counting "
                                f"the FP64 cache itself instead of its digits)"),
                "route": f"node interpolation, r = {r} Chebyshev nodes on [{alphas.min():.3g}, {alphas.max():.3g}]",
                "share_of_step": shares,
                "node_operator_gemm": {"ms_per_step": nodeop_ms / args.steps, "gbs": basis_gbs,
                                       "gbs_vs_fp64_cache_bytes": basis_cache_bytes * args.steps
                                       / (nodeop_ms * 1e-3) / 1e9,
                                       "fp64_equivalent_flops": fp_basis},
                "node_product_gemm": {"kernel": f"ozgemm_kernel<{S},1,2>", "bound": "tensor",
                                      "ms_per_step": i8_ms / args.steps, "achieved_tops": prod_tops,
                                      "peak_tops": peaks["int8_tops"], "frac": prod_tops / peaks["int8_tops"],
                                      "peak_source": peaks["int8_src"],
                                      "algorithmic": f"2*(r*N)*(2B)*N = {fp_prod:.4g} FP64-equivalent flops x "
                                                     f"{products} digit products",
                                      "fp64_equivalent_tflops": fp_prod * args.steps / (i8_ms * 1e-3) / 1e12,
                                      "dmma_peak_tflops": peaks["fp64_tflops"]},
                "combine_kernel": {"ms_per_step": cb_ms / args.steps, "flops_per_step": cb_flops,
                                   "tflops": cb_flops * args.steps / (cb_ms * 1e-3) / 1e12,
                                   "form": "Y = P_C Z' (DMMA) + loss; dL/da from the node Gram of [Z'; Xc]",
                                   "peak_dmma_tflops": peaks["fp64_tflops"]}}
    elif power_route:
        S = int(L_.fgfrft_int8_digits())
        products = S * (S + 1) // 2
        fp64eq = 2.0 * (2 * L * n) * (2 * b) * n
        i8_ops = fp64eq * products
        achieved = i8_ops * args.steps / (i8_ms * 1e-3) / 1e12
        cb_ms, cb_n = prof["combine"]
        # combine: Y = C Z (2*A*(2L+1)*2nB DMMA flops) + either S = G Z^T (same again) or, for an
        # orthogonal F, the 2(2L+1) dot products R_q = <Xc, Z_q>, gamma(d) = <X, F^d X> (FP64 FMA)
        gram = cache.orthogonality() is not None and 0 <= cache.orthogonality() <= 1e-12
        y_flops = 2.0 * A * (2 * L + 1) * 2 * n * b
        cb_flops = y_flops + (2.0 * 2 * (2 * L + 1) * 2 * n * b if gram else y_flops)
        cb_form = ("Y = C Z (DMMA) + Gram sequence / R dot products (F orthogonal: "
                   f"residual {cache.orthogonality():.2e})" if gram else "Y = C Z and S = G Z^T (DMMA)")
        traffic = ncu_traffic(f"void ozgemm_kernel<{S}, 1, 2>")
        roof = {"bound": "tensor",
                "kernel": f"ozgemm_kernel<{S},1,2> (tcgen05.mma kind::i8, TMEM digit accumulators)",
                "achieved": achieved, "peak": peaks["int8_tops"], "unit": "TOPS",
                "frac": achieved / peaks["int8_tops"], "traffic": traffic,
                "traffic_note": ("bytes per launch, DRAM read + write from profiles/r01_ncu_final_summary.csv "
                                 "(ncu --set full); algorithmic: sliced cache 2L*N*N*S bytes read once + Z "
                                 "2L*N*2B*8 written = %.3g" % (2 * L * n * n * S + 2 * L * n * 2 * b * 8)),
                "peak_source": peaks["int8_src"],
                "algorithmic": "per step 2*(2L*N)*(2B)*N FP64-equivalent flops (Z = F^k X, k = +-1..+-L, real F x "
                               f"complex X) = {products} int8 digit-product GEMMs of that size (Ozaki scheme, "
                               f"{S} base-254 digits)",
                "fp64_equivalent_tflops": fp64eq * args.steps / (i8_ms * 1e-3) / 1e12,
                "fp64_equivalent_frac_of_dmma_peak": fp64eq * args.steps / (i8_ms * 1e-3) / 1e12 / peaks["fp64_tflops"],
                "dmma_peak_tflops": peaks["fp64_tflops"],
                "launches_timed": i8_n, "share_of_step": shares,
                "combine_kernel": {"ms_per_step": cb_ms / args.steps,
                                   "flops_per_step": cb_flops,
                                   "tflops": cb_flops * args.steps / (cb_ms * 1e-3) / 1e12,
                                   "form": cb_form,
                                   "peak_dmma_tflops": peaks["fp64_tflops"]}}
    else:
        gemm_ms, gemm_n = prof["dmma_zgemm"]
        gemm_flops_step = 2 * A * (4.0 if real else 8.0) * n * n * b
        gemm_tflops = gemm_flops_step * args.steps / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None
        roof = {"bound": "tensor",
                "kernel": ("rgemm_kernel (FP64 DMMA, real Q x complex X)" if real
                           else "zgemm_dmma_kernel (FP64 DMMA complex GEMM)"),
                "achieved": gemm_tflops, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                "frac": (gemm_tflops / peaks["fp64_tflops"]) if gemm_tflops else None,
                "traffic": None, "peak_source": peaks["fp64_src"],
                "algorithmic": ("4*N^2*B flops per order per GEMM (real F: real x complex), "
                                "2 GEMMs per order" if real else
                                "8*N^2*B flops per order per GEMM, 2 GEMMs per order"),
                "launches_timed": gemm_n, "share_of_step": shares}

    # ---- the same step on the FP64-tensor-core (DMMA) engine, for comparison
    dmma_ms = None
    if power_route:
        cache.set_engine(fg.ENGINE_DMMA)
        with torch.cuda.stream(stream):
            for _ in range(2):
                step_dev()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            step_dev()
        e1.record(stream)
        e1.synchronize()
        dmma_ms = e0.elapsed_time(e1) / 5
        cache.set_engine(fg.ENGINE_AUTO)

    # ---- synthesis GB/s (metric's first half): 64-order sweep and a single order, device output
    qbuf = torch.empty((A, n, n), dtype=torch.complex128, device=f"cuda:{local}")

    def synth(al):
        fg._check(L_.fgfrft_synthesize_dev(cache.handle, al.ctypes.data, len(al), 0, 0, qbuf.data_ptr()))

    syn = {}
    for tag, al in (("sweep64", alphas), ("single", alphas[23:24].copy())):
        with torch.cuda.stream(stream):
            for _ in range(3):
                synth(al)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(stream)
        for _ in range(reps):
            synth(al)
        e1.record(stream)
        e1.synchronize()
        t = e0.elapsed_time(e1) / reps
        nbytes = (L * (8.0 if real else 16.0) + len(al) * 16.0) * n * n
        syn[tag] = {"orders": len(al), "ms": t, "gbs": nbytes / (t * 1e-3) / 1e9,
                    "frac_hbm": nbytes / (t * 1e-3) / 1e9 / peaks["hbm_gbs"], "algorithmic_bytes": nbytes,
                    "flops": 8.0 * L * n * n * len(al)}
    del qbuf

    # ---- e2e: through the C ABI with pinned host buffers (H2D X, Xc + D2H loss, dL/dalpha)
    xh = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).pin_memory()
    xch = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).pin_memory()
    lh = torch.empty(A, dtype=torch.float64).pin_memory()
    dh = torch.empty(A, dtype=torch.float64).pin_memory()

    def step_e2e():
        fg._check(L_.fgfrft_mse_step(cache.handle, alphas.ctypes.data, A, xh.data_ptr(), xch.data_ptr(), b, None,
                                     lh.data_ptr(), dh.data_ptr()))

    for _ in range(args.warmup):
        step_e2e()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        step_e2e()
    e1.record(stream)
    e1.synchronize()
    t_wall = (time.perf_counter() - t_wall) / args.steps
    e2e_dev_ms = e0.elapsed_time(e1) / args.steps
    e2e_ms = max_over_ranks(max(e2e_dev_ms, t_wall * 1e3))
    e2e_value = n * b * A * ws / (e2e_ms * 1e-3)

    # Orders that change every step (a learning loop): two order sets differing by 1e-9 alternate,
    # so each call re-plans on the host (node count, interpolation check, coefficient tables) and
    # re-uploads the tables; the device work is the same as in the timed step above, where the
    # library reuses the host tables of an unchanged order set.
    alphas_b = alphas + 1e-9
    alt = [alphas, alphas_b]

    def step_alt(i):
        al = alt[i & 1]
        fg._check(L_.fgfrft_mse_step_dev(cache.handle, al.ctypes.data, A, xd.data_ptr(), xcd.data_ptr(), b,
                                         None, loss_d.data_ptr(), dlda_d.data_ptr()))

    for i in range(2):
        step_alt(i)
    torch.cuda.synchronize()
    ea0, ea1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea0.record(stream)
    t_alt = time.perf_counter()
    for i in range(args.steps):
        step_alt(i)
    ea1.record(stream)
    ea1.synchronize()
    t_alt = (time.perf_counter() - t_alt) / args.steps
    alt_ms = max_over_ranks(max(ea0.elapsed_time(ea1) / args.steps, t_alt * 1e3))
    orders_changing = {"ms_per_step": alt_ms, "value": n * b * A * ws / (alt_ms * 1e-3), "unit": UNIT,
                       "note": "orders change every step (two sets 1e-9 apart alternate): host re-plan + "
                               "coefficient upload per call; max of device and wall time per step"}

    cpu = cpu1 = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg)
        cpu1 = cpu_baseline(cfg, budget_s=8.0, cores=1)  # the reference's single-threaded configuration

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": workload_config(cfg, ws),
            "roofline": roof,
            "route": (f"node interpolation: Q(a) through r = {nodes} Chebyshev nodes of the order interval; the "
                      "node operators W_j by one INT8 tensor-core Ozaki GEMM over the cache's 2L terms, Z'_j = W_j X "
                      "by a second, then Y and the loss of every order by one DMMA pass that also forms the node Gram, "
                      "from which dL/da follows for every order"
                      if route == 2 else
                      "power products: Z = F^k X by one INT8 tensor-core Ozaki GEMM over the stacked cache, "
                      "then per-order combination + MSE + dL/da on DMMA" if power_route else
                      "per-order synthesis Q(a) + DMMA GEMMs"),
            "dmma_engine_ms_per_step": dmma_ms,
            "synthesis": {"unit": "GB/s", "peak_hbm_gbs": peaks["hbm_gbs"], "peak_source": peaks["hbm_src"],
                          "layout": "S = L stored slabs (F^-k read as conjugate-transposed tile pairs); "
                                    + ("real F: slabs stored as real doubles (8 B/element), output complex128"
                                       if real else "complex128 slabs"),
                          **syn},
            "cache_build": {"seconds": build_s, "wall_tflops": build_flops / build_s / 1e12,
                            "gemm_ms": build_gemm_ms,
                            "gemm_tflops": build_flops / (build_gemm_ms * 1e-3) / 1e12 if build_gemm_ms else None,
                            "gemm_frac_fp64": (build_flops / (build_gemm_ms * 1e-3) / 1e12 / peaks["fp64_tflops"]
                                               if build_gemm_ms else None),
                            "flops": build_flops,
                            "note": "seconds: host wall clock incl. H2D of F, allocations and the orthogonality "
                                    "check; gemm_*: CUDA-event time of the DMMA products (doubling build, "
                                    "P_(s+j) = P_j P_s, batched per level)",
                            "int8_slices_seconds": slices_s},
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms,
                    "device_ms": e2e_dev_ms, "wall_ms": t_wall * 1e3,
                    "h2d_bytes_per_step": 2 * n * b * 16, "d2h_bytes_per_step": 2 * A * 8},
            "orders_changing": orders_changing,
            "gpu_launches": launches,
            "clocks": clk,
            "parity_check": check,
            "cpu_baseline": cpu,
            "cpu_baseline_single_thread": cpu1,
        }
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
