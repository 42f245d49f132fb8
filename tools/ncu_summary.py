"""Compact per-kernel summary of an ncu --set full report (run here, without a GPU):

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/r02_ncu_c3_summary.csv

Columns: kernel, duration_us, dram_read_bytes, dram_write_bytes, dram_pct (of peak sustained),
sm_throughput_pct, tensor_pipe_pct (any tensor pipe), fp64_pipe_pct, issue_active_pct, regs,
smem_dyn_bytes, grid, block. bench.py reads `traffic` (dram read + write per launch) from it.
"""
import csv
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                                                "nsecond": 1e-3}),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", {}),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", {}),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", {}),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", {}),
    "regs": ("launch__registers_per_thread", {}),
    "smem_dyn_bytes": ("launch__shared_mem_per_block_dynamic", None),
    "grid": ("launch__grid_size", {}),
    "block": ("launch__block_size", {}),
}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "Kbyte/block": 1e3, "byte/block": 1.0, "Mbyte/block": 1e6}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    head, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(head)}
    tensor_cols = [i for i, h in enumerate(head)
                   if h.startswith("sm__pipe_tensor") and h.endswith("pct_of_peak_sustained_active")]
    w = csv.writer(sys.stdout)
    w.writerow(["kernel"] + list(METRICS) + ["tensor_pipe_pct"])
    for r in rows[2:]:
        out = [r[idx["Kernel Name"]]]
        for key, (m, scale) in METRICS.items():
            if m not in idx:
                out.append("")
                continue
            v, u = r[idx[m]].replace(",", ""), units[idx[m]]
            try:
                x = float(v)
            except ValueError:
                out.append("")
                continue
            if scale is None:
                x *= BYTES.get(u, 1.0)
            elif scale:
                x *= scale.get(u, 1.0)
            out.append(f"{x:.6g}")
        tp = []
        for i in tensor_cols:
            try:
                tp.append(float(r[i]))
            except ValueError:
                pass
        out.append(f"{max(tp):.4g}" if tp else "")
        w.writerow(out)


if __name__ == "__main__":
    main()
