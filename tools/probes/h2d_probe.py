"""Host->device copy rates on the GPU box: one pinned 134 MB copy (config 3's X + Xc per step) as
one copy, as chunks on one stream, and split over 2 / 4 concurrent streams (copy engines)."""
import json
import subprocess

import torch

nb = 2 * 4096 * 1024 * 16
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
h.fill_(1)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(ns, chunks):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(streams[0])
    for s in streams[1:ns]:
        s.wait_event(ev0)
    per = nb // chunks
    for c in range(chunks):
        s = streams[c % ns]
        with torch.cuda.stream(s):
            d[c * per:(c + 1) * per].copy_(h[c * per:(c + 1) * per], non_blocking=True)
    for s in streams[1:ns]:
        e = torch.cuda.Event()
        e.record(s)
        streams[0].wait_event(e)
    ev1.record(streams[0])
    ev1.synchronize()
    return ev0.elapsed_time(ev1)


out = {}
for ns, ch in [(1, 1), (1, 4), (2, 2), (2, 8), (4, 4), (4, 16)]:
    ts = sorted(run(ns, ch) for _ in range(7))
    out[f"streams{ns}_chunks{ch}"] = {"ms": ts[3], "gbs": nb / (ts[3] * 1e-3) / 1e9}
try:
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-600:]
except Exception as ex:
    out["topo"] = str(ex)
print(json.dumps(out, indent=1))
