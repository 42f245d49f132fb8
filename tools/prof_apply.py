"""Per-kernel-class profile of the config-2 64-order apply (and the MSE step) on a caller stream."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2602_20870_b200 as fg, prep
cfg = prep.config2()
cache = fg.PowerCache(cfg.f, cfg.l, memory_budget=8 << 30)
stream = torch.cuda.Stream()
if "--own" not in sys.argv:
    cache.set_stream(stream.cuda_stream)
lib = fg.lib()
al = np.ascontiguousarray(cfg.alphas, dtype=np.float64); A = len(al)
x = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda()
y = torch.empty((A, cfg.b, cfg.n), dtype=torch.complex128, device="cuda")
def app():
    fg._check(lib.fgfrft_apply_dev(cache.handle, al.ctypes.data, A, 0, 0, x.data_ptr(), cfg.b, y.data_ptr()))
for _ in range(3):
    app()
torch.cuda.synchronize()
fg.profile_enable(True); fg.profile_read(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
t0 = time.perf_counter()
for _ in range(5):
    app()
e1.record(stream)
torch.cuda.synchronize()
print("wall ms/apply", (time.perf_counter() - t0) / 5 * 1e3, "event ms", e0.elapsed_time(e1) / 5)
print(fg.profile_read(True))
