"""Per-kernel-class profile (fgfrft_profile_*) of one config's MSE step: python tools/prof_step.py 3"""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2602_20870_b200 as fg, prep
which = sys.argv[1] if len(sys.argv) > 1 else "3"
cfg = {"2": prep.config2, "3": prep.config3, "4": prep.config4}[which]()
cache = fg.PowerCache(cfg.f, cfg.l, memory_budget=140 << 30)
lib = fg.lib()
al = np.ascontiguousarray(cfg.alphas, dtype=np.float64); A = len(al)
x = torch.from_numpy(np.ascontiguousarray(cfg.x.T)).cuda()
xc = torch.from_numpy(np.ascontiguousarray(cfg.x_clean.T)).cuda()
loss = torch.empty(A, dtype=torch.float64, device="cuda"); dl = torch.empty_like(loss)
def step():
    fg._check(lib.fgfrft_mse_step_dev(cache.handle, al.ctypes.data, A, x.data_ptr(), xc.data_ptr(), cfg.b, None,
                                      loss.data_ptr(), dl.data_ptr()))
for _ in range(3):
    step()
torch.cuda.synchronize()
fg.profile_enable(True); fg.profile_read(True)
t0 = time.perf_counter()
for _ in range(5):
    step()
torch.cuda.synchronize()
print("C" + which, "wall ms/step", (time.perf_counter() - t0) / 5 * 1e3)
for k, (ms, cnt) in fg.profile_read(True).items():
    if cnt:
        print(f"  {k:12s} {ms / 5:8.3f} ms/step  launches/step {cnt / 5:.1f}")
