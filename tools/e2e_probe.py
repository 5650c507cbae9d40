import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2405_12866_b200 import inputs as I, qfs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = I.make_problem(cfg, init="R")
ctx = qfs.Context(p.n, p.pairs)
ctx.set_samples(p.x, p.y, p.xv, p.yv)
m = p.m_init
prm = dict(dist_tol=-1.0, diff_tol_r=1e-3, plateau_window=0, min_iter=6, max_iter=1, m_init=m, overtrain_ratio=1e300, beta=0.0, stop_on_first=0)
g = p.init
hx = torch.from_numpy(p.x).pin_memory(); hy = torch.from_numpy(p.y).pin_memory()
hxv = torch.from_numpy(p.xv).pin_memory(); hyv = torch.from_numpy(p.yv).pin_memory()
def q():
    ctx.set_samples_async_host_ptr(hx.shape[0], hx.data_ptr(), hy.data_ptr(), hxv.shape[0], hxv.data_ptr(), hyv.data_ptr())
for _ in range(3):
    q(); g, _, _ = ctx.instantiate(g, prm)
steps = 20
# a) full e2e
torch.cuda.synchronize(); t0 = time.perf_counter(); q()
for s in range(steps):
    if s + 1 < steps: q()
    g, _, _ = ctx.instantiate(g, prm)
ta = (time.perf_counter() - t0) / steps
# b) no sample upload
t0 = time.perf_counter()
for s in range(steps):
    g, _, _ = ctx.instantiate(g, prm)
tb = (time.perf_counter() - t0) / steps
# c) one call with max_iter = steps
t0 = time.perf_counter()
g, _, _ = ctx.instantiate(g, dict(prm, max_iter=steps))
tc = (time.perf_counter() - t0) / steps
# d) synchronous set_samples each step (no overlap)
t0 = time.perf_counter()
for s in range(steps):
    ctx.set_samples_host_ptr(hx.shape[0], hx.data_ptr(), hy.data_ptr(), hxv.shape[0], hxv.data_ptr(), hyv.data_ptr())
    g, _, _ = ctx.instantiate(g, prm)
td = (time.perf_counter() - t0) / steps
print(f"{cfg}: ms/step e2e-async {ta*1e3:.3f}  no-upload {tb*1e3:.3f}  one-call {tc*1e3:.3f}  sync-upload {td*1e3:.3f}")
# e) queued upload, copy finished before the call (consume cost without concurrent DMA)
tot = 0.0
for s in range(steps):
    q()
    torch.cuda.synchronize()
    time.sleep(0.002)
    t0 = time.perf_counter()
    g, _, _ = ctx.instantiate(g, prm)
    tot += time.perf_counter() - t0
te = tot / steps
print(f"{cfg}: ms/call with the staged copy already done {te*1e3:.3f} (consume on the critical path only)")
