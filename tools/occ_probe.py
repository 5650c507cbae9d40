import time, sys
sys.path.insert(0, '/root/repo')
from paper_2405_12866_b200 import build, inputs as I, qfs
build.build()
for cfg in ("c3",):
    for s in (64, 30, 12, 5, 2, 1):
        p = I.make_problem(cfg, init="W", s=s)
        ctx = qfs.Context(p.n, p.pairs); ctx.set_samples(p.x, p.y, p.xv, p.yv)
        t0 = time.perf_counter(); ctx.trace_sweeps(p.init, 16, 1, env=False); t1 = time.perf_counter()
        ctx.trace_sweeps(p.init, 16, 1, env=False); t2 = time.perf_counter()
        print(cfg, s, "first %.3f s  second %.3f s" % (t1 - t0, t2 - t1), flush=True)
