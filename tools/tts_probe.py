"""Time-to-solution probe: instantiate a W instance twice (cold, warm) per path."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import build, inputs as I, qfs
build.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
p = I.make_problem(cfg, init="W")
for path in ("auto", "streamed"):
    ctx = qfs.Context(p.n, p.pairs); ctx.set_path(path); ctx.set_samples(p.x, p.y, p.xv, p.yv)
    prm = dict(p.params, max_iter=300)
    ctx.instantiate(p.init, dict(prm, max_iter=2))
    for rep in range(3):
        t0 = time.perf_counter(); g, r, w = ctx.instantiate(p.init, prm); dt = time.perf_counter() - t0
        print(cfg, path, rep, "%.4f s" % dt, r[w]["sweeps"], r[w]["term"], "launches", ctx.launch_count(), flush=True)
    ctx.close()
