"""Warm-start strength vs convergence on C5 (GPU instantiate, real stopping rules)."""
import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2405_12866_b200 import build, qfs, inputs as I
build.build()
for eps in (0.1, 0.05, 0.02):
    p = I.make_problem("c5", init="W", eps=eps)
    ctx = qfs.Context(p.n, p.pairs)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    t = time.time()
    g, r, w = ctx.instantiate(p.init, dict(p.params, max_iter=400))
    print(eps, r[w], "%.2fs" % (time.time() - t), flush=True)
