import numpy as np, sys
sys.path.insert(0, '.')
import oracle
from paper_2405_12866_b200 import inputs as I, qfs
p = I.make_problem("c3", init="R", s=8)
ctx = qfs.Context(p.n, p.pairs)
ctx.set_samples(p.x, p.y, p.xv, p.yv)
gt = ctx.trace_sweeps(p.init, 16, 5)
ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, 16, 5)
d = np.abs(gt["sigma"] - ot["sigma"])
idx = np.argwhere(d > 1e-9)
print("bad", len(idx), idx[:10], gt["sigma"][tuple(idx[0])] if len(idx) else None, ot["sigma"][tuple(idx[0])] if len(idx) else None)
