"""C5 (n=14, K=300, M=64): GPU trace vs oracle for the first sweep(s), full size."""
import sys, time
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle
from paper_2405_12866_b200 import build, qfs, inputs as I
build.build()
p = I.make_problem("c5", init="W")
ctx = qfs.Context(p.n, p.pairs)
ctx.set_samples(p.x, p.y, p.xv, p.yv)
gt = ctx.trace_sweeps(p.init, 64, 3, env=False, gates=False)
print("gpu cost", gt["cost"][:, 0])
t = time.time()
ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, 64, 1, threads=1)
print("oracle cost", ot["cost"][:, 0], "%.1fs" % (time.time() - t))
print("sigma max rel diff sweep0", np.abs(gt["sigma"][0] - ot["sigma"][0]).max() / np.abs(ot["sigma"][0]).max())
