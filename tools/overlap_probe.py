"""Probe: does running the apply of two column halves on two streams (two handles) overlap the
SpMM of one half with the C2R passes of the other?  Prints ms per full 4096-column step."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2004_11610_b200 import inputs as I, xc
cfg = I.CONFIGS["c5"]
x, _, _ = xc.gauss_rule(cfg.kind, cfg.N)
T1 = xc.Transform(cfg.kind, x, cfg.eps)
T2 = xc.Transform(cfg.kind, x, cfg.eps)
B = 4096
X = torch.from_numpy(I.config_rhs(cfg, B=B)).cuda()
Y = torch.empty_like(X)
X1, X2 = X[:, :B // 2].contiguous(), X[:, B // 2:].contiguous()
Y1, Y2 = torch.empty_like(X1), torch.empty_like(X2)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
T1.graphs(False); T2.graphs(False)
def one():
    T1.apply(X, out=Y)
def two(stagger):
    with torch.cuda.stream(s1):
        T1.apply(X1, out=Y1)
    if stagger:
        e = torch.cuda.Event(); e.record(s1); s2.wait_event(e)
    with torch.cuda.stream(s2):
        T2.apply(X2, out=Y2)
for name, f in (("single", one), ("two-streams", lambda: two(False)), ("two-staggered", lambda: two(True))):
    for _ in range(3): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10): f()
    torch.cuda.synchronize()
    print(name, (time.perf_counter() - t0) / 10 * 1e3, "ms")
