"""Time the c5 precompute (xc_build_compressed) phases: run once to warm up, then once timed."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2004_11610_b200 import inputs as I, xc
cfg = I.CONFIGS["c5"]
t0 = time.perf_counter()
x, _, _ = xc.gauss_rule(cfg.kind, cfg.N)
print("gauss", time.perf_counter() - t0, flush=True)
for rep in range(2):
    t0 = time.perf_counter()
    T = xc.Transform(cfg.kind, x, cfg.eps)
    torch.cuda.synchronize()
    print("build", rep, time.perf_counter() - t0, flush=True)
    T.close()
