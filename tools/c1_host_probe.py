"""c1 (N = 512, B = 1): per-apply cost through Transform.apply vs a bare ctypes xc_apply call vs a
torch CUDA graph of K applies (GPU-only time).  Measurement helper, not a test."""
import ctypes
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_11610_b200 import inputs as I  # noqa: E402
from paper_2004_11610_b200 import xc  # noqa: E402

cfg = I.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
sys.path.insert(0, ROOT)
import bench  # noqa: E402
x, wt = bench._nodes(cfg, 0)
T = xc.Transform(cfg.kind, x, cfg.eps, alpha=cfg.alpha, beta=cfg.beta, weights=wt, device=0, eta=cfg.eta,
                 n_rows=cfg.M, eps2=cfg.eps2 if cfg.eps2 != 1e-2 else 0.0)
B = cfg.B
X = torch.from_numpy(I.config_rhs(cfg, B)).cuda()
if X.dim() == 1:
    X = X[:, None]
Y = torch.empty((T.rows(xc.XC_DIR_A)[1], B), dtype=torch.float64, device="cuda")
T.reserve(B)
st = torch.cuda.current_stream()
K = 2000


def timed(fn, k=K):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(k):
        fn()
    e1.record(st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3, (t1 - t0) / k * 1e6


print("Transform.apply          gpu %.2f us/apply  host %.2f us/call" % timed(lambda: T.apply(X, xc.XC_DIR_A, out=Y)))
lib, h = T._lib, T._h
args = (h, xc.XC_DIR_A, ctypes.c_void_p(X.data_ptr()), X.stride(0), ctypes.c_void_p(Y.data_ptr()), Y.stride(0), B,
        ctypes.c_void_p(st.cuda_stream))
print("bare ctypes xc_apply     gpu %.2f us/apply  host %.2f us/call" % timed(lambda: lib.xc_apply(*args)))
