"""Precompute time of the trig kinds: direct (entries + FFT per node) vs Appendix A (R-22).

Usage: python tools/appa_build_time.py  (one GPU).  Prints one JSON line per case."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_11610_b200 import inputs as I  # noqa: E402
from paper_2004_11610_b200 import xc  # noqa: E402


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        T = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        info = T.block_info(0)
        T.close()
    return min(ts), info


cases = [("c2_cos", xc.XC_COS, 4096, 1e-10), ("cos_65536", xc.XC_COS, 65536, 1e-12),
         ("cos_262144", xc.XC_COS, 262144, 1e-12), ("c6_exp", xc.XC_EXP, 4096, 1e-10),
         ("exp_131072", xc.XC_EXP, 131072, 1e-12)]
xc.Transform(xc.XC_COS, I.cos_nodes(64, 0), 1e-10).close()  # context / module load
for name, kind, N, eps in cases:
    nodes = I.cos_nodes(N, 1) if kind == xc.XC_COS else I.exp_nodes(N, 6)
    td, bd = timed(lambda: xc.Transform(kind, nodes, eps))
    ta, ba = timed(lambda: xc.Transform(kind, nodes, eps, trig_precompute=1))
    print(json.dumps({"case": name, "N": N, "L": bd["L"], "eps": eps, "direct_s": round(td, 4),
                      "appA_s": round(ta, 4), "speedup": round(td / ta, 2), "nnz_direct": bd["nnz"],
                      "nnz_appA": ba["nnz"], "q_taps": ba["q_taps"]}), flush=True)
