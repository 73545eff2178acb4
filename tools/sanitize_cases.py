#!/usr/bin/env python
"""Small cases of every kernel family (for compute-sanitizer where it is open; on the B200 pool it is
closed, so with XC_WS_GUARD=1 every case also checks the workspace guard zones, xc_debug_guards):
Legendre c1 (B = 1) and a reduced c3 (block chain, split-K, tail, forked streams), both directions
of Laguerre, the exp and spectral-Laguerre kinds (complex SpMM, C2C), the 2D block method, the
Appendix-A precompute, the global threshold, degenerate sizes N = 2..64, the host-buffer pipeline,
an attached workspace.  Product path only (no oracle); prints one line per case."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_11610_b200 import inputs as I  # noqa: E402
from paper_2004_11610_b200 import xc  # noqa: E402


GUARD = os.environ.get("XC_WS_GUARD") == "1"


def check_guards(name, T):
    if GUARD:
        bad, checked = T.debug_guards()
        assert checked > 0 and bad == 0, (name, bad, checked)


def run(name, T, X, dirs=(xc.XC_DIR_A,)):
    for d in dirs:
        for path_B in (X.shape[1], 1):   # the batch, then one column (other grid shapes)
            Y = T.apply(torch.from_numpy(np.ascontiguousarray(X[:, :path_B])).cuda(), d)
            torch.cuda.synchronize()
            assert torch.isfinite(Y).all(), name
    check_guards(name, T)
    print("ok", name, flush=True)


def main():
    x, w, wt = xc.gauss_rule(xc.XC_JACOBI, 512)
    run("c1", xc.Transform(xc.XC_JACOBI, x, 1e-12), I.rhs(512, 1, 0))
    run("c1_tiled", xc.Transform(xc.XC_JACOBI, x, 1e-12, apply_path=1), I.rhs(512, 33, 0))
    x2 = I.cos_nodes(4096, 1)
    run("c2", xc.Transform(xc.XC_COS, x2, 1e-10), I.rhs(4096, 64, 1))
    run("c2_small", xc.Transform(xc.XC_COS, x2, 1e-10, apply_path=2), I.rhs(4096, 70, 1))
    x, w, wt = xc.gauss_rule(xc.XC_JACOBI, 2048, 0.5, -0.3)
    T = xc.Transform(xc.XC_JACOBI, x, 1e-12, alpha=0.5, beta=-0.3, dirs=3, weights=w)
    run("c3_reduced", T, I.rhs(2048, 96, 2), (1, 2))
    s = torch.cuda.Stream()
    ws = torch.empty(T.workspace_bytes(96) // 8 + 64, dtype=torch.float64, device="cuda")
    T.attach_workspace(s.cuda_stream, ws)
    Y = T.apply(torch.from_numpy(I.rhs(2048, 96, 3)).cuda(), stream=s.cuda_stream)
    torch.cuda.synchronize()
    check_guards("attached_workspace", T)
    print("ok attached_workspace", flush=True)
    Xh = I.rhs(2048, 130, 4)
    Yh = T.apply_host(Xh)
    assert np.isfinite(Yh).all()
    check_guards("host_pipeline", T)
    print("ok host_pipeline", flush=True)
    x, w, wt = xc.gauss_rule(xc.XC_LAGUERRE, 1024)
    run("laguerre_both", xc.Transform(xc.XC_LAGUERRE, x, 1e-11, dirs=3, weights=wt), I.rhs(1024, 40, 3), (1, 2))
    t = I.exp_nodes(96, 2)
    T = xc.Transform(xc.XC_EXP, t, 1e-12, dirs=3, weights=np.ones(96))
    Xc = I.complex_rhs(96, 3, 2)
    run("exp_small", T, np.concatenate([Xc.real, Xc.imag]), (1, 2))
    cfg = I.CONFIGS["c7"]
    T = xc.Transform(xc.XC_LAGSPEC, I.lagspec_freqs(cfg.N, cfg.T), cfg.eps, eta=cfg.eta, n_rows=cfg.M)
    F = I.config_rhs(cfg, 8)
    run("lagspec_c7", T, np.concatenate([F.real, F.imag]))
    cfg = I.CONFIGS["c8"]
    run("lag2d_small", xc.Transform(xc.XC_LAG2D, I.lag2d_grid(512, cfg.eta), 1e-10), I.rhs(512, 17, 8))
    run("cos_appA", xc.Transform(xc.XC_COS, I.cos_nodes(3000, 1), 1e-10, trig_precompute=1), I.rhs(3000, 9, 1))
    x, w, wt = xc.gauss_rule(xc.XC_JACOBI, 900)
    run("global_threshold", xc.Transform(xc.XC_JACOBI, x, 1e-12, thresh_mode=1), I.rhs(900, 20, 5))
    for N in (2, 3, 7, 33, 64):
        x, w, wt = xc.gauss_rule(xc.XC_JACOBI, N)
        run(f"degenerate_N{N}", xc.Transform(xc.XC_JACOBI, x, 1e-12, dirs=3, weights=w), I.rhs(N, 5, N), (1, 2))
    print("all cases done", flush=True)


if __name__ == "__main__":
    main()
