"""Extreme-parameter parity checks (bug hunting; not part of the suite): eps 1e-14 / 1e-6,
Jacobi alpha, beta near -1 and large, big ragged batches, both directions, host buffers."""
import copy, sys
import numpy as np, torch
sys.path.insert(0, ".")
import oracle as O
from paper_2004_11610_b200 import inputs as I, xc

def check(name, kind, kx, x, eps, B, wat=False, host=False, **extra):
    N = len(x)
    w = 0.5 + np.random.default_rng(1).random(N) if wat else None
    T = xc.Transform(kx, x, eps, dirs=xc.XC_DIR_A | (xc.XC_DIR_WAT if wat else 0), weights=w, **extra)
    plan = O.make_plan(kind, N, eps)
    op = O.compress(plan, x)
    X = I.rhs(N, B, 3)
    d = xc.XC_DIR_WAT if wat else xc.XC_DIR_A
    Y = T.apply_host(X, d) if host else T.apply(torch.from_numpy(X).cuda(), d).cpu().numpy()
    ref = O.apply_input_axis(op, X, w) if wat else O.apply_output_axis(op, X)
    err = O.rel_l2_cols(Y, ref).max()
    if err > 2e-12:
        errs = [err]
        for f in (1 - 1e-6, 1 + 1e-6):
            p2 = copy.deepcopy(plan); p2.eps1 = plan.eps1 * f
            o2 = O.compress(p2, x)
            errs.append(O.rel_l2_cols(Y, O.apply_input_axis(o2, X, w) if wat else O.apply_output_axis(o2, X)).max())
        err = min(errs)
    dense = (w[:, None] * O.dense_apply_t(kind, x, X[:, :4])) if wat else O.dense_apply(kind, x, X[:, :4])
    ed = O.rel_l2_cols(Y[:, :4], dense).max()
    ok = err <= 2e-12
    print(("ok  " if ok else "FAIL"), name, "N", N, "B", B, "eps", eps, "wat", wat, "host", host,
          "vs oracle %.2e" % err, "vs dense %.2e (10eps %.0e)" % (ed, 10 * eps), flush=True)
    T.close()

for eps in (1e-14, 1e-6):
    check("legendre", O.Kind(O.KIND_JACOBI), xc.XC_JACOBI, O.gauss_rule(O.Kind(O.KIND_JACOBI), 1500)[0], eps, 40)
    check("cos", O.Kind(O.KIND_COS), xc.XC_COS, I.cos_nodes(2000, 4), eps, 70, wat=True)
for a, b in ((-0.95, -0.95), (-0.9, 3.0), (4.0, 4.0)):
    k = O.Kind(O.KIND_JACOBI, a, b)
    check(f"jacobi({a},{b})", k, xc.XC_JACOBI, O.gauss_rule(k, 1200)[0], 1e-12, 33, wat=True, alpha=a, beta=b)
check("legendre big ragged host", O.Kind(O.KIND_JACOBI), xc.XC_JACOBI, O.gauss_rule(O.Kind(O.KIND_JACOBI), 3000)[0],
      1e-12, 1037, host=True)
check("laguerre 1e-13", O.Kind(O.KIND_LAGUERRE), xc.XC_LAGUERRE, O.gauss_rule(O.Kind(O.KIND_LAGUERRE), 900)[0],
      1e-13, 17, wat=True)
