#!/usr/bin/env python
"""Record the c5 parity numbers (GPU vs the oracle's cached c5 reference) as JSON on stdout:
max relative L2 over the 16 check columns for the same-operator and the GPU-built operator."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2004_11610_b200 import inputs as I  # noqa: E402
from paper_2004_11610_b200 import xc  # noqa: E402

c = I.CONFIGS["c5"]
z = np.load(os.path.join(ROOT, "oracle_cache", "c5_oracle.npz"))
X = torch.from_numpy(I.config_rhs(c)).cuda()
out = {"config": c.name, "B": c.B, "cols": z["cols"].tolist()}
bands = [(z[f"start{i}"], z[f"len{i}"], z[f"vals{i}"]) for i in range(len(z["L"]))]
for name, T in (("same_operator", xc.Transform.from_bands(xc.XC_JACOBI, z["x"], c.eps, bands)),
                ("gpu_built", xc.Transform(xc.XC_JACOBI, z["x"], c.eps))):
    Y = T.apply(X)[:, z["cols"]].cpu().numpy()
    out[name] = {"rel_l2_vs_oracle_compressed": float(O.rel_l2_cols(Y, z["Y_alg"]).max()),
                 "rel_l2_vs_dense": float(O.rel_l2_cols(Y, z["Y_dense"]).max()), "nnz": T.info()["nnz"]}
    T.close()
xg, wg, _ = xc.gauss_rule(xc.XC_JACOBI, c.N)
out["gauss_rule_max_ulp"] = float(np.max(np.abs(xg - z["x"]) / np.spacing(np.abs(z["x"]))))
import json  # noqa: E402
print(json.dumps(out))
