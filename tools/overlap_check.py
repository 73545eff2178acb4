#!/usr/bin/env python
"""Bitwise check of an apply-schedule switch (e.g. XC_OVERLAP) against the default schedule:
applies the config's batch in this process (schedule from the environment) and in a child
process without any XC_* switch, and compares the results."""
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_11610_b200 import inputs as I  # noqa: E402
from paper_2004_11610_b200 import xc  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
c = I.CONFIGS[cfg]
x, w, wt = xc.gauss_rule(c.kind, c.N, c.alpha, c.beta)
T = xc.Transform(c.kind, x, c.eps, alpha=c.alpha, beta=c.beta)
X = torch.from_numpy(I.config_rhs(c)).cuda()
Y = T.apply(X).cpu().numpy()
if os.environ.get("OV_CHILD"):
    np.save(sys.argv[2], Y)
    sys.exit(0)
out = os.path.join(ROOT, "gpurun_out", f"ov_{os.getpid()}.npy")
env = {k: v for k, v in os.environ.items() if not k.startswith("XC_")}
env["OV_CHILD"] = "1"
subprocess.check_call([sys.executable, os.path.abspath(__file__), cfg, out], env=env)
Y0 = np.load(out)
os.unlink(out)
print(cfg, {k: v for k, v in os.environ.items() if k.startswith("XC_")}, "bitwise equal:", np.array_equal(Y, Y0),
      "max abs diff", float(np.abs(Y - Y0).max()))
