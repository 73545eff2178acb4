#!/usr/bin/env python
"""Build the oracle's c5 reference (BASELINE configs[4]: Legendre N = 65536, eps = 1e-12) and cache it.

Calls only ``oracle/`` (and the seeded input generator ``paper_2004_11610_b200.inputs``): the
oracle's Gauss-Legendre rule, its block chain, its compressed operator (entries in double-double,
Kaiser window, unitary DFT, per-node threshold: P:104-110), its
compressed apply (Alg. 2 block form) and its dense direct product on the
16 check columns b = 256 i of the seeded c5 batch.  Nothing here comes from the CUDA path.

    python tools/make_c5_oracle.py            # writes oracle_cache/c5_oracle.npz (~3-5 min, 8 cores)

The cache is git-ignored (about 200 MB) but not gpurun-ignored, so it travels to the GPU box with
the snapshot; ``tests/golden/c5_oracle_manifest.json`` (committed) holds the SHA-256 of every array
so the GPU test can check that the cache is this script's output.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2004_11610_b200 import inputs as I  # noqa: E402

OUT = os.path.join(ROOT, "oracle_cache", "c5_oracle.npz")
MANIFEST = os.path.join(ROOT, "tests", "golden", "c5_oracle_manifest.json")
COLS = 256 * np.arange(16)


def runs_of(S):
    """One run per node (start = first kept bin, len = last - first + 1) with the dropped interior
    bins as explicit zeros: the node-band layout xc_build_from_bands takes (glue, no arithmetic)."""
    S = S.tocsr()
    S.sort_indices()
    N = S.shape[0]
    ip, idx = S.indptr, S.indices
    cnt = np.diff(ip)
    has = cnt > 0
    start = np.zeros(N, np.int64)
    last = np.zeros(N, np.int64)
    start[has] = idx[ip[:-1][has]]
    last[has] = idx[ip[1:][has] - 1]
    ln = np.where(has, last - start + 1, 0)
    off = np.concatenate([[0], np.cumsum(ln)])
    vals = np.zeros(int(off[-1]), np.complex128)
    row = np.repeat(np.arange(N), cnt)
    vals[off[row] + (idx - start[row])] = S.data
    return start.astype(np.int32), ln.astype(np.int32), vals


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest() + f":{a.dtype.str}:{a.shape}"


def main():
    c = I.CONFIGS["c5"]
    kind = O.Kind(c.kind, c.alpha, c.beta)
    t0 = time.time()
    x, w, _ = O.gauss_rule(kind, c.N)
    t_nodes = time.time() - t0
    plan = O.make_plan(kind, c.N, c.eps)
    t0 = time.time()
    op = O.compress(plan, x, node_chunk=1024)
    t_build = time.time() - t0
    X = np.ascontiguousarray(I.config_rhs(c)[:, COLS])
    t0 = time.time()
    Ya = O.apply_output_axis(op, X)
    t_apply = time.time() - t0
    t0 = time.time()
    Yd = O.dense_apply(kind, x, X)
    t_dense = time.time() - t0
    arrays = {"x": x, "w": w, "cols": COLS, "X": X, "Y_alg": Ya, "Y_dense": Yd,
              "L": np.array([b.L for b in plan.blocks]), "m_off": np.array([b.m_off for b in plan.blocks]),
              "keep_lo": np.array([b.keep_lo for b in plan.blocks]),
              "keep_hi": np.array([b.keep_hi for b in plan.blocks]),
              "tail": np.array([plan.tail]), "zeta": np.array([plan.zeta])}
    for i, S in enumerate(op.S):
        st, ln, v = runs_of(S)
        arrays[f"start{i}"], arrays[f"len{i}"], arrays[f"vals{i}"] = st, ln, v
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez(OUT, **arrays)
    man = {"config": c.name, "N": c.N, "eps": c.eps, "cols": COLS.tolist(), "nnz": O.nnz(op),
           "rel_l2_alg_vs_dense": float(O.rel_l2_cols(Ya, Yd).max()),
           "seconds": {"gauss_rule": round(t_nodes, 1), "compress": round(t_build, 1),
                       "compressed_apply_16_cols": round(t_apply, 2), "dense_16_cols": round(t_dense, 1)},
           "threads": os.cpu_count(), "script": "tools/make_c5_oracle.py",
           "sha256": {k: digest(v) for k, v in sorted(arrays.items())}}
    with open(MANIFEST, "w") as f:
        json.dump(man, f, indent=1)
    print(json.dumps({k: man[k] for k in ("nnz", "rel_l2_alg_vs_dense", "seconds")}))


if __name__ == "__main__":
    main()
