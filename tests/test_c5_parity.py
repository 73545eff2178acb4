"""c5 (BASELINE configs[4]: Legendre N = 65536, B = 4096, eps = 1e-12) at the 1e-12 bar.

The oracle's c5 reference comes from tools/make_c5_oracle.py (calls only oracle/; ~10 min on
8 cores, so it is cached under oracle_cache/ and its arrays' SHA-256 are committed in
tests/golden/c5_oracle_manifest.json): the oracle's Gauss-Legendre nodes, its compressed operator
(block chain, double-double entries, Kaiser window, unitary DFT, per-node threshold), its compressed
apply (Alg. 2 block form) and its dense product on the 16 check columns
b = 256 i of the seeded batch.  The GPU runs at the bench's launch configuration (all 4096 columns
in one xc_apply); the sampled columns are compared.
"""
import functools
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2004_11610_b200 import inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CACHE = os.path.join(ROOT, "oracle_cache", "c5_oracle.npz")
MANIFEST = os.path.join(ROOT, "tests", "golden", "c5_oracle_manifest.json")
C5 = I.CONFIGS["c5"]


def _digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest() + f":{a.dtype.str}:{a.shape}"


@functools.lru_cache(maxsize=1)
def _cache():
    if not os.path.exists(CACHE):
        pytest.skip("oracle cache missing: run tools/make_c5_oracle.py (about 10 min on 8 cores)")
    man = json.load(open(MANIFEST))
    z = dict(np.load(CACHE))
    for k, d in man["sha256"].items():   # the cache is the committed script's output
        assert _digest(z[k]) == d, f"oracle cache array {k} does not match the manifest"
    return z, man


def test_c5_oracle_cache_pins():
    """The cached oracle result against the plain definition (CPU): the oracle's compressed apply
    is within 10 eps of its dense product on the 16 columns, its chain is the oracle planner's
    (Table 1 shape tested elsewhere), and its nodes are a Gauss-Legendre rule (sum w = 2,
    symmetric nodes: x_k = -x_{N-1-k})."""
    z, man = _cache()
    assert O.rel_l2_cols(z["Y_alg"], z["Y_dense"]).max() <= 10 * C5.eps
    plan = O.make_plan(O.Kind(C5.kind), C5.N, C5.eps)
    assert [b.L for b in plan.blocks] == list(z["L"]) and plan.tail == int(z["tail"][0])
    x, w = z["x"], z["w"]
    assert abs(w.sum() - 2.0) <= 1e-13 and np.abs(x + x[::-1]).max() <= 4e-16
    X = I.config_rhs(C5)[:, z["cols"]]
    assert np.array_equal(X, z["X"])   # the seeded batch's check columns


def _xc():
    from paper_2004_11610_b200 import xc
    return xc


@functools.lru_cache(maxsize=1)
def _X_gpu():
    import torch
    return torch.from_numpy(I.config_rhs(C5)).cuda()


def _bands(z):
    return [(z[f"start{i}"], z[f"len{i}"], z[f"vals{i}"]) for i in range(len(z["L"]))]


@pytest.mark.gpu
def test_c5_same_operator_parity():
    """The oracle's own c5 operator (its kept entries, xc_build_from_bands) through the GPU
    computation stage at B = 4096: <= 1e-12 vs the oracle's compressed apply, <= 10 eps vs dense."""
    xc = _xc()
    z, _ = _cache()
    T = xc.Transform.from_bands(xc.XC_JACOBI, z["x"], C5.eps, _bands(z))
    Y = T.apply(_X_gpu())[:, z["cols"]].cpu().numpy()
    T.close()
    e = O.rel_l2_cols(Y, z["Y_alg"])
    assert e.max() <= 1e-12, e
    assert O.rel_l2_cols(Y, z["Y_dense"]).max() <= 10 * C5.eps


@pytest.mark.gpu
def test_c5_gpu_built_parity():
    """The GPU precompute of c5 (double-double entries, FFT, threshold on the GPU) from the oracle's
    nodes, applied at B = 4096: <= 1e-12 vs the oracle's compressed apply, <= 10 eps vs dense."""
    xc = _xc()
    z, _ = _cache()
    T = xc.Transform(xc.XC_JACOBI, z["x"], C5.eps)
    assert [b["L"] for b in T.blocks()] == list(z["L"])
    Y = T.apply(_X_gpu())[:, z["cols"]].cpu().numpy()
    e = O.rel_l2_cols(Y, z["Y_alg"])
    assert e.max() <= 1e-12, e
    assert O.rel_l2_cols(Y, z["Y_dense"]).max() <= 10 * C5.eps
    # kept sets at 40 sampled nodes per block (both ends included): equal except at threshold
    # ties (|S| within 1e-9 relative of tau = eps1 max |S_k|); values to 1e-13 of the node max
    rng = np.random.default_rng(5)
    ks = np.unique(np.r_[0, 1, C5.N // 2, C5.N - 2, C5.N - 1, rng.integers(0, C5.N, 35)])
    for i in range(len(z["L"])):
        st, ln, v = z[f"start{i}"], z[f"len{i}"], z[f"vals{i}"]
        off = np.concatenate([[0], np.cumsum(ln.astype(np.int64))])
        H = int(z["L"][i]) // 2 + 1
        for k in ks:
            o = np.zeros(H, np.complex128)
            o[st[k]:st[k] + ln[k]] = v[off[k]:off[k + 1]]
            g = T.node_spectrum(i, int(k))
            m = max(np.abs(o).max(), np.abs(g).max())
            tau = C5.eps * m
            only = (o != 0) != (g != 0)
            assert np.all(np.abs(np.abs(np.where(o != 0, o, g))[only] - tau) <= 1e-9 * tau), (i, k)
            both = (o != 0) & (g != 0)
            assert np.abs(g[both] - o[both]).max(initial=0.0) <= 1e-13 * m, (i, k)
    T.close()


@pytest.mark.gpu
def test_c5_gpu_gauss_rule_vs_oracle():
    """The product's Gauss-Legendre rule at N = 65536 (the nodes bench.py builds c5 from) equals
    the oracle's to 4 ulp (weights to 1e-12 relative)."""
    xc = _xc()
    z, _ = _cache()
    x, w, _ = xc.gauss_rule(xc.XC_JACOBI, C5.N)
    assert np.all(np.abs(x - z["x"]) <= 4 * np.spacing(np.abs(z["x"])) + 1e-300)
    np.testing.assert_allclose(w, z["w"], rtol=1e-12)
