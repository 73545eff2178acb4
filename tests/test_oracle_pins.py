"""Pins for the CPU oracle: every part checked against something other than itself.

Each test names the paper passage (P:<line> of /root/reference/PAPER.md) or the
mathematical fact it uses.  Independent references: mpmath (arbitrary precision
special functions), scipy (DCT-II, Gauss rules at small N, i0e+brentq), closed
forms, and brute force at tiny N.  Runs on CPU (-m "not gpu").
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest
import scipy.fft
import scipy.optimize
import scipy.special

import oracle as O
from paper_2004_11610_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden")
LEG = O.Kind(O.KIND_JACOBI, 0.0, 0.0)
JAC = O.Kind(O.KIND_JACOBI, 0.5, -0.3)
CHEB = O.Kind(O.KIND_JACOBI, -0.5, -0.5)
LAG = O.Kind(O.KIND_LAGUERRE)
COS = O.Kind(O.KIND_COS)


# --------------------------------------------------------------------------- Bessel / Kaiser
@pytest.mark.parametrize("x", [0.0, 0.5, 3.0, 16.1, 25.56, 30.25, 50.0])
def test_bessel_i0_i1_vs_mpmath(x):
    """I0, I1 against mpmath's arbitrary-precision Bessel functions."""
    mp.mp.dps = 40
    assert abs(O.bessel_i0(x) / float(mp.besseli(0, x)) - 1) < 2e-15
    if x > 0:
        assert abs(O.bessel_i1(x) / float(mp.besseli(1, x)) - 1) < 2e-15


def test_kaiser_closed_forms():
    """w_0 = w_N = 1/I0(zeta); w_{N/2} = 1; symmetric; zeta = 0 gives ones."""
    z = 25.5
    w = O.kaiser(z, 100)
    assert w[0] == pytest.approx(1 / float(mp.besseli(0, z)), rel=1e-15)
    assert w[-1] == w[0]
    assert w[50] == 1.0
    np.testing.assert_array_equal(w, w[::-1])
    np.testing.assert_array_equal(O.kaiser(0.0, 37), np.ones(38))
    assert np.all(np.diff(w[:51]) > 0)


@pytest.mark.parametrize("eps1", [1e-6, 1e-10, 1e-11, 1e-12, 1e-15])
def test_zeta_solves_its_equation(eps1):
    """1/I0(zeta) = eps1; checked with mpmath and against scipy brentq on i0e."""
    z = O.solve_zeta(eps1)
    mp.mp.dps = 40
    assert abs(1 / float(mp.besseli(0, z)) / eps1 - 1) < 1e-12
    zb = scipy.optimize.brentq(lambda t: math.log(scipy.special.i0e(t)) + t + math.log(eps1), 1, 100,
                               xtol=1e-15)
    assert z == pytest.approx(zb, abs=1e-10)


@pytest.mark.parametrize("span,eps2,two", [(512, 1e-2, False), (16384, 1e-2, False), (4096, 1e-2, True),
                                           (1000, 1e-3, False), (777, 1e-4, True)])
def test_s_rule_definition(span, eps2, two):
    """Reading R-2 of P:184: s is the smallest s >= 1 with w^{zeta,L-1}_s >= eps2."""
    z = O.solve_zeta(1e-12)
    s = O.minimal_s(z, span, eps2, two)
    L = span + (2 * s if two else s)
    assert O.kaiser_at(z, L - 1, s) >= eps2
    if s > 1:
        Lm = span + (2 * (s - 1) if two else s - 1)
        assert O.kaiser_at(z, Lm - 1, s - 1) < eps2
    # monotone: a larger eps2 needs at least as many extra components
    assert O.minimal_s(z, span, eps2 * 3, two) >= s


def test_smooth5_brute_force():
    """R-9 (P:450 'locally optimal FFT size'): smallest even 2,3,5-smooth >= n."""
    def smooth(m):
        for p in (2, 3, 5):
            while m % p == 0:
                m //= p
        return m == 1
    for n in list(range(1, 400)) + [86399, 21601, 65537 + 20000]:
        m = O.smooth5_even_at_least(n)
        assert m >= n and m % 2 == 0 and smooth(m)
        assert not any(smooth(k) and k % 2 == 0 for k in range(n, m))


def test_block_chain_shape_vs_table1():
    """P:491-518 (Table 1): first-block order N_1/N within 5 % and block count within 1,
    for the minimal-s chain of reading R-2 (only the chain shape is pinned, C-9)."""
    g = json.load(open(os.path.join(GOLD, "table1_block_orders.json")))
    for col, e1, e2 in (("1e-6", g["eps1_1e-6"], g["eps2_1e-6"]), ("1e-10", g["eps1_1e-10"], g["eps2_1e-10"])):
        z = O.solve_zeta(e1)
        for Ns, row in g["rows"].items():
            N = int(Ns)
            if N < 1024:
                continue
            e, chain = N, []
            while e > 32:
                s = O.minimal_s(z, e, e2, False)
                chain.append(e + s)
                e = s
            paper = row[col]
            assert abs(chain[0] / paper[0] - 1) < 0.05, (N, col, chain, paper)
            assert abs(len(chain) - len(paper)) <= 1, (N, col, chain, paper)


def test_chain_is_self_consistent():
    """R-8: block i keeps positions [s_i, s_{i-1}); L_i = s_{i-1} + s_i; tail <= cutoff."""
    for cfg in ("c1", "c3", "c4", "c5"):
        c = I.CONFIGS[cfg]
        kind = O.Kind(c.kind, c.alpha, c.beta)
        p = O.make_plan(kind, c.N, c.eps)
        e = c.N
        for b in p.blocks:
            assert b.keep_hi == e and b.L == b.keep_hi + b.keep_lo and b.m_off == 0
            assert O.kaiser_at(p.zeta, b.L - 1, b.keep_lo) >= p.eps2
            e = b.keep_lo
        assert p.tail == e <= 32


# --------------------------------------------------------------------------- DFT convention
def test_unitary_dft_convention():
    """Eq. (1): unitary forward DFT with e^{-2 pi i jk/N}; F F* = I.
    The oracle's DFT step is numpy's FFT with norm='ortho'; pin the convention."""
    L = 30
    e0 = np.zeros(L)
    e0[0] = 1
    np.testing.assert_allclose(np.fft.rfft(e0, norm="ortho"), np.full(L // 2 + 1, 1 / math.sqrt(L)), atol=1e-16)
    x = np.random.default_rng(0).standard_normal(L)
    direct = np.array([sum(x[j] * np.exp(-2j * np.pi * j * k / L) for j in range(L)) for k in range(L // 2 + 1)])
    np.testing.assert_allclose(np.fft.rfft(x, norm="ortho"), direct / math.sqrt(L), atol=1e-14)
    np.testing.assert_allclose(np.fft.irfft(np.fft.rfft(x, norm="ortho"), n=L, norm="ortho"), x, atol=1e-15)


def test_convolution_theorem_appendix_a():
    """(A.1) P:641-649: F(X . Y) = F X * F Y with the 1/sqrt(N) circular convolution."""
    N = 24
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(N), rng.standard_normal(N)
    F = lambda v: np.fft.fft(v, norm="ortho")
    fx, fy = F(x), F(y)
    conv = np.array([sum(fx[m] * fy[(n - m) % N] for m in range(N)) for n in range(N)]) / math.sqrt(N)
    np.testing.assert_allclose(F(x * y), conv, atol=1e-14)


def _closed_form_exp(theta, L):
    """(y3) P:671: (1/sqrt(N)) sum_j e^{i j theta} w^{jk} = (e^{iN theta} - 1)/(e^{i theta} w^k - 1)/sqrt(N)."""
    wk = np.exp(-2j * np.pi * np.arange(L) / L)
    return (np.exp(1j * L * theta) - 1) / (np.exp(1j * theta) * wk - 1) / math.sqrt(L)


def test_trig_row_spectrum_closed_form():
    """Appendix A: with the window switched off (zeta = 0), the oracle's
    per-node spectrum of a cos row equals the closed form
    y^cos_k(theta) = (y^exp_k(theta) + y^exp_k(-theta)) / 2 built from (y3),
    and the corrected (y1) of reading R-12."""
    L = 48
    plan = O.Plan(COS, 40, 1e-12, 1e-2, 0.0)
    blk = O.Block(L, 0, 0, L)
    t = np.array([0.1234, 0.4321, 0.77])
    S = O.node_spectra(plan, blk, t)                     # (3, L/2+1)
    for i, tk in enumerate(t):
        th = math.pi * tk
        y = 0.5 * (_closed_form_exp(th, L) + _closed_form_exp(-th, L))
        np.testing.assert_allclose(S[i], y[:L // 2 + 1], atol=1e-14)
        wk = np.exp(-2j * np.pi * np.arange(L) / L)
        A = (math.cos(L * th) - 1) * math.cos(th) + math.sin(th) * math.sin(L * th)
        y1 = (wk * A - (math.cos(L * th) - 1)) / (wk ** 2 - 2 * wk * math.cos(th) + 1) / math.sqrt(L)
        np.testing.assert_allclose(S[i], y1[:L // 2 + 1], atol=1e-13)


# --------------------------------------------------------------------------- special functions
def test_legendre_closed_values():
    """P_2(1/2) = -1/8; P_j(1) = 1, P_j(-1) = (-1)^j; orthonormal p_j = sqrt((2j+1)/2) P_j (R-4)."""
    E = O.entries(LEG, np.array([0.5, 1.0, -1.0]), 0, 200)
    j = np.arange(200)
    nrm = np.sqrt((2 * j + 1) / 2)
    assert E[0, 2] == pytest.approx(-0.125 * math.sqrt(2.5), rel=1e-15)
    np.testing.assert_allclose(E[1], nrm, rtol=1e-15)
    np.testing.assert_allclose(E[2], nrm * (-1.0) ** j, rtol=1e-15)


def test_chebyshev_is_jacobi_minus_half():
    """Jacobi(-1/2,-1/2) orthonormal = sqrt(2/pi) cos(j theta), 1/sqrt(pi) for j = 0."""
    th = np.array([0.3, 1.1, 2.9])
    E = O.entries(CHEB, np.cos(th), 0, 3000)
    j = np.arange(3000)
    ref = math.sqrt(2 / math.pi) * np.cos(np.outer(th, j))
    ref[:, 0] = 1 / math.sqrt(math.pi)
    np.testing.assert_allclose(E, ref, atol=2e-15)


@pytest.mark.parametrize("a,b", [(0.0, 0.0), (0.5, -0.3), (1.0, 1.0), (-0.7, 2.5)])
def test_jacobi_vs_mpmath(a, b):
    """Orthonormal Jacobi p_n (chi read as the squared norm, R-4) vs mpmath.jacobi,
    normalised by h_n = 2^{a+b+1}/(2n+a+b+1) G(n+a+1)G(n+b+1)/(G(n+a+b+1) n!), up to n = 3000."""
    mp.mp.dps = 50
    xs = [-0.999, -0.31, 0.0123, 0.77, 0.9999]
    ns = [0, 1, 2, 7, 100, 1234, 2999]
    E = O.entries(O.Kind(O.KIND_JACOBI, a, b), np.array(xs), 0, 3000)
    for i, x in enumerate(xs):
        for n in ns:
            h = mp.mpf(2) ** (a + b + 1) / (2 * n + a + b + 1) * mp.gamma(n + a + 1) * mp.gamma(n + b + 1) / (
                mp.gamma(n + a + b + 1) * mp.factorial(n))
            ref = float(mp.jacobi(n, a, b, mp.mpf(x)) / mp.sqrt(h))
            assert abs(E[i, n] - ref) <= 4e-15 * max(1.0, abs(ref)), (x, n, E[i, n], ref)


def test_laguerre_vs_mpmath():
    """l_n(t) = e^{-t/2} L_n(t) vs mpmath.laguerre, including t far beyond fp64's exp range."""
    mp.mp.dps = 60
    xs = [0.0, 0.5, 2.0, 37.0, 900.0, 3000.0, 20000.0]
    E = O.entries(LAG, np.array(xs), 0, 2001)
    assert E[2, 0] == pytest.approx(math.exp(-1), rel=1e-15)
    assert E[2, 1] == pytest.approx(-math.exp(-1), rel=1e-15)   # l_1(2) = -e^{-1}
    np.testing.assert_array_equal(E[0], np.ones(2001))          # l_n(0) = 1
    for i, x in enumerate(xs):
        for n in (0, 1, 5, 150, 1000, 2000):
            ref = mp.exp(-mp.mpf(x) / 2) * mp.laguerre(n, 0, mp.mpf(x))
            r = float(ref)
            if abs(r) < 1e-300:
                assert abs(E[i, n]) < 1e-290
            else:
                assert abs(E[i, n] - r) <= 1e-14 * abs(r) + 1e-300, (x, n, E[i, n], r)


def test_cos_entries_exact_reduction():
    """cos(pi m t) (P:68 with theta = pi t) vs mpmath at large m, negative m."""
    mp.mp.dps = 50
    t = np.array([0.1, 0.333333333333, 0.9999999])
    E = O.entries(COS, t, 0, 20000, m_off=-5000)
    for i, tk in enumerate(t):
        for m in (-5000, -1, 0, 3, 9999, 14999):
            ref = float(mp.cos(mp.pi * m * mp.mpf(tk)))
            assert abs(E[i, m + 5000] - ref) < 3e-16


# --------------------------------------------------------------------------- Gauss rules
def test_gauss_small_closed_forms():
    """N = 2: Gauss-Legendre +-1/sqrt(3), w = 1; Gauss-Laguerre 2 -+ sqrt(2), w = (2 +- sqrt 2)/4."""
    x, w, _ = O.gauss_rule(LEG, 2)
    np.testing.assert_allclose(x, [-1 / math.sqrt(3), 1 / math.sqrt(3)], rtol=1e-15)
    np.testing.assert_allclose(w, [1, 1], rtol=1e-15)
    x, w, wt = O.gauss_rule(LAG, 2)
    np.testing.assert_allclose(x, [2 - math.sqrt(2), 2 + math.sqrt(2)], rtol=1e-15)
    np.testing.assert_allclose(w, [(2 + math.sqrt(2)) / 4, (2 - math.sqrt(2)) / 4], rtol=1e-15)
    np.testing.assert_allclose(wt, w * np.exp(x), rtol=1e-14)


@pytest.mark.parametrize("kind", [LEG, JAC, CHEB, O.Kind(O.KIND_JACOBI, 2.0, 0.5)])
def test_gauss_jacobi_identities(kind):
    """sum w = 2^{a+b+1} G(a+1)G(b+1)/G(a+b+2); sum x = N(b-a)/(2N+a+b); p_N(x_k) = 0 (mpmath);
    exact on monomials up to 2N-1; nodes match scipy at small N."""
    a, b = kind.alpha, kind.beta
    for N in (5, 64, 700):
        x, w, _ = O.gauss_rule(kind, N)
        mu0 = 2 ** (a + b + 1) * math.gamma(a + 1) * math.gamma(b + 1) / math.gamma(a + b + 2)
        assert w.sum() == pytest.approx(mu0, rel=1e-13)
        assert x.sum() == pytest.approx(N * (b - a) / (2 * N + a + b), abs=1e-12)
        if N <= 64:
            xs, ws = scipy.special.roots_jacobi(N, a, b)
            np.testing.assert_allclose(x, xs, atol=1e-14)
            np.testing.assert_allclose(w, ws, rtol=1e-11)   # scipy itself is ~1e-12
            mp.mp.dps = 40
            for deg in range(2 * N):
                ex = mp.quad(lambda t: (1 - t) ** a * (1 + t) ** b * t ** deg, [-1, 0, 1])
                assert float(np.dot(w, x ** deg)) == pytest.approx(float(ex), abs=1e-13)
    mp.mp.dps = 40
    N = 700
    x, _, _ = O.gauss_rule(kind, N)
    for k in (0, 1, N // 2, N - 1):
        v = mp.jacobi(N, a, b, mp.mpf(x[k]))
        d = mp.diff(lambda t: mp.jacobi(N, a, b, t), mp.mpf(x[k]))
        assert abs(float(v / d)) <= 2 * np.spacing(abs(x[k])) + 1e-300


def test_gauss_laguerre_identities():
    """Gauss-Laguerre: sum w = 1, sum x = N^2, L_N(x_k) = 0 (mpmath), wt = 1/sum_j l_j(x_k)^2."""
    N = 300
    x, w, wt = O.gauss_rule(LAG, N)
    assert w.sum() == pytest.approx(1.0, rel=1e-13)
    assert x.sum() == pytest.approx(N * N, rel=1e-14)
    mp.mp.dps = 60
    for k in (0, 1, N // 2, N - 1):
        v = mp.laguerre(N, 0, mp.mpf(x[k]))
        d = mp.diff(lambda t: mp.laguerre(N, 0, t), mp.mpf(x[k]))
        assert abs(float(v / d)) <= 2 * np.spacing(x[k])
        s = sum((mp.exp(-mp.mpf(x[k]) / 2) * mp.laguerre(j, 0, mp.mpf(x[k]))) ** 2 for j in range(N))
        assert wt[k] == pytest.approx(float(1 / s), rel=1e-13)


@pytest.mark.parametrize("kind,N", [(LEG, 512), (JAC, 1024), (LAG, 512)])
def test_discrete_orthogonality(kind, N):
    """Gauss quadrature makes the transform orthogonal: A diag(w) A^T = I_N
    (Laguerre functions with wt = w e^x)."""
    x, w, wt = O.gauss_rule(kind, N)
    E = O.entries(kind, x, 0, N)                 # E[k, j] = phi_j(x_k)
    G = E.T @ (wt[:, None] * E)
    assert np.abs(G - np.eye(N)).max() < 5e-13


# --------------------------------------------------------------------------- dense product
def test_dense_vs_mpmath_matrix():
    """The plain definition Y = A X against a matrix built from mpmath entries (N = 24)."""
    mp.mp.dps = 30
    N = 24
    x, _, _ = O.gauss_rule(LEG, N)
    A = np.array([[float(mp.sqrt((2 * j + 1) / mp.mpf(2)) * mp.legendre(j, mp.mpf(xk))) for xk in x]
                  for j in range(N)])
    X = I.rhs(N, 3, 7)
    np.testing.assert_allclose(O.dense_apply(LEG, x, X), A @ X, atol=1e-13)
    np.testing.assert_allclose(O.dense_apply_t(LEG, x, X), A.T @ X, atol=1e-13)


def test_dense_cos_is_dct2():
    """at t_k = (k + 1/2)/N the cos transform is the DCT-II: y_j = (1/2) dct2(x)_j (scipy)."""
    N = 300
    t = (np.arange(N) + 0.5) / N
    X = I.rhs(N, 4, 3)
    np.testing.assert_allclose(O.dense_apply(COS, t, X), 0.5 * scipy.fft.dct(X, type=2, axis=0), atol=1e-12)


def test_dense_chebyshev_gauss_is_dct2():
    """Jacobi(-1/2,-1/2) at Gauss-Chebyshev nodes: y_j = sqrt(2/pi) (1/2) dct2(x reversed)_j, j >= 1;
    y_0 = sum x / sqrt(pi); weights pi/N."""
    N = 256
    x, w, _ = O.gauss_rule(CHEB, N)
    np.testing.assert_allclose(w, np.full(N, math.pi / N), rtol=1e-11)
    X = I.rhs(N, 2, 4)
    Y = O.dense_apply(CHEB, x, X)
    d = 0.5 * scipy.fft.dct(X[::-1], type=2, axis=0)   # ascending x = descending theta
    np.testing.assert_allclose(Y[1:], math.sqrt(2 / math.pi) * d[1:], atol=1e-12)
    np.testing.assert_allclose(Y[0], X.sum(axis=0) / math.sqrt(math.pi), atol=1e-12)


# --------------------------------------------------------------------------- compressed algorithm
def test_threshold_soundness():
    """P:106 per-node threshold (R-3): every dropped |S| < eps1 * node max, every kept one >=."""
    x, _, _ = O.gauss_rule(JAC, 256)
    plan = O.make_plan(JAC, 256, 1e-10)
    blk = plan.blocks[0]
    S = O.node_spectra(plan, blk, x)
    K = O.threshold(S, plan.eps1)
    m = np.abs(S).max(axis=1, keepdims=True)
    assert np.all(np.abs(S[K == 0]) < (plan.eps1 * m * np.ones_like(S))[K == 0] * (1 + 1e-12))
    assert np.all(np.abs(K[K != 0]) >= (plan.eps1 * m * np.ones_like(S))[K != 0] * (1 - 1e-12))
    # Hermitian symmetry of real rows: bins 0 and L/2 real
    assert np.all(S[:, 0].imag == 0) and np.all(S[:, -1].imag == 0)


def test_spectrum_brute_force_tiny():
    """Brute force (N = 16): the windowed-row spectrum equals the naive Eq.-(1) sum in mpmath."""
    mp.mp.dps = 30
    N = 16
    x, _, _ = O.gauss_rule(LEG, N)
    plan = O.make_plan(LEG, N, 1e-6, dense_cutoff=2)
    blk = plan.blocks[0]
    S = O.node_spectra(plan, blk, x)
    w = O.kaiser(plan.zeta, blk.L - 1)
    for k in (0, 5, 15):
        for q in range(blk.H):
            ref = sum(w[m] * mp.sqrt((2 * m + 1) / mp.mpf(2)) * mp.legendre(m, mp.mpf(x[k])) *
                      mp.expj(-2 * mp.pi * m * q / blk.L) for m in range(blk.L)) / mp.sqrt(blk.L)
            assert abs(complex(S[k, q]) - complex(ref)) < 1e-14


@pytest.mark.parametrize("kind,N", [(LEG, 48), (JAC, 64), (LAG, 40), (COS, 50)])
def test_keep_all_is_exact(kind, N):
    """eps1 threshold -> 0 keeps every entry: both computation stages reproduce the dense
    product (the extended identities comp1/comp2) to rounding x 1/eps2."""
    if kind.kind == O.KIND_COS:
        x = I.cos_nodes(N, 9)
        wt = None
    else:
        x, _, wt = O.gauss_rule(kind, N)
    plan = O.make_plan(kind, N, 1e-12, dense_cutoff=8)
    plan.eps1 = 0.0                            # keep all (threshold only; zeta stays)
    op = O.compress(plan, x)
    X = I.rhs(N, 3, 11)
    err = O.rel_l2_cols(O.apply_output_axis(op, X), O.dense_apply(kind, x, X))
    assert err.max() < 1e-13
    Yt = O.apply_input_axis(op, X)
    err = O.rel_l2_cols(Yt, O.dense_apply_t(kind, x, X))
    assert err.max() < 1e-13


def test_compressed_cos_vs_dct2():
    """P:74 + Alg. 2: the compressed non-uniform cos transform at DCT-II nodes meets 10 eps vs scipy."""
    N = 512
    t = (np.arange(N) + 0.5) / N
    plan = O.make_plan(COS, N, 1e-10)
    op = O.compress(plan, t)
    X = I.rhs(N, 4, 6)
    ref = 0.5 * scipy.fft.dct(X, type=2, axis=0)
    assert O.rel_l2_cols(O.apply_output_axis(op, X), ref).max() < 1e-9


@pytest.mark.parametrize("cfg,N", [("c1", 512), ("c2", 1024), ("c3", 1024), ("c4", 512)])
def test_compressed_error_within_10eps(cfg, N):
    """Calibration (parity unpinned by the paper, which states only 'accuracy ~ eps1/eps2'):
    the oracle's compressed apply meets BASELINE's 10*eps bar against the dense product."""
    c = I.CONFIGS[cfg]
    kind = O.Kind(c.kind, c.alpha, c.beta)
    if c.kind == O.KIND_COS:
        x = I.cos_nodes(N, c.seed)
    else:
        x, _, wt = O.gauss_rule(kind, N)
    plan = O.make_plan(kind, N, c.eps)
    op = O.compress(plan, x)
    X = I.rhs(N, 8, c.seed)
    err = O.rel_l2_cols(O.apply_output_axis(op, X), O.dense_apply(kind, x, X))
    assert err.max() < 10 * c.eps, err


def test_laguerre_round_trip():
    """C-15: with Gauss-Laguerre nodes, backward = diag(wt) A^T and forward = A are inverse
    (Gauss exactness); the compressed pair reproduces C to ~eps."""
    N = 384
    x, _, wt = O.gauss_rule(LAG, N)
    plan = O.make_plan(LAG, N, 1e-11)
    op = O.compress(plan, x)
    C = I.laguerre_coeffs(N, 4, 3)
    Xf = O.apply_input_axis(op, C, wt)                   # backward (values at nodes)
    Xd = wt[:, None] * O.dense_apply_t(LAG, x, C)
    assert O.rel_l2_cols(Xf, Xd).max() < 1e-10
    C2 = O.apply_output_axis(op, Xf)                     # forward
    assert O.rel_l2_cols(C2, C).max() < 1e-9


# --------------------------------------------------------------------------- kind EXP (NEXT-3)
EXPK = O.Kind(O.KIND_EXP)


def test_exp_entries_vs_mpmath():
    """phi_m(t) = e^{i pi m t}, exactly reduced (m may be negative): vs mpmath."""
    mp.mp.dps = 30
    t = np.array([0.0, 0.3, 1.0, 1.37, 1.999])
    E = O.entries(EXPK, t, -40, 60)
    for k, tk in enumerate(t):
        for m in (-40, -1, 0, 7, 59):
            ref = mp.expj(mp.pi * m * mp.mpf(tk))
            assert abs(complex(E[k, m + 40]) - complex(ref)) < 2e-16


def test_exp_row_spectrum_is_y3():
    """Appendix A (y3): with the window off the oracle's spectrum of an exp row is the
    closed form (e^{iL theta} - 1) / (e^{i theta} w^q - 1) / sqrt(L), all L bins (complex rows)."""
    L = 40
    plan = O.Plan(EXPK, 30, 1e-12, 1e-2, 0.0)
    blk = O.Block(L, 0, 0, L)
    t = np.array([0.11, 0.73, 1.41])
    S = O.node_spectra(plan, blk, t)
    assert S.shape == (3, L)
    for i, tk in enumerate(t):
        np.testing.assert_allclose(S[i], _closed_form_exp(math.pi * tk, L), atol=1e-14)


def test_exp_dense_uniform_nodes_is_inverse_dft():
    """At t_k = 2k/N the exp transform is the DFT matrix: A X = N ifft(X) (numpy)."""
    N = 96
    t = 2.0 * np.arange(N) / N
    X = I.rhs(N, 3, 4) + 1j * I.rhs(N, 3, 5)
    np.testing.assert_allclose(O.dense_apply(EXPK, t, X), N * np.fft.ifft(X, axis=0), atol=1e-11)


def test_exp_compressed_uniform_nodes_vs_ifft():
    """Alg. 2 with complex rows at uniform nodes meets 10 eps against numpy's inverse DFT."""
    N = 256
    t = 2.0 * np.arange(N) / N
    op = O.compress(O.make_plan(EXPK, N, 1e-10), t)
    X = I.rhs(N, 4, 7) + 1j * I.rhs(N, 4, 8)
    ref = N * np.fft.ifft(X, axis=0)
    assert O.rel_l2_cols(O.apply_output_axis(op, X), ref).max() < 1e-9


def test_exp_keep_all_and_cos_consistency():
    """Keep-all (eps1 -> 0) reproduces the dense complex product; and for t in [0,1] and real X
    the real part of the exp transform is the cos transform (Re e^{i pi j t} = cos pi j t)."""
    N = 60
    t = np.sort(np.random.default_rng(3).random(N) * 2.0)
    plan = O.make_plan(EXPK, N, 1e-12)
    plan.eps1 = 0.0
    op = O.compress(plan, t)
    X = I.rhs(N, 2, 1) + 1j * I.rhs(N, 2, 2)
    assert O.rel_l2_cols(O.apply_output_axis(op, X), O.dense_apply(EXPK, t, X)).max() < 1e-13
    tc = I.cos_nodes(N, 4)
    Xr = I.rhs(N, 2, 3)
    np.testing.assert_allclose(O.dense_apply(EXPK, tc, Xr).real, O.dense_apply(COS, tc, Xr), atol=1e-12)


def test_exp_input_axis_closed_forms():
    """Input axis of the exp kind (Alg. 1 with complex rows): at uniform nodes A^T C = N ifft(C)
    (A symmetric there); keep-all reproduces the dense transpose; compressed meets 10 eps."""
    N = 128
    t = 2.0 * np.arange(N) / N
    C = I.rhs(N, 3, 1) + 1j * I.rhs(N, 3, 2)
    np.testing.assert_allclose(O.dense_apply_t(EXPK, t, C), N * np.fft.ifft(C, axis=0), atol=1e-11)
    op = O.compress(O.make_plan(EXPK, N, 1e-10), t)
    assert O.rel_l2_cols(O.apply_input_axis(op, C), N * np.fft.ifft(C, axis=0)).max() < 1e-9
    tr = np.sort(np.random.default_rng(5).random(60) * 2.0)
    plan = O.make_plan(EXPK, 60, 1e-12)
    plan.eps1 = 0.0
    op = O.compress(plan, tr)
    C2 = I.rhs(60, 2, 3) + 1j * I.rhs(60, 2, 4)
    assert O.rel_l2_cols(O.apply_input_axis(op, C2), O.dense_apply_t(EXPK, tr, C2)).max() < 1e-13


# --------------------------------------------------------------------------- rectangular / LAGSPEC
def test_exp_rectangular_uniform_nodes():
    """Rectangular exp operator (M degrees x N nodes, R-21): at t_k = 2k/N, A[m,k] = e^{2 pi i mk/N}
    is periodic in m, so A X = N ifft(X)[m mod N] and A^T C = N ifft(sum of C's rows folded mod N)."""
    N = 128
    t = 2.0 * np.arange(N) / N
    X = I.rhs(N, 3, 4) + 1j * I.rhs(N, 3, 5)
    for M in (77, 200):
        ref = (N * np.fft.ifft(X, axis=0))[np.arange(M) % N]
        np.testing.assert_allclose(O.dense_apply(EXPK, t, X, M=M), ref, atol=1e-11)
        op = O.compress(O.make_plan(EXPK, N, 1e-10, M=M), t)
        assert op.plan.blocks[0].keep_hi - op.plan.blocks[0].keep_lo == M
        assert O.rel_l2_cols(O.apply_output_axis(op, X), ref).max() < 1e-9
        C = I.rhs(M, 3, 6) + 1j * I.rhs(M, 3, 7)
        Cf = np.zeros((N, 3), dtype=np.complex128)
        np.add.at(Cf, np.arange(M) % N, C)
        reft = N * np.fft.ifft(Cf, axis=0)
        np.testing.assert_allclose(O.dense_apply_t(EXPK, t, C), reft, atol=1e-10)
        assert O.rel_l2_cols(O.apply_input_axis(op, C), reft).max() < 1e-9


def _lagk(eta):
    return O.Kind(O.KIND_LAGSPEC, eta=eta)


def test_lagspec_entries_vs_mpmath_power_form():
    """C^T[m,j] = (-eta/2 - i k_j)^m / (eta/2 - i k_j)^(m+1) (Eq. main_formula2) in 40-digit
    arithmetic, including m < 0 (the left extra components of the trig form)."""
    mp.mp.dps = 40
    eta = 2500.0
    k = I.lagspec_freqs(501, 4.0)[[0, 1, 7, 250, 500]]
    E = O.entries(_lagk(eta), k, -300, 700)
    for j, kj in enumerate(k):
        for m in (-300, -1, 0, 1, 5, 345, 699):
            ref = mp.mpc(-eta / 2, -kj) ** m / mp.mpc(eta / 2, -kj) ** (m + 1)
            assert abs(complex(E[j, m + 300]) - complex(ref)) <= 2e-16 * abs(complex(ref))


def test_lagspec_entries_are_laplace_transform_of_laguerre_functions():
    """Where the formula comes from: v_m = int_0^inf e^{i k t} l_m(eta t) dt for one
    Fourier mode, l_m(x) = e^{-x/2} L_m(x).  scipy quad (Fourier weight) with scipy's Laguerre
    polynomials -- an independent route to every entry."""
    import scipy.integrate as si
    eta = 3.0
    k = np.array([0.0, 0.7, 2.5])
    E = O.entries(_lagk(eta), k, 0, 6)
    for j, kj in enumerate(k):
        for m in range(6):
            f = lambda x, m=m: math.exp(-eta * x / 2) * scipy.special.eval_laguerre(m, eta * x)
            # e^{-eta x / 2} < 1e-24 beyond x = 40: the finite interval is the integral
            re = si.quad(lambda x: f(x) * math.cos(kj * x), 0, 40, epsabs=1e-15, epsrel=1e-13, limit=500)[0]
            im = si.quad(lambda x: f(x) * math.sin(kj * x), 0, 40, epsabs=1e-15, epsrel=1e-13, limit=500)[0]
            assert abs(E[j, m] - (re + 1j * im)) < 1e-10


def test_lagspec_phase_reading():
    """Reading R-21 of P:402-405: the ratio r_j = (-eta/2 - i k_j)/(eta/2 - i k_j) is unimodular with
    argument pi + 2 atan(2 k_j / eta), so C^T[m,j] = e^{i m theta_j} / (eta/2 - i k_j): the exp kind at
    t_j = 1 + (2/pi) atan(2 k_j/eta) in (0, 2), ascending in k_j, scaled per node.  The printed
    i exp(-i m phi) / (eta/2 - i k_j) differs from the power form already at m = 0 (factor i)."""
    eta = 2500.0
    k = I.lagspec_freqs(501, 4.0)
    E = O.entries(_lagk(eta), k, -5, 40)
    d = 1.0 / (eta / 2 - 1j * k)
    t = 1.0 + (2.0 / np.pi) * np.arctan(2.0 * k / eta)
    assert np.all(np.diff(t) > 0) and t[0] == 1.0 and t[-1] < 2.0
    Ee = O.entries(EXPK, t, -5, 40) * d[:, None]
    # t_j rounded to fp64: phase error <= pi |m| 2 * 2^-53 (|m| <= 40 here)
    np.testing.assert_allclose(E, Ee, rtol=0, atol=(np.pi * 40 * 2 ** -52 + 4e-16) * np.abs(d).max())
    printed = 1j * d                                        # the printed form at m = 0
    assert np.abs(printed - E[:, 5]).min() > 0.5 * np.abs(d).min()


@pytest.mark.parametrize("eps", [1e-10, 1e-12])
def test_lagspec_fig_lag_row_compressed(eps):
    """The paper's Fig. lag_row operator: C^T is 649 x 501, eta = 2500, k_j = 2 pi j/T,
    T = 4.  Compressed (Alg. 2 with complex rows, both directions) vs the dense C^T within 10 eps;
    keep-all within 1e-13."""
    cfg = I.CONFIGS["c7"]
    k = I.lagspec_freqs(cfg.N, cfg.T)
    kind = _lagk(cfg.eta)
    F = I.config_rhs(cfg, 4)
    op = O.compress(O.make_plan(kind, cfg.N, eps, M=cfg.M), k)
    V = O.apply_output_axis(op, F)
    assert V.shape == (cfg.M, 4)
    assert O.rel_l2_cols(V, O.dense_apply(kind, k, F, M=cfg.M)).max() < 10 * eps
    G = I.complex_rhs(cfg.M, 4, 70, skip_nodes=False)
    Yt = O.apply_input_axis(op, G)
    assert Yt.shape == (cfg.N, 4)
    assert O.rel_l2_cols(Yt, O.dense_apply_t(kind, k, G)).max() < 10 * eps
    plan = O.make_plan(kind, 60, 1e-12, M=85)
    plan.eps1 = 0.0
    kk = I.lagspec_freqs(60, 4.0)
    op0 = O.compress(plan, kk)
    assert O.rel_l2_cols(O.apply_output_axis(op0, F[:60]), O.dense_apply(kind, kk, F[:60], M=85)).max() < 1e-13


# --------------------------------------------------------------------------- Appendix A (NEXT-2)
def test_appA_closed_row_spectra_vs_fft():
    """(y3) / the cos and LAGSPEC rows in closed form = numpy's FFT of the extended rows."""
    L, m_off = 90, -13
    t = np.array([0.0, 0.013, 0.5, 0.77, 1.0])
    for kind, nodes in ((COS, t), (EXPK, np.r_[t, 1.31, 1.999]), (_lagk(40.0), np.array([-30.0, 0.0, 2.5, 90.0]))):
        y = O.row_spectra_closed(kind, nodes, L, m_off)
        E = O.entries(kind, nodes, 0, L, m_off)
        np.testing.assert_allclose(y, np.fft.fft(E, axis=1, norm="ortho"), atol=1e-13 * np.sqrt(L))


def test_appA_closed_form_at_resonance_vs_mpmath():
    """Near and at resonance (theta = 2 pi k / L, where (y3) is 0/0) the Dirichlet form is exact: vs
    the 40-digit geometric sum."""
    mp.mp.dps = 40
    L, m_off = 64, -5
    for t in (2 * 7 / L, 2 * 7 / L + 1e-13, 2 * 7 / L - 3e-16, 2 * 63 / L):
        y = O.row_spectra_closed(EXPK, np.array([t]), L, m_off)[0]
        for k in (6, 7, 8, 63):
            ref = mp.fsum(mp.expj(mp.pi * (p + m_off) * mp.mpf(t)) * mp.expj(-2 * mp.pi * p * k / L) for p in range(L))
            assert abs(complex(y[k]) - complex(ref) / math.sqrt(L)) < 1e-14 * math.sqrt(L), (t, k)


def test_appA_printed_y1_is_conjugated():
    """Reading R-22: the printed (y1) equals the sum with w_N^{-jk}, i.e. the conjugate of the sum it
    names (the oracle uses (y3(theta) + y3(-theta))/2); (y3) as printed is right."""
    N, th = 50, 0.7123
    k = np.arange(N)
    om = np.exp(-2j * np.pi / N)
    c, s_ = np.cos(N * th), np.sin(N * th)
    y1 = om ** k * (((c - 1) * np.cos(th) + np.sin(th) * s_) - (c - 1) * om ** k) / (om ** (2 * k) - 2 * om ** k * np.cos(th) + 1) / np.sqrt(N)
    y = O.row_spectra_closed(COS, np.array([th / np.pi]), N, 0)[0]
    np.testing.assert_allclose(y1, np.conj(y), atol=1e-12)
    assert np.abs(y1 - y).max() > 1.0
    y3 = (np.exp(1j * N * th) - 1) / (np.exp(1j * th) * om ** k - 1) / np.sqrt(N)
    np.testing.assert_allclose(y3, O.row_spectra_closed(EXPK, np.array([th / np.pi]), N, 0)[0], atol=1e-12)


def test_appA_untruncated_convolution_is_the_direct_dft():
    """Eq. (A.1) with every window coefficient (Q = L/2) reproduces the direct windowed DFT
    (node_spectra) -- the convolution theorem with the 1/sqrt(N) of P:645."""
    N, eps = 40, 1e-10
    t = I.cos_nodes(N, 3)
    for kind, nodes in ((COS, t), (EXPK, 2 * t)):
        plan = O.make_plan(kind, N, eps)
        blk = plan.blocks[0]
        xt = np.fft.fft(O.kaiser(plan.zeta, blk.L - 1), norm="ortho")
        S = O.node_spectra_appA(plan, blk, nodes, xt)
        np.testing.assert_allclose(S, O.node_spectra(plan, blk, nodes), atol=1e-13)


def test_appA_window_truncation():
    """Q, x~ and w' (R-22): w' = F* of the kept coefficients, real; |w' - w| <= L^-1/2 sum of the
    dropped |x~_m|; q = 2Q + 1 is small (the paper: "a small number of coefficients")."""
    for eps, L in ((1e-10, 7200), (1e-12, 1080)):
        z = O.solve_zeta(eps)
        Q, xq, wq = O.window_spectrum_truncated(z, L, eps)
        w = O.kaiser(z, L - 1)
        xt = np.fft.fft(w, norm="ortho")
        assert 6 <= Q <= 16
        assert np.count_nonzero(xq) == 2 * Q + 1
        assert np.abs(xt[Q + 1:L - Q]).max() < eps * abs(xt[0]) <= np.abs(xt[Q])
        bound = np.abs(xt[Q + 1:L - Q]).sum() / np.sqrt(L)
        assert np.abs(wq - w).max() <= bound * (1 + 1e-9) + 1e-15


@pytest.mark.parametrize("which", ["cos", "exp", "lagspec"])
def test_appA_operator_meets_10eps(which):
    """The Appendix-A operator (closed-form rows, q-term convolution, w' divided out) meets 10 eps
    against the dense product, with the kept-entry count of the direct build (+-2 %)."""
    eps = 1e-10
    if which == "cos":
        kind, N, M = COS, 1024, None
        nodes = I.cos_nodes(N, 1)
        X = I.rhs(N, 3, 1, skip_cos_nodes=True)
    elif which == "exp":
        kind, N, M = EXPK, 1024, None
        nodes = I.exp_nodes(N, 6)
        X = I.complex_rhs(N, 3, 6)
    else:
        cfg = I.CONFIGS["c7"]
        kind, N, M = _lagk(cfg.eta), cfg.N, cfg.M
        nodes = I.lagspec_freqs(N, cfg.T)
        X = I.config_rhs(cfg, 3)
    plan = O.make_plan(kind, N, eps, M=M)
    opA = O.compress_appA(plan, nodes)
    Y = O.apply_output_axis(opA, X)
    Yd = O.dense_apply(kind, nodes, X, M=M) if M else O.dense_apply(kind, nodes, X)
    assert O.rel_l2_cols(Y, Yd).max() < 10 * eps
    op = O.compress(plan, nodes)
    assert abs(O.nnz(opA)[0] / O.nnz(op)[0] - 1) < 0.02
    if which == "exp":
        C = I.complex_rhs(N, 2, 60, skip_nodes=False)
        assert O.rel_l2_cols(O.apply_input_axis(opA, C), O.dense_apply_t(kind, nodes, C)).max() < 10 * eps


# --------------------------------------------------------------------------- 2D (NEXT-1)
def _plan2d(N, eps, eps2=0.1, cutoff=32):
    return O.make_plan(LAG, N, eps, eps2=eps2, dense_cutoff=cutoff)


def test_2d_spectrum_is_the_two_sided_transform():
    """Eq. (comp_2d): D2 = F W_M D W_N F with the unitary DFT of Eq. (1) on both sides --
    written with explicit DFT matrices on a tiny block."""
    x = I.lag2d_grid(12, 100.0)
    plan = _plan2d(12, 1e-10, cutoff=4)
    op = O.compress_2d(plan, x)
    b = plan.blocks[0]
    E = O.entries(LAG, O.lag2d_nodes_ext(x, b.L), 0, b.L)
    w = O.kaiser(plan.zeta, b.L - 1)
    F = np.exp(-2j * np.pi * np.outer(np.arange(b.L), np.arange(b.L)) / b.L) / np.sqrt(b.L)
    ref = F @ (w[:, None] * E * w[None, :]) @ F
    ref = np.where(np.abs(ref) >= plan.eps1 * np.abs(ref).max(), ref, 0)
    np.testing.assert_allclose(op.D2[0][0].toarray(), ref, atol=1e-13 * np.abs(ref).max())


def test_2d_keep_all_reproduces_the_series_sum():
    """Keep-all (eps1 -> 0): the 2D block method is exact -- W_b^-1 F* D2 F* W_a^-1 = E on every
    block pair and the pairs + tails partition D -- so Y = D C to rounding (vs the dense sum)."""
    N = 200
    x = I.lag2d_grid(N, 100.0)
    plan = _plan2d(N, 1e-12)
    plan.eps1 = 0.0
    C = I.laguerre_coeffs(N, 3, 8)
    Y = O.apply_2d(O.compress_2d(plan, x), C)
    assert O.rel_l2_cols(Y, O.dense_apply_t(LAG, x, C)).max() < 1e-12


@pytest.mark.parametrize("eta", [100.0, 1000.0])
def test_2d_compressed_meets_10eps(eta):
    """Compressed (eps1 = 1e-10, eps2 = 0.1, R-23) vs the dense series sum within 10 eps."""
    N, eps = 1024, 1e-10
    x = I.lag2d_grid(N, eta)
    op = O.compress_2d(_plan2d(N, eps), x)
    C = I.rhs(N, 3, 8)
    assert O.rel_l2_cols(O.apply_2d(op, C), O.dense_apply_t(LAG, x, C)).max() < 10 * eps


def test_2d_compression_paper_claims():
    """Fig. lag_matrix2: the 2D compression keeps fewer entries than the 1D one along
    either axis; 'compressed up to 3-4 % of the initial number of elements' -- at N = 4096,
    eta = 100 the block-pair scheme keeps < 5 % of N^2 (the Hermitian half stored)."""
    N, eps = 1024, 1e-10
    x = I.lag2d_grid(N, 100.0)
    plan = _plan2d(N, eps)
    op = O.compress_2d(plan, x)
    n2 = O.nnz_2d(op, half=False)
    D = O.entries(LAG, x, 0, N)                                  # D[i, j] = l_j(x_i)
    for A in (D, D.T):                                           # 1D along the degree / time axis
        w = O.kaiser(O.solve_zeta(eps), N - 1)
        S = np.fft.fft(A * w[None, :], axis=1, norm="ortho")
        kept = np.abs(S) >= eps * np.abs(S).max()
        assert n2 < kept.sum()
    N = 4096
    op = O.compress_2d(_plan2d(N, eps), I.lag2d_grid(N, 100.0))
    assert O.nnz_2d(op) / N ** 2 < 0.05


def test_2d_all_tail_is_the_direct_sum():
    """N <= the cutoff: no block pair, the 2D method is the direct method exactly."""
    N = 20
    x = I.lag2d_grid(N, 100.0)
    op = O.compress_2d(_plan2d(N, 1e-12), x)
    assert not op.D2
    C = I.rhs(N, 2, 3)
    np.testing.assert_allclose(O.apply_2d(op, C), O.dense_apply_t(LAG, x, C), rtol=0, atol=1e-12)


# --------------------------------------------------------------------------- c5-range pins
# c5 evaluates degrees up to L_1 - 1 = 86399 (block 1 of N = 65536), where recurrence error grows
# (P:475).  These pins reach those degrees with references that are not the oracle's recurrence:
# closed forms at x = 0, +-1 and mpmath's hypergeometric series next to +-1 (where it converges).

C5_DEGREES = (20000, 65534, 65535, 86398, 86399)


def _h_jacobi(n, a, b):
    """Squared norm of P_n^(a,b) (chi_n, read as the squared norm, R-4)."""
    return mp.mpf(2) ** (a + b + 1) / (2 * n + a + b + 1) * mp.exp(
        mp.loggamma(n + a + 1) + mp.loggamma(n + b + 1) - mp.loggamma(n + a + b + 1) - mp.loggamma(n + 1))


@pytest.mark.parametrize("kind", [LEG, JAC], ids=["legendre", "jacobi_0.5_-0.3"])
def test_jacobi_c5_degrees_closed_forms(kind):
    """p_n(1) = C(n+a, n)/sqrt(h_n), p_n(-1) = (-1)^n C(n+b, n)/sqrt(h_n) at the c5 degrees; for
    Legendre also p_n(0) = sqrt((2n+1)/2) (-1)^{n/2} C(n, n/2)/2^n (n even), 0 (n odd).  Relative
    1e-14 of the row scale |p_n(1)|."""
    mp.mp.dps = 40
    a, b = kind.alpha, kind.beta
    E = O.entries(kind, np.array([-1.0, 0.0, 1.0]), 0, max(C5_DEGREES) + 1)
    for n in C5_DEGREES:
        sh = mp.sqrt(_h_jacobi(n, a, b))
        p1 = float(mp.binomial(n + a, n) / sh)
        pm1 = float((-1) ** n * mp.binomial(n + b, n) / sh)
        assert abs(E[2, n] - p1) <= 1e-14 * abs(p1), (n, E[2, n], p1)
        assert abs(E[0, n] - pm1) <= 1e-14 * abs(p1), (n, E[0, n], pm1)
        if a == 0.0 and b == 0.0:
            p0 = 0.0 if n % 2 else float(mp.sqrt(mp.mpf(2 * n + 1) / 2) * (-1) ** (n // 2) * mp.binomial(n, n // 2)
                                         / mp.mpf(2) ** n)
            assert abs(E[1, n] - p0) <= 1e-14 * abs(p1), (n, E[1, n], p0)


@pytest.mark.parametrize("kind", [LEG, JAC], ids=["legendre", "jacobi_0.5_-0.3"])
def test_jacobi_c5_degrees_near_the_ends_vs_mpmath(kind):
    """Next to x = +-1 (the outermost Gauss nodes of N = 65536 and two more) the hypergeometric series
    of P_n^(a,b) converges fast even at n = 86399: mpmath (40 digits) vs the oracle's double-double
    recurrence at the c5 degrees, 1e-14 of the row scale.  x -> -x via P_n^(a,b)(-x) = (-1)^n P_n^(b,a)(x)."""
    mp.mp.dps = 40
    a, b = kind.alpha, kind.beta
    th = [2.404825557695773 / 65536.5, 5.520078110286311 / 65536.5, 3e-5]
    xs = [math.cos(t) for t in th]
    x = np.array(sorted([-v for v in xs] + xs))
    E = O.entries(kind, x, 0, max(C5_DEGREES) + 1)
    for n in C5_DEGREES:
        sh = mp.sqrt(_h_jacobi(n, a, b))
        scale = float(mp.binomial(n + a, n) / sh)
        for i, xv in enumerate(x):
            X = mp.mpf(float(xv))
            if xv > 0:
                ref = mp.jacobi(n, a, b, X, maxterms=10 ** 6) / sh
            else:
                ref = (-1) ** n * mp.jacobi(n, b, a, -X, maxterms=10 ** 6) / sh
            assert abs(E[i, n] - float(ref)) <= 1e-14 * scale, (n, xv, E[i, n], float(ref))


def _gauss_rows_orthogonality(x, w, rows, chunk=1024):
    """G = A_S diag(w) A_S^T for the sampled degree rows S (entries in node chunks)."""
    jmax = int(max(rows)) + 1
    G = np.zeros((len(rows), len(rows)))
    for k0 in range(0, x.size, chunk):
        E = O.entries(LEG, x[k0:k0 + chunk], 0, jmax)[:, rows]      # E[k, s] = p_{rows[s]}(x_k)
        G += E.T @ (w[k0:k0 + chunk, None] * E)
    return G


# Bar of the sampled-row orthogonality: N eps.  The Gauss nodes are rounded to fp64 (relative error
# eps), and p_j(x~_k) moves by ~ j |x~_k - x_k| / sqrt(1 - x^2) per node, which leaves
# A diag(w) A^T - I at ~ 0.5 N eps for every row (measured with 80-bit accumulation: 3.7e-13 at
# N = 4096, 9.2e-13 at 16384, 7.5e-12 at 65536 -- growing as N, not the summation).  An fp64
# (not double-double) recurrence misses this bar by two orders (3.6e-10 at N = 16384, SURVEY PR-10).


def test_discrete_orthogonality_sampled_rows_16384():
    """A diag(w) A^T = I on 64 sampled degree rows of the N = 16384 Gauss-Legendre transform
    (both ends of the degree range included), N eps."""
    N = 16384
    x, w, _ = O.gauss_rule(LEG, N)
    rows = np.unique(np.r_[0, 1, N - 2, N - 1, np.random.default_rng(1).integers(0, N, 60)])
    G = _gauss_rows_orthogonality(x, w, rows)
    assert np.abs(G - np.eye(len(rows))).max() <= N * np.finfo(float).eps


def test_discrete_orthogonality_sampled_rows_65536():
    """The same at N = 65536 (c5), with the oracle's Gauss rule from tools/make_c5_oracle.py's cache
    (its N = 65536 Newton solve takes minutes; skipped without the cache)."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle_cache",
                        "c5_oracle.npz")
    if not os.path.exists(path):
        pytest.skip("oracle cache missing: tools/make_c5_oracle.py")
    z = np.load(path)
    x, w = z["x"], z["w"]
    N = x.size
    rows = np.unique(np.r_[0, 1, N - 2, N - 1, np.random.default_rng(2).integers(0, N, 60)])
    G = _gauss_rows_orthogonality(x, w, rows)
    assert np.abs(G - np.eye(len(rows))).max() <= N * np.finfo(float).eps


@pytest.mark.parametrize("L", [720, 2250, 2916])
def test_dft_step_vs_naive_dft(L):
    """The oracle's DFT step (numpy rfft, unitary: Eq. 1) at radix-3/5 block lengths of c1/c3/c5
    against the naive O(L^2) sum in 80-bit arithmetic with exactly reduced twiddle indices
    e^{-2 pi i ((p q) mod L) / L}: relative 1e-14 of the spectrum's max."""
    blk = O.Block(L, 0, L // 4, L)
    plan = O.Plan(LEG, 64, 1e-12, 1e-2, O.solve_zeta(1e-12), [blk], 0)
    x = np.array([-0.93, -0.2, 0.41, 0.999])
    S = O.node_spectra(plan, blk, x)
    w = O.kaiser(plan.zeta, L - 1).astype(np.longdouble)
    E = O.entries(LEG, x, 0, L).astype(np.longdouble) * w[None, :]
    p = np.arange(L, dtype=np.int64)
    H = L // 2 + 1
    pq = (p[:, None] * p[None, :H]) % L
    ang = -2 * np.pi * pq.astype(np.longdouble) / L
    re = E @ np.cos(ang) / np.sqrt(np.longdouble(L))
    im = E @ np.sin(ang) / np.sqrt(np.longdouble(L))
    ref = (re + 1j * im).astype(np.complex128)
    m = np.abs(ref).max(axis=1, keepdims=True)
    assert np.all(np.abs(S - ref) <= 1e-14 * m)


# --------------------------------------------------------------------------- global threshold
def test_global_threshold_soundness_and_subset():
    """thresh_mode = 1, the global threshold of Alg. 1/2 step 1.3: every kept |S| >= eps1 x the
    max over the block's whole matrix, every dropped one below it (max taken here over all nodes at
    once, the oracle takes it in a first pass over node chunks); the kept set is a subset of the
    per-node threshold's (eps1 x a node's max <= eps1 x the block max)."""
    N = 300
    x, _, _ = O.gauss_rule(JAC, N)
    plan = O.make_plan(JAC, N, 1e-10)
    opg = O.compress(plan, x, node_chunk=64, thresh_mode=1)
    opn = O.compress(plan, x, node_chunk=64)
    for blk, Sg, Sn in zip(plan.blocks, opg.S, opn.S):
        S = O.node_spectra(plan, blk, x)
        tau = plan.eps1 * np.abs(S).max()
        G = Sg.toarray()
        assert np.all(np.abs(G[G != 0]) >= tau * (1 - 1e-12))
        assert np.all(np.abs(S[G == 0]) < tau * (1 + 1e-12))
        assert np.all((Sn.toarray() != 0) | (G == 0))          # subset of the per-node kept set
        assert Sg.nnz < Sn.nnz


def test_global_threshold_keep_all_and_error():
    """Global threshold: eps1 -> 0 keeps everything (the dense product to 1e-13, as per node), and at
    eps = 1e-12 the error against the dense product is larger than the per-node threshold's but
    bounded (calibration, SURVEY PR-7: 7.1e-11 vs 2.3e-12 at N = 1024): <= 1000 eps."""
    N = 512
    x, _, _ = O.gauss_rule(JAC, N)
    plan = O.make_plan(JAC, N, 1e-12)
    X = I.rhs(N, 6, 12)
    Yd = O.dense_apply(JAC, x, X)
    eg = O.rel_l2_cols(O.apply_output_axis(O.compress(plan, x, thresh_mode=1), X), Yd).max()
    en = O.rel_l2_cols(O.apply_output_axis(O.compress(plan, x), X), Yd).max()
    assert en < eg <= 1000 * 1e-12, (en, eg)
    plan0 = O.make_plan(JAC, N, 1e-12)
    plan0.eps1 = 0.0
    e0 = O.rel_l2_cols(O.apply_output_axis(O.compress(plan0, x, thresh_mode=1), X), Yd).max()
    assert e0 < 1e-13


# --------------------------------------------------------------------------- naive DFT step
@pytest.mark.parametrize("L", [30, 108, 288, 720, 2250])
def test_naive_dft_vs_library_fft(L):
    """The oracle's written-out DFT step (naive_dft: the O(L^2) sum of Eq. 1, exactly reduced
    twiddle indices) against numpy's FFT, both signs, and the unitary round trip F* F = I."""
    rng = np.random.default_rng(L)
    x = rng.standard_normal((L, 3)) + 1j * rng.standard_normal((L, 3))
    f = O.naive_dft(x, -1)
    g = O.naive_dft(x, +1)
    assert np.abs(f - np.fft.fft(x, axis=0, norm="ortho")).max() <= 1e-14 * np.abs(f).max() * math.log2(L)
    assert np.abs(g - np.fft.ifft(x, axis=0, norm="ortho")).max() <= 1e-14 * np.abs(g).max() * math.log2(L)
    assert np.abs(O.naive_dft(f, +1) - x).max() <= 1e-13
    d = np.zeros(L, complex)
    d[1] = 1.0
    assert np.allclose(O.naive_dft(d, -1), np.exp(-2j * np.pi * np.arange(L) / L) / math.sqrt(L), atol=1e-15)


@pytest.mark.parametrize("kind,dirs", [(LEG, "A"), (JAC, "AW"), (COS, "A")])
def test_compressed_algorithm_with_naive_dft(kind, dirs):
    """BASELINE's oracle as written: the compressed algorithm with a naive DFT, in both steps where
    the method takes one (precompute S = F W e_k; apply v = F* u, P:218 / z' = F* z,
    P:201).  At c1's size (N = 512, blocks L = 720, 288, 108) it builds the same kept sets as the
    library-FFT form (up to threshold ties) with entries equal to 1e-14 of each node's max, applies
    to 1e-14 of it on either operator, and meets the 10 eps bar against the dense product."""
    N, eps = 512, 1e-12
    if kind.kind == O.KIND_COS:
        x, wt = I.cos_nodes(N, 1), None
    else:
        x, _, wt = O.gauss_rule(kind, N)
    plan = O.make_plan(kind, N, eps)
    opf = O.compress(plan, x)
    opn = O.compress(plan, x, dft="naive")
    for Sf, Sn in zip(opf.S, opn.S):
        A, B = Sf.toarray(), Sn.toarray()
        m = np.abs(A).max(axis=1, keepdims=True)
        both = (A != 0) & (B != 0)
        assert np.all(np.abs(A - B)[both] <= 1e-14 * np.broadcast_to(m, A.shape)[both])
        flip = (A != 0) != (B != 0)                                # ties at the threshold only
        assert np.all(np.abs(np.where(flip, A + B, 0)) <= plan.eps1 * m * (1 + 1e-10))
    X = I.rhs(N, 4, 0)
    ref = O.apply_output_axis(opf, X)
    Yn = O.apply_output_axis(opn, X, dft="naive")
    assert O.rel_l2_cols(O.apply_output_axis(opf, X, dft="naive"), ref).max() <= 1e-14
    assert O.rel_l2_cols(Yn, ref).max() <= 1e-13
    assert O.rel_l2_cols(Yn, O.dense_apply(kind, x, X)).max() <= 10 * eps
    if "W" in dirs:
        C = I.rhs(N, 4, 1)
        r = O.apply_input_axis(opf, C, wt)
        assert O.rel_l2_cols(O.apply_input_axis(opf, C, wt, dft="naive"), r).max() <= 1e-14
