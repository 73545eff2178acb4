"""CPU oracle for the extra-component method -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementation of what the B200 hot path
computes, written from the paper (Terekhov, arXiv 2004.11610;
``P:<n>`` = /root/reference/PAPER.md line n) and the readings listed in
DESIGN.md ("R-<n>").  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with ``paper_2004_11610_b200`` (the product); the
only common module is the seeded input generator
``paper_2004_11610_b200.inputs``, which holds none of the method's arithmetic.

Two things are computed:

* the plain definition, ``Y = A X`` (or ``diag(w~) A^T C``) with every entry
  ``A[j,k] = phi_j(x_k)`` regenerated in double-double and rounded once
  (``dense_apply``; C helper ``liborc.so``), and
* the algorithm step by step in the paper's order: zeta, s,
  block chain, extended/windowed rows, unitary DFT (Eq. 1, P:24;
  library FFT as the DFT step), threshold, then the computation stage
  of Algorithm 2 / its block form for the output axis and of
  Algorithm 1 / block form for the input axis.

Functions whose result is not pinned by a closed form or an independent
library routine say so ("parity unpinned") in their docstring; see DESIGN.md.
"""
from __future__ import annotations

import ctypes
import functools
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

KIND_COS, KIND_JACOBI, KIND_LAGUERRE, KIND_EXP, KIND_LAGSPEC, KIND_LAG2D = 1, 2, 3, 4, 5, 6


def is_complex(kind) -> bool:
    """Complex rows (full spectrum of L bins, complex X and Y): kinds EXP and LAGSPEC."""
    return kind.kind in (KIND_EXP, KIND_LAGSPEC)


def build_lib() -> str:
    """Compile oracle/orc_special.c into oracle/liborc.so (plain gcc, OpenMP)."""
    src = os.path.join(_HERE, "orc_special.c")
    out = os.path.join(_HERE, "liborc.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-o", out, src, "-lm"])
    return out


def _lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build_lib())
        dp = ctypes.POINTER(ctypes.c_double)
        _LIB.orc_jacobi_entries.argtypes = [ctypes.c_double, ctypes.c_double, dp, ctypes.c_int64,
                                            ctypes.c_int, ctypes.c_int, dp]
        _LIB.orc_laguerre_entries.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, dp]
        _LIB.orc_cos_entries.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         dp]
        _LIB.orc_sin_entries.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         dp]
        _LIB.orc_gauss_newton.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_int64, dp, dp, dp, ctypes.c_int]
        _LIB.orc_dense_apply.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                         dp, ctypes.c_int64, ctypes.c_int64, dp, ctypes.c_int64, dp]
        _LIB.orc_jacobi_mu0.restype = ctypes.c_double
        _LIB.orc_jacobi_mu0.argtypes = [ctypes.c_double, ctypes.c_double]
    return _LIB


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ---------------------------------------------------------------------------
# Special-function entries (double-double recurrences, rounded once)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Kind:
    """Which special function generates A[j,k] = phi_j(x_k) (operator convention R-1).

    kind COS:      phi_j(t) = cos(pi j t), nodes t in [0,1]
    kind EXP:      phi_j(t) = exp(i pi j t), nodes t in [0,2): the non-uniform DFT, complex
                   (the exp row of Appendix A, Eq. A.4 / y3; NEXT-3)
    kind JACOBI:   phi_j(x) = p_j^(alpha,beta)(x), orthonormal on [-1,1] (R-4)
    kind LAGUERRE: phi_j(x) = exp(-x/2) L_j(x), x >= 0
    kind LAGSPEC:  phi_m(k) = (-eta/2 - i k)^m / (eta/2 - i k)^(m+1): the matrix C^T of the
                   spectral Laguerre forward transform V = C^T F (Eq. main_formula2 / lag_matrix,
                   P:395-412); nodes = Fourier frequencies k_j (any real, ascending); complex
    """
    kind: int
    alpha: float = 0.0
    beta: float = 0.0
    eta: float = 0.0   # LAGSPEC only: the Laguerre scale eta > 0


def entries(kind: Kind, nodes: np.ndarray, m0: int, m1: int, m_off: int = 0) -> np.ndarray:
    """E[k, m-m0] = phi_{m+m_off}(x_k) for m in [m0, m1) (node-major)."""
    x = np.ascontiguousarray(nodes, dtype=np.float64)
    out = np.empty((x.size, m1 - m0), dtype=np.float64)
    lib = _lib()
    if kind.kind == KIND_EXP:  # complex: e^{i pi m t} = cos + i sin, both exactly reduced
        im = np.empty_like(out)
        lib.orc_cos_entries(_p(x), x.size, m0, m1, m_off, _p(out))
        lib.orc_sin_entries(_p(x), x.size, m0, m1, m_off, _p(im))
        return out + 1j * im
    if kind.kind == KIND_LAGSPEC:
        # the power form of Eq. (main_formula2), evaluated as written in 80-bit complex
        # arithmetic and rounded once; m < 0 (the left extra components) by the same formula
        a = np.longdouble(kind.eta) / 2
        kk = x.astype(np.longdouble)
        den = a - 1j * kk
        r = (-a - 1j * kk) / den
        m = np.arange(m0 + m_off, m1 + m_off).astype(np.clongdouble)
        return (np.power(r[:, None], m[None, :]) / den[:, None]).astype(np.complex128)
    if kind.kind == KIND_COS:
        lib.orc_cos_entries(_p(x), x.size, m0, m1, m_off, _p(out))
    elif kind.kind == KIND_JACOBI:
        assert m_off == 0
        lib.orc_jacobi_entries(kind.alpha, kind.beta, _p(x), x.size, m0, m1, _p(out))
    elif kind.kind == KIND_LAGUERRE:
        assert m_off == 0
        lib.orc_laguerre_entries(_p(x), x.size, m0, m1, _p(out))
    else:
        raise ValueError(kind)
    return out


def jacobi_mu0(alpha: float, beta: float) -> float:
    return _lib().orc_jacobi_mu0(alpha, beta)


# ---------------------------------------------------------------------------
# Gauss rules (inputs of the Legendre/Jacobi/Laguerre configs)
# ---------------------------------------------------------------------------
def gauss_rule(kind: Kind, N: int, newton: int = 2):
    """Gauss nodes (ascending) and weights for the kind's orthogonality weight.

    Initial guesses: a library routine (scipy's asymptotic Gauss-Legendre rule,
    else the eigenvalues of the fp64 Jacobi matrix via scipy), then Newton in
    double-double on p_N and weights by Christoffel-Darboux, all in liborc.
    Returns (x, w, wt) where wt = w e^{x} (= 1/sum_j l_j(x)^2) for Laguerre,
    wt = w otherwise.
    """
    import scipy.linalg
    import scipy.special
    if kind.kind == KIND_JACOBI and kind.alpha == 0.0 and kind.beta == 0.0:
        x0, _ = scipy.special.roots_legendre(N)
        iters = max(1, newton - 1)
    elif kind.kind == KIND_JACOBI:
        a, b = kind.alpha, kind.beta
        n = np.arange(N, dtype=np.float64)
        t = 2 * n + a + b
        with np.errstate(divide="ignore", invalid="ignore"):
            d = (b * b - a * a) / (t * (t + 2))
        d[0] = (b - a) / (a + b + 2)
        m = np.arange(1, N, dtype=np.float64)
        t = 2 * m + a + b
        e2 = 4 * m * (m + a) * (m + b) * (m + a + b) / (t * t * (t + 1) * (t - 1))
        e2[0] = 4 * (1 + a) * (1 + b) / ((2 + a + b) ** 2 * (3 + a + b))
        x0 = scipy.linalg.eigvalsh_tridiagonal(d, np.sqrt(e2))
        iters = newton + 1
    elif kind.kind == KIND_LAGUERRE:
        n = np.arange(N, dtype=np.float64)
        x0 = scipy.linalg.eigvalsh_tridiagonal(2 * n + 1, np.arange(1, N, dtype=np.float64))
        iters = newton + 2
    else:
        raise ValueError("Gauss rule needs JACOBI or LAGUERRE")
    x = np.ascontiguousarray(np.sort(x0), dtype=np.float64)
    w = np.empty_like(x)
    wt = np.empty_like(x)
    bad = _lib().orc_gauss_newton(kind.kind, kind.alpha, kind.beta, N, _p(x), _p(w), _p(wt), iters)
    if bad:
        raise ArithmeticError("Gauss Newton produced non-finite nodes")
    return x, w, wt


# ---------------------------------------------------------------------------
# Plain definition: the dense product (the paper's "direct method")
# ---------------------------------------------------------------------------
def dense_apply(kind: Kind, nodes: np.ndarray, X: np.ndarray, M: int | None = None) -> np.ndarray:
    """Y[j,b] = sum_k phi_j(x_k) X[k,b], j < M (Y = A X; output indexed by degree; M = N unless
    given: rectangular for the complex kinds)."""
    if is_complex(kind):  # complex: the entries matrix (rounded once), a plain matmul
        A = entries(kind, nodes, 0, len(nodes) if M is None else M).T   # A[j, k] = phi_j(x_k)
        return A @ np.asarray(X, dtype=np.complex128)
    X = np.ascontiguousarray(X, dtype=np.float64)
    N, B = X.shape
    Y = np.empty((N, B), dtype=np.float64)
    x = np.ascontiguousarray(nodes, dtype=np.float64)
    rc = _lib().orc_dense_apply(kind.kind, kind.alpha, kind.beta, 1, _p(x), N, N, _p(X), B, _p(Y))
    assert rc == 0
    return Y


def dense_apply_rows(kind: Kind, nodes: np.ndarray, X: np.ndarray, ndeg: int) -> np.ndarray:
    """Rows [0, ndeg) of Y = A X (a row sample of the dense product; same arithmetic)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    N, B = X.shape
    Y = np.empty((ndeg, B), dtype=np.float64)
    x = np.ascontiguousarray(nodes, dtype=np.float64)
    rc = _lib().orc_dense_apply(kind.kind, kind.alpha, kind.beta, 1, _p(x), N, ndeg, _p(X), B, _p(Y))
    assert rc == 0
    return Y


def dense_apply_t(kind: Kind, nodes: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Y[k,b] = sum_j phi_j(x_k) C[j,b] (Y = A^T C; output indexed by node; j < rows of C)."""
    if is_complex(kind):  # complex: Y[k] = sum_j phi_j(x_k) C[j] (no conjugate)
        return entries(kind, nodes, 0, C.shape[0]) @ np.asarray(C, dtype=np.complex128)
    C = np.ascontiguousarray(C, dtype=np.float64)
    N, B = C.shape
    Y = np.empty((N, B), dtype=np.float64)
    x = np.ascontiguousarray(nodes, dtype=np.float64)
    rc = _lib().orc_dense_apply(kind.kind, kind.alpha, kind.beta, 2, _p(x), N, N, _p(C), B, _p(Y))
    assert rc == 0
    return Y


# ---------------------------------------------------------------------------
# Kaiser window, zeta(eps1), s(zeta, eps2)
# ---------------------------------------------------------------------------
def bessel_i0(x: float) -> float:
    """I_0(x) = sum_k (x/2)^{2k} / (k!)^2 (power series, math.fsum)."""
    x = float(x)
    q = 0.25 * x * x
    terms, t, k = [1.0], 1.0, 0
    while True:
        k += 1
        t *= q / (k * k)
        terms.append(t)
        if t < 1e-18 * terms[0] and k > q:
            break
    return math.fsum(terms)


def bessel_i1(x: float) -> float:
    """I_1(x) = sum_k (x/2)^{2k+1} / (k! (k+1)!)."""
    x = float(x)
    q = 0.25 * x * x
    t = 0.5 * x
    terms, k = [t], 0
    while True:
        k += 1
        t *= q / (k * (k + 1))
        terms.append(t)
        if t < 1e-18 * terms[0] and k > q:
            break
    return math.fsum(terms)


def kaiser(zeta: float, npts: int) -> np.ndarray:
    """w_n^{zeta,npts} = I0(zeta sqrt(1-(2n/npts-1)^2)) / I0(zeta), n = 0..npts.

    A window over L positions uses npts = L - 1 (L samples; reading R-6).  The values of one
    (zeta, npts) are computed once and memoised (the per-point series is slow in Python; a node
    chunk of c5's first block would otherwise spend 4 s recomputing its 86400-point window).
    """
    return _kaiser_memo(float(zeta), int(npts)).copy()


@functools.lru_cache(maxsize=64)
def _kaiser_memo(zeta: float, npts: int) -> np.ndarray:
    n = np.arange(npts + 1, dtype=np.float64)
    r = (2.0 * n - npts) / npts
    arg = zeta * np.sqrt(np.maximum(0.0, 1.0 - r * r))
    i0z = bessel_i0(zeta)
    return np.array([bessel_i0(a) for a in arg]) / i0z


def kaiser_at(zeta: float, npts: int, n: int) -> float:
    r = (2.0 * n - npts) / npts
    return bessel_i0(zeta * math.sqrt(max(0.0, 1.0 - r * r))) / bessel_i0(zeta)


def solve_zeta(eps1: float, zeta0: float = 50.0, tol: float = 1e-14) -> float:
    """zeta with 1/I0(zeta) = eps1, Newton from zeta0 = 50.

    Newton is applied to the equivalent equation ln I0(zeta) = -ln eps1 (the
    literal 1/I0 form diverges from zeta0 = 50; reading R-7).
    """
    z = zeta0
    target = -math.log(eps1)
    for _ in range(200):
        g = math.log(bessel_i0(z)) - target
        step = g / (bessel_i1(z) / bessel_i0(z))
        z -= step
        if abs(step) < tol * max(1.0, z):
            return z
    raise ArithmeticError("zeta Newton did not converge")


def smooth5_even_at_least(n: int) -> int:
    """Smallest even integer >= n whose only prime factors are 2, 3, 5 (R-9)."""
    m = max(2, n + (n & 1))
    while True:
        r = m
        for p in (2, 3, 5):
            while r % p == 0:
                r //= p
        if r == 1:
            return m
        m += 2


@dataclass
class Block:
    """One block of the (block) extra-component method.

    Positions p in [0, L) carry degree p + m_off; the kept (real) degrees are
    positions [keep_lo, keep_hi); the others are the extra components (P:131-180
    for the trig form, P:281-301 for the block form).
    """
    L: int
    m_off: int
    keep_lo: int
    keep_hi: int

    @property
    def H(self) -> int:
        return self.L // 2 + 1


@dataclass
class Plan:
    kind: Kind
    N: int          # nodes (columns of A)
    eps1: float
    eps2: float
    zeta: float
    blocks: list = field(default_factory=list)
    tail: int = 0   # dense degrees [0, tail)
    M: int = 0      # degrees (rows of A); 0 = N (square)

    @property
    def rows(self) -> int:
        return self.M if self.M > 0 else self.N


def minimal_s(zeta: float, span: int, eps2: float, two_sided: bool) -> int:
    """Smallest s >= 1 with w^{zeta, L-1}_s >= eps2, L = span + s (block) or span + 2s (trig).

    Reading R-2 of P:184 (the printed '<' is satisfied by s = 0).
    """
    for s in range(1, 4 * span + 64):
        L = span + (2 * s if two_sided else s)
        if kaiser_at(zeta, L - 1, s) >= eps2:
            return s
    raise ArithmeticError("s search did not terminate (eps2 too close to 1?)")


def make_plan(kind: Kind, N: int, eps: float, eps1: float | None = None, eps2: float | None = None,
              dense_cutoff: int = 32, M: int | None = None) -> Plan:
    """Block chain (R-2, R-3, R-8, R-9): see DESIGN.md.  M: degrees (rows) when they differ from
    the N nodes -- complex kinds only (the C^T of P:412 is (M+1) x (Nx+1), R-21)."""
    eps1 = eps if eps1 is None else eps1
    eps2 = 1e-2 if eps2 is None else eps2
    zeta = solve_zeta(eps1)
    plan = Plan(kind, N, eps1, eps2, zeta)
    if M is not None and M != N:
        assert is_complex(kind), "rectangular operators: complex kinds only"
        plan.M = M
    if kind.kind in (KIND_COS, KIND_EXP, KIND_LAGSPEC):
        # trig form: extra components on both sides (Alg. 2); span = the degrees
        R = plan.rows
        s0 = minimal_s(zeta, R, eps2, two_sided=True)
        L = smooth5_even_at_least(R + 2 * s0)
        s = (L - R) // 2
        plan.blocks.append(Block(L, -s, s, s + R))
        plan.tail = 0
        return plan
    e = N
    while e > dense_cutoff:
        s0 = minimal_s(zeta, e, eps2, two_sided=False)
        L = smooth5_even_at_least(e + s0)
        s = L - e
        if s >= e:   # the next block's span [s_{i+1}, s_i) must shrink (R-8)
            raise ArithmeticError("block chain does not shrink (eps2 too close to 1)")
        plan.blocks.append(Block(L, 0, s, e))
        e = s
    plan.tail = e
    return plan


# ---------------------------------------------------------------------------
# Compression (precomputation stage)
# ---------------------------------------------------------------------------
# ---------------------------------------------------------------------------
# The DFT step written out (BASELINE north star: "the compressed algorithm with a naive DFT").
# Eq. 1: (F f)_q = (1/sqrt(L)) sum_p f_p e^{-2 pi i p q / L}; F* has the + sign.  The
# twiddle of p q is taken at the exactly reduced index (p q mod L) from a table evaluated in long
# double, and the O(L^2) sum is one matrix product.  dft="fft" (default) uses numpy's FFT for the
# same step; the two are pinned against each other in tests/test_oracle_pins.py.
# ---------------------------------------------------------------------------
NAIVE_MAX_L = 4096


@functools.lru_cache(maxsize=6)
def _dft_matrix(L: int, sign: int) -> np.ndarray:
    """F[q, p] = e^{sign 2 pi i (p q mod L) / L} / sqrt(L) (L x L, complex128)."""
    if L > NAIVE_MAX_L:
        raise ValueError(f"naive DFT limited to L <= {NAIVE_MAX_L} (O(L^2) memory)")
    m = np.arange(L, dtype=np.longdouble)
    # angles in long double: 2 pi m / L with pi to long-double precision
    pi_l = np.longdouble("3.14159265358979323846264338327950288")
    ang = 2 * pi_l * m / np.longdouble(L)
    tw = (np.cos(ang) + sign * 1j * np.sin(ang)).astype(np.complex128)
    idx = np.outer(np.arange(L, dtype=np.int64), np.arange(L, dtype=np.int64)) % L
    return tw[idx] / math.sqrt(L)


def naive_dft(x: np.ndarray, sign: int, axis: int = 0) -> np.ndarray:
    """Unitary DFT of length L = x.shape[axis] by the direct sum (sign -1: F, +1: F*)."""
    x = np.moveaxis(np.asarray(x, dtype=np.complex128), axis, 0)
    y = _dft_matrix(x.shape[0], sign) @ x.reshape(x.shape[0], -1)
    return np.moveaxis(y.reshape(x.shape), 0, axis)


def _half_to_real_inverse(u: np.ndarray, L: int, dft: str) -> np.ndarray:
    """v = F* U (real), U the Hermitian spectrum whose bins 0..L/2 are u (rows)."""
    if dft == "fft":
        return np.fft.irfft(u, n=L, axis=0, norm="ortho")
    H = u.shape[0]
    U = np.zeros((L,) + u.shape[1:], dtype=np.complex128)
    U[:H] = u
    U[0] = U[0].real                                   # bins 0 and L/2 of a real signal are real
    if L % 2 == 0:
        U[L // 2] = U[L // 2].real
    U[L - np.arange(1, (L + 1) // 2)] = np.conj(u[1:(L + 1) // 2])
    return naive_dft(U, +1, axis=0).real


def node_spectra(plan: Plan, blk: Block, nodes: np.ndarray, dft: str = "fft") -> np.ndarray:
    """S[k, q] = (F W e_k)_q: unitary DFT (Eq. 1) of the windowed extended row of node k.

    Returns the half spectrum q in [0, H) (real rows).  Bins 0 and L/2
    are real by symmetry and their imaginary part is set to exactly 0.  Kind EXP (complex
    rows): the full spectrum q in [0, L).  dft="naive": the direct sum (naive_dft).
    """
    w = kaiser(plan.zeta, blk.L - 1)
    E = entries(plan.kind, nodes, 0, blk.L, blk.m_off)          # E[k, p] = phi_{p+m_off}(x_k)
    if dft == "naive":
        S = naive_dft(E * w[None, :], -1, axis=1)
        if is_complex(plan.kind):
            return S
        S = S[:, :blk.H].copy()
    elif is_complex(plan.kind):                                 # complex rows: the full spectrum
        return np.fft.fft(E * w[None, :], axis=1, norm="ortho")
    else:
        S = np.fft.rfft(E * w[None, :], axis=1, norm="ortho")  # e^{-2 pi i p q / L} / sqrt(L)
    S[:, 0] = S[:, 0].real
    S[:, -1] = S[:, -1].real
    return S


def threshold(S: np.ndarray, eps1: float) -> np.ndarray:
    """Per-node relative threshold (reading R-3): drop |S| < eps1 * max_q |S[k,q]|."""
    mag2 = S.real ** 2 + S.imag ** 2
    tau2 = (eps1 * eps1) * mag2.max(axis=1, keepdims=True)
    return np.where(mag2 >= tau2, S, 0.0)


@dataclass
class Operator:
    plan: Plan
    S: list          # per block: scipy.sparse.csr_matrix (N x H) complex, kept entries
    windows: list    # per block: Kaiser window on L points
    P_tail: np.ndarray  # (tail x N) dense, phi_j(x_k) for j < tail


def threshold_global(S: np.ndarray, eps1: float, gmax2: float) -> np.ndarray:
    """Global threshold of Algorithm 1/2 step 1.3: drop |S| < eps1 * ||A_e||_max, the max
    over the block's whole compressed matrix (gmax2 = that max squared)."""
    mag2 = S.real ** 2 + S.imag ** 2
    return np.where(mag2 >= (eps1 * eps1) * gmax2, S, 0.0)


def compress(plan: Plan, nodes: np.ndarray, node_chunk: int = 512, thresh_mode: int = 0,
             dft: str = "fft") -> Operator:
    """The compressed operator of every block.  thresh_mode 0: the per-node
    relative threshold (reading R-3); 1: the global threshold of step 1.3 -- a first
    pass over the nodes finds the block's max |S|, the second thresholds."""
    S_list, W_list = [], []
    for blk in plan.blocks:
        parts = []
        gmax2 = 0.0
        if thresh_mode == 1:
            for k0 in range(0, plan.N, node_chunk):
                S = node_spectra(plan, blk, nodes[k0:k0 + node_chunk], dft)
                gmax2 = max(gmax2, float((S.real ** 2 + S.imag ** 2).max()))
        for k0 in range(0, plan.N, node_chunk):
            S = node_spectra(plan, blk, nodes[k0:k0 + node_chunk], dft)
            Sk = threshold_global(S, plan.eps1, gmax2) if thresh_mode == 1 else threshold(S, plan.eps1)
            parts.append(sp.csr_matrix(Sk))
        S_list.append(sp.vstack(parts).tocsr())
        W_list.append(kaiser(plan.zeta, blk.L - 1))
    P_tail = entries(plan.kind, nodes, 0, plan.tail).T.copy() if plan.tail > 0 else np.zeros((0, plan.N))
    return Operator(plan, S_list, W_list, P_tail)


# ---------------------------------------------------------------------------
# Appendix A: fast precompute of the trig kinds (NEXT-2, reading R-22)
# ---------------------------------------------------------------------------
def window_spectrum_truncated(zeta: float, L: int, eps1: float):
    """Step 1 of Appendix A: the Kaiser window's unitary DFT x~ = F w (one library FFT,
    "performed once for all rows"), truncated to the q = 2Q+1 coefficients |m| <= Q, Q the largest
    |m| <= L/2 with |x~_m| >= eps1 |x~_0| (R-22).  Returns (Q, x~ truncated (length L), w' = F* x~
    truncated): w' is the window of the whole method (divided out in the computation stage)."""
    w = kaiser(zeta, L - 1)
    xt = np.fft.fft(w, norm="ortho")
    m = np.minimum(np.arange(L), L - np.arange(L))
    big = np.abs(xt) >= eps1 * abs(xt[0])
    Q = int(m[big].max())
    xq = np.where(m <= Q, xt, 0.0)
    wq = np.fft.ifft(xq, norm="ortho").real        # x~ Hermitian (w real) => w' real
    return Q, xq, wq


def _dirichlet_exp(t, L: int, m_off: int) -> np.ndarray:
    """Eq. (y3) for the extended row p -> e^{i pi (p + m_off) t}, p in [0, L): all L bins,
    y~_k = L^-1/2 e^{i pi m_off t} (e^{i L theta} - 1) / (e^{i theta} w_L^k - 1), theta = pi t, written in
    its equivalent Dirichlet form e^{i pi (L-1) s / L} sin(pi s) / sin(pi s / L), s = L t / 2 - k
    (reduced to (-L/2, L/2]; the limit L at s = 0) so that it is exact near resonance.  80-bit."""
    t = np.asarray(t, dtype=np.longdouble)
    k = np.arange(L, dtype=np.longdouble)
    Ld = np.longdouble(L)
    s = Ld * t[:, None] / 2 - k[None, :]
    s = s - Ld * np.round(s / Ld)
    pi = np.longdouble(np.pi)
    den = np.sin(pi * s / Ld)
    ratio = np.where(s == 0, Ld, np.sin(pi * s) / np.where(s == 0, 1, den))
    a = (Ld - 1) * s / Ld + np.longdouble(m_off) * t[:, None]   # phase / pi
    a = a - 2 * np.round(a / 2)
    y = ratio * (np.cos(pi * a) + 1j * np.sin(pi * a)) / np.sqrt(Ld)
    return y.astype(np.complex128)


def row_spectra_closed(kind: Kind, nodes: np.ndarray, L: int, m_off: int) -> np.ndarray:
    """Step 3 of Appendix A: the unitary DFT of every extended (unwindowed) row in closed form,
    all L bins.  exp: (y3); cos: (y3(theta) + y3(-theta)) / 2 (the printed (y1) is the complex
    conjugate of the sum it names, R-22); LAGSPEC: (y3) at e^{i theta_j} = r_j times 1/(eta/2 - i k_j)."""
    x = np.asarray(nodes, dtype=np.float64)
    if kind.kind == KIND_EXP:
        return _dirichlet_exp(x, L, m_off)
    if kind.kind == KIND_COS:
        return 0.5 * (_dirichlet_exp(x, L, m_off) + _dirichlet_exp(-x, L, m_off))
    if kind.kind == KIND_LAGSPEC:
        a = np.longdouble(kind.eta) / 2
        kk = x.astype(np.longdouble)
        r = (-a - 1j * kk) / (a - 1j * kk)
        th = np.angle(r) / np.longdouble(np.pi)        # r = e^{i pi th}
        d = (1 / (a - 1j * kk)).astype(np.complex128)
        return _dirichlet_exp(th, L, m_off) * d[:, None]
    raise ValueError("Appendix A covers the trigonometric kinds only")


def node_spectra_appA(plan: Plan, blk: Block, nodes: np.ndarray, xq: np.ndarray) -> np.ndarray:
    """Step 2 of Appendix A: F(w' . row) = x~ * y~ (Eq. A.1: (x~*y~)_n =
    L^-1/2 sum_m x~_m y~_{(n-m) mod L}) over the 2Q+1 nonzero x~_m, every bin (the oracle does
    not skip bins; the product evaluates only a window around each node's peak)."""
    L = blk.L
    y = row_spectra_closed(plan.kind, nodes, L, blk.m_off)
    S = np.zeros_like(y)
    for m in np.nonzero(xq)[0]:
        S += xq[m] * np.roll(y, m, axis=1)            # y~_{(n - m) mod L}
    S /= np.sqrt(L)
    if is_complex(plan.kind):
        return S
    S = S[:, :blk.H].copy()
    S[:, 0] = S[:, 0].real
    S[:, -1] = S[:, -1].real
    return S


def compress_appA(plan: Plan, nodes: np.ndarray, node_chunk: int = 256) -> Operator:
    """The trig operator by Appendix A: per block the truncated window spectrum, closed-form row
    spectra, convolution, then the same per-node threshold; the window the computation
    stage divides by is w' (R-22)."""
    assert plan.kind.kind in (KIND_COS, KIND_EXP, KIND_LAGSPEC)
    S_list, W_list = [], []
    for blk in plan.blocks:
        Q, xq, wq = window_spectrum_truncated(plan.zeta, blk.L, plan.eps1)
        parts = []
        for k0 in range(0, plan.N, node_chunk):
            Sk = threshold(node_spectra_appA(plan, blk, nodes[k0:k0 + node_chunk], xq), plan.eps1)
            parts.append(sp.csr_matrix(Sk))
        S_list.append(sp.vstack(parts).tocsr())
        W_list.append(wq)
    return Operator(plan, S_list, W_list, np.zeros((0, plan.N)))


# ---------------------------------------------------------------------------
# 2D (both-sided) block extra-component method, time-domain Laguerre (NEXT-1, reading R-23)
# ---------------------------------------------------------------------------
def lag2d_nodes_ext(nodes: np.ndarray, n: int) -> np.ndarray:
    """The equispaced grid x_i (t_i = 12 i / (N-1)) continued to n points: the given
    N nodes, then x_{N-1} + i h, h = (x_{N-1} - x_0) / (N - 1) (the extra rows of the 2D blocks)."""
    x = np.asarray(nodes, dtype=np.float64)
    N = x.size
    if n <= N:
        return x[:n].copy()
    h = (x[-1] - x[0]) / (N - 1)
    return np.concatenate([x, x[-1] + h * np.arange(1, n - N + 1, dtype=np.float64)])


@dataclass
class Operator2D:
    plan: Plan        # the block chain, used on both axes (square N x N)
    D2: list          # D2[b][a]: scipy.sparse (L_b x L_a) complex, thresholded 2D spectrum
    windows: list     # Kaiser window of each block
    tail_rows: np.ndarray   # D[i, j], i < t (all degrees)
    tail_cols: np.ndarray   # D[i, j], i >= t, j < t


def compress_2d(plan: Plan, nodes: np.ndarray) -> Operator2D:
    """D[i,j] = l_j(x_i) on the equispaced grid, compressed per block pair (a, b) of the chain used
    on both axes (Fig. test322; R-23): the extended block E_ab[p, q] =
    l_q(x_p), p in [0, L_b) (time positions; extra rows continue the grid), q in [0, L_a) (degrees;
    extra degrees continue the recurrence), then D2_ab = F W_b E_ab W_a F (Eq. comp_2d, P:428;
    unitary 2D DFT), thresholded at eps1 * max |D2_ab| (the global form of P:198)."""
    assert plan.kind.kind == KIND_LAGUERRE
    N, t = plan.N, plan.tail
    Lmax = max((b.L for b in plan.blocks), default=0)   # N <= cutoff: no block, all direct
    W = [kaiser(plan.zeta, b.L - 1) for b in plan.blocks]
    D2 = []
    for b, wb in zip(plan.blocks, W):
        Et = entries(plan.kind, lag2d_nodes_ext(nodes, b.L), 0, Lmax)   # Et[p, q] = l_q(x_p)
        row = []
        for a, wa in zip(plan.blocks, W):
            S = np.fft.fft2(wb[:, None] * Et[:, :a.L] * wa[None, :], norm="ortho")
            S = np.where(np.abs(S) >= plan.eps1 * np.abs(S).max(), S, 0.0)
            row.append(sp.csr_matrix(S))
        D2.append(row)
    x = np.asarray(nodes, dtype=np.float64)
    tail_rows = entries(plan.kind, x[:t], 0, N) if t > 0 else np.zeros((0, N))
    tail_cols = entries(plan.kind, x[t:], 0, t) if t > 0 else np.zeros((N, 0))
    return Operator2D(plan, D2, W, tail_rows, tail_cols)


def apply_2d(op: Operator2D, C: np.ndarray) -> np.ndarray:
    """Y = D C (values at the grid from Laguerre coefficients, the backward transform of P:528):
    per degree block a, z_a = F* W_a^-1 pad_a(C) (Alg. 1 prologue); per time block b,
    u_b = sum_a D2_ab z_a, v_b = F* u_b, Y[kept_b] = v_b / w_b (Alg. 2 epilogue);
    tails by the direct method: rows i < t in full, columns j < t for i >= t."""
    plan = op.plan
    C = np.asarray(C, dtype=np.float64)
    N, B = C.shape
    Y = np.zeros((N, B))
    zs = []
    for a, wa in zip(plan.blocks, op.windows):
        z = np.zeros((a.L, B))
        z[a.keep_lo:a.keep_hi] = C[a.keep_lo:a.keep_hi] / wa[a.keep_lo:a.keep_hi, None]
        zs.append(np.fft.ifft(z, axis=0, norm="ortho"))
    for b, wb, row in zip(plan.blocks, op.windows, op.D2):
        u = np.zeros((b.L, B), dtype=np.complex128)
        for S, z in zip(row, zs):
            u += S @ z
        v = np.fft.ifft(u, axis=0, norm="ortho").real      # Hermitian u: real up to rounding
        Y[b.keep_lo:b.keep_hi] = v[b.keep_lo:b.keep_hi] / wb[b.keep_lo:b.keep_hi, None]
    t = plan.tail
    if t > 0:
        Y[t:] += op.tail_cols @ C[:t]
        Y[:t] = op.tail_rows @ C
    return Y


def nnz_2d(op: Operator2D, half: bool = True) -> int:
    """Kept entries of all block pairs (half: rows k <= L_b/2 only, the Hermitian half stored)."""
    tot = 0
    for b, row in zip(op.plan.blocks, op.D2):
        for S in row:
            tot += S[:b.L // 2 + 1].nnz if half else S.nnz
    return tot


# ---------------------------------------------------------------------------
# Computation stage
# ---------------------------------------------------------------------------
def apply_output_axis(op: Operator, X: np.ndarray, dft: str = "fft") -> np.ndarray:
    """Y = A X, output indexed by degree (Alg. 2; block form P:281).

    Per block: u = S^T X (sparse), v = F* u (unitary inverse DFT, real
    output), Y[kept] = v[kept] / w[kept]; the extra positions are discarded
    (Fe2).  Tail degrees by the direct method.  dft="naive": the inverse
    DFT by the direct sum (naive_dft), blocks with L <= NAIVE_MAX_L.
    """
    if is_complex(op.plan.kind):                                # complex input and output
        X = np.asarray(X, dtype=np.complex128)
        Y = np.zeros((op.plan.rows, X.shape[1]), dtype=np.complex128)
        for blk, S, w in zip(op.plan.blocks, op.S, op.windows):
            u = S.T @ X                                         # (L x B): full spectrum
            v = naive_dft(u, +1) if dft == "naive" else np.fft.ifft(u, axis=0, norm="ortho")
            lo, hi = blk.keep_lo, blk.keep_hi
            Y[lo + blk.m_off:hi + blk.m_off] = v[lo:hi] / w[lo:hi, None]
        return Y
    X = np.asarray(X, dtype=np.float64)
    N, B = X.shape
    Y = np.zeros((N, B))
    for blk, S, w in zip(op.plan.blocks, op.S, op.windows):
        u = S.T @ X                                             # (H x B) complex
        v = _half_to_real_inverse(u, blk.L, dft)                # e^{+2 pi i p q / L} / sqrt(L)
        lo, hi = blk.keep_lo, blk.keep_hi
        Y[lo + blk.m_off:hi + blk.m_off] = v[lo:hi] / w[lo:hi, None]
    if op.plan.tail:
        Y[:op.plan.tail] = op.P_tail @ X
    return Y


def apply_input_axis(op: Operator, C: np.ndarray, wt: np.ndarray | None = None, dft: str = "fft") -> np.ndarray:
    """Y = diag(wt) A^T C, input indexed by degree (Alg. 1; block form P:281-301).

    Per block: z = pad(C) / w (zeros outside the kept range, Fe1/Fe3), z' = F* z,
    Y[k] += sum over the full spectrum of S[k,q] z'[q], evaluated on the half
    spectrum as c_q Re(S z') with c_0 = c_{L/2} = 1, else 2 (real case).
    """
    if is_complex(op.plan.kind):  # complex rows: full spectrum, no fold, complex result
        C = np.asarray(C, dtype=np.complex128)
        B = C.shape[1]
        Y = np.zeros((op.plan.N, B), dtype=np.complex128)
        for blk, S, w in zip(op.plan.blocks, op.S, op.windows):
            z = np.zeros((blk.L, B), dtype=np.complex128)
            lo, hi = blk.keep_lo, blk.keep_hi
            z[lo:hi] = C[lo + blk.m_off:hi + blk.m_off] / w[lo:hi, None]
            zf = naive_dft(z, +1) if dft == "naive" else np.fft.ifft(z, axis=0, norm="ortho")
            Y += S @ zf                                         # sum_q S[k,q] (F* z)_q
        if wt is not None:
            Y *= wt[:, None]
        return Y
    C = np.asarray(C, dtype=np.float64)
    N, B = C.shape
    Y = np.zeros((N, B))
    for blk, S, w in zip(op.plan.blocks, op.S, op.windows):
        z = np.zeros((blk.L, B))
        lo, hi = blk.keep_lo, blk.keep_hi
        z[lo:hi] = C[lo + blk.m_off:hi + blk.m_off] / w[lo:hi, None]
        if dft == "naive":
            zq = naive_dft(z, +1)[:blk.H]                       # (F* z)_q, q in [0, H)
        else:
            zq = np.conj(np.fft.rfft(z, axis=0, norm="ortho"))  # (F* z)_q, q in [0, H)
        c = np.full(blk.H, 2.0)
        c[0] = 1.0
        c[-1] = 1.0
        Y += (S @ (c[:, None] * zq)).real
    if op.plan.tail:
        Y += op.P_tail.T @ C[:op.plan.tail]
    if wt is not None:
        Y *= wt[:, None]
    return Y


def rel_l2_cols(Y: np.ndarray, Yref: np.ndarray) -> np.ndarray:
    """Per-column relative L2 error ||y - y_ref|| / ||y_ref|| (reading R-11)."""
    num = np.linalg.norm(Y - Yref, axis=0)
    den = np.linalg.norm(Yref, axis=0)
    return num / np.where(den == 0, 1.0, den)


def nnz(op: Operator) -> list:
    return [int(S.nnz) for S in op.S]
