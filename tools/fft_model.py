"""Dev tool: numpy model of the CUDA FFT index math (Stockham passes + 4-step).
Not used by tests or the product; it only validated the kernel's indexing."""
import numpy as np

def factors(R):
    f = []
    for r in (8, 4, 5, 3, 2):
        while R % r == 0 and (r != 4 or R % 8 != 0 or True):
            if r == 8 and R % 8: break
            f.append(r); R //= r
    assert R == 1
    return f

def dft_r(v, r, s):
    t = np.arange(r)
    return np.array([np.sum(v * np.exp(s * 2j * np.pi * t * u / r)) for u in range(r)])

def stockham(x, s):
    R = len(x); Ns = 1; data = x.astype(complex)
    for r in factors(R):
        out = np.empty_like(data)
        for j in range(R // r):
            k = j % Ns
            v = np.array([data[j + t * (R // r)] for t in range(r)])
            w = np.exp(s * 2j * np.pi * (k * (R // (Ns * r))) / R)
            v = v * w ** np.arange(r)
            v = dft_r(v, r, s)
            idxD = (j // Ns) * Ns * r + k
            for u in range(r):
                out[idxD + u * Ns] = v[u]
        data = out; Ns *= r
    return data

def four_step(x, L1, L2, s):
    L = L1 * L2
    T = np.empty(L, complex)
    for n2 in range(L2):
        seq = np.array([x[L2 * n1 + n2] for n1 in range(L1)])
        y = stockham(seq, s)
        for k1 in range(L1):
            T[k1 * L2 + n2] = y[k1] * np.exp(s * 2j * np.pi * ((n2 * k1) % L) / L)
    X = np.empty(L, complex)
    for k1 in range(L1):
        y = stockham(T[k1 * L2: k1 * L2 + L2], s)
        for k2 in range(L2):
            X[k1 + L1 * k2] = y[k2]
    return X

rng = np.random.default_rng(0)
for R in (8, 12, 30, 45, 60, 64, 100, 108, 120, 300):
    x = rng.standard_normal(R) + 1j * rng.standard_normal(R)
    print(R, factors(R), np.abs(stockham(x, -1) - np.fft.fft(x)).max(), np.abs(stockham(x, 1) - np.fft.ifft(x) * R).max())
for L1, L2 in ((8, 9), (12, 30), (45, 50)):
    x = rng.standard_normal(L1 * L2) + 1j * rng.standard_normal(L1 * L2)
    print(L1, L2, np.abs(four_step(x, L1, L2, -1) - np.fft.fft(x)).max())
