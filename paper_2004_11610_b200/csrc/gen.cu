// gen.cu -- GPU precomputation of the compressed operator (precomputation stage,
// Alg. 1/2 steps 1.2-1.3; block form P:281).
//
//  * entry generation: phi_m(x_k) for all positions m of a block, one thread per
//    node running the three-term recurrence in double-double and rounding once
//    (R-5; "accumulation of errors when using the three-term recurrence"),
//    times the Kaiser window (W_M);
//  * band detection / compaction after the FFT: per node, keep |S| >= eps1 * max
//    (R-3), one contiguous run per node (start, len) with the dropped
//    entries inside the run stored as exact zeros;
//  * tile fill for the tensor-core SpMM (spmm.cu).
#include <math.h>

#include <algorithm>

#include "xc_internal.cuh"

namespace {

// 1/(2 ln 2) and ln 2 as double-double
__device__ const double kI2L2_H = 0.7213475204444817, kI2L2_L = 1.0177636870465517e-17;
__device__ const double kLN2_H = 0.6931471805599453, kLN2_L = 2.3190468138462996e-17;

template <bool CPLX>
__device__ __forceinline__ void put(void* F, int64_t idx, double v) {
  if (CPLX)
    reinterpret_cast<double2*>(F)[idx] = make_double2(v, 0.0);
  else
    reinterpret_cast<double*>(F)[idx] = v;
}

// Orthonormal Jacobi: x p_n = a_{n+1} p_{n+1} + b_n p_n + a_n p_{n-1}  (R-4)
template <bool CPLX>
__global__ void gen_jacobi(GenParams g, void* F, int64_t ld) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= g.nc) return;
  const ddv x = dv(g.nodes[k]);
  ddv p = g.p0, pm1 = dv(0.0);
  for (int n = 0; n < g.L; ++n) {
    double e = ddround(p);
    put<CPLX>(F, (int64_t)n * ld + k, g.w ? g.w[n] * e : e);
    const double2 bn = g.jab[3 * n + 0], an = g.jab[3 * n + 1], ia = g.jab[3 * (n + 1) + 2];
    ddv t = ddsub(ddmul(ddsub(x, ddv{bn.x, bn.y}), p), ddmul(ddv{an.x, an.y}, pm1));
    pm1 = p;
    p = ddmul(t, ddv{ia.x, ia.y});
  }
}

__device__ ddv dexp_neg_small(ddv gv) {
  // exp(-g), 0 <= g < ln 2: Taylor series in double-double
  ddv term = dv(1.0), sum = dv(1.0), mg = ddneg(gv);
  for (int n = 1; n < 40; ++n) {
    term = dddiv(ddmul(term, mg), dv((double)n));
    sum = ddadd(sum, term);
    if (fabs(term.h) < 1e-34) break;
  }
  return sum;
}

// Laguerre functions l_n = exp(-x/2) L_n(x) with a tracked binary exponent
template <bool CPLX>
__global__ void gen_laguerre(GenParams g, void* F, int64_t ld) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= g.nc) return;
  const double xk = g.nodes[k];
  ddv y = ddmuld(ddv{kI2L2_H, kI2L2_L}, xk);  // x / (2 ln 2)
  double ny = floor(y.h);
  ddv f = ddsub(y, dv(ny));
  if (f.h < 0.0) {
    ny -= 1.0;
    f = ddadd(f, dv(1.0));
  }
  const ddv ef = dexp_neg_small(ddmul(f, ddv{kLN2_H, kLN2_L}));  // 2^{-f}
  int E = -(int)ny;
  const ddv x = dv(xk);
  ddv Lc = dv(1.0), Lm = dv(0.0);
  for (int n = 0; n < g.L; ++n) {
    double r = ddround(ddmul(Lc, ef));
    double v = (E < -2200) ? 0.0 : ldexp(r, E);
    put<CPLX>(F, (int64_t)n * ld + k, g.w ? g.w[n] * v : v);
    // L_{n+1} = ((2n+1-x) L_n - n L_{n-1}) / (n+1)
    ddv t = ddsub(ddmul(ddsub(dv(2.0 * n + 1.0), x), Lc), ddmuld(Lm, (double)n));
    ddv Ln = dddiv(t, dv((double)(n + 1)));
    Lm = Lc;
    Lc = Ln;
    double a = fabs(Lc.h);
    if (a > 0x1p512) {
      Lc = ddv{ldexp(Lc.h, -512), ldexp(Lc.l, -512)};
      Lm = ddv{ldexp(Lm.h, -512), ldexp(Lm.l, -512)};
      E += 512;
    }
  }
}

// cos(pi m t), m = p + m_off: exact product and exact reduction mod 2
template <bool CPLX>
__global__ void gen_cos(GenParams g, void* F, int64_t ld) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t tot = (int64_t)g.L * g.nc;
  if (idx >= tot) return;
  int p = (int)(idx / g.nc), k = (int)(idx - (int64_t)p * g.nc);
  double m = (double)(p + g.m_off);
  ddv r = tprod(m, g.nodes[k]);
  double n2 = 2.0 * rint(0.5 * r.h);
  r = ddsub(r, dv(n2));
  double s, c;
  sincospi(r.h, &s, &c);
  double v = fma(-3.141592653589793 * r.l, s, c);
  put<CPLX>(F, (int64_t)p * ld + k, g.w ? g.w[p] * v : v);
}

// e^{i pi m t} = (cos, sin)(pi m t), m = p + m_off: the same exact reduction (NEXT-3; the exp row
// of Appendix A)
__global__ void gen_exp(GenParams g, double2* F, int64_t ld) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t tot = (int64_t)g.L * g.nc;
  if (idx >= tot) return;
  int p = (int)(idx / g.nc), k = (int)(idx - (int64_t)p * g.nc);
  double m = (double)(p + g.m_off);
  ddv r = tprod(m, g.nodes[k]);
  if (g.nodes_lo) r = ddadd(r, dv(m * g.nodes_lo[k]));  // t = hi + lo (XC_LAGSPEC phases)
  double n2 = 2.0 * rint(0.5 * r.h);
  r = ddsub(r, dv(n2));
  double s, c;
  sincospi(r.h, &s, &c);
  const double d = 3.141592653589793 * r.l;  // first-order correction for the low part
  double vc = fma(-d, s, c), vs = fma(d, c, s);
  const double wp = g.w ? g.w[p] : 1.0;
  if (g.cscale) {  // per-node complex scale d_k (XC_LAGSPEC: 1 / (eta/2 - i k))
    const double2 sc = g.cscale[k];
    const double re = vc * sc.x - vs * sc.y, im = vc * sc.y + vs * sc.x;
    vc = re;
    vs = im;
  }
  F[(int64_t)p * ld + k] = make_double2(wp * vc, wp * vs);
}

// ---- band detection: per node, max |S|^2 then the kept run -------------------------
// circ (complex rows, full spectrum of L = H bins): the run is circular -- the shortest arc
// holding every kept bin (the complement of the longest circular gap); start in [0, H),
// start + len may exceed H (bins taken mod H).
__global__ void band_detect_circ_k(const double2* __restrict__ spec, int H, int nc, double eps1, double thr_abs2,
                                   int* start, int* len) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nc) return;
  double mx = 0.0;
  for (int q = 0; q < H; ++q) {
    double2 v = spec[(int64_t)q * nc + k];
    mx = fmax(mx, v.x * v.x + v.y * v.y);
  }
  const double thr = thr_abs2 > 0.0 ? thr_abs2 : (eps1 * eps1) * mx;  // global or per node
  int first = -1, prev = -1, gap = -1, gap_end = 0;
  if (mx > 0.0)
    for (int q = 0; q < H; ++q) {
      double2 v = spec[(int64_t)q * nc + k];
      if (v.x * v.x + v.y * v.y >= thr) {
        if (first < 0) first = q;
        if (prev >= 0 && q - prev - 1 > gap) {
          gap = q - prev - 1;
          gap_end = q;
        }
        prev = q;
      }
    }
  if (first < 0) {
    start[k] = 0;
    len[k] = 0;
    return;
  }
  const int wrap = first + (H - 1 - prev);  // unkept bins across the end of the spectrum
  if (wrap >= gap) {                         // the longest gap wraps: run [first, prev]
    start[k] = first;
    len[k] = prev - first + 1;
  } else {                                   // the longest gap is inside: run starts after it
    start[k] = gap_end;
    len[k] = H - gap;
  }
}

__global__ void band_detect_k(const double2* __restrict__ spec, int H, int nc, double eps1, double thr_abs2, int* start,
                              int* len) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nc) return;
  double mx = 0.0;
  for (int q = 0; q < H; ++q) {
    double2 v = spec[(int64_t)q * nc + k];
    mx = fmax(mx, v.x * v.x + v.y * v.y);
  }
  const double thr = thr_abs2 > 0.0 ? thr_abs2 : (eps1 * eps1) * mx;  // global or per node
  int first = -1, last = -1;
  if (mx > 0.0) {
    for (int q = 0; q < H; ++q) {
      double2 v = spec[(int64_t)q * nc + k];
      if (v.x * v.x + v.y * v.y >= thr) {
        if (first < 0) first = q;
        last = q;
      }
    }
  }
  start[k] = first < 0 ? 0 : first;
  len[k] = first < 0 ? 0 : last - first + 1;
}

__global__ void band_store_k(const double2* __restrict__ spec, int H, int nc, double eps1, double thr_abs2,
                             const int* start, const int* len, const int64_t* off, double2* vals, bool circ) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nc) return;
  double mx = 0.0;
  for (int q = 0; q < H; ++q) {
    double2 v = spec[(int64_t)q * nc + k];
    mx = fmax(mx, v.x * v.x + v.y * v.y);
  }
  const double thr = thr_abs2 > 0.0 ? thr_abs2 : (eps1 * eps1) * mx;
  int s = start[k], n = len[k];
  int64_t o = off[k];
  for (int i = 0; i < n; ++i) {
    int q = s + i;
    if (circ && q >= H) q -= H;
    double2 v = spec[(int64_t)q * nc + k];
    if (!circ && (q == 0 || q == H - 1)) v.y = 0.0;  // bins 0 and L/2 of a real row are real
    vals[o + i] = (v.x * v.x + v.y * v.y >= thr) ? v : make_double2(0.0, 0.0);
  }
}

// max |S|^2 over a spectrum chunk (the global threshold's reference, Alg. 1/2 step 1.3):
// non-negative doubles order as their bit patterns, so the max is an exact integer atomicMax
__global__ void spec_max2_k(const double2* __restrict__ spec, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = spec[i];
    m = fmax(m, v.x * v.x + v.y * v.y);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

}  // namespace

xc_status spec_max2(const double2* spec, int64_t n, unsigned long long* out, cudaStream_t st) {
  if (n <= 0) return XC_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 4 * sm_count());
  spec_max2_k<<<grid, 256, 0, st>>>(spec, n, out);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status gen_entries(const GenParams& g, double2* F, cudaStream_t st) {
  if (g.nc <= 0 || g.L <= 0) return XC_OK;
  if (g.kind == XC_EXP) {
    int64_t tot = (int64_t)g.L * g.nc;
    gen_exp<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(g, F, g.nc);
  } else if (g.kind == XC_COS) {
    int64_t tot = (int64_t)g.L * g.nc;
    gen_cos<true><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(g, F, g.nc);
  } else if (g.kind == XC_JACOBI) {
    gen_jacobi<true><<<(g.nc + 127) / 128, 128, 0, st>>>(g, F, g.nc);
  } else {
    gen_laguerre<true><<<(g.nc + 127) / 128, 128, 0, st>>>(g, F, g.nc);
  }
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status gen_entries_real(const GenParams& g, double* E, int64_t ldE, cudaStream_t st) {
  if (g.nc <= 0 || g.L <= 0) return XC_OK;  // nothing to generate (e.g. an empty tail part)
  if (g.kind == XC_COS) {
    int64_t tot = (int64_t)g.L * g.nc;
    gen_cos<false><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(g, E, ldE);
  } else if (g.kind == XC_JACOBI) {
    gen_jacobi<false><<<(g.nc + 127) / 128, 128, 0, st>>>(g, E, ldE);
  } else {
    gen_laguerre<false><<<(g.nc + 127) / 128, 128, 0, st>>>(g, E, ldE);
  }
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status band_detect(const double2* spec, int H, int nc, double eps1, double thr_abs2, int* start, int* len,
                      bool circ, cudaStream_t st) {
  if (circ) band_detect_circ_k<<<(nc + 127) / 128, 128, 0, st>>>(spec, H, nc, eps1, thr_abs2, start, len);
  else band_detect_k<<<(nc + 127) / 128, 128, 0, st>>>(spec, H, nc, eps1, thr_abs2, start, len);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status band_store(const double2* spec, int H, int nc, double eps1, double thr_abs2, const int* start,
                     const int* len, const int64_t* off, double2* vals, bool circ, cudaStream_t st) {
  band_store_k<<<(nc + 127) / 128, 128, 0, st>>>(spec, H, nc, eps1, thr_abs2, start, len, off, vals, circ);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}
