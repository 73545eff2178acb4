// appa.cu -- Appendix A fast precompute of the trigonometric kinds (SURVEY NEXT-2,
// reading R-22 in DESIGN.md).  Product side; independent of oracle/.
//
// Per node, instead of generating the L entries of the extended row and FFT-ing them, the kept
// bins of S = F(W' row) are evaluated directly:
//   S_n = L^-1/2 sum_{|m| <= Q} xq_m y_{n-m}                       (Eq. A.1)
// with xq the window's DFT truncated to 2Q+1 coefficients (W' = F* xq is the method's window)
// and y the closed-form DFT of the unwindowed row, (y3) of P:667-671 in its Dirichlet form
//   y_j = L^-1/2 e^{i pi (m_off t + (L-1) s / L)} sin(pi s) / sin(pi s / L),  s = L t / 2 - j,
// exact near resonance (s -> integer multiples of L), the cos row as (y(t) + y(-t)) / 2.
// Only a window of 2W+1 bins around the node's peak L t / 2 is evaluated ("about 24
// convolutions per row"); a kept bin on the window's edge raises a flag and the host
// retries with a wider window.  One warp per node; the y values of the window +- Q sit in
// shared memory.
#include <math.h>

#include "xc_internal.cuh"

namespace {

// sin(pi x) for a double-double x (|x| moderate): exact reduction to the nearest integer, then
// sinpi of the high part plus the first-order low-part correction.
__device__ __forceinline__ double sinpi_dd(ddv x) {
  const double n0 = rint(x.h);
  ddv f = ddsub(x, dv(n0));
  double s, c;
  sincospi(f.h, &s, &c);
  s = fma(3.141592653589793 * f.l, c, s);
  return (fmod(n0, 2.0) != 0.0) ? -s : s;
}

// y_j (unnormalised by L^-1/2) for the row p -> e^{i pi (p + m_off) t}, t = sg * (th + tl)
__device__ __forceinline__ double2 dirichlet(double th, double tl, double sg, int L, int m_off, int64_t j) {
  // s = L t / 2 - j in double-double, reduced to (-L/2, L/2]
  ddv u = tprod((double)L, th);
  u = ddadd(u, dv((double)L * tl));
  u.h *= 0.5 * sg;
  u.l *= 0.5 * sg;
  ddv s = ddsub(u, dv((double)j));
  const double r = rint(s.h / (double)L);
  if (r != 0.0) s = ddsub(s, tprod(r, (double)L));
  double ratio;
  if (s.h == 0.0 && s.l == 0.0) {
    ratio = (double)L;
  } else {
    const double den = sinpi((s.h + s.l) / (double)L);
    ratio = sinpi_dd(s) / den;
  }
  // phase / pi = m_off t + s - s / L   (mod 2)
  ddv a = tprod((double)m_off, sg * th);
  a = ddadd(a, dv((double)m_off * sg * tl));
  a = ddadd(a, s);
  a = ddsub(a, dv((s.h + s.l) / (double)L));
  const double n2 = 2.0 * rint(0.5 * a.h);
  a = ddsub(a, dv(n2));
  double sn, cs;
  sincospi(a.h, &sn, &cs);
  const double d = 3.141592653589793 * a.l;
  return make_double2(ratio * fma(-d, sn, cs), ratio * fma(d, cs, sn));
}

struct AppAArgs {
  int kind;        // XC_COS (half spectrum) or XC_EXP (full spectrum; LAGSPEC runs as XC_EXP)
  int L, H, m_off, Q, W;
  const double* th;        // nodes (chunk), high parts
  const double* tl;        // low parts or null
  const double2* cscale;   // per-node scale or null
  const double2* xq;       // xq_m, m = -Q..Q at index m + Q
  int nc;
  double eps1;
  double2* spec;           // full-spectrum mode: spec[q * nc + k], zeroed beforehand; or null
  double2* win;            // window mode: win[k * (2W+1) + i] = S at bin c - W + i
  int* start;              // window mode: kept run per node (band_detect's convention)
  int* len;
  int* wfirst;             // window mode: window index of the run's first bin
  double* thr;             // window mode: eps1^2 max |S|^2 per node
  int* flag;               // set to 1 if a kept bin touches the evaluated window's edge
};

constexpr int kWarps = 4;

__global__ void __launch_bounds__(32 * kWarps) appa_spectra_k(AppAArgs a) {
  extern __shared__ double2 ysm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * kWarps + warp;
  if (k >= a.nc) return;
  const int R = 2 * (a.W + a.Q) + 1, Wn = 2 * a.W + 1;
  double2* y = ysm + (size_t)warp * R;
  const double th = a.th[k], tl = a.tl ? a.tl[k] : 0.0;
  const bool cosk = a.kind == XC_COS;
  const int64_t c = (int64_t)floor(0.5 * (double)a.L * th);  // peak bin (window centre)
  const int64_t j0 = c - a.W - a.Q;
  for (int i = lane; i < R; i += 32) {
    double2 v = dirichlet(th, tl, 1.0, a.L, a.m_off, j0 + i);
    if (cosk) {
      const double2 w = dirichlet(th, tl, -1.0, a.L, a.m_off, j0 + i);
      v = make_double2(0.5 * (v.x + w.x), 0.5 * (v.y + w.y));
    }
    y[i] = v;
  }
  __syncwarp();
  const double isL = 1.0 / (double)a.L;  // L^-1/2 (A.1) x L^-1/2 (y3)
  double2 sc = a.cscale ? a.cscale[k] : make_double2(1.0, 0.0);
  double mx = 0.0, edge = 0.0;
  for (int i = lane; i < Wn; i += 32) {
    const int64_t n = c - a.W + i;
    int64_t q = n;
    // complex rows with 2W + 1 = L + 1 (full circle): the last bin repeats the first -- skipped
    const bool valid = cosk ? (n >= 0 && n < a.H) : !(2 * a.W + 1 > a.L && i == Wn - 1);
    double re = 0.0, im = 0.0;
    if (valid) {
      if (!cosk) q = ((n % a.L) + a.L) % a.L;
#pragma unroll 4
      for (int m = -a.Q; m <= a.Q; ++m) {
        const double2 x = __ldg(&a.xq[m + a.Q]);
        const double2 v = y[i + a.Q - m];  // y_{n - m}
        re = fma(x.x, v.x, fma(-x.y, v.y, re));
        im = fma(x.x, v.y, fma(x.y, v.x, im));
      }
      re *= isL;
      im *= isL;
      const double sr = re * sc.x - im * sc.y, si = re * sc.y + im * sc.x;
      re = sr;
      im = si;
      if (cosk && (q == 0 || q == a.L / 2)) im = 0.0;  // real rows: bins 0 and L/2 are real
      if (a.spec) a.spec[q * a.nc + k] = make_double2(re, im);
      const double m2 = re * re + im * im;
      mx = fmax(mx, m2);
      const bool at_edge = (i == 0 && !(cosk && n <= 0)) || (i == Wn - 1 && !(cosk && n >= a.H - 1));
      if (at_edge) edge = fmax(edge, m2);
    }
    if (a.win) a.win[(int64_t)k * Wn + i] = make_double2(re, im);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    edge = fmax(edge, __shfl_xor_sync(0xffffffffu, edge, o));
  }
  const double thr = (a.eps1 * a.eps1) * mx;
  if (lane == 0 && mx > 0.0 && edge >= thr) atomicOr(a.flag, 1);
  if (!a.win) return;
  __syncwarp();
  // the kept run inside the window: first and last bin with |S|^2 >= thr (the window holds less
  // than half the circle, so for complex rows this linear span is the shortest arc, R-18)
  int first = Wn, last = -1;
  if (mx > 0.0)
    for (int i = lane; i < Wn; i += 32) {
      const double2 v = a.win[(int64_t)k * Wn + i];
      if (v.x * v.x + v.y * v.y >= thr) {
        first = min(first, i);
        last = max(last, i);
      }
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
  }
  if (lane == 0) {
    if (last < 0) {
      a.start[k] = 0;
      a.len[k] = 0;
      a.wfirst[k] = 0;
    } else {
      const int64_t n = c - a.W + first;
      a.start[k] = (int)(cosk ? n : ((n % a.L) + a.L) % a.L);
      a.len[k] = last - first + 1;
      a.wfirst[k] = first;
    }
    a.thr[k] = thr;
  }
}

// kept values of the window mode into the node-ordered value array (band_store's convention:
// bins of the run below the threshold are stored as explicit zeros)
__global__ void appa_store_k(const double2* __restrict__ win, int Wn, const int* __restrict__ wfirst,
                             const int* __restrict__ len, const double* __restrict__ thr,
                             const int64_t* __restrict__ off, double2* vals, int nc) {
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= nc) return;
  const int n = len[k], f = wfirst[k];
  const double t = thr[k];
  for (int i = lane; i < n; i += 32) {
    const double2 v = win[(int64_t)k * Wn + f + i];
    vals[off[k] + i] = (v.x * v.x + v.y * v.y >= t) ? v : make_double2(0.0, 0.0);
  }
}

}  // namespace

// Host side: truncated window spectrum and the window W' = F* xq (long double), R-22.
xc_status appa_window(const std::vector<double>& w, int L, double eps1, std::vector<double2>& xq, int& Q,
                      std::vector<double>& wq) {
  const long double PI2 = 6.283185307179586476925286766559005768L;
  const long double isL = 1.0L / sqrtl((long double)L);
  std::vector<long double> ct(L), st(L);  // e^{2 pi i n / L}, exact index reduction below
  for (int n = 0; n < L; ++n) {
    const long double ang = PI2 * (long double)n / (long double)L;
    ct[n] = cosl(ang);
    st[n] = sinl(ang);
  }
  const int mmax = std::min(64, L / 2);
  std::vector<long double> xr(mmax + 1), xi(mmax + 1);
  for (int m = 0; m <= mmax; ++m) {
    long double sr = 0, si = 0;
    int64_t idx = 0;  // (m p) mod L
    for (int p = 0; p < L; ++p) {
      sr += (long double)w[p] * ct[idx];
      si -= (long double)w[p] * st[idx];
      idx += m;
      if (idx >= L) idx -= L;
    }
    xr[m] = sr * isL;
    xi[m] = si * isL;
  }
  const long double a0 = fabsl(xr[0]);
  Q = 0;
  for (int m = 1; m <= mmax; ++m)
    if (sqrtl(xr[m] * xr[m] + xi[m] * xi[m]) >= (long double)eps1 * a0) Q = m;
  if (2 * Q + 1 > L) {
    xc_set_error("Appendix A: window spectrum does not decay (L too small)");
    return XC_EUNSUPPORTED;
  }
  xq.assign(2 * Q + 1, make_double2(0, 0));
  for (int m = -Q; m <= Q; ++m) {  // xq_{-m} = conj(xq_m) (w real)
    const int am = m < 0 ? -m : m;
    xq[m + Q] = make_double2((double)xr[am], (double)(m < 0 ? -xi[am] : xi[am]));
  }
  wq.assign(L, 0.0);
  for (int p = 0; p < L; ++p) {
    long double v = xr[0];
    int64_t idx = 0;
    for (int m = 1; m <= Q; ++m) {  // 2 Re(xq_m e^{2 pi i m p / L}); the m = L/2 term once
      idx += p;
      idx %= L;
      const long double t = xr[m] * ct[idx] - xi[m] * st[idx];
      v += (2 * m == L) ? t : 2.0L * t;
    }
    wq[p] = (double)(v * isL);
  }
  return XC_OK;
}

xc_status appa_spectra(int kind, int L, int H, int m_off, int Q, int W, const double* th, const double* tl,
                       const double2* cscale, const double2* xq, int nc, double eps1, double2* spec, int* flag,
                       cudaStream_t st, AppAWin* wm) {
  AppAArgs a{kind, L, H, m_off, Q, W, th, tl, cscale, xq, nc, eps1, spec, nullptr, nullptr, nullptr, nullptr,
             nullptr, flag};
  if (wm) {
    a.win = wm->win;
    a.start = wm->start;
    a.len = wm->len;
    a.wfirst = wm->wfirst;
    a.thr = wm->thr;
  }
  const size_t smem = (size_t)kWarps * (2 * (W + Q) + 1) * sizeof(double2);
  if (smem > 200 * 1024) {
    xc_set_error("Appendix A: evaluation window too wide");
    return XC_EUNSUPPORTED;
  }
  XC_CUDA(cudaFuncSetAttribute(appa_spectra_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  appa_spectra_k<<<(nc + kWarps - 1) / kWarps, 32 * kWarps, smem, st>>>(a);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status appa_store(const AppAWin& wm, int W, const int64_t* off, double2* vals, int nc, cudaStream_t st) {
  appa_store_k<<<(nc + 7) / 8, 256, 0, st>>>(wm.win, 2 * W + 1, wm.wfirst, wm.len, wm.thr, off, vals, nc);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}
