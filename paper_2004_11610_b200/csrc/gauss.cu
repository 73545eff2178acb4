// gauss.cu -- Gauss rules on the GPU (inputs of the Legendre / Jacobi / Laguerre
// transforms; the paper discretises with Gauss quadratures).
//
// 1. Eigenvalues of the symmetric tridiagonal Jacobi matrix by Sturm-sequence
//    bisection, one thread per eigenvalue (robust for every kind).
// 2. Two Newton steps on p_N in double-double from the recurrence (R-5).
// 3. Weights by Christoffel-Darboux at the returned fp64 node:
//    sum_{j<N} p_j(x)^2 = a_N (p_N'(x) p_{N-1}(x) - p_N(x) p_{N-1}'(x)),  w = 1 / sum.
//    Laguerre (orthonormal L_n in e^{-x}): p_n = (-1)^n L_n, a_N = N, and
//    wt = w e^{x} = 1 / sum_j l_j(x)^2 with a tracked binary exponent.
#include <math.h>

#include <vector>

#include "xc_internal.cuh"

namespace {

__device__ const double gI2L2_H = 0.7213475204444817, gI2L2_L = 1.0177636870465517e-17;
__device__ const double gLN2_H = 0.6931471805599453, gLN2_L = 2.3190468138462996e-17;

__global__ void sturm_bisect(const double* d, const double* e2, int N, double lo0, double hi0, double pivmin,
                             double* x) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  double lo = lo0, hi = hi0;
  for (int it = 0; it < 300; ++it) {
    double mid = 0.5 * (lo + hi);
    if (!(mid > lo && mid < hi)) break;
    // number of eigenvalues < mid
    int cnt = 0;
    double q = d[0] - mid;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += (q < 0.0);
    for (int i = 1; i < N; ++i) {
      q = (d[i] - mid) - e2[i] / q;
      if (fabs(q) < pivmin) q = -pivmin;
      cnt += (q < 0.0);
    }
    if (cnt > k)
      hi = mid;
    else
      lo = mid;
  }
  x[k] = 0.5 * (lo + hi);
}

__device__ ddv exp2_neg_frac(ddv f) {
  // 2^{-f} = exp(-f ln2), 0 <= f < 1
  ddv g = ddmul(f, ddv{gLN2_H, gLN2_L});
  ddv term = dv(1.0), sum = dv(1.0), mg = ddneg(g);
  for (int n = 1; n < 40; ++n) {
    term = dddiv(ddmul(term, mg), dv((double)n));
    sum = ddadd(sum, term);
    if (fabs(term.h) < 1e-34) break;
  }
  return sum;
}

// Newton polish + Christoffel-Darboux weights.  kind 2: Jacobi (tab = b_n, a_n, 1/a_n).
__global__ void newton_cd(int kind, const double2* tab, ddv p0, int N, double* x, double* w, double* wt, int iters) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  ddv X = dv(x[k]);
  ddv pN = dv(0), dpN = dv(1), pNm1 = dv(0), dpNm1 = dv(0);
  int E = 0;
  for (int it = 0; it <= iters; ++it) {
    ddv pm = dv(0.0), p = (kind == XC_JACOBI) ? p0 : dv(1.0), dpm = dv(0.0), dp = dv(0.0);
    E = 0;
    for (int n = 0; n < N; ++n) {
      ddv pn, dpn;
      if (kind == XC_JACOBI) {
        double2 bn = tab[3 * n], an = tab[3 * n + 1], ia = tab[3 * (n + 1) + 2];
        ddv xb = ddsub(X, ddv{bn.x, bn.y});
        ddv A = ddv{an.x, an.y}, IA = ddv{ia.x, ia.y};
        pn = ddmul(ddsub(ddmul(xb, p), ddmul(A, pm)), IA);
        dpn = ddmul(ddadd(ddsub(ddmul(xb, dp), ddmul(A, dpm)), p), IA);
      } else {
        ddv cf = ddsub(dv(2.0 * n + 1.0), X);
        ddv inv = dddiv(dv(1.0), dv((double)(n + 1)));
        pn = ddmul(ddsub(ddmul(cf, p), ddmuld(pm, (double)n)), inv);
        dpn = ddmul(ddsub(ddsub(ddmul(cf, dp), ddmuld(dpm, (double)n)), p), inv);
      }
      pm = p;
      p = pn;
      dpm = dp;
      dp = dpn;
      if (fmax(fabs(p.h), fabs(dp.h)) > 0x1p400) {
        p = ddv{ldexp(p.h, -400), ldexp(p.l, -400)};
        pm = ddv{ldexp(pm.h, -400), ldexp(pm.l, -400)};
        dp = ddv{ldexp(dp.h, -400), ldexp(dp.l, -400)};
        dpm = ddv{ldexp(dpm.h, -400), ldexp(dpm.l, -400)};
        E += 400;
      }
    }
    pN = p;
    dpN = dp;
    pNm1 = pm;
    dpNm1 = dpm;
    if (it < iters) X = ddsub(X, dddiv(pN, dpN));
    if (it == iters - 1) X = dv(ddround(X));
  }
  double xr = ddround(X);
  x[k] = xr;
  ddv cd = ddsub(ddmul(dpN, pNm1), ddmul(pN, dpNm1));
  if (kind == XC_JACOBI) {
    double2 aN = tab[3 * N + 1];
    double wk = ddround(dddiv(dv(1.0), ddmul(ddv{aN.x, aN.y}, cd)));
    w[k] = wk;
    wt[k] = wk;
  } else {
    ddv s = ddmuld(cd, -(double)N);  // true sum = s * 2^{2E}
    w[k] = ldexp(ddround(dddiv(dv(1.0), s)), -2 * E);
    // e^{x} = 2^{x/ln2} = 2^{ny} 2^{f}
    ddv y = ddmuld(ddv{gI2L2_H, gI2L2_L}, 2.0 * xr);
    double ny = floor(y.h);
    ddv f = ddsub(y, dv(ny));
    if (f.h < 0) {
      ny -= 1.0;
      f = ddadd(f, dv(1.0));
    }
    ddv ef = dddiv(dv(1.0), exp2_neg_frac(f));
    wt[k] = ldexp(ddround(dddiv(ef, s)), (int)ny - 2 * E);
  }
}

}  // namespace

xc_status gauss_rule_device(int kind, double alpha, double beta, int64_t N64, double* x_out, double* w_out,
                            double* wt_out, int device) {
  if (N64 < 1 || N64 > (1 << 26)) {
    xc_set_error("gauss_rule: N out of range");
    return XC_EINVAL;
  }
  if (kind != XC_JACOBI && kind != XC_LAGUERRE) {
    xc_set_error("gauss_rule: kind must be XC_JACOBI or XC_LAGUERRE");
    return XC_EINVAL;
  }
  if (kind == XC_JACOBI && !(alpha > -1.0 && beta > -1.0)) {
    xc_set_error("gauss_rule: alpha, beta must be > -1");
    return XC_EINVAL;
  }
  XC_CUDA(cudaSetDevice(device));
  const int N = (int)N64;
  std::vector<double> d(N), e2(N, 0.0);
  std::vector<double2> tab;
  ddv p0 = dv(1.0);
  double lo, hi;
  if (kind == XC_JACOBI) {
    jacobi_coeffs(alpha, beta, N + 1, tab, p0);
    for (int n = 0; n < N; ++n) d[n] = tab[3 * n].x + tab[3 * n].y;
    for (int n = 1; n < N; ++n) {
      double a = tab[3 * n + 1].x;
      e2[n] = a * a;
    }
    lo = -1.0;
    hi = 1.0;
  } else {
    for (int n = 0; n < N; ++n) d[n] = 2.0 * n + 1.0;
    for (int n = 1; n < N; ++n) e2[n] = (double)n * n;
    lo = 0.0;
    hi = 4.0 * N + 2.0;
  }
  double emax = 1.0;
  for (int n = 1; n < N; ++n) emax = fmax(emax, e2[n]);
  double pivmin = 1e-300 * emax;
  DevBuf bd, be, bx, bw, bwt, btab;
  xc_status s = XC_OK;
  auto fin = [&]() {
    dev_free(bd); dev_free(be); dev_free(bx); dev_free(bw); dev_free(bwt); dev_free(btab);
  };
  if ((s = dev_alloc(bd, N * 8)) || (s = dev_alloc(be, N * 8)) || (s = dev_alloc(bx, N * 8)) ||
      (s = dev_alloc(bw, N * 8)) || (s = dev_alloc(bwt, N * 8)) ||
      (s = dev_alloc(btab, std::max<size_t>(16, tab.size() * sizeof(double2))))) {
    fin();
    return s;
  }
  cudaError_t ce = cudaSuccess;
  ce = cudaMemcpy(bd.p, d.data(), N * 8, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemcpy(be.p, e2.data(), N * 8, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && !tab.empty())
    ce = cudaMemcpy(btab.p, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) {
    sturm_bisect<<<(N + 127) / 128, 128>>>((double*)bd.p, (double*)be.p, N, lo, hi, pivmin, (double*)bx.p);
    ce = cudaGetLastError();
  }
  if (ce == cudaSuccess) {
    newton_cd<<<(N + 127) / 128, 128>>>(kind, (double2*)btab.p, p0, N, (double*)bx.p, (double*)bw.p,
                                        (double*)bwt.p, kind == XC_LAGUERRE ? 3 : 2);
    ce = cudaGetLastError();
  }
  if (ce == cudaSuccess) ce = cudaMemcpy(x_out, bx.p, N * 8, cudaMemcpyDeviceToHost);
  if (ce == cudaSuccess && w_out) ce = cudaMemcpy(w_out, bw.p, N * 8, cudaMemcpyDeviceToHost);
  if (ce == cudaSuccess && wt_out) ce = cudaMemcpy(wt_out, bwt.p, N * 8, cudaMemcpyDeviceToHost);
  fin();
  if (ce != cudaSuccess) {
    xc_set_error(std::string("gauss_rule: ") + cudaGetErrorString(ce));
    return XC_ECUDA;
  }
  return XC_OK;
}
