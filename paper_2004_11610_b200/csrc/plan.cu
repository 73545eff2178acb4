// plan.cu -- host planning of the extra-component method (product side).
//
//  zeta(eps1): Newton for 1/I0(zeta) = eps1 from zeta0 = 50, applied to the
//              equivalent ln I0(zeta) = -ln eps1 (R-7);
//  s(zeta, eps2): smallest s with w_s >= eps2 on the block window (R-2 of P:184);
//  L: smallest even 2-3-5-smooth length >= span + s (R-9);
//  block chain: extra columns on the right only, the first s_i degrees handed to
//              the next block, dense tail below the cutoff (R-8).
//  Jacobi recurrence coefficients in double-double (R-4).
#include <math.h>

#include <vector>

#include "plan.h"
#include "xc_internal.cuh"

// I0 and I1 by their power series in long double (64-bit significand).
long double bessel_i0l(long double x) {
  long double q = 0.25L * x * x, t = 1.0L, s = 1.0L;
  for (int k = 1; k < 500; ++k) {
    t *= q / ((long double)k * k);
    s += t;
    if (t < 1e-22L * s) break;
  }
  return s;
}
long double bessel_i1l(long double x) {
  long double q = 0.25L * x * x, t = 0.5L * x, s = t;
  for (int k = 1; k < 500; ++k) {
    t *= q / ((long double)k * (k + 1));
    s += t;
    if (t < 1e-22L * s) break;
  }
  return s;
}

double kaiser_value(double zeta, int npts, int n) {
  // w_n^{zeta,npts} = I0(zeta sqrt(1 - (2n/npts - 1)^2)) / I0(zeta)
  long double r = ((long double)2 * n - npts) / (long double)npts;
  long double a = 1.0L - r * r;
  if (a < 0) a = 0;
  return (double)(bessel_i0l(zeta * sqrtl(a)) / bessel_i0l(zeta));
}

void kaiser_window(double zeta, int L, std::vector<double>& w) {
  w.resize(L);
  long double i0z = bessel_i0l(zeta);
  int npts = L - 1;
  for (int n = 0; n < L; ++n) {
    long double r = ((long double)2 * n - npts) / (long double)npts;
    long double a = 1.0L - r * r;
    if (a < 0) a = 0;
    w[n] = (double)(bessel_i0l(zeta * sqrtl(a)) / i0z);
  }
}

bool solve_zeta(double eps1, double& zeta) {
  long double z = 50.0L, target = -logl((long double)eps1);
  for (int it = 0; it < 200; ++it) {
    long double i0 = bessel_i0l(z);
    long double step = (logl(i0) - target) / (bessel_i1l(z) / i0);
    z -= step;
    if (fabsl(step) < 1e-15L * (z > 1 ? z : 1)) {
      zeta = (double)z;
      return true;
    }
  }
  return false;
}

int smooth5_even_ge(int n) {
  int m = n < 2 ? 2 : n + (n & 1);
  for (;; m += 2) {
    int r = m;
    while (r % 2 == 0) r /= 2;
    while (r % 3 == 0) r /= 3;
    while (r % 5 == 0) r /= 5;
    if (r == 1) return m;
  }
}

bool minimal_s(double zeta, int span, double eps2, bool two_sided, int& s_out) {
  for (int s = 1; s < 4 * span + 64; ++s) {
    int L = span + (two_sided ? 2 * s : s);
    if (kaiser_value(zeta, L - 1, s) >= eps2) {
      s_out = s;
      return true;
    }
  }
  return false;
}

xc_status make_chain(int kind, int64_t N, double eps1, double eps2, int cutoff, PlanOut& out) {
  if (!solve_zeta(eps1, out.zeta)) {
    xc_set_error("zeta Newton did not converge");
    return XC_ENUMERIC;
  }
  out.blocks.clear();
  if (kind == XC_COS || kind == XC_EXP) {  // trigonometric: one block, extras on both sides
    int s0;
    if (!minimal_s(out.zeta, (int)N, eps2, true, s0)) {
      xc_set_error("s search did not terminate");
      return XC_ENUMERIC;
    }
    int L = smooth5_even_ge((int)N + 2 * s0);
    int s = (L - (int)N) / 2;
    out.blocks.push_back(PlanBlock{L, -s, s, s + (int)N});
    out.tail = 0;
    return XC_OK;
  }
  int e = (int)N;
  while (e > cutoff) {
    int s0;
    if (!minimal_s(out.zeta, e, eps2, false, s0)) {
      xc_set_error("s search did not terminate");
      return XC_ENUMERIC;
    }
    int L = smooth5_even_ge(e + s0);
    int s = L - e;
    // the chain must shrink (the next block holds the first s_i degrees of this one);
    // s >= e happens only for eps2 close to 1 -- reject instead of looping
    if (s >= e) {
      xc_set_error("block chain does not shrink (s >= span): eps2 too close to 1");
      return XC_ENUMERIC;
    }
    if ((int)out.blocks.size() + 1 >= XC_MAX_BLOCKS) {
      xc_set_error("block chain longer than " + std::to_string(XC_MAX_BLOCKS - 1) + " blocks");
      return XC_ENUMERIC;
    }
    out.blocks.push_back(PlanBlock{L, 0, s, e});
    e = s;
  }
  out.tail = e;
  return XC_OK;
}

double jacobi_mu0(double a, double b) {
  long double l = (a + b + 1.0L) * logl(2.0L) + lgammal(a + 1.0L) + lgammal(b + 1.0L) - lgammal(a + b + 2.0L);
  return (double)expl(l);
}

// tab[3n+0] = b_n, tab[3n+1] = a_n, tab[3n+2] = 1/a_n (each as (hi, lo)), n = 0..nmax
void jacobi_coeffs(double alpha, double beta, int nmax, std::vector<double2>& tab, ddv& p0) {
  tab.assign(3 * (size_t)(nmax + 1), make_double2(0, 0));
  ddv A = dv(alpha), B = dv(beta), AB = ddadd(A, B), one = dv(1.0), two = dv(2.0);
  auto put = [&](int i, ddv v) { tab[i] = make_double2(v.h, v.l); };
  put(0, dddiv(ddsub(B, A), ddadd(AB, two)));
  for (int n = 1; n <= nmax; ++n) {
    ddv Nn = dv((double)n);
    ddv t = ddadd(ddmuld(Nn, 2.0), AB);
    put(3 * n, dddiv(ddmul(ddsub(B, A), AB), ddmul(t, ddadd(t, two))));
    ddv a2;
    if (n == 1) {
      a2 = dddiv(ddmuld(ddmul(ddadd(A, one), ddadd(B, one)), 4.0), ddmul(ddmul(t, t), ddadd(t, one)));
    } else {
      ddv num = ddmuld(ddmul(ddmul(Nn, ddadd(Nn, A)), ddmul(ddadd(Nn, B), ddadd(Nn, AB))), 4.0);
      ddv den = ddmul(ddmul(t, t), ddmul(ddadd(t, one), ddsub(t, one)));
      a2 = dddiv(num, den);
    }
    ddv an = ddsqrt(a2);
    put(3 * n + 1, an);
    put(3 * n + 2, dddiv(one, an));
  }
  p0 = dddiv(one, ddsqrt(dv(jacobi_mu0(alpha, beta))));
}
