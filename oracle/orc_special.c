/*
 * oracle/orc_special.c -- TEST INFRASTRUCTURE ONLY (the CPU oracle).
 *
 * Plain, slow, obviously-correct evaluation of the special-function entries that
 * define the transform matrices of Terekhov, "An extra-component method for
 * evaluating fast matrix-vector multiplication with special functions"
 * (arXiv 2004.11610; /root/reference/PAPER.md = "P:<line>").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  It shares no code with the CUDA product path.
 *
 * Everything that goes through a three-term recurrence is carried in
 * double-double (two fp64 words, ~106-bit significand) and rounded to fp64 once
 * at the end, because the fp64 recurrence error grows with the degree
 * and would exceed the 10*eps parity bar at N = 16384+ (reading R-5).
 *
 * Functions (all fp64 in/out, node-major outputs):
 *   orc_jacobi_entries   p_m^(a,b)(x_k), orthonormal Jacobi (C-5)
 *   orc_laguerre_entries l_m(x_k) = exp(-x_k/2) L_m(x_k)
 *   orc_cos_entries      cos(pi * m * t_k)
 *   orc_sin_entries      sin(pi * m * t_k)  (with cos: e^{i pi m t_k}, NEXT-3)
 *   orc_gauss_newton     Newton polish of Gauss nodes + Christoffel weights
 *   orc_dense_apply      Y = A X or Y = A^T C with entries regenerated on the fly
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* double-double arithmetic (Dekker / Knuth error-free transformations)      */
/* ------------------------------------------------------------------------ */
typedef struct { double hi, lo; } dd;

static inline dd mk(double h, double l) { dd r; r.hi = h; r.lo = l; return r; }
static inline dd d2dd(double a) { return mk(a, 0.0); }
static inline dd two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return mk(s, (a - (s - bb)) + (b - bb));
}
static inline dd fast_two_sum(double a, double b) {
  double s = a + b;
  return mk(s, b - (s - a));
}
static inline dd two_prod(double a, double b) {
  double p = a * b;
  return mk(p, fma(a, b, -p));
}
static inline dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return fast_two_sum(s.hi, s.lo);
}
static inline dd dd_neg(dd a) { return mk(-a.hi, -a.lo); }
static inline dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
static inline dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return fast_two_sum(p.hi, p.lo);
}
static inline dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return fast_two_sum(p.hi, p.lo);
}
static inline dd dd_div(dd a, dd b) {
  double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul_d(b, q1));
  double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul_d(b, q2));
  double q3 = r.hi / b.hi;
  return dd_add(fast_two_sum(q1, q2), d2dd(q3));
}
static inline dd dd_sqrt(dd a) {
  if (a.hi <= 0.0) return d2dd(0.0);
  double x = sqrt(a.hi);
  /* one Newton step in dd: x + (a - x^2) / (2x) */
  dd x2 = two_prod(x, x);
  dd r = dd_sub(a, x2);
  return dd_add(d2dd(x), d2dd(r.hi / (2.0 * x)));
}
static inline double dd_round(dd a) { return a.hi + a.lo; }

/* ln 2 and 1/(2 ln 2) as double-double (mpmath, 200 bits). */
static const double LN2_HI = 0.6931471805599453, LN2_LO = 2.3190468138462996e-17;
static const double I2LN2_HI = 0.7213475204444817, I2LN2_LO = 1.0177636870465517e-17;

/* exp(-g) for 0 <= g < 0.7 by its Taylor series in double-double. */
static dd dd_exp_neg_small(dd g) {
  dd term = d2dd(1.0), sum = d2dd(1.0);
  dd mg = dd_neg(g);
  for (int n = 1; n < 40; ++n) {
    term = dd_div(dd_mul(term, mg), d2dd((double)n));
    sum = dd_add(sum, term);
    if (fabs(term.hi) < 1e-34) break;
  }
  return sum;
}

/* ------------------------------------------------------------------------ */
/* Jacobi orthonormal recurrence (chi_m read as the squared norm,  */
/* DESIGN.md reading R-4).  x p_n = a_{n+1} p_{n+1} + b_n p_n + a_n p_{n-1}.  */
/* ------------------------------------------------------------------------ */
typedef struct {
  int nmax;
  dd *a;      /* a[n], n >= 1 */
  dd *inva;   /* 1 / a[n]    */
  dd *b;      /* b[n], n >= 0 */
  dd p0;      /* p_0 = 1/sqrt(mu_0) */
} jac_coef;

static void jac_coef_init(jac_coef *c, double al, double be, int nmax, double mu0) {
  c->nmax = nmax;
  c->a = (dd *)malloc(sizeof(dd) * (nmax + 2));
  c->inva = (dd *)malloc(sizeof(dd) * (nmax + 2));
  c->b = (dd *)malloc(sizeof(dd) * (nmax + 2));
  dd A = d2dd(al), B = d2dd(be), AB = dd_add(A, B);
  /* b_0 = (beta - alpha) / (alpha + beta + 2) */
  c->b[0] = dd_div(dd_sub(B, A), dd_add(AB, d2dd(2.0)));
  c->a[0] = d2dd(0.0);
  c->inva[0] = d2dd(0.0);
  for (int n = 1; n <= nmax + 1; ++n) {
    dd N = d2dd((double)n);
    dd t = dd_add(dd_mul_d(N, 2.0), AB);                       /* 2n + a + b */
    /* b_n = (b^2 - a^2) / ((2n+a+b)(2n+a+b+2)) */
    c->b[n] = dd_div(dd_mul(dd_sub(B, A), AB), dd_mul(t, dd_add(t, d2dd(2.0))));
    dd a2;
    if (n == 1) {
      /* a_1^2 = 4 (1+a)(1+b) / ((2+a+b)^2 (3+a+b)) (cancelled form, valid for a+b = -1) */
      dd num = dd_mul_d(dd_mul(dd_add(A, d2dd(1.0)), dd_add(B, d2dd(1.0))), 4.0);
      dd den = dd_mul(dd_mul(t, t), dd_add(t, d2dd(1.0)));
      a2 = dd_div(num, den);
    } else {
      /* a_n^2 = 4 n (n+a)(n+b)(n+a+b) / ((2n+a+b)^2 (2n+a+b+1)(2n+a+b-1)) */
      dd num = dd_mul_d(dd_mul(dd_mul(N, dd_add(N, A)), dd_mul(dd_add(N, B), dd_add(N, AB))), 4.0);
      dd den = dd_mul(dd_mul(t, t), dd_mul(dd_add(t, d2dd(1.0)), dd_sub(t, d2dd(1.0))));
      a2 = dd_div(num, den);
    }
    c->a[n] = dd_sqrt(a2);
    c->inva[n] = dd_div(d2dd(1.0), c->a[n]);
  }
  /* mu_0 is passed in (computed by the caller with lgamma, a uniform scale) */
  c->p0 = dd_div(d2dd(1.0), dd_sqrt(d2dd(mu0)));
}
static void jac_coef_free(jac_coef *c) { free(c->a); free(c->inva); free(c->b); }

/* mu_0 = int_{-1}^{1} (1-x)^a (1+x)^b dx = 2^{a+b+1} G(a+1) G(b+1) / G(a+b+2) */
double orc_jacobi_mu0(double al, double be) {
  long double l = (al + be + 1.0L) * logl(2.0L) + lgammal(al + 1.0L) + lgammal(be + 1.0L) -
                  lgammal(al + be + 2.0L);
  return (double)expl(l);
}

/* out[k*(m1-m0) + (m-m0)] = p_m(x_k), m in [m0, m1) */
int orc_jacobi_entries(double al, double be, const double *x, int64_t nx, int m0, int m1,
                       double *out) {
  if (m1 <= m0 || nx <= 0) return 0;
  jac_coef c;
  jac_coef_init(&c, al, be, m1 + 1, orc_jacobi_mu0(al, be));
  int64_t W = m1 - m0;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = 0; k < nx; ++k) {
    dd X = d2dd(x[k]);
    dd pm1 = d2dd(0.0), p = c.p0;
    double *o = out + k * W;
    for (int n = 0; n < m1; ++n) {
      if (n >= m0) o[n - m0] = dd_round(p);
      /* p_{n+1} = ((x - b_n) p_n - a_n p_{n-1}) / a_{n+1} */
      dd t = dd_sub(dd_mul(dd_sub(X, c.b[n]), p), dd_mul(c.a[n], pm1));
      dd pn = dd_mul(t, c.inva[n + 1]);
      pm1 = p;
      p = pn;
    }
  }
  jac_coef_free(&c);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Laguerre functions l_n(x) = exp(-x/2) L_n(x), exponent-tracked */
/* L_{n+1} = ((2n+1-x) L_n - n L_{n-1}) / (n+1),  L_0 = 1, L_1 = 1 - x.      */
/* ------------------------------------------------------------------------ */
int orc_laguerre_entries(const double *x, int64_t nx, int m0, int m1, double *out) {
  if (m1 <= m0 || nx <= 0) return 0;
  int64_t W = m1 - m0;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = 0; k < nx; ++k) {
    double xk = x[k];
    /* exp(-x/2) = 2^{-y}, y = x / (2 ln 2) = ny + f, f in [0,1) */
    dd y = dd_mul_d(mk(I2LN2_HI, I2LN2_LO), xk);
    double ny = floor(y.hi);
    dd f = dd_sub(y, d2dd(ny));
    if (f.hi < 0) { ny -= 1.0; f = dd_add(f, d2dd(1.0)); }
    dd g = dd_mul(f, mk(LN2_HI, LN2_LO));          /* f ln2 in [0, ln2) */
    dd ef = dd_exp_neg_small(g);                  /* 2^{-f}            */
    long E = -(long)ny;                           /* binary exponent   */
    dd X = d2dd(xk);
    dd Lm1 = d2dd(0.0), L = d2dd(1.0);
    double *o = out + k * W;
    for (int n = 0; n < m1; ++n) {
      if (n >= m0) {
        dd v = dd_mul(L, ef);
        double r = dd_round(v);
        long e = E;
        if (e < -2200) r = 0.0;
        else r = ldexp(r, (int)e);
        o[n - m0] = r;
      }
      dd t = dd_sub(dd_mul(dd_sub(d2dd(2.0 * n + 1.0), X), L), dd_mul_d(Lm1, (double)n));
      dd Ln = dd_div(t, d2dd((double)(n + 1)));
      Lm1 = L;
      L = Ln;
      /* keep the pair in range: rescale by 2^{-/+512} */
      double a = fabs(L.hi);
      if (a > 0x1p512) {
        L = mk(ldexp(L.hi, -512), ldexp(L.lo, -512));
        Lm1 = mk(ldexp(Lm1.hi, -512), ldexp(Lm1.lo, -512));
        E += 512;
      } else if (a < 0x1p-512 && a > 0.0 && fabs(Lm1.hi) < 0x1p-512) {
        L = mk(ldexp(L.hi, 512), ldexp(L.lo, 512));
        Lm1 = mk(ldexp(Lm1.hi, 512), ldexp(Lm1.lo, 512));
        E -= 512;
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* cos(pi * m * t_k) (P:66-70 with theta = pi t; m may be negative).   */
/* m * t is exact in double-double; the reduction mod 2 is exact; the cosine  */
/* of the reduced argument is evaluated in 80-bit long double and rounded.    */
/* ------------------------------------------------------------------------ */
static double cospi_exact_product(double m, double t) {
  dd r = two_prod(m, t);                 /* exact */
  double n2 = 2.0 * nearbyint(r.hi * 0.5);
  r = dd_sub(r, d2dd(n2));                /* exact: subtract an even integer */
  long double a = (long double)r.hi + (long double)r.lo;
  const long double PI_L = 3.141592653589793238462643383279502884L;
  return (double)cosl(PI_L * a);
}

/* sin(pi * m * t_k), same exact argument reduction (the imaginary part of e^{i pi m t}). */
static double sinpi_exact_product(double m, double t) {
  dd r = two_prod(m, t);
  double n2 = 2.0 * nearbyint(r.hi * 0.5);
  r = dd_sub(r, d2dd(n2));
  long double a = (long double)r.hi + (long double)r.lo;
  const long double PI_L = 3.141592653589793238462643383279502884L;
  return (double)sinl(PI_L * a);
}

int orc_sin_entries(const double *t, int64_t nx, int m0, int m1, int m_off, double *out) {
  if (m1 <= m0 || nx <= 0) return 0;
  int64_t W = m1 - m0;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nx; ++k)
    for (int m = m0; m < m1; ++m)
      out[k * W + (m - m0)] = sinpi_exact_product((double)(m + m_off), t[k]);
  return 0;
}

int orc_cos_entries(const double *t, int64_t nx, int m0, int m1, int m_off, double *out) {
  if (m1 <= m0 || nx <= 0) return 0;
  int64_t W = m1 - m0;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nx; ++k)
    for (int m = m0; m < m1; ++m)
      out[k * W + (m - m0)] = cospi_exact_product((double)(m + m_off), t[k]);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Gauss rules: Newton polish in double-double + Christoffel-Darboux weights  */
/* kind 2 = Jacobi(al,be) on [-1,1] (orthonormal p_n), kind 3 = Laguerre.     */
/* x: in = initial guesses (fp64), out = polished nodes.                      */
/* w: Gauss weights; wt (Laguerre only): w_k e^{x_k} = 1 / sum_j l_j(x_k)^2.  */
/* iters double-double Newton steps (p_N / p_N').                             */
/* ------------------------------------------------------------------------ */
int orc_gauss_newton(int kind, double al, double be, int64_t N, double *x, double *w, double *wt,
                     int iters) {
  jac_coef c;
  int jac = (kind == 2);
  if (jac) jac_coef_init(&c, al, be, (int)N + 1, orc_jacobi_mu0(al, be));
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : bad)
  for (int64_t k = 0; k < N; ++k) {
    dd X = d2dd(x[k]);
    dd pN = d2dd(0.0), dpN = d2dd(1.0), pNm1 = d2dd(0.0), dpNm1 = d2dd(0.0);
    long E = 0;
    for (int it = 0; it <= iters; ++it) {
      dd pm1 = d2dd(0.0), p, dpm1 = d2dd(0.0), dp = d2dd(0.0);
      E = 0;
      if (jac) p = c.p0; else p = d2dd(1.0);
      for (int n = 0; n < N; ++n) {
        dd pn, dpn;
        if (jac) {
          dd xb = dd_sub(X, c.b[n]);
          pn = dd_mul(dd_sub(dd_mul(xb, p), dd_mul(c.a[n], pm1)), c.inva[n + 1]);
          dpn = dd_mul(dd_add(dd_sub(dd_mul(xb, dp), dd_mul(c.a[n], dpm1)), p), c.inva[n + 1]);
        } else {
          dd cf = dd_sub(d2dd(2.0 * n + 1.0), X);
          dd inv = dd_div(d2dd(1.0), d2dd((double)(n + 1)));
          pn = dd_mul(dd_sub(dd_mul(cf, p), dd_mul_d(pm1, (double)n)), inv);
          dpn = dd_mul(dd_sub(dd_sub(dd_mul(cf, dp), dd_mul_d(dpm1, (double)n)), p), inv);
        }
        pm1 = p; p = pn; dpm1 = dp; dp = dpn;
        double a = fmax(fabs(p.hi), fabs(dp.hi));
        if (a > 0x1p400) {
          p = mk(ldexp(p.hi, -400), ldexp(p.lo, -400));
          pm1 = mk(ldexp(pm1.hi, -400), ldexp(pm1.lo, -400));
          dp = mk(ldexp(dp.hi, -400), ldexp(dp.lo, -400));
          dpm1 = mk(ldexp(dpm1.hi, -400), ldexp(dpm1.lo, -400));
          E += 400;
        }
      }
      pN = p; dpN = dp; pNm1 = pm1; dpNm1 = dpm1;
      if (it < iters) X = dd_sub(X, dd_div(pN, dpN));
      /* the weights are evaluated at the fp64 node actually returned */
      if (it == iters - 1) X = d2dd(dd_round(X));
    }
    double xr = dd_round(X);
    if (!isfinite(xr)) bad++;
    x[k] = xr;
    /* Christoffel-Darboux: sum_{j<N} p_j(x)^2 = a_N (p_N' p_{N-1} - p_N p_{N-1}') */
    dd cd = dd_sub(dd_mul(dpN, pNm1), dd_mul(pN, dpNm1));
    if (jac) {
      dd s = dd_mul(c.a[N], cd);               /* scale 2^{2E}, E = 0 for Jacobi */
      w[k] = dd_round(dd_div(d2dd(1.0), s));
      if (wt) wt[k] = w[k];
    } else {
      /* Laguerre (L_n orthonormal in e^{-x}): p_n = (-1)^n L_n has a_N = N, so
         sum_j L_j^2 = -N (L_N' L_{N-1} - L_N L_{N-1}') ; stored values are 2^{-E} true */
      dd s = dd_mul_d(cd, -(double)N);
      /* w = 1/(s 2^{2E}); wt = e^x w = 2^{x/ln2 - 2E} / s */
      double ls = log2(fabs(s.hi)) + 2.0 * E;
      w[k] = ldexp(dd_round(dd_div(d2dd(1.0), s)), (int)(-2 * E));
      dd yx = dd_mul_d(mk(I2LN2_HI, I2LN2_LO), 2.0 * xr);     /* x / ln 2 */
      double ny = floor(yx.hi);
      dd f = dd_sub(yx, d2dd(ny));
      if (f.hi < 0) { ny -= 1; f = dd_add(f, d2dd(1.0)); }
      /* 2^{f} = 1 / 2^{-f} */
      dd ef = dd_div(d2dd(1.0), dd_exp_neg_small(dd_mul(f, mk(LN2_HI, LN2_LO))));
      dd v = dd_div(ef, s);
      (void)ls;
      if (wt) wt[k] = ldexp(dd_round(v), (int)(ny - 2 * E));
    }
  }
  if (jac) jac_coef_free(&c);
  return bad;
}

/* ------------------------------------------------------------------------ */
/* Dense products (the "direct method"): entries regenerated per node  */
/* in double-double, fp64 accumulation in ascending node order.               */
/*   dir 1: Y[j,b] = sum_k phi_j(x_k) X[k,b], j < nout    (Y = A X)           */
/*   dir 2: Y[k,b] = sum_j phi_j(x_k) X[j,b], j < ndeg    (Y = A^T X)         */
/* kind 1 = cos(pi m t) (m_off applies), 2 = Jacobi(al,be), 3 = Laguerre.     */
/* X is row-major (rows x B), ldx = B.                                        */
/* ------------------------------------------------------------------------ */
static int entries(int kind, double al, double be, int m_off, const double *x, int64_t nx,
                   int m0, int m1, double *out) {
  if (kind == 1) return orc_cos_entries(x, nx, m0, m1, m_off, out);
  if (kind == 2) return orc_jacobi_entries(al, be, x, nx, m0, m1, out);
  if (kind == 3) return orc_laguerre_entries(x, nx, m0, m1, out);
  return -1;
}

int orc_dense_apply(int kind, double al, double be, int dir, const double *nodes, int64_t N,
                    int64_t ndeg, const double *X, int64_t B, double *Y) {
  const int64_t KB = 64; /* node block */
  double *E = (double *)malloc(sizeof(double) * KB * ndeg);
  if (!E) return -2;
  if (dir == 1) memset(Y, 0, sizeof(double) * ndeg * B);
  for (int64_t k0 = 0; k0 < N; k0 += KB) {
    int64_t nk = (N - k0 < KB) ? (N - k0) : KB;
    entries(kind, al, be, 0, nodes + k0, nk, 0, (int)ndeg, E); /* E[kk*ndeg + j] */
    if (dir == 1) {
#pragma omp parallel for schedule(static)
      for (int64_t j = 0; j < ndeg; ++j) {
        double *y = Y + j * B;
        for (int64_t kk = 0; kk < nk; ++kk) {
          double e = E[kk * ndeg + j];
          const double *xr = X + (k0 + kk) * B;
          for (int64_t b = 0; b < B; ++b) y[b] += e * xr[b];
        }
      }
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t kk = 0; kk < nk; ++kk) {
        double *y = Y + (k0 + kk) * B;
        for (int64_t b = 0; b < B; ++b) y[b] = 0.0;
        for (int64_t j = 0; j < ndeg; ++j) {
          double e = E[kk * ndeg + j];
          const double *xr = X + j * B;
          for (int64_t b = 0; b < B; ++b) y[b] += e * xr[b];
        }
      }
    }
  }
  free(E);
  return 0;
}
