// plan.h -- host planning helpers (plan.cu)
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/xc.h"

// longest block chain (+ the dense tail) the apply's per-source tables hold (XC_MAX_SRC)
constexpr int XC_MAX_BLOCKS = 40;

struct PlanBlock {
  int L, m_off, keep_lo, keep_hi;
};
struct PlanOut {
  double zeta = 0;
  std::vector<PlanBlock> blocks;
  int tail = 0;
};

double kaiser_value(double zeta, int npts, int n);
void kaiser_window(double zeta, int L, std::vector<double>& w);
bool solve_zeta(double eps1, double& zeta);
int smooth5_even_ge(int n);
bool minimal_s(double zeta, int span, double eps2, bool two_sided, int& s_out);
xc_status make_chain(int kind, int64_t N, double eps1, double eps2, int cutoff, PlanOut& out);
