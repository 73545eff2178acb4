// build.h -- tile fill (build.cu)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/xc.h"

struct FillItem {
  int64_t a_off;
  int k0;
  int nsteps;
  int g;
  int pad;
};

enum { FILL_OUT_CPLX = 0, FILL_OUT_REAL = 1, FILL_IN_CPLX = 2, FILL_IN_REAL = 3 };

xc_status fill_tiles(int mode, const FillItem* fi, int n, const int* start, const int* len, const int64_t* off,
                     const double2* vals, const double* P, int t, int N, int H, double* tiles, cudaStream_t st);
