// build.h -- tile fill (build.cu)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/xc.h"

// Fill descriptor of one SpMM item: two M-tiles (g0, g1; -1 = empty) over the B rows
// [k0, k0 + 4 nsteps); tiles[a_off + 64 s + 2 lane + mt] is lane's A fragment of M-tile mt.
struct FillItem {
  int64_t a_off;
  int k0;
  int nsteps;
  int g0, g1;
};

enum { FILL_OUT_CPLX = 0, FILL_OUT_REAL = 1, FILL_IN_CPLX = 2, FILL_IN_REAL = 3 };

xc_status fill_tiles(int mode, const FillItem* fi, int n, const int* start, const int* len, const int64_t* off,
                     const double2* vals, const double* P, int t, int N, int H, double* tiles, cudaStream_t st);
