// build.h -- tile fill (build.cu)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/xc.h"

// Fill descriptor of one M-tile of an SpMM item: group g over the B rows [k0, k0 + 4 nsteps)
// in slot mt (0 or 1) of the item's A stream; tiles[a_off + 64 s + 2 lane + mt] is lane's A
// fragment of that M-tile.
struct FillItem {
  int64_t a_off;
  int k0;       // first B row of the item's stream
  int nsteps;
  int g, mt;
  int lo, hi;   // this M-tile's own B rows: entries outside [lo, hi) are zero (a chunked
                // group must not count a row of its neighbouring chunk twice)
};

enum { FILL_OUT_CPLX = 0, FILL_OUT_REAL = 1, FILL_IN_CPLX = 2, FILL_IN_REAL = 3, FILL_OUT_CC = 4, FILL_IN_CC = 5 };

xc_status fill_tiles(int mode, const FillItem* fi, int n, const int* start, const int* len, const int64_t* off,
                     const double2* vals, const double* P, int t, int N, int H, double* tiles, cudaStream_t st);
