// lag2d.cu -- kernels of the 2D (both-sided) block extra-component method for the time-domain
// Laguerre sum D c, D[i,j] = l_j(x_i) on an equispaced grid (SURVEY NEXT-1,
// reading R-23 in DESIGN.md).  Product side; independent of oracle/.
//
// Precompute helpers (per block pair): the time-axis window, a complex transpose, the block's
// max |D2|^2, per-row counts and the ordered compaction of the kept entries of the Hermitian half.
// Apply: the complex x complex CSR product u_b[k] = sum_e D2[k, q_e] z_{a_e}[q_e] over the
// prologue planes of all degree blocks (z[-q] = conj z[q]), and the dense tails.
#include <stdlib.h>

#include "xc_internal.cuh"

namespace {

// F[q * nc + k] *= w[k]  (the time-axis window W_b on the rows of the extended block)
__global__ void scale_nodes_k(double2* F, int64_t n, int nc, const double* __restrict__ w) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = w[i % nc];
  double2 v = F[i];
  F[i] = make_double2(v.x * s, v.y * s);
}

// out[c * R + r] = in[r * C + c]
__global__ void transpose_k(const double2* __restrict__ in, double2* __restrict__ out, int R, int C) {
  __shared__ double2 t[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = r0 + j, c = c0 + threadIdx.x;
    if (r < R && c < C) t[j][threadIdx.x] = in[(int64_t)r * C + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int c = c0 + j, r = r0 + threadIdx.x;
    if (r < R && c < C) out[(int64_t)c * R + r] = t[threadIdx.x][j];
  }
}

// *mx = max |S|^2 (non-negative doubles order like their bit patterns)
__global__ void maxabs2_k(const double2* __restrict__ S, int64_t n, unsigned long long* mx) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = S[i];
    m = fmax(m, v.x * v.x + v.y * v.y);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, (unsigned long long)__double_as_longlong(m));
}

// cnt[k] = #{q : |S[k, q]|^2 >= thr}, one warp per row
__global__ void count_rows_k(const double2* __restrict__ S, int rows, int cols, const unsigned long long* mx,
                             double eps1, int* cnt) {
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= rows) return;
  const double thr = eps1 * eps1 * __longlong_as_double((long long)*mx);
  int c = 0;
  for (int q = lane; q < cols; q += 32) {
    const double2 v = S[(int64_t)k * cols + q];
    c += (v.x * v.x + v.y * v.y >= thr) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[k] = c;
}

// kept entries of row k in ascending q at ptr[k] (ballot compaction), one warp per row
__global__ void scatter_rows_k(const double2* __restrict__ S, int rows, int cols, const unsigned long long* mx,
                               double eps1, const int64_t* __restrict__ ptr, int* qout, double2* vout) {
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= rows) return;
  const double thr = eps1 * eps1 * __longlong_as_double((long long)*mx);
  int64_t o = ptr[k];
  for (int q0 = 0; q0 < cols; q0 += 32) {
    const int q = q0 + lane;
    double2 v = make_double2(0.0, 0.0);
    if (q < cols) v = S[(int64_t)k * cols + q];
    const bool keep = q < cols && v.x * v.x + v.y * v.y >= thr;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int pos = __popc(bal & ((1u << lane) - 1u));
      qout[o + pos] = q;
      vout[o + pos] = v;
    }
    o += __popc(bal);
  }
}

// u[k][col] = sum_e v_e * z_e[col]; z_e = row re_e of the interleaved prologue spectra z (double2),
// conjugated when im_e != 0.  One warp per row; each lane owns CPL columns (lane + 32 c) of a
// 32*CPL-column tile; the row's entries are fetched 32 at a time (one per lane, coalesced) and
// broadcast with shuffles, so the z gathers of consecutive entries are independent loads.
template <int CPL>
__global__ void __launch_bounds__(256) csr2d_k(const int64_t* __restrict__ ptr, const Ent2D* __restrict__ ent,
                                                const int* __restrict__ order, int rows,
                                                const double2* __restrict__ z, int64_t ldz,
                                                double2* __restrict__ U, int64_t ldu, int B) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int k = order[r];  // rows longest first (the grid's tail is the short rows)
  const int cb = blockIdx.y * 32 * CPL + lane;
  double ar[CPL], ai[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) ar[c] = ai[c] = 0.0;
  const int64_t e0 = ptr[k], e1 = ptr[k + 1];
  for (int64_t eb = e0; eb < e1; eb += 32) {
    const int n = (e1 - eb) < 32 ? (int)(e1 - eb) : 32;
    Ent2D mine = {make_double2(0.0, 0.0), 0, 0};
    if (lane < n) mine = ent[eb + lane];
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
      const double vx = __shfl_sync(0xffffffffu, mine.v.x, j);
      const double vy0 = __shfl_sync(0xffffffffu, mine.v.y, j);
      const int row = __shfl_sync(0xffffffffu, mine.re, j), cj = __shfl_sync(0xffffffffu, mine.im, j);
      const double2* zr = z + (int64_t)row * ldz;
      // conj(z) = (xr, -xi): (vx + i vy)(xr - i xi) = conj((vx - i vy)(xr + i xi)) -- with
      // s = -1 for a conjugated entry: re = vx xr - s' vy xi, im = s'' ... written out:
      const double vy = cj ? -vy0 : vy0;       // value conjugated
      const double sg = cj ? -1.0 : 1.0;       // result conjugated
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = cb + 32 * c;
        if (col < B) {
          const double2 x = __ldg(zr + col);
          // t = (vx + i vy) x ;  conj case: conj((vx - i vy0) x) = (vx + i vy0) conj(x)
          const double tr = fma(vx, x.x, -vy * x.y), ti = fma(vx, x.y, vy * x.x);
          ar[c] += tr;
          ai[c] = fma(sg, ti, ai[c]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int col = cb + 32 * c;
    if (col < B) U[(int64_t)k * ldu + col] = make_double2(ar[c], ai[c]);
  }
}

// The same product on the FP64 tensor cores (BSR form): the rows of the stacked u_b in groups
// of 8, each group a list of 8 x 4 blocks over 4 consecutive rows r4.. of the interleaved prologue
// spectra z.  A block holds four DMMA A fragments (32 doubles each, element [i][j] at 4 i + j):
//   re += Crr z_re + Cri z_im,   im += Cir z_re + Cii z_im
// (a conjugated spectrum value folds into the signs of the coefficients).  One warp per (group,
// 32 columns): per block 4 A fragments (reused over 4 column tiles), per column tile one 16-byte
// z load per lane (both B fragments) and 4 DMMAs.
__device__ __forceinline__ void dmma2(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) bsr2d_k(Bsr2D m, const double2* __restrict__ z, int64_t ldz,
                                                double2* __restrict__ U, int64_t ldu, double2* __restrict__ part,
                                                int B) {
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= m.nseg) return;
  const int sg = m.order[w];
  const int c0 = blockIdx.y * 32;
  double dr[4][2], di[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) dr[t][0] = dr[t][1] = di[t][0] = di[t][1] = 0.0;
  const int zrow_l = lane & 3, zcol_l = lane >> 2;
  const int64_t e0 = m.sptr[sg], e1 = m.sptr[sg + 1];
  // software pipeline: the next block's A fragments and z row are loaded before this one's DMMAs
  double arr = 0, ari = 0, air = 0, aii = 0;
  int r4 = 0;
  if (e0 < e1) {
    const double* A = m.tiles + e0 * 128;
    arr = __ldg(A + lane); ari = __ldg(A + 32 + lane); air = __ldg(A + 64 + lane); aii = __ldg(A + 96 + lane);
    r4 = __ldg(m.r4s + e0);
  }
  for (int64_t e = e0; e < e1; ++e) {
    const double2* zr = z + (int64_t)(r4 + zrow_l) * ldz;
    double2 x[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int col = c0 + 8 * t + zcol_l;
      x[t] = col < B ? __ldg(zr + col) : make_double2(0.0, 0.0);
    }
    const double brr = arr, bri = ari, bir = air, bii = aii;
    if (e + 1 < e1) {
      const double* A = m.tiles + (e + 1) * 128;
      arr = __ldg(A + lane); ari = __ldg(A + 32 + lane); air = __ldg(A + 64 + lane); aii = __ldg(A + 96 + lane);
      r4 = __ldg(m.r4s + e + 1);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      dmma2(dr[t][0], dr[t][1], brr, x[t].x);
      dmma2(dr[t][0], dr[t][1], bri, x[t].y);
      dmma2(di[t][0], di[t][1], bir, x[t].x);
      dmma2(di[t][0], di[t][1], bii, x[t].y);
    }
  }
  const int i = lane >> 2;  // D fragment: row lane/4, columns 2 (lane%4) + {0, 1}
  const int slot = m.sslot[sg];
  double2* u;
  int64_t ld;
  if (slot < 0) {  // the group's only segment: straight into u
    if (i >= m.snv[sg]) return;
    u = U + (int64_t)(m.srow[sg] + i) * ldu;
    ld = ldu;
  } else {         // one of several segments: 8 partial rows, summed in order by bsr_reduce_k
    u = part + ((int64_t)slot * 8 + i) * B;
    ld = B;
  }
  (void)ld;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int col = c0 + 8 * t + 2 * (lane & 3);
    if (col < B) u[col] = make_double2(dr[t][0], di[t][0]);
    if (col + 1 < B) u[col + 1] = make_double2(dr[t][1], di[t][1]);
  }
}

// groups cut into several segments: u rows = sum of the segments' partial rows in segment order
__global__ void bsr_reduce_k(const int* __restrict__ rrow, const int* __restrict__ rnv, const int* __restrict__ rslot,
                             const int* __restrict__ rcnt, int nred, const double2* __restrict__ part,
                             double2* __restrict__ U, int64_t ldu, int B) {
  const int g = blockIdx.y;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nred || idx >= (int64_t)8 * B) return;
  const int i = (int)(idx / B), col = (int)(idx - (int64_t)i * B);
  if (i >= rnv[g]) return;
  double2 s = make_double2(0.0, 0.0);
  for (int c = 0; c < rcnt[g]; ++c) {
    const double2 v = part[((int64_t)(rslot[g] + c) * 8 + i) * B + col];
    s.x += v.x;
    s.y += v.y;
  }
  U[(int64_t)(rrow[g] + i) * ldu + col] = s;
}

__global__ void tail_reduce_k(const double* __restrict__ part, int nch, int K, int B, double* Y, int64_t ldy,
                              int acc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)K * B) return;
  const int k = (int)(i / B), col = (int)(i - (int64_t)k * B);
  double s = 0.0;
  for (int c = 0; c < nch; ++c) s += part[((int64_t)c * K + k) * B + col];
  double* y = Y + (int64_t)k * ldy + col;
  *y = acc ? *y + s : s;
}

// The tails (the direct method) on the FP64 tensor cores: Y[m][col] (+)= sum_j E[j * ldE + m] X[j][col], j in the
// chunk blockIdx.z (length JC, a multiple of 4).  One warp per 8 rows x 32 columns (4 DMMA column
// tiles): A fragment lane = E[k0 + lane%4][m0 + lane/4], B fragment lane = X[k0 + lane%4][col].
__global__ void __launch_bounds__(256) dense_tn_mma_k(const double* __restrict__ E, int J, int K, int64_t ldE,
                                                       const double* __restrict__ X, int64_t ldx, double* Y,
                                                       int64_t ldy, int B, int acc, int JC, double* part) {
  const int lane = threadIdx.x & 31;
  const int m0 = (blockIdx.y * 8 + (threadIdx.x >> 5)) * 8;
  if (m0 >= K) return;
  const int c0 = blockIdx.x * 32;
  const int j0 = blockIdx.z * JC, j1 = min(J, j0 + JC);
  const int am = m0 + (lane >> 2), kk = lane & 3;
  double d[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) d[t][0] = d[t][1] = 0.0;
  for (int k = j0; k < j1; k += 4) {
    const int kr = k + kk;
    const double a = (kr < j1 && am < K) ? __ldg(E + (int64_t)kr * ldE + am) : 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int col = c0 + 8 * t + (lane >> 2);
      const double b = (kr < j1 && col < B) ? __ldg(X + (int64_t)kr * ldx + col) : 0.0;
      dmma2(d[t][0], d[t][1], a, b);
    }
  }
  const int m = m0 + (lane >> 2);
  if (m >= K) return;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int col = c0 + 8 * t + 2 * (lane & 3) + q;
      if (col >= B) continue;
      if (part) {
        part[((int64_t)blockIdx.z * K + m) * B + col] = d[t][q];
      } else {
        double* y = Y + (int64_t)m * ldy + col;
        *y = acc ? *y + d[t][q] : d[t][q];
      }
    }
  }
}

}  // namespace

xc_status lag2d_scale_nodes(double2* F, int L, int nc, const double* w, cudaStream_t st) {
  const int64_t n = (int64_t)L * nc;
  scale_nodes_k<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(F, n, nc, w);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status lag2d_transpose(const double2* in, double2* out, int R, int C, cudaStream_t st) {
  transpose_k<<<dim3((C + 31) / 32, (R + 31) / 32), dim3(32, 8), 0, st>>>(in, out, R, C);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status lag2d_compact_rows(const double2* S, int rows, int cols, double eps1, unsigned long long* dmx, int* dcnt,
                             std::vector<int64_t>& ptr, DevBuf& q, DevBuf& v, cudaStream_t st) {
  XC_CUDA(cudaMemsetAsync(dmx, 0, sizeof(unsigned long long), st));
  const int64_t n = (int64_t)rows * cols;
  maxabs2_k<<<(unsigned)std::min<int64_t>(4 * 148 * 8, (n + 255) / 256), 256, 0, st>>>(S, n, dmx);
  count_rows_k<<<(rows + 7) / 8, 256, 0, st>>>(S, rows, cols, dmx, eps1, dcnt);
  XC_CUDA(cudaGetLastError());
  std::vector<int> cnt(rows);
  XC_CUDA(cudaMemcpyAsync(cnt.data(), dcnt, rows * sizeof(int), cudaMemcpyDeviceToHost, st));
  XC_CUDA(cudaStreamSynchronize(st));
  ptr.assign(rows + 1, 0);
  for (int k = 0; k < rows; ++k) ptr[k + 1] = ptr[k] + cnt[k];
  DevBuf dptr;
  XC_TRY(dev_alloc(dptr, ptr.size() * sizeof(int64_t)));
  XC_CUDA(cudaMemcpyAsync(dptr.p, ptr.data(), ptr.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  XC_TRY(dev_alloc(q, (size_t)std::max<int64_t>(1, ptr[rows]) * sizeof(int)));
  XC_TRY(dev_alloc(v, (size_t)std::max<int64_t>(1, ptr[rows]) * sizeof(double2)));
  scatter_rows_k<<<(rows + 7) / 8, 256, 0, st>>>(S, rows, cols, dmx, eps1, (const int64_t*)dptr.p, (int*)q.p,
                                                 (double2*)v.p);
  XC_CUDA(cudaGetLastError());
  XC_CUDA(cudaStreamSynchronize(st));
  dev_free(dptr);
  return XC_OK;
}

xc_status lag2d_spmm(const int64_t* ptr, const Ent2D* ent, const int* order, int rows, const double2* z, int64_t ldz,
                     double2* U, int64_t ldu, int B, cudaStream_t st) {
  if (rows <= 0) return XC_OK;
  static const int cpl = getenv("XC_CSR_CPL") ? atoi(getenv("XC_CSR_CPL")) : 4;
  if (cpl == 8 && B > 128)
    csr2d_k<8><<<dim3((rows + 7) / 8, (B + 255) / 256), 256, 0, st>>>(ptr, ent, order, rows, z, ldz, U, ldu, B);
  else if (cpl >= 4 && B > 64)
    csr2d_k<4><<<dim3((rows + 7) / 8, (B + 127) / 128), 256, 0, st>>>(ptr, ent, order, rows, z, ldz, U, ldu, B);
  else
    csr2d_k<2><<<dim3((rows + 7) / 8, (B + 63) / 64), 256, 0, st>>>(ptr, ent, order, rows, z, ldz, U, ldu, B);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status lag2d_bsr(const Bsr2D& m, const double2* z, int64_t ldz, double2* U, int64_t ldu, double2* part, int B,
                    cudaStream_t st) {
  if (m.nseg <= 0) return XC_OK;
  bsr2d_k<<<dim3((m.nseg + 7) / 8, (B + 31) / 32), 256, 0, st>>>(m, z, ldz, U, ldu, part, B);
  XC_CUDA(cudaGetLastError());
  if (m.nred > 0) {
    bsr_reduce_k<<<dim3((unsigned)((8 * B + 255) / 256), m.nred), 256, 0, st>>>(m.rrow, m.rnv, m.rslot, m.rcnt, m.nred,
                                                                                 part, U, ldu, B);
    XC_CUDA(cudaGetLastError());
  }
  return XC_OK;
}

xc_status dense_tn(const double* E, int J, int K, int64_t ldE, const double* X, int64_t ldx, double* Y, int64_t ldy,
                   int B, bool acc, double* part, int64_t part_cap, cudaStream_t st) {
  if (K <= 0 || J <= 0) return XC_OK;
  // long sums are cut into chunks of 128 (grid parallelism), reduced in a second pass
  int nch = (J + 127) / 128;
  if (nch > 1 && (!part || (int64_t)nch * K * B > part_cap)) nch = 1;
  const int JC = ((J + nch - 1) / nch + 3) / 4 * 4;
  nch = (J + JC - 1) / JC;
  dense_tn_mma_k<<<dim3((B + 31) / 32, (K + 63) / 64, nch), 256, 0, st>>>(E, J, K, ldE, X, ldx, Y, ldy, B, acc ? 1 : 0,
                                                                          JC, nch > 1 ? part : nullptr);
  XC_CUDA(cudaGetLastError());
  if (nch > 1) {
    const int64_t n = (int64_t)K * B;
    tail_reduce_k<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, nch, K, B, Y, ldy, acc ? 1 : 0);
    XC_CUDA(cudaGetLastError());
  }
  return XC_OK;
}
