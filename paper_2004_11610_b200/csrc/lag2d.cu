// lag2d.cu -- kernels of the 2D (both-sided) block extra-component method for the time-domain
// Laguerre sum D c, D[i,j] = l_j(x_i) on an equispaced grid (SURVEY NEXT-1,
// reading R-23 in DESIGN.md).  Product side; independent of oracle/.
//
// Precompute helpers (per block pair): the time-axis window, a complex transpose, the block's
// max |D2|^2, per-row counts and the ordered compaction of the kept entries of the Hermitian half.
// Apply: the complex x complex CSR product u_b[k] = sum_e D2[k, q_e] z_{a_e}[q_e] over the
// prologue planes of all degree blocks (z[-q] = conj z[q]), and the dense tails.
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

// u[k][col] = sum_e v_e * z_e[col]; z_e = zre[re_e] + i zim-row, conjugated when im_e < 0
// (row index -im_e - 1).  One warp per row; each lane owns CPL columns (lane + 32 c) of a
// 32*CPL-column tile; the row's entries are fetched 32 at a time (one per lane, coalesced) and
// broadcast with shuffles, so the z gathers of consecutive entries are independent loads.
template <int CPL>
__global__ void __launch_bounds__(256) csr2d_k(const int64_t* __restrict__ ptr, const Ent2D* __restrict__ ent,
                                                int rows, const double* __restrict__ z, int64_t ldz,
                                                double2* __restrict__ U, int64_t ldu, int B) {
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= rows) return;
  const int cb = blockIdx.y * 32 * CPL + lane;
  double ar[CPL], ai[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) ar[c] = ai[c] = 0.0;
  const int64_t e0 = ptr[k], e1 = ptr[k + 1];
  for (int64_t eb = e0; eb < e1; eb += 32) {
    const int n = (e1 - eb) < 32 ? (int)(e1 - eb) : 32;
    Ent2D mine = {make_double2(0.0, 0.0), 0, 0};
    if (lane < n) mine = ent[eb + lane];
    for (int j = 0; j < n; ++j) {
      const double vx = __shfl_sync(0xffffffffu, mine.v.x, j), vy = __shfl_sync(0xffffffffu, mine.v.y, j);
      const int re = __shfl_sync(0xffffffffu, mine.re, j), im = __shfl_sync(0xffffffffu, mine.im, j);
      const bool cj = im < 0;
      const double* zr = z + (int64_t)re * ldz;
      const double* zi = z + (cj ? -(int64_t)im - 1 : (int64_t)im) * ldz;
      const double sy = cj ? -vy : vy;  // conj(z): (xr, -xi); fold the sign into the value
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = cb + 32 * c;
        if (col < B) {
          const double xr = __ldg(zr + col), xi = __ldg(zi + col);
          // (vx + i vy)(xr + i s xi), s = +-1:  re = vx xr - s vy xi,  im = s vx xi + vy xr
          ar[c] = fma(vx, xr, fma(-sy, xi, ar[c]));
          ai[c] = fma(cj ? -vx : vx, xi, fma(vy, xr, ai[c]));
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

// Y[k][col] (+)= sum_j E[j * ldE + k] X[j][col]   (the direct method for the tails).
// One CTA per (row k, 32 columns); its 8 warps split j and are summed in a fixed order.
__global__ void __launch_bounds__(256) dense_tn_k(const double* __restrict__ E, int J, int K, int64_t ldE,
                                                   const double* __restrict__ X, int64_t ldx, double* Y,
                                                   int64_t ldy, int B, int acc) {
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;
  const int k = blockIdx.y;
  double s = 0.0;
  if (col < B)
    for (int j = w; j < J; j += 8) s = fma(__ldg(E + (int64_t)j * ldE + k), __ldg(X + (int64_t)j * ldx + col), s);
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && col < B) {
    double t = part[0][lane];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += part[i][lane];
    double* y = Y + (int64_t)k * ldy + col;
    *y = acc ? *y + t : t;
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

xc_status lag2d_spmm(const int64_t* ptr, const Ent2D* ent, int rows, const double* z, int64_t ldz, double2* U,
                     int64_t ldu, int B, cudaStream_t st) {
  if (rows <= 0) return XC_OK;
  csr2d_k<2><<<dim3((rows + 7) / 8, (B + 63) / 64), 256, 0, st>>>(ptr, ent, rows, z, ldz, U, ldu, B);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

xc_status dense_tn(const double* E, int J, int K, int64_t ldE, const double* X, int64_t ldx, double* Y, int64_t ldy,
                   int B, bool acc, cudaStream_t st) {
  if (K <= 0 || J <= 0) return XC_OK;
  dense_tn_k<<<dim3((B + 31) / 32, K), 256, 0, st>>>(E, J, K, ldE, X, ldx, Y, ldy, B, acc ? 1 : 0);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}
