// xc_internal.cuh -- shared declarations of the libxc CUDA sources (product side).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/xc.h"

// ---------------------------------------------------------------------------
// Error-free fp64 pairs ("double-double") for the entry generation (R-5).
// Product-side implementation (host + device); independent of oracle/.
// ---------------------------------------------------------------------------
struct ddv {
  double h, l;
};

__host__ __device__ __forceinline__ ddv dv(double a) { return ddv{a, 0.0}; }
__host__ __device__ __forceinline__ ddv qsum(double a, double b) {
  double s = a + b;
  return ddv{s, b - (s - a)};
}
__host__ __device__ __forceinline__ ddv tsum(double a, double b) {
  double s = a + b;
  double v = s - a;
  return ddv{s, (a - (s - v)) + (b - v)};
}
__host__ __device__ __forceinline__ ddv tprod(double a, double b) {
  double p = a * b;
#ifdef __CUDA_ARCH__
  return ddv{p, __fma_rn(a, b, -p)};
#else
  return ddv{p, fma(a, b, -p)};
#endif
}
__host__ __device__ __forceinline__ ddv ddadd(ddv a, ddv b) {
  ddv s = tsum(a.h, b.h);
  ddv t = tsum(a.l, b.l);
  s.l += t.h;
  s = qsum(s.h, s.l);
  s.l += t.l;
  return qsum(s.h, s.l);
}
__host__ __device__ __forceinline__ ddv ddneg(ddv a) { return ddv{-a.h, -a.l}; }
__host__ __device__ __forceinline__ ddv ddsub(ddv a, ddv b) { return ddadd(a, ddneg(b)); }
__host__ __device__ __forceinline__ ddv ddmul(ddv a, ddv b) {
  ddv p = tprod(a.h, b.h);
#ifdef __CUDA_ARCH__
  p.l = __fma_rn(a.h, b.l, __fma_rn(a.l, b.h, p.l));
#else
  p.l += a.h * b.l + a.l * b.h;
#endif
  return qsum(p.h, p.l);
}
__host__ __device__ __forceinline__ ddv ddmuld(ddv a, double b) {
  ddv p = tprod(a.h, b);
#ifdef __CUDA_ARCH__
  p.l = __fma_rn(a.l, b, p.l);
#else
  p.l += a.l * b;
#endif
  return qsum(p.h, p.l);
}
__host__ __device__ __forceinline__ ddv dddiv(ddv a, ddv b) {
  double q1 = a.h / b.h;
  ddv r = ddsub(a, ddmuld(b, q1));
  double q2 = r.h / b.h;
  r = ddsub(r, ddmuld(b, q2));
  double q3 = r.h / b.h;
  return ddadd(qsum(q1, q2), dv(q3));
}
__host__ __device__ __forceinline__ ddv ddsqrt(ddv a) {
  if (a.h <= 0.0) return dv(0.0);
  double s = sqrt(a.h);
  ddv r = ddsub(a, tprod(s, s));
  return ddadd(dv(s), dv(r.h / (2.0 * s)));
}
__host__ __device__ __forceinline__ double ddround(ddv a) { return a.h + a.l; }

// ---------------------------------------------------------------------------
// Error handling
// ---------------------------------------------------------------------------
void xc_set_error(const std::string& msg);

#define XC_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e__ = (call);                                                          \
    if (e__ != cudaSuccess) {                                                          \
      xc_set_error(std::string(#call) + ": " + cudaGetErrorString(e__) + " @" +        \
                   __FILE__ + ":" + std::to_string(__LINE__));                         \
      return e__ == cudaErrorMemoryAllocation ? XC_ENOMEM : XC_ECUDA;                  \
    }                                                                                  \
  } while (0)

#define XC_TRY(call)                  \
  do {                                \
    xc_status s__ = (call);           \
    if (s__ != XC_OK) return s__;     \
  } while (0)

// ---------------------------------------------------------------------------
// Device buffers (owned by the handle)
// ---------------------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};
xc_status dev_alloc(DevBuf& b, size_t bytes);
void dev_free(DevBuf& b);

// One-time per-device setup (function attributes are per device): true the first time it is
// called for the current device with this mask.
#include <atomic>
inline bool first_on_device(std::atomic<unsigned long long>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const unsigned long long bit = 1ull << dev;
  return (mask.fetch_or(bit) & bit) == 0;
}
inline int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// ---------------------------------------------------------------------------
// FFT engine (fft.cu): batched complex FFT of 2-3-5-smooth length L along the
// slow axis of a batch-fastest layout, 1 pass (L <= 1024) or 2 passes
// (four-step, L = L1 * L2) through an L2-resident scratch.
// ---------------------------------------------------------------------------
enum FftPro { PRO_PLAIN = 0, PRO_XREAL = 2, PRO_XCPLX = 3 };  // PRO_XCPLX: XC_EXP input axis
enum FftEpi { EPI_PLAIN = 0, EPI_ZPLANES = 2, EPI_CY = 3 };  // EPI_CY: XC_EXP output (planar, W^{-1}, Fe2)

struct FftPlan {
  int L = 0, L1 = 0, L2 = 0;       // L = L1 * L2; single pass when L2 == 1
  int nf1 = 0, f1[12] = {0};       // radices of the first (or only) pass
  int nf2 = 0, f2[12] = {0};
  double2* tw1 = nullptr;          // e^{+2 pi i n / L1}, n < L1
  double2* tw2 = nullptr;          // e^{+2 pi i n / L2}
  double2* twL = nullptr;          // e^{+2 pi i n / L}  (two-pass only)
  DevBuf mem;
};

struct FftIO {
  // prologue sources
  const double2* src = nullptr; int64_t lds = 0;           // PRO_PLAIN
  const double2* Uc = nullptr; int64_t ldu = 0;            // c2r_run: half spectrum u_q at Uc[q*ldu + col], q <= M
  const double2* twh = nullptr; int M = 0;                 // c2r_run: e^{+2 pi i n / (2M)}, n < M
  int H = 0;
  const double* X = nullptr; int64_t ldx = 0;              // PRO_XREAL
  const double* winv = nullptr;                            // 1/w_p (PRO_XREAL, PRO_XCPLX)
  int64_t xpl = 0;                                         // PRO_XCPLX: offset of the imaginary plane of X
  int keep_lo = 0, keep_hi = 0, m_off = 0;
  // epilogue destinations
  double2* dst = nullptr; int64_t ldd = 0; int kmax = 0;    // EPI_PLAIN: bins [0,kmax)
  double* Y = nullptr; int64_t ldy = 0;                    // c2r_run: output rows
  const double* yscale = nullptr;                          // c2r_run / EPI_CY: 1/(sqrt(L) w_p)
  int64_t ypl = 0;                                         // EPI_CY: offset of the imaginary plane of Y
  double* zre = nullptr; double* zim = nullptr; int64_t ldz = 0;  // EPI_ZPLANES
  double scale = 1.0;                                      // EPI_PLAIN / EPI_ZPLANES
};

xc_status fft_plan_make(FftPlan& p, int L, bool c2r = false);

// Radix plan of a C2R sub-transform (c2r.cu, and its cost model in fft.cu): 8s, then 9s, then 6s
// (a 2 with a 3), then 4, 2, 5s, 3s -- few stages (every stage is a shared-memory round trip).
struct C2RRadices {
  int nf;
  int f[16];
};
constexpr C2RRadices c2r_radices(int R) {
  C2RRadices p{};
  int x = R;
  while (x % 8 == 0) { p.f[p.nf++] = 8; x /= 8; }
  while (x % 9 == 0) { p.f[p.nf++] = 9; x /= 9; }
  while (x % 6 == 0) { p.f[p.nf++] = 6; x /= 6; }
  while (x % 4 == 0) { p.f[p.nf++] = 4; x /= 4; }
  while (x % 2 == 0) { p.f[p.nf++] = 2; x /= 2; }
  while (x % 5 == 0) { p.f[p.nf++] = 5; x /= 5; }
  while (x % 3 == 0) { p.f[p.nf++] = 3; x /= 3; }
  if (x != 1) p.nf = -1;
  return p;
}  // c2r: split chosen for c2r_run
void fft_plan_free(FftPlan& p);
// sigma = -1 forward (Eq. 1), +1 inverse.  ncol columns.  scratch: L*ncol double2 (2-pass only).
xc_status fft_run(const FftPlan& p, int sigma, FftPro pro, FftEpi epi, const FftIO& io, int ncol,
                  double2* scratch, cudaStream_t st);
// Output-axis real-output inverse (c2r.cu): persistent prefetching passes, half spectrum
// io.Uc (ldu) -> Y rows (io.Y, ldy) with the W^{-1}/truncate epilogue.  scratch: M*ncol double2.
xc_status c2r_run(const FftPlan& p, const FftIO& io, int ncol, double2* scratch, cudaStream_t st);
// two-pass lengths run in column chunks of c2r_chunk_cols(p, ncol) columns (scratch: M x that)
int64_t c2r_chunk_cols(const FftPlan& p, int64_t ncol);
// kernel launches of c2r_run for ncol columns
int64_t c2r_launch_count(const FftPlan& p, int64_t ncol);
// the length's twiddle tables (allocated once per device; call at build time, not in an apply)
xc_status c2r_prepare(const FftPlan& p);
// 1 if c2r.cu has a 512-thread big-tile kernel for this pass (mode 0 first / 1 second) and length
bool c2r_has_big(int mode, int R);
// 1 if c2r.cu has a compile-time specialised kernel for this pass and length (the generic one runs
// ~1.4x the instructions)
bool c2r_has_spec(int mode, int R);
// 1 if c2r.cu has a "wide" kernel (512 threads, 6400-point tiles) for this pass and length
bool c2r_has_wide(int mode, int R);

// ---------------------------------------------------------------------------
// SpMM on the FP64 tensor cores (spmm.cu)
// Each item computes two 8 x (8*NT) output tiles D_mt = A_mt (8 x 4*nsteps) * Bm (mt = 0, 1)
// sharing the B fragments; row R of Bm is gathered from a source (plain rows or re/im planes).
// ---------------------------------------------------------------------------
struct SpmmItem {
  int64_t a_off;      // offset (doubles) of the A stream: 64 doubles per step (2 M-tiles x 32 lanes)
  int64_t out_row[2]; // first of the 8 output rows of M-tile 0 / 1 (-1: M-tile absent)
  int k0;             // first B row of the item (B row R -> plane R&1, row R>>1 for re/im sources)
  int nsteps;         // 4 B rows per step
  int src;            // index into SpmmSrcs
  int cplx;           // 1: output rows are 4 complex bins, stored interleaved (re, im) per column
};

// A window of B rows [r0, r1) (r1 - r0 <= XC_WMAX) and the items [i0, i1) inside it.
#define XC_WMAX 192
#define XC_WARPS 8  // warps per SpMM CTA
#define XC_WIN_ITEMS 128  // max items per SpMM window (the CTA stages them in shared memory)
struct SpmmWin {
  int r0, r1;
  int i0, i1;
  int src;
  int pad;
  int wo[XC_WARPS + 1];  // items [i0 + wo[w], i0 + wo[w+1]) run on warp w (balanced on the host)
};

#define XC_MAX_SRC 40
struct SpmmSrcs {
  const double* re[XC_MAX_SRC];
  const double* im[XC_MAX_SRC];   // null => plain rows (row r -> k0 + r)
  int nrows[XC_MAX_SRC];          // rows available (loads beyond are zero)
  int64_t ld[XC_MAX_SRC];
};

xc_status spmm_run(const SpmmWin* wins, int nwins, const SpmmItem* items, const double* tiles,
                   const SpmmSrcs& srcs, double* part, int64_t ldp, int ncols, cudaStream_t st);
int spmm_nt_for(int64_t B);

// ---------------------------------------------------------------------------
// Reductions of the partial sums (spmm.cu)
// ---------------------------------------------------------------------------
// Y[deg][b] = sum_c part[(base(g) + 8c + deg % 8)][b], g = deg / 8, deg in [0, t)
xc_status reduce_rows8(const double* part, int64_t ldp, const int64_t* base, const int* nch, int nrows,
                       const double* rowscale, double* Y, int64_t ldy, int ncols, int maxn, cudaStream_t st);

// ---------------------------------------------------------------------------
// Precompute kernels (gen.cu)
// ---------------------------------------------------------------------------
struct GenParams {
  int kind;            // XC_COS / XC_JACOBI / XC_LAGUERRE / XC_EXP (complex entries)
  int L;               // positions [0, L)
  int m_off;           // degree = position + m_off
  const double* nodes; // device, chunk
  int nc;              // nodes in chunk
  const double* w;     // window on L positions (device) or null (=1)
  const double2* jab;  // Jacobi: per n: (b_n.h, b_n.l), (a_n.h, a_n.l), (inva_n.h, inva_n.l) = 3 double2
  ddv p0;              // Jacobi p_0
  const double* nodes_lo = nullptr;  // XC_EXP: low parts of the nodes (t = hi + lo), or null
  const double2* cscale = nullptr;   // XC_EXP: per-node complex scale of the entries, or null
};
// F[p * nc + k] = (w_p * phi_{p+m_off}(x_k), 0)   (complex, batch = nodes)
xc_status gen_entries(const GenParams& g, double2* F, cudaStream_t st);
// E[j * ldE + k] = phi_j(x_k) (real), j in [0, L)
xc_status gen_entries_real(const GenParams& g, double* E, int64_t ldE, cudaStream_t st);

// Band detection and compaction on a spectrum chunk Spec[q * nc + k], q < H.
// circ: complex rows (XC_EXP), full circular spectrum of H = L bins; runs may wrap (mod H).
// Appendix A (appa.cu): truncated window spectrum xq (2Q+1, index m+Q) and W' = F* xq on the host;
// the per-node windowed spectra around each node's peak into spec (zeroed by the caller).
xc_status appa_window(const std::vector<double>& w, int L, double eps1, std::vector<double2>& xq, int& Q,
                      std::vector<double>& wq);
// Window mode (wm != null): only the 2W+1 bins around each node's peak, the kept run (start, len)
// found in the window, then appa_store copies it; spec may then be null.
struct AppAWin {
  double2* win;   // nc x (2W+1)
  int* start;
  int* len;
  int* wfirst;
  double* thr;
};
xc_status appa_spectra(int kind, int L, int H, int m_off, int Q, int W, const double* th, const double* tl,
                       const double2* cscale, const double2* xq, int nc, double eps1, double2* spec, int* flag,
                       cudaStream_t st, AppAWin* wm = nullptr);
xc_status appa_store(const AppAWin& wm, int W, const int64_t* off, double2* vals, int nc, cudaStream_t st);
// 2D block method (lag2d.cu, R-23): one kept entry of a D2 row: value, the row of the interleaved
// prologue spectra it multiplies (re) and whether that spectrum value is conjugated (im != 0)
struct Ent2D {
  double2 v;
  int re, im;
};
xc_status lag2d_scale_nodes(double2* F, int L, int nc, const double* w, cudaStream_t st);
xc_status lag2d_transpose(const double2* in, double2* out, int R, int C, cudaStream_t st);
xc_status lag2d_compact_rows(const double2* S, int rows, int cols, double eps1, unsigned long long* dmx, int* dcnt,
                             std::vector<int64_t>& ptr, DevBuf& q, DevBuf& v, cudaStream_t st);
xc_status lag2d_spmm(const int64_t* ptr, const Ent2D* ent, const int* order, int rows, const double2* z, int64_t ldz,
                     double2* U, int64_t ldu, int B, cudaStream_t st);
// The same product in 8 x 4 blocks on the FP64 tensor cores (device pointers, built by build_2d):
// groups of 8 u rows, their blocks cut into segments of at most kBsrSeg blocks (one warp each)
constexpr int kBsrSeg = 24;
struct Bsr2D {
  const int64_t* sptr;  // blocks of segment s: [sptr[s], sptr[s+1])
  const int* r4s;       // first z row of each block
  const double* tiles;  // 128 doubles per block: the Crr, Cri, Cir, Cii A fragments
  const int* srow;      // first u row of the segment's group
  const int* snv;       // valid rows of the group (<= 8)
  const int* sslot;     // -1: the group's only segment; else its partial slot
  const int* order;     // segments, most blocks first
  int nseg;
  const int* rrow;      // groups with several segments: u row, valid rows, first slot, slots
  const int* rnv;
  const int* rslot;
  const int* rcnt;
  int nred;
  int nslots;
};
xc_status lag2d_bsr(const Bsr2D& m, const double2* z, int64_t ldz, double2* U, int64_t ldu, double2* part, int B,
                    cudaStream_t st);
// Y[k][col] (+)= sum_j E[j * ldE + k] X[j][col]; part: optional scratch (part_cap doubles) for
// a split-j pass with a deterministic second-pass reduction
xc_status dense_tn(const double* E, int J, int K, int64_t ldE, const double* X, int64_t ldx, double* Y, int64_t ldy,
                   int B, bool acc, double* part, int64_t part_cap, cudaStream_t st);
// thr_abs2 > 0: the global threshold |S|^2 >= thr_abs2 (Alg. 1/2 step 1.3); else per node
// |S|^2 >= eps1^2 max_q |S[k,q]|^2 (R-3)
xc_status band_detect(const double2* spec, int H, int nc, double eps1, double thr_abs2, int* start, int* len,
                      bool circ, cudaStream_t st);
xc_status band_store(const double2* spec, int H, int nc, double eps1, double thr_abs2, const int* start,
                     const int* len, const int64_t* off, double2* vals, bool circ, cudaStream_t st);
// *out = max(*out, max_i |spec_i|^2) as the bit pattern of a non-negative double
xc_status spec_max2(const double2* spec, int64_t n, unsigned long long* out, cudaStream_t st);

// Gauss rules (gauss.cu)
xc_status gauss_rule_device(int kind, double alpha, double beta, int64_t N, double* x, double* w,
                            double* wt, int device);

// Host-side Jacobi recurrence coefficients in double-double (plan.cu)
void jacobi_coeffs(double alpha, double beta, int nmax, std::vector<double2>& tab, ddv& p0);
double jacobi_mu0(double alpha, double beta);

// ---------------------------------------------------------------------------
// Small operators (small.cu): the two-launch apply of XC_DIR_A for real kinds when every block's
// M = L/2 <= kSmallMaxM: a bin-major gather for all u_i and the tail, then every block's C2R in
// shared memory.
// ---------------------------------------------------------------------------
constexpr int kSmallMaxM = 4096;
constexpr int kSmallMaxBlocks = 8;
struct SmallOp {
  const int64_t* ptr;   // rows + 1: entries of row r at [ptr[r], ptr[r+1])
  const int* node;      // node index of each entry (ascending within a row)
  const double2* val;   // S_i[k, q] (block bins) or (phi_j(x_k), 0) (tail degrees)
  const int64_t* out;   // >= 0: complex u row (double2 units, ld = ldu); < 0: tail degree -out-1
  int rows;
  const int* longrows;  // rows with more than kSmallLong entries (one warp each)
  int nlong;
};
constexpr int kSmallLong = 64;
constexpr int kSmallSub = 4;  // lanes per short (row, column) of the gather (kSmallLong / kSmallSub loads each)
struct SmallBlk {
  int M, nf, f[16];
  int m_off, keep_lo, keep_hi;
  int64_t urow;           // first complex u row of the block
  const double2* twh;     // e^{+i pi n / M}, n < M (pairing)
  const double2* twM;     // e^{+2 pi i n / M}, n < M (stage twiddles)
  const double* yscale;   // 1 / (sqrt(L) w_p)
};
struct SmallBlocks {
  SmallBlk blk[kSmallMaxBlocks];
  int nb, maxM;
};
xc_status small_spmm(const SmallOp& op, const double* X, int64_t ldx, double2* U, int64_t ldu, double* Y, int64_t ldy,
                     int B, int N, cudaStream_t st);
xc_status small_c2r(const SmallBlocks& sb, const double2* U, int64_t ldu, double* Y, int64_t ldy, int B,
                    cudaStream_t st);
bool small_radices(int M, int* f, int& nf);
