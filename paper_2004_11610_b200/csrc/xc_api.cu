// xc_api.cu -- the C ABI (include/xc.h): build orchestration and apply.
//
// Precomputation (xc_build_compressed; Alg. 1/2 step 1):
//   host plan (zeta, s_i, L_i, tail)  ->  per block, per node chunk on the GPU:
//   entries (double-double) x window -> forward FFT (Eq. 1) -> per-node threshold ->
//   node bands  ->  tensor-core tiles for the output axis (bin groups x nodes) and,
//   if requested, the input axis (node groups x bins).
// Computation (xc_apply):
//   XC_DIR_A  : SpMM (all blocks + dense tail, one launch) -> per block inverse FFT
//               with the partial-sum reduction fused in its prologue and the
//               W^{-1}/truncation fused in its epilogue (Alg. 2 step 2);
//               tail rows reduced directly.
//   XC_DIR_WAT: per block inverse FFT of pad(X)/w (Alg. 1 step 2.2 / Fe1, Fe3) ->
//               SpMM over all blocks + tail -> reduction times the weights.
#include <math.h>
#include <cmath>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <algorithm>
#include <array>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "build.h"
#include "plan.h"
#include "xc_internal.cuh"

static_assert(XC_MAX_BLOCKS == XC_MAX_SRC, "block chain bound = apply source table size");

static thread_local std::string g_err;
void xc_set_error(const std::string& msg) { g_err = msg; }

xc_status dev_alloc(DevBuf& b, size_t bytes) {
  dev_free(b);
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    b.p = nullptr;
    cudaGetLastError();
    xc_set_error("cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    return XC_ENOMEM;
  }
  b.bytes = bytes;
  return XC_OK;
}
void dev_free(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

namespace {

constexpr int KC = 184;      // node chunk of a split output-axis item (multiple of 4, <= XC_WMAX)
constexpr int KSPLIT = 184;  // blocks whose bin groups span more nodes than this are split
constexpr int QC = 64;       // bin chunk of an input-axis item (2 QC B rows <= XC_WMAX)
constexpr int WIN_ITEMS = XC_WIN_ITEMS;  // max items per SpMM window (CTA)

struct BlockData {
  int L = 0, H = 0, m_off = 0, keep_lo = 0, keep_hi = 0;
  FftPlan fft;   // length L: precompute (forward) and the input-axis prologue
  FftPlan fftM;  // length M = L/2: output-axis real-output inverse (C2R)
  DevBuf twh;    // e^{+2 pi i n / L}, n < M
  bool split = false;
  int64_t ubase = 0;  // first U row of the block in the output-axis partial array
  std::vector<double> h_w;
  DevBuf w, yscale, winv;
  std::vector<int> h_start, h_len;
  std::vector<int64_t> h_off;
  DevBuf start, len, off, vals;
  int64_t nnz = 0;
  int max_band = 0;
  int appQ = -1;  // Appendix A precompute: Q of the truncated window spectrum (-1: direct)
  double gmax2 = 0;  // thresh_mode = 1: max |S|^2 over the whole block (all ranks)
  int ngroups = 0;
  int64_t loc_count = 0;  // values of the locally computed node range (distributed precompute)
  DevBuf grp_base, grp_nch;  // output axis groups
  int grp_nch_max = 0;       // the longest chunk chain (reduce_rows8's instance)
};

template <typename T>
xc_status upload(DevBuf& b, const std::vector<T>& v) {
  XC_TRY(dev_alloc(b, v.size() * sizeof(T)));
  if (!v.empty()) XC_CUDA(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return XC_OK;
}

}  // namespace

// One workspace of xc_apply: the per-call scratch arrays for up to B columns, carved from one
// device range (ws_layout), plus the forked block streams and the captured graphs that use them.
constexpr int kAux = 4;  // forked streams: block 2 alone, blocks 3.. round robin over 3
struct GraphEntry {      // CUDA graph of one xc_apply argument set (captured at its 2nd call)
  const void* X;
  void* Y;
  int64_t ldx, ldy, B;
  int dir;
  cudaStream_t st;
  int seen;
  cudaGraphExec_t exec;
};
struct Ws {
  int64_t B = 0;              // columns the layout is carved for (0: none yet)
  DevBuf own;                 // the handle's own workspace; empty for an attached one
  char* base = nullptr;       // device range (own.p or the caller's)
  size_t bytes = 0;
  cudaStream_t bound = nullptr;  // attached: the stream it serves
  double* partA = nullptr;    // output axis: SpMM rows (u of every block, split-K partials, tail)
  double* partW = nullptr;    // input axis: SpMM partial rows
  double* zpl = nullptr;      // input axis / 2D: prologue spectra (z' planes)
  double* tailpart = nullptr; // 2D: split-j partial sums of the tails
  double2* bsr_part = nullptr;  // 2D: partial rows of the split DMMA groups
  double2* scratch = nullptr;   // FFT scratch of the caller's stream
  double2* scratch_aux[kAux] = {};  // ... and of each forked stream
  std::vector<int64_t> zoff;  // per block offset (doubles) of its z' planes in zpl
  cudaStream_t s_aux[kAux] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kAux] = {};
  int naux = 2;               // forked streams of the current apply (naux_for)
  std::vector<GraphEntry> graphs;
  std::vector<std::pair<size_t, size_t>> guards;  // debug guard zones (XC_WS_GUARD): offset, bytes
};

struct xc_op {
  int kind = 0;   // machinery kind (XC_LAGSPEC runs as XC_EXP, R-21)
  int ukind = 0;  // the kind the caller built
  bool appA = false;  // Appendix A trig precompute (R-22)
  int thresh_mode = 0;  // 0: per-node relative threshold (R-3); 1: global
  int apply_path = 0;   // xc_params.apply_path: 0 auto, 1 tiled, 2 small (two launches)
  bool small_on = false;   // XC_DIR_A runs the small-operator path (small.cu)
  DevBuf sm_ptr, sm_node, sm_val, sm_out, sm_twM, sm_long;  // its bin-major operator and stage twiddles
  SmallOp sm_op{};
  SmallBlocks sm_blocks{};
  std::vector<double> user_nodes, user_wt;  // the caller's nodes / weights (xc_export)
  double eta = 0;
  int dense_cutoff = 32;
  DevBuf tailR, tailC;  // XC_LAG2D: direct-method tails (rows i < t: N x t; columns j < t: t x (N-t))
  DevBuf ptr2d, ent2d, order2d;  // XC_LAG2D: CSR of the Hermitian halves of sum_a D2_ab, time blocks
  int rows2d = 0;                 // stacked; order2d: rows longest first
  DevBuf bsr_sptr, bsr_r4, bsr_tiles, bsr_srow, bsr_snv, bsr_sslot, bsr_order;  // XC_LAG2D: 8 x 4
  DevBuf bsr_rrow, bsr_rnv, bsr_rslot, bsr_rcnt;                       // DMMA blocks
  int bsr_nseg = 0, bsr_nred = 0, bsr_nslots = 0;
  int64_t zrows2d = 0;  // rows of the stacked prologue spectra
  double alpha = 0, beta = 0;
  int64_t N = 0;  // nodes
  int64_t M = 0;  // degrees (rows of A); == N unless rectangular
  DevBuf nodes_lo, cscale;  // XC_LAGSPEC: low parts of t_j, per-node scale 1/(eta/2 - i k_j)
  double eps1 = 0, eps2 = 0, zeta = 0;
  int tail = 0, dirs = 0, device = 0;
  std::vector<BlockData> blocks;
  DevBuf nodes, wt, tailP;
  // output axis
  DevBuf itemsA, tilesA, winsA;
  int nitemsA = 0, nwinsA = 0;
  int64_t rowsA = 0, tilesA_n = 0, mtstepsA = 0;  // M-tile steps issued (DMMA accounting)
  int ntailg = 0;
  DevBuf tail_base, tail_nch;
  int tail_nch_max = 0;
  // input axis
  DevBuf itemsW, tilesW, winsW;
  int nitemsW = 0, nwinsW = 0;
  int64_t rowsW = 0, tilesW_n = 0, mtstepsW = 0;
  DevBuf nodeg_base, nodeg_nch;
  int nodeg_nch_max = 0;
  DevBuf nodeg_base_im;  // XC_EXP: partial rows of the imaginary parts per node group
  // workspaces: the handle's own (xc_reserve; also the host-buffer pipeline's) and the ones the
  // caller attaches to streams (xc_attach_workspace); xc_apply uses the one bound to its stream
  Ws def;
  std::vector<Ws*> att;
  std::mutex att_mu;
  DevBuf Xh, Yh;  // host-buffer pipeline slots
  bool use_graphs = true;
  // xc_apply_host pipeline: copy-in / copy-out streams and per-slot events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  bool use_fork = true;
  static constexpr int kSlots = 3;  // device slots of the host-buffer pipeline
  cudaEvent_t ev_in[kSlots] = {}, ev_cmp[kSlots] = {}, ev_out[kSlots] = {};
  cudaEvent_t ev_start = nullptr;
  cudaStream_t hst = nullptr;  // apply stream of the last host-buffer call (valid if hst_set)
  bool hst_set = false;
  int64_t hchunk = 0;          // chunks enqueued since the slots were (re)allocated
  int64_t hBc = 0, hN = 0;     // chunk shape (columns, rows) the slots are laid out for
  xc_info_t info{};
  // build state (kept between the phases of a distributed precompute)
  DevBuf djtab;
  ddv p0{1.0, 0.0};
  cudaStream_t bst = nullptr;
  int node_chunk = 0;
  int rank = 0, nranks = 1, npr = 0, xstage = 0;  // npr: nodes per rank (padded)
  int xstage_next = 0;  // stage of the exchange being prepared (0 max, 1 bands, 2 values: 3, 1, 2)
  DevBuf xsend, xrecv;
  std::vector<int64_t> xmaxc;  // per block: max over ranks of the local value count
  // phase profiling (ring of event sets: start, after phase 1, after phase 2, end)
  static constexpr int kRing = 512;
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_dir;     // direction recorded in the slot, 0 = free
  int64_t ev_count = 0;
  double ms_spmm = 0, ms_fft = 0, ms_red = 0, ms_tot = 0;
  int64_t n_prof = 0;
};

namespace {

int64_t pad_cols(int64_t B) {
  int64_t t = 8 * spmm_nt_for(B);
  return (B + t - 1) / t * t;
}

void clear_graphs(Ws& w) {
  for (auto& g : w.graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  w.graphs.clear();
}

// Forked stream of block ib >= 1 (fork_stream): block 2 on its own, blocks 3.. round robin over
// naux - 1 streams.  Large batches use naux = 2 (blocks 3.. in one stream: more concurrent
// streams slowed c5's FFT phase 3.94 -> 4.09 ms), small ones all four (c3 0.255 -> 0.225 ms).
inline int aux_of(int ib, int naux) { return ib == 1 ? 0 : 1 + (ib - 2) % (naux - 1); }
inline int naux_for(int64_t N, int64_t B) {
  static const int force = getenv("XC_NAUX") ? atoi(getenv("XC_NAUX")) : 0;  // measurement switch
  if (force >= 2 && force <= kAux) return force;
  return N * B <= (32LL << 20) ? kAux : 2;
}

// Columns of one C2R column chunk of a two-pass block (c2r_run): the four-step scratch of a chunk
// (M x chunk complex) is kept near 40 MB so that it stays in L2 between the two passes.
int64_t c2r_cols(const BlockData& b, int64_t B) { return c2r_chunk_cols(b.fftM, B); }

// FFT scratch (double2 elements) one block needs on its stream for B columns
size_t block_scratch(const xc_op* h, const BlockData& b, int64_t B) {
  const bool two_d = h->ukind == XC_LAG2D;  // prologue planes (as XC_DIR_WAT) + C2R (as XC_DIR_A)
  size_t n = 0;
  if ((two_d || (h->dirs & XC_DIR_WAT)) && b.fft.L2 > 1) n = std::max(n, (size_t)b.L * (size_t)B);
  if (((h->dirs & XC_DIR_A) || two_d) && h->kind != XC_EXP && b.fftM.L2 > 1)
    n = std::max(n, (size_t)b.fftM.L * (size_t)c2r_cols(b, B));
  if ((h->dirs & XC_DIR_A) && h->kind == XC_EXP && b.fft.L2 > 1)  // C2C inverse of length L
    n = std::max(n, (size_t)b.L * (size_t)B);
  return n;
}

// The workspace of B columns: part sizes in carve order (256-byte aligned), total returned.  With
// w and base it also sets w's pointers into [base, base + total).  xc_workspace_query is this total.
// Debug guard zones (XC_WS_GUARD=1, read once): kGuard bytes after every workspace part, filled with
// 0x7F at carve time; xc_debug_guards counts the bytes a kernel overwrote (an out-of-bounds write
// past a part).  compute-sanitizer is closed on the GPU pool, so this is the write check the tests run.
constexpr size_t kGuard = 64 * 1024;
bool ws_guard() {
  static const bool on = getenv("XC_WS_GUARD") && atoi(getenv("XC_WS_GUARD")) != 0;
  return on;
}

size_t ws_layout(const xc_op* h, int64_t B, Ws* w, char* base) {
  const int64_t Bp = pad_cols(B);
  const bool two_d = h->ukind == XC_LAG2D;
  size_t off = 0;
  std::vector<std::pair<size_t, size_t>> guards;
  auto take = [&](size_t bytes) -> char* {
    // parts of 2 MB and more start on a 2 MB boundary (relative to the range, which cudaMalloc
    // aligns so): their rows then keep the alignment separate allocations had (c5: 10.68 ms with
    // 256-byte aligned parts vs 10.56 ms in round 1)
    if (bytes >= (2u << 20)) off = (off + (2u << 20) - 1) / (2u << 20) * (2u << 20);
    char* p = base ? base + off : nullptr;
    off += (std::max<size_t>(bytes, 16) + 255) / 256 * 256;
    if (ws_guard()) {
      guards.push_back({off, kGuard});
      off += kGuard;
    }
    return p;
  };
  size_t scr = 1;
  for (size_t i = 0; i < h->blocks.size(); ++i)
    if (i == 0 || h->kind == XC_EXP) scr = std::max(scr, block_scratch(h, h->blocks[i], B));
  size_t an[kAux] = {};
  if (h->kind != XC_EXP)
    for (size_t i = 1; i < h->blocks.size(); ++i) {
      const size_t n = block_scratch(h, h->blocks[i], B);
      scr = std::max(scr, n);  // without forked streams every block runs on the caller's
      for (int na : {2, (int)kAux})  // scratch for either stream assignment (naux_for)
        an[aux_of((int)i, na)] = std::max(an[aux_of((int)i, na)], n);
    }
  double2* p_scr = (double2*)take(scr * sizeof(double2));
  double2* p_aux[kAux];
  for (int i = 0; i < kAux; ++i) p_aux[i] = an[i] ? (double2*)take(an[i] * sizeof(double2)) : nullptr;
  double* p_partA = (h->dirs & XC_DIR_A) ? (double*)take((size_t)h->rowsA * Bp * sizeof(double)) : nullptr;
  double2* p_bsr = (two_d && h->bsr_nslots > 0) ? (double2*)take((size_t)h->bsr_nslots * 8 * Bp * sizeof(double2))
                                                 : nullptr;
  double* p_tail = (two_d && h->tail > 0)
                       ? (double*)take((size_t)((h->N + 127) / 128) * h->tail * Bp * sizeof(double))
                       : nullptr;
  double* p_partW = ((h->dirs & XC_DIR_WAT) && !two_d) ? (double*)take((size_t)h->rowsW * Bp * sizeof(double))
                                                      : nullptr;
  std::vector<int64_t> zoff;
  double* p_zpl = nullptr;
  if ((h->dirs & XC_DIR_WAT) || two_d) {
    int64_t tot = 0;
    for (auto& b : h->blocks) {
      zoff.push_back(tot);
      tot += 2 * (int64_t)b.H * Bp;
    }
    if (two_d) tot += 2 * 4 * Bp;  // the DMMA blocks may reach 3 rows past the last spectrum row
    p_zpl = (double*)take((size_t)tot * sizeof(double));
  }
  if (w && base) {
    w->scratch = p_scr;
    for (int i = 0; i < kAux; ++i) w->scratch_aux[i] = p_aux[i];
    w->partA = p_partA;
    w->bsr_part = p_bsr;
    w->tailpart = p_tail;
    w->partW = p_partW;
    w->zpl = p_zpl;
    w->zoff = zoff;
    w->guards = guards;
  }
  return off;
}

// The forked-stream events and streams of a workspace (created once, before any apply uses it).
xc_status ws_streams(Ws& w) {
  if (w.s_aux[0]) return XC_OK;
  int lo = 0, hi = 0;
  XC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  for (int i = 0; i < kAux; ++i) {
    XC_CUDA(cudaStreamCreateWithPriority(&w.s_aux[i], cudaStreamNonBlocking, hi));
    XC_CUDA(cudaEventCreateWithFlags(&w.ev_join[i], cudaEventDisableTiming));
  }
  XC_CUDA(cudaEventCreateWithFlags(&w.ev_fork, cudaEventDisableTiming));
  return XC_OK;
}

// Carve workspace w for B columns from [w.base, w.base + w.bytes) (no allocation).
xc_status ws_carve(const xc_op* h, Ws& w, int64_t B) {
  const size_t need = ws_layout(h, B, nullptr, nullptr);
  if (need > w.bytes) {
    xc_set_error("workspace of " + std::to_string(w.bytes) + " bytes is short of the " + std::to_string(need) +
                 " needed for B = " + std::to_string(B) + " (xc_workspace_query)");
    return XC_ENOMEM;
  }
  ws_layout(h, B, &w, w.base);
  w.B = B;
  for (auto& g : w.guards) XC_CUDA(cudaMemset(w.base + g.first, 0x7F, g.second));  // debug mode only
  clear_graphs(w);  // captured graphs reference the old layout
  return XC_OK;
}

// The handle's own workspace for up to B columns (allocates: xc_reserve, the host pipeline).
xc_status ensure_ws(xc_op* h, int64_t B) {
  XC_TRY(ws_streams(h->def));
  if (B <= h->def.B) return XC_OK;
  const size_t need = ws_layout(h, B, nullptr, nullptr);
  clear_graphs(h->def);
  XC_TRY(dev_alloc(h->def.own, need));
  h->def.base = (char*)h->def.own.p;
  h->def.bytes = need;
  XC_TRY(ws_carve(h, h->def, B));  // (the 2D padding rows are zeroed by every apply)
  return XC_OK;
}

// Kernel launches of one apply of B columns (xc_launches; xc_info's counts are for B = 1).
int64_t c2r_launches_b(const BlockData& b, int64_t B) { return c2r_launch_count(b.fftM, B); }
int64_t count_launches(const xc_op* h, int dir, int64_t B) {
  auto spmm_launches = [](int n) -> int64_t { return n <= 0 ? 0 : (n + 65535 - 1) / 65535; };
  int64_t n = 0;
  if (h->ukind == XC_LAG2D) {
    for (auto& b : h->blocks) n += ((b.fft.L2 > 1) ? 2 : 1) + c2r_launches_b(b, B);
    return n + 1 + (h->bsr_nred > 0 ? 1 : 0) + (h->tail > 0 ? 2 + (h->N > 128 ? 1 : 0) : 0);
  }
  if (dir == XC_DIR_A && h->small_on) {  // small_spmm / small_c2r grid.y chunks
    return 2 * ((B + 65534) / 65535);
  }
  if (dir == XC_DIR_A) {
    if (!(h->dirs & XC_DIR_A)) return 0;
    n = spmm_launches(h->nwinsA) + (h->tail > 0 ? 1 : 0);
    for (auto& b : h->blocks)
      n += (b.split ? 1 : 0) + (h->kind == XC_EXP ? ((b.fft.L2 > 1) ? 2 : 1) : c2r_launches_b(b, B));
    return n;
  }
  if (!(h->dirs & XC_DIR_WAT)) return 0;
  n = spmm_launches(h->nwinsW) + (h->kind == XC_EXP ? 2 : 1);
  for (auto& b : h->blocks) n += (b.fft.L2 > 1) ? 2 : 1;
  return n;
}

xc_status validate_nodes(int kind, const double* x, int64_t N) {
  for (int64_t k = 0; k < N; ++k) {
    if (!std::isfinite(x[k])) {
      xc_set_error("nodes: non-finite value at " + std::to_string(k));
      return XC_EINVAL;
    }
    if (k > 0 && !(x[k] > x[k - 1])) {
      xc_set_error("nodes: not strictly ascending at " + std::to_string(k));
      return XC_EINVAL;
    }
  }
  bool ok = true;
  if (kind == XC_COS) ok = x[0] >= 0.0 && x[N - 1] <= 1.0;
  if (kind == XC_EXP) ok = x[0] >= 0.0 && x[N - 1] < 2.0;
  if (kind == XC_JACOBI) ok = x[0] >= -1.0 && x[N - 1] <= 1.0;
  if (kind == XC_LAGUERRE || kind == XC_LAG2D) ok = x[0] >= 0.0;  // XC_LAGSPEC: any real frequency
  if (ok && kind == XC_LAG2D && N > 2) {  // equispaced (the extra rows continue the grid, R-23)
    const double hh = (x[N - 1] - x[0]) / (double)(N - 1);
    for (int64_t k = 1; k < N && ok; ++k) ok = fabs((x[k] - x[k - 1]) - hh) <= 1e-9 * fmax(hh, fabs(x[k]));
    if (!ok) {
      xc_set_error("XC_LAG2D: nodes must be equispaced");
      return XC_EINVAL;
    }
  }
  if (!ok) {
    xc_set_error("nodes: outside the domain of the kind");
    return XC_EINVAL;
  }
  return XC_OK;
}

// --- the per-block precompute: entries -> FFT -> threshold -> node bands ------------
// Per block: FFT plans, twiddles, the window and its derived scales (and, for the Appendix A
// precompute, the truncated window spectrum in dxq).
xc_status block_setup(xc_op* h, BlockData& b, DevBuf& dxq) {
  const bool cplx_rows = h->kind == XC_EXP;  // complex rows: the full spectrum (no Hermitian half)
  b.H = cplx_rows ? b.L : b.L / 2 + 1;
  XC_TRY(fft_plan_make(b.fft, b.L));
  if (!cplx_rows) XC_TRY(fft_plan_make(b.fftM, b.L / 2, true));
  {
    std::vector<double2> tw(b.L / 2);
    const long double PI2 = 6.283185307179586476925286766559005768L;
    for (int n = 0; n < b.L / 2; ++n) {
      long double a = PI2 * (long double)n / (long double)b.L;
      tw[n] = make_double2((double)cosl(a), (double)sinl(a));
    }
    XC_TRY(upload(b.twh, tw));
  }
  kaiser_window(h->zeta, b.L, b.h_w);
  if (h->appA) {  // R-22: the truncated window W' = F* xq is the method's window from here on
    std::vector<double2> xq;
    std::vector<double> wq;
    XC_TRY(appa_window(b.h_w, b.L, h->eps1, xq, b.appQ, wq));
    b.h_w = wq;
    XC_TRY(upload(dxq, xq));
  }
  std::vector<double> ys(b.L), wi(b.L);
  const double isL = 1.0 / sqrt((double)b.L);
  for (int p = 0; p < b.L; ++p) {
    ys[p] = isL / b.h_w[p];
    wi[p] = 1.0 / b.h_w[p];
  }
  XC_TRY(upload(b.w, b.h_w));
  XC_TRY(upload(b.yscale, ys));
  XC_TRY(upload(b.winv, wi));
  return XC_OK;
}

// The windowed extended rows of nodes [k0, k0 + n) and their unitary DFT (Eq. 1): spec[q * n + k],
// q < H (the direct precompute, p2-p3).
xc_status chunk_spectra(xc_op* h, BlockData& b, const DevBuf& djtab, ddv p0, int k0, int n, DevBuf& F, DevBuf& scr,
                        DevBuf& spec, cudaStream_t st) {
  GenParams g{};
  g.kind = h->kind;
  g.L = b.L;
  g.m_off = b.m_off;
  g.nodes = (const double*)h->nodes.p + k0;
  if (h->nodes_lo.p) g.nodes_lo = (const double*)h->nodes_lo.p + k0;
  if (h->cscale.p) g.cscale = (const double2*)h->cscale.p + k0;
  g.nc = n;
  g.w = (const double*)b.w.p;
  g.jab = (const double2*)djtab.p;
  g.p0 = p0;
  XC_TRY(gen_entries(g, (double2*)F.p, st));
  FftIO io{};
  io.src = (const double2*)F.p;
  io.lds = n;
  io.dst = (double2*)spec.p;
  io.ldd = n;
  io.kmax = b.H;
  io.scale = 1.0 / sqrt((double)b.L);  // unitary DFT of Eq. (1)
  return fft_run(b.fft, -1, PRO_PLAIN, EPI_PLAIN, io, n, (double2*)scr.p, st);
}

// Nodes per precompute chunk of block b: F, the FFT scratch and the spectra (48 B per position and
// node) take at most a third of the free device memory (capped at 48 GB): the entry recurrence runs
// one thread per node, so the chunk is the generation's parallelism (c5 block 1: ~9K nodes per
// chunk instead of 776 with a 3 GB budget -- 10x faster precompute)
int chunk_nodes(const BlockData& b, int node_chunk, int64_t per_node, int N) {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = 3ull << 30;
  const int64_t budget = std::max<int64_t>(1LL << 30, std::min<int64_t>((int64_t)(fr / 3), 48LL << 30));
  int nc = node_chunk > 0 ? node_chunk : (int)std::max<int64_t>(64, std::min<int64_t>(budget / per_node, 1 << 24));
  return std::min(nc, std::max(1, N));
}

// Global threshold reference (thresh_mode = 1, Alg. 1/2 step 1.3): max |S|^2 over the block's
// spectra of nodes [n0, n1) -- the first of the two passes over the nodes.
xc_status block_max2(xc_op* h, BlockData& b, const DevBuf& djtab, ddv p0, int node_chunk, int n0, int n1,
                     double& mx2, cudaStream_t st) {
  DevBuf dxq;
  XC_TRY(block_setup(h, b, dxq));
  const int nc = chunk_nodes(b, node_chunk, (int64_t)b.L * 48, n1 - n0);
  DevBuf F, scr, spec, dmx;
  XC_TRY(dev_alloc(F, (size_t)b.L * nc * sizeof(double2)));
  if (b.fft.L2 > 1) XC_TRY(dev_alloc(scr, (size_t)b.L * nc * sizeof(double2)));
  XC_TRY(dev_alloc(spec, (size_t)b.H * nc * sizeof(double2)));
  XC_TRY(dev_alloc(dmx, sizeof(unsigned long long)));
  XC_CUDA(cudaMemsetAsync(dmx.p, 0, sizeof(unsigned long long), st));
  for (int k0 = n0; k0 < n1; k0 += nc) {
    const int n = std::min(nc, n1 - k0);
    XC_TRY(chunk_spectra(h, b, djtab, p0, k0, n, F, scr, spec, st));
    XC_TRY(spec_max2((const double2*)spec.p, (int64_t)b.H * n, (unsigned long long*)dmx.p, st));
  }
  unsigned long long bits = 0;
  XC_CUDA(cudaMemcpyAsync(&bits, dmx.p, sizeof(bits), cudaMemcpyDeviceToHost, st));
  XC_CUDA(cudaStreamSynchronize(st));
  memcpy(&mx2, &bits, sizeof(double));
  dev_free(F);
  dev_free(scr);
  dev_free(spec);
  dev_free(dmx);
  return XC_OK;
}

xc_status build_block(xc_op* h, BlockData& b, const DevBuf& djtab, ddv p0, int node_chunk, int n0, int n1,
                      cudaStream_t st) {
  const int N = (int)h->N;
  const bool cplx_rows = h->kind == XC_EXP;
  DevBuf dxq;
  XC_TRY(block_setup(h, b, dxq));

  // global threshold (thresh_mode = 1): |S|^2 >= eps1^2 max over the whole block (set by the caller)
  const double thr2 = h->thresh_mode == 1 ? (h->eps1 * h->eps1) * b.gmax2 : 0.0;
  // Appendix A, window mode: only 2W+1 bins per node are evaluated and kept in memory; for
  // complex rows the window must stay under half the circle (its linear span is then the
  // shortest arc holding the kept bins, R-18); short blocks take the full-spectrum mode
  int appW = b.appQ + 16;
  const int appWmax = cplx_rows ? (b.L / 2 - 1) / 2 : b.H;
  const bool app_win = h->appA && appW <= appWmax;
  int64_t per_node = app_win ? (int64_t)16 * 4 * (2 * appW + 1) + 32 : (int64_t)b.L * 48;
  const int nc = chunk_nodes(b, node_chunk, per_node, N);
  DevBuf F, scr, spec, st_len, d_start, d_len, dflag, dwin, dwfirst, dthr;
  if (!h->appA) {
    XC_TRY(dev_alloc(F, (size_t)b.L * nc * sizeof(double2)));
    if (b.fft.L2 > 1) XC_TRY(dev_alloc(scr, (size_t)b.L * nc * sizeof(double2)));
  } else {
    XC_TRY(dev_alloc(dflag, sizeof(int)));
  }
  if (app_win) {
    XC_TRY(dev_alloc(dwfirst, (size_t)nc * sizeof(int)));
    XC_TRY(dev_alloc(dthr, (size_t)nc * sizeof(double)));
  } else {
    XC_TRY(dev_alloc(spec, (size_t)b.H * nc * sizeof(double2)));
  }
  XC_TRY(dev_alloc(b.start, (size_t)N * sizeof(int)));
  XC_TRY(dev_alloc(b.len, (size_t)N * sizeof(int)));
  b.h_start.assign(N, 0);
  b.h_len.assign(N, 0);
  b.h_off.assign(N + 1, 0);
  std::vector<DevBuf> chunk_vals;
  std::vector<int64_t> chunk_base;
  DevBuf choff;

  for (int k0 = n0; k0 < n1; k0 += nc) {
    int n = std::min(nc, n1 - k0);
    int W = 0;  // Appendix A: evaluated half-window around the peak (kept runs lie within Q + 3, R-22)
    AppAWin wm{};
    if (h->appA) {
      for (;;) {
        // full-spectrum mode: 2 Wmax + 1 >= L covers every bin of the circle (for even L one bin
        // is evaluated twice, with the same value); window mode: under half the circle
        const int Wmax = app_win ? appWmax : (cplx_rows ? b.L / 2 : b.H);
        W = std::min(appW, Wmax);
        int flag = 0;
        XC_CUDA(cudaMemsetAsync(dflag.p, 0, sizeof(int), st));
        const double* th = (const double*)h->nodes.p + k0;
        const double* tl = h->nodes_lo.p ? (const double*)h->nodes_lo.p + k0 : nullptr;
        const double2* cs = h->cscale.p ? (const double2*)h->cscale.p + k0 : nullptr;
        if (app_win) {
          const size_t wb = (size_t)n * (2 * W + 1) * sizeof(double2);
          if (dwin.bytes < wb) {
            dev_free(dwin);
            XC_TRY(dev_alloc(dwin, wb));
          }
          wm = AppAWin{(double2*)dwin.p, (int*)b.start.p + k0, (int*)b.len.p + k0, (int*)dwfirst.p, (double*)dthr.p};
          XC_TRY(appa_spectra(h->kind, b.L, b.H, b.m_off, b.appQ, W, th, tl, cs, (const double2*)dxq.p, n, h->eps1,
                              nullptr, (int*)dflag.p, st, &wm));
        } else {
          XC_CUDA(cudaMemsetAsync(spec.p, 0, (size_t)b.H * n * sizeof(double2), st));
          XC_TRY(appa_spectra(h->kind, b.L, b.H, b.m_off, b.appQ, W, th, tl, cs, (const double2*)dxq.p, n, h->eps1,
                              (double2*)spec.p, (int*)dflag.p, st));
        }
        XC_CUDA(cudaMemcpyAsync(&flag, dflag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        XC_CUDA(cudaStreamSynchronize(st));
        if (!flag) break;
        if (W == Wmax) {
          if (!app_win) break;  // every bin evaluated
          xc_set_error("Appendix A: a kept run spans a quarter of the circle; use trig_precompute = 0");
          return XC_ENUMERIC;
        }
        appW = 2 * appW;  // a kept bin on the window's edge: widen and redo the chunk
      }
    } else {
      XC_TRY(chunk_spectra(h, b, djtab, p0, k0, n, F, scr, spec, st));
    }
    int* ds = (int*)b.start.p + k0;
    int* dl = (int*)b.len.p + k0;
    if (!app_win) XC_TRY(band_detect((const double2*)spec.p, b.H, n, h->eps1, thr2, ds, dl, cplx_rows, st));
    XC_CUDA(cudaMemcpyAsync(b.h_start.data() + k0, ds, n * sizeof(int), cudaMemcpyDeviceToHost, st));
    XC_CUDA(cudaMemcpyAsync(b.h_len.data() + k0, dl, n * sizeof(int), cudaMemcpyDeviceToHost, st));
    XC_CUDA(cudaStreamSynchronize(st));
    std::vector<int64_t> loc(n);
    int64_t tot = 0;
    for (int i = 0; i < n; ++i) {
      loc[i] = tot;
      b.h_off[k0 + i] = b.h_off[k0] + tot;  // fixed below (global prefix)
      tot += b.h_len[k0 + i];
    }
    DevBuf cv;
    XC_TRY(dev_alloc(cv, (size_t)std::max<int64_t>(1, tot) * sizeof(double2)));
    XC_TRY(upload(choff, loc));
    if (app_win)
      XC_TRY(appa_store(wm, W, (const int64_t*)choff.p, (double2*)cv.p, n, st));
    else
      XC_TRY(band_store((const double2*)spec.p, b.H, n, h->eps1, thr2, ds, dl, (const int64_t*)choff.p,
                        (double2*)cv.p, cplx_rows, st));
    XC_CUDA(cudaStreamSynchronize(st));
    chunk_vals.push_back(cv);
    chunk_base.push_back(tot);
  }
  // the local node range's values, contiguous in node order
  int64_t acc = 0;
  for (int64_t c : chunk_base) acc += c;
  XC_TRY(dev_alloc(b.vals, (size_t)std::max<int64_t>(1, acc) * sizeof(double2)));
  int64_t pos = 0;
  for (size_t c = 0; c < chunk_vals.size(); ++c) {
    if (chunk_base[c] > 0)
      XC_CUDA(cudaMemcpyAsync((double2*)b.vals.p + pos, chunk_vals[c].p, chunk_base[c] * sizeof(double2),
                              cudaMemcpyDeviceToDevice, st));
    pos += chunk_base[c];
  }
  XC_CUDA(cudaStreamSynchronize(st));
  for (auto& cv : chunk_vals) dev_free(cv);
  dev_free(choff);
  b.loc_count = acc;
  dev_free(F);
  dev_free(scr);
  dev_free(spec);
  dev_free(dflag);
  dev_free(dxq);
  dev_free(dwin);
  dev_free(dwfirst);
  dev_free(dthr);
  return XC_OK;
}

// Global band offsets once every node's band is known (h_start/h_len for all N nodes,
// b.vals holding all values in node order).
xc_status finalize_bands(xc_op* h, BlockData& b) {
  const int N = (int)h->N;
  int64_t acc = 0;
  b.max_band = 0;
  for (int k = 0; k < N; ++k) {
    b.h_off[k] = acc;
    acc += b.h_len[k];
    b.max_band = std::max(b.max_band, b.h_len[k]);
  }
  b.h_off[N] = acc;
  XC_TRY(upload(b.off, b.h_off));
  // kept nonzeros (the stored runs contain explicit zeros for dropped interior bins)
  b.nnz = acc;
  return XC_OK;
}

// --- SpMM items: M-tiles, single or paired ------------------------------------------------
// An M-tile is one 8-row slice of the operator (a bin group, a degree group or a node group)
// over its exact range of B rows [k0, k1) with its output rows.  Two M-tiles over nearly the
// same rows may be paired into one item: they then share the B fragments (half the shared-
// memory traffic per DMMA) but both run over the union of the ranges.  Pairing is used only
// where the union adds little (kPairSlack); otherwise the item carries one M-tile.
constexpr double kPairSlackDefault = 1.08;
double pair_slack() {  // XC_PAIR_SLACK overrides (measurement switch)
  static const double v = getenv("XC_PAIR_SLACK") ? atof(getenv("XC_PAIR_SLACK")) : kPairSlackDefault;
  return v;
}

struct MTile {
  int fam;        // block index, or -1 for the dense tail
  int g;          // group index within the family
  int chunk;      // execution-order key (B-row window)
  int k0, k1;     // B rows
  int64_t out_row;
  int cplx;
};

struct ItemSet {
  std::vector<SpmmItem> items;
  std::vector<FillItem> fills;  // one per M-tile
  std::vector<int> fam;         // family of each fill
  int64_t aoff = 0;
};

bool worth_pairing(const MTile& a, const MTile& b) {
  const int la = std::max(0, a.k1 - a.k0), lb = std::max(0, b.k1 - b.k0);
  if (la == 0 || lb == 0) return false;
  const int u0 = std::min(a.k0, b.k0), u1 = std::max(a.k1, b.k1);
  if (u1 - u0 > XC_WMAX - 3) return false;  // the pair must fit one shared-memory window
  return 2.0 * (u1 - u0) <= pair_slack() * (la + lb);
}

// Emit one item for M-tile a (and b, if non-null) reading operand source `src`.
void emit_item(const MTile& a, const MTile* b, int src, ItemSet& out) {
  int k0 = a.k0, k1 = a.k1;
  if (b) {
    k0 = std::min(k0, b->k0);
    k1 = std::max(k1, b->k1);
  }
  SpmmItem it{};
  it.a_off = out.aoff;
  it.out_row[0] = a.out_row;
  it.out_row[1] = b ? b->out_row : -1;
  it.k0 = k1 > k0 ? k0 : 0;
  it.nsteps = std::max(0, (k1 - k0 + 3) / 4);
  it.src = src;
  it.cplx = a.cplx;
  out.items.push_back(it);
  out.fills.push_back(FillItem{out.aoff, it.k0, it.nsteps, a.g, 0, a.k0, a.k1});
  out.fam.push_back(a.fam);
  if (b) {
    out.fills.push_back(FillItem{out.aoff, it.k0, it.nsteps, b->g, 1, b->k0, b->k1});
    out.fam.push_back(b->fam);
  }
  out.aoff += 64LL * ((it.nsteps + 1) & ~1);  // steps in pairs (build.cu)
}

// Pair neighbours of an ordered list greedily where worth it.
void pair_list(const std::vector<MTile>& mt, int src, ItemSet& out) {
  size_t i = 0;
  while (i < mt.size()) {
    if (i + 1 < mt.size() && mt[i + 1].cplx == mt[i].cplx && worth_pairing(mt[i], mt[i + 1])) {
      emit_item(mt[i], &mt[i + 1], src, out);
      i += 2;
    } else {
      emit_item(mt[i], nullptr, src, out);
      i += 1;
    }
  }
}

// items per output-axis window (XC_WIN_ITEMS_A overrides; measurement switch)
int out_win_items() {
  static const int v = getenv("XC_WIN_ITEMS_A") ? atoi(getenv("XC_WIN_ITEMS_A")) : 64;
  return std::max(8, v);
}

xc_status upload_and_fill(xc_op* h, ItemSet& S, bool input_axis, DevBuf& d_items, DevBuf& d_wins,
                          DevBuf& d_tiles, int& nitems, int& nwins, int64_t& ntiles, cudaStream_t st) {
  const int N = (int)h->N;
  ntiles = S.aoff;
  int64_t& mts = input_axis ? h->mtstepsW : h->mtstepsA;
  mts = 0;
  for (auto& it : S.items) mts += (int64_t)it.nsteps * (it.out_row[1] >= 0 ? 2 : 1);
  XC_TRY(dev_alloc(d_tiles, (size_t)std::max<int64_t>(1, S.aoff) * sizeof(double)));
  XC_CUDA(cudaMemsetAsync(d_tiles.p, 0, (size_t)std::max<int64_t>(1, S.aoff) * sizeof(double), st));  // unpaired slots
  DevBuf dfill;
  for (int fam = -1; fam < (int)h->blocks.size(); ++fam) {
    std::vector<FillItem> part;
    for (size_t i = 0; i < S.fills.size(); ++i)
      if (S.fam[i] == fam && S.fills[i].nsteps > 0) part.push_back(S.fills[i]);  // per M-tile
    if (part.empty()) continue;
    XC_TRY(upload(dfill, part));
    if (fam >= 0) {
      BlockData& b = h->blocks[fam];
      XC_TRY(fill_tiles(input_axis ? (h->kind == XC_EXP ? FILL_IN_CC : FILL_IN_CPLX)
                                   : (h->kind == XC_EXP ? FILL_OUT_CC : FILL_OUT_CPLX),
                        (FillItem*)dfill.p, (int)part.size(),
                        (int*)b.start.p, (int*)b.len.p, (int64_t*)b.off.p, (double2*)b.vals.p, nullptr, 0, N, b.H,
                        (double*)d_tiles.p, st));
    } else {
      XC_TRY(fill_tiles(input_axis ? FILL_IN_REAL : FILL_OUT_REAL, (FillItem*)dfill.p, (int)part.size(), nullptr,
                        nullptr, nullptr, nullptr, (double*)h->tailP.p, h->tail, N, 0, (double*)d_tiles.p, st));
    }
    XC_CUDA(cudaStreamSynchronize(st));
  }
  dev_free(dfill);
  // windows: items sorted by (source, first B row); a window takes consecutive items while
  // their B rows fit XC_WMAX rows (one CTA stages them in shared memory)
  std::vector<size_t> ord(S.items.size());
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
    if (S.items[a].src != S.items[b].src) return S.items[a].src < S.items[b].src;
    return S.items[a].k0 < S.items[b].k0;
  });
  std::vector<SpmmItem> sorted(S.items.size());
  for (size_t i = 0; i < ord.size(); ++i) sorted[i] = S.items[ord[i]];
  // tiny operators (fewer than 16 items per SM, e.g. c1): fewer items per window, so that the
  // single-column-tile grid still has >= 2 CTAs per SM
  const int64_t nsm = sm_count();
  // otherwise the output axis takes at most 64 items per window (c4 forward SpMM 1.366 -> 1.314
  // ms; c5 unchanged, its windows are bounded by their 192 rows), the input axis 128 (64 there
  // made c4 backward 2.5 % slower)
  const int win_items = (int64_t)sorted.size() < 16 * nsm
                            ? (int)std::max<int64_t>(8, ((int64_t)sorted.size() + 2 * nsm - 1) / (2 * nsm))
                            : (input_axis ? WIN_ITEMS : std::min(out_win_items(), WIN_ITEMS));
  std::vector<SpmmWin> wins;
  std::vector<int64_t> wcost;  // the window's critical path: its most loaded warp
  size_t i = 0;
  while (i < sorted.size()) {
    SpmmWin w{};
    w.src = sorted[i].src;
    w.r0 = sorted[i].k0;
    w.r1 = sorted[i].k0 + 4 * sorted[i].nsteps;
    w.i0 = (int)i;
    size_t j = i + 1;
    while (j < sorted.size() && sorted[j].src == w.src && (int)(j - i) < win_items) {
      int e = sorted[j].k0 + 4 * sorted[j].nsteps;
      if (std::max(e, w.r1) - w.r0 > XC_WMAX) break;
      w.r1 = std::max(w.r1, e);
      ++j;
    }
    w.i1 = (int)j;
    // balance the window's items over the CTA's warps: longest first onto the least-loaded
    // warp (cost ~ M-tile steps + a fixed per-item overhead); each warp's items contiguous
    {
      const int n = w.i1 - w.i0;
      std::vector<int> ord(n);
      for (int q = 0; q < n; ++q) ord[q] = q;
      auto cost = [&](int q) {
        const SpmmItem& it = sorted[w.i0 + q];
        return (int64_t)it.nsteps * (it.out_row[1] >= 0 ? 2 : 1) + 6;
      };
      std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return cost(x) > cost(y); });
      std::vector<int64_t> load(XC_WARPS, 0);
      std::vector<std::vector<int>> per(XC_WARPS);
      for (int q : ord) {
        int best = 0;
        for (int k = 1; k < XC_WARPS; ++k)
          if (load[k] < load[best]) best = k;
        load[best] += cost(q);
        per[best].push_back(q);
      }
      std::vector<SpmmItem> tmp;
      w.wo[0] = 0;
      for (int k = 0; k < XC_WARPS; ++k) {
        for (int q : per[k]) tmp.push_back(sorted[w.i0 + q]);
        w.wo[k + 1] = (int)tmp.size();
      }
      std::copy(tmp.begin(), tmp.end(), sorted.begin() + w.i0);
      wcost.push_back(*std::max_element(load.begin(), load.end()));
    }
    wins.push_back(w);
    i = j;
  }
  // a second copy of the windows, heaviest first: CTAs are dispatched in grid order, so with it
  // the last wave holds the light windows (list scheduling, longest first).  Used for grids of
  // a few waves (wins_for); long grids keep node order (measured: c5 SpMM 6.87 vs 7.08 ms)
  {
    std::vector<size_t> wo(wins.size());
    for (size_t q = 0; q < wo.size(); ++q) wo[q] = q;
    std::stable_sort(wo.begin(), wo.end(), [&](size_t x, size_t y) { return wcost[x] > wcost[y]; });
    const size_t nw = wins.size();
    for (size_t q = 0; q < nw; ++q) wins.push_back(wins[wo[q]]);
  }
  XC_TRY(upload(d_items, sorted));
  XC_TRY(upload(d_wins, wins));
  nitems = (int)sorted.size();
  nwins = (int)wins.size() / 2;
  return XC_OK;
}

// --- output-axis items and tiles ---------------------------------------------------------
// Per block, bin group g = bins [4g, 4g+4) owns U rows ubase + 8g + 2(q%4) + comp, i.e. the
// complex half spectrum u_q interleaved in double rows ubase + 2q, +1.  Blocks whose groups
// span few nodes (the large-L blocks) get one M-tile per group writing U directly; blocks
// whose groups span many nodes (small L: ~18N nonzeros over few bins) are split into node
// chunks whose partial sums are reduced into U in fixed order (deterministic split-K).
xc_status build_output_axis(xc_op* h, cudaStream_t st) {
  const int N = (int)h->N;
  const int N4 = (N + 3) / 4 * 4;
  ItemSet S;
  int64_t rows = 0;
  std::vector<MTile> pool;  // split-block M-tiles of every block, paired across blocks per chunk
  // B rows per node: 1 (real X), 2 for XC_EXP (planar complex X: row 2k real part, 2k+1 imag)
  const int kb = h->kind == XC_EXP ? 2 : 1;
  for (size_t bi = 0; bi < h->blocks.size(); ++bi) {
    BlockData& b = h->blocks[bi];
    b.ngroups = (b.H + 3) / 4;
    // per group: the B-row range touched in each node chunk of KC B rows (chunks ascending)
    struct Seg {
      int c, lo, hi;
    };
    std::vector<std::vector<Seg>> seg(b.ngroups);
    std::vector<int> last_node(b.ngroups, -1);
    for (int k = 0; k < N; ++k) {
      const int len = b.h_len[k];
      if (len == 0) continue;
      const int r0 = kb * k, r1 = kb * (k + 1), c = r0 / KC;
      for (int j = 0; j < len; ++j) {
        const int q = (b.h_start[k] + j) % b.H;  // complex rows may wrap around the spectrum
        const int g = q / 4;
        if (last_node[g] == k) continue;         // this node already counted for group g
        last_node[g] = k;
        auto& v = seg[g];
        if (!v.empty() && v.back().c == c) v.back().hi = r1;
        else v.push_back(Seg{c, r0, r1});
      }
    }
    b.ubase = rows;
    rows += 8LL * b.ngroups;
    std::vector<int64_t> gbase(b.ngroups, 0);
    std::vector<int> gnch(b.ngroups, -1);  // -1: the group's items write U directly
    std::vector<MTile> mt;
    b.split = false;
    for (int g = 0; g < b.ngroups; ++g) {
      const auto& v = seg[g];
      const int a = v.empty() ? 0 : v.front().lo, e = v.empty() ? 0 : v.back().hi;
      if (e - a <= KSPLIT) {  // one item over the whole range writes the group's U rows
        mt.push_back(MTile{(int)bi, g, 0, a, e, b.ubase + 8LL * g, 1});  // empty group -> zeros
        continue;
      }
      // long (or wrapping) group: one partial M-tile per touched chunk, reduced in fixed order
      b.split = true;
      gbase[g] = rows;
      gnch[g] = 0;
      for (const Seg& sg : v) {
        pool.push_back(MTile{(int)bi, g, sg.c, sg.lo, sg.hi, rows, 1});
        rows += 8;
        gnch[g]++;
      }
    }
    if (b.split) {
      XC_TRY(upload(b.grp_base, gbase));
      XC_TRY(upload(b.grp_nch, gnch));
      b.grp_nch_max = gnch.empty() ? 0 : *std::max_element(gnch.begin(), gnch.end());
    }
    pair_list(mt, 0, S);  // the direct groups, consecutive in g
  }
  // split blocks: per node chunk, all blocks' M-tiles ordered by range, paired across blocks
  std::stable_sort(pool.begin(), pool.end(), [](const MTile& x, const MTile& y) {
    if (x.chunk != y.chunk) return x.chunk < y.chunk;
    if (x.k0 != y.k0) return x.k0 < y.k0;
    return x.k1 < y.k1;
  });
  pair_list(pool, 0, S);
  // dense tail: groups of 8 degrees x node chunks
  h->ntailg = (h->tail + 7) / 8;
  std::vector<int64_t> tbase(std::max(1, h->ntailg), 0);
  std::vector<int> tnch(std::max(1, h->ntailg), 0);
  std::vector<MTile> mt;
  for (int g = 0; g < h->ntailg; ++g) {
    tbase[g] = rows;
    for (int k0 = 0; k0 < N4; k0 += KC) {
      mt.push_back(MTile{-1, g, k0 / KC, k0, std::min(N, k0 + KC), rows, 0});
      rows += 8;
      tnch[g]++;
    }
  }
  std::stable_sort(mt.begin(), mt.end(), [](const MTile& x, const MTile& y) { return x.chunk < y.chunk; });
  pair_list(mt, 0, S);
  XC_TRY(upload(h->tail_base, tbase));
  XC_TRY(upload(h->tail_nch, tnch));
  h->tail_nch_max = tnch.empty() ? 0 : *std::max_element(tnch.begin(), tnch.end());
  h->rowsA = rows;
  return upload_and_fill(h, S, false, h->itemsA, h->winsA, h->tilesA, h->nitemsA, h->nwinsA, h->tilesA_n, st);
}

// --- input-axis items and tiles ----------------------------------------------------------
// Node group G = nodes [8G, 8G+8); per block its bins are the union of the nodes' bands,
// in B rows 2q (re plane) and 2q+1 (im plane) of that block's z' planes; split into bin
// chunks.  Items of one node group are allocated consecutive output rows and reduced (times
// the weights) in fixed order.
// XC_EXP input axis (Alg. 1 with complex rows, R-20): node group G = nodes [8G, 8G+8), bins of
// the full circular spectrum in chunks of QC; per (G, chunk) two M-tiles over the same B rows
// (2q, 2q+1: the z' planes) -- the real and the imaginary parts of Y -- always paired.  Partial
// rows of G: real parts at base[G] + 8c, imaginary parts at base_im[G] + 8c, c < nch[G].
xc_status build_input_axis_cc(xc_op* h, cudaStream_t st) {
  const int N = (int)h->N;
  const int NG = (N + 7) / 8;
  BlockData& b = h->blocks[0];  // the exp kind has one block and no tail
  const int nch_bins = (b.H + QC - 1) / QC;
  std::vector<int> gnch(NG, 0);
  std::vector<int64_t> gbase(NG, 0), gbase_im(NG, 0);
  struct Rng {
    int G, c, q0, q1;
  };
  std::vector<Rng> rng;
  std::vector<int> lo(nch_bins), hi(nch_bins);
  for (int G = 0; G < NG; ++G) {
    std::fill(lo.begin(), lo.end(), b.H);
    std::fill(hi.begin(), hi.end(), -1);
    for (int k = 8 * G; k < std::min(N, 8 * G + 8); ++k)
      for (int j = 0; j < b.h_len[k]; ++j) {
        const int q = (b.h_start[k] + j) % b.H, c = q / QC;
        lo[c] = std::min(lo[c], q);
        hi[c] = std::max(hi[c], q);
      }
    for (int c = 0; c < nch_bins; ++c)
      if (hi[c] >= lo[c]) {
        rng.push_back(Rng{G, c, lo[c] / 2 * 2, (hi[c] + 2) / 2 * 2});
        gnch[G]++;
      }
  }
  int64_t rows = 0;
  for (int G = 0; G < NG; ++G) {
    gbase[G] = rows;
    gbase_im[G] = rows + 8LL * gnch[G];
    rows += 16LL * gnch[G];
  }
  std::vector<int> used(NG, 0);
  std::vector<MTile> mt;
  for (auto& r : rng) {
    const int u = used[r.G]++;
    mt.push_back(MTile{0, 2 * r.G + 0, r.c, 2 * r.q0, 2 * r.q1, gbase[r.G] + 8LL * u, 0});
    mt.push_back(MTile{0, 2 * r.G + 1, r.c, 2 * r.q0, 2 * r.q1, gbase_im[r.G] + 8LL * u, 0});
  }
  ItemSet S;
  for (size_t i = 0; i + 1 < mt.size(); i += 2) emit_item(mt[i], &mt[i + 1], 0, S);  // re / im share B rows
  XC_TRY(upload(h->nodeg_base, gbase));
  XC_TRY(upload(h->nodeg_base_im, gbase_im));
  XC_TRY(upload(h->nodeg_nch, gnch));
  h->nodeg_nch_max = gnch.empty() ? 0 : *std::max_element(gnch.begin(), gnch.end());
  h->rowsW = rows;
  return upload_and_fill(h, S, true, h->itemsW, h->winsW, h->tilesW, h->nitemsW, h->nwinsW, h->tilesW_n, st);
}

xc_status build_input_axis(xc_op* h, cudaStream_t st) {
  if (h->kind == XC_EXP) return build_input_axis_cc(h, st);
  const int N = (int)h->N;
  const int NG = (N + 7) / 8;
  const int nb = (int)h->blocks.size();
  std::vector<std::vector<MTile>> fam_tiles(nb + 1);
  std::vector<int> gnch(NG, 0);
  std::vector<int64_t> gbase(NG, 0);
  // first pass: count M-tiles per node group (rows are allocated group-major)
  struct Rng {
    int fam, G, chunk, k0, k1;
  };
  std::vector<Rng> rng;
  for (int bi = 0; bi < nb; ++bi) {
    BlockData& b = h->blocks[bi];
    for (int G = 0; G < NG; ++G) {
      int qlo = b.H, qhi = 0;
      for (int k = 8 * G; k < std::min(N, 8 * G + 8); ++k) {
        if (b.h_len[k] == 0) continue;
        qlo = std::min(qlo, b.h_start[k]);
        qhi = std::max(qhi, b.h_start[k] + b.h_len[k]);
      }
      if (qlo >= qhi) continue;
      int a = qlo / 2 * 2, e = (qhi + 1) / 2 * 2;  // 2 bins = 4 B rows per step
      for (int c = a / QC; c * QC < e; ++c) {
        int q0 = std::max(a, c * QC), q1 = std::min(e, (c + 1) * QC);
        if (q1 <= q0) continue;
        rng.push_back(Rng{bi, G, c, 2 * q0, 2 * q1});
        gnch[G]++;
      }
    }
  }
  if (h->tail > 0) {
    int t4 = (h->tail + 3) / 4 * 4;
    for (int G = 0; G < NG; ++G) {
      rng.push_back(Rng{-1, G, 0, 0, t4});
      gnch[G]++;
    }
  }
  int64_t rows = 0;
  for (int G = 0; G < NG; ++G) {
    gbase[G] = rows;
    rows += 8LL * gnch[G];
  }
  std::vector<int> used(NG, 0);
  for (auto& r : rng) {
    int64_t orow = gbase[r.G] + 8LL * used[r.G]++;
    fam_tiles[r.fam + 1].push_back(MTile{r.fam, r.G, r.chunk, r.k0, r.k1, orow, 0});
  }
  ItemSet S;
  for (int f = 0; f <= nb; ++f) {
    auto& mt = fam_tiles[f];
    std::stable_sort(mt.begin(), mt.end(), [](const MTile& x, const MTile& y) {
      return x.chunk != y.chunk ? x.chunk < y.chunk : x.g < y.g;
    });
    pair_list(mt, f == 0 ? nb : f - 1, S);
  }
  XC_TRY(upload(h->nodeg_base, gbase));
  XC_TRY(upload(h->nodeg_nch, gnch));
  h->nodeg_nch_max = gnch.empty() ? 0 : *std::max_element(gnch.begin(), gnch.end());
  h->rowsW = rows;
  return upload_and_fill(h, S, true, h->itemsW, h->winsW, h->tilesW, h->nitemsW, h->nwinsW, h->tilesW_n, st);
}

double fft_flops(int L) { return 2.5 * L * log2((double)L); }  // real FFT = half of 5 L log2 L

// Phase 1 of the precompute: validation, plan (p1), per-block windows / FFT plans, nodes.
xc_status build_begin(xc_kind kind, const xc_params* prm, const double* nodes, int64_t N, double eps, xc_op* h) {
  xc_params p;
  xc_params_default(&p);
  if (prm) p = *prm;
  if (kind != XC_COS && kind != XC_JACOBI && kind != XC_LAGUERRE && kind != XC_EXP && kind != XC_LAGSPEC &&
      kind != XC_LAG2D) {
    xc_set_error("unknown kind");
    return XC_EINVAL;
  }
  const bool cplx = kind == XC_EXP || kind == XC_LAGSPEC;
  const int64_t M = p.n_rows > 0 ? p.n_rows : N;
  if (p.n_rows < 0 || (M != N && !cplx) || M < 2 || M > (1 << 24)) {
    xc_set_error("n_rows: 0, or in [2, 2^24] for the complex kinds (XC_EXP, XC_LAGSPEC)");
    return XC_EINVAL;
  }
  if (p.trig_precompute != 0 && (p.trig_precompute != 1 || !(cplx || kind == XC_COS))) {
    xc_set_error("trig_precompute: 0, or 1 (Appendix A) for XC_COS / XC_EXP / XC_LAGSPEC");
    return XC_EINVAL;
  }
  if (kind == XC_LAGSPEC && !(std::isfinite(p.eta) && p.eta > 0.0)) {
    xc_set_error("XC_LAGSPEC needs eta > 0");
    return XC_EINVAL;
  }
  if (N < 2 || N > (1 << 24) || !nodes) {
    xc_set_error("N must be in [2, 2^24] and nodes non-null");
    return XC_EINVAL;
  }
  if (!(eps > 0.0 && eps < 1.0)) {
    xc_set_error("eps must be in (0,1)");
    return XC_EINVAL;
  }
  h->kind = kind == XC_LAGSPEC ? XC_EXP : (kind == XC_LAG2D ? XC_LAGUERRE : kind);
  h->ukind = kind;
  h->appA = p.trig_precompute == 1;
  if (p.thresh_mode != 0 && p.thresh_mode != 1) {
    xc_set_error("thresh_mode: 0 (per node, P:106) or 1 (global, P:198)");
    return XC_EINVAL;
  }
  if (p.thresh_mode == 1 && h->appA) {
    xc_set_error("thresh_mode = 1 with the Appendix A precompute");
    return XC_EUNSUPPORTED;
  }
  h->thresh_mode = kind == XC_LAG2D ? 1 : p.thresh_mode;  // the 2D blocks have no node axis (R-23)
  if (p.apply_path < 0 || p.apply_path > 2) {
    xc_set_error("apply_path: 0 (auto), 1 (tiled) or 2 (small-operator path)");
    return XC_EINVAL;
  }
  h->apply_path = p.apply_path;
  h->use_fork = getenv("XC_NO_FORK") == nullptr;  // A/B switch for measurements
  h->alpha = p.alpha;
  h->beta = p.beta;
  h->N = N;
  h->M = M;
  h->eps1 = p.eps1 > 0 ? p.eps1 : eps;
  h->eps2 = p.eps2 > 0 ? p.eps2 : (kind == XC_LAG2D ? 0.1 : 1e-2);
  h->dirs = p.dirs ? p.dirs : XC_DIR_A;
  if (kind == XC_LAG2D && h->dirs != XC_DIR_A) {
    xc_set_error("XC_LAG2D: XC_DIR_A only");
    return XC_EUNSUPPORTED;
  }
  h->device = p.device;
  if (!(h->eps1 < h->eps2) || !(h->eps2 < 1.0)) {
    xc_set_error("need eps1 < eps2 < 1");
    return XC_EINVAL;
  }
  if (kind == XC_JACOBI && !(p.alpha > -1.0 && p.beta > -1.0)) {
    xc_set_error("Jacobi alpha, beta must be > -1");
    return XC_EINVAL;
  }
  if ((h->dirs & XC_DIR_WAT) && !p.weights) {
    xc_set_error("XC_DIR_WAT needs weights");
    return XC_EINVAL;
  }
  // the input axis's tail items stage the t dense degrees as B rows of one shared-memory window
  // (<= XC_WMAX rows), so the cutoff is bounded
  if (p.dense_cutoff < 0 || p.dense_cutoff > XC_WMAX - 4) {
    xc_set_error("dense_cutoff: 0 (default 32) or in [1, " + std::to_string(XC_WMAX - 4) + "]");
    return XC_EINVAL;
  }
  XC_TRY(validate_nodes(kind, nodes, N));
  XC_CUDA(cudaSetDevice(p.device));
  h->user_nodes.assign(nodes, nodes + N);  // for xc_export
  if (h->dirs & XC_DIR_WAT) h->user_wt.assign(p.weights, p.weights + N);
  h->eta = p.eta;
  h->dense_cutoff = p.dense_cutoff > 0 ? p.dense_cutoff : 32;
  cudaStream_t st = (cudaStream_t)p.stream;

  PlanOut plan;
  XC_TRY(make_chain(h->kind, M, h->eps1, h->eps2, p.dense_cutoff > 0 ? p.dense_cutoff : 32, plan));
  h->zeta = plan.zeta;
  h->tail = plan.tail;
  h->blocks.resize(plan.blocks.size());
  int Lmax = 0;
  for (size_t i = 0; i < plan.blocks.size(); ++i) {
    h->blocks[i].L = plan.blocks[i].L;
    h->blocks[i].m_off = plan.blocks[i].m_off;
    h->blocks[i].keep_lo = plan.blocks[i].keep_lo;
    h->blocks[i].keep_hi = plan.blocks[i].keep_hi;
    Lmax = std::max(Lmax, plan.blocks[i].L);
  }
  if (kind == XC_LAGSPEC) {
    // R-21: C^T[m,j] = r_j^m / (eta/2 - i k_j), r_j = e^{i pi t_j}, t_j = 1 + (2/pi) atan(2 k_j / eta)
    // in (0, 2), ascending in k_j; t_j carried as hi + lo (80-bit), the scale folded into the entries
    std::vector<double> th(N), tl(N);
    std::vector<double2> sc(N);
    const long double PI = 3.141592653589793238462643383279502884L, e2 = 0.5L * (long double)p.eta;
    for (int64_t j = 0; j < N; ++j) {
      const long double kj = nodes[j];
      const long double t = 1.0L + (2.0L / PI) * atanl(kj / e2);
      th[j] = (double)t;
      tl[j] = (double)(t - (long double)th[j]);
      const long double den = e2 * e2 + kj * kj;
      sc[j] = make_double2((double)(e2 / den), (double)(kj / den));  // 1/(e2 - i k) = (e2 + i k)/den
    }
    if (!(th[0] > 0.0) || !(th[N - 1] < 2.0)) {
      xc_set_error("XC_LAGSPEC: |k| / eta too large (phase node at the circle's seam)");
      return XC_EINVAL;
    }
    XC_TRY(upload(h->nodes, th));
    XC_TRY(upload(h->nodes_lo, tl));
    XC_TRY(upload(h->cscale, sc));
  } else if (kind == XC_LAG2D) {
    // the grid continued past x_{N-1} for the extra rows of the 2D blocks (as the oracle's
    // lag2d_nodes_ext: x_{N-1} + i h, h = (x_{N-1} - x_0) / (N - 1))
    std::vector<double> xe(nodes, nodes + N);
    const double hh = (nodes[N - 1] - nodes[0]) / (double)(N - 1);
    for (int64_t i = 1; N - 1 + i < std::max<int64_t>(N, Lmax); ++i) {
      volatile double d = hh * (double)i;  // no contraction: the same two roundings as the oracle
      xe.push_back(nodes[N - 1] + d);
    }
    XC_TRY(upload(h->nodes, xe));
  } else {
    XC_TRY(upload(h->nodes, std::vector<double>(nodes, nodes + N)));
  }
  if (h->dirs & XC_DIR_WAT) XC_TRY(upload(h->wt, std::vector<double>(p.weights, p.weights + N)));

  h->bst = st;
  h->node_chunk = p.node_chunk;
  if (kind == XC_JACOBI) {
    std::vector<double2> jtab;
    jacobi_coeffs(p.alpha, p.beta, std::max(Lmax, h->tail) + 2, jtab, h->p0);
    XC_TRY(upload(h->djtab, jtab));
  }
  return XC_OK;
}

// Phase 2 (p2-p4): node bands of the nodes [n0, n1) of every block.
xc_status build_bands(xc_op* h, int n0, int n1) {
  for (auto& b : h->blocks) XC_TRY(build_block(h, b, h->djtab, h->p0, h->node_chunk, n0, n1, h->bst));
  return XC_OK;
}

// Phase 2a (thresh_mode = 1): each block's max |S|^2 over the nodes [n0, n1) into gmax2.
xc_status build_maxima(xc_op* h, int n0, int n1) {
  for (auto& b : h->blocks) XC_TRY(block_max2(h, b, h->djtab, h->p0, h->node_chunk, n0, n1, b.gmax2, h->bst));
  return XC_OK;
}

// The small-operator path (small.cu): eligible when XC_DIR_A of a real kind has at most
// kSmallMaxBlocks blocks, each with M = L/2 <= kSmallMaxM (one CTA's shared memory) and a
// 2-3-5 radix plan, and at most 4M entries in all (bins and tail); the choice depends on the
// operator only.  Builds the bin-major transpose of the node bands (nodes ascending per bin) and
// the tail rows, and the per-block tables of the in-shared-memory C2R.
xc_status build_small(xc_op* h, cudaStream_t st) {
  h->small_on = false;
  if (h->apply_path == 1 || !(h->dirs & XC_DIR_A) || h->kind == XC_EXP || h->ukind == XC_LAG2D) return XC_OK;
  bool ok = (int)h->blocks.size() <= kSmallMaxBlocks;
  int64_t ents = (int64_t)h->tail * h->N;
  // auto: blocks with M <= 1024 (c1); a longer block (c2: M = 3600) is faster on the tiled path
  // (two C2R passes spread over the SMs beat one shared-memory FFT per CTA and column: 27 vs 33 us)
  const int maxM = h->apply_path == 2 ? kSmallMaxM : 1024;
  for (auto& b : h->blocks) {
    ok = ok && b.L / 2 <= maxM;
    ents += b.nnz;
  }
  ok = ok && ents <= (4LL << 20);
  SmallBlocks sb{};
  for (size_t i = 0; ok && i < h->blocks.size(); ++i) {
    ok = small_radices(h->blocks[i].L / 2, sb.blk[i].f, sb.blk[i].nf);
  }
  if (!ok) {
    if (h->apply_path == 2) {
      xc_set_error("apply_path = 2: the operator is too large for the small-operator path");
      return XC_EUNSUPPORTED;
    }
    return XC_OK;
  }
  const int N = (int)h->N;
  // rows: every block's bins q < H (complex u rows), then the tail degrees
  std::vector<int64_t> cnt, out;
  for (auto& b : h->blocks) {
    for (int q = 0; q < b.H; ++q) out.push_back(b.ubase / 2 + q);
  }
  for (int j = 0; j < h->tail; ++j) out.push_back(-(int64_t)j - 1);
  const int rows = (int)out.size();
  std::vector<int64_t> ptr(rows + 1, 0);
  int64_t r0 = 0;
  for (auto& b : h->blocks) {
    for (int k = 0; k < N; ++k)
      for (int j = 0; j < b.h_len[k]; ++j) ptr[r0 + b.h_start[k] + j + 1]++;
    r0 += b.H;
  }
  for (int j = 0; j < h->tail; ++j) ptr[r0 + j + 1] = N;
  for (int r = 0; r < rows; ++r) ptr[r + 1] += ptr[r];
  std::vector<int> node(std::max<int64_t>(1, ptr[rows]));
  std::vector<double2> val(std::max<int64_t>(1, ptr[rows]));
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  r0 = 0;
  for (auto& b : h->blocks) {
    std::vector<double2> v(std::max<int64_t>(1, b.nnz));
    if (b.nnz > 0) XC_CUDA(cudaMemcpy(v.data(), b.vals.p, b.nnz * sizeof(double2), cudaMemcpyDeviceToHost));
    for (int k = 0; k < N; ++k)  // nodes ascending: the fixed summation order of every bin
      for (int j = 0; j < b.h_len[k]; ++j) {
        const int64_t e = fill[r0 + b.h_start[k] + j]++;
        node[e] = k;
        val[e] = v[b.h_off[k] + j];
      }
    r0 += b.H;
  }
  if (h->tail > 0) {
    std::vector<double> P((size_t)h->tail * N);
    XC_CUDA(cudaMemcpy(P.data(), h->tailP.p, P.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (int j = 0; j < h->tail; ++j)
      for (int k = 0; k < N; ++k) {
        const int64_t e = fill[r0 + j]++;
        node[e] = k;
        val[e] = make_double2(P[(size_t)j * N + k], 0.0);
      }
  }
  XC_TRY(upload(h->sm_ptr, ptr));
  XC_TRY(upload(h->sm_node, node));
  XC_TRY(upload(h->sm_val, val));
  XC_TRY(upload(h->sm_out, out));
  std::vector<int> lr;
  for (int r = 0; r < rows; ++r)
    if (ptr[r + 1] - ptr[r] > kSmallLong) lr.push_back(r);
  XC_TRY(upload(h->sm_long, lr));
  h->sm_op = SmallOp{(const int64_t*)h->sm_ptr.p, (const int*)h->sm_node.p, (const double2*)h->sm_val.p,
                     (const int64_t*)h->sm_out.p, rows, (const int*)h->sm_long.p, (int)lr.size()};
  // stage twiddles e^{+2 pi i n / M} of every block, concatenated
  std::vector<double2> tw;
  std::vector<size_t> twoff;
  const long double PI2 = 6.283185307179586476925286766559005768L;
  for (auto& b : h->blocks) {
    const int M = b.L / 2;
    twoff.push_back(tw.size());
    for (int n = 0; n < M; ++n) {
      const long double a = PI2 * (long double)n / (long double)M;
      tw.push_back(make_double2((double)cosl(a), (double)sinl(a)));
    }
  }
  XC_TRY(upload(h->sm_twM, tw));
  sb.nb = (int)h->blocks.size();
  sb.maxM = 0;
  for (int i = 0; i < sb.nb; ++i) {
    const BlockData& b = h->blocks[i];
    SmallBlk& k = sb.blk[i];
    k.M = b.L / 2;
    k.m_off = b.m_off;
    k.keep_lo = b.keep_lo;
    k.keep_hi = b.keep_hi;
    k.urow = b.ubase / 2;
    k.twh = (const double2*)b.twh.p;
    k.twM = (const double2*)h->sm_twM.p + twoff[i];
    k.yscale = (const double*)b.yscale.p;
    sb.maxM = std::max(sb.maxM, k.M);
  }
  h->sm_blocks = sb;
  h->small_on = true;
  (void)st;
  return XC_OK;
}

// Phase 3: global band offsets, dense tail entries, tensor-core tiles, info.
xc_status build_end(xc_op* h) {
  const int64_t N = h->N;
  const xc_kind kind = (xc_kind)h->kind;
  cudaStream_t st = h->bst;
  for (auto& b : h->blocks) XC_TRY(finalize_bands(h, b));
  // dense tail entries P[j][k] = phi_j(x_k), j < t
  if (h->tail > 0) {
    XC_TRY(dev_alloc(h->tailP, (size_t)h->tail * N * sizeof(double)));
    GenParams g{};
    g.kind = kind;
    g.L = h->tail;
    g.m_off = 0;
    g.nodes = (const double*)h->nodes.p;
    g.nc = (int)N;
    g.w = nullptr;
    g.jab = (const double2*)h->djtab.p;
    g.p0 = h->p0;
    XC_TRY(gen_entries_real(g, (double*)h->tailP.p, N, st));
    XC_CUDA(cudaStreamSynchronize(st));
  }
  if (h->dirs & XC_DIR_A) XC_TRY(build_output_axis(h, st));
  if (h->dirs & XC_DIR_WAT) XC_TRY(build_input_axis(h, st));
  if ((h->dirs & XC_DIR_A) && h->kind != XC_EXP)  // C2R twiddle tables now, not inside an apply
    for (auto& b : h->blocks) XC_TRY(c2r_prepare(b.fftM));
  XC_TRY(build_small(h, st));
  dev_free(h->djtab);
  XC_CUDA(cudaStreamSynchronize(st));

  // info
  xc_info_t& in = h->info;
  in.N = N;
  in.M = h->M;
  in.kind = h->ukind;
  in.zeta = h->zeta;
  in.eps1 = h->eps1;
  in.eps2 = h->eps2;
  in.n_blocks = (int)h->blocks.size();
  in.tail = h->tail;
  in.dirs = h->dirs;
  int64_t nnz = 0;
  double fft = 0;
  for (auto& b : h->blocks) {
    nnz += b.nnz;
    fft += fft_flops(b.L);
  }
  in.nnz = nnz;
  // complex x real: 2 FMA per kept entry; XC_EXP complex x complex: 4 FMA (and a complex FFT)
  in.flops_per_col_A = (kind == XC_EXP ? 8.0 : 4.0) * nnz + 2.0 * h->tail * N + (kind == XC_EXP ? 2.0 : 1.0) * fft;
  in.flops_per_col_WAT = in.flops_per_col_A;
  in.dmma_flops_per_col_A = 64.0 * h->mtstepsA;   // 8 x 4 FMA per M-tile step and column
  in.dmma_flops_per_col_WAT = 64.0 * h->mtstepsW;
  in.op_bytes_A = h->tilesA_n * 8 + (int64_t)h->nitemsA * sizeof(SpmmItem);
  in.op_bytes_WAT = h->tilesW_n * 8 + (int64_t)h->nitemsW * sizeof(SpmmItem);
  in.launches_A = (int)count_launches(h, XC_DIR_A, 1);
  in.launches_WAT = (int)count_launches(h, XC_DIR_WAT, 1);
  in.alg_bytes_per_col = (kind == XC_EXP ? 16.0 : 8.0) * (double)(h->N + h->M);
  in.alg_bytes_fixed = 20.0 * (double)nnz + 8.0 * h->tail * (double)N;
  return XC_OK;
}

// XC_LAG2D (R-23): per block pair (a = degree block, b = time block) the extended block E_ab,
// windowed on both axes, its 2D DFT (degree axis, transpose, time axis; rows k <= L_b/2 kept),
// the global threshold, then per time block the rows of all pairs merged into one CSR whose
// entries point at the prologue planes of their degree block.
xc_status build_2d(xc_op* h) {
  cudaStream_t st = h->bst;
  const int N = (int)h->N, t = h->tail, nb = (int)h->blocks.size();
  DevBuf none;
  for (auto& b : h->blocks) XC_TRY(block_setup(h, b, none));
  std::vector<int64_t> zrow(nb + 1, 0);  // rows of degree block a's prologue spectrum (interleaved)
  for (int a = 0; a < nb; ++a) zrow[a + 1] = zrow[a] + (int64_t)h->blocks[a].H;
  int Lmax = 0;
  for (auto& b : h->blocks) Lmax = std::max(Lmax, b.L);
  DevBuf F, S1, T, S2, scr, dmx, dcnt;
  const size_t big = (size_t)Lmax * Lmax * sizeof(double2);
  XC_TRY(dev_alloc(F, big));
  XC_TRY(dev_alloc(S1, big));
  XC_TRY(dev_alloc(T, big));
  XC_TRY(dev_alloc(S2, big));
  XC_TRY(dev_alloc(scr, big));
  XC_TRY(dev_alloc(dmx, sizeof(unsigned long long)));
  XC_TRY(dev_alloc(dcnt, (size_t)Lmax * sizeof(int)));
  int64_t total = 0;
  std::vector<int64_t> gptr(1, 0);  // all time blocks' rows stacked (one launch of the product)
  std::vector<Ent2D> gent;
  // the BSR form: groups of 8 rows of one time block, 8 x 4 blocks over z rows r4..r4+3
  std::vector<int64_t> bptr(1, 0);
  std::vector<int> br4, bgrow, bgnv;
  std::vector<double> btiles;
  int64_t urow = 0;  // first stacked u row of the current time block
  h->rowsA = 0;  // the apply's u_b buffers (Hermitian half, complex): 2 H_b double rows each
  for (auto& b : h->blocks) h->rowsA += 2 * (int64_t)b.H;
  for (int ib = 0; ib < nb; ++ib) {
    BlockData& bb = h->blocks[ib];
    const int Lb = bb.L, Hb = bb.H;
    std::vector<std::vector<int64_t>> pptr(nb);
    std::vector<std::vector<int>> pq(nb);
    std::vector<std::vector<double2>> pv(nb);
    for (int ia = 0; ia < nb; ++ia) {
      BlockData& ba = h->blocks[ia];
      const int La = ba.L;
      GenParams g{};
      g.kind = XC_LAGUERRE;
      g.L = La;
      g.m_off = 0;
      g.nodes = (const double*)h->nodes.p;  // time positions p < L_b: x_p of the continued grid
      g.nc = Lb;
      g.w = (const double*)ba.w.p;           // degree window W_a
      XC_TRY(gen_entries(g, (double2*)F.p, st));  // F[q * L_b + p] = w_a[q] l_q(x_p)
      XC_TRY(lag2d_scale_nodes((double2*)F.p, La, Lb, (const double*)bb.w.p, st));  // W_b
      FftIO io{};
      io.src = (const double2*)F.p;
      io.lds = Lb;
      io.dst = (double2*)S1.p;
      io.ldd = Lb;
      io.kmax = La;
      io.scale = 1.0 / sqrt((double)La);
      XC_TRY(fft_run(ba.fft, -1, PRO_PLAIN, EPI_PLAIN, io, Lb, (double2*)scr.p, st));  // degree axis
      XC_TRY(lag2d_transpose((const double2*)S1.p, (double2*)T.p, La, Lb, st));    // T[p * L_a + q]
      FftIO io2{};
      io2.src = (const double2*)T.p;
      io2.lds = La;
      io2.dst = (double2*)S2.p;
      io2.ldd = La;
      io2.kmax = Hb;  // the Hermitian half of the time axis
      io2.scale = 1.0 / sqrt((double)Lb);
      XC_TRY(fft_run(bb.fft, -1, PRO_PLAIN, EPI_PLAIN, io2, La, (double2*)scr.p, st));  // time axis
      DevBuf dq, dv;
      XC_TRY(lag2d_compact_rows((const double2*)S2.p, Hb, La, h->eps1, (unsigned long long*)dmx.p, (int*)dcnt.p,
                                pptr[ia], dq, dv, st));
      const int64_t n = pptr[ia][Hb];
      pq[ia].resize(n);
      pv[ia].resize(n);
      if (n > 0) {
        XC_CUDA(cudaMemcpy(pq[ia].data(), dq.p, n * sizeof(int), cudaMemcpyDeviceToHost));
        XC_CUDA(cudaMemcpy(pv[ia].data(), dv.p, n * sizeof(double2), cudaMemcpyDeviceToHost));
      }
      dev_free(dq);
      dev_free(dv);
    }
    // merge the pairs row by row (degree blocks in order, q ascending)
    std::vector<int64_t> ptr(Hb + 1, 0);
    for (int k = 0; k < Hb; ++k) {
      int64_t c = 0;
      for (int ia = 0; ia < nb; ++ia) c += pptr[ia][k + 1] - pptr[ia][k];
      ptr[k + 1] = ptr[k] + c;
    }
    std::vector<Ent2D> ent(ptr[Hb]);
    for (int k = 0; k < Hb; ++k) {
      int64_t o = ptr[k];
      for (int ia = 0; ia < nb; ++ia) {
        const int La = h->blocks[ia].L, Ha = h->blocks[ia].H;
        for (int64_t e = pptr[ia][k]; e < pptr[ia][k + 1]; ++e) {
          const int q = pq[ia][e];
          const bool cj = q >= Ha;  // z_a[q] = conj z_a[L_a - q] (real input)
          const int r = cj ? La - q : q;
          Ent2D en;
          en.v = pv[ia][e];
          en.re = (int)(zrow[ia] + r);
          en.im = cj ? 1 : 0;
          ent[o++] = en;
        }
      }
    }
    for (int k = 0; k < Hb; ++k) gptr.push_back(gptr.back() + (ptr[k + 1] - ptr[k]));
    gent.insert(gent.end(), ent.begin(), ent.end());
    for (int k0 = 0; k0 < Hb; k0 += 8) {
      std::map<int, std::array<double, 128>> blk;  // r4 -> Crr | Cri | Cir | Cii (ordered: deterministic)
      for (int i = 0; i < 8 && k0 + i < Hb; ++i)
        for (int64_t e = ptr[k0 + i]; e < ptr[k0 + i + 1]; ++e) {
          const Ent2D& en = ent[e];
          const int r4 = en.re & ~3, j = en.re - r4;
          auto it = blk.find(r4);
          if (it == blk.end()) {
            std::array<double, 128> z{};
            it = blk.emplace(r4, z).first;
          }
          double* T = it->second.data();
          const double vr = en.v.x, vi = en.v.y;
          const int f = 4 * i + j;
          T[f] += vr;                          // Crr
          T[32 + f] += en.im ? vi : -vi;       // Cri
          T[64 + f] += vi;                     // Cir
          T[96 + f] += en.im ? -vr : vr;       // Cii
        }
      for (auto& kv : blk) {
        br4.push_back(kv.first);
        btiles.insert(btiles.end(), kv.second.begin(), kv.second.end());
      }
      bptr.push_back(bptr.back() + (int64_t)blk.size());
      bgrow.push_back((int)(urow + k0));
      bgnv.push_back(std::min(8, Hb - k0));
    }
    urow += Hb;
    bb.nnz = ptr[Hb];
    total += bb.nnz;
  }
  for (auto& b : h->blocks) XC_TRY(c2r_prepare(b.fftM));  // C2R twiddle tables (not in an apply)
  XC_TRY(upload(h->ptr2d, gptr));
  XC_TRY(upload(h->ent2d, gent));
  h->rows2d = (int)gptr.size() - 1;
  std::vector<int> order(h->rows2d);
  for (int r = 0; r < h->rows2d; ++r) order[r] = r;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return gptr[a + 1] - gptr[a] > gptr[b + 1] - gptr[b]; });
  XC_TRY(upload(h->order2d, order));
  // segments of at most kBsrSeg blocks (one warp each); groups cut in several are summed in order
  std::vector<int64_t> sptr(1, 0);
  std::vector<int> srow, snv, sslot, rrow, rnv, rslot, rcnt;
  int nslots = 0;
  for (size_t g = 0; g + 1 < bptr.size(); ++g) {
    const int64_t nbk = bptr[g + 1] - bptr[g];
    const int ns = std::max<int64_t>(1, (nbk + kBsrSeg - 1) / kBsrSeg);
    for (int c = 0; c < ns; ++c) {
      sptr.push_back(std::min(bptr[g + 1], bptr[g] + (int64_t)(c + 1) * kBsrSeg));
      srow.push_back(bgrow[g]);
      snv.push_back(bgnv[g]);
      sslot.push_back(ns == 1 ? -1 : nslots + c);
    }
    if (ns > 1) {
      rrow.push_back(bgrow[g]);
      rnv.push_back(bgnv[g]);
      rslot.push_back(nslots);
      rcnt.push_back(ns);
      nslots += ns;
    }
  }
  sptr.back() = bptr.back();
  h->bsr_nseg = (int)srow.size();
  h->bsr_nred = (int)rrow.size();
  h->bsr_nslots = nslots;
  std::vector<int> sorder(h->bsr_nseg);
  for (int g = 0; g < h->bsr_nseg; ++g) sorder[g] = g;
  std::stable_sort(sorder.begin(), sorder.end(),
                   [&](int a, int b) { return sptr[a + 1] - sptr[a] > sptr[b + 1] - sptr[b]; });
  XC_TRY(upload(h->bsr_sptr, sptr));
  XC_TRY(upload(h->bsr_r4, br4));
  XC_TRY(upload(h->bsr_tiles, btiles));
  XC_TRY(upload(h->bsr_srow, srow));
  XC_TRY(upload(h->bsr_snv, snv));
  XC_TRY(upload(h->bsr_sslot, sslot));
  XC_TRY(upload(h->bsr_order, sorder));
  XC_TRY(upload(h->bsr_rrow, rrow));
  XC_TRY(upload(h->bsr_rnv, rnv));
  XC_TRY(upload(h->bsr_rslot, rslot));
  XC_TRY(upload(h->bsr_rcnt, rcnt));
  h->zrows2d = zrow[nb];
  dev_free(F);
  dev_free(S1);
  dev_free(T);
  dev_free(S2);
  dev_free(scr);
  dev_free(dmx);
  dev_free(dcnt);
  // direct-method tails: E[j * ld + k] = l_j(x_k)
  if (t > 0) {
    XC_TRY(dev_alloc(h->tailR, (size_t)N * t * sizeof(double)));
    XC_TRY(dev_alloc(h->tailC, (size_t)t * (N - t) * sizeof(double)));
    GenParams g{};
    g.kind = XC_LAGUERRE;
    g.m_off = 0;
    g.w = nullptr;
    g.L = N;
    g.nodes = (const double*)h->nodes.p;
    g.nc = t;
    XC_TRY(gen_entries_real(g, (double*)h->tailR.p, t, st));
    g.L = t;
    g.nodes = (const double*)h->nodes.p + t;
    g.nc = N - t;
    XC_TRY(gen_entries_real(g, (double*)h->tailC.p, N - t, st));
  }
  XC_CUDA(cudaStreamSynchronize(st));
  // info
  xc_info_t& in = h->info;
  in.N = N;
  in.M = N;
  in.kind = XC_LAG2D;
  in.zeta = h->zeta;
  in.eps1 = h->eps1;
  in.eps2 = h->eps2;
  in.n_blocks = nb;
  in.tail = t;
  in.dirs = h->dirs;
  in.nnz = total;
  double fft = 0;
  for (auto& b : h->blocks) fft += 2.0 * fft_flops(b.L);  // the prologue and the C2R epilogue
  // complex x complex: 4 FMA per stored entry; tails: 2 t N - t^2 FMA
  in.flops_per_col_A = 8.0 * total + 2.0 * (2.0 * t * N - (double)t * t) + fft;
  in.flops_per_col_WAT = 0;
  in.op_bytes_A = total * (int64_t)sizeof(Ent2D);
  in.launches_A = (int)count_launches(h, XC_DIR_A, 1);
  in.alg_bytes_per_col = 16.0 * (double)N;
  in.alg_bytes_fixed = 24.0 * (double)total + 8.0 * (2.0 * t * N - (double)t * t);  // Ent2D values + indices
  return XC_OK;
}

xc_status build_impl(xc_kind kind, const xc_params* prm, const double* nodes, int64_t N, double eps, xc_op* h) {
  XC_TRY(build_begin(kind, prm, nodes, N, eps, h));
  if (h->ukind == XC_LAG2D) return build_2d(h);
  if (h->thresh_mode == 1) XC_TRY(build_maxima(h, 0, (int)N));  // two passes: max, then threshold
  XC_TRY(build_bands(h, 0, (int)N));
  return build_end(h);
}

xc_status prof_harvest(xc_op* h, int slot) {
  if (h->ev_dir[slot] == 0) return XC_OK;
  cudaEvent_t* e = &h->ev[4 * slot];
  XC_CUDA(cudaEventSynchronize(e[3]));
  float t01, t12, t23, t03;
  XC_CUDA(cudaEventElapsedTime(&t01, e[0], e[1]));
  XC_CUDA(cudaEventElapsedTime(&t12, e[1], e[2]));
  XC_CUDA(cudaEventElapsedTime(&t23, e[2], e[3]));
  XC_CUDA(cudaEventElapsedTime(&t03, e[0], e[3]));
  if (h->ev_dir[slot] == XC_DIR_A) {
    h->ms_spmm += t01;
    h->ms_fft += t12;
  } else {
    h->ms_fft += t01;
    h->ms_spmm += t12;
  }
  h->ms_red += t23;
  h->ms_tot += t03;
  h->n_prof++;
  h->ev_dir[slot] = 0;
  return XC_OK;
}

// SpMM windows for a batch of B columns: node order, or heaviest first (the copy behind it) when
// the grid is only a few waves deep
const SpmmWin* wins_for(const DevBuf& w, int nwins, int64_t B) {
  const int64_t ctas = (int64_t)nwins * ((B + 63) / 64);
  return (const SpmmWin*)w.p + ((ctas < 16 * (int64_t)sm_count()) ? nwins : 0);
}

// Per-block phases (the blocks are independent there): block 1 stays on the caller's stream,
// block 2 goes to s_aux[0], blocks 3.. round robin to s_aux[1..3] (high priority: their few CTAs
// are dispatched ahead of block 1's persistent grid), each stream with its own FFT scratch;
// fork/join by events, so the phase also works under CUDA-graph capture.
bool fork_begin(xc_op* h, Ws& w, cudaStream_t st, int64_t B, xc_status& err) {
  err = XC_OK;
  w.naux = naux_for(h->N, B);
  if (!h->use_fork || h->blocks.size() < 2 || !w.scratch_aux[0] || !w.s_aux[0]) return false;
  auto fail = [&](cudaError_t e) {
    xc_set_error(std::string("fork: ") + cudaGetErrorString(e));
    err = XC_ECUDA;
    return false;
  };
  cudaError_t e;
  if ((e = cudaEventRecord(w.ev_fork, st)) != cudaSuccess) return fail(e);
  const int na = std::min<int>(w.naux, (int)h->blocks.size() - 1);  // streams in use
  for (int i = 0; i < na; ++i)
    if ((e = cudaStreamWaitEvent(w.s_aux[i], w.ev_fork, 0)) != cudaSuccess) return fail(e);
  return true;
}

xc_status fork_end(xc_op* h, Ws& w, cudaStream_t st, bool fork) {
  if (!fork) return XC_OK;
  const int na = std::min<int>(w.naux, (int)h->blocks.size() - 1);
  for (int i = 0; i < na; ++i) {
    XC_CUDA(cudaEventRecord(w.ev_join[i], w.s_aux[i]));
    XC_CUDA(cudaStreamWaitEvent(st, w.ev_join[i], 0));
  }
  return XC_OK;
}

cudaStream_t fork_stream(const Ws& w, cudaStream_t st, bool fork, int ib) {
  return (fork && ib > 0) ? w.s_aux[aux_of(ib, w.naux)] : st;
}

double2* fork_scratch(const Ws& w, bool fork, int ib) {
  return (fork && ib > 0) ? w.scratch_aux[aux_of(ib, w.naux)] : w.scratch;
}

xc_status apply_impl(xc_op* h, Ws& w, xc_dir dir, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t B,
                     cudaStream_t st) {
  if (B < 1 || ldx < B || ldy < B || !X || !Y) {
    xc_set_error("apply: need B >= 1, ldx >= B, ldy >= B, non-null X and Y");
    return XC_EINVAL;
  }
  if (B > (1 << 24)) {
    xc_set_error("apply: B too large");
    return XC_EINVAL;
  }
  if (!(h->dirs & dir) || h->xstage != 0) {
    xc_set_error(h->xstage ? "apply: distributed build not finished" : "apply: direction was not built");
    return XC_ESTATE;
  }
  if (B > w.B) {
    xc_set_error("apply: B exceeds the workspace (xc_reserve / xc_attach_workspace first)");
    return XC_ESTATE;
  }
  cudaEvent_t* ev = nullptr;
  if (h->prof) {
    int slot = (int)(h->ev_count++ % xc_op::kRing);
    XC_TRY(prof_harvest(h, slot));
    ev = &h->ev[4 * slot];
    // XC_LAG2D phases: prologue FFTs, products, C2R + tails -- the input axis's order
    h->ev_dir[slot] = h->ukind == XC_LAG2D ? XC_DIR_WAT : dir;
  }
  auto mark = [&](int i) -> xc_status {
    if (ev) XC_CUDA(cudaEventRecord(ev[i], st));
    return XC_OK;
  };
  const int64_t Bp = pad_cols(B);
  const int N = (int)h->N;
  XC_TRY(mark(0));
  if (h->ukind == XC_LAG2D) {  // R-23: prologues, merged 2D products + C2R per time block, tails
    const int nb = (int)h->blocks.size();
    xc_status ferr;
    bool fork = fork_begin(h, w, st, B, ferr);
    XC_TRY(ferr);
    int64_t zrow = 0;  // plane rows of the degree blocks, stacked with the row stride Bp of this call
    for (int a = 0; a < nb; ++a) {
      BlockData& b = h->blocks[a];
      FftIO io{};
      io.X = X;
      io.ldx = ldx;
      io.winv = (const double*)b.winv.p;
      io.keep_lo = b.keep_lo;
      io.keep_hi = b.keep_hi;
      io.m_off = b.m_off;
      io.dst = (double2*)w.zpl + zrow * Bp;  // the rows the CSR entries address (build_2d)
      zrow += b.H;
      io.ldd = Bp;
      io.kmax = b.H;
      io.scale = 1.0 / sqrt((double)b.L);
      XC_TRY(fft_run(b.fft, +1, PRO_XREAL, EPI_PLAIN, io, (int)B, fork_scratch(w, fork, a),
                     fork_stream(w, st, fork, a)));
    }
    XC_TRY(fork_end(h, w, st, fork));
    // the 4 rows past the last spectrum row: read by the DMMA blocks (times zero), so finite
    XC_CUDA(cudaMemsetAsync(w.zpl + 2 * zrow * Bp, 0, 8 * Bp * sizeof(double), st));
    XC_TRY(mark(1));
    // the products of all time blocks in one launch (u_b stacked in partA), then the C2R
    // epilogues and the tails
    static const bool use_csr = getenv("XC_2D_CSR") != nullptr;  // the DFMA CSR product (comparison)
    if (use_csr) {
      XC_TRY(lag2d_spmm((const int64_t*)h->ptr2d.p, (const Ent2D*)h->ent2d.p, (const int*)h->order2d.p, h->rows2d,
                        (const double2*)w.zpl, Bp, (double2*)w.partA, Bp, (int)B, st));
    } else {
      Bsr2D m{(const int64_t*)h->bsr_sptr.p, (const int*)h->bsr_r4.p,  (const double*)h->bsr_tiles.p,
              (const int*)h->bsr_srow.p,     (const int*)h->bsr_snv.p, (const int*)h->bsr_sslot.p,
              (const int*)h->bsr_order.p,    h->bsr_nseg,              (const int*)h->bsr_rrow.p,
              (const int*)h->bsr_rnv.p,      (const int*)h->bsr_rslot.p, (const int*)h->bsr_rcnt.p,
              h->bsr_nred,                   h->bsr_nslots};
      XC_TRY(lag2d_bsr(m, (const double2*)w.zpl, Bp, (double2*)w.partA, Bp, w.bsr_part, (int)B,
                       st));
    }
    XC_TRY(mark(2));
    fork = fork_begin(h, w, st, B, ferr);
    XC_TRY(ferr);
    int64_t uoff = 0;
    for (int ib = 0; ib < nb; ++ib) {
      BlockData& b = h->blocks[ib];
      double2* U = (double2*)w.partA + uoff * Bp;
      uoff += b.H;
      FftIO io{};
      io.Uc = U;
      io.ldu = Bp;
      io.twh = (const double2*)b.twh.p;
      io.M = b.L / 2;
      io.H = b.H;
      io.Y = Y;
      io.ldy = ldy;
      io.yscale = (const double*)b.yscale.p;
      io.keep_lo = b.keep_lo;
      io.keep_hi = b.keep_hi;
      io.m_off = b.m_off;
      XC_TRY(c2r_run(b.fftM, io, (int)B, fork_scratch(w, fork, ib), fork_stream(w, st, fork, ib)));
    }
    XC_TRY(fork_end(h, w, st, fork));  // the tail columns add into rows the epilogues wrote
    const int t = h->tail;
    if (t > 0) {
      const int64_t cap = (int64_t)((h->N + 127) / 128) * h->tail * Bp;
      XC_TRY(dense_tn((const double*)h->tailR.p, N, t, t, X, ldx, Y, ldy, (int)B, false, w.tailpart, cap,
                      st));
      XC_TRY(dense_tn((const double*)h->tailC.p, t, N - t, N - t, X, ldx, Y + (int64_t)t * ldy, ldy, (int)B, true,
                      w.tailpart, cap, st));
    }
    return mark(3);
  }
  if (dir == XC_DIR_A && h->kind == XC_EXP) {
    // complex input in planar form: B row 2k = Re X[k], 2k+1 = Im X[k] (rows N.. are the imag plane)
    SpmmSrcs s{};
    s.re[0] = X;
    s.im[0] = X + (int64_t)N * ldx;
    s.nrows[0] = N;
    s.ld[0] = ldx;
    XC_TRY(spmm_run(wins_for(h->winsA, h->nwinsA, B), h->nwinsA, (const SpmmItem*)h->itemsA.p,
                    (const double*)h->tilesA.p, s, w.partA, Bp, (int)B, st));
    XC_TRY(mark(1));
    for (auto& b : h->blocks) {
      double* U = w.partA + b.ubase * Bp;
      if (b.split)
        XC_TRY(reduce_rows8(w.partA, Bp, (const int64_t*)b.grp_base.p, (const int*)b.grp_nch.p,
                            8 * b.ngroups, nullptr, U, Bp, (int)Bp, b.grp_nch_max, st));
      // v = F* u over all L bins (complex inverse DFT), then Fe2 discard and W^{-1}
      FftIO io{};
      io.src = reinterpret_cast<const double2*>(U);
      io.lds = Bp;
      io.Y = Y;
      io.ldy = ldy;
      io.ypl = h->M * ldy;  // planar complex output: M degree rows
      io.yscale = (const double*)b.yscale.p;
      io.keep_lo = b.keep_lo;
      io.keep_hi = b.keep_hi;
      io.m_off = b.m_off;
      XC_TRY(fft_run(b.fft, +1, PRO_PLAIN, EPI_CY, io, (int)B, w.scratch, st));
    }
    XC_TRY(mark(2));
    return mark(3);
  }
  if (dir == XC_DIR_A && h->small_on) {  // small operators: two launches (small.cu)
    XC_TRY(small_spmm(h->sm_op, X, ldx, (double2*)w.partA, Bp, Y, ldy, (int)B, N, st));
    XC_TRY(mark(1));
    XC_TRY(small_c2r(h->sm_blocks, (const double2*)w.partA, Bp, Y, ldy, (int)B, st));
    XC_TRY(mark(2));
    return mark(3);
  }
  if (dir == XC_DIR_A) {
    SpmmSrcs s{};
    s.re[0] = X;
    s.im[0] = nullptr;
    s.nrows[0] = N;
    s.ld[0] = ldx;
    XC_TRY(spmm_run(wins_for(h->winsA, h->nwinsA, B), h->nwinsA, (const SpmmItem*)h->itemsA.p,
                    (const double*)h->tilesA.p, s, w.partA, Bp, (int)B, st));
    XC_TRY(mark(1));
    const int nb = (int)h->blocks.size();
    xc_status ferr;
    const bool fork = fork_begin(h, w, st, B, ferr);
    XC_TRY(ferr);
    for (int ib = 0; ib < nb; ++ib) {
      BlockData& b = h->blocks[ib];
      cudaStream_t sb = fork_stream(w, st, fork, ib);
      double2* scr = fork_scratch(w, fork, ib);
      double* U = w.partA + b.ubase * Bp;
      if (b.split)  // interleaved complex rows: reduce all Bp doubles of each double row
        XC_TRY(reduce_rows8(w.partA, Bp, (const int64_t*)b.grp_base.p, (const int*)b.grp_nch.p,
                            8 * b.ngroups, nullptr, U, Bp, (int)Bp, b.grp_nch_max, sb));
      FftIO io{};
      io.Uc = reinterpret_cast<const double2*>(U);
      io.ldu = Bp;
      io.twh = (const double2*)b.twh.p;
      io.M = b.L / 2;
      io.H = b.H;
      io.Y = Y;
      io.ldy = ldy;
      io.yscale = (const double*)b.yscale.p;
      io.keep_lo = b.keep_lo;
      io.keep_hi = b.keep_hi;
      io.m_off = b.m_off;
      XC_TRY(c2r_run(b.fftM, io, (int)B, scr, sb));
      // the dense tail's rows [0, t) are disjoint from every block's kept rows [s_i, e_i) (the
      // chain ends at s = t, m_off = 0), so its reduction runs beside the FFT phase, after block
      // 2 on that block's stream (the lightest), instead of after the join (c3: 19 us at the end)
      if (ib == std::min(1, nb - 1) && h->tail > 0)
        XC_TRY(reduce_rows8(w.partA, Bp, (const int64_t*)h->tail_base.p, (const int*)h->tail_nch.p,
                            h->tail, nullptr, Y, ldy, (int)B, h->tail_nch_max, sb));
    }
    XC_TRY(fork_end(h, w, st, fork));
    XC_TRY(mark(2));
    if (nb == 0 && h->tail > 0)  // a tail-only operator (N <= the dense cutoff)
      XC_TRY(reduce_rows8(w.partA, Bp, (const int64_t*)h->tail_base.p, (const int*)h->tail_nch.p,
                          h->tail, nullptr, Y, ldy, (int)B, h->tail_nch_max, st));
    return mark(3);
  }
  // XC_DIR_WAT
  if (h->kind == XC_EXP) {
    BlockData& b = h->blocks[0];
    double* zre = w.zpl + w.zoff[0];
    double* zim = zre + (int64_t)b.H * Bp;
    FftIO io{};
    io.X = X;
    io.ldx = ldx;
    io.xpl = h->M * ldx;  // planar complex input: M degree rows
    io.winv = (const double*)b.winv.p;
    io.keep_lo = b.keep_lo;
    io.keep_hi = b.keep_hi;
    io.m_off = b.m_off;
    io.zre = zre;
    io.zim = zim;
    io.ldz = Bp;
    io.H = b.H;
    io.scale = 1.0 / sqrt((double)b.L);
    XC_TRY(fft_run(b.fft, +1, PRO_XCPLX, EPI_ZPLANES, io, (int)B, w.scratch, st));
    SpmmSrcs s{};
    s.re[0] = zre;
    s.im[0] = zim;
    s.nrows[0] = b.H;
    s.ld[0] = Bp;
    XC_TRY(mark(1));
    XC_TRY(spmm_run(wins_for(h->winsW, h->nwinsW, B), h->nwinsW, (const SpmmItem*)h->itemsW.p,
                    (const double*)h->tilesW.p, s, w.partW, Bp, (int)B, st));
    XC_TRY(mark(2));
    XC_TRY(reduce_rows8(w.partW, Bp, (const int64_t*)h->nodeg_base.p, (const int*)h->nodeg_nch.p,
                        N, (const double*)h->wt.p, Y, ldy, (int)B, h->nodeg_nch_max, st));
    XC_TRY(reduce_rows8(w.partW, Bp, (const int64_t*)h->nodeg_base_im.p,
                        (const int*)h->nodeg_nch.p, N, (const double*)h->wt.p, Y + (int64_t)N * ldy, ldy, (int)B, h->nodeg_nch_max, st));
    return mark(3);
  }
  SpmmSrcs s{};
  const int nb = (int)h->blocks.size();
  xc_status ferr;
  const bool fork = fork_begin(h, w, st, B, ferr);
  XC_TRY(ferr);
  for (int i = 0; i < nb; ++i) {
    BlockData& b = h->blocks[i];
    double* zre = w.zpl + w.zoff[i];
    double* zim = zre + (int64_t)b.H * Bp;
    FftIO io{};
    io.X = X;
    io.ldx = ldx;
    io.winv = (const double*)b.winv.p;
    io.keep_lo = b.keep_lo;
    io.keep_hi = b.keep_hi;
    io.m_off = b.m_off;
    io.zre = zre;
    io.zim = zim;
    io.ldz = Bp;
    io.H = b.H;
    io.scale = 1.0 / sqrt((double)b.L);
    XC_TRY(fft_run(b.fft, +1, PRO_XREAL, EPI_ZPLANES, io, (int)B, fork_scratch(w, fork, i),
                   fork_stream(w, st, fork, i)));
    s.re[i] = zre;
    s.im[i] = zim;
    s.nrows[i] = b.H;
    s.ld[i] = Bp;
  }
  XC_TRY(fork_end(h, w, st, fork));
  s.re[nb] = X;
  s.im[nb] = nullptr;
  s.nrows[nb] = h->tail;
  s.ld[nb] = ldx;
  XC_TRY(mark(1));
  XC_TRY(spmm_run(wins_for(h->winsW, h->nwinsW, B), h->nwinsW, (const SpmmItem*)h->itemsW.p,
                  (const double*)h->tilesW.p, s, w.partW, Bp, (int)B, st));
  XC_TRY(mark(2));
  XC_TRY(reduce_rows8(w.partW, Bp, (const int64_t*)h->nodeg_base.p, (const int*)h->nodeg_nch.p, N,
                      (const double*)h->wt.p, Y, ldy, (int)B, h->nodeg_nch_max, st));
  return mark(3);
}

void ws_release(Ws& w) {
  clear_graphs(w);
  for (int i = 0; i < kAux; ++i)
    if (w.s_aux[i]) {
      cudaStreamSynchronize(w.s_aux[i]);
      cudaStreamDestroy(w.s_aux[i]);
      cudaEventDestroy(w.ev_join[i]);
      w.s_aux[i] = nullptr;
    }
  if (w.ev_fork) cudaEventDestroy(w.ev_fork);
  w.ev_fork = nullptr;
  dev_free(w.own);
  w.base = nullptr;
  w.bytes = 0;
  w.B = 0;
}

void destroy_impl(xc_op* h) {
  for (auto& e : h->ev) cudaEventDestroy(e);
  h->ev.clear();
  ws_release(h->def);
  for (Ws* w : h->att) {
    ws_release(*w);
    delete w;
  }
  h->att.clear();
  if (h->s_in) {
    cudaStreamSynchronize(h->s_in);
    cudaStreamSynchronize(h->s_out);
    cudaStreamDestroy(h->s_in);
    cudaStreamDestroy(h->s_out);
    for (int i = 0; i < xc_op::kSlots; ++i) {
      cudaEventDestroy(h->ev_in[i]);
      cudaEventDestroy(h->ev_cmp[i]);
      cudaEventDestroy(h->ev_out[i]);
    }
    cudaEventDestroy(h->ev_start);
    h->s_in = h->s_out = nullptr;
  }
  for (auto& b : h->blocks) {
    fft_plan_free(b.fft);
    fft_plan_free(b.fftM);
    dev_free(b.twh);
    dev_free(b.w); dev_free(b.yscale); dev_free(b.winv);
    dev_free(b.start); dev_free(b.len); dev_free(b.off); dev_free(b.vals);
    dev_free(b.grp_base); dev_free(b.grp_nch);
  }
  DevBuf* all[] = {&h->nodes, &h->wt, &h->tailP, &h->itemsA, &h->tilesA, &h->winsA, &h->tail_base, &h->tail_nch,
                   &h->itemsW, &h->tilesW, &h->winsW, &h->nodeg_base, &h->nodeg_nch, &h->nodeg_base_im,
                   &h->Xh, &h->Yh, &h->xsend, &h->xrecv, &h->djtab, &h->nodes_lo, &h->cscale,
                   &h->tailR, &h->tailC, &h->ptr2d, &h->ent2d, &h->order2d,
                   &h->bsr_sptr, &h->bsr_r4, &h->bsr_tiles, &h->bsr_srow, &h->bsr_snv, &h->bsr_sslot,
                   &h->bsr_order, &h->bsr_rrow, &h->bsr_rnv, &h->bsr_rslot, &h->bsr_rcnt,
                   &h->sm_ptr, &h->sm_node, &h->sm_val, &h->sm_out, &h->sm_twM, &h->sm_long};
  for (DevBuf* b : all) dev_free(*b);
}

}  // namespace

// =========================================================================== C ABI
extern "C" {

xc_status xc_params_default(xc_params* p) {
  if (!p) return XC_EINVAL;
  memset(p, 0, sizeof(*p));
  return XC_OK;
}

xc_status xc_build_compressed(xc_kind kind, const xc_params* p, const double* nodes, int64_t N, double eps,
                              xc_handle* out) {
  if (!out) {
    xc_set_error("out is null");
    return XC_EINVAL;
  }
  *out = nullptr;
  xc_op* h = new xc_op();
  xc_status s = build_impl(kind, p, nodes, N, eps, h);
  if (s != XC_OK) {
    destroy_impl(h);
    delete h;
    return s;
  }
  *out = h;
  return XC_OK;
}

namespace {

// The computation stage on given node bands (xc_build_from_bands, xc_import).  windows (import):
// the exported per-block windows, which the rebuilt plan must reproduce bit for bit.
xc_status from_bands_impl(xc_kind kind, const xc_params* p, const double* nodes, int64_t N, double eps,
                          const int* const* start, const int* const* len, const double* const* vals,
                          const std::vector<std::vector<double>>* windows, xc_op* h) {
  XC_TRY(build_begin(kind, p, nodes, N, eps, h));
  if (windows && windows->size() != h->blocks.size()) {
    xc_set_error("import: the file's block chain differs from the plan of its parameters");
    return XC_EINVAL;
  }
  for (size_t i = 0; i < h->blocks.size(); ++i) {
    BlockData& b = h->blocks[i];
    DevBuf none;
    XC_TRY(block_setup(h, b, none));
    if (windows && (*windows)[i] != b.h_w) {
      xc_set_error("import: block " + std::to_string(i) + "'s window differs from the plan's");
      return XC_EINVAL;
    }
    if (!start[i] || !len[i] || !vals[i]) {
      xc_set_error("build_from_bands: null band arrays of block " + std::to_string(i));
      return XC_EINVAL;
    }
    b.h_start.assign(start[i], start[i] + N);
    b.h_len.assign(len[i], len[i] + N);
    b.h_off.assign(N + 1, 0);
    int64_t tot = 0;
    for (int64_t k = 0; k < N; ++k) {
      if (b.h_len[k] < 0 || b.h_len[k] > b.H || b.h_start[k] < 0 || b.h_start[k] >= std::max(1, b.H) ||
          (h->kind != XC_EXP && b.h_start[k] + b.h_len[k] > b.H)) {
        xc_set_error("build_from_bands: band out of range at block " + std::to_string(i) + ", node " +
                     std::to_string(k));
        return XC_EINVAL;
      }
      tot += b.h_len[k];
    }
    std::vector<double2> v(std::max<int64_t>(1, tot));
    for (int64_t q = 0; q < tot; ++q) v[q] = make_double2(vals[i][2 * q], vals[i][2 * q + 1]);
    XC_TRY(upload(b.vals, v));
    XC_TRY(upload(b.start, b.h_start));
    XC_TRY(upload(b.len, b.h_len));
    b.loc_count = tot;
  }
  return build_end(h);
}

// ---- operator files (xc_export / xc_import), little-endian, version 1 -----------------------
constexpr char kOpMagic[8] = {'X', 'C', 'O', 'P', 'E', 'R', '0', '1'};
struct OpFileHdr {
  char magic[8];
  int32_t kind, thresh_mode, trig_precompute, dense_cutoff, dirs, n_blocks, tail, reserved;
  int64_t N, M;
  double alpha, beta, eta, eps1, eps2, zeta;
};
struct OpFileBlk {
  int32_t L, m_off, keep_lo, keep_hi;
  int64_t nnz;
};

}  // namespace

xc_status xc_build_from_bands(xc_kind kind, const xc_params* p, const double* nodes, int64_t N, double eps,
                              const int* const* start, const int* const* len, const double* const* vals,
                              xc_handle* out) {
  if (!out || !start || !len || !vals) {
    xc_set_error("build_from_bands: null argument");
    return XC_EINVAL;
  }
  *out = nullptr;
  if (kind == XC_LAG2D || (p && p->trig_precompute != 0)) {
    xc_set_error("build_from_bands: node bands of the 1D operators with the Kaiser window only");
    return XC_EUNSUPPORTED;
  }
  xc_op* h = new xc_op();
  xc_status s = from_bands_impl(kind, p, nodes, N, eps, start, len, vals, nullptr, h);
  if (s != XC_OK) {
    destroy_impl(h);
    delete h;
    return s;
  }
  *out = h;
  return XC_OK;
}

xc_status xc_export(xc_handle h, const char* path) {
  if (!h || !path) {
    xc_set_error("export: null argument");
    return XC_EINVAL;
  }
  if (h->ukind == XC_LAG2D || h->xstage != 0) {
    xc_set_error(h->xstage ? "export: distributed build not finished" : "export: XC_LAG2D operators are not exported");
    return h->xstage ? XC_ESTATE : XC_EUNSUPPORTED;
  }
  XC_CUDA(cudaSetDevice(h->device));
  OpFileHdr hd{};
  memcpy(hd.magic, kOpMagic, 8);
  hd.kind = h->ukind;
  hd.thresh_mode = h->thresh_mode;
  hd.trig_precompute = h->appA ? 1 : 0;
  hd.dense_cutoff = h->dense_cutoff;
  hd.dirs = h->dirs;
  hd.n_blocks = (int32_t)h->blocks.size();
  hd.tail = h->tail;
  hd.N = h->N;
  hd.M = h->M;
  hd.alpha = h->alpha;
  hd.beta = h->beta;
  hd.eta = h->eta;
  hd.eps1 = h->eps1;
  hd.eps2 = h->eps2;
  hd.zeta = h->zeta;
  FILE* f = fopen(path, "wb");
  if (!f) {
    xc_set_error(std::string("export: cannot open ") + path);
    return XC_EINVAL;
  }
  bool ok = fwrite(&hd, sizeof(hd), 1, f) == 1;
  ok = ok && fwrite(h->user_nodes.data(), sizeof(double), h->N, f) == (size_t)h->N;
  if (h->dirs & XC_DIR_WAT) ok = ok && fwrite(h->user_wt.data(), sizeof(double), h->N, f) == (size_t)h->N;
  for (auto& b : h->blocks) {
    if (!ok) break;
    OpFileBlk bk{b.L, b.m_off, b.keep_lo, b.keep_hi, b.nnz};
    std::vector<double2> v(std::max<int64_t>(1, b.nnz));
    if (b.nnz > 0) {
      cudaError_t e = cudaMemcpy(v.data(), b.vals.p, b.nnz * sizeof(double2), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) {
        fclose(f);
        xc_set_error(std::string("export: ") + cudaGetErrorString(e));
        return XC_ECUDA;
      }
    }
    ok = fwrite(&bk, sizeof(bk), 1, f) == 1;
    ok = ok && fwrite(b.h_w.data(), sizeof(double), b.L, f) == (size_t)b.L;
    ok = ok && fwrite(b.h_start.data(), sizeof(int), h->N, f) == (size_t)h->N;
    ok = ok && fwrite(b.h_len.data(), sizeof(int), h->N, f) == (size_t)h->N;
    ok = ok && (b.nnz == 0 || fwrite(v.data(), sizeof(double2), b.nnz, f) == (size_t)b.nnz);
  }
  if (fclose(f) != 0) ok = false;
  if (!ok) {
    xc_set_error(std::string("export: write failed: ") + path);
    return XC_EINVAL;
  }
  return XC_OK;
}

xc_status xc_import(const char* path, const xc_params* prm, xc_handle* out) {
  if (!path || !out) {
    xc_set_error("import: null argument");
    return XC_EINVAL;
  }
  *out = nullptr;
  FILE* f = fopen(path, "rb");
  if (!f) {
    xc_set_error(std::string("import: cannot open ") + path);
    return XC_EINVAL;
  }
  auto bad = [&](const std::string& m) {
    fclose(f);
    xc_set_error("import: " + m + " (" + path + ")");
    return XC_EINVAL;
  };
  OpFileHdr hd{};
  if (fread(&hd, sizeof(hd), 1, f) != 1 || memcmp(hd.magic, kOpMagic, 8) != 0) return bad("not an operator file");
  if (hd.N < 2 || hd.N > (1 << 24) || hd.n_blocks < 0 || hd.n_blocks >= XC_MAX_BLOCKS) return bad("bad header");
  const int64_t N = hd.N;
  std::vector<double> nodes(N), wt;
  if (fread(nodes.data(), sizeof(double), N, f) != (size_t)N) return bad("truncated nodes");
  if (hd.dirs & XC_DIR_WAT) {
    wt.resize(N);
    if (fread(wt.data(), sizeof(double), N, f) != (size_t)N) return bad("truncated weights");
  }
  std::vector<std::vector<int>> st(hd.n_blocks), ln(hd.n_blocks);
  std::vector<std::vector<double>> vals(hd.n_blocks), win(hd.n_blocks);
  std::vector<OpFileBlk> bks(hd.n_blocks);
  for (int i = 0; i < hd.n_blocks; ++i) {
    OpFileBlk& bk = bks[i];
    if (fread(&bk, sizeof(bk), 1, f) != 1 || bk.L < 2 || bk.nnz < 0) return bad("bad block header");
    win[i].resize(bk.L);
    st[i].resize(N);
    ln[i].resize(N);
    vals[i].resize(2 * std::max<int64_t>(1, bk.nnz));
    if (fread(win[i].data(), sizeof(double), bk.L, f) != (size_t)bk.L ||
        fread(st[i].data(), sizeof(int), N, f) != (size_t)N || fread(ln[i].data(), sizeof(int), N, f) != (size_t)N ||
        (bk.nnz > 0 && fread(vals[i].data(), sizeof(double2), bk.nnz, f) != (size_t)bk.nnz))
      return bad("truncated block " + std::to_string(i));
  }
  fclose(f);
  xc_params p;
  xc_params_default(&p);
  if (prm) {  // device and stream from the caller; everything that shapes the operator from the file
    p.device = prm->device;
    p.stream = prm->stream;
    p.node_chunk = prm->node_chunk;
    p.apply_path = prm->apply_path;
  }
  p.alpha = hd.alpha;
  p.beta = hd.beta;
  p.eps1 = hd.eps1;
  p.eps2 = hd.eps2;
  p.eta = hd.eta;
  p.dense_cutoff = hd.dense_cutoff;
  p.dirs = hd.dirs;
  p.n_rows = hd.M != N ? hd.M : 0;
  p.trig_precompute = hd.trig_precompute;
  p.thresh_mode = hd.thresh_mode;
  p.weights = wt.empty() ? nullptr : wt.data();
  std::vector<const int*> sp(hd.n_blocks), lp(hd.n_blocks);
  std::vector<const double*> vp(hd.n_blocks);
  for (int i = 0; i < hd.n_blocks; ++i) {
    sp[i] = st[i].data();
    lp[i] = ln[i].data();
    vp[i] = vals[i].data();
  }
  xc_op* h = new xc_op();
  xc_status s = from_bands_impl((xc_kind)hd.kind, &p, nodes.data(), N, hd.eps1, sp.data(), lp.data(), vp.data(),
                                &win, h);
  if (s == XC_OK) {
    for (int i = 0; i < hd.n_blocks && s == XC_OK; ++i) {
      const BlockData& b = h->blocks[i];
      if (b.L != bks[i].L || b.m_off != bks[i].m_off || b.keep_lo != bks[i].keep_lo || b.keep_hi != bks[i].keep_hi ||
          b.nnz != bks[i].nnz) {
        xc_set_error("import: block " + std::to_string(i) + " differs from the plan of the file's parameters");
        s = XC_EINVAL;
      }
    }
    if (s == XC_OK && (h->tail != hd.tail || h->zeta != hd.zeta)) {
      xc_set_error("import: the plan's tail or zeta differs from the file's");
      s = XC_EINVAL;
    }
  }
  if (s != XC_OK) {
    destroy_impl(h);
    delete h;
    return s;
  }
  *out = h;
  return XC_OK;
}

// ---- distributed precompute: node range per rank + two all-gathers ----------
namespace {

// Every rank's part of an exchange starts with this header; after the caller's all-gather the
// slot of rank r must carry rank r's header of the current stage (else XC_ENCCL: the all-gather
// was incomplete, out of rank order, or mixed stages).
struct ExHdr {
  uint32_t magic, stage, rank, nranks;
};
constexpr uint32_t kExMagic = 0x58434558u;  // "XCEX"
constexpr size_t kExHdr = sizeof(ExHdr);     // 16 bytes: keeps the double2 payload aligned

xc_status put_exchange(xc_op* h, const void* payload, size_t bytes, bool device_payload) {
  ExHdr hd{kExMagic, (uint32_t)h->xstage_next, (uint32_t)h->rank, (uint32_t)h->nranks};
  XC_TRY(dev_alloc(h->xsend, kExHdr + bytes));
  XC_TRY(dev_alloc(h->xrecv, (kExHdr + bytes) * h->nranks));
  XC_CUDA(cudaMemset(h->xsend.p, 0, kExHdr + bytes));
  XC_CUDA(cudaMemcpy(h->xsend.p, &hd, kExHdr, cudaMemcpyHostToDevice));
  if (bytes && payload)
    XC_CUDA(cudaMemcpy((char*)h->xsend.p + kExHdr, payload, bytes,
                       device_payload ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  return XC_OK;
}

// Check the headers of the completed exchange (per = one rank's slot in bytes).
xc_status check_exchange(xc_op* h, size_t per) {
  for (int r = 0; r < h->nranks; ++r) {
    ExHdr hd{};
    XC_CUDA(cudaMemcpy(&hd, (const char*)h->xrecv.p + (size_t)r * per, kExHdr, cudaMemcpyDeviceToHost));
    if (hd.magic != kExMagic || hd.stage != (uint32_t)h->xstage || hd.rank != (uint32_t)r ||
        hd.nranks != (uint32_t)h->nranks) {
      xc_set_error("exchange " + std::to_string(h->xstage) + ": slot " + std::to_string(r) + " holds rank " +
                   std::to_string(hd.rank) + " of stage " + std::to_string(hd.stage) +
                   " (the all-gather is incomplete or out of rank order)");
      return XC_ENCCL;
    }
  }
  return XC_OK;
}

// Exchange 0 (thresh_mode = 1): this rank's max |S|^2 per block (the global threshold's reference,
// an all-reduce(max) done as an all-gather + max, so one exchange primitive serves all).
xc_status stage_exchange0(xc_op* h) {
  std::vector<double> mx;
  for (auto& b : h->blocks) mx.push_back(b.gmax2);
  h->xstage_next = 3;
  return put_exchange(h, mx.data(), mx.size() * sizeof(double), false);
}

xc_status stage_maxima(xc_op* h) {
  const int nb = (int)h->blocks.size();
  const size_t per = kExHdr + (size_t)nb * sizeof(double);
  XC_TRY(check_exchange(h, per));
  std::vector<char> all(per * h->nranks);
  XC_CUDA(cudaMemcpy(all.data(), h->xrecv.p, all.size(), cudaMemcpyDeviceToHost));
  for (int i = 0; i < nb; ++i) {
    double m = 0.0;
    for (int r = 0; r < h->nranks; ++r) {
      double v;
      memcpy(&v, all.data() + (size_t)r * per + kExHdr + (size_t)i * sizeof(double), sizeof(double));
      m = std::max(m, v);
    }
    h->blocks[i].gmax2 = m;
  }
  return XC_OK;
}

// Exchange 1: per block, the (start, len) of this rank's nodes, padded to npr nodes.
xc_status stage_exchange1(xc_op* h) {
  const int nb = (int)h->blocks.size();
  const int n0 = h->rank * h->npr, n1 = std::min<int>((int)h->N, n0 + h->npr);
  std::vector<int> buf((size_t)nb * 2 * h->npr, 0);
  for (int i = 0; i < nb; ++i) {
    BlockData& b = h->blocks[i];
    for (int k = n0; k < n1; ++k) {
      buf[((size_t)i * 2 + 0) * h->npr + (k - n0)] = b.h_start[k];
      buf[((size_t)i * 2 + 1) * h->npr + (k - n0)] = b.h_len[k];
    }
  }
  h->xstage_next = 1;
  return put_exchange(h, buf.data(), buf.size() * sizeof(int), false);
}

// After exchange 1: every node's band; exchange 2 carries each rank's values per block,
// padded to the largest rank's count.
xc_status stage_exchange2(xc_op* h) {
  const int nb = (int)h->blocks.size();
  const int N = (int)h->N;
  const size_t per1 = kExHdr + (size_t)nb * 2 * h->npr * sizeof(int);
  XC_TRY(check_exchange(h, per1));
  std::vector<char> raw(per1 * h->nranks);
  XC_CUDA(cudaMemcpy(raw.data(), h->xrecv.p, raw.size(), cudaMemcpyDeviceToHost));
  h->xmaxc.assign(nb, 1);
  for (int i = 0; i < nb; ++i) {
    BlockData& b = h->blocks[i];
    for (int r = 0; r < h->nranks; ++r) {
      const int* slot = reinterpret_cast<const int*>(raw.data() + (size_t)r * per1 + kExHdr);
      const int* st = slot + ((size_t)i * 2 + 0) * h->npr;
      const int* ln = slot + ((size_t)i * 2 + 1) * h->npr;
      int64_t cnt = 0;
      for (int j = 0; j < h->npr && r * h->npr + j < N; ++j) {
        b.h_start[r * h->npr + j] = st[j];
        b.h_len[r * h->npr + j] = ln[j];
        cnt += ln[j];
      }
      h->xmaxc[i] = std::max<int64_t>(h->xmaxc[i], cnt);
    }
  }
  size_t per = 0;
  for (int i = 0; i < nb; ++i) per += (size_t)h->xmaxc[i] * sizeof(double2);
  h->xstage_next = 2;
  XC_TRY(put_exchange(h, nullptr, per, true));
  size_t off = kExHdr;
  for (int i = 0; i < nb; ++i) {
    BlockData& b = h->blocks[i];
    if (b.loc_count > 0)
      XC_CUDA(cudaMemcpy((char*)h->xsend.p + off, b.vals.p, b.loc_count * sizeof(double2), cudaMemcpyDeviceToDevice));
    off += (size_t)h->xmaxc[i] * sizeof(double2);
  }
  return XC_OK;
}

// After exchange 2: the full value arrays, then the rest of the build.
xc_status stage_finish(xc_op* h) {
  const int nb = (int)h->blocks.size();
  const int N = (int)h->N;
  size_t per = kExHdr;
  for (int i = 0; i < nb; ++i) per += (size_t)h->xmaxc[i] * sizeof(double2);
  XC_TRY(check_exchange(h, per));
  size_t boff = kExHdr;
  for (int i = 0; i < nb; ++i) {
    BlockData& b = h->blocks[i];
    int64_t total = 0;
    for (int k = 0; k < N; ++k) total += b.h_len[k];
    XC_TRY(dev_alloc(b.vals, (size_t)std::max<int64_t>(1, total) * sizeof(double2)));
    int64_t pos = 0;
    for (int r = 0; r < h->nranks; ++r) {
      int64_t cnt = 0;
      for (int j = 0; j < h->npr && r * h->npr + j < N; ++j) cnt += b.h_len[r * h->npr + j];
      if (cnt > 0)
        XC_CUDA(cudaMemcpy((double2*)b.vals.p + pos, (const char*)h->xrecv.p + r * per + boff,
                           cnt * sizeof(double2), cudaMemcpyDeviceToDevice));
      pos += cnt;
    }
    boff += (size_t)h->xmaxc[i] * sizeof(double2);
    XC_CUDA(cudaMemcpy(b.start.p, b.h_start.data(), N * sizeof(int), cudaMemcpyHostToDevice));
    XC_CUDA(cudaMemcpy(b.len.p, b.h_len.data(), N * sizeof(int), cudaMemcpyHostToDevice));
  }
  dev_free(h->xsend);
  dev_free(h->xrecv);
  return build_end(h);
}

void set_exchange(xc_op* h, xc_exchange_t* ex) {
  ex->send = h->xsend.p;
  ex->recv = h->xrecv.p;
  ex->bytes_per_rank = h->xsend.p ? h->xsend.bytes : 0;
}

}  // namespace

xc_status xc_build_local(xc_kind kind, const xc_params* p, const double* nodes, int64_t N, double eps, int rank,
                         int nranks, xc_handle* out, xc_exchange_t* ex) {
  if (!out || !ex || nranks < 1 || rank < 0 || rank >= nranks) {
    xc_set_error("build_local: need out, ex and 0 <= rank < nranks");
    return XC_EINVAL;
  }
  *out = nullptr;
  xc_op* h = new xc_op();
  auto fail = [&](xc_status s) {
    destroy_impl(h);
    delete h;
    return s;
  };
  if (kind == XC_LAG2D) {
    xc_set_error("build_local: XC_LAG2D has no distributed precompute");
    return fail(XC_EUNSUPPORTED);
  }
  xc_status s = build_begin(kind, p, nodes, N, eps, h);
  if (s != XC_OK) return fail(s);
  h->rank = rank;
  h->nranks = nranks;
  h->npr = (int)((N + nranks - 1) / nranks);
  const int n0 = std::min<int>((int)N, rank * h->npr), n1 = std::min<int>((int)N, n0 + h->npr);
  if (h->thresh_mode == 1) {  // global threshold: first the block maxima of every rank (exchange 0)
    if ((s = build_maxima(h, n0, n1)) != XC_OK) return fail(s);
    if ((s = stage_exchange0(h)) != XC_OK) return fail(s);
  } else {
    if ((s = build_bands(h, n0, n1)) != XC_OK) return fail(s);
    if ((s = stage_exchange1(h)) != XC_OK) return fail(s);
  }
  h->xstage = h->xstage_next;
  set_exchange(h, ex);
  *out = h;
  return XC_OK;
}

xc_status xc_build_step(xc_handle h, xc_exchange_t* ex) {
  if (!h || !ex || h->xstage < 1 || h->xstage > 3) {
    xc_set_error("build_step: handle is not in a distributed build");
    return XC_ESTATE;
  }
  XC_CUDA(cudaSetDevice(h->device));
  if (h->xstage == 3) {  // block maxima of all ranks -> global thresholds -> this rank's bands
    XC_TRY(stage_maxima(h));
    const int n0 = std::min<int>((int)h->N, h->rank * h->npr), n1 = std::min<int>((int)h->N, n0 + h->npr);
    XC_TRY(build_bands(h, n0, n1));
    XC_TRY(stage_exchange1(h));
    h->xstage = 1;
    set_exchange(h, ex);
    return XC_OK;
  }
  if (h->xstage == 1) {
    XC_TRY(stage_exchange2(h));
    h->xstage = 2;
    set_exchange(h, ex);
    return XC_OK;
  }
  XC_TRY(stage_finish(h));
  h->xstage = 0;
  set_exchange(h, ex);
  return XC_OK;
}

// Test entry point: the output-axis real-output inverse DFT engine alone (c2r_run with the plan
// a block of length L would use), W = 1: Y[p] = (F*_L u)_p (unitary) for p < L.
xc_status xc_c2r_check(int64_t L, const double* U, int64_t ldu, double* Y, int64_t ldy, int64_t B, void* stream) {
  if (L < 4 || (L & 1) || !U || !Y || B < 1 || ldu < B || ldy < B) {
    xc_set_error("c2r_check: need even L >= 4, B >= 1, ld >= B");
    return XC_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  FftPlan plan;
  XC_TRY(fft_plan_make(plan, (int)(L / 2), true));
  std::vector<double2> tw(L / 2);
  const long double PI2 = 6.283185307179586476925286766559005768L;
  for (int64_t n = 0; n < L / 2; ++n) {
    long double a = PI2 * (long double)n / (long double)L;
    tw[n] = make_double2((double)cosl(a), (double)sinl(a));
  }
  std::vector<double> ys(L, 1.0 / sqrt((double)L));
  DevBuf dtw, dys, scr;
  xc_status s = upload(dtw, tw);
  if (s == XC_OK) s = upload(dys, ys);
  if (s == XC_OK && plan.L2 > 1) s = dev_alloc(scr, (size_t)(L / 2) * B * sizeof(double2));
  if (s == XC_OK) {
    FftIO io{};
    io.Uc = reinterpret_cast<const double2*>(U);
    io.ldu = ldu;
    io.twh = (const double2*)dtw.p;
    io.M = (int)(L / 2);
    io.H = (int)(L / 2 + 1);
    io.Y = Y;
    io.ldy = ldy;
    io.yscale = (const double*)dys.p;
    io.keep_lo = 0;
    io.keep_hi = (int)L;
    io.m_off = 0;
    s = c2r_run(plan, io, (int)B, (double2*)scr.p, st);
  }
  if (s == XC_OK && cudaStreamSynchronize(st) != cudaSuccess) {
    xc_set_error("c2r_check: kernel failed");
    s = XC_ECUDA;
  }
  dev_free(dtw);
  dev_free(dys);
  dev_free(scr);
  fft_plan_free(plan);
  return s;
}

xc_status xc_apply(xc_handle h, xc_dir dir, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t B,
                   void* stream) {
  if (!h) {
    xc_set_error("null handle");
    return XC_EINVAL;
  }
  XC_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  Ws* wp = &h->def;
  {
    std::lock_guard<std::mutex> lk(h->att_mu);
    for (Ws* a : h->att)
      if (a->bound == st) wp = a;
  }
  Ws& w = *wp;
  if (wp != &h->def && B > w.B) XC_TRY(ws_carve(h, w, B));  // the caller's memory: no allocation
  if (!h->use_graphs || h->prof || h->xstage != 0) return apply_impl(h, w, dir, X, ldx, Y, ldy, B, st);
  GraphEntry* e = nullptr;
  for (auto& g : w.graphs)
    if (g.X == X && g.Y == Y && g.ldx == ldx && g.ldy == ldy && g.B == B && g.dir == dir && g.st == st) e = &g;
  if (e && e->exec) {
    XC_CUDA(cudaGraphLaunch(e->exec, st));
    return XC_OK;
  }
  if (!e) {  // first call with these arguments: run directly (one-time kernel attributes)
    XC_TRY(apply_impl(h, w, dir, X, ldx, Y, ldy, B, st));
    if (w.graphs.size() >= 16) clear_graphs(w);
    w.graphs.push_back(GraphEntry{X, Y, ldx, ldy, B, (int)dir, st, 1, nullptr});
    return XC_OK;
  }
  // second call: capture the apply once, then replay it
  cudaStreamCaptureStatus cs;
  XC_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone || st == nullptr)  // caller is capturing, or legacy stream
    return apply_impl(h, w, dir, X, ldx, Y, ldy, B, st);
  cudaGraph_t graph = nullptr;
  XC_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  xc_status s = apply_impl(h, w, dir, X, ldx, Y, ldy, B, st);
  cudaError_t ce = cudaStreamEndCapture(st, &graph);
  if (s != XC_OK) {
    if (graph) cudaGraphDestroy(graph);
    return s;
  }
  XC_CUDA(ce);
  cudaGraphExec_t exec = nullptr;
  ce = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  XC_CUDA(ce);
  e->exec = exec;
  XC_CUDA(cudaGraphLaunch(exec, st));
  return XC_OK;
}

xc_status xc_attach_workspace(xc_handle h, void* stream, void* dptr, size_t bytes) {
  if (!h) {
    xc_set_error("null handle");
    return XC_EINVAL;
  }
  XC_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(h->att_mu);
  for (size_t i = 0; i < h->att.size(); ++i)
    if (h->att[i]->bound == st) {  // replace (or detach): the old one's work must be done
      XC_CUDA(cudaStreamSynchronize(st));
      ws_release(*h->att[i]);
      delete h->att[i];
      h->att.erase(h->att.begin() + i);
      break;
    }
  if (!dptr) return XC_OK;
  if (bytes < 256 || ((uintptr_t)dptr & 255)) {
    xc_set_error("attach_workspace: need a 256-byte aligned device range");
    return XC_EINVAL;
  }
  Ws* w = new Ws();
  w->bound = st;
  w->base = (char*)dptr;
  w->bytes = bytes;
  xc_status s = ws_streams(*w);
  if (s != XC_OK) {
    ws_release(*w);
    delete w;
    return s;
  }
  h->att.push_back(w);
  return XC_OK;
}

xc_status xc_set_graphs(xc_handle h, int enable) {
  if (!h) return XC_EINVAL;
  h->use_graphs = enable != 0;
  if (!enable) {
    clear_graphs(h->def);
    std::lock_guard<std::mutex> lk(h->att_mu);
    for (Ws* w : h->att) clear_graphs(*w);
  }
  return XC_OK;
}

// Host buffers: the batch is cut into column chunks that flow through a 3-stage pipeline
// (H2D on s_in, the apply on `stream`, D2H on s_out; two device slots), so the PCIe
// copies in both directions overlap each other and the apply.
namespace {

// Enqueue one host-buffer apply on the pipeline (no host synchronisation).  Chunk slots and
// their events carry over between calls, so consecutive calls overlap (the next call's first
// copy in runs under this call's last copy out).
xc_status host_enqueue(xc_op* h, xc_dir dir, const double* Xh, double* Yh, int64_t B, cudaStream_t st) {
  if (!h->s_in) {
    int lo = 0, hi = 0;
    XC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    XC_CUDA(cudaStreamCreateWithPriority(&h->s_in, cudaStreamNonBlocking, hi));
    XC_CUDA(cudaStreamCreateWithPriority(&h->s_out, cudaStreamNonBlocking, hi));
    for (int i = 0; i < xc_op::kSlots; ++i) {
      XC_CUDA(cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming));
      XC_CUDA(cudaEventCreateWithFlags(&h->ev_cmp[i], cudaEventDisableTiming));
      XC_CUDA(cudaEventCreateWithFlags(&h->ev_out[i], cudaEventDisableTiming));
    }
    XC_CUDA(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming));
  }
  // rows of X and Y: nodes N / degrees M by direction (planar complex: twice)
  const int64_t cf = h->kind == XC_EXP ? 2 : 1;
  const int64_t NI = cf * (dir == XC_DIR_A ? h->N : h->M), NO = cf * (dir == XC_DIR_A ? h->M : h->N);
  const int64_t N = std::max(NI, NO);
  // chunk: a multiple of 64 columns (the SpMM column tile), at least 64
  int64_t nparts = 12;  // ~B/12 columns per chunk: the measured optimum at c5 (2D DMA efficiency vs pipeline fill)
  static const int env_parts = getenv("XC_HOST_CHUNKS") ? atoi(getenv("XC_HOST_CHUNKS")) : 0;
  if (env_parts > 0) nparts = env_parts;
  int64_t Bc = std::min<int64_t>(B, std::max<int64_t>(64, ((B + nparts - 1) / nparts + 63) / 64 * 64));
  const int64_t nchunk = (B + Bc - 1) / Bc;
  const size_t slot = (size_t)N * Bc * sizeof(double);
  const int NS = xc_op::kSlots;
  // slot i sits at i * N * Bc: a call with another chunk shape (B or direction) would move the
  // slots under chunks still in flight, so a shape change drains the pipeline first (as does a
  // reallocation)
  if (h->Xh.bytes < NS * slot || Bc > h->def.B || Bc != h->hBc || N != h->hN) {
    XC_CUDA(cudaStreamSynchronize(h->s_in));
    XC_CUDA(cudaStreamSynchronize(h->s_out));
    if (h->hst_set) XC_CUDA(cudaStreamSynchronize(h->hst));
    h->hchunk = 0;
    h->hBc = Bc;
    h->hN = N;
    if (h->Xh.bytes < NS * slot) {
      XC_TRY(dev_alloc(h->Xh, NS * slot));
      XC_TRY(dev_alloc(h->Yh, NS * slot));
    }
    XC_TRY(ensure_ws(h, Bc));
  }
  if (h->hst_set && h->hst != st) {  // the previous calls' apply stream must be done with the slots
    XC_CUDA(cudaEventRecord(h->ev_start, h->hst));
    XC_CUDA(cudaStreamWaitEvent(st, h->ev_start, 0));
  }
  h->hst = st;
  h->hst_set = true;
  // the copy streams start after the work already queued on `stream`
  XC_CUDA(cudaEventRecord(h->ev_start, st));
  XC_CUDA(cudaStreamWaitEvent(h->s_in, h->ev_start, 0));
  XC_CUDA(cudaStreamWaitEvent(h->s_out, h->ev_start, 0));
  for (int64_t c = 0; c < nchunk; ++c, ++h->hchunk) {
    const int i = (int)(h->hchunk % NS);
    const bool reused = h->hchunk >= NS;
    const int64_t c0 = c * Bc, bc = std::min(Bc, B - c0);
    double* xs = (double*)h->Xh.p + (size_t)i * N * Bc;
    double* ys = (double*)h->Yh.p + (size_t)i * N * Bc;
    if (reused) XC_CUDA(cudaStreamWaitEvent(h->s_in, h->ev_cmp[i], 0));  // slot's X consumed
    XC_CUDA(cudaMemcpy2DAsync(xs, bc * sizeof(double), Xh + c0, B * sizeof(double), bc * sizeof(double), NI,
                              cudaMemcpyHostToDevice, h->s_in));
    XC_CUDA(cudaEventRecord(h->ev_in[i], h->s_in));
    XC_CUDA(cudaStreamWaitEvent(st, h->ev_in[i], 0));
    if (reused) XC_CUDA(cudaStreamWaitEvent(st, h->ev_out[i], 0));     // slot's Y copied out
    XC_TRY(apply_impl(h, h->def, dir, xs, bc, ys, bc, bc, st));
    XC_CUDA(cudaEventRecord(h->ev_cmp[i], st));
    XC_CUDA(cudaStreamWaitEvent(h->s_out, h->ev_cmp[i], 0));
    XC_CUDA(cudaMemcpy2DAsync(Yh + c0, B * sizeof(double), ys, bc * sizeof(double), bc * sizeof(double), NO,
                              cudaMemcpyDeviceToHost, h->s_out));
    XC_CUDA(cudaEventRecord(h->ev_out[i], h->s_out));
  }
  return XC_OK;
}

xc_status host_sync(xc_op* h) {
  if (h->s_out) XC_CUDA(cudaStreamSynchronize(h->s_out));
  if (h->s_in) XC_CUDA(cudaStreamSynchronize(h->s_in));
  if (h->hst_set) XC_CUDA(cudaStreamSynchronize(h->hst));
  return XC_OK;
}

}  // namespace

// Host buffers: the batch is cut into column chunks that flow through a 3-stage pipeline
// (H2D on s_in, the apply on `stream`, D2H on s_out; two device slots), so the PCIe
// copies in both directions overlap each other and the apply.
xc_status xc_apply_host(xc_handle h, xc_dir dir, const double* Xh, double* Yh, int64_t B, void* stream) {
  if (!h || !Xh || !Yh || B < 1) {
    xc_set_error("apply_host: bad arguments");
    return XC_EINVAL;
  }
  XC_CUDA(cudaSetDevice(h->device));
  XC_TRY(host_enqueue(h, dir, Xh, Yh, B, (cudaStream_t)stream));
  return host_sync(h);
}

xc_status xc_apply_host_async(xc_handle h, xc_dir dir, const double* Xh, double* Yh, int64_t B, void* stream) {
  if (!h || !Xh || !Yh || B < 1) {
    xc_set_error("apply_host_async: bad arguments");
    return XC_EINVAL;
  }
  XC_CUDA(cudaSetDevice(h->device));
  return host_enqueue(h, dir, Xh, Yh, B, (cudaStream_t)stream);
}

xc_status xc_host_wait(xc_handle h) {
  if (!h) return XC_EINVAL;
  XC_CUDA(cudaSetDevice(h->device));
  return host_sync(h);
}

xc_status xc_reserve(xc_handle h, int64_t B) {
  if (!h || B < 1) return XC_EINVAL;
  XC_CUDA(cudaSetDevice(h->device));
  return ensure_ws(h, B);
}

xc_status xc_debug_guards(xc_handle h, int64_t* bad, int64_t* checked) {
  if (!h || !bad) return XC_EINVAL;
  XC_CUDA(cudaSetDevice(h->device));
  XC_CUDA(cudaDeviceSynchronize());
  int64_t nb = 0, nc = 0;
  std::vector<unsigned char> buf;
  std::lock_guard<std::mutex> lk(h->att_mu);
  std::vector<Ws*> all{&h->def};
  for (Ws* w : h->att) all.push_back(w);
  for (Ws* w : all)
    for (auto& g : w->guards) {
      buf.resize(g.second);
      XC_CUDA(cudaMemcpy(buf.data(), w->base + g.first, g.second, cudaMemcpyDeviceToHost));
      for (unsigned char c : buf) nb += c != 0x7F;
      nc += (int64_t)g.second;
    }
  *bad = nb;
  if (checked) *checked = nc;
  return XC_OK;
}

xc_status xc_launches(xc_handle h, xc_dir dir, int64_t B, int64_t* n) {
  if (!h || !n || B < 1) return XC_EINVAL;
  *n = count_launches(h, dir, B);
  return XC_OK;
}

xc_status xc_workspace_query(xc_handle h, int64_t B, size_t* bytes) {
  if (!h || !bytes || B < 1) return XC_EINVAL;
  *bytes = ws_layout(h, B, nullptr, nullptr);
  return XC_OK;
}

xc_status xc_info(xc_handle h, xc_info_t* out) {
  if (!h || !out) return XC_EINVAL;
  *out = h->info;
  return XC_OK;
}

xc_status xc_block_info(xc_handle h, int i, xc_block_info_t* out) {
  if (!h || !out || i < 0 || i >= (int)h->blocks.size()) {
    xc_set_error("block_info: bad block index");
    return XC_EINVAL;
  }
  const BlockData& b = h->blocks[i];
  out->L = b.L;
  out->H = b.H;
  out->m_off = b.m_off;
  out->keep_lo = b.keep_lo;
  out->keep_hi = b.keep_hi;
  out->nnz = b.nnz;
  out->max_band = b.max_band;
  out->q_taps = b.appQ >= 0 ? 2 * b.appQ + 1 : 0;
  return XC_OK;
}

xc_status xc_block_window(xc_handle h, int i, double* w) {
  if (!h || !w || i < 0 || i >= (int)h->blocks.size()) return XC_EINVAL;
  memcpy(w, h->blocks[i].h_w.data(), h->blocks[i].h_w.size() * sizeof(double));
  return XC_OK;
}

xc_status xc_node_spectrum(xc_handle h, int i, int64_t k, double* re, double* im) {
  if (!h || !re || !im || i < 0 || i >= (int)h->blocks.size() || k < 0 || k >= h->N || h->ukind == XC_LAG2D) {
    xc_set_error("node_spectrum: bad arguments");
    return XC_EINVAL;
  }
  const BlockData& b = h->blocks[i];
  for (int q = 0; q < b.H; ++q) re[q] = im[q] = 0.0;
  int n = b.h_len[k];
  if (n == 0) return XC_OK;
  std::vector<double2> v(n);
  XC_CUDA(cudaSetDevice(h->device));
  XC_CUDA(cudaMemcpy(v.data(), (double2*)b.vals.p + b.h_off[k], n * sizeof(double2), cudaMemcpyDeviceToHost));
  for (int j = 0; j < n; ++j) {
    const int q = (b.h_start[k] + j) % b.H;  // runs of complex rows may wrap (XC_EXP)
    re[q] = v[j].x;
    im[q] = v[j].y;
  }
  return XC_OK;
}

xc_status xc_gauss_rule(xc_kind kind, double alpha, double beta, int64_t N, double* nodes, double* weights,
                        double* wt, int device) {
  if (!nodes) return XC_EINVAL;
  std::vector<double> w(N), t(N);
  xc_status s = gauss_rule_device(kind, alpha, beta, N, nodes, w.data(), t.data(), device);
  if (s != XC_OK) return s;
  if (weights) memcpy(weights, w.data(), N * sizeof(double));
  if (wt) memcpy(wt, t.data(), N * sizeof(double));
  return XC_OK;
}

xc_status xc_profile_enable(xc_handle h, int enable) {
  if (!h) return XC_EINVAL;
  XC_CUDA(cudaSetDevice(h->device));
  if (enable && h->ev.empty()) {
    h->ev.resize(4 * xc_op::kRing);
    h->ev_dir.assign(xc_op::kRing, 0);
    for (auto& e : h->ev) XC_CUDA(cudaEventCreate(&e));
  }
  h->prof = enable != 0;
  return XC_OK;
}

xc_status xc_profile_read(xc_handle h, double* ms_spmm, double* ms_fft, double* ms_reduce, double* ms_total,
                          int64_t* n) {
  if (!h) return XC_EINVAL;
  XC_CUDA(cudaSetDevice(h->device));
  for (int slot = 0; slot < (int)h->ev_dir.size(); ++slot) XC_TRY(prof_harvest(h, slot));
  if (ms_spmm) *ms_spmm = h->ms_spmm;
  if (ms_fft) *ms_fft = h->ms_fft;
  if (ms_reduce) *ms_reduce = h->ms_red;
  if (ms_total) *ms_total = h->ms_tot;
  if (n) *n = h->n_prof;
  h->ms_spmm = h->ms_fft = h->ms_red = h->ms_tot = 0;
  h->n_prof = 0;
  return XC_OK;
}

xc_status xc_plan_chain(xc_kind kind, int64_t N, double eps1, double eps2, int cutoff, double* zeta, int* nb,
                        int* L, int* m_off, int* keep_lo, int* keep_hi, int max_blocks, int* tail) {
  if (!zeta || !nb || !L || !m_off || !keep_lo || !keep_hi || !tail || N < 2 || !(eps1 > 0 && eps1 < 1)) {
    xc_set_error("plan_chain: bad arguments");
    return XC_EINVAL;
  }
  if (eps2 <= 0) eps2 = 1e-2;
  if (!(eps1 < eps2 && eps2 < 1)) {
    xc_set_error("plan_chain: need eps1 < eps2 < 1");
    return XC_EINVAL;
  }
  PlanOut p;
  XC_TRY(make_chain(kind, N, eps1, eps2, cutoff > 0 ? cutoff : 32, p));
  if ((int)p.blocks.size() > max_blocks) {
    xc_set_error("plan_chain: too many blocks for the output arrays");
    return XC_EINVAL;
  }
  *zeta = p.zeta;
  *nb = (int)p.blocks.size();
  *tail = p.tail;
  for (size_t i = 0; i < p.blocks.size(); ++i) {
    L[i] = p.blocks[i].L;
    m_off[i] = p.blocks[i].m_off;
    keep_lo[i] = p.blocks[i].keep_lo;
    keep_hi[i] = p.blocks[i].keep_hi;
  }
  return XC_OK;
}

void xc_destroy(xc_handle h) {
  if (!h) return;
  cudaSetDevice(h->device);
  destroy_impl(h);
  delete h;
}

const char* xc_last_error(void) { return g_err.c_str(); }

const char* xc_version(void) { return "xc-b200 0.1 (sm_100a, fp64 DMMA)"; }

}  // extern "C"
