/*
 * xc.h -- C ABI of the B200-native extra-component transform library (libxc.so).
 *
 * Method: A. V. Terekhov, "An extra-component method for evaluating fast
 * matrix-vector multiplication with special functions", arXiv 2004.11610.
 * Citations "P:<n>" refer to lines of the paper's text; readings
 * "R-<n>" are listed in DESIGN.md.
 *
 * Operator convention (R-1): A[j,k] = phi_j(x_k); row j = degree / frequency,
 * column k = node.  All arithmetic is fp64.  Matrices X, Y are row-major with
 * the right-hand-side (RHS) index fastest: element (row r, rhs b) at r*ld + b.
 *
 * Ownership: the handle owns the compressed operator, its plans, twiddle
 * tables and an internal workspace; the caller owns X, Y and the nodes.
 * Nodes and weights are copied at build time.
 *
 * Errors: every call returns an xc_status; xc_last_error() returns a
 * thread-local message for the last failing call on the calling thread.
 * CUDA errors are reported as XC_ECUDA (the library never aborts).
 */
#ifndef XC_H_
#define XC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct xc_op* xc_handle;

typedef enum {
  XC_OK = 0,
  XC_EINVAL = 1,        /* bad argument: N < 2, B < 1, ld < B, non-finite / unsorted /
                           out-of-domain nodes, eps outside (0,1), eps1 >= eps2      */
  XC_ENUMERIC = 2,      /* zeta Newton did not converge, s search did not terminate  */
  XC_ESTATE = 3,        /* direction applied that was not built                       */
  XC_ENOMEM = 4,        /* device allocation failed                                   */
  XC_ECUDA = 5,         /* CUDA runtime error                                         */
  XC_EUNSUPPORTED = 6,  /* size beyond the FFT engine's range (L > 1024^2, ...)       */
  XC_ENCCL = 7          /* distributed precompute: the caller's all-gather (NCCL) did not
                           deliver every rank's part of the exchange in rank order      */
} xc_status;

typedef enum {
  XC_COS = 1,       /* A[j,k] = cos(pi j t_k), nodes t_k in [0,1] (P:66-70 with theta = pi t;
                       non-block Algorithm 2/1 with extra components on both sides) */
  XC_JACOBI = 2,    /* A[j,k] = p_j^(alpha,beta)(x_k), orthonormal on [-1,1]; Legendre = (0,0)
                       (chi read as the squared norm, R-4; block form P:280-301)     */
  XC_LAGUERRE = 3,  /* A[j,k] = l_j(x_k) = exp(-x_k/2) L_j(x_k), x_k >= 0 (block form) */
  XC_EXP = 4,       /* A[j,k] = exp(i pi j t_k), nodes t_k in [0,2): the non-uniform DFT, complex
                       (the exp row of Appendix A).  Both directions
                       (XC_DIR_WAT: Y = diag(wts) A^T X, no conjugate).  X and Y
                       are complex in planar form: 2N rows, real parts in rows [0,N), imaginary
                       parts in rows [N,2N), same ld; the full spectrum of L bins is kept.
                       May be rectangular: p->n_rows = M degrees (rows) != N nodes; then
                       XC_DIR_A maps 2N planar rows to 2M, XC_DIR_WAT 2M to 2N.                  */
  XC_LAGSPEC = 5,   /* the spectral Laguerre forward V = C^T F (Fig. lag_row):
                       A[m,j] = (-eta/2 - i k_j)^m / (eta/2 - i k_j)^(m+1), m < M = p->n_rows
                       (0 => N), nodes = frequencies k_j (finite, strictly ascending, any sign),
                       eta = p->eta > 0.  Computed as XC_EXP at t_j = 1 + (2/pi) atan(2 k_j/eta)
                       with the per-node scale 1/(eta/2 - i k_j) folded into the operator (R-21);
                       complex planar X / Y as XC_EXP, both directions.                          */
  XC_LAG2D = 6      /* the time-domain Laguerre sum Y = D X, D[i,j] = l_j(x_i) = exp(-x_i/2) L_j(x_i),
                       i, j < N, on an EQUISPACED grid x_i >= 0 (nodes ascending, spacing equal to
                       1e-9 relative), by the 2D block method (R-23): the
                       block chain on both axes, D2 = F W D W F per block pair.  XC_DIR_A only
                       (output indexed by node); eps2 defaults to 0.1 for this kind.             */
} xc_kind;

typedef enum {
  XC_DIR_A = 1,     /* Y = A X: output indexed by degree (Algorithm 2 / block form) */
  XC_DIR_WAT = 2    /* Y = diag(wt) A^T X: input indexed by degree (Algorithm 1 / block form,
                       P:188-204); wt are the weights passed at build time          */
} xc_dir;

typedef struct {
  double alpha, beta;      /* XC_JACOBI parameters (> -1)                                    */
  double eps1, eps2;       /* 0 => eps1 = eps (threshold), eps2 = 1e-2 (extra components, R-2) */
  int dense_cutoff;        /* 0 => 32: degrees [0, t) with t <= cutoff done densely  */
  int dirs;                /* bitmask of xc_dir layouts to build; 0 => XC_DIR_A only          */
  const double* weights;   /* host, length N; required iff dirs & XC_DIR_WAT (copied)        */
  int device;              /* CUDA device ordinal                                            */
  void* stream;            /* cudaStream_t for the build (NULL = default stream)             */
  int node_chunk;          /* 0 => auto: nodes per precompute chunk (device memory bound)    */
  double eta;              /* XC_LAGSPEC: Laguerre scale eta > 0                      */
  int64_t n_rows;          /* XC_EXP / XC_LAGSPEC: degrees M (rows of A); 0 => N (square)     */
  int trig_precompute;     /* trig kinds (XC_COS, XC_EXP, XC_LAGSPEC): 0 = entries + FFT per node;
                              1 = Appendix A (R-22): closed-form row spectra convolved
                              with the 2Q+1 leading window coefficients, only the bins around each
                              node's peak evaluated; the truncated window W' is then the method's
                              window (xc_block_window returns it).  XC_EINVAL for other kinds.  */
  int thresh_mode;         /* 0: per-node relative threshold |S| >= eps1 max_q |S[k,q]| (P:106,
                              R-3; default); 1: the global threshold of Alg. 1/2 step 1.3,
                              |S| >= eps1 max over the block's whole compressed matrix:
                              two passes over the nodes (and one more exchange, of the block
                              maxima, in a distributed build).  XC_LAG2D is always global (R-23);
                              XC_EUNSUPPORTED with trig_precompute = 1.                       */
  int apply_path;          /* XC_DIR_A of the real kinds: 0 = auto (the small-operator path when
                              every block has L/2 <= 4096 in at most 8 blocks and the operator has
                              <= 4M entries -- c1, c2 -- else tiled); 1 = tiled (tensor-core SpMM
                              over node windows + C2R passes); 2 = the small-operator path (two
                              launches: a bin-major gather for every u_i and the tail, then every
                              block's C2R in shared memory; XC_EUNSUPPORTED if not eligible).
                              The choice depends on the operator only, never on B.            */
} xc_params;

typedef struct {
  int64_t N;               /* transform size (degrees = nodes = N)                            */
  int kind;
  double zeta, eps1, eps2; /* Kaiser shape zeta(eps1) and thresholds                  */
  int n_blocks;            /* number of compressed blocks (1 for XC_COS)                      */
  int tail;                /* dense degrees [0, tail)                                         */
  int dirs;                /* layouts built                                                   */
  int64_t nnz;             /* kept complex entries over all blocks (half spectrum)            */
  int64_t op_bytes_A;      /* device bytes of the XC_DIR_A apply operator (tiles + metadata)  */
  int64_t op_bytes_WAT;    /* device bytes of the XC_DIR_WAT apply operator                   */
  double flops_per_col_A;  /* algorithmic fp64 flops per RHS column, XC_DIR_A   */
  double flops_per_col_WAT;
  double dmma_flops_per_col_A;   /* flops the tensor-core (DMMA) tiles actually issue         */
  double dmma_flops_per_col_WAT;
  int launches_A;          /* kernel launches per xc_apply(XC_DIR_A)                         */
  int launches_WAT;        /* kernel launches per xc_apply(XC_DIR_WAT)                       */
  int64_t M;               /* degrees (rows of A): N unless rectangular (complex kinds)       */
  double alg_bytes_per_col;  /* algorithmic HBM bytes per RHS column of an apply:
                                X read + Y written (16 N, planar complex twice)                 */
  double alg_bytes_fixed;    /* ... and per apply: the operator once (20 B per kept entry:
                                complex value + index) and the dense tail (8 t N)               */
} xc_info_t;

typedef struct {
  int L;            /* FFT length of the block (even, 2-3-5-smooth, R-9)                      */
  int H;            /* half-spectrum bins L/2 + 1                                     */
  int m_off;        /* position p carries degree p + m_off                                    */
  int keep_lo;      /* kept positions [keep_lo, keep_hi) (Fe2/Fe3)      */
  int keep_hi;
  int64_t nnz;      /* kept complex entries                                                   */
  int max_band;     /* widest kept run of any node (bins)                                     */
  int q_taps;       /* Appendix A precompute: window coefficients 2Q+1 (0: direct precompute) */
} xc_block_info_t;

/* Fill *p with defaults (all zero / NULL; device 0). */
xc_status xc_params_default(xc_params* p);

/* Precomputation stage (Alg. 1/2 step 1; block chain P:280-301):
 * plans zeta/s/L_i on the host, then generates the special-function entries in
 * double-double on the GPU, windows them, FFTs along the degree axis, thresholds
 * per node (|S| >= eps1 * max_q |S[k,q]|, R-3) and builds the tensor-core tiles.
 * nodes: host, length N, strictly ascending, finite, in the kind's domain.
 * eps: accuracy parameter in (0,1); used as eps1 unless p->eps1 > 0.
 * On success *out owns all device memory; destroy with xc_destroy. */
xc_status xc_build_compressed(xc_kind kind, const xc_params* p, const double* nodes, int64_t N,
                              double eps, xc_handle* out);

/* The computation stage on node bands given by the caller instead of the GPU precompute (p2-p4):
 * the plan (zeta, chain, windows) is this library's for (kind, p, nodes, N, eps) -- query it with
 * xc_plan_chain -- and for block i node k keeps bins [start[i][k], start[i][k] + len[i][k]) of the
 * block's spectrum (real rows: half spectrum, start + len <= L/2 + 1; XC_EXP / XC_LAGSPEC: all L
 * bins, the run taken mod L), values vals[i] = (re, im) pairs, the runs of all nodes concatenated
 * in node order (len[i][k] pairs per node; zeros allowed).  Host pointers, copied.  The tests use
 * it to apply the oracle's own operator (same kept entries).  XC_EUNSUPPORTED for
 * XC_LAG2D and trig_precompute = 1; XC_EINVAL for runs out of range. */
xc_status xc_build_from_bands(xc_kind kind, const xc_params* p, const double* nodes, int64_t N, double eps,
                              const int* const* start, const int* const* len, const double* const* vals,
                              xc_handle* out);

/* Operator persistence (checkpoint / resume of the precompute, which costs "several orders of
 * magnitude" more than an apply).  xc_export writes the handle's compressed operator to
 * `path`: a versioned little-endian file -- header (magic "XCOPER01", kind, thresh_mode,
 * trig_precompute, dense_cutoff, dirs, block count, tail, N, M, alpha, beta, eta, eps1, eps2,
 * zeta), the caller's nodes (and weights if XC_DIR_WAT was built), then per block (L, m_off,
 * keep_lo, keep_hi, nnz), its window (L doubles), the node bands start[N], len[N] (int32) and the
 * kept values (nnz complex, run-contiguous in node order: the layout of xc_build_from_bands).
 * xc_import rebuilds the operator from such a file: the plan is recomputed from the file's
 * parameters and must reproduce its chain, windows and counts (else XC_EINVAL); the kept values
 * are the file's, so applies are bit-identical to the exporting handle's.  Only device, stream
 * and node_chunk are taken from p (may be NULL).  Errors: XC_EINVAL (I/O, not an operator file,
 * truncated, plan mismatch), XC_EUNSUPPORTED (export of XC_LAG2D), XC_ESTATE (export during a
 * distributed build), XC_ECUDA / XC_ENOMEM. */
xc_status xc_export(xc_handle h, const char* path);
xc_status xc_import(const char* path, const xc_params* p, xc_handle* out);

/* Distributed precompute (the node range of the operator is split over ranks).
 * Each exchange: the caller copies `send` (bytes_per_rank device bytes) of every rank into
 * `recv` in rank order (recv + r * bytes_per_rank), e.g. one NCCL all-gather.
 * xc_build_local: phase 1 and the node bands (entries, FFT, threshold; p2-p4) of nodes
 *   [rank * ceil(N/nranks), (rank + 1) * ceil(N/nranks)) only; *ex describes the first exchange
 *   (every node's band start and length; with thresh_mode = 1 first the block maxima of this
 *   rank's nodes, the reference of the global threshold).  Same arguments as xc_build_compressed.
 * xc_build_step: consumes the completed exchange; sets *ex to the next one (the bands after the
 *   maxima, the kept values, padded to the largest rank's count, after the bands) or, after the
 *   last, finishes the build (tiles of the whole operator, identical to xc_build_compressed's)
 *   and sets ex->bytes_per_rank = 0.
 * Every rank's part starts with a 16-byte header (magic, stage, rank, nranks) that
 * xc_build_step checks in every slot of `recv`.
 * The buffers in *ex are owned by the handle and valid until the next call on it.
 * Errors: XC_EINVAL (bad rank / nranks, as xc_build_compressed), XC_ESTATE (step outside a
 * distributed build), XC_ENCCL (a slot of `recv` does not hold that rank's part of this
 * exchange: the all-gather failed or ordered the ranks differently).  The handle is unusable for
 * xc_apply until the build has finished. */
typedef struct {
  void* send;             /* device, bytes_per_rank bytes                                   */
  void* recv;             /* device, nranks * bytes_per_rank bytes, rank-major              */
  size_t bytes_per_rank;  /* 0: no exchange pending (build finished)                        */
} xc_exchange_t;

xc_status xc_build_local(xc_kind kind, const xc_params* p, const double* nodes, int64_t N, double eps,
                         int rank, int nranks, xc_handle* out, xc_exchange_t* ex);
xc_status xc_build_step(xc_handle h, xc_exchange_t* ex);

/* Computation stage (Alg. 2 step 2 / Alg. 1 step 2 per block):
 * X, Y: DEVICE pointers, row-major N x B with leading dimensions ldx, ldy >= B.
 * Enqueues on `stream` only: no host synchronisation and no allocation.  The workspace is the
 * one attached to `stream` (xc_attach_workspace) or else the handle's own, reserved beforehand
 * with xc_reserve(h, >= B) -- XC_ESTATE if B exceeds it, XC_ENOMEM if an attached workspace is
 * shorter than xc_workspace_query(h, B).  Reentrant across streams that have distinct workspaces
 * (one attached per stream; concurrent calls from several host threads are allowed then); calls
 * sharing one workspace must be ordered on one stream.  The handle's operator is read-only here. */
xc_status xc_apply(xc_handle h, xc_dir dir, const double* X, int64_t ldx, double* Y, int64_t ldy,
                   int64_t B, void* stream);

/* Bind a caller-owned DEVICE workspace [dptr, dptr + bytes) (256-byte aligned) to `stream`:
 * xc_apply on that stream uses it instead of the handle's own (size it with xc_workspace_query;
 * the caller keeps ownership and must not free it before detaching).  dptr = NULL detaches the
 * stream's workspace; attaching to a stream that has one replaces it.  Both wait for the work
 * queued on `stream`.  Creates the workspace's forked block streams (no device allocation).
 * Errors: XC_EINVAL (null handle, misaligned or tiny range). */
xc_status xc_attach_workspace(xc_handle h, void* stream, void* dptr, size_t bytes);

/* CUDA graphs of xc_apply (default on): the second call with the same (X, Y, ldx, ldy, B,
 * dir, stream) captures the apply's launches into a graph, later calls replay it with one
 * launch.  Not used while profiling, on the legacy default stream, or when the caller is itself
 * capturing.  Graphs are dropped when the workspace grows.  enable = 0 turns them off. */
xc_status xc_set_graphs(xc_handle h, int enable);

/* Test entry point: the computation stage's real-output inverse DFT engine alone, for the
 * block length L (even) with the window switched off: Y[p] = (F*_L u)_p, p < L (unitary, P:24,
 * real case P:444).  U: DEVICE, L/2 + 1 complex rows x B (interleaved re, im per column; row
 * pitch ldu complex), the half spectrum u_0..u_{L/2}; Y: DEVICE, L x B, ld ldy.  Synchronises
 * `stream`.  XC_EINVAL for odd L, L < 4, B < 1 or ld < B. */
xc_status xc_c2r_check(int64_t L, const double* U, int64_t ldu, double* Y, int64_t ldy, int64_t B, void* stream);

/* Same as xc_apply with HOST buffers X_host, Y_host (row-major N x B, ld = B):
 * copies X to the device, applies, copies Y back, and synchronises `stream`.
 * The batch is processed in column chunks (about B/16 columns, a multiple of 64) through a
 * pipeline: host-to-device copy, apply, device-to-host copy on three streams, so both copy
 * directions and the apply overlap.  Work already queued on `stream` is ordered before it.
 * Host buffers should be pinned for full bandwidth and must not overlap. */
xc_status xc_apply_host(xc_handle h, xc_dir dir, const double* X_host, double* Y_host, int64_t B,
                        void* stream);

/* Streaming form of xc_apply_host: enqueues the same pipeline and returns without waiting; the
 * pipeline state carries over, so back-to-back calls overlap (a call's first copy in runs under
 * the previous call's last copy out).  X_host must stay unchanged and Y_host unread until
 * xc_host_wait(h) (which waits for every enqueued call).  Errors as xc_apply_host. */
xc_status xc_apply_host_async(xc_handle h, xc_dir dir, const double* X_host, double* Y_host, int64_t B,
                              void* stream);
xc_status xc_host_wait(xc_handle h);

/* Reserve the handle's own workspace for up to B right-hand sides (allocates if B exceeds the
 * reserve so far; the host-buffer calls reserve their chunk width themselves). */
xc_status xc_reserve(xc_handle h, int64_t B);

/* Kernel launches one xc_apply(dir) of B columns makes (xc_info's launches_* are for B = 1;
 * the two-pass inverse DFTs run in column chunks, so the count grows with B). */
xc_status xc_launches(xc_handle h, xc_dir dir, int64_t B, int64_t* n);

/* Debug aid (the GPU pool's compute-sanitizer is closed): with the environment variable
 * XC_WS_GUARD=1 set before the first call, every workspace part is followed by a 64 KB guard zone
 * filled with 0x7F when it is carved; this synchronises the device and returns in *bad the number
 * of guard bytes some kernel overwrote (0: no write past a workspace part) and in *checked (may be
 * NULL) the guard bytes examined (0 when guards are off). */
xc_status xc_debug_guards(xc_handle h, int64_t* bad, int64_t* checked);

/* Bytes of workspace xc_apply needs for B right-hand sides (what xc_attach_workspace must get). */
xc_status xc_workspace_query(xc_handle h, int64_t B, size_t* bytes);

xc_status xc_info(xc_handle h, xc_info_t* out);
xc_status xc_block_info(xc_handle h, int block, xc_block_info_t* out);

/* Kaiser window of block `block` (host out, L values: w_p, p = 0..L-1, R-6). */
xc_status xc_block_window(xc_handle h, int block, double* w_out);

/* Kept spectrum of node k in block `block`: re/im host arrays of H values
 * (dropped entries are 0).  For parity tests against the oracle. */
xc_status xc_node_spectrum(xc_handle h, int block, int64_t k, double* re, double* im);

/* Gauss rule of the kind's orthogonality weight, computed on device `device`
 * (Sturm bisection on the Jacobi matrix + double-double Newton, Christoffel-Darboux
 * weights).  nodes, weights: host out, length N (ascending).  wt (may be NULL):
 * weights times e^{x} for XC_LAGUERRE (= 1/sum_j l_j(x)^2), else a copy of weights. */
xc_status xc_gauss_rule(xc_kind kind, double alpha, double beta, int64_t N, double* nodes,
                        double* weights, double* wt, int device);

/* Per-phase timing of xc_apply: when enabled, each xc_apply records CUDA events on
 * its own stream at the phase boundaries (no host synchronisation inside the call;
 * a ring of 512 event sets is recycled).  enable != 0 turns it on, 0 off. */
xc_status xc_profile_enable(xc_handle h, int enable);

/* Waits for all recorded events, returns the summed milliseconds of the SpMM launch
 * (FP64 tensor cores), of the FFT launches, of the reduction/tail launch and of the
 * whole apply, plus the number of applies recorded; then resets the sums. */
xc_status xc_profile_read(xc_handle h, double* ms_spmm, double* ms_fft, double* ms_reduce, double* ms_total,
                          int64_t* n_applies);

/* Host-only planning (no GPU needed): zeta(eps1), the block chain and
 * FFT lengths (R-2, R-8, R-9).  Arrays L, m_off, keep_lo, keep_hi have room for
 * max_blocks entries; *n_blocks receives the count, *tail the dense degrees.
 * eps2 = 0 selects 1e-2, dense_cutoff = 0 selects 32. */
xc_status xc_plan_chain(xc_kind kind, int64_t N, double eps1, double eps2, int dense_cutoff, double* zeta,
                        int* n_blocks, int* L, int* m_off, int* keep_lo, int* keep_hi, int max_blocks,
                        int* tail);

/* Release all device memory of the handle (NULL is ignored). */
void xc_destroy(xc_handle h);

/* Thread-local message of the last failing call ("" if none). */
const char* xc_last_error(void);

/* Library version string. */
const char* xc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* XC_H_ */
