// c2r.cu -- the output-axis inverse DFT of the computation stage (Alg. 2 steps 2.1-2.2,
// P:217-219; real case P:444; Fe2 discard + W^{-1}), as persistent,
// prefetching passes over the RHS batch.
//
// v = F*_L u for a real output of length L = 2M from the half spectrum u_0..u_M:
//   Z[n] = (u_n + conj u_{M-n}) + i e^{2 pi i n/L} (u_n - conj u_{M-n}),  n < M
//   z = IDFT_M(Z),  v[2k] = Re z_k,  v[2k+1] = Im z_k
// and Y[p + m_off] = v[p] * yscale[p] for the kept positions p (yscale = 1/(sqrt(L) w_p)).
// M <= 512 runs in one pass; longer M = L1 * L2 as a four-step pair of passes
//   pass 0: for each n2, the L1-point IDFT over n = L2 n1 + n2 (pairing fused in its first
//           radix stage), times e^{2 pi i n2 k1 / M}, to scratch row k1 L2 + n2;
//   pass 1: for each k1, the L2-point IDFT over scratch rows k1 L2 + n2, output
//           k = k1 + L1 k2 written as Y rows 2k, 2k+1 (scale, truncate).
//
// Design (sm_100a, HBM-bound): a tile is `nseq` = cb columns x sc sub-sequences of R
// points (R * nseq <= 2048, 32 KB).  Each CTA is persistent over tiles and keeps two
// buffers: LD (the tile being loaded by cp.async) and WK (the tile being transformed).
// The first radix stage reads LD (and forms Z there), so LD is free after it and the
// next tile's loads are issued immediately -- they stay in flight during the remaining
// stages and the epilogue.  Middle stages run in place in WK (read, barrier, write);
// the last stage writes global memory straight from registers (columns are the fast
// index, so every store is a contiguous run of cb * 16 or cb * 8 bytes).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "bfly.cuh"
#include "xc_internal.cuh"

namespace {

using namespace xcb;

constexpr int NTH = 256;   // threads per CTA
constexpr int TILE = 2048; // R * nseq per buffer (32 KB); 2 buffers -> 3 CTAs per SM

struct StageC {
  int r, Rr, Ns;          // radix, butterflies per sequence R/r, span Ns
  int twoff;              // offset of this stage's table w_{Ns r}^{k t}, [k][t-1], in C2RArgs::stw
  unsigned magic;         // ceil(2^32 / Ns): j / Ns by __umulhi (exact for j < 2^16)
};

// Tile geometry: sub-transform length and log2(sequences per tile).  Compile-time constants
// in the specialised kernels (all smem offsets fold to immediates), runtime in the generic one.
struct Geo {
  int R, lgn;
};

// The radix plan of a length (c2r_radices) with spans, twiddle offsets and magic numbers.
struct StagePlan {
  int nf;
  StageC st[16];
};
constexpr StagePlan stages_of(int R) {
  StagePlan p{};
  const C2RRadices rp = c2r_radices(R);
  p.nf = rp.nf;
  int Ns = 1, off = 0;
  for (int i = 0; i < rp.nf; ++i) {
    p.st[i].r = rp.f[i];
    p.st[i].Rr = R / rp.f[i];
    p.st[i].Ns = Ns;
    p.st[i].twoff = off;
    p.st[i].magic = (Ns == 1) ? 0u : (unsigned)((0x100000000ULL + Ns - 1) / Ns);
    off += Ns * (rp.f[i] - 1);
    Ns *= rp.f[i];
  }
  return p;
}

struct C2RArgs {
  int mode;              // 0: first of two, 1: second of two, 2: single pass
  int R, nf;             // sub-transform length and its radix stages
  StageC st[16];
  const double2* stw;    // per-stage twiddle tables (exact, long double on the host)
  const double2* ptw;    // pairing twiddle e^{i pi n / M}: pass 0 at [n2 L1 + e] (n = L2 e + n2), else [e]
  const double2* ftw;    // pass 0 four-step twiddle e^{2 pi i n2 k1 / M} at [n2 L1 + k1]
  int M, L1, L2;
  int S;                 // sub-sequences per column
  int P;                 // slot pairs per column (pass 0)
  int ncol, cb, lgcb, sc, lgn;
  int ntx, ntiles;
  double2* scr;          // four-step scratch, row (k1 L2 + n2), ld = lds (offsets < 2^31)
  int lds;
  int big;               // 1: 512-thread CTAs, tiles up to 2 TILE points
  int nstw;              // entries of the stage-twiddle table (staged in smem once per CTA)
  int naux;              // entries of one per-tile auxiliary slice (sc * R; MODE 2: R)
};

// Shared-memory partition (double2 units): LD | WK | nyq | stw | aux, where aux holds
//   MODE 0: ptw slice [slot][e] (used by the first stage) + 2 x ftw slice [slot][k1]
//   MODE 1: 2 x yscale slice [slot][k2] as (yscale[2k], yscale[2k+1])
//   MODE 2: the whole ptw [e] and yscale [k] tables (loaded once per CTA)
// The slices used by the last stage are double-buffered: the next tile's are prefetched
// while the current tile's last stage still reads them.
struct Smem {
  double2 *ld, *wk, *nyq, *stw, *ptw, *aux2;  // aux2: two slices of a.naux
};
__device__ __forceinline__ Smem smem_parts(const C2RArgs& a, double2* base) {
  Smem p;
  const int tn = a.R << a.lgn;
  p.ld = base;
  p.wk = base + tn;
  p.nyq = base + 2 * tn;
  p.stw = p.nyq + (1 << a.lgn);
  p.ptw = p.stw + a.nstw;
  p.aux2 = p.ptw + ((a.mode == 1) ? 0 : a.naux);
  return p;
}

// Per-thread view of the current tile (offsets in elements; all < 2^31, checked on the host).
struct Slot {
  int sub;      // sub-sequence of this thread's sequence (clamped to 0 when invalid)
  int col;
  bool valid;
  int pmode;    // 0: partner element R-e in own sequence (sub 0; e = 0 -> Nyquist), 1: R-1-e own, 2: R-1-e other slot
  int psq;      // partner's sequence index (own or other slot)
  int sl;       // slot of this thread's sequence within the tile
};

// sub-sequence held by slot sl of sequence-group gy (-1: none)
template <int MODE>
__device__ __forceinline__ int slot_sub(const C2RArgs& a, int gy, int sl) {
  if (MODE == 0) {
    const int p = gy * (a.sc >> 1) + (sl >> 1);
    const int which = sl & 1;
    if (p >= a.P) return -1;
    if (p == 0) return which ? ((a.S & 1) ? -1 : a.S / 2) : 0;
    return which ? a.S - p : p;
  }
  if (MODE == 1) {
    const int sub = gy * a.sc + sl;
    return sub < a.S ? sub : -1;
  }
  return 0;
}

template <int MODE>
__device__ __forceinline__ Slot slot_of(const C2RArgs& a, int tile, int sq) {
  Slot s;
  const int gy = tile / a.ntx;
  const int gx = tile - gy * a.ntx;
  const int sl = sq >> a.lgcb, cl = sq & (a.cb - 1);
  s.col = gx * a.cb + cl;
  s.sl = sl;
  int sub;
  if (MODE == 0) {
    const int p = gy * (a.sc >> 1) + (sl >> 1);
    const int which = sl & 1;
    sub = -1;
    if (p < a.P) {
      if (p == 0) sub = which ? ((a.S & 1) ? -1 : a.S / 2) : 0;
      else sub = which ? a.S - p : p;
    }
    s.pmode = (sub == 0) ? 0 : ((2 * sub == a.S) ? 1 : 2);
  } else if (MODE == 1) {
    sub = gy * a.sc + sl;
    if (sub >= a.S) sub = -1;
    s.pmode = 0;
  } else {
    sub = 0;
    s.pmode = 0;
  }
  s.valid = sub >= 0 && s.col < a.ncol;
  s.sub = s.valid ? sub : 0;
  if (!s.valid) s.col = 0;
  s.psq = (s.pmode == 2) ? (sq ^ a.cb) : sq;
  return s;
}

__device__ __forceinline__ void cp16(double2* dst, const double2* src, bool v) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(v ? 16 : 0));
}

// coff: column offset of the tile's chunk in u / Y; soff: element offset of its scratch buffer
// (both 0 outside the fused two-pass kernel)
template <int MODE>
__device__ __forceinline__ void issue_loads(const C2RArgs& a, const FftIO& io, int tile, const Smem& sp, int abuf,
                                            int sq, int e0, int estep, int nth, int coff = 0, unsigned soff = 0) {
  Slot s = slot_of<MODE>(a, tile, sq);
  const double2* g;
  int gstep;
  if (MODE == 0) {
    g = io.Uc + (size_t)((unsigned)s.sub * (unsigned)io.ldu + s.col + coff);
    gstep = a.L2 * (int)io.ldu;
  } else if (MODE == 1) {
    g = a.scr + (size_t)(soff + (unsigned)s.sub * (unsigned)(a.L2 * a.lds) + s.col);
    gstep = a.lds;
  } else {
    g = io.Uc + s.col + coff;
    gstep = (int)io.ldu;
  }
  double2* d = sp.ld + (e0 << a.lgn) + sq;
  const int dstep = estep << a.lgn;
  for (int e = e0; e < a.R; e += estep, d += dstep) cp16(d, g + (size_t)((unsigned)e * (unsigned)gstep), s.valid);
  if (MODE != 1 && e0 == 0) {
    const bool v = s.valid && s.sub == 0;
    cp16(sp.nyq + sq, io.Uc + (size_t)((unsigned)a.M * (unsigned)io.ldu + s.col + coff), v);
  }
  if (MODE != 2) {  // this tile's twiddle / scale slices
    const int gy = tile / a.ntx;
    double2* aux = sp.aux2 + abuf * a.naux;
    for (int idx = threadIdx.x; idx < a.naux; idx += nth) {
      const int sl = idx / a.R, e = idx - sl * a.R;
      const int sub = slot_sub<MODE>(a, gy, sl);
      const int su = sub < 0 ? 0 : sub;
      if (MODE == 0) {
        cp16(sp.ptw + idx, a.ptw + su * a.R + e, true);
        cp16(aux + idx, a.ftw + su * a.R + e, true);
      } else {
        cp16(aux + idx, reinterpret_cast<const double2*>(io.yscale) + (su + a.L1 * e), true);
      }
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

// Z[e] of this thread's sequence (pairing of the half spectrum); branch-free.
template <int MODE>
__device__ __forceinline__ double2 zval(const Geo g, const Smem& sp, const Slot& s, int sq, int e) {
  double2 u = sp.ld[(e << g.lgn) + sq];
  const int pe = (s.pmode == 0) ? g.R - e : g.R - 1 - e;   // pe == R only for pmode 0, e == 0
  const double2* pp = (pe == g.R) ? sp.nyq + sq : sp.ld + (pe << g.lgn) + s.psq;
  double2 v = *pp;
  const double2 w = sp.ptw[(MODE == 0) ? s.sl * g.R + e : e];
  double evr = u.x + v.x, evi = u.y - v.y;  // u_n + conj u_{M-n}
  double dr = u.x - v.x, di = u.y + v.y;    // u_n - conj u_{M-n}
  double odr = dr * w.x - di * w.y, odi = dr * w.y + di * w.x;
  return make_double2(evr - odi, evi + odr);
}

// Epilogue context: per-tile base offsets so each store is one 32-bit multiply-add.
struct Epi {
  int base;   // MODE 0: sub * lds + col (scratch); MODE 1/2: column col of Y row 0 (+ m_off)
  int kstep;  // MODE 0: L2 * lds;   MODE 1/2: output k advances by L1 (MODE 1) or 1 per kk
};

template <int MODE>
__device__ __forceinline__ void store_out(const C2RArgs& a, const FftIO& io, const Geo g, const Slot& s,
                                          const Epi& ep, const double2* aux, int kk, double2 v, bool act) {
  if (MODE == 0) {
    const double2 w = aux[s.sl * g.R + kk];
    if (act) a.scr[(unsigned)(ep.base + kk * ep.kstep)] = c_mul(v, w);
  } else {
    const int k = (MODE == 1) ? s.sub + a.L1 * kk : kk;
    const int p = 2 * k;
    const double2 ys = aux[(MODE == 1) ? s.sl * g.R + kk : kk];  // (yscale[p], yscale[p+1])
    // signed: with m_off < 0 (trigonometric kind) rows below keep_lo give negative offsets (not stored)
    double* y = io.Y + (ptrdiff_t)(ep.base + p * (int)io.ldy);
    const bool k0 = act && p >= io.keep_lo && p < io.keep_hi;
    const bool k1 = act && p + 1 >= io.keep_lo && p + 1 < io.keep_hi;
    const double y0 = v.x * ys.x, y1 = v.y * ys.y;
    if (k0) __stcs(y, y0);
    if (k1) __stcs(y + io.ldy, y1);
  }
}

enum { IN_Z = 0, IN_LD = 1, IN_WK = 2 };
enum { OUT_WK = 0, OUT_G = 1 };

// One Stockham radix-r stage for this thread's sequence: butterflies j = e0 + b*estep < R/r.
// Out-of-range butterflies of the last round are computed on a clamped (valid) index and
// their stores suppressed, so there is no divergent control flow inside the stage.
template <int r, int IN, int OUT, int MODE, bool FIRST>
__device__ __forceinline__ void stage(const C2RArgs& a, const FftIO& io, const Geo g, const Smem& sp,
                                      const double2* aux, const Slot& s, const Epi& ep, int sq, int e0, int estep,
                                      const StageC c) {
  const double2* ld = sp.ld;
  double2* wk = sp.wk;
  constexpr int MB = (TILE / NTH + r - 1) / r;  // butterflies per thread (R * nseq <= TILE)
  const int lgn = g.lgn;
  double2 v[MB][r];
  bool act[MB], wact[MB];
  int jj[MB];
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    const int j = e0 + b * estep;
    act[b] = j < c.Rr;
    wact[b] = __any_sync(0xffffffffu, act[b]);  // warp-uniform: rounds with no work are skipped
    jj[b] = act[b] ? j : c.Rr - 1;
#pragma unroll
    for (int t = 0; t < r; ++t) {
      const int e = jj[b] + t * c.Rr;
      if (!wact[b]) v[b][t] = make_double2(0.0, 0.0);
      else if (IN == IN_Z) v[b][t] = zval<MODE>(g, sp, s, sq, e);
      else if (IN == IN_LD) v[b][t] = ld[(e << lgn) + sq];
      else v[b][t] = wk[(e << lgn) + sq];
    }
  }
  if (IN == IN_WK && OUT == OUT_WK) __syncthreads();  // in place: all reads before any write
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    if (!wact[b]) continue;
    int jd = jj[b], k = 0;
    if (!FIRST) {
      jd = (int)__umulhi((unsigned)jj[b], c.magic);
      k = jj[b] - jd * c.Ns;
      const double2* tw = sp.stw + c.twoff + k * (r - 1);
#pragma unroll
      for (int t = 1; t < r; ++t) v[b][t] = c_mul(v[b][t], tw[t - 1]);
    }
    bfly<r>(v[b]);
    const int idxD = FIRST ? jd * r : jd * c.Ns * r + k;
    const int ustep = FIRST ? 1 : c.Ns;
    const bool gact = act[b] && s.valid;
#pragma unroll
    for (int u = 0; u < r; ++u) {
      if (OUT == OUT_WK) {
        if (act[b]) wk[((idxD + u * ustep) << lgn) + sq] = v[b][u];
      } else {
        store_out<MODE>(a, io, g, s, ep, aux, idxD + u * ustep, v[b][u], gact);
      }
    }
  }
}

template <int IN, int OUT, int MODE, bool FIRST>
__device__ __forceinline__ void stage_r(const C2RArgs& a, const FftIO& io, const Geo g, const Smem& sp,
                                        const double2* aux, const Slot& s, const Epi& ep, int sq, int e0, int estep,
                                        const StageC& c) {
  switch (c.r) {
    case 2: stage<2, IN, OUT, MODE, FIRST>(a, io, g, sp, aux, s, ep, sq, e0, estep, c); break;
    case 3: stage<3, IN, OUT, MODE, FIRST>(a, io, g, sp, aux, s, ep, sq, e0, estep, c); break;
    case 4: stage<4, IN, OUT, MODE, FIRST>(a, io, g, sp, aux, s, ep, sq, e0, estep, c); break;
    case 5: stage<5, IN, OUT, MODE, FIRST>(a, io, g, sp, aux, s, ep, sq, e0, estep, c); break;
    case 6: stage<6, IN, OUT, MODE, FIRST>(a, io, g, sp, aux, s, ep, sq, e0, estep, c); break;
    case 9: stage<9, IN, OUT, MODE, FIRST>(a, io, g, sp, aux, s, ep, sq, e0, estep, c); break;
    default: stage<8, IN, OUT, MODE, FIRST>(a, io, g, sp, aux, s, ep, sq, e0, estep, c); break;
  }
}

// Compile-time stage sequence (specialised kernels): stages ST .. NF-2 in place, then the last.
template <int MODE, int RC, int ST>
__device__ __forceinline__ void stages_ct(const C2RArgs& a, const FftIO& io, const Geo g, const Smem& sp,
                                          const double2* aux, const Slot& s, const Epi& ep, int sq, int e0,
                                          int estep) {
  constexpr StagePlan P = stages_of(RC);
  constexpr StageC c = P.st[ST];
  if constexpr (ST + 1 < P.nf) {
    stage<c.r, IN_WK, OUT_WK, MODE, false>(a, io, g, sp, aux, s, ep, sq, e0, estep, c);
    __syncthreads();
    stages_ct<MODE, RC, ST + 1>(a, io, g, sp, aux, s, ep, sq, e0, estep);
  } else {
    stage<c.r, IN_WK, OUT_G, MODE, false>(a, io, g, sp, aux, s, ep, sq, e0, estep, c);
  }
}

// RC = 0: generic kernel (runtime length and radix plan); RC > 0: specialised for sub-length
// RC with 2^LGNC sequences per tile.
template <int MODE, int RC, int LGNC, int BIG = 0>
__global__ void __launch_bounds__(BIG ? 2 * NTH : NTH, BIG ? 1 : 3)
    c2r_pass(const __grid_constant__ C2RArgs a, const __grid_constant__ FftIO io) {
  constexpr int NT = BIG ? 2 * NTH : NTH;  // BIG: 512 threads, tiles up to 2 TILE (one CTA per SM)
  extern __shared__ double2 smem[];
  const Smem sp = smem_parts(a, smem);
  const Geo g = RC ? Geo{RC, LGNC >= 0 ? LGNC : a.lgn} : Geo{a.R, a.lgn};  // LGNC < 0: runtime
  const int tid = threadIdx.x;
  const int sq = tid & ((1 << g.lgn) - 1);
  const int e0 = tid >> g.lgn, estep = NT >> g.lgn;
  constexpr int IN0 = (MODE == 1) ? IN_LD : IN_Z;

  // once per CTA: the stage twiddles (and, single pass, the whole pairing / scale tables)
  for (int i = tid; i < a.nstw; i += NT) cp16(sp.stw + i, a.stw + i, true);
  if (MODE == 2)
    for (int i = tid; i < a.naux; i += NT) {
      cp16(sp.ptw + i, a.ptw + i, true);
      cp16(sp.aux2 + i, reinterpret_cast<const double2*>(io.yscale) + i, true);
    }
  int tile = blockIdx.x, abuf = 0;
  if (tile < a.ntiles) issue_loads<MODE>(a, io, tile, sp, abuf, sq, e0, estep, NT);
  for (; tile < a.ntiles; tile += gridDim.x, abuf ^= 1) {
    const Slot s = slot_of<MODE>(a, tile, sq);
    const double2* aux = (MODE == 2) ? sp.aux2 : sp.aux2 + abuf * a.naux;
    Epi ep;
    if (MODE == 0) {
      ep.base = s.sub * a.lds + s.col;
      ep.kstep = a.L2 * a.lds;
    } else {
      ep.base = io.m_off * (int)io.ldy + s.col;
      ep.kstep = 0;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();  // LD, nyq, slices complete for every thread; WK free (previous tile done)
    const bool more = tile + (int)gridDim.x < a.ntiles;
    if constexpr (RC > 0) {
      constexpr StagePlan P = stages_of(RC);
      constexpr StageC c0 = P.st[0];
      if constexpr (P.nf == 1) {
        stage<c0.r, IN0, OUT_G, MODE, true>(a, io, g, sp, aux, s, ep, sq, e0, estep, c0);
        __syncthreads();
        if (more) issue_loads<MODE>(a, io, tile + gridDim.x, sp, abuf ^ 1, sq, e0, estep, NT);
      } else {
        stage<c0.r, IN0, OUT_WK, MODE, true>(a, io, g, sp, aux, s, ep, sq, e0, estep, c0);
        __syncthreads();  // LD and the pairing slice consumed, WK written
        if (more) issue_loads<MODE>(a, io, tile + gridDim.x, sp, abuf ^ 1, sq, e0, estep, NT);
        stages_ct<MODE, RC, 1>(a, io, g, sp, aux, s, ep, sq, e0, estep);
      }
    } else {
      if (a.nf == 1) {
        stage_r<IN0, OUT_G, MODE, true>(a, io, g, sp, aux, s, ep, sq, e0, estep, a.st[0]);
        __syncthreads();
        if (more) issue_loads<MODE>(a, io, tile + gridDim.x, sp, abuf ^ 1, sq, e0, estep, NT);
        continue;
      }
      stage_r<IN0, OUT_WK, MODE, true>(a, io, g, sp, aux, s, ep, sq, e0, estep, a.st[0]);
      __syncthreads();  // LD and the pairing slice consumed, WK written
      if (more) issue_loads<MODE>(a, io, tile + gridDim.x, sp, abuf ^ 1, sq, e0, estep, NT);
      for (int st = 1; st + 1 < a.nf; ++st) {
        stage_r<IN_WK, OUT_WK, MODE, false>(a, io, g, sp, aux, s, ep, sq, e0, estep, a.st[st]);
        __syncthreads();
      }
      stage_r<IN_WK, OUT_G, MODE, false>(a, io, g, sp, aux, s, ep, sq, e0, estep, a.st[a.nf - 1]);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ---- fused two-pass C2R: both passes of a long length in one persistent kernel ----------------
// The batch is cut into chunks of cw columns; chunk c's four-step scratch (M x cw complex) lives
// in buffer c % nbuf (nbuf x ~22 MB: L2-resident), so pass 1 reads what pass 0 wrote from L2 and
// the 2 x 2.8 GB scratch round trip of c5's block 1 never reaches HBM.  CTAs claim tiles from one
// counter in the order P0(0), P0(1), P1(0), P0(2), P1(1), ..., P1(n-1) (Pp(c): the pass-p tiles of
// chunk c); a pass-1 tile waits until every pass-0 tile of its chunk is done, a pass-0 tile until
// the pass-1 tiles of the chunk nbuf before it (same buffer) are done.  Every tile it waits for
// was claimed earlier by a running CTA, so the waits end (no inter-launch dependency; one launch
// instead of 2 per chunk -- the per-launch ramps made the chunked two-launch form slower).
struct FusedCtl {
  unsigned* counter;  // tile claims (zeroed before the launch)
  unsigned* done0;    // per chunk: finished pass-0 tiles
  unsigned* done1;    // per chunk: finished pass-1 tiles
  int nchunk, cw, n0, n1, nbuf;
  unsigned sstride;   // elements between scratch buffers (M x cw)
};

__device__ __forceinline__ void fused_decode(const FusedCtl& f, int t, int& pass, int& c, int& lt) {
  if (t < f.n0) {
    pass = 0;
    c = 0;
    lt = t;
    return;
  }
  const int u = t - f.n0, blk = f.n0 + f.n1, k = u / blk, r = u - k * blk;
  if (k < f.nchunk - 1) {
    if (r < f.n0) {
      pass = 0;
      c = k + 1;
      lt = r;
    } else {
      pass = 1;
      c = k;
      lt = r - f.n0;
    }
  } else {
    pass = 1;
    c = f.nchunk - 1;
    lt = r;
  }
}

__device__ __forceinline__ bool fused_ready(const FusedCtl& f, int pass, int c) {
  if (pass == 1) return *(volatile unsigned*)(f.done0 + c) >= (unsigned)f.n0;
  return c < f.nbuf || *(volatile unsigned*)(f.done1 + c - f.nbuf) >= (unsigned)f.n1;
}

// One tile of pass MODE (sub-length RC, 2^LGNC sequences) with the next tile's loads issued after
// its first stage when ready.  Returns whether they were.
template <int MODE, int RC, int LGNC>
__device__ __forceinline__ bool fused_tile(const C2RArgs& a, const C2RArgs& an, int pn, const FftIO& io,
                                           const Smem& sp, int lt, int coff, unsigned soff, double2* aux,
                                           int ln, int cn_off, unsigned sn_off, double2* auxn, const Smem& spn,
                                           int lgnn, int* s_flag, bool next_ok) {
  constexpr int NT = 2 * NTH;
  const Geo g{RC, LGNC};
  const int tid = threadIdx.x;
  const int sq = tid & ((1 << LGNC) - 1), e0 = tid >> LGNC, estep = NT >> LGNC;
  constexpr int IN0 = (MODE == 1) ? IN_LD : IN_Z;
  const Slot s = slot_of<MODE>(a, lt, sq);
  Epi ep;
  if (MODE == 0) {
    ep.base = (int)(soff + (unsigned)(s.sub * a.lds + s.col));
    ep.kstep = a.L2 * a.lds;
  } else {
    ep.base = io.m_off * (int)io.ldy + s.col + coff;
    ep.kstep = 0;
  }
  constexpr StagePlan P = stages_of(RC);
  constexpr StageC c0 = P.st[0];
  static_assert(P.nf >= 2, "fused passes have two or more radix stages");
  stage<c0.r, IN0, OUT_WK, MODE, true>(a, io, g, sp, aux, s, ep, sq, e0, estep, c0);
  __syncthreads();  // LD consumed, WK written; s_flag set by thread 0 before this barrier
  const bool go = next_ok && *s_flag;
  if (go) {
    const int sqn = tid & ((1 << lgnn) - 1), e0n = tid >> lgnn, esn = NT >> lgnn;
    if (pn == 0) issue_loads<0>(an, io, ln, spn, 0, sqn, e0n, esn, NT, cn_off, sn_off);
    else issue_loads<1>(an, io, ln, spn, 0, sqn, e0n, esn, NT, cn_off, sn_off);
  }
  stages_ct<MODE, RC, 1>(a, io, g, sp, aux, s, ep, sq, e0, estep);
  (void)auxn;
  return go;
}

template <int R0, int L0, int R1, int L1>
__global__ void __launch_bounds__(2 * NTH, 1)
    c2r_fused(const __grid_constant__ C2RArgs a0, const __grid_constant__ C2RArgs a1,
              const __grid_constant__ FftIO io, const FusedCtl f) {
  constexpr int NT = 2 * NTH;
  constexpr int T0 = R0 << L0, T1 = R1 << L1, TT = T0 > T1 ? T0 : T1;
  constexpr int NQ = (1 << (L0 > L1 ? L0 : L1));
  extern __shared__ double2 smem[];
  __shared__ int s_tile, s_flag;
  const int naxm = a0.naux > a1.naux ? a0.naux : a1.naux;
  Smem b0, b1;  // the two passes' views of one layout: LD | WK | nyq | stw0 | stw1 | ptw | 2 aux slots
  b0.ld = b1.ld = smem;
  b0.wk = b1.wk = smem + TT;
  b0.nyq = b1.nyq = smem + 2 * TT;
  b0.stw = b0.nyq + NQ;
  b1.stw = b0.stw + a0.nstw;
  b0.ptw = b1.ptw = b1.stw + a1.nstw;
  double2* auxbase = b0.ptw + a0.naux;
  b0.aux2 = b1.aux2 = auxbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < a0.nstw; i += NT) cp16(b0.stw + i, a0.stw + i, true);
  for (int i = tid; i < a1.nstw; i += NT) cp16(b1.stw + i, a1.stw + i, true);
  const int total = f.nchunk * (f.n0 + f.n1);
  auto slot_view = [&](const Smem& b, int ab) {
    Smem v = b;
    v.aux2 = auxbase + ab * naxm;
    return v;
  };
  if (tid == 0) s_tile = (int)atomicAdd(f.counter, 1u);
  __syncthreads();
  int t = s_tile, abuf = 0;
  bool loaded = false;
  // the first tile's loads (after its dependency)
  if (t < total) {
    int p, c, lt;
    fused_decode(f, t, p, c, lt);
    if (tid == 0)
      while (!fused_ready(f, p, c)) __nanosleep(200);
    __threadfence();
    __syncthreads();
    const Smem v = slot_view(p == 0 ? b0 : b1, 0);
    const int lg = p == 0 ? L0 : L1;
    const int sq = tid & ((1 << lg) - 1), e0 = tid >> lg, es = NT >> lg;
    if (p == 0) issue_loads<0>(a0, io, lt, v, 0, sq, e0, es, NT, c * f.cw, (unsigned)(c % f.nbuf) * f.sstride);
    else issue_loads<1>(a1, io, lt, v, 0, sq, e0, es, NT, c * f.cw, (unsigned)(c % f.nbuf) * f.sstride);
    loaded = true;
  }
  while (t < total) {
    int p, c, lt;
    fused_decode(f, t, p, c, lt);
    __syncthreads();  // every thread has read s_tile of this tile
    if (tid == 0) s_tile = (int)atomicAdd(f.counter, 1u);  // claim the next tile now
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();  // this tile's data in; s_tile = the next tile
    const int tn = s_tile;
    int pn = 0, cn = 0, ln = 0;
    const bool has_next = tn < total;
    if (has_next) fused_decode(f, tn, pn, cn, ln);
    if (tid == 0) s_flag = has_next && fused_ready(f, pn, cn);  // read before the tile's first barrier
    const Smem cur = slot_view(p == 0 ? b0 : b1, abuf);
    const Smem nxt = slot_view(pn == 0 ? b0 : b1, abuf ^ 1);
    const int coff = c * f.cw, cnoff = cn * f.cw;
    const unsigned soff = (unsigned)(c % f.nbuf) * f.sstride, snoff = (unsigned)(cn % f.nbuf) * f.sstride;
    bool went;
    if (p == 0)
      went = fused_tile<0, R0, L0>(a0, pn == 0 ? a0 : a1, pn, io, cur, lt, coff, soff, cur.aux2, ln, cnoff, snoff,
                                   nxt.aux2, nxt, pn == 0 ? L0 : L1, &s_flag, has_next);
    else
      went = fused_tile<1, R1, L1>(a1, pn == 0 ? a0 : a1, pn, io, cur, lt, coff, soff, cur.aux2, ln, cnoff, snoff,
                                   nxt.aux2, nxt, pn == 0 ? L0 : L1, &s_flag, has_next);
    // this tile's results visible device-wide, then count it
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(p == 0 ? f.done0 + c : f.done1 + c, 1u);
    if (has_next && !went) {  // its dependency was not met at the first stage: wait, then load
      if (tid == 0)
        while (!fused_ready(f, pn, cn)) __nanosleep(200);
      __threadfence();
      __syncthreads();
      const int lg = pn == 0 ? L0 : L1;
      const int sq = tid & ((1 << lg) - 1), e0 = tid >> lg, es = NT >> lg;
      if (pn == 0) issue_loads<0>(a0, io, ln, nxt, 0, sq, e0, es, NT, cnoff, snoff);
      else issue_loads<1>(a1, io, ln, nxt, 0, sq, e0, es, NT, cnoff, snoff);
    } else if (has_next) {
      __threadfence();  // acquire side of the ready flag read by thread 0 (loads already issued)
    }
    t = tn;
    abuf ^= 1;
  }
  (void)loaded;
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

int ilog2i(int v) {
  int l = 0;
  while ((1 << (l + 1)) <= v) ++l;
  return l;
}


void set_radices(C2RArgs& a) {
  const StagePlan P = stages_of(a.R);
  a.nf = P.nf;
  int off = 0;
  for (int i = 0; i < P.nf; ++i) {
    a.st[i] = P.st[i];
    off = P.st[i].twoff + P.st[i].Ns * (P.st[i].r - 1);
  }
  a.nstw = std::max(off, 1);
}

// e^{+2 pi i m / n} with exact integer reduction of m
double2 cis(int64_t m, int64_t n) {
  const long double PI2 = 6.283185307179586476925286766559005768L;
  m %= n;
  if (m < 0) m += n;
  const long double ang = PI2 * (long double)m / (long double)n;
  return make_double2((double)cosl(ang), (double)sinl(ang));
}

void stage_table(int R, std::vector<double2>& t) {
  t.clear();
  const StagePlan P = stages_of(R);
  for (int i = 0; i < P.nf; ++i)
    for (int k = 0; k < P.st[i].Ns; ++k)
      for (int q = 1; q < P.st[i].r; ++q) t.push_back(cis((int64_t)k * q, (int64_t)P.st[i].Ns * P.st[i].r));
  if (t.empty()) t.push_back(make_double2(1.0, 0.0));
}

// Twiddle tables of one length M (cached per device; a few MB at most per length).
struct C2RTables {
  int dev = -1, M = 0, L1 = 0, L2 = 0;
  DevBuf stw0, stw1, ptw, ftw;
};
std::mutex g_tab_mu;
std::vector<C2RTables*> g_tabs;

template <typename T>
xc_status put(DevBuf& b, const std::vector<T>& v) {
  XC_TRY(dev_alloc(b, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) XC_CUDA(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return XC_OK;
}

xc_status tables_for(const FftPlan& p, const C2RTables** out) {
  int dev = 0;
  XC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_tab_mu);
  for (auto* t : g_tabs)
    if (t->dev == dev && t->M == p.L && t->L1 == p.L1 && t->L2 == p.L2) {
      *out = t;
      return XC_OK;
    }
  auto* t = new C2RTables();
  t->dev = dev;
  t->M = p.L;
  t->L1 = p.L1;
  t->L2 = p.L2;
  std::vector<double2> v;
  stage_table(p.L1, v);
  XC_TRY(put(t->stw0, v));
  if (p.L2 > 1) {
    stage_table(p.L2, v);
    XC_TRY(put(t->stw1, v));
  }
  const int64_t M = p.L, L1 = p.L1, L2 = p.L2;
  v.assign(M, make_double2(0, 0));
  for (int64_t n2 = 0; n2 < L2; ++n2)
    for (int64_t e = 0; e < L1; ++e) v[n2 * L1 + e] = cis(L2 * e + n2, 2 * M);  // e^{i pi n / M}
  XC_TRY(put(t->ptw, v));
  if (p.L2 > 1) {
    for (int64_t n2 = 0; n2 < L2; ++n2)
      for (int64_t k1 = 0; k1 < L1; ++k1) v[n2 * L1 + k1] = cis(n2 * k1, M);
    XC_TRY(put(t->ftw, v));
  }
  g_tabs.push_back(t);
  *out = t;
  return XC_OK;
}

// nseq = cb * sc (powers of two) with R * nseq <= TILE; columns first (cb <= 16), sc >= smin.
void choose(C2RArgs& a, int smin) {
  const int tile = a.big ? 2 * TILE : TILE, nth = a.big ? 2 * NTH : NTH;
  int nseq = 1;
  while (2 * nseq * a.R <= tile && nseq < nth && nseq < smin * a.S * std::max(1, a.ncol)) nseq *= 2;
  int cb = 1;
  while (cb < a.ncol && cb < 16 && 2 * cb * smin <= nseq) cb *= 2;
  a.cb = cb;
  a.sc = nseq / cb;
  a.lgcb = ilog2i(cb);
  a.lgn = ilog2i(nseq);
}

typedef void (*C2RKernel)(C2RArgs, FftIO);

// Specialised (mode, sub-length, log2 nseq) instances: the long passes of the configured
// workloads (c5: 43200 = 200 x 216, 13824 = 64 x 216, 4500 = 45 x 100, 1458 = 27 x 54;
// c3/c4: 10800 = 60 x 180, 5400 = 25 x 216, 3456 = 36 x 96, 1728 = 9 x 192).  Anything else
// runs the generic kernel.
struct Spec {
  int mode, R, lgn, big;
  C2RKernel k;
};
#define XC_SPEC(M, R, L) {M, R, L, 0, (C2RKernel)c2r_pass<M, R, L>}
#define XC_BIG(M, R, L) {M, R, L, 1, (C2RKernel)c2r_pass<M, R, L, 1>}
// BIG (512 threads, 64 KB tiles, 1 CTA / SM): the longest passes, so that a tile row is >= 128 B
const Spec kSpecs[] = {
    XC_BIG(0, 200, 4),
    XC_BIG(1, 432, 3), XC_BIG(1, 512, 3),  // second passes of M = 86400 = 200 x 432, 27648 = 54 x 512 (N = 131072)
    XC_SPEC(1, 216, 3), XC_SPEC(0, 54, 5),  XC_SPEC(1, 256, 3), XC_SPEC(0, 45, 5), XC_SPEC(1, 100, 4),
    XC_SPEC(0, 27, 6),  XC_SPEC(1, 54, 5),  XC_SPEC(1, 240, 3), XC_SPEC(1, 64, 5), XC_SPEC(0, 32, 6),
    XC_SPEC(0, 36, 5),  XC_SPEC(0, 9, 7),
    XC_SPEC(0, 25, 6),  XC_SPEC(1, 45, 5),  XC_SPEC(0, 15, 7),  XC_SPEC(1, 36, 5), XC_SPEC(1, 50, 5),  // c3, c8
    // single-pass lengths (M <= 512) of the configured workloads, any sequences per tile: a
    // compact kernel instead of the generic one (12.7K instructions; a one-CTA launch at B = 1
    // spends most of its 15 us fetching them)
    XC_SPEC(2, 360, -1), XC_SPEC(2, 144, -1), XC_SPEC(2, 54, -1),  XC_SPEC(2, 375, -1), XC_SPEC(2, 128, -1),
    XC_SPEC(2, 40, -1),  XC_SPEC(2, 200, -1), XC_SPEC(2, 64, -1),  XC_SPEC(2, 480, -1), XC_SPEC(2, 180, -1),
    XC_SPEC(2, 72, -1),  XC_SPEC(2, 30, -1),  XC_SPEC(2, 225, -1), XC_SPEC(2, 96, -1),  XC_SPEC(2, 45, -1),
};
#undef XC_SPEC
#undef XC_BIG

}  // namespace

namespace {
bool has_big(int mode, int R);
}

bool c2r_has_big(int mode, int R) { return has_big(mode, R); }

bool c2r_has_spec(int mode, int R) {
  for (const Spec& sp : kSpecs)
    if (sp.mode == mode && sp.R == R) return true;
  return false;
}

namespace {

// Big tiles (512 threads, 4096 points) for pass `mode` of length R: where a specialised big kernel
// exists, and for the lengths the specialised kernels do not cover whenever the 2048-point tile
// would leave rows narrower than 8 columns (128 B; R > 128 with paired sub-sequences, R > 256
// otherwise): the generic big kernel then doubles the row width (the passes' HBM throughput tracks
// it: 64 B rows 2.35 TB/s, 128 B 3.7 TB/s; tools/stride_probe.cu).
bool has_big(int mode, int R) {
  static const bool off = getenv("XC_C2R_GENERIC") || getenv("XC_C2R_NOBIG");  // measurement switches
  if (off) return false;
  bool spec = false;
  for (const Spec& sp : kSpecs)
    if (sp.mode == mode && sp.R == R) {
      if (sp.big) return true;
      spec = true;
    }
  if (spec || mode == 2) return false;
  return R > (mode == 0 ? 128 : 256);
}

template <int MODE>
xc_status launch(C2RArgs& a, const FftIO& io, cudaStream_t st) {
  static std::atomic<unsigned long long> once{0};
  if (first_on_device(once)) {
    XC_CUDA(cudaFuncSetAttribute(c2r_pass<MODE, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    XC_CUDA(cudaFuncSetAttribute(c2r_pass<MODE, 0, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (const Spec& sp : kSpecs)
      if (sp.mode == MODE)
        XC_CUDA(cudaFuncSetAttribute((const void*)sp.k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  const int nsm = sm_count();
  a.mode = MODE;
  a.ntx = (a.ncol + a.cb - 1) / a.cb;
  int nty;
  if (MODE == 0) nty = (a.P + a.sc / 2 - 1) / (a.sc / 2);
  else if (MODE == 1) nty = (a.S + a.sc - 1) / a.sc;
  else nty = 1;
  a.ntiles = a.ntx * nty;
  a.naux = (MODE == 2) ? a.R : a.sc * a.R;
  const int nseq = 1 << a.lgn;
  const size_t ent = 2 * (size_t)a.R * nseq + nseq + a.nstw + (MODE == 1 ? 0 : a.naux) +
                     (MODE == 2 ? 1 : 2) * (size_t)a.naux;
  const size_t sm = ent * sizeof(double2);
  if (sm > 200 * 1024) {
    xc_set_error("c2r: tile does not fit shared memory");
    return XC_EUNSUPPORTED;
  }
  C2RKernel k = a.big ? (C2RKernel)c2r_pass<MODE, 0, 0, 1> : (C2RKernel)c2r_pass<MODE, 0, 0>;
  int nt = a.big ? 2 * NTH : NTH;
  static const bool generic = getenv("XC_C2R_GENERIC") != nullptr;
  if (!generic)
    for (const Spec& sp : kSpecs)
      if (sp.mode == MODE && sp.R == a.R && (sp.lgn == a.lgn || sp.lgn < 0) && sp.big == a.big) {
        k = sp.k;
        nt = sp.big ? 2 * NTH : NTH;
      }
  static const bool log_generic = getenv("XC_C2R_LOG") != nullptr;  // which passes run generic
  if (log_generic && (k == (C2RKernel)c2r_pass<MODE, 0, 0> || k == (C2RKernel)c2r_pass<MODE, 0, 0, 1>))
    fprintf(stderr, "c2r generic: mode %d R %d lgn %d big %d\n", MODE, a.R, a.lgn, a.big);
  if (a.big && nt == NTH) {
    xc_set_error("c2r: big tile without a big kernel");
    return XC_EUNSUPPORTED;
  }
  int per_sm = 0;
  XC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, nt, sm));
  const int grid = std::min(a.ntiles, std::max(1, per_sm) * std::max(1, nsm));
  k<<<grid, nt, sm, st>>>(a, io);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

}  // namespace

int c2r_launches(const FftPlan& p) { return p.L2 > 1 ? 2 : 1; }

// Column chunk of a two-pass length: with XC_C2R_CHUNK_MB = m > 0 the four-step scratch of one chunk
// (M x chunk complex) is held near m MB so that pass 1 could read it from L2 right after pass 0
// wrote it.  Measured at c5 (B = 4096): the scratch traffic does leave HBM, but the FFT phase
// grows 3.94 -> 4.70 / 4.79 / 4.92 ms at m = 20 / 40 / 80 (2 x 64 launches for block 1 instead of
// 2, each a short persistent grid with its own ramp and tail; these passes are issue-bound, not
// HBM-bound), so the default is one chunk (m = 0); the switch stays for measurements.
int64_t c2r_chunk_cols(const FftPlan& p, int64_t B) {
  if (p.L2 <= 1 || B <= 64) return B;
  static const int64_t mb = getenv("XC_C2R_CHUNK_MB") ? atoll(getenv("XC_C2R_CHUNK_MB")) : 0;
  if (mb <= 0) return B;
  int64_t c = (mb << 20) / (16 * (int64_t)p.L) / 64 * 64;
  return std::min<int64_t>(B, std::max<int64_t>(64, c));
}

xc_status c2r_prepare(const FftPlan& p) {
  const C2RTables* tb = nullptr;
  return tables_for(p, &tb);
}

static xc_status c2r_run_cols(const FftPlan& p, const FftIO& io, int ncol, double2* scratch, cudaStream_t st);

// Fused instances (first pass R0 with 2^L0 sequences, second R1 with 2^L1; 512 threads, big tiles)
typedef void (*FusedKernel)(C2RArgs, C2RArgs, FftIO, FusedCtl);
struct FusedSpec {
  int R0, L0, R1, L1;
  FusedKernel k;
};
const FusedSpec kFused[] = {
    {200, 4, 216, 4, (FusedKernel)c2r_fused<200, 4, 216, 4>},   // c5 block 1: M = 43200
    {200, 4, 432, 3, (FusedKernel)c2r_fused<200, 4, 432, 3>},   // N = 131072 block 1: M = 86400
};

// Geometry of one pass for ncol columns with big tiles (launch<MODE>'s tile counts, no launch)
void pass_geometry(C2RArgs& a, int mode, int ncol) {
  a.mode = mode;
  a.ncol = ncol;
  a.lds = ncol;
  a.big = 1;
  set_radices(a);
  choose(a, mode == 0 ? 2 : 1);
  a.ntx = (a.ncol + a.cb - 1) / a.cb;
  const int nty = mode == 0 ? (a.P + a.sc / 2 - 1) / (a.sc / 2) : (a.S + a.sc - 1) / a.sc;
  a.ntiles = a.ntx * nty;
  a.naux = a.sc * a.R;
}

// The fused two-pass C2R when an instance exists for the plan's split and the batch has at least
// nbuf + 1 chunks (the control words sit in the scratch after the nbuf chunk buffers).
// XC_FUSED=0 turns it off; XC_FUSED_CW (columns per chunk, default 32), XC_FUSED_CTAS (grid).
xc_status c2r_fused_run(const FftPlan& p, const FftIO& io, int ncol, double2* scratch, cudaStream_t st, bool& done,
                        bool dry = false) {
  done = false;
  static const bool off = getenv("XC_FUSED") && atoi(getenv("XC_FUSED")) == 0;
  static const int cw_env = getenv("XC_FUSED_CW") ? atoi(getenv("XC_FUSED_CW")) : 32;
  static const int ctas_env = getenv("XC_FUSED_CTAS") ? atoi(getenv("XC_FUSED_CTAS")) : 0;
  if (off || p.L2 <= 1 || (!scratch && !dry)) return XC_OK;
  const int cw = std::max(16, cw_env / 16 * 16), nbuf = 3;
  if (ncol % cw != 0 || ncol < (nbuf + 1) * cw) return XC_OK;
  const C2RTables* tb = nullptr;
  XC_TRY(tables_for(p, &tb));
  C2RArgs a0{}, a1{};
  for (C2RArgs* a : {&a0, &a1}) {
    a->ptw = (const double2*)tb->ptw.p;
    a->ftw = (const double2*)tb->ftw.p;
    a->M = p.L;
    a->L1 = p.L1;
    a->L2 = p.L2;
    a->scr = scratch;
  }
  a0.R = p.L1;
  a0.S = p.L2;
  a0.P = (a0.S & 1) ? (a0.S + 1) / 2 : a0.S / 2;
  a0.stw = (const double2*)tb->stw0.p;
  pass_geometry(a0, 0, cw);
  a1.R = p.L2;
  a1.S = p.L1;
  a1.stw = (const double2*)tb->stw1.p;
  pass_geometry(a1, 1, cw);
  FusedKernel k = nullptr;
  for (const FusedSpec& f : kFused)
    if (f.R0 == a0.R && f.L0 == a0.lgn && f.R1 == a1.R && f.L1 == a1.lgn) k = f.k;
  if (!k || a0.sc < 2) return XC_OK;
  if ((int64_t)p.L * nbuf * cw >= (1LL << 31)) return XC_OK;
  if (dry) {
    done = true;
    return XC_OK;
  }
  FusedCtl f{};
  f.nchunk = ncol / cw;
  f.cw = cw;
  f.n0 = a0.ntiles;
  f.n1 = a1.ntiles;
  f.nbuf = nbuf;
  f.sstride = (unsigned)((int64_t)p.L * cw);
  unsigned* ctl = reinterpret_cast<unsigned*>(scratch + (size_t)nbuf * f.sstride);
  f.counter = ctl;
  f.done0 = ctl + 1;
  f.done1 = ctl + 1 + f.nchunk;
  XC_CUDA(cudaMemsetAsync(ctl, 0, (1 + 2 * (size_t)f.nchunk) * sizeof(unsigned), st));
  const int TT = std::max(a0.R << a0.lgn, a1.R << a1.lgn), NQ = 1 << std::max(a0.lgn, a1.lgn);
  const size_t sm = (size_t)(2 * TT + NQ + a0.nstw + a1.nstw + a0.naux + 2 * std::max(a0.naux, a1.naux)) *
                    sizeof(double2);
  if (sm > 220 * 1024) return XC_OK;
  static std::atomic<unsigned long long> once{0};
  if (first_on_device(once))
    for (const FusedSpec& fs : kFused)
      XC_CUDA(cudaFuncSetAttribute((const void*)fs.k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  const int nsm = sm_count();
  const int total = f.nchunk * (f.n0 + f.n1);
  const int grid = std::min(total, ctas_env > 0 ? ctas_env : nsm);
  k<<<grid, 2 * NTH, sm, st>>>(a0, a1, io, f);
  XC_CUDA(cudaGetLastError());
  done = true;
  return XC_OK;
}

int64_t c2r_launch_count(const FftPlan& p, int64_t ncol) {
  if (p.L2 <= 1) return 1;
  bool fused = false;
  FftIO io{};
  if (c2r_fused_run(p, io, (int)ncol, nullptr, nullptr, fused, true) == XC_OK && fused) return 1;
  const int64_t cw = c2r_chunk_cols(p, ncol);
  return 2 * ((ncol + cw - 1) / cw);
}

xc_status c2r_run(const FftPlan& p, const FftIO& io, int ncol, double2* scratch, cudaStream_t st) {
  bool fused = false;
  XC_TRY(c2r_fused_run(p, io, ncol, scratch, st, fused));
  if (fused) return XC_OK;
  const int64_t cw = c2r_chunk_cols(p, ncol);
  if (cw >= ncol) return c2r_run_cols(p, io, ncol, scratch, st);
  for (int64_t c0 = 0; c0 < ncol; c0 += cw) {  // columns are independent: chunk by chunk
    FftIO ic = io;
    ic.Uc = io.Uc + c0;
    ic.Y = io.Y + c0;
    XC_TRY(c2r_run_cols(p, ic, (int)std::min<int64_t>(cw, ncol - c0), scratch, st));
  }
  return XC_OK;
}

static xc_status c2r_run_cols(const FftPlan& p, const FftIO& io, int ncol, double2* scratch, cudaStream_t st) {
  C2RArgs a{};
  // 32-bit element offsets inside the kernels
  if ((int64_t)p.L * ncol >= (1LL << 31) || (int64_t)(io.keep_hi + io.m_off + 1) * io.ldy >= (1LL << 31) ||
      (int64_t)(p.L + 1) * io.ldu >= (1LL << 31)) {
    xc_set_error("c2r: batch too large for 32-bit offsets (split the batch)");
    return XC_EUNSUPPORTED;
  }
  const C2RTables* tb = nullptr;
  XC_TRY(tables_for(p, &tb));
  a.ptw = (const double2*)tb->ptw.p;
  a.ftw = (const double2*)tb->ftw.p;
  a.M = p.L;
  a.L1 = p.L1;
  a.L2 = p.L2;
  a.ncol = ncol;
  a.scr = scratch;
  a.lds = ncol;
  if (p.L2 == 1) {
    a.mode = 2;
    a.R = p.L1;
    a.S = 1;
    set_radices(a);
    a.stw = (const double2*)tb->stw0.p;
    // one sequence per column: every slot is a column
    int nseq = 1;
    while (2 * nseq * a.R <= TILE && nseq < NTH && nseq < ncol) nseq *= 2;
    a.cb = nseq;
    a.sc = 1;
    a.lgcb = a.lgn = ilog2i(nseq);
    if (a.R * nseq > TILE) {
      xc_set_error("c2r: length too long for one pass");
      return XC_EUNSUPPORTED;
    }
    return launch<2>(a, io, st);
  }
  if (!scratch) {
    xc_set_error("c2r: two-pass length needs scratch");
    return XC_EINVAL;
  }
  // pass 0: L1-point transforms over the L2 sub-sequences, slots paired {p, L2 - p}
  a.mode = 0;
  a.R = p.L1;
  a.S = p.L2;
  a.P = (a.S & 1) ? (a.S + 1) / 2 : a.S / 2;
  set_radices(a);
  a.stw = (const double2*)tb->stw0.p;
  a.big = has_big(0, a.R) && ncol >= 64;
  choose(a, 2);
  if (a.sc < 2 || a.R * (1 << a.lgn) > (a.big ? 2 : 1) * TILE) {
    xc_set_error("c2r: first-pass length too long");
    return XC_EUNSUPPORTED;
  }
  XC_TRY(launch<0>(a, io, st));
  // pass 1: L2-point transforms over the L1 sub-sequences
  a.mode = 1;
  a.R = p.L2;
  a.S = p.L1;
  set_radices(a);
  a.stw = (const double2*)tb->stw1.p;
  a.big = has_big(1, a.R) && ncol >= 64;
  choose(a, 1);
  if (a.R * (1 << a.lgn) > (a.big ? 2 : 1) * TILE) {
    xc_set_error("c2r: second-pass length too long");
    return XC_EUNSUPPORTED;
  }
  return launch<1>(a, io, st);
}
