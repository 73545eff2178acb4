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
template <int r, int IN, int OUT, int MODE, bool FIRST, int PPT = TILE / NTH>
__device__ __forceinline__ void stage(const C2RArgs& a, const FftIO& io, const Geo g, const Smem& sp,
                                      const double2* aux, const Slot& s, const Epi& ep, int sq, int e0, int estep,
                                      const StageC c) {
  const double2* ld = sp.ld;
  double2* wk = sp.wk;
  constexpr int MB = (PPT + r - 1) / r;  // butterflies per thread (R * nseq <= PPT * threads)
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
template <int MODE, int RC, int ST, int PPT = TILE / NTH>
__device__ __forceinline__ void stages_ct(const C2RArgs& a, const FftIO& io, const Geo g, const Smem& sp,
                                          const double2* aux, const Slot& s, const Epi& ep, int sq, int e0,
                                          int estep) {
  constexpr StagePlan P = stages_of(RC);
  constexpr StageC c = P.st[ST];
  if constexpr (ST + 1 < P.nf) {
    stage<c.r, IN_WK, OUT_WK, MODE, false, PPT>(a, io, g, sp, aux, s, ep, sq, e0, estep, c);
    __syncthreads();
    stages_ct<MODE, RC, ST + 1, PPT>(a, io, g, sp, aux, s, ep, sq, e0, estep);
  } else {
    stage<c.r, IN_WK, OUT_G, MODE, false, PPT>(a, io, g, sp, aux, s, ep, sq, e0, estep, c);
  }
}

// RC = 0: generic kernel (runtime length and radix plan); RC > 0: specialised for sub-length
// RC with 2^LGNC sequences per tile.
// BIG = 1: 512 threads, tiles up to 2 TILE points (one CTA per SM); BIG = 2 ("wide"): 512 threads,
// tiles up to kWide points (~200 KB of double-buffered tiles), so that a first pass of 200 points
// has 32 sequences = 16 columns (256-B rows)
constexpr int kWide = 6400;
template <int MODE, int RC, int LGNC, int BIG = 0>
__global__ void __launch_bounds__(BIG ? 2 * NTH : NTH, BIG ? 1 : 3)
    c2r_pass(const __grid_constant__ C2RArgs a, const __grid_constant__ FftIO io) {
  constexpr int NT = BIG ? 2 * NTH : NTH;
  constexpr int PPT = BIG == 2 ? (kWide + 2 * NTH - 1) / (2 * NTH) : TILE / NTH;  // points per thread
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
        stage<c0.r, IN0, OUT_G, MODE, true, PPT>(a, io, g, sp, aux, s, ep, sq, e0, estep, c0);
        __syncthreads();
        if (more) issue_loads<MODE>(a, io, tile + gridDim.x, sp, abuf ^ 1, sq, e0, estep, NT);
      } else {
        stage<c0.r, IN0, OUT_WK, MODE, true, PPT>(a, io, g, sp, aux, s, ep, sq, e0, estep, c0);
        __syncthreads();  // LD and the pairing slice consumed, WK written
        if (more) issue_loads<MODE>(a, io, tile + gridDim.x, sp, abuf ^ 1, sq, e0, estep, NT);
        stages_ct<MODE, RC, 1, PPT>(a, io, g, sp, aux, s, ep, sq, e0, estep);
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
  const int tile = a.big == 2 ? kWide : (a.big ? 2 * TILE : TILE), nth = a.big ? 2 * NTH : NTH;
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
#define XC_WIDE(M, R, L) {M, R, L, 2, (C2RKernel)c2r_pass<M, R, L, 2>}
// BIG (512 threads, 64 KB tiles, 1 CTA / SM): the longest passes, so that a tile row is >= 128 B
const Spec kSpecs[] = {
    XC_BIG(0, 200, 4), XC_WIDE(0, 200, 5),
    XC_BIG(1, 432, 3), XC_BIG(1, 512, 3),  // second passes of M = 86400 = 200 x 432, 27648 = 54 x 512 (N = 131072)
    XC_BIG(0, 100, 5),  // first pass of M = 43200 = 100 x 432 with 16-column (256-B) tile rows
                        // (c5 block 1 10.92 -> 10.74 ms, N = 32768 5.13 -> 5.00 ms vs 200 x 216)
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
#undef XC_WIDE

}  // namespace

namespace {
bool has_big(int mode, int R);
}

bool c2r_has_big(int mode, int R) { return has_big(mode, R); }

bool c2r_has_wide(int mode, int R) {
  static const bool off = getenv("XC_C2R_GENERIC") || getenv("XC_C2R_NOBIG") || getenv("XC_C2R_NOWIDE");
  if (off) return false;
  for (const Spec& sp : kSpecs)
    if (sp.mode == mode && sp.R == R && sp.big == 2) return true;
  return false;
}

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
    XC_CUDA(cudaFuncSetAttribute(c2r_pass<MODE, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    XC_CUDA(cudaFuncSetAttribute(c2r_pass<MODE, 0, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    for (const Spec& sp : kSpecs)
      if (sp.mode == MODE)
        XC_CUDA(cudaFuncSetAttribute((const void*)sp.k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
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
  if (sm > 227 * 1024) {
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

int64_t c2r_launch_count(const FftPlan& p, int64_t ncol) {
  if (p.L2 <= 1) return 1;
  const int64_t cw = c2r_chunk_cols(p, ncol);
  return 2 * ((ncol + cw - 1) / cw);
}

xc_status c2r_run(const FftPlan& p, const FftIO& io, int ncol, double2* scratch, cudaStream_t st) {
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
  a.big = ncol >= 64 ? (c2r_has_wide(0, a.R) && ncol >= 128 ? 2 : (has_big(0, a.R) ? 1 : 0)) : 0;
  choose(a, 2);
  if (a.sc < 2 || a.R * (1 << a.lgn) > (a.big == 2 ? kWide : (a.big ? 2 : 1) * TILE)) {
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
