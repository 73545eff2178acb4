// fft.cu -- batched fp64 mixed-radix FFT for the extra-component method (sm_100a).
//
// The transform of Eq. (1) along the slow axis of a batch-fastest array
// (element (n, col) at n*ld + col), for any 2-3-5-smooth length L (R-9).
// Lengths up to 1024 run in one pass; longer ones as a four-step L = L1*L2:
//   pass 1: for each n2, L1-point FFT over n = L2*n1 + n2, times w_L^{sigma n2 k1},
//           stored at scratch[k1*L2 + n2]  (L2-resident: the scratch of one block)
//   pass 2: for each k1, L2-point FFT over scratch[k1*L2 + n2], output k = k1 + L1*k2.
// Each pass stages `cb` columns x `sc` sub-sequences in shared memory (ping-pong
// buffers) and runs self-sorting Stockham radix-{8,4,5,3,2} stages with the
// butterflies in registers; twiddles come from exact tables (long double on the
// host), raised to the r-th power by complex multiplication.
//
// The prologue of the first pass can fuse the input-axis pre-processing (P:137-156 Fe1 pad +
// W^{-1}; PRO_XREAL) and the epilogue of the last the z' planes layout (EPI_ZPLANES), see
// FftPro / FftEpi in xc_internal.cuh.  Serves the precompute (forward, Eq. 1) and the input
// axis; the output-axis real-output inverse has its own engine (c2r.cu).
#include <math.h>

#include <algorithm>
#include <vector>

#include <stdio.h>

#include "xc_internal.cuh"

namespace {

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 c_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by S*i
template <int S>
__device__ __forceinline__ double2 c_si(double2 a) {
  return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <int S>
__device__ __forceinline__ void bfly2(double2* v) {
  double2 t = c_sub(v[0], v[1]);
  v[0] = c_add(v[0], v[1]);
  v[1] = t;
}
template <int S>
__device__ __forceinline__ void bfly4(double2& v0, double2& v1, double2& v2, double2& v3) {
  double2 a = c_add(v0, v2), b = c_sub(v0, v2), c = c_add(v1, v3), d = c_si<S>(c_sub(v1, v3));
  v0 = c_add(a, c);
  v2 = c_sub(a, c);
  v1 = c_add(b, d);
  v3 = c_sub(b, d);
}
template <int S>
__device__ __forceinline__ void bfly8(double2* v) {
  const double R2 = 0.70710678118654752440;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  bfly4<S>(e0, e1, e2, e3);
  bfly4<S>(o0, o1, o2, o3);
  // o1 *= e^{S i pi/4}, o2 *= S i, o3 *= e^{S 3 i pi/4}
  o1 = make_double2(R2 * (o1.x - S * o1.y), R2 * (o1.y + S * o1.x));
  o2 = c_si<S>(o2);
  o3 = make_double2(R2 * (-o3.x - S * o3.y), R2 * (-o3.y + S * o3.x));
  v[0] = c_add(e0, o0);
  v[4] = c_sub(e0, o0);
  v[1] = c_add(e1, o1);
  v[5] = c_sub(e1, o1);
  v[2] = c_add(e2, o2);
  v[6] = c_sub(e2, o2);
  v[3] = c_add(e3, o3);
  v[7] = c_sub(e3, o3);
}
template <int S>
__device__ __forceinline__ void bfly3(double2* v) {
  const double C = -0.5, SN = S * 0.86602540378443864676;
  double2 a = c_add(v[1], v[2]), b = c_sub(v[1], v[2]);
  double2 m = make_double2(v[0].x + C * a.x, v[0].y + C * a.y);
  double2 ib = make_double2(-SN * b.y, SN * b.x);  // i * SN * b
  v[0] = c_add(v[0], a);
  v[1] = c_add(m, ib);
  v[2] = c_sub(m, ib);
}
template <int S>
__device__ __forceinline__ void bfly5(double2* v) {
  const double C1 = 0.30901699437494742410, C2 = -0.80901699437494742410;
  const double S1 = S * 0.95105651629515357212, S2 = S * 0.58778525229247312917;
  double2 a1 = c_add(v[1], v[4]), b1 = c_sub(v[1], v[4]);
  double2 a2 = c_add(v[2], v[3]), b2 = c_sub(v[2], v[3]);
  double2 x0 = v[0];
  double2 m1 = make_double2(x0.x + C1 * a1.x + C2 * a2.x, x0.y + C1 * a1.y + C2 * a2.y);
  double2 m2 = make_double2(x0.x + C2 * a1.x + C1 * a2.x, x0.y + C2 * a1.y + C1 * a2.y);
  double2 t1 = make_double2(S1 * b1.x + S2 * b2.x, S1 * b1.y + S2 * b2.y);
  double2 t2 = make_double2(S2 * b1.x - S1 * b2.x, S2 * b1.y - S1 * b2.y);
  // i * t = (-t.y, t.x)
  v[0] = make_double2(x0.x + a1.x + a2.x, x0.y + a1.y + a2.y);
  v[1] = make_double2(m1.x - t1.y, m1.y + t1.x);
  v[4] = make_double2(m1.x + t1.y, m1.y - t1.x);
  v[2] = make_double2(m2.x - t2.y, m2.y + t2.x);
  v[3] = make_double2(m2.x + t2.y, m2.y - t2.x);
}

// One self-sorting Stockham radix-r stage over nseq = 2^lgn interleaved sequences of length R
// (smem layout [n][seq]); twiddle w_{Ns r}^{k t} from the length-R table.  j / Ns by a
// precomputed multiplier (exact for j < 2^16).
template <int r, int SIG>
__device__ __forceinline__ void stockham_stage(const double2* __restrict__ bin, double2* __restrict__ bout, int R,
                                               int Ns, unsigned magic, int lgn, const double2* __restrict__ tw,
                                               int sq, int j0, int jstep) {
  // this thread's sequence sq is fixed (blockDim is a multiple of nseq); j runs over butterflies
  const int Rr = R / r;
  const int twstep = R / (Ns * r);
  for (int j = j0; j < Rr; j += jstep) {
    int jd = (Ns == 1) ? j : (int)__umulhi((unsigned)j, magic);  // j / Ns
    int k = j - jd * Ns;
    double2 v[r];
#pragma unroll
    for (int t = 0; t < r; ++t) v[t] = bin[((j + t * Rr) << lgn) + sq];
    if (k > 0) {
      double2 w = __ldg(tw + k * twstep);
      if (SIG < 0) w.y = -w.y;
      double2 wt = w;
#pragma unroll
      for (int t = 1; t < r; ++t) {
        v[t] = c_mul(v[t], wt);
        if (t + 1 < r) wt = c_mul(wt, w);
      }
    }
    if (r == 2) bfly2<SIG>(v);
    else if (r == 3) bfly3<SIG>(v);
    else if (r == 4) bfly4<SIG>(v[0], v[1], v[2], v[3]);
    else if (r == 5) bfly5<SIG>(v);
    else bfly8<SIG>(v);
    int idxD = jd * Ns * r + k;
#pragma unroll
    for (int u = 0; u < r; ++u) bout[((idxD + u * Ns) << lgn) + sq] = v[u];
  }
}

struct PassArgs {
  int R;             // sub-FFT length of this pass
  int nf;            // number of radix stages
  int f[12];         // radices
  unsigned magic[12];// ceil(2^32 / Ns) of each stage
  const double2* tw; // e^{+2 pi i n/R}
  const double2* twL;// e^{+2 pi i n/L} (stage 0 only)
  int L, L1, L2;
  int stage;         // 0 = first of two, 1 = second of two, 2 = single
  int S;             // number of sub-sequences per column
  int ncol, cb, sc;  // cb, sc powers of two
  int lgcb, lgn;     // log2(cb), log2(cb * sc)
  double2* scratch;  // two-pass intermediate, index (k1*L2 + n2)*ncol + col
};

template <int PRO>
__device__ __forceinline__ double2 pro_load(const FftIO& io, int n, int col) {
  if (PRO == PRO_PLAIN) {
    return io.src[(int64_t)n * io.lds + col];
  } else if (PRO == PRO_XCPLX) {  // XC_EXP: planar complex input (rows N.. imaginary), pad + W^{-1}
    if (n >= io.keep_lo && n < io.keep_hi) {
      const int64_t o = (int64_t)(n + io.m_off) * io.ldx + col;
      return make_double2(io.X[o] * io.winv[n], io.X[io.xpl + o] * io.winv[n]);
    }
    return make_double2(0.0, 0.0);
  } else {  // PRO_XREAL: pad + W^{-1} (Fe1 / Fe3)
    if (n >= io.keep_lo && n < io.keep_hi)
      return make_double2(io.X[(int64_t)(n + io.m_off) * io.ldx + col] * io.winv[n], 0.0);
    return make_double2(0.0, 0.0);
  }
}

template <int EPI>
__device__ __forceinline__ void epi_store(const FftIO& io, int k, int col, double2 v) {
  if (EPI == EPI_PLAIN) {
    if (k < io.kmax) io.dst[(int64_t)k * io.ldd + col] = c_scale(v, io.scale);
  } else if (EPI == EPI_CY) {
    // XC_EXP: complex output position k kept (Fe2), times 1/(sqrt(L) w_k); planar Y
    if (k >= io.keep_lo && k < io.keep_hi) {
      const int64_t o = (int64_t)(k + io.m_off) * io.ldy + col;
      io.Y[o] = v.x * io.yscale[k];
      io.Y[io.ypl + o] = v.y * io.yscale[k];
    }
  } else {  // EPI_ZPLANES
    if (k < io.H) {
      io.zre[(int64_t)k * io.ldz + col] = v.x * io.scale;
      io.zim[(int64_t)k * io.ldz + col] = v.y * io.scale;
    }
  }
}

template <int PRO, int EPI, int SIG>
__global__ void __launch_bounds__(256, 3) fft_pass(PassArgs a, FftIO io) {
  extern __shared__ double2 smem[];
  const int nseq = 1 << a.lgn;
  double2* bin = smem;
  double2* bout = smem + a.R * nseq;
  const int tid = threadIdx.x, nth = blockDim.x;
  // per-thread constants (nth is a multiple of nseq): sequence sq, its slot, sub-sequence and column
  const int sq = tid & (nseq - 1);
  const int e0 = tid >> a.lgn, estep = nth >> a.lgn;
  const int slot = sq >> a.lgcb, cl = sq & (a.cb - 1);
  const int sub = blockIdx.y * a.sc + slot;
  const int col = blockIdx.x * a.cb + cl;
  const bool valid = sub < a.S && col < a.ncol;

  // ---- load (prologue) ----
  if ((PRO == PRO_XREAL || PRO == PRO_XCPLX) && a.stage != 1) {
    // real input scaled by W^{-1}: through registers
    for (int e = e0; e < a.R; e += 4 * estep) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int ee = e + u * estep;
        v[u] = make_double2(0.0, 0.0);
        if (valid && ee < a.R) v[u] = pro_load<PRO>(io, (a.stage == 0) ? a.L2 * ee + sub : ee, col);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int ee = e + u * estep;
        if (ee < a.R) bin[(ee << a.lgn) + sq] = v[u];
      }
    }
  } else if (valid) {
    // complex input: asynchronous 16-byte copies global -> shared, all in flight at once
    const double2* g;
    int64_t gstep;
    if (a.stage == 1) {
      g = a.scratch + ((int64_t)sub * a.L2) * a.ncol + col;
      gstep = a.ncol;
    } else {
      const int nstride = (a.stage == 0) ? a.L2 : 1;
      g = io.src + (int64_t)sub * io.lds + col;
      gstep = (int64_t)nstride * io.lds;
    }
    for (int e = e0; e < a.R; e += estep) {
      unsigned sa = (unsigned)__cvta_generic_to_shared(bin + (e << a.lgn) + sq);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g + e * gstep));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  } else {
    for (int e = e0; e < a.R; e += estep) bin[(e << a.lgn) + sq] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  // ---- Stockham stages ----
  int Ns = 1;
  for (int st = 0; st < a.nf; ++st) {
    const int r = a.f[st];
    const unsigned mg = a.magic[st];
    switch (r) {
      case 2: stockham_stage<2, SIG>(bin, bout, a.R, Ns, mg, a.lgn, a.tw, sq, e0, estep); break;
      case 3: stockham_stage<3, SIG>(bin, bout, a.R, Ns, mg, a.lgn, a.tw, sq, e0, estep); break;
      case 4: stockham_stage<4, SIG>(bin, bout, a.R, Ns, mg, a.lgn, a.tw, sq, e0, estep); break;
      case 5: stockham_stage<5, SIG>(bin, bout, a.R, Ns, mg, a.lgn, a.tw, sq, e0, estep); break;
      default: stockham_stage<8, SIG>(bin, bout, a.R, Ns, mg, a.lgn, a.tw, sq, e0, estep); break;
    }
    __syncthreads();
    double2* t = bin;
    bin = bout;
    bout = t;
    Ns *= r;
  }

  // ---- store (epilogue) ----
  if (!valid) return;
  if (a.stage == 0) {
    // four-step twiddle w_L^{sigma n2 k1}, n2 = sub, k1 = e (n2 k1 < L)
    double2* dstp = a.scratch + (int64_t)sub * a.ncol + col;
    const int64_t dstep = (int64_t)a.L2 * a.ncol;
    for (int e = e0; e < a.R; e += estep) {
      double2 w = __ldg(a.twL + sub * e);
      if (SIG < 0) w.y = -w.y;
      dstp[e * dstep] = c_mul(bin[(e << a.lgn) + sq], w);
    }
  } else {
    const int kstride = (a.stage == 1) ? a.L1 : 1;
    for (int e = e0; e < a.R; e += estep) epi_store<EPI>(io, sub + kstride * e, col, bin[(e << a.lgn) + sq]);
  }
}

void factorize(int R, int& nf, int* f) {
  nf = 0;
  while (R % 8 == 0) { f[nf++] = 8; R /= 8; }
  while (R % 4 == 0) { f[nf++] = 4; R /= 4; }
  while (R % 2 == 0) { f[nf++] = 2; R /= 2; }
  while (R % 5 == 0) { f[nf++] = 5; R /= 5; }
  while (R % 3 == 0) { f[nf++] = 3; R /= 3; }
  if (R != 1) nf = -1;
}

void twiddle_table(int n, std::vector<double2>& t) {
  t.resize(n);
  const long double PI2 = 6.283185307179586476925286766559005768L;
  for (int i = 0; i < n; ++i) {
    long double ang = PI2 * (long double)i / (long double)n;
    t[i] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
}

template <int PRO, int EPI, int SIG>
xc_status launch_pass(const PassArgs& a, const FftIO& io, cudaStream_t st) {
  const int nseq = 1 << a.lgn;
  size_t sm = 2ull * a.R * nseq * sizeof(double2);
  static std::atomic<unsigned long long> once{0};
  if (first_on_device(once))
    XC_CUDA(cudaFuncSetAttribute(fft_pass<PRO, EPI, SIG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 120 * 1024));
  int gy = (a.S + a.sc - 1) / a.sc;
  dim3 grid((a.ncol + a.cb - 1) / a.cb, gy);
  int work = a.R * nseq / 2;
  int th = work >= 256 ? 256 : (work >= 128 ? 128 : 64);
  fft_pass<PRO, EPI, SIG><<<grid, th, sm, st>>>(a, io);
  XC_CUDA(cudaGetLastError());
  return XC_OK;
}

template <int SIG>
xc_status dispatch(FftPro pro, FftEpi epi, const PassArgs& a, const FftIO& io, cudaStream_t st) {
  // pass-1-of-2 uses only the prologue, pass-2-of-2 only the epilogue
  if (a.stage == 0) {
    if (pro == PRO_PLAIN) return launch_pass<PRO_PLAIN, EPI_PLAIN, SIG>(a, io, st);
    if (pro == PRO_XCPLX) return launch_pass<PRO_XCPLX, EPI_PLAIN, SIG>(a, io, st);
    return launch_pass<PRO_XREAL, EPI_PLAIN, SIG>(a, io, st);
  }
  if (a.stage == 1) {
    if (epi == EPI_PLAIN) return launch_pass<PRO_PLAIN, EPI_PLAIN, SIG>(a, io, st);
    if (epi == EPI_CY) return launch_pass<PRO_PLAIN, EPI_CY, SIG>(a, io, st);
    return launch_pass<PRO_PLAIN, EPI_ZPLANES, SIG>(a, io, st);
  }
#define XC_CASE(P, E) \
  if (pro == P && epi == E) return launch_pass<P, E, SIG>(a, io, st);
  XC_CASE(PRO_PLAIN, EPI_PLAIN)
  XC_CASE(PRO_PLAIN, EPI_ZPLANES)
  XC_CASE(PRO_PLAIN, EPI_CY)
  XC_CASE(PRO_XREAL, EPI_PLAIN)
  XC_CASE(PRO_XREAL, EPI_ZPLANES)
  XC_CASE(PRO_XCPLX, EPI_ZPLANES)
#undef XC_CASE
  xc_set_error("fft: bad prologue/epilogue");
  return XC_EINVAL;
}

int ilog2(int v) {
  int l = 0;
  while ((1 << (l + 1)) <= v) ++l;
  return l;
}

// Tile: nseq = cb * sc sequences of length R in ping-pong smem of 32 R nseq bytes;
// cb, sc powers of two.
constexpr int kTileElems = 1792;  // R * nseq per CTA: 2 buffers x 16 B -> 56 KB, 3-4 CTAs per SM

void choose_tile(int R, int ncol, int sc, int& cb) {
  int nseq = sc;
  while (nseq < 16 * sc && 2 * nseq * R <= kTileElems) nseq *= 2;
  cb = nseq / sc;
  while (cb > 1 && cb / 2 >= ncol) cb /= 2;
}

void set_stages(PassArgs& a, int nf, const int* f) {
  a.nf = nf;
  int Ns = 1;
  for (int i = 0; i < nf; ++i) {
    a.f[i] = f[i];
    a.magic[i] = (Ns == 1) ? 0u : (unsigned)((0x100000000ULL + Ns - 1) / Ns);
    Ns *= f[i];
  }
}

}  // namespace

// Cost model of one C2R pass (c2r.cu) per element: warp-rounds of its radix stages (256 threads,
// tiles of R * nseq <= 2048 points -- 512 / 4096 for the big-tile kernels --, nseq a power of two
// with at least smin sub-sequences, rounds without an active lane skipped per warp) times the
// measured throughput penalty of its tile-row width (cb columns x 16 B: 64 B rows ran at 2.35,
// 128 B at 3.75, 256 B at 5.8 TB/s on c5).
double c2r_pass_cost(int R, int smin, int mode) {
  const C2RRadices pl = c2r_radices(R);
  if (pl.nf < 0) return 1e30;
  const bool wide = c2r_has_wide(mode, R), big = wide || c2r_has_big(mode, R);
  const int tile = wide ? 6400 : (big ? 4096 : 2048), nth = big ? 512 : 256;
  int nseq = 1;
  while (2 * nseq * R <= tile && nseq < nth) nseq *= 2;
  if (nseq < smin) return 1e30;
  const int cb = std::min(16, nseq / smin);
  const double pen = cb >= 16 ? 1.0 : cb >= 8 ? 1.55 : cb >= 4 ? 2.5 : cb >= 2 ? 4.0 : 6.0;
  const int lgn = ilog2(nseq);
  const int estep = nth >> lgn;
  double warps = 0;
  for (int i = 0; i < pl.nf; ++i) {
    const int ppt = wide ? 13 : 8;  // points per thread of the tile (c2r.cu: TILE / NTH, or kWide / 512)
    const int r = pl.f[i], Rr = R / r, MB = (ppt + r - 1) / r;
    for (int b = 0; b < MB; ++b)
      for (int w = 0; w < nth / 32; ++w) {
        const int e0min = (32 * w) >> lgn;
        if (e0min + b * estep < Rr) warps += 1;
      }
  }
  // a big second pass runs one 512-thread CTA per SM against three 256-thread ones: measured
  // slower than the model's rounds say (c5 block 1: 432-point big pass 1.17 ms vs 216-point pass
  // 0.96 ms), hence the occupancy factor 1.7
  const double occ = (mode == 1 && big) ? 1.7 : 1.0;
  return warps * 32.0 / ((double)R * nseq) * pen * occ * (c2r_has_spec(mode, R) ? 1.0 : 1.4);
}

xc_status fft_plan_make(FftPlan& p, int L, bool c2r) {
  p.L = L;
  if (L <= 512) {
    p.L1 = L;
    p.L2 = 1;
  } else {
    int best = -1;
    // XC_C2R_SPLIT="M:L1[,M:L1...]" forces the split of the listed C2R lengths (measurement switch)
    static const char* forced = getenv("XC_C2R_SPLIT");
    if (c2r && forced) {
      const char* q = forced;
      while (*q) {
        int m = 0, l1 = 0;
        if (sscanf(q, "%d:%d", &m, &l1) == 2 && m == L && l1 > 1 && L % l1 == 0) best = l1;
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    }
    if (c2r && best < 0) {  // the split with the cheapest pair of C2R passes (first pass pairs sub-sequences)
      double bc = 1e30;
      // first pass (paired sub-sequences) <= 256 points, second <= 512: every M up to 131072
      // splits (c5 at N = 131072: M = 86400 = 200 x 432, both passes on 128-B tile rows)
      for (int d = 2; d <= 256; ++d) {
        if (L % d || L / d > 512) continue;
        const double c = c2r_pass_cost(d, 2, 0) + c2r_pass_cost(L / d, 1, 1);
        if (c < bc - 1e-9) {
          bc = c;
          best = d;
        }
      }
    }
    if (best < 0)
      for (int d = 2; (int64_t)d * d <= L; ++d)
        if (L % d == 0) best = d;
    if (best < 0 || L / best > 1024) {
      xc_set_error("fft: length " + std::to_string(L) + " not splittable into two factors <= 1024");
      return XC_EUNSUPPORTED;
    }
    p.L1 = best;
    p.L2 = L / best;
  }
  factorize(p.L1, p.nf1, p.f1);
  factorize(p.L2, p.nf2, p.f2);
  if (p.nf1 < 0 || p.nf2 < 0) {
    xc_set_error("fft: length " + std::to_string(L) + " is not 2-3-5-smooth");
    return XC_EUNSUPPORTED;
  }
  std::vector<double2> t1, t2, tL;
  twiddle_table(p.L1, t1);
  twiddle_table(p.L2, t2);
  if (p.L2 > 1) twiddle_table(L, tL);
  size_t bytes = (t1.size() + t2.size() + tL.size()) * sizeof(double2);
  XC_TRY(dev_alloc(p.mem, bytes));
  double2* base = (double2*)p.mem.p;
  p.tw1 = base;
  p.tw2 = base + t1.size();
  p.twL = tL.empty() ? nullptr : base + t1.size() + t2.size();
  XC_CUDA(cudaMemcpy(p.tw1, t1.data(), t1.size() * sizeof(double2), cudaMemcpyHostToDevice));
  XC_CUDA(cudaMemcpy(p.tw2, t2.data(), t2.size() * sizeof(double2), cudaMemcpyHostToDevice));
  if (!tL.empty()) XC_CUDA(cudaMemcpy(p.twL, tL.data(), tL.size() * sizeof(double2), cudaMemcpyHostToDevice));
  return XC_OK;
}

void fft_plan_free(FftPlan& p) { dev_free(p.mem); }

xc_status fft_run(const FftPlan& p, int sigma, FftPro pro, FftEpi epi, const FftIO& io, int ncol,
                  double2* scratch, cudaStream_t st) {
  PassArgs a{};
  a.L = p.L;
  a.L1 = p.L1;
  a.L2 = p.L2;
  a.ncol = ncol;
  a.scratch = scratch;
  a.twL = p.twL;
  if (pro != PRO_PLAIN && pro != PRO_XREAL && pro != PRO_XCPLX) {
    xc_set_error("fft_run: the output-axis inverse runs in c2r_run");
    return XC_EINVAL;
  }
  if (p.L2 == 1) {
    a.R = p.L1;
    set_stages(a, p.nf1, p.f1);
    a.tw = p.tw1;
    a.stage = 2;
    a.S = 1;
    a.sc = 1;
    choose_tile(a.R, ncol, 1, a.cb);
    a.lgcb = ilog2(a.cb);
    a.lgn = a.lgcb;
    return sigma > 0 ? dispatch<1>(pro, epi, a, io, st) : dispatch<-1>(pro, epi, a, io, st);
  }
  if (!scratch) {
    xc_set_error("fft: two-pass length needs scratch");
    return XC_EINVAL;
  }
  // pass 1: L1-point FFTs, L2 sub-sequences per column
  a.R = p.L1;
  set_stages(a, p.nf1, p.f1);
  a.tw = p.tw1;
  a.stage = 0;
  a.S = p.L2;
  a.sc = 1;
  choose_tile(a.R, ncol, a.sc, a.cb);
  {  // spread spare sequences over sub-sequences when there are few columns
    int nseq = a.cb;
    while (nseq < 16 && 2 * nseq * a.R <= kTileElems) nseq *= 2;
    a.sc = nseq / a.cb;
  }
  a.lgcb = ilog2(a.cb);
  a.lgn = ilog2(a.cb * a.sc);
  XC_TRY(sigma > 0 ? dispatch<1>(pro, epi, a, io, st) : dispatch<-1>(pro, epi, a, io, st));
  // pass 2: L2-point FFTs, L1 sub-sequences per column
  a.R = p.L2;
  set_stages(a, p.nf2, p.f2);
  a.tw = p.tw2;
  a.stage = 1;
  a.S = p.L1;
  choose_tile(a.R, ncol, 1, a.cb);
  {
    int nseq = a.cb;
    while (nseq < 16 && 2 * nseq * a.R <= kTileElems) nseq *= 2;
    a.sc = nseq / a.cb;
  }
  a.lgcb = ilog2(a.cb);
  a.lgn = ilog2(a.cb * a.sc);
  return sigma > 0 ? dispatch<1>(pro, epi, a, io, st) : dispatch<-1>(pro, epi, a, io, st);
}
