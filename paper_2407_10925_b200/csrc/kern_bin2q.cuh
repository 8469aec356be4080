#pragma once
// kern_bin2q.cuh -- the binary (sigma = d = 2) two-array sweep on the symmetry-folded ("quarter")
// table: one stored entry per class of states with provably equal values -- orbits of
// {id, complement c, string swap s, psi = c s}, and for same-head states also the tail
// complement t (reading R18) -- 3/16 of the logical states.
//
// Method: identical arithmetic to kern_bin2_tma.cu (Eqs. F1/F0
// PAPER.md:752-779), same tile pairing {t, psi(t)} and the same adv_b windows.  Only the
// storage changes (DESIGN.md §6 "quarter table"):
//
//  * Half-table index space [0, 2^(2l-1)) (a_0 = 0, complement folded, Eq. comp_eq) is cut into
//    blocks of 4^K entries; a block is fixed by its top l-K characters pairs ("prefix").  The
//    residual symmetries of the half table map blocks onto blocks with a digit-wise permutation
//    inside: Q1 blocks (heads 01) pair under psi (pairswap of the complement); Q0 blocks
//    (heads 00) fold under {id, s, t, s t} (s: swap the two bits of every pair; t: complement
//    every tail digit, i.e. reverse the block).  Of each block orbit only the smallest prefix is
//    stored ("canonical", mode 0); the others read it through the permutation (mode 1 = s,
//    2 = psi or s t, 3 = t).  map[block] = (slot << 2) | mode, built by the host.  The string
//    swap W(a,b) = W(b,a) is an exact invariant of every iterate (reading R19), the complement
//    one is Eq. comp_eq, the tail complement of same-head states is v'[00t] = v'[00t~] (R18).
//  * Reads: a tile's adv_b window (2T entries with free low 2M+1 bits) of a mode-0 block is one
//    contiguous run; of a pairswapped block two runs of T (bit 2M+1 <-> bit 2M exchanged),
//    loaded with two bulk copies into the same smem slots; of a tail-complemented block one run
//    read reversed.  The consumer indexes smem through the permutation.  Every half-table
//    window is loaded once, so a stored block is requested once per logical image (twice for
//    Q1 blocks, four times for Q0 blocks).
//  * Item order: the host's L2 schedule (lcsb_api.cu quarter_schedule) lists the tile pairs in
//    waves that share stored blocks, and thread 0 of each CTA claims items in that order from a
//    global counter, so the items in flight stay within about one grid-width of the list and
//    most repeated block loads hit L2.
//  * Writes: of every output run (Q1 tile, Q0 row run, Q0 mirror run) only those lying in a
//    canonical block are stored -- each stored entry is written exactly once.  psi(t)'s outputs
//    equal t's (the pair computes one max for both), so exactly one of the two Q1 runs is
//    written unless the block is psi-fixed; a Q0 row run and its mirror run are t-images, so
//    one of the two is written.
//  => per sweep every logical window of the half table is loaded once (from DRAM ~1.6 x the
//     stored table at l = 17) and 3/8 of the half table is written.
//  * Bound pass (WMODE, reading R21): the same item walk without stores; at every stored
//    output x it reads u[x] (the table the pass reads, = v_n) and v_prev[x] and accumulates
//    R_max = max(u - v_prev), R_min = min(u - v_prev) (Alg. 5 line 7 / PAPER.md:694) and
//    D = min(F(u,u) - u) with F(u,u)[x] in fp64 (not rounded to storage), so one pass gives
//    E = max(0, max W) = max(0, R - D) for both R (W = u + R - F(u,u), PAPER.md:400 with
//    Alg. 5 line 8): the R reduction and the W pass of the old two-pass bound in one read.
//  * Residual storage (RES, reading R24): the table holds a residual e against a fixed fp32 base
//    H (v = H + e + o); every window is loaded from both and added in fp64 (exact), outputs
//    store round((F + shift) - H[x]) and the bound reads H at the outputs too.
//  * fp32 tiles of 4^6 (the config-4/5 default, round 2): bin2q_qp_kernel pipelines the sweep by
//    window quarters (quad tid + 256 q of every thread reads one quarter of each window) with a
//    producer warp, and bin2q_qpw_kernel does the same for the bound pass and the tracking sweep
//    (DIFF, reading R25) with u (and v_prev) at each quarter's outputs staged by TMA; the
//    whole-stage bin2q_kernel remains for the other tiles, fp64 and the A/B knobs.
#include <math.h>
#include <stdlib.h>

// The kernel templates live here; the instantiations are split over four translation units
// (compiled in parallel): kern_bin2q.cu (the sweep), kern_bin2q_bound.cu (the one-pass bound),
// kern_bin2q_ext.cu (the integer-offset and residual-storage sweeps), kern_bin2q_diff.cu (the
// tracking sweep).
#include "lcsb_internal.cuh"
#include "tma.cuh"

namespace lcsbk {
namespace {

__device__ __forceinline__ uint64_t pairswap(uint64_t v) {
  return ((v & 0xAAAAAAAAAAAAAAAAull) >> 1) | ((v & 0x5555555555555555ull) << 1);
}
__device__ __forceinline__ uint32_t pairswap32(uint32_t v) {
  return ((v & 0xAAAAAAAAu) >> 1) | ((v & 0x55555555u) << 1);
}

// Q0 output from one row of 4 in the oracle's summation order (Alg. 3 "SameFirstBit"):
// 1 + max(0, cand) with the z = head option's 0 (reading R3).  The iterates are non-negative
// (v_0 = 0 and F maps non-negative tables to non-negative tables), so cand >= 0 and the max is
// cand itself: the compare is dropped, the value is unchanged.
__device__ __forceinline__ double q0_val(double v0, double v1, double v2, double v3) {
  const double r = ((v0 + v1) + v2) + v3;
#ifdef LCSB_Q0_FMA  // A/B: 0.25 r is exact, so one fused op rounds exactly as DMUL + DADD do
  return __fma_rn(0.25, r, 1.0);
#else
  return 1.0 + 0.25 * r;
#endif
}

constexpr int kThreads = 256;
constexpr uint64_t kNone = ~0ull;
// fp32 bound pass: the register-lean quad order (pair_quads_w32); LCSB_BOUND_WIDE (compile-time,
// A/B only) restores the generic order
#ifndef LCSB_BOUND_WIDE
constexpr bool WLEAN = true;
#else
constexpr bool WLEAN = false;
#endif

// output stores: nothing in a sweep re-reads them, so they are streaming stores (st.global.cs,
// evict-first) that leave L2 to the input windows (A/B at l = 17 fp32: 5.161 -> 5.132 ms;
// LCSB_BIN2Q_NO_STCS builds the plain stores)
template <typename V>
__device__ __forceinline__ void st_out(V* p, V v) {
#ifndef LCSB_BIN2Q_NO_STCS
  __stcs(p, v);
#else
  *p = v;
#endif
}

template <typename T, int M, int S, bool WMODE, int MINB = 1, bool RES = false>
struct QCfg {
  static constexpr uint32_t TT = 1u << (2 * M);  // Q1 outputs per tile
  static constexpr uint32_t WIN = 2 * TT;        // entries per adv_b window
  // the stage holds the item's two windows (RES: of the residual, then of the base); the bound
  // pass reads u and v_prev at the outputs straight from global memory (streaming loads, issued
  // before the window reads)
  static constexpr uint32_t STAGE = 2 * WIN * (RES ? 2 : 1);
  // + the bound pass's next-item map entries (QItem, 32 bytes, fetched by cp.async)
  static constexpr size_t SMEM = (size_t)S * STAGE * sizeof(T) + (size_t)S * sizeof(uint64_t) +
                                 (size_t)S * 8 * sizeof(uint64_t) + (WMODE ? 32 : 0);
};

struct QGeo {
  int K;
  uint64_t q1, lmask, amask, bmask, kmask;
  uint64_t ntiles;  // 4^(l-1-M)
};

__device__ __forceinline__ void qtile(const QGeo& g, uint64_t tau, uint32_t LOG, uint64_t& x0,
                                      uint64_t& p0, uint64_t& taup) {
  x0 = g.q1 + (tau << LOG);
  p0 = pairswap(~x0 & g.lmask) & ~((1ull << LOG) - 1);  // first output of tile psi(tau)
  taup = (p0 - g.q1) >> LOG;
}
__device__ __forceinline__ uint64_t qwin(const QGeo& g, uint64_t x) {  // adv_b window base
  return (x & g.amask) | ((x & g.bmask & ~g.q1) << 2);
}
// stored index of the first entry of a run starting at half-table index s if the run lies in
// a canonical block, else kNone
__device__ __forceinline__ uint64_t qrun(const QGeo& g, uint32_t m, uint64_t s) {
  return (m & 3u) ? kNone : (((uint64_t)(m >> 2) << (2 * g.K)) | (s & g.kmask));
}

// ---- window addressing.  Logical window position w (0 <= w < 2T): bit 2M = the appended b
// character of the tile's top free pair, low 2M bits = the tile's free pairs.  A window loaded
// from a permuted block sits in smem as two runs of T (bit 2M+1 <-> bit 2M exchanged) with the
// pairs inside permuted: mode 1 (s) pairswap, mode 2 (psi) pairswap of the complement.
// A "group" = the 4 logical positions with equal bits >= 2 (the last character pair of the
// window state free); it is 4 consecutive smem entries in every mode, in the order comp<MODE>.
template <uint32_t TT, int MODE>
__device__ __forceinline__ uint32_t gbase(uint32_t g) {  // smem start of the group at logical g
  if (MODE == 0) return g;
  if (MODE == 3) return 2u * TT - 4u - g;  // tail complement: the window reversed
  const uint32_t w = (MODE == 1) ? g : (~(g + 3u) & (2u * TT - 1u));
  return (w & TT) | pairswap32(w & (TT - 1u));
}
template <int MODE>
__device__ __forceinline__ constexpr uint32_t comp(uint32_t d) {  // smem slot of logical digit d
  return MODE == 0 ? d
                   : (MODE == 1 ? (((d & 1u) << 1) | (d >> 1))
                                : (MODE == 3 ? 3u - d : ((((3u - d) & 1u) << 1) | ((3u - d) >> 1))));
}

template <typename T>
__device__ __forceinline__ void ld4(const T* p, double (&v)[4]);
template <>
__device__ __forceinline__ void ld4<float>(const float* p, double (&v)[4]) {
  const float4 f = *reinterpret_cast<const float4*>(p);
  v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
}
template <>
__device__ __forceinline__ void ld4<double>(const double* p, double (&v)[4]) {
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
// raw 4-entry group in the storage type (no widening)
__device__ __forceinline__ void ld4r(const float* p, float (&v)[4]) {
  const float4 f = *reinterpret_cast<const float4*>(p);
  v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
}
__device__ __forceinline__ void sel4f(bool s, const float (&x)[4], const float (&y)[4],
                                      float (&a)[4], float (&b)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = s ? y[k] : x[k];
    b[k] = s ? x[k] : y[k];
  }
}
__device__ __forceinline__ void widen4(const float (&x)[4], double (&v)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = (double)x[k];
}

template <typename T>
__device__ __forceinline__ void st4(T* p, double a, double b, double c, double d);
template <>
__device__ __forceinline__ void st4<float>(float* p, double a, double b, double c, double d) {
  *reinterpret_cast<float4*>(p) = make_float4((float)a, (float)b, (float)c, (float)d);
}
template <>
__device__ __forceinline__ void st4<double>(double* p, double a, double b, double c, double d) {
  reinterpret_cast<double2*>(p)[0] = make_double2(a, b);
  reinterpret_cast<double2*>(p)[1] = make_double2(c, d);
}
__device__ __forceinline__ void sel4(bool s, const double (&x)[4], const double (&y)[4],
                                     double (&a)[4], double (&b)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = s ? y[k] : x[k];
    b[k] = s ? x[k] : y[k];
  }
}
// bound pass accumulators at one stored output: u = v_n[x], p = v_{n-1}[x], f = F(u,u)[x]
// (sweep with integer offsets: rmin = min of the stored values, sh = the shift -c, reading R23)
struct BAcc {
  double rmax, rmin, dmin;
  double sh;
};
__device__ __forceinline__ void bacc(double u, double p, double f, BAcc& b) {
  const double dd = u - p;
  b.rmax = dmax(b.rmax, dd);
  b.rmin = dmin(b.rmin, dd);
  b.dmin = dmin(b.dmin, f - u);
}
// tracking sweep (DIFF): at one stored output, u = the table read (v_{n-1}) there, f = F(u,u) in
// fp64 and st = the stored value (v_n): R of v_n (max / min of v_n - v_{n-1}, the one-pass bound's
// expression) and D of v_{n-1} (min of F(u,u) - u, reading R21)
__device__ __forceinline__ void dacc(double u, double f, double st, BAcc& b) {
  const double dd = st - u;
  b.rmax = dmax(b.rmax, dd);
  b.rmin = dmin(b.rmin, dd);
  b.dmin = dmin(b.dmin, f - u);
}
// streaming 4-entry load in the storage type (widened at use)
__device__ __forceinline__ void ld4s(const float* p, float (&v)[4]) {
  const float4 f = __ldcs(reinterpret_cast<const float4*>(p));
  v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
}
__device__ __forceinline__ void ld4s(const double* p, double (&v)[4]) {
  const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// Each thread takes quads of Q1 outputs o0..o0+3 of tile t (and the same values at psi(t)).
// adv_b pairs of outputs (o0, o0+2) form x-window group A = logical 2 pairswap(o0), (o0+1, o0+3)
// group B = A + 4; in the psi window (o0+3, o0+2) form A' = 2 (T-4-o0), (o0+1, o0) B' = A' + 4.
// Over all quads every group of both windows is loaded exactly once, and a group is also a
// complete Q0 row (Alg. 3): row r = group/4 -> Q0 output r of the window's run and its mirror
// (the complemented tail, row read reversed).  So each window entry is read from smem and
// widened to fp64 once.  The A/B load order alternates across threads so each 128-bit smem load
// is conflict-free (2-way for permuted x windows).
// bound pass (WMODE): src = u = v_n, prev = v_{n-1}; nothing is stored
template <typename T, int MODE, bool WMODE, bool OFS = false, bool RES = false, bool DIFF = false>
__device__ __forceinline__ void q0_group(const double (&G)[4], uint32_t r, uint32_t half_rows,
                                         const T* src, T* dst, uint64_t of, uint64_t om,
                                         const T* prev, BAcc& ba, const T* base = nullptr) {
  const double v0 = G[comp<MODE>(0)], v1 = G[comp<MODE>(1)], v2 = G[comp<MODE>(2)],
               v3 = G[comp<MODE>(3)];
  // a row run and its mirror run are images of each other, so usually only one is stored:
  // each value is formed only when its run is (the branches are uniform per item)
  if (WMODE) {
    const uint32_t rm = half_rows - 1 - r;
    // RES: u = H + e and v_prev = H + e_prev (both exact in fp64)
    if (of != kNone) {
      const double h = RES ? (double)__ldcs(base + of + r) : 0.0;
      bacc(h + (double)__ldcs(src + of + r), prev ? h + (double)__ldcs(prev + of + r) : 0.0,
           q0_val(v0, v1, v2, v3), ba);
    }
    if (om != kNone) {
      const double h = RES ? (double)__ldcs(base + om + rm) : 0.0;
      bacc(h + (double)__ldcs(src + om + rm), prev ? h + (double)__ldcs(prev + om + rm) : 0.0,
           q0_val(v3, v2, v1, v0), ba);
    }
  } else if (DIFF) {  // store round(F), reduce against the table read at the same position
    if (of != kNone) {
      const double f = q0_val(v0, v1, v2, v3);
      const T st = (T)f;
      const double u = (double)__ldcs(src + of + r);
      st_out(dst + of + r, st);
      dacc(u, f, (double)st, ba);
    }
    if (om != kNone) {
      const uint32_t rm = half_rows - 1 - r;
      const double f = q0_val(v3, v2, v1, v0);
      const T st = (T)f;
      const double u = (double)__ldcs(src + om + rm);
      st_out(dst + om + rm, st);
      dacc(u, f, (double)st, ba);
    }
  } else if (OFS) {  // store round(F(s) - c) (RES: - H[x]); track the min of s (= H + e)
    if (of != kNone) {
      const double h = RES ? (double)__ldcs(base + of + r) : 0.0;
      const T st = (T)((q0_val(v0, v1, v2, v3) + ba.sh) - h);
      st_out(dst + of + r, st);
      ba.rmin = dmin(ba.rmin, h + (double)st);
    }
    if (om != kNone) {
      const uint32_t rm = half_rows - 1 - r;
      const double h = RES ? (double)__ldcs(base + om + rm) : 0.0;
      const T st = (T)((q0_val(v3, v2, v1, v0) + ba.sh) - h);
      st_out(dst + om + rm, st);
      ba.rmin = dmin(ba.rmin, h + (double)st);
    }
  } else {
    if (of != kNone) st_out(dst + of + r, (T)q0_val(v0, v1, v2, v3));
    if (om != kNone) st_out(dst + om + (half_rows - 1 - r), (T)q0_val(v3, v2, v1, v0));
  }
}

// smem offset of window entry P (the window's smem layout, gbase) inside the quarter buffer of
// the quarter-pipelined sweep (bin2q_qp_kernel): modes 0 / 3 keep contiguous quarters (P's top
// two bits fixed), the pairswapped modes fix bits 12 and 10 of P (two runs of 1024; bit 11 -> 10)
template <uint32_t TT, int MODE>
__device__ __forceinline__ uint32_t qloc(uint32_t P) {
  static_assert(TT == 4096, "quarter buffers for tiles of 4^6");
  if (MODE == 0 || MODE == 3) return P & 2047u;
  return ((P >> 1) & 1024u) | (P & 1023u);
}

// fp32 storage, sweep: one quad of Q1 outputs o0..o0+3 (o0 = 4 qd) of the tile pair, its Q0 rows;
// the Q1 values in fp32 (see the comment inside).  QP: bw / bp are the quarter buffers of the
// quad's quarter (bin2q_qp_kernel) instead of the whole windows.
// an item's stored output runs (meta[1..6]), read once per item into registers (the stores to
// global memory between the quads would otherwise make the compiler re-read them from shared
// memory, as it cannot rule out aliasing)
struct QRuns {
  float *pQ1, *pQ1p, *pf, *pm, *ppf, *ppm;  // run starts in the output table (nullptr: not stored)
};
__device__ __forceinline__ QRuns qruns(const uint64_t* meta, bool self, float* dst) {
  QRuns r;
  auto ptr = [&](uint64_t o) { return o != kNone ? dst + o : nullptr; };
  r.pQ1 = ptr(meta[1]);
  r.pQ1p = ptr(meta[2]);
  r.pf = ptr(meta[3]);
  r.pm = ptr(meta[4]);
  r.ppf = self ? nullptr : ptr(meta[5]);
  r.ppm = self ? nullptr : ptr(meta[6]);
  return r;
}
// the stored Q0 outputs of one row (row run at pf, mirror run at pm), as q0_group's sweep branch
template <uint32_t TT, int MODE>
__device__ __forceinline__ void q0_store_f32(const double (&G)[4], uint32_t r, float* pf,
                                             float* pm) {
  const double v0 = G[comp<MODE>(0)], v1 = G[comp<MODE>(1)], v2 = G[comp<MODE>(2)],
               v3 = G[comp<MODE>(3)];
  if (pf) st_out(pf + r, (float)q0_val(v0, v1, v2, v3));
  if (pm) st_out(pm + (TT / 2 - 1 - r), (float)q0_val(v3, v2, v1, v0));
}

template <typename T, uint32_t TT, int MW, int MP, bool QP = false>
__device__ __forceinline__ void quad_f32(const T* bw, const T* bp, const QRuns& R, uint32_t qd) {
  static_assert(sizeof(T) == 4, "fp32 storage");
  constexpr uint32_t SX = (MW == 0 || MW == 3) ? 2 : 0, SP = (MP == 0 || MP == 3) ? 2 : 1;
  // fp32 storage, sweep: the Q1 value round32(max(0.5 (x0 + x1), 0.5 (y0 + y1))) of fp64
  // arithmetic equals the same expression evaluated in fp32 (a two-term fp32 sum is exact in
  // fp64 or off by less than half an fp32 ulp, so no double rounding; halving and max commute
  // with rounding), so Q1 stays in fp32; only the Q0 rows that are stored widen to fp64 (their
  // four-term sums are not exact in fp32).
  const uint32_t o0 = 4 * qd;
  const uint32_t g = 2 * pairswap32(o0), u = 2 * (TT - 4 - o0);
  auto ax = [&](uint32_t gg) -> uint32_t {
    if constexpr (QP) return qloc<TT, MW>(gbase<TT, MW>(gg));
    else return gbase<TT, MW>(gg);
  };
  auto ap = [&](uint32_t gg) -> uint32_t {
    if constexpr (QP) return qloc<TT, MP>(gbase<TT, MP>(gg));
    else return gbase<TT, MP>(gg);
  };
  // X1 / X2 hold the groups A (row g/4) and B (row g/4 + 1) in a per-thread order (sx: B
  // first) that keeps the 128-bit smem loads conflict-free; the pair sums are formed per loaded
  // group and only they are put back in A/B order (4 selects instead of 8 per window)
  float X1[4], X2[4], P1[4], P2[4];
  const bool sx = (qd >> SX) & 1u, sp = (qd >> SP) & 1u;
  ld4r(reinterpret_cast<const float*>(bw) + ax(sx ? g + 4 : g), X1);
  ld4r(reinterpret_cast<const float*>(bw) + ax(sx ? g : g + 4), X2);
  ld4r(reinterpret_cast<const float*>(bp) + ap(sp ? u + 4 : u), P1);
  ld4r(reinterpret_cast<const float*>(bp) + ap(sp ? u : u + 4), P2);
  constexpr uint32_t c0 = comp<MW>(0), c1 = comp<MW>(1), c2 = comp<MW>(2), c3 = comp<MW>(3);
  constexpr uint32_t d0 = comp<MP>(0), d1 = comp<MP>(1), d2 = comp<MP>(2), d3 = comp<MP>(3);
  const float x1l = 0.5f * (X1[c0] + X1[c1]), x1h = 0.5f * (X1[c2] + X1[c3]);
  const float x2l = 0.5f * (X2[c0] + X2[c1]), x2h = 0.5f * (X2[c2] + X2[c3]);
  const float p1l = 0.5f * (P1[d0] + P1[d1]), p1h = 0.5f * (P1[d2] + P1[d3]);
  const float p2l = 0.5f * (P2[d0] + P2[d1]), p2h = 0.5f * (P2[d2] + P2[d3]);
  // bx = {A lo, B lo, A hi, B hi}; bq = {Bp hi, Bp lo, Ap hi, Ap lo}
  const float bx[4] = {sx ? x2l : x1l, sx ? x1l : x2l, sx ? x2h : x1h, sx ? x1h : x2h};
  const float bq[4] = {sp ? p1h : p2h, sp ? p1l : p2l, sp ? p2h : p1h, sp ? p2l : p1l};
  float v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = fmaxf(bx[k], bq[k]);  // one FMNMX (no NaN, no -0)
  const uint32_t qb = pairswap32(~o0 & (TT - 1) & ~3u);
  if (R.pQ1) st_out(reinterpret_cast<float4*>(R.pQ1 + o0), make_float4(v[0], v[1], v[2], v[3]));
  if (R.pQ1p)
    st_out(reinterpret_cast<float4*>(R.pQ1p + qb), make_float4(v[3], v[1], v[2], v[0]));
  double G[4];
  if (R.pf || R.pm) {  // X1 is row g/4 + sx, X2 row g/4 + 1 - sx
    widen4(X1, G);
    q0_store_f32<TT, MW>(G, (g >> 2) + sx, R.pf, R.pm);
    widen4(X2, G);
    q0_store_f32<TT, MW>(G, (g >> 2) + 1 - sx, R.pf, R.pm);
  }
  if (R.ppf || R.ppm) {
    widen4(P1, G);
    q0_store_f32<TT, MP>(G, (u >> 2) + sp, R.ppf, R.ppm);
    widen4(P2, G);
    q0_store_f32<TT, MP>(G, (u >> 2) + 1 - sp, R.ppf, R.ppm);
  }
}

// fp32 storage, sweep: every quad of the tile pair (the whole windows in the stage)
template <typename T, uint32_t TT, int MW, int MP>
__device__ __forceinline__ void pair_quads_f32(const T* bw, const T* bp, const T* src, T* dst,
                                               const uint64_t* meta, bool self) {
  (void)src;
  const QRuns R = qruns(meta, self, reinterpret_cast<float*>(dst));
  for (uint32_t qd = threadIdx.x; qd < TT / 4; qd += blockDim.x)
    quad_f32<T, TT, MW, MP>(bw, bp, R, qd);
}

// one Q0 row of the fp32 bound pass / tracking sweep (pair_quads_w32), with u (and v_prev) at
// its output loaded up front by the caller: (fu, fpv) at the row run's entry when `of` is stored,
// else (mu, mpv) at the mirror run's (the mirror of row r sits at half - 1 - r).  When both runs
// are stored (tail-complement-fixed blocks) the mirror's entries are read here directly.
template <uint32_t TT, int MODE, bool DIFF>
__device__ __forceinline__ void q0_rows_w(const double (&G)[4], uint32_t r, uint64_t of,
                                          uint64_t om, float fu, float fpv, float mu, float mpv,
                                          const float* src, const float* prev, float* dst,
                                          BAcc& ba) {
  (void)fpv;
  (void)mpv;  // v_prev: unused by the tracking sweep (DIFF)
  const double v0 = G[comp<MODE>(0)], v1 = G[comp<MODE>(1)], v2 = G[comp<MODE>(2)],
               v3 = G[comp<MODE>(3)];
  if (of != kNone) {
    const double f = q0_val(v0, v1, v2, v3);
    if constexpr (DIFF) {
      const float st = (float)f;
      st_out(dst + of + r, st);
      dacc((double)fu, f, (double)st, ba);
    } else {
      bacc((double)fu, prev ? (double)fpv : 0.0, f, ba);
    }
  }
  if (om != kNone) {
    const uint32_t rm = TT / 2 - 1 - r;
    if (of != kNone) {  // both runs stored: the caller loaded the row run's entries
      mu = __ldcs(src + om + rm);
      if constexpr (!DIFF) {
        if (prev) mpv = __ldcs(prev + om + rm);
      }
    }
    const double f = q0_val(v3, v2, v1, v0);
    if constexpr (DIFF) {
      const float st = (float)f;
      st_out(dst + om + rm, st);
      dacc((double)mu, f, (double)st, ba);
    } else {
      bacc((double)mu, prev ? (double)mpv : 0.0, f, ba);
    }
  }
}

// fp32 storage, bound pass: the arithmetic of pair_quads<float, ..., WMODE> (every value and
// every accumulated u, v_prev, F(u,u) identical; max / min are order-free) in an order that keeps
// fewer values live -- the x window's pair sums and Q0 rows are finished before the psi window's
// groups are loaded (the kernel runs at its 80-register cap; the fp64 group arrays of both
// windows held at once spilled to local memory)
// DIFF (the tracking sweep, kern_bin2q_diff.cu): the same walk storing round32(F) at every stored
// output and reducing against u = the table read there (dacc); v_prev is not read
template <uint32_t TT, int MW, int MP, bool DIFF = false>
__device__ __forceinline__ void pair_quads_w32(const float* bw, const float* bp, const float* src,
                                               const uint64_t* meta, bool self, const float* prev,
                                               BAcc& ba, float* dst = nullptr) {
  constexpr uint32_t SX = (MW == 0 || MW == 3) ? 2 : 0, SP = (MP == 0 || MP == 3) ? 2 : 1;
  const uint64_t oQ1 = meta[1], oQ1p = meta[2];
  const uint64_t of = meta[3], om = meta[4], opf = meta[5], opm = meta[6];
  const bool rows_x = of != kNone || om != kNone;
  const bool rows_p = !self && (opf != kNone || opm != kNone);
  const bool rdp = !DIFF && prev;  // v_prev is read (the one-pass bound; not the D-only pass)
  for (uint32_t qd = threadIdx.x; qd < TT / 4; qd += kThreads) {
    const uint32_t o0 = 4 * qd;
    const uint32_t g = 2 * pairswap32(o0), u = 2 * (TT - 4 - o0);
    const uint32_t qb = pairswap32(~o0 & (TT - 1) & ~3u);
    const uint32_t rx = g >> 2, rp = u >> 2;  // the first of the two rows of each window (even)
    // every global load of the quad first, so their latencies overlap each other and the window
    // arithmetic: u and v_prev at the stored Q1 outputs (4 consecutive entries) and at the two
    // rows of each window (2 consecutive entries of the row run, or of the mirror run reversed:
    // mirror of row r at half - 1 - r)
    float uu[4] = {0, 0, 0, 0}, pp[4] = {0, 0, 0, 0};
    const uint64_t q = oQ1 != kNone ? oQ1 + o0 : (oQ1p != kNone ? oQ1p + qb : kNone);
    if (q != kNone) {
      ld4s(src + q, uu);
      if (rdp) ld4s(prev + q, pp);
    }
    const uint64_t xo = of != kNone ? of + rx : (om != kNone ? om + (TT / 2 - 2 - rx) : kNone);
    const uint64_t po = !rows_p ? kNone
                                : (opf != kNone ? opf + rp : opm + (TT / 2 - 2 - rp));
    float2 ux = make_float2(0.f, 0.f), px = ux, up = ux, pq = ux;
    if (xo != kNone) {
      ux = __ldcs(reinterpret_cast<const float2*>(src + xo));
      if (rdp) px = __ldcs(reinterpret_cast<const float2*>(prev + xo));
    }
    if (po != kNone) {
      up = __ldcs(reinterpret_cast<const float2*>(src + po));
      if (rdp) pq = __ldcs(reinterpret_cast<const float2*>(prev + po));
    }
    const bool sx = (qd >> SX) & 1u, sp = (qd >> SP) & 1u;
    constexpr uint32_t c0 = comp<MW>(0), c1 = comp<MW>(1), c2 = comp<MW>(2), c3 = comp<MW>(3);
    constexpr uint32_t d0 = comp<MP>(0), d1 = comp<MP>(1), d2 = comp<MP>(2), d3 = comp<MP>(3);
    double tx[4];
    {
      float X1[4], X2[4], a[4], b[4];
      ld4r(bw + gbase<TT, MW>(sx ? g + 4 : g), X1);
      ld4r(bw + gbase<TT, MW>(sx ? g : g + 4), X2);
      sel4f(sx, X1, X2, a, b);
      tx[0] = (double)a[c0] + (double)a[c1];
      tx[1] = (double)b[c0] + (double)b[c1];
      tx[2] = (double)a[c2] + (double)a[c3];
      tx[3] = (double)b[c2] + (double)b[c3];
      if (rows_x) {
        double G[4];
        widen4(a, G);
        q0_rows_w<TT, MW, DIFF>(G, rx, of, om, ux.x, px.x, ux.y, px.y, src, prev, dst, ba);
        widen4(b, G);
        q0_rows_w<TT, MW, DIFF>(G, rx + 1, of, om, ux.y, px.y, ux.x, px.x, src, prev, dst, ba);
      }
    }
    double tq[4];
    {
      float P1[4], P2[4], ap[4], bq[4];
      ld4r(bp + gbase<TT, MP>(sp ? u + 4 : u), P1);
      ld4r(bp + gbase<TT, MP>(sp ? u : u + 4), P2);
      sel4f(sp, P1, P2, ap, bq);
      tq[0] = (double)bq[d2] + (double)bq[d3];
      tq[1] = (double)bq[d0] + (double)bq[d1];
      tq[2] = (double)ap[d2] + (double)ap[d3];
      tq[3] = (double)ap[d0] + (double)ap[d1];
      if (rows_p) {
        double G[4];
        widen4(ap, G);
        q0_rows_w<TT, MP, DIFF>(G, rp, opf, opm, up.x, pq.x, up.y, pq.y, src, prev, dst, ba);
        widen4(bq, G);
        q0_rows_w<TT, MP, DIFF>(G, rp + 1, opf, opm, up.y, pq.y, up.x, pq.x, src, prev, dst,
                                ba);
      }
    }
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = 0.5 * dmax(tx[k], tq[k]);
    if constexpr (DIFF) {
      float st[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) st[k] = (float)v[k];
      if (oQ1 != kNone)
        st_out(reinterpret_cast<float4*>(dst + oQ1 + o0), make_float4(st[0], st[1], st[2], st[3]));
      if (oQ1p != kNone)
        st_out(reinterpret_cast<float4*>(dst + oQ1p + qb), make_float4(st[3], st[1], st[2], st[0]));
      if (oQ1 != kNone) {
#pragma unroll
        for (int k = 0; k < 4; ++k) dacc((double)uu[k], v[k], (double)st[k], ba);
      } else if (oQ1p != kNone) {
        dacc((double)uu[3], v[0], (double)st[0], ba);
        dacc((double)uu[1], v[1], (double)st[1], ba);
        dacc((double)uu[2], v[2], (double)st[2], ba);
        dacc((double)uu[0], v[3], (double)st[3], ba);
      }
    } else if (oQ1 != kNone) {
#pragma unroll
      for (int k = 0; k < 4; ++k) bacc((double)uu[k], (double)pp[k], v[k], ba);
    } else if (oQ1p != kNone) {
      bacc((double)uu[3], (double)pp[3], v[0], ba);
      bacc((double)uu[1], (double)pp[1], v[1], ba);
      bacc((double)uu[2], (double)pp[2], v[2], ba);
      bacc((double)uu[0], (double)pp[0], v[3], ba);
    }
  }
}

template <typename T, uint32_t TT, int MW, int MP, bool WMODE, int NT = kThreads, int UNR = 1,
          bool OFS = false, bool RES = false, bool DIFF = false>
__device__ __forceinline__ void pair_quads(const T* bw, const T* bp, const T* src, T* dst,
                                           const uint64_t* meta, bool self, const T* prev,
                                           BAcc& ba, const T* base = nullptr) {
  // A/B load order select bits (bank conflicts): modes 0 and 3 (contiguous, possibly reversed)
  // alternate on bit 2, the pairswapped modes on bit 0 (x window) / bit 1 (psi window)
  constexpr uint32_t SX = (MW == 0 || MW == 3) ? 2 : 0, SP = (MP == 0 || MP == 3) ? 2 : 1;
  const uint64_t oQ1 = meta[1], oQ1p = meta[2];
  const uint64_t of = meta[3], om = meta[4], opf = meta[5], opm = meta[6];
  const bool rows_x = of != kNone || om != kNone;
  const bool rows_p = !self && (opf != kNone || opm != kNone);
  // UNR > 1 (bound pass): several quads unrolled, so their global loads of u and v_prev are
  // issued together (more loads in flight per thread)
#pragma unroll UNR
  for (uint32_t qd = threadIdx.x; qd < TT / 4; qd += NT) {
    const uint32_t o0 = 4 * qd;
    const uint32_t g = 2 * pairswap32(o0), u = 2 * (TT - 4 - o0);
    // psi(o0 + k) sits at oQ1p + qb + pairswap(3 - k): the quad reversed as (3, 1, 2, 0)
    const uint32_t qb = pairswap32(~o0 & (TT - 1) & ~3u);
    // bound pass: u and v_prev at the quad's stored Q1 outputs, loaded first (their latency
    // overlaps the window reads and the arithmetic); W(psi x) = W(x), so either copy serves
    T uu[4] = {0, 0, 0, 0}, pp[4] = {0, 0, 0, 0};  // initialised: keeps them out of local memory
    T hq[4] = {0, 0, 0, 0}, hp[4] = {0, 0, 0, 0};  // RES: the base at the Q1 outputs
    if (WMODE || DIFF) {
      const uint64_t q = oQ1 != kNone ? oQ1 + o0 : (oQ1p != kNone ? oQ1p + qb : kNone);
      if (q != kNone) {
        ld4s(src + q, uu);
        if (WMODE && prev) ld4s(prev + q, pp);
        if (RES) ld4s(base + q, hq);
      }
    } else if (RES) {
      if (oQ1 != kNone) ld4s(base + oQ1 + o0, hq);
      if (oQ1p != kNone) ld4s(base + oQ1p + qb, hp);
    }
    double A[4], B[4], Ap[4], Bp[4];
    const bool sx = (qd >> SX) & 1u, sp = (qd >> SP) & 1u;
    if constexpr (sizeof(T) == 4) {  // select the raw floats, then widen (half the selects)
      float X1[4], X2[4], P1[4], P2[4], a[4], b[4], ap[4], bpp[4];
      ld4r(reinterpret_cast<const float*>(bw) + gbase<TT, MW>(sx ? g + 4 : g), X1);
      ld4r(reinterpret_cast<const float*>(bw) + gbase<TT, MW>(sx ? g : g + 4), X2);
      ld4r(reinterpret_cast<const float*>(bp) + gbase<TT, MP>(sp ? u + 4 : u), P1);
      ld4r(reinterpret_cast<const float*>(bp) + gbase<TT, MP>(sp ? u : u + 4), P2);
      sel4f(sx, X1, X2, a, b);
      sel4f(sp, P1, P2, ap, bpp);
      widen4(a, A);
      widen4(b, B);
      widen4(ap, Ap);
      widen4(bpp, Bp);
      if constexpr (RES) {  // + the base's windows (same smem layout, 2 WIN further): H + e
        const float* hw = reinterpret_cast<const float*>(bw) + 2 * 2 * TT;
        const float* hpw = reinterpret_cast<const float*>(bp) + 2 * 2 * TT;
        ld4r(hw + gbase<TT, MW>(sx ? g + 4 : g), X1);
        ld4r(hw + gbase<TT, MW>(sx ? g : g + 4), X2);
        ld4r(hpw + gbase<TT, MP>(sp ? u + 4 : u), P1);
        ld4r(hpw + gbase<TT, MP>(sp ? u : u + 4), P2);
        sel4f(sx, X1, X2, a, b);
        sel4f(sp, P1, P2, ap, bpp);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          A[k] = (double)a[k] + A[k];
          B[k] = (double)b[k] + B[k];
          Ap[k] = (double)ap[k] + Ap[k];
          Bp[k] = (double)bpp[k] + Bp[k];
        }
      }
    } else {
      double X1[4], X2[4], P1[4], P2[4];
      ld4(bw + gbase<TT, MW>(sx ? g + 4 : g), X1);
      ld4(bw + gbase<TT, MW>(sx ? g : g + 4), X2);
      ld4(bp + gbase<TT, MP>(sp ? u + 4 : u), P1);
      ld4(bp + gbase<TT, MP>(sp ? u : u + 4), P2);
      sel4(sx, X1, X2, A, B);
      sel4(sp, P1, P2, Ap, Bp);
    }
    constexpr uint32_t c0 = comp<MW>(0), c1 = comp<MW>(1), c2 = comp<MW>(2), c3 = comp<MW>(3);
    constexpr uint32_t d0 = comp<MP>(0), d1 = comp<MP>(1), d2 = comp<MP>(2), d3 = comp<MP>(3);
    double v[4];
    // adv_b(x) and adv_b(psi x) = adv_a(x), each (g[c=0] + g[c=1]) / 2 in the oracle's order
    // max(s/2, t/2) = max(s, t)/2 exactly (halving is exact and monotone): one multiply per output
    const double tx[4] = {A[c0] + A[c1], B[c0] + B[c1], A[c2] + A[c3], B[c2] + B[c3]};
    const double tq[4] = {Bp[d2] + Bp[d3], Bp[d0] + Bp[d1], Ap[d2] + Ap[d3], Ap[d0] + Ap[d1]};
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = 0.5 * dmax(tx[k], tq[k]);
    if (WMODE) {
      if (oQ1 != kNone) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          bacc((double)hq[k] + (double)uu[k], (double)hq[k] + (double)pp[k], v[k], ba);
      } else if (oQ1p != kNone) {
        bacc((double)hq[3] + (double)uu[3], (double)hq[3] + (double)pp[3], v[0], ba);
        bacc((double)hq[1] + (double)uu[1], (double)hq[1] + (double)pp[1], v[1], ba);
        bacc((double)hq[2] + (double)uu[2], (double)hq[2] + (double)pp[2], v[2], ba);
        bacc((double)hq[0] + (double)uu[0], (double)hq[0] + (double)pp[0], v[3], ba);
      }
    } else if (DIFF) {  // the sweep's stores + R of v_n and D of v_{n-1} against the table read
      const T s0 = (T)v[0], s1 = (T)v[1], s2 = (T)v[2], s3 = (T)v[3];
      if (oQ1 != kNone) st4(dst + oQ1 + o0, (double)s0, (double)s1, (double)s2, (double)s3);
      if (oQ1p != kNone) st4(dst + oQ1p + qb, (double)s3, (double)s1, (double)s2, (double)s0);
      if (oQ1 != kNone) {
        dacc((double)uu[0], v[0], (double)s0, ba);
        dacc((double)uu[1], v[1], (double)s1, ba);
        dacc((double)uu[2], v[2], (double)s2, ba);
        dacc((double)uu[3], v[3], (double)s3, ba);
      } else if (oQ1p != kNone) {  // position j of the psi run holds output (3, 1, 2, 0)[j]
        dacc((double)uu[3], v[0], (double)s0, ba);
        dacc((double)uu[1], v[1], (double)s1, ba);
        dacc((double)uu[2], v[2], (double)s2, ba);
        dacc((double)uu[0], v[3], (double)s3, ba);
      }
    } else if (OFS && RES) {  // round((F(s) - c) - H[x]) at each stored copy; min of H + e
      if (oQ1 != kNone) {
        T st[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          st[k] = (T)((v[k] + ba.sh) - (double)hq[k]);
          ba.rmin = dmin(ba.rmin, (double)hq[k] + (double)st[k]);
        }
        st4(dst + oQ1 + o0, (double)st[0], (double)st[1], (double)st[2], (double)st[3]);
      }
      if (oQ1p != kNone) {  // position j holds output (3, 1, 2, 0)[j]
        const double vv[4] = {v[3], v[1], v[2], v[0]};
        T st[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          st[k] = (T)((vv[k] + ba.sh) - (double)hp[k]);
          ba.rmin = dmin(ba.rmin, (double)hp[k] + (double)st[k]);
        }
        st4(dst + oQ1p + qb, (double)st[0], (double)st[1], (double)st[2], (double)st[3]);
      }
    } else if (OFS) {  // round(F(s) - c) (the shift is an integer: exact before the rounding)
      const T s0 = (T)(v[0] + ba.sh), s1 = (T)(v[1] + ba.sh), s2 = (T)(v[2] + ba.sh),
              s3 = (T)(v[3] + ba.sh);
      if (oQ1 != kNone) st4(dst + oQ1 + o0, (double)s0, (double)s1, (double)s2, (double)s3);
      if (oQ1p != kNone) st4(dst + oQ1p + qb, (double)s3, (double)s1, (double)s2, (double)s0);
      if (oQ1 != kNone || oQ1p != kNone)
        ba.rmin = dmin(ba.rmin, dmin(dmin((double)s0, (double)s1), dmin((double)s2, (double)s3)));
    } else {
      if (oQ1 != kNone) st4(dst + oQ1 + o0, v[0], v[1], v[2], v[3]);
      if (oQ1p != kNone) st4(dst + oQ1p + qb, v[3], v[1], v[2], v[0]);
    }
    // Q0 rows of the four groups
    if (rows_x) {
      q0_group<T, MW, WMODE, OFS, RES, DIFF>(A, g >> 2, TT / 2, src, dst, of, om, prev, ba, base);
      q0_group<T, MW, WMODE, OFS, RES, DIFF>(B, (g >> 2) + 1, TT / 2, src, dst, of, om, prev, ba,
                                              base);
    }
    if (rows_p) {
      q0_group<T, MP, WMODE, OFS, RES, DIFF>(Ap, u >> 2, TT / 2, src, dst, opf, opm, prev, ba,
                                              base);
      q0_group<T, MP, WMODE, OFS, RES, DIFF>(Bp, (u >> 2) + 1, TT / 2, src, dst, opf, opm, prev,
                                              ba, base);
    }
  }
}

// next item >= c (step G) whose tile is the smaller member of its psi pair
__device__ __forceinline__ uint64_t qnext(const QGeo& g, uint64_t c, uint64_t G, uint32_t LOG) {
  while (c < g.ntiles) {
    uint64_t x0, p0, taup;
    qtile(g, c, LOG, x0, p0, taup);
    if (taup >= c) return c;
    c += G;
  }
  return c;
}

// map entries an item needs: windows t, psi t; runs Q1 t, Q1 psi t, rows/mirrors of both windows
struct QItem {
  uint32_t m[8];
};
__device__ __forceinline__ void cp_async4(uint32_t* smem, const uint32_t* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
template <int M, bool ASYNC>
__device__ __forceinline__ void qlookup(const QGeo& g, const uint32_t* __restrict__ map,
                                        uint64_t tau, QItem& it) {
  constexpr uint32_t TT = 1u << (2 * M), LOG = 2 * M;
  uint64_t x0, p0, taup;
  qtile(g, tau, LOG, x0, p0, taup);
  const uint64_t wb = qwin(g, x0), wp = qwin(g, p0);
  const uint64_t yf = wb >> 2, ypf = wp >> 2;
  const int sh = 2 * g.K;
  if constexpr (ASYNC) {
    // straight into shared memory (cp.async; `it` is in shared memory): needed at the next fill
    // only, and no register holds them across the consumer loop in between (qlookup_wait)
    cp_async4(&it.m[0], map + (wb >> sh));
    cp_async4(&it.m[1], map + (wp >> sh));
    cp_async4(&it.m[2], map + (x0 >> sh));
    cp_async4(&it.m[3], map + (p0 >> sh));
    cp_async4(&it.m[4], map + (yf >> sh));
    cp_async4(&it.m[5], map + ((g.q1 - yf - TT / 2) >> sh));
    cp_async4(&it.m[6], map + (ypf >> sh));
    cp_async4(&it.m[7], map + ((g.q1 - ypf - TT / 2) >> sh));
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    it.m[0] = __ldg(map + (wb >> sh));
    it.m[1] = __ldg(map + (wp >> sh));
    it.m[2] = __ldg(map + (x0 >> sh));
    it.m[3] = __ldg(map + (p0 >> sh));
    it.m[4] = __ldg(map + (yf >> sh));
    it.m[5] = __ldg(map + ((g.q1 - yf - TT / 2) >> sh));
    it.m[6] = __ldg(map + (ypf >> sh));
    it.m[7] = __ldg(map + ((g.q1 - ypf - TT / 2) >> sh));
  }
}
__device__ __forceinline__ void qlookup_wait() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Thread 0: bulk-load the two windows of tile pair tau into a stage and record the item's
// metadata: meta[0] = window modes (bits 0-1: window t, 2-3: window psi t, bit 4: self pair),
// meta[1..6] = stored run starts (Q1 t, Q1 psi t, rows t, mirrors t, rows psi t, mirrors psi t;
// kNone = not stored).
template <typename T, int M, bool WMODE = false, bool RES = false, bool DIFF = false>
__device__ __forceinline__ void qissue(const QGeo& g, const QItem& it, uint64_t tau, T* buf,
                                       uint64_t* bar, uint64_t* meta, const T* src,
                                       uint32_t hints, uint64_t keep, const T* prev = nullptr,
                                       const T* base = nullptr) {
  constexpr uint32_t TT = 1u << (2 * M), LOG = 2 * M;
  uint64_t x0, p0, taup;
  qtile(g, tau, LOG, x0, p0, taup);
  const bool self = taup == tau;
  const uint64_t wb = qwin(g, x0), wp = qwin(g, p0);
  const uint64_t yf = wb >> 2, ym = g.q1 - yf - TT / 2, ypf = wp >> 2, ypm = g.q1 - ypf - TT / 2;
  const int sh = 2 * g.K;
  const uint32_t mw = it.m[0], mp = it.m[1];
  meta[0] = (mw & 3u) | ((mp & 3u) << 2) | (self ? 16u : 0u);
  meta[1] = qrun(g, it.m[2], x0);
  meta[2] = self ? kNone : qrun(g, it.m[3], p0);
  meta[3] = qrun(g, it.m[4], yf);
  meta[4] = qrun(g, it.m[5], ym);
  meta[5] = self ? kNone : qrun(g, it.m[6], ypf);
  meta[6] = self ? kNone : qrun(g, it.m[7], ypm);
  mbar_expect_tx(bar, 2 * 2 * TT * (uint32_t)sizeof(T) * (RES ? 2 : 1));
  // bound pass: u and v_prev at the item's stored output runs go to L2 now (bulk prefetch), so
  // the consumers' direct loads of them, one item later, hit L2 (RES: the base there too, in
  // the sweep as well)
  // (tracking sweep, DIFF: the table read at the output runs, likewise)
  if ((WMODE || RES || DIFF) && ((TT / 2) * sizeof(T)) % 16 == 0) {
    const uint64_t q = meta[1] != kNone ? meta[1] : meta[2];
    if (q != kNone) {
      if (WMODE || DIFF) bulk_prefetch_l2(src + q, TT * (uint32_t)sizeof(T));
      if (WMODE && prev) bulk_prefetch_l2(prev + q, TT * (uint32_t)sizeof(T));
      if (RES) bulk_prefetch_l2(base + q, TT * (uint32_t)sizeof(T));
    }
    if (RES && !WMODE && meta[1] != kNone && meta[2] != kNone)
      bulk_prefetch_l2(base + meta[2], TT * (uint32_t)sizeof(T));
#pragma unroll
    for (int k = 3; k < 7; ++k)
      if (meta[k] != kNone) {
        if (WMODE || DIFF) bulk_prefetch_l2(src + meta[k], TT / 2 * (uint32_t)sizeof(T));
        if (WMODE && prev) bulk_prefetch_l2(prev + meta[k], TT / 2 * (uint32_t)sizeof(T));
        if (RES) bulk_prefetch_l2(base + meta[k], TT / 2 * (uint32_t)sizeof(T));
      }
  }
#pragma unroll
  for (int k = 0; k < (RES ? 4 : 2); ++k) {  // RES: k = 2, 3 load the base's windows
    const uint32_t m = (k & 1) ? mp : mw;
    const uint64_t w = (k & 1) ? wp : wb;
    T* dst = buf + k * 2 * TT;
    const T* blk = (k < 2 ? src : base) + ((uint64_t)(m >> 2) << sh);
    const uint64_t e = w & g.kmask;
    // L2 policy per piece (quarter_schedule): reloaded soon -> `keep`, else evict-first
    const uint32_t hb = hints >> (2 * (k & 1));
    const uint64_t pol0 = (hb & 1u) ? keep : kL2EvictFirst, pol1 = (hb & 2u) ? keep : kL2EvictFirst;
    const uint64_t pol01 = (hb & 3u) ? keep : kL2EvictFirst;
    if ((m & 3u) == 0) {
      tma_load_1d_hint(dst, blk + e, 2 * TT * (uint32_t)sizeof(T), bar, pol01);
    } else if ((m & 3u) == 3) {  // tail complement: one contiguous run, read reversed
      tma_load_1d_hint(dst, blk + ((~e & g.kmask) & ~(2ull * TT - 1)), 2 * TT * (uint32_t)sizeof(T),
                       bar, pol01);
    } else {
      const uint64_t f = ((m & 3u) == 1) ? pairswap(e) : pairswap(~e & g.kmask);
      const uint64_t start = (f & ~(4ull * TT - 1)) | (f & TT);
      tma_load_1d_hint(dst, blk + start, TT * (uint32_t)sizeof(T), bar, pol0);
      tma_load_1d_hint(dst + TT, blk + start + 2 * TT, TT * (uint32_t)sizeof(T), bar, pol1);
    }
  }
}

template <typename T, int M, int S, bool WMODE, int MINB = 1, int NT = kThreads, int UNR = 1,
          bool OFS = false, bool RES = false, int DEPTH = 1, bool DIFF = false>
__global__ void __launch_bounds__(NT, MINB) bin2q_kernel(Bin2QArgs a) {
  using C = QCfg<T, M, S, WMODE, MINB, RES>;
  constexpr uint32_t TT = C::TT, WIN = C::WIN;
  constexpr uint32_t LOG = 2 * M;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* in = reinterpret_cast<T*>(smem_raw);  // [S][STAGE]
  uint64_t* bars = reinterpret_cast<uint64_t*>(in + (size_t)S * C::STAGE);
  uint64_t* metas = bars + S;  // [S][8]

  // the geometry comes precomputed in the launch arguments (launch_q): constant-bank operands
  // that ptxas re-reads where needed instead of holding (or spilling) them across the item loop
  QGeo g;
  g.K = a.K;
  g.lmask = a.geo[0];
  g.q1 = a.geo[1];
  g.amask = a.geo[2];
  g.bmask = a.geo[3];
  g.kmask = a.geo[4];
  g.ntiles = a.geo[5];
  const T* src = reinterpret_cast<const T*>(a.src);
  T* dst = reinterpret_cast<T*>(a.dst);
  const uint32_t* map = a.map;
  const int tid = threadIdx.x;
  const uint64_t G = gridDim.x;

  BAcc ba{-INFINITY, INFINITY, INFINITY, 0.0};
  if (OFS) ba.sh = a.ost->shift;
  const T* base = RES ? reinterpret_cast<const T*>(a.base) : nullptr;
  const T* prev = reinterpret_cast<const T*>(a.prev);
  // items: with a schedule, item c is the tile pair of tile sched[c] (c = blockIdx.x + k G);
  // without one, the pair representatives in tile order
  const uint32_t* sched = (a.sched && a.sched_m == M) ? a.sched : nullptr;
  const uint64_t nitems = sched ? a.nitems : g.ntiles;
  // item claims (thread 0): dynamic -- the next index of the shared counter; static -- this
  // CTA's next representative in round-robin order
  unsigned long long* counter = sched ? a.counter : nullptr;
  auto first = [&](uint64_t c) { return sched ? c : qnext(g, c, G, LOG); };
  auto claim = [&](uint64_t prev) -> uint64_t {
    if (counter) return (uint64_t)atomicAdd(counter, 1ull);
    return first(prev == ~0ull ? (uint64_t)blockIdx.x : prev + G);
  };
  auto entry = [&](uint64_t c) -> uint32_t { return sched ? __ldg(sched + c) : (uint32_t)c; };
  // hint bits only come with a schedule; without one every piece keeps the default policy
  const uint64_t keep = (a.l2keep != 0) ? kL2EvictLast : kL2EvictNormal;
  // producer (thread 0); at depth 3 software-pipelined over three items so none of its dependent
  // memory latencies (claim -> schedule entry -> map entries) stalls the CTA: at each fill it
  // issues item pc (map entries in pit), starts pit's loads for p1 (entry e1 loaded a fill
  // earlier), loads the entry of p2 (claimed a fill earlier) and claims the next item
  uint64_t pc = 0, p1 = 0, p2 = 0;
  uint32_t e0 = 0, e1 = 0;
  // DEPTH 3 (sweeps with dynamic claiming) or 1: the claim, the entry and the map lookups of the
  // next item back to back.  Depth 3 pays only where the claim is an atomic (A/B at l = 17: fp32
  // sweep 5.12 -> 5.07-5.10 ms, fp64 12.99 -> 12.56); with static claims (the residual sweep
  // 19.9 -> 21.2) and in the bound pass, which runs at its 80-register cap (10.86 -> 11.95: the
  // extra producer state spills), it costs
  constexpr int depth = DEPTH;
  static_assert(DEPTH == 1 || DEPTH == 3, "producer depth 1 or 3");
  // the next item's map entries (thread 0, qlookup): registers in the sweeps; in shared memory,
  // fetched by cp.async, in the bound pass, which runs at its register cap (A/B at l = 17: bound
  // fp32 10.64 -> 10.21 ms, fp64 20.8 -> 17.3; the sweeps lose 0.3-1 % that way)
  constexpr bool ASYNC = WMODE;
  static_assert(sizeof(QItem) == 32, "QCfg::SMEM reserves 32 bytes");
  QItem pit_r;
  QItem& pit = ASYNC ? *reinterpret_cast<QItem*>(metas + 8 * S) : pit_r;
  auto ent_of = [&](uint64_t c) -> uint32_t { return c < nitems ? entry(c) : 0u; };
  auto tile_e = [&](uint32_t e) -> uint64_t {
    return sched ? (uint64_t)(e & kQTileMask) : (uint64_t)e;
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // a stage either receives an item (meta[7] = 0, TMA completes its phase) or the end marker
  // (meta[7] = 1, a plain arrive completes it); the claims are monotone, so after the first end
  // marker every later stage is an end marker too
  auto fill = [&](int s, T* sbuf) {
    uint64_t* meta = metas + 8 * s;
    if (pc < nitems) {
      meta[7] = 0;
      if constexpr (ASYNC) qlookup_wait();
      qissue<T, M, WMODE, RES, DIFF>(g, pit, tile_e(e0), sbuf, &bars[s], meta, src,
                               sched ? (e0 >> kQHintShift) : 0xFu, keep, prev, base);
      if constexpr (depth == 1) {  // claim, entry and map lookups back to back
        pc = claim(pc);
        e0 = ent_of(pc);
      } else {  // claim two fills ahead, the entry one
        pc = p1;
        e0 = e1;
        p1 = p2;
        e1 = ent_of(p1);
        p2 = claim(p2);
      }
      if (pc < nitems) qlookup<M, ASYNC>(g, map, tile_e(e0), pit);
    } else {
      meta[7] = 1;
      mbar_arrive(&bars[s]);
    }
  };
  if (tid == 0) {
    pc = claim(~0ull);
    if constexpr (depth == 3) {
      p1 = claim(pc);
      p2 = claim(p1);
      e1 = ent_of(p1);
    }
    e0 = ent_of(pc);
    if (pc < nitems) qlookup<M, ASYNC>(g, map, tile_e(e0), pit);
    for (int s = 0; s < S; ++s) fill(s, in + (size_t)s * C::STAGE);
  }

  for (uint32_t i = 0;; ++i) {
    const uint32_t s = i % S;
    const uint32_t parity = (i / S) & 1u;
    T* buf = in + (size_t)s * C::STAGE;
    const uint64_t* meta = metas + 8 * s;
    mbar_wait(&bars[s], parity);
    __syncthreads();
    if (meta[7]) break;  // end marker: no more items for this CTA
    const uint32_t modes = (uint32_t)meta[0];
    const uint32_t mw = modes & 3u, mp = (modes >> 2) & 3u;  // 3 only for Q0 (same-head) blocks
    const bool self = (modes & 16u) != 0;
    const T* bw = buf;
    const T* bp = buf + WIN;
#define LCSB_Q1(MW, MP)                                                            \
  if constexpr (sizeof(T) == 4 && !WMODE && !OFS && !RES && !DIFF)                 \
    pair_quads_f32<T, TT, MW, MP>(bw, bp, src, dst, meta, self);                   \
  else if constexpr (sizeof(T) == 4 && (WMODE || DIFF) && !RES && NT == kThreads && UNR == 1 && WLEAN) \
    pair_quads_w32<TT, MW, MP, DIFF>(reinterpret_cast<const float*>(bw),           \
                                     reinterpret_cast<const float*>(bp),           \
                                     reinterpret_cast<const float*>(src), meta, self, \
                                     reinterpret_cast<const float*>(prev), ba,     \
                                     reinterpret_cast<float*>(dst));               \
  else                                                                             \
    pair_quads<T, TT, MW, MP, WMODE, NT, UNR, OFS, RES, DIFF>(bw, bp, src, dst, meta, self, prev, \
                                                              ba, base)
    switch (mw * 4 + mp) {
      case 0: LCSB_Q1(0, 0); break;
      case 1: LCSB_Q1(0, 1); break;
      case 2: LCSB_Q1(0, 2); break;
      case 3: LCSB_Q1(0, 3); break;
      case 4: LCSB_Q1(1, 0); break;
      case 5: LCSB_Q1(1, 1); break;
      case 6: LCSB_Q1(1, 2); break;
      case 7: LCSB_Q1(1, 3); break;
      case 8: LCSB_Q1(2, 0); break;
      case 9: LCSB_Q1(2, 1); break;
      case 10: LCSB_Q1(2, 2); break;
      case 11: LCSB_Q1(2, 3); break;
      case 12: LCSB_Q1(3, 0); break;
      case 13: LCSB_Q1(3, 1); break;
      case 14: LCSB_Q1(3, 2); break;
      default: LCSB_Q1(3, 3); break;
    }
#undef LCSB_Q1
    __syncthreads();  // stage s (data and metadata) is free again
    if (tid == 0) fill((int)s, buf);
  }
  if (WMODE || DIFF) block_red3_to(ba.rmax, ba.rmin, ba.dmin, a.red_out);
  if (OFS && !WMODE) block_min_to(ba.rmin, a.omin);
}

// ---- quarter-pipelined fp32 sweep (tiles of 4^6, round 2).  In bin2q_kernel a CTA's single
// 64 KB stage is refilled only after all four of its quads per thread are done, so each CTA
// alternates between waiting for its windows and computing; when the SM clock drops (the board's
// power cap) the computing share grows and fewer bytes are in flight.  Here the
// stage is four 16 KB quarter buffers: quad qd = tid + 256 q of every thread reads only logical
// quarter swap2(q) of the x window and quarter 3 - q of the psi window (g = 2 pairswap(4 qd),
// u = 2 (TT - 4 - 4 qd)), so quarter q of the NEXT item is loaded as soon as all threads are past
// quad q of the current one -- loads stay in flight while the CTA computes.  Values, stores and
// item order are those of bin2q_kernel (bit-identical tables).
struct QPGeo {
  static constexpr uint32_t TT = 4096, Q = 2048;  // Q1 outputs per tile; entries per window quarter
};
// thread 0: the global start of a window's loaded layout (qissue's TMA sources)
__device__ __forceinline__ const float* qp_wstart(const QGeo& g, const float* src, uint32_t m,
                                                  uint64_t w) {
  constexpr uint64_t TT = QPGeo::TT;
  const float* blk = src + ((uint64_t)(m >> 2) << (2 * g.K));
  const uint64_t e = w & g.kmask;
  if ((m & 3u) == 0) return blk + e;
  if ((m & 3u) == 3u) return blk + ((~e & g.kmask) & ~(2 * TT - 1));
  const uint64_t f = ((m & 3u) == 1u) ? pairswap(e) : pairswap(~e & g.kmask);
  return blk + ((f & ~(4 * TT - 1)) | (f & TT));
}
// thread 0: logical quarter L of one window (mode m, loaded layout starting at gs) into its
// quarter buffer (qloc's layout): modes 0 / 3 one contiguous 8 KB run (mode 3 reversed: physical
// quarter 3 - L); pairswapped modes two 4 KB runs (physical bits 12 and 10 fixed)
__device__ __forceinline__ void qp_issue_win(float* dst, const float* gs, uint32_t m, uint32_t L,
                                             uint64_t* bar) {
  constexpr uint32_t TT = QPGeo::TT, Q = QPGeo::Q;
  if (m == 0u) {
    tma_load_1d(dst, gs + (size_t)Q * L, Q * 4u, bar);
  } else if (m == 3u) {
    tma_load_1d(dst, gs + (size_t)Q * (3u - L), Q * 4u, bar);
  } else {
    const uint32_t Lw = (m == 1u) ? L : 3u - L;  // psi reads w = ~(g + 3): quarter 3 - L
    const float* b = gs + (size_t)(Lw >> 1) * 2 * TT + (Lw & 1u) * 1024u;
    tma_load_1d(dst, b, 1024u * 4u, bar);
    tma_load_1d(dst + 1024, b + 2048, 1024u * 4u, bar);
  }
}
constexpr int kQPMeta = 10;  // per item: [0] modes, [1..6] runs, [7] end, [8] / [9] window starts

// The producer side shared by bin2q_qp_kernel and bin2q_qpw_kernel (one lane of the producer
// warp): item claims as bin2q_kernel (the L2 schedule with the dynamic work counter, else static
// round robin), pipelined DEPTH deep (3: claim two items ahead, load the schedule entry one
// ahead), and each item's metadata -- modes, stored output runs, window starts -- from the map
// entries requested one item earlier.
template <int DEPTH>
struct QPItems {
  static constexpr int M = 6;
  static constexpr uint32_t TT = QPGeo::TT, LOG = 2 * M;
  QGeo g;
  const float* src;
  const uint32_t* map;
  const uint32_t* sched;
  unsigned long long* counter;
  uint64_t nitems, G;
  uint64_t pc = 0, p1 = 0, p2 = 0;
  uint32_t e0 = 0, e1 = 0;
  QItem pit;
  __device__ explicit QPItems(const Bin2QArgs& a) {
    g.K = a.K;
    g.lmask = a.geo[0];
    g.q1 = a.geo[1];
    g.amask = a.geo[2];
    g.bmask = a.geo[3];
    g.kmask = a.geo[4];
    g.ntiles = a.geo[5];
    src = reinterpret_cast<const float*>(a.src);
    map = a.map;
    sched = (a.sched && a.sched_m == M) ? a.sched : nullptr;
    nitems = sched ? a.nitems : g.ntiles;
    counter = sched ? a.counter : nullptr;
    G = gridDim.x;
  }
  __device__ uint64_t claim(uint64_t prev) {
    if (counter) return (uint64_t)atomicAdd(counter, 1ull);
    const uint64_t c = prev == ~0ull ? (uint64_t)blockIdx.x : prev + G;
    return sched ? c : qnext(g, c, G, LOG);
  }
  __device__ uint32_t ent_of(uint64_t c) const {
    return c < nitems ? (sched ? __ldg(sched + c) : (uint32_t)c) : 0u;
  }
  __device__ uint64_t tile_e(uint32_t e) const {
    return sched ? (uint64_t)(e & kQTileMask) : (uint64_t)e;
  }
  __device__ void start() {
    pc = claim(~0ull);
    if constexpr (DEPTH == 3) {
      p1 = claim(pc);
      p2 = claim(p1);
      e1 = ent_of(p1);
    }
    e0 = ent_of(pc);
    if (pc < nitems) qlookup<M, false>(g, map, tile_e(e0), pit);
  }
  // the metadata of item pc into meta (false and the end marker when no item is left), then
  // the pipeline moves on and the map entries of the new pc are requested
  __device__ bool prep(uint64_t* meta) {
    if (pc >= nitems) {
      meta[7] = 1;
      return false;
    }
    const uint64_t tau = tile_e(e0);
    uint64_t x0, p0, taup;
    qtile(g, tau, LOG, x0, p0, taup);
    const bool self = taup == tau;
    const uint64_t wb = qwin(g, x0), wp = qwin(g, p0);
    const uint64_t yf = wb >> 2, ym = g.q1 - yf - TT / 2, ypf = wp >> 2, ypm = g.q1 - ypf - TT / 2;
    meta[0] = (pit.m[0] & 3u) | ((pit.m[1] & 3u) << 2) | (self ? 16u : 0u);
    meta[1] = qrun(g, pit.m[2], x0);
    meta[2] = self ? kNone : qrun(g, pit.m[3], p0);
    meta[3] = qrun(g, pit.m[4], yf);
    meta[4] = qrun(g, pit.m[5], ym);
    meta[5] = self ? kNone : qrun(g, pit.m[6], ypf);
    meta[6] = self ? kNone : qrun(g, pit.m[7], ypm);
    meta[7] = 0;
    meta[8] = reinterpret_cast<uint64_t>(qp_wstart(g, src, pit.m[0], wb));
    meta[9] = reinterpret_cast<uint64_t>(qp_wstart(g, src, pit.m[1], wp));
    if constexpr (DEPTH == 1) {
      pc = claim(pc);
      e0 = ent_of(pc);
    } else {
      pc = p1;
      e0 = e1;
      p1 = p2;
      e1 = ent_of(p1);
      p2 = claim(p2);
    }
    if (pc < nitems) qlookup<M, false>(g, map, tile_e(e0), pit);
    return true;
  }
};

// LCSB_QP_SPIN (A/B): plain probe loops instead of the suspend-hint waits
#ifdef LCSB_QP_SPIN
#define QP_WAIT mbar_wait
#else
#define QP_WAIT mbar_wait_sleep
#endif
// consumer threads of bin2q_qp_kernel (LCSB_QP_CONSUMERS, compile-time A/B: 128 = four warps
// with two quads per thread per quarter)
#ifndef LCSB_QP_CONSUMERS
#define LCSB_QP_CONSUMERS 256
#endif
constexpr int kQPC = LCSB_QP_CONSUMERS;
static_assert(kThreads % kQPC == 0 && kQPC % 32 == 0, "consumer threads");
// the consumer side of one item of bin2q_qp_kernel: its four quarters in order, each after its
// buffer has landed (full[q]); each warp then releases the buffer (empty[q])
template <int MW, int MP>
__device__ __forceinline__ void qp_item(const float* qbuf, uint64_t* full, uint64_t* empty,
                                        uint32_t parity, const float* src, float* dst,
                                        const uint64_t* meta, bool self, uint32_t tid, int lane) {
  constexpr uint32_t TT = QPGeo::TT, Q = QPGeo::Q;
  (void)src;
  const QRuns R = qruns(meta, self, dst);
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    if (q) QP_WAIT(&full[q], parity);
    const float* bw = qbuf + (size_t)(2 * q) * Q;
#pragma unroll 1
    for (uint32_t j = 0; j < (uint32_t)(kThreads / kQPC); ++j)
      quad_f32<float, TT, MW, MP, true>(bw, bw + Q, R, tid + kQPC * j + kThreads * (uint32_t)q);
    __syncwarp();  // the warp's reads of buffer q are done
    if (lane == 0) mbar_arrive(&empty[q]);
  }
}

// warp-specialised: warps 0-7 consume (one quad per thread per quarter), warp 8 (one lane)
// produces -- it waits on empty[q] (all 8 consumer warps past quarter q of the previous item)
// and refills buffer q with the next item's quarter, so no CTA-wide barrier stalls the loop
constexpr int kQPThreads = kQPC + 32;
template <int DEPTH>
__global__ void __launch_bounds__(kQPThreads, 3) bin2q_qp_kernel(Bin2QArgs a) {
  constexpr int M = 6;
  constexpr uint32_t TT = QPGeo::TT, Q = QPGeo::Q;
  static_assert(TT == (1u << (2 * M)) && TT / 4 == 4 * kThreads, "256 quads per quarter");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* qbuf = reinterpret_cast<float*>(smem_raw);  // [quarter][x / psi][Q]
  uint64_t* bars = reinterpret_cast<uint64_t*>(qbuf + 8 * Q);  // full[4]
  uint64_t* empty = bars + 4;                                  // empty[4]
  uint64_t* metas = empty + 4;                                 // [2][kQPMeta]
  float* dst = reinterpret_cast<float*>(a.dst);
  const float* src = reinterpret_cast<const float*>(a.src);
  const int tid = threadIdx.x;
  // thread 0: quarter q of the item in `slot` (or a plain arrive after the last item)
  auto issue = [&](int q, int slot) {
    const uint64_t* meta = metas + kQPMeta * slot;
    if (meta[7]) {
      mbar_arrive(&bars[q]);
      return;
    }
    const uint32_t modes = (uint32_t)meta[0];
    mbar_expect_tx(&bars[q], 2u * Q * 4u);
    const uint32_t sq = ((q & 1) << 1) | (q >> 1);  // x window: logical quarter swap2(q)
    qp_issue_win(qbuf + (size_t)(2 * q) * Q, reinterpret_cast<const float*>(meta[8]), modes & 3u,
                 sq, &bars[q]);
    qp_issue_win(qbuf + (size_t)(2 * q + 1) * Q, reinterpret_cast<const float*>(meta[9]),
                 (modes >> 2) & 3u, 3u - (uint32_t)q, &bars[q]);
  };
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) {
      mbar_init(&bars[q], 1);
      mbar_init(&empty[q], kQPC / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= kQPC) {  // the producer warp
    if (tid != kQPC) return;
    QPItems<DEPTH> P(a);
    P.start();
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i & 1u);
      // buffer q and meta slot `slot` are free once every consumer warp is past quarter q of
      // item i - 1 (for q = 0 that also means past item i - 2, the slot's previous item)
      if (i) QP_WAIT(&empty[0], (i - 1) & 1u);
      const bool end = !P.prep(metas + kQPMeta * slot);
      issue(0, slot);
      if (end) return;  // the consumers stop at this item's quarter 0
      for (int q = 1; q < 4; ++q) {
        if (i) QP_WAIT(&empty[q], (i - 1) & 1u);
        issue(q, slot);
      }
    }
  }
  const int lane = tid & 31;
  for (uint32_t i = 0;; ++i) {
    const int slot = (int)(i & 1u);
    const uint64_t* meta = metas + kQPMeta * slot;
    QP_WAIT(&bars[0], i & 1u);
    if (meta[7]) break;  // end marker: no more items for this CTA
    const uint32_t modes = (uint32_t)meta[0];
    const uint32_t mw = modes & 3u, mp = (modes >> 2) & 3u;
    const bool self = (modes & 16u) != 0;
    // one (mode x mode) code path per item: the quarter loop runs inside it (dispatching per
    // quarter through the jump table stalled the warps on instruction fetch)
#define LCSB_QP(MW, MP) \
  qp_item<MW, MP>(qbuf, bars, empty, i & 1u, src, dst, meta, self, (uint32_t)tid, lane)
    switch (mw * 4 + mp) {
      case 0: LCSB_QP(0, 0); break;
      case 1: LCSB_QP(0, 1); break;
      case 2: LCSB_QP(0, 2); break;
      case 3: LCSB_QP(0, 3); break;
      case 4: LCSB_QP(1, 0); break;
      case 5: LCSB_QP(1, 1); break;
      case 6: LCSB_QP(1, 2); break;
      case 7: LCSB_QP(1, 3); break;
      case 8: LCSB_QP(2, 0); break;
      case 9: LCSB_QP(2, 1); break;
      case 10: LCSB_QP(2, 2); break;
      case 11: LCSB_QP(2, 3); break;
      case 12: LCSB_QP(3, 0); break;
      case 13: LCSB_QP(3, 1); break;
      case 14: LCSB_QP(3, 2); break;
      default: LCSB_QP(3, 3); break;
    }
#undef LCSB_QP
  }
}

// ---- staged, quarter-pipelined fp32 bound pass (tiles of 4^6, round 2).  The one-pass bound
// (reading R21) of bin2q_kernel<..., WMODE> reads u and v_prev at every stored output with direct
// loads; they make it long-scoreboard bound.  Here every quarter-step of an item (the quarter
// buffers of bin2q_qp_kernel) also carries, staged by TMA, u and v_prev at the quarter's outputs:
// the Q1 outputs of quads tid + 256 q are one contiguous 1024-entry range of the stored Q1 run
// (quarter q of t's run, or quarter swap2(3 - q) of psi(t)'s), the x window's rows one
// 512-entry range of the row run (quarter swap2(q); mirror run: quarter 3 - swap2(q)) and the
// psi window's likewise (quarter 3 - q).  A quarter-step buffer is 32 KB (windows 16 KB, u and
// v_prev 8 KB each), two per CTA; a producer warp refills them.  Same arithmetic and reductions
// as the direct-load pass (bit-identical R, D).
constexpr uint32_t kQWBuf = 8192;  // floats per quarter-step buffer
// One quad of the staged bound pass (round 2), in two parts: the (mode x mode)-specific window
// loads, the groups put into logical order (register renaming), and one mode-independent part
// for the fp64 arithmetic of quad_w32 (pair_quads_w32), the staged u / v_prev (the quarter's
// [Q1 1024 | x rows 512 | psi rows 512]) and the reductions, shared by the sixteen combinations
// (sixteen full copies of the whole quad kept ~30 % of the warps waiting on instruction fetch).
// DF (the tracking sweep of reading R25): store round32(F) at every stored output and reduce
// against the staged u (dacc), as quad_w32<..., DIFF>; v_prev is not read.
template <int MW, int MP>
__device__ __forceinline__ void wq_load(const float* bw, const float* bp, uint32_t qd,
                                        float (&a)[4], float (&b)[4], float (&ap)[4],
                                        float (&bq)[4]) {
  constexpr uint32_t TT = QPGeo::TT;
  constexpr uint32_t SX = (MW == 0 || MW == 3) ? 2 : 0, SP = (MP == 0 || MP == 3) ? 2 : 1;
  const uint32_t o0 = 4 * qd;
  const uint32_t g = 2 * pairswap32(o0), u = 2 * (TT - 4 - o0);
  const bool sx = (qd >> SX) & 1u, sp = (qd >> SP) & 1u;
  float X1[4], X2[4], P1[4], P2[4], A[4], B[4], Ap[4], Bp[4];
  ld4r(bw + qloc<TT, MW>(gbase<TT, MW>(sx ? g + 4 : g)), X1);
  ld4r(bw + qloc<TT, MW>(gbase<TT, MW>(sx ? g : g + 4)), X2);
  ld4r(bp + qloc<TT, MP>(gbase<TT, MP>(sp ? u + 4 : u)), P1);
  ld4r(bp + qloc<TT, MP>(gbase<TT, MP>(sp ? u : u + 4)), P2);
  sel4f(sx, X1, X2, A, B);
  sel4f(sp, P1, P2, Ap, Bp);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = A[comp<MW>(k)];
    b[k] = B[comp<MW>(k)];
    ap[k] = Ap[comp<MP>(k)];
    bq[k] = Bp[comp<MP>(k)];
  }
}
// the mode-independent part on logical-order groups
template <bool DF>
__device__ __forceinline__ void wq_common(const float (&a)[4], const float (&b)[4],
                                          const float (&ap)[4], const float (&bq)[4],
                                          const float* su, const float* spv,
                                          const uint64_t* meta, bool self, const float* src,
                                          const float* prev, BAcc& ba, uint32_t qd, float* dst) {
  constexpr uint32_t TT = QPGeo::TT;
  const uint64_t oQ1 = meta[1], oQ1p = meta[2];
  const uint64_t of = meta[3], om = meta[4], opf = meta[5], opm = meta[6];
  const bool rows_x = of != kNone || om != kNone;
  const bool rows_p = !self && (opf != kNone || opm != kNone);
  const bool rdp = prev != nullptr;
  const uint32_t o0 = 4 * qd;
  const uint32_t g = 2 * pairswap32(o0), u = 2 * (TT - 4 - o0);
  const uint32_t qb = pairswap32(~o0 & (TT - 1) & ~3u);
  const uint32_t rx = g >> 2, rp = u >> 2;
  double tx[4];
  tx[0] = (double)a[0] + (double)a[1];
  tx[1] = (double)b[0] + (double)b[1];
  tx[2] = (double)a[2] + (double)a[3];
  tx[3] = (double)b[2] + (double)b[3];
  if (rows_x) {
    const uint32_t xi = of != kNone ? (rx & 511u) : (510u - (rx & 511u));
    const float2 ux = *reinterpret_cast<const float2*>(su + 1024 + xi);
    const float2 px = rdp ? *reinterpret_cast<const float2*>(spv + 1024 + xi) : make_float2(0.f, 0.f);
    double G[4];
    widen4(a, G);
    q0_rows_w<TT, 0, DF>(G, rx, of, om, ux.x, px.x, ux.y, px.y, src, prev, dst, ba);
    widen4(b, G);
    q0_rows_w<TT, 0, DF>(G, rx + 1, of, om, ux.y, px.y, ux.x, px.x, src, prev, dst, ba);
  }
  double tq[4];
  tq[0] = (double)bq[2] + (double)bq[3];
  tq[1] = (double)bq[0] + (double)bq[1];
  tq[2] = (double)ap[2] + (double)ap[3];
  tq[3] = (double)ap[0] + (double)ap[1];
  if (rows_p) {
    const uint32_t pi = opf != kNone ? (rp & 511u) : (510u - (rp & 511u));
    const float2 up = *reinterpret_cast<const float2*>(su + 1536 + pi);
    const float2 pq = rdp ? *reinterpret_cast<const float2*>(spv + 1536 + pi) : make_float2(0.f, 0.f);
    double G[4];
    widen4(ap, G);
    q0_rows_w<TT, 0, DF>(G, rp, opf, opm, up.x, pq.x, up.y, pq.y, src, prev, dst, ba);
    widen4(bq, G);
    q0_rows_w<TT, 0, DF>(G, rp + 1, opf, opm, up.y, pq.y, up.x, pq.x, src, prev, dst, ba);
  }
  double v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = 0.5 * dmax(tx[k], tq[k]);
  if (oQ1 != kNone || oQ1p != kNone) {
    const uint32_t qi = oQ1 != kNone ? (o0 & 1023u) : (qb & 1023u);
    float uu[4], pp[4] = {0, 0, 0, 0};
    ld4r(su + qi, uu);
    if (rdp) ld4r(spv + qi, pp);
    if constexpr (DF) {
      float st[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) st[k] = (float)v[k];
      if (oQ1 != kNone)
        st_out(reinterpret_cast<float4*>(dst + oQ1 + o0), make_float4(st[0], st[1], st[2], st[3]));
      if (oQ1p != kNone)
        st_out(reinterpret_cast<float4*>(dst + oQ1p + qb), make_float4(st[3], st[1], st[2], st[0]));
      if (oQ1 != kNone) {
#pragma unroll
        for (int k = 0; k < 4; ++k) dacc((double)uu[k], v[k], (double)st[k], ba);
      } else {
        dacc((double)uu[3], v[0], (double)st[0], ba);
        dacc((double)uu[1], v[1], (double)st[1], ba);
        dacc((double)uu[2], v[2], (double)st[2], ba);
        dacc((double)uu[0], v[3], (double)st[3], ba);
      }
      return;
    }
    if (oQ1 != kNone) {
#pragma unroll
      for (int k = 0; k < 4; ++k) bacc((double)uu[k], (double)pp[k], v[k], ba);
    } else {
      bacc((double)uu[3], (double)pp[3], v[0], ba);
      bacc((double)uu[1], (double)pp[1], v[1], ba);
      bacc((double)uu[2], (double)pp[2], v[2], ba);
      bacc((double)uu[0], (double)pp[0], v[3], ba);
    }
  }
}

constexpr int kQPWThreads = kThreads + 32;  // the bound pass: 8 consumer warps + the producer
template <int DEPTH, bool DF>
__global__ void __launch_bounds__(kQPWThreads, 3) bin2q_qpw_kernel(Bin2QArgs a) {
  constexpr uint32_t Q = QPGeo::Q;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* qbuf = reinterpret_cast<float*>(smem_raw);  // [2][kQWBuf]
  uint64_t* bars = reinterpret_cast<uint64_t*>(qbuf + 2 * kQWBuf);  // full[2]
  uint64_t* empty = bars + 2;                                        // empty[2]
  uint64_t* metas = empty + 2;                                       // [2][kQPMeta]
  __shared__ double r0[8], r1[8], r2[8];
  const float* src = reinterpret_cast<const float*>(a.src);
  // DF (tracking sweep): the table read is staged at the outputs, v_prev is not read, the new
  // values go to dst
  const float* prev = DF ? nullptr : reinterpret_cast<const float*>(a.prev);
  float* dst = DF ? reinterpret_cast<float*>(a.dst) : nullptr;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[b], 1);
      mbar_init(&empty[b], kThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= kThreads) {  // the producer warp (one lane)
    if (tid != kThreads) return;
    QPItems<DEPTH> P(a);
    P.start();
    for (uint64_t k = 0;; ++k) {
      const int q = (int)(k & 3u), b = (int)(k & 1u), slot = (int)((k >> 2) & 1u);
      if (k >= 2) QP_WAIT(&empty[b], (uint32_t)(((k >> 1) - 1) & 1u));
      uint64_t* meta = metas + kQPMeta * slot;
      if (q == 0 && !P.prep(meta)) {  // no item left: the end marker completes buffer 0
        mbar_arrive(&bars[b]);
        return;
      }
      // quarter q: both windows' quarters, u and v_prev at its outputs
      const uint32_t modes = (uint32_t)meta[0];
      const bool self = (modes & 16u) != 0;
      const uint32_t sq = (((uint32_t)q & 1u) << 1) | ((uint32_t)q >> 1);  // swap2(q)
      const uint64_t oQ1 = meta[1], oQ1p = meta[2], of = meta[3], om = meta[4], opf = meta[5],
                     opm = meta[6];
      const uint64_t q1s = oQ1 != kNone ? oQ1 + 1024u * (uint32_t)q
                                        : (oQ1p != kNone ? oQ1p + 1024u * (((3u - q) & 1u) << 1 | ((3u - q) >> 1)) : kNone);
      const uint64_t xs = of != kNone ? of + 512u * sq : (om != kNone ? om + 512u * (3u - sq) : kNone);
      const uint64_t ps = self ? kNone
                               : (opf != kNone ? opf + 512u * (3u - q)
                                               : (opm != kNone ? opm + 512u * (uint32_t)q : kNone));
      const int na = prev ? 2 : 1;
      uint32_t bytes = 2u * Q * 4u;
      bytes += (uint32_t)na * ((q1s != kNone ? 4096u : 0u) + (xs != kNone ? 2048u : 0u) +
                               (ps != kNone ? 2048u : 0u));
      mbar_expect_tx(&bars[b], bytes);
      float* buf = qbuf + (size_t)b * kQWBuf;
      qp_issue_win(buf, reinterpret_cast<const float*>(meta[8]), modes & 3u, sq, &bars[b]);
      qp_issue_win(buf + Q, reinterpret_cast<const float*>(meta[9]), (modes >> 2) & 3u,
                   3u - (uint32_t)q, &bars[b]);
      for (int ar = 0; ar < na; ++ar) {
        const float* base = ar ? prev : src;
        float* st = buf + 4096 + 2048 * ar;
        if (q1s != kNone) tma_load_1d(st, base + q1s, 4096u, &bars[b]);
        if (xs != kNone) tma_load_1d(st + 1024, base + xs, 2048u, &bars[b]);
        if (ps != kNone) tma_load_1d(st + 1536, base + ps, 2048u, &bars[b]);
      }
      (void)self;
    }
  }
  const int lane = tid & 31;
  BAcc ba{-INFINITY, INFINITY, INFINITY, 0.0};
  for (uint32_t i = 0;; ++i) {
    const uint64_t* meta = metas + kQPMeta * (i & 1u);
    QP_WAIT(&bars[0], 0u);
    if (meta[7]) break;
    const uint32_t modes = (uint32_t)meta[0];
    const uint32_t mw = modes & 3u, mp = (modes >> 2) & 3u;
    const bool self = (modes & 16u) != 0;
    const uint32_t combo = mw * 4 + mp;
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
      const int bb = q & 1;
      if (q) QP_WAIT(&bars[bb], (uint32_t)(q >> 1));
      const float* buf = qbuf + (size_t)bb * kQWBuf;
      const uint32_t qd = (uint32_t)tid + kThreads * (uint32_t)q;
      float xa[4], xb[4], pa[4], pb[4];
#define LCSB_QPW(MW, MP) wq_load<MW, MP>(buf, buf + 2048, qd, xa, xb, pa, pb)
      switch (combo) {
        case 0: LCSB_QPW(0, 0); break;
        case 1: LCSB_QPW(0, 1); break;
        case 2: LCSB_QPW(0, 2); break;
        case 3: LCSB_QPW(0, 3); break;
        case 4: LCSB_QPW(1, 0); break;
        case 5: LCSB_QPW(1, 1); break;
        case 6: LCSB_QPW(1, 2); break;
        case 7: LCSB_QPW(1, 3); break;
        case 8: LCSB_QPW(2, 0); break;
        case 9: LCSB_QPW(2, 1); break;
        case 10: LCSB_QPW(2, 2); break;
        case 11: LCSB_QPW(2, 3); break;
        case 12: LCSB_QPW(3, 0); break;
        case 13: LCSB_QPW(3, 1); break;
        case 14: LCSB_QPW(3, 2); break;
        default: LCSB_QPW(3, 3); break;
      }
#undef LCSB_QPW
      wq_common<DF>(xa, xb, pa, pb, buf + 4096, buf + 6144, meta, self, src, prev, ba, qd, dst);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[bb]);
    }
  }
  // block reduction over the 8 consumer warps (named barrier 1: the producer has left)
  double x = ba.rmax, y = ba.rmin, z = ba.dmin;
  for (int o = 16; o > 0; o >>= 1) {
    x = dmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    y = dmin(y, __shfl_xor_sync(0xffffffffu, y, o));
    z = dmin(z, __shfl_xor_sync(0xffffffffu, z, o));
  }
  const int wid = tid >> 5;
  if (lane == 0) {
    r0[wid] = x;
    r1[wid] = y;
    r2[wid] = z;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
  if (tid == 0) {
    for (int w = 1; w < kThreads / 32; ++w) {
      x = dmax(x, r0[w]);
      y = dmin(y, r1[w]);
      z = dmin(z, r2[w]);
    }
    atomicMax(a.red_out + 0, ord_enc(x));
    atomicMin(a.red_out + 1, ord_enc(y));
    atomicMin(a.red_out + 2, ord_enc(z));
  }
}

template <int DEPTH, bool DF = false>
cudaError_t launch_qpw(const Bin2QArgs& a, cudaStream_t s, int sms) {
  constexpr size_t SMEM = 2 * kQWBuf * sizeof(float) + 4 * sizeof(uint64_t) +
                          2 * kQPMeta * sizeof(uint64_t);
  static uint64_t cap = 0;
  if (cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(bin2q_qpw_kernel<DEPTH, DF>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bin2q_qpw_kernel<DEPTH, DF>,
                                                      kQPWThreads, SMEM) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = (uint64_t)per_sm * sms;
  }
  if (a.K < 7 || a.ell < a.K + 1) return cudaErrorInvalidValue;
  const uint64_t ntiles = (a.sched && a.sched_m == 6) ? a.nitems : (1ull << (2 * (a.ell - 7)));
  uint64_t blocks = cap < ntiles ? cap : ntiles;
  if (blocks < 1) blocks = 1;
  Bin2QArgs b = a;
  const int L = 2 * a.ell;
  b.geo[0] = (1ull << L) - 1;
  b.geo[1] = 1ull << (L - 2);
  b.geo[2] = 0xAAAAAAAAAAAAAAAAull & b.geo[0];
  b.geo[3] = 0x5555555555555555ull & b.geo[0];
  b.geo[4] = (1ull << (2 * a.K)) - 1;
  b.geo[5] = 1ull << (2 * (a.ell - 7));
  bin2q_qpw_kernel<DEPTH, DF><<<(unsigned)blocks, kQPWThreads, SMEM, s>>>(b);
  return cudaGetLastError();
}

template <int DEPTH>
cudaError_t launch_qp(const Bin2QArgs& a, cudaStream_t s, int sms) {
  constexpr size_t SMEM = 8 * QPGeo::Q * sizeof(float) + 8 * sizeof(uint64_t) +
                          2 * kQPMeta * sizeof(uint64_t);
  static uint64_t cap = 0;
  if (cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(bin2q_qp_kernel<DEPTH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bin2q_qp_kernel<DEPTH>, kQPThreads,
                                                      SMEM) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = (uint64_t)per_sm * sms;
  }
  if (a.K < 7 || a.ell < a.K + 1) return cudaErrorInvalidValue;
  const uint64_t ntiles = (a.sched && a.sched_m == 6) ? a.nitems : (1ull << (2 * (a.ell - 7)));
  uint64_t blocks = cap < ntiles ? cap : ntiles;
  if (blocks < 1) blocks = 1;
  Bin2QArgs b = a;
  const int L = 2 * a.ell;
  b.geo[0] = (1ull << L) - 1;
  b.geo[1] = 1ull << (L - 2);
  b.geo[2] = 0xAAAAAAAAAAAAAAAAull & b.geo[0];
  b.geo[3] = 0x5555555555555555ull & b.geo[0];
  b.geo[4] = (1ull << (2 * a.K)) - 1;
  b.geo[5] = 1ull << (2 * (a.ell - 7));
  bin2q_qp_kernel<DEPTH><<<(unsigned)blocks, kQPThreads, SMEM, s>>>(b);
  return cudaGetLastError();
}

// the launch claims items dynamically (a schedule for these tiles and a work counter)
inline bool q_dynamic(const Bin2QArgs& a, int M) {
  return a.counter && a.sched && a.sched_m == M;
}

template <typename T, int M, int S, bool WMODE, int MINB = 1, int NT = kThreads, int UNR = 1,
          bool OFS = false, bool RES = false, int DEPTH = 1, bool DIFF = false>
cudaError_t launch_q(const Bin2QArgs& a, cudaStream_t s, int sms) {
  using C = QCfg<T, M, S, WMODE, MINB, RES>;
  static uint64_t cap = 0;
  if (cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(bin2q_kernel<T, M, S, WMODE, MINB, NT, UNR, OFS, RES, DEPTH, DIFF>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm,
                                                      bin2q_kernel<T, M, S, WMODE, MINB, NT, UNR, OFS, RES, DEPTH, DIFF>,
                                                      NT, C::SMEM) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = (uint64_t)per_sm * sms;
  }
  if (a.K < M + 1 || a.ell < a.K + 1) return cudaErrorInvalidValue;
  const uint64_t ntiles =
      (a.sched && a.sched_m == M) ? a.nitems : (1ull << (2 * (a.ell - 1 - M)));
  uint64_t blocks = cap < ntiles ? cap : ntiles;
  if (blocks < 1) blocks = 1;
  Bin2QArgs b = a;
  const int L = 2 * a.ell;
  b.geo[0] = (1ull << L) - 1;
  b.geo[1] = 1ull << (L - 2);
  b.geo[2] = 0xAAAAAAAAAAAAAAAAull & b.geo[0];
  b.geo[3] = 0x5555555555555555ull & b.geo[0];
  b.geo[4] = (1ull << (2 * a.K)) - 1;
  b.geo[5] = 1ull << (2 * (a.ell - 1 - M));
  bin2q_kernel<T, M, S, WMODE, MINB, NT, UNR, OFS, RES, DEPTH, DIFF><<<(unsigned)blocks, NT, C::SMEM, s>>>(b);
  return cudaGetLastError();
}

}  // namespace
}  // namespace lcsbk
