// kern_q4.cu -- KS-form (and two-array) sweep and W pass for d = 2 strings over sigma = 4
// (BASELINE config 3) on
// the complement-folded table, reading each stored entry once per sweep.
//
// Recurrence (Eq. ineq3, Alg. 1, reading R1): for the pair
// (a, b) = (h_a alpha, h_b beta) with tails alpha, beta of length l-1,
//   h_a == h_b :  v' = 1 + max(0, P)                         (z = h: N empty -> 0; other z: P)
//   h_a != h_b :  v' = max(adv_b, adv_a, P)                  (z = h_a, z = h_b, the two other z)
//   P     = 1/16 sum_{c1,c2} g2[(alpha c1, beta c2)]          (|N| = 2 reads two sweeps back)
//   adv_b = 1/4  sum_c      g1[(h_a alpha, beta c)]           (|N| = 1 reads one sweep back)
//   adv_a = 1/4  sum_c      g1[(alpha c, h_b beta)]
// Layout (reading R14): x = h_a<<(4l-2) | h_b<<(4l-4) | t with t = interleave(alpha, beta), one
// 4-bit group (a digit, b digit) per character position.  adv_b's 4 entries are contiguous at
//   y = h_a<<(4l-2) | (t & A) | ((t & B) << 4) | c     (A / B = a / b digit bits of each group).
//
// Storage:
//  * complement fold: relabelling every symbol d -> 3-d is an alphabet permutation, under which
//    every iterate is invariant (reading R19 generalised; Eq. comp_eq for sigma = 2), and it maps
//    x to N-1-x.  Only h_a in {0, 1} is stored (x < N/2); the rest is read at N-1-x;
//  * pooled history: g2 is read ONLY through P, the mean of a 16-entry row, and P depends only on
//    the tails t.  Every sweep also writes the row means of the table it produces (fp64, one per
//    stored row, each summed in Alg. 1's order from the stored values in shared memory), and the
//    sweep two later reads those instead of g2: the ring holds 2 tables + 3 mean arrays.
//
// Two-array form (Q4Args::flags & kQ4TwoArray, reading R20): every option reads the
// previous sweep and h_a != h_b offers no P (the drop-both option), so
//   h_a == h_b :  v' = 1 + max(0, P1),  h_a != h_b :  v' = max(adv_b, adv_a)
// with P1 the row means of g1 itself -- the means the previous sweep wrote (ring of 2 suffices).
//
// Work unit: a unit is 16^M consecutive tails.  adv_a is adv_b of the string-swapped state:
// adv_a(h_a, h_b, t) = adv_b(h_b, h_a, swap t); for h_b >= 2 that window is folded -- it is the
// window of head 3-h_b of the complemented tails, read reversed.  So a CTA takes the group
// {u, s u, c u, c s u} (s = swap the two digits of every tail group, c = complement) and loads,
// for each unit of the group, its two stored adv_b windows (heads 0, 1) and, for the units whose
// first tail character is < 2, their row means of g2 (the others read their complement's,
// reversed).  From these it computes all stored outputs of the four units (h_a in {0,1}, every
// h_b): every stored window is read exactly once per sweep, every stored entry written once:
// 2 x (stored table) + 2 x (stored means) bytes per sweep, 4.5 B per logical state in fp32.
//
// Pipeline: a persistent grid (3 CTAs/SM); thread 0 walks this CTA's items (every G-th unit that
// is the smallest of its group), issues the TMA loads of the next item as soon as the current
// stage is consumed, and publishes the item's record (its units and the slots of their swapped /
// complemented partners) in shared memory with the loads; an end-of-work record completes the
// stage's mbarrier phase with a plain arrive.  Each thread owns one tail of every unit.
#include <math.h>
#include <stdlib.h>

#include "lcsb_internal.cuh"
#include "tma.cuh"

namespace lcsbk {
namespace {

constexpr int kThreads = 256;
// Q4Args::flags: issue the next item's loads as soon as the input stage is consumed (before the
// row-mean phase), and the bank-conflict-free tail order below
constexpr int kQ4EarlyIssue = 1, kQ4TailPerm = 2;
// Thread order of the 16 tails (a0, b0) of a row (i & 15 = 4 a0 + b0): each quarter-warp's 8
// 128-bit window loads (adv_b at 16 a0 + 64 b0 bytes, adv_a of the swapped and complemented
// swapped units at 16 b0 + 64 a0) then fall in 8 distinct 16-byte bank groups.
constexpr uint64_t kTailPerm = 0xFE985432DCBA7610ull;  // nibble k = tail of lane k
__device__ __forceinline__ uint32_t tail_of(uint32_t j, bool perm) {
  return perm ? ((j & ~15u) | (uint32_t)((kTailPerm >> (4 * (j & 15))) & 15)) : j;
}
constexpr uint64_t kA4 = 0xCCCCCCCCCCCCCCCCull;  // a digit (bits 2-3) of every 4-bit group
constexpr uint64_t kB4 = 0x3333333333333333ull;  // b digit (bits 0-1)

__device__ __forceinline__ uint64_t digit_swap(uint64_t v) {  // (a, b) -> (b, a) in every group
  return ((v & kA4) >> 2) | ((v & kB4) << 2);
}

template <typename T>
struct V4T;
template <>
struct V4T<float> {
  using type = float4;
};
template <>
struct V4T<double> {
  using type = double4;
};

// r <- r + (v + shift), c = 0..3 in order (Alg. 1 line 8); REV: the window is folded, logical
// c is stored entry 3-c.  SHIFT = false (sweeps, shift 0): v + 0.0 == v exactly for the
// non-negative iterate values (never -0.0), so the add is dropped.
template <typename T, bool REV, bool SHIFT>
__device__ __forceinline__ double sum4(const T* p, double sh) {
  const typename V4T<T>::type v = *reinterpret_cast<const typename V4T<T>::type*>(p);
  const double x = v.x, y = v.y, z = v.z, w = v.w;
  const double a0 = REV ? w : x, a1 = REV ? z : y, a2 = REV ? y : z, a3 = REV ? x : w;
  if (!SHIFT) return ((a0 + a1) + a2) + a3;
  double r = 0.0;
  r = r + (a0 + sh);
  r = r + (a1 + sh);
  r = r + (a2 + sh);
  r = r + (a3 + sh);
  return r;
}

constexpr int kGroup = 4;  // units per item (u, s u, c u, c s u), deduplicated
// per-stage item record written by the producer with the loads (the consumers read it after the
// mbarrier wait instead of recomputing the claim walk and the group): [0] = n | slot bits
// (kNoItem = end of work), [1..4] = the units
constexpr int kMeta = 6;
constexpr uint64_t kNoItem = ~0ull;

template <typename T, int M, int S, bool WMODE = false, bool GR = false>
struct Q4Cfg {
  static constexpr uint32_t TT = 1u << (4 * M);  // tails per unit
  static constexpr uint32_t WB = 4 * TT;         // g1 entries per adv_b window
  static constexpr uint32_t WIN = 2 * WB;        // the two stored windows of a unit (heads 0, 1)
  static constexpr uint32_t PR = TT * 8 / sizeof(T);  // a unit's TT row means (fp64), in T slots
  // W pass: also u at the unit's 8 stored output runs (h_a < 2, every h_b; TT tails each)
  static constexpr uint32_t UOUT = WMODE ? 8 * TT : 0;
  static constexpr uint32_t UNIT = WIN + PR + UOUT;
  static constexpr uint32_t STAGE = kGroup * UNIT;
  // sweep: the group's outputs staged for the row means of the new table, transposed so a row's
  // 16 values are 16 "c-rows" apart: [unit][head pair (8)][c][NR + 1] (NR = TT/16 rows per
  // head pair, +1 pad: stores and in-order row reads are bank-conflict-free)
  static constexpr uint32_t NR = TT / 16;
  // GR: no staging -- the row means re-read the just-written rows from global memory (L2)
  static constexpr uint32_t OUTS = (WMODE || GR) ? 0 : kGroup * 8 * 16 * (NR + 1);
  static constexpr size_t SMEM =
      (size_t)S * STAGE * sizeof(T) + (size_t)OUTS * sizeof(T) + (size_t)S * sizeof(uint64_t) +
      (size_t)S * kMeta * sizeof(uint64_t);
};

struct Q4Geo {
  int ell;
  uint32_t tail_bits;  // 4 (l - 1)
  uint32_t ubits;      // tail_bits - 4M: bits of a unit index
  uint64_t nunits;
  int p;               // sharded: 2^p shards (0 = unsharded), items of shard `shard` only
  uint32_t shard;
};

// shard key of a unit (its first tail groups; lcsb_internal.cuh q4_key): the key of both windows
// of every unit of its group
__device__ __forceinline__ uint32_t unit_key(const Q4Geo& g, uint64_t u) {
  const int B = (int)g.ubits;
  const uint32_t k1 = q4dig(u, B, 0, 1) ^ q4dig(u, B, 0, 0);
  if (g.p == 1) return k1 >> 1;
  if (g.p == 2) return k1;
  return (k1 << 1) | ((q4dig(u, B, 1, 1) ^ q4dig(u, B, 1, 0)) >> 1);
}

__device__ __forceinline__ uint64_t unit_comp(const Q4Geo& g, uint64_t u) {
  return ~u & (g.nunits - 1);
}
// first tail character of the unit's tails (its a digit) < 2: its row means are stored
__device__ __forceinline__ bool unit_low(const Q4Geo& g, uint64_t u) {
  return ((u >> (g.ubits - 1)) & 1ull) == 0;
}
__device__ __forceinline__ uint64_t group_min(const Q4Geo& g, uint64_t u) {
  const uint64_t su = digit_swap(u), cu = unit_comp(g, u), csu = unit_comp(g, su);
  uint64_t m = u < su ? u : su;
  m = m < cu ? m : cu;
  return m < csu ? m : csu;
}
// the group's distinct units in the fixed order (u, s u, c u, c s u); returns the count
__device__ __forceinline__ int group_units(const Q4Geo& g, uint64_t u, uint64_t (&U)[kGroup]) {
  const uint64_t cand[kGroup] = {u, digit_swap(u), unit_comp(g, u), unit_comp(g, digit_swap(u))};
  int n = 1;
  U[0] = u;
#pragma unroll
  for (int k = 1; k < kGroup; ++k) {
    bool dup = false;
#pragma unroll
    for (int j = 0; j < k; ++j) dup = dup || (cand[j] == cand[k]);
    if (!dup) {  // U[n++] = cand[k], with constant indices (U stays in registers)
#pragma unroll
      for (int p = 1; p <= k; ++p)
        if (n == p) U[p] = cand[k];
      ++n;
    }
  }
  return n;
}
__device__ __forceinline__ int slot_of(const uint64_t (&U)[kGroup], int n, uint64_t v) {
  int k = 0;
#pragma unroll
  for (int j = 0; j < kGroup; ++j)
    if (j < n && U[j] == v) k = j;
  return k;
}

// next item >= c (step G): a unit that is the smallest of its group (sharded: of this shard)
__device__ __forceinline__ uint64_t q4_next(const Q4Geo& g, uint64_t c, uint64_t G) {
  while (c < g.nunits) {
    if (group_min(g, c) == c && (g.p == 0 || unit_key(g, c) == g.shard)) return c;
    c += G;
  }
  return c;
}

template <typename T, int M, int S, bool WMODE>
__device__ __forceinline__ void q4_issue(const Q4Geo& g, uint64_t u, T* buf, uint64_t* bar,
                                         uint64_t* meta, const T* g1, const double* pin,
                                         const Q4Args& a) {
  using C = Q4Cfg<T, M, S, WMODE>;
  if (u >= g.nunits) {  // no item left: an end marker completes the stage's phase
    meta[0] = kNoItem;
    mbar_arrive(bar);
    return;
  }
  uint64_t U[kGroup] = {0, 0, 0, 0};
  const int n = group_units(g, u, U);
  // slots (2 bits each) of the swapped, complemented-swapped and complemented unit of each unit
  uint64_t rec = (uint64_t)n;
#pragma unroll
  for (int k = 0; k < kGroup; ++k) {
    const uint64_t X = U[k], sX = digit_swap(X);
    const uint64_t slots = (uint64_t)slot_of(U, n, sX) | ((uint64_t)slot_of(U, n, unit_comp(g, sX)) << 2) |
                           ((uint64_t)slot_of(U, n, unit_comp(g, X)) << 4);
    rec |= slots << (8 + 8 * k);
    meta[1 + k] = X;
  }
  meta[0] = rec;
  uint32_t bytes = 0;
  for (int k = 0; k < n; ++k) {
    bytes += C::WIN * (uint32_t)sizeof(T);
    if (unit_low(g, U[k])) bytes += C::TT * (uint32_t)sizeof(double);
    if (WMODE) bytes += C::UOUT * (uint32_t)sizeof(T);
  }
  mbar_expect_tx(bar, bytes);
  for (int k = 0; k < n; ++k) {
    const uint64_t t0 = U[k] << (4 * M);
    T* ub = buf + (size_t)k * C::UNIT;
    const uint64_t low = (t0 & kA4) | ((t0 & kB4) << 4);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t yb = ((uint64_t)h << (g.tail_bits + 2)) | low;
      // sharded: the window lies in this shard (its key is the item's), contiguously
      tma_load_1d(ub + h * C::WB, g1 + (g.p ? q4_local(yb, g.ell, g.p) : yb), C::WB * sizeof(T),
                  bar);
    }
    if (unit_low(g, U[k]))
      tma_load_1d(ub + C::WIN, pin + (g.p ? q4_mlocal(t0, g.ell, g.p) : t0),
                  C::TT * sizeof(double), bar);
    if (WMODE) {  // u (= g1, the newest table) at the unit's 8 stored output runs
      T* uo = ub + C::WIN + C::PR;
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        const uint64_t hx = ((uint64_t)(hh >> 2) << (g.tail_bits + 2)) |
                            ((uint64_t)(hh & 3) << g.tail_bits);
        // sharded: the run's owner (any shard; a peer's table through its mapped pointer)
        const T* src = g.p ? reinterpret_cast<const T*>(a.g1_sh[q4_key(hx | t0, g.ell, g.p)]) +
                                 q4_local(hx | t0, g.ell, g.p)
                           : g1 + (hx | t0);
        tma_load_1d(uo + hh * C::TT, src, C::TT * sizeof(T), bar);
      }
    }
  }
}

// sum of the 16 values of a row in order (Alg. 1: c = (c1, c2) lexicographic), read from global
// memory through L2 only (.cg: the rows were written by this CTA before the barrier)
template <typename T>
__device__ __forceinline__ double row16_sum(const T* p) {
  double sum = 0.0;
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(p) + q);
      sum = sum + (double)v.x;
      sum = sum + (double)v.y;
      sum = sum + (double)v.z;
      sum = sum + (double)v.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(p) + q);
      sum = sum + v.x;
      sum = sum + v.y;
    }
  }
  return sum;
}

template <typename T, int M, int S, bool WMODE, bool GR = false, bool SH = false, bool OFS = false>
__global__ void __launch_bounds__(kThreads, GR ? 4 : ((WMODE && sizeof(T) == 8) ? 1 : 3)) q4_kernel(Q4Args a) {
  using C = Q4Cfg<T, M, S, WMODE, GR>;
  constexpr uint32_t TT = C::TT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* in = reinterpret_cast<T*>(smem_raw);
  T* outs = in + (size_t)S * C::STAGE;  // Q4Cfg::OUTS layout (sweep only)
  uint64_t* bars = reinterpret_cast<uint64_t*>(outs + C::OUTS);
  uint64_t* metas = bars + S;  // [S][kMeta]

  Q4Geo g;
  g.ell = a.ell;
  g.tail_bits = 4u * (uint32_t)(a.ell - 1);
  g.ubits = g.tail_bits - 4 * M;
  g.nunits = 1ull << g.ubits;
  g.p = SH ? a.p : 0;  // unsharded instantiations: every shard branch folds away
  g.shard = (uint32_t)a.shard;
  const T* g1 = reinterpret_cast<const T*>(a.g1);
  const double* pin = a.pin;
  double* pout = a.pout;
  T* dst = reinterpret_cast<T*>(a.dst);
  const int tid = threadIdx.x;
  const uint64_t G = gridDim.x;
  const uint32_t hbit_a = g.tail_bits + 2, hbit_b = g.tail_bits;

  // W pass: W = (v + 2R) - F(v + R, v + 0R) for R in {R_max, R_min} (Alg. 2 line 6, d = 2)
  double R[2] = {0.0, 0.0}, wmax[2] = {-INFINITY, -INFINITY};
  if (WMODE) {
    R[0] = dec_ord(a.red_in[0]);
    R[1] = dec_ord(a.red_in[1]);
  }

  uint64_t pc = 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    pc = q4_next(g, blockIdx.x, G);
    for (int s = 0; s < S; ++s) {
      q4_issue<T, M, S, WMODE>(g, pc, in + (size_t)s * C::STAGE, &bars[s], metas + s * kMeta, g1,
                               pin, a);
      if (pc < g.nunits) pc = q4_next(g, pc + G, G);
    }
  }

  const bool ta = (a.flags & kQ4TwoArray) != 0;
  // integer offsets (OFS, sweep only; readings R23, R26): the row means read are of the table two
  // back (KS; one back in the two-array form, shift 0) and get gpost added after the mean; every
  // output gets shift = -c before the storage rounding; omn = min of the stored values.  The
  // |N| = 0 option (-o_n in stored terms, R26) never wins against P + gpost[2] >= -o_n, so
  // h_a == h_b stays 1 + P
  static_assert(!(OFS && WMODE), "offsets: sweeps only");
  [[maybe_unused]] double psh = 0.0, osh = 0.0, omn = INFINITY;
  [[maybe_unused]] float omn32 = INFINITY;  // fp32 storage: the min of the stored values
  if constexpr (OFS) {
    psh = a.ost->gpost[ta ? 1 : 2];
    osh = a.ost->shift;
  }
  static_assert(TT == kThreads, "one tail per thread and unit");
  const uint32_t i = tail_of((uint32_t)tid, (a.flags & kQ4TailPerm) != 0);
  const uint32_t i2 = (uint32_t)digit_swap(i);  // this tail's offset in the swapped unit
  const uint32_t offU = (uint32_t)((i & kA4) | ((i & kB4) << 4));
  const uint32_t offS = (uint32_t)((i2 & kA4) | ((i2 & kB4) << 4));
  const uint32_t i3 = TT - 1 - i2;  // in the complemented swapped unit
  const uint32_t offCS = (uint32_t)((i3 & kA4) | ((i3 & kB4) << 4));
  for (uint32_t it = 0;; ++it) {
    const uint32_t s = it % S;
    T* buf = in + (size_t)s * C::STAGE;
    mbar_wait(&bars[s], (it / S) & 1u);
    const uint64_t* meta = metas + s * kMeta;
    const uint64_t rec = meta[0];
    if (rec == kNoItem) break;
    const int n = (int)(rec & 7u);
    uint64_t U[kGroup];
#pragma unroll
    for (int k = 0; k < kGroup; ++k) U[k] = meta[1 + k];
    __syncthreads();  // every thread has the record before the producer may overwrite it

    // one tail per thread and unit (TT == kThreads): i and its window offsets are per-thread
    // constants (hoisted above the item loop)
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {  // unrolled: U[] stays in registers
      if (k >= n) break;
      const uint64_t X = U[k];
      const uint32_t sl = (uint32_t)(rec >> (8 + 8 * k));
      T* const drow = (WMODE || g.p) ? nullptr : dst + ((X << (4 * M)) + i);
      const T* ubX = buf + (size_t)k * C::UNIT;
      const T* ubS = buf + (size_t)(sl & 3u) * C::UNIT;
      const T* ubCS = buf + (size_t)((sl >> 2) & 3u) * C::UNIT;
      // P: the mean of the g2 row of these tails (|N| = 2, shift (d-2) R = 0); stored for units
      // whose first tail character is < 2, else the complement unit's, reversed
      double pu;
      if (unit_low(g, X)) {
        pu = reinterpret_cast<const double*>(ubX + C::WIN)[i];
      } else {
        const T* ubC = buf + (size_t)((sl >> 4) & 3u) * C::UNIT;
        pu = reinterpret_cast<const double*>(ubC + C::WIN)[TT - 1 - i];
      }
      if constexpr (OFS) pu = pu + psh;
#pragma unroll
      for (int m = 0; m < (WMODE ? 2 : 1); ++m) {
        const double sh = (WMODE && !ta) ? R[m] : 0.0;  // KS |N| = 1: shift (d-1) R = R
        double bU[2], bS[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) bU[h] = 0.25 * sum4<T, false, WMODE>(ubX + h * C::WB + offU, sh);
        // adv_a(h_a, h_b, t) = adv_b(h_b, h_a, swap t): stored for h_b < 2; for h_b >= 2 the
        // folded window of head 3 - h_b of the complemented swapped tails, read reversed
        bS[0] = 0.25 * sum4<T, false, WMODE>(ubS + 0 * C::WB + offS, sh);
        bS[1] = 0.25 * sum4<T, false, WMODE>(ubS + 1 * C::WB + offS, sh);
        bS[2] = 0.25 * sum4<T, true, WMODE>(ubCS + 1 * C::WB + offCS, sh);
        bS[3] = 0.25 * sum4<T, true, WMODE>(ubCS + 0 * C::WB + offCS, sh);
        // fp32 storage, sweep: round32(max(a, b, c)) = max(round32(a), round32(b), round32(c))
        // (rounding is monotone), so the candidates are rounded once each (7 conversions instead
        // of 8 fp64 max chains + 8 conversions) and the maxima taken in fp32 (one FMNMX each; no
        // NaN, no -0); the stored values are unchanged bit for bit
        // (OFS: x -> round32(x - c) is monotone too, so each candidate gets -c in fp64 first)
        [[maybe_unused]] float fU[2], fS[4], fpu = 0.f, fsame = 0.f;
        if constexpr (sizeof(T) == 4 && !WMODE) {
          auto shc = [osh](double x) {  // OFS: x - c; otherwise x itself (no instruction)
            if constexpr (OFS) return x + osh;
            else return x;
          };
          fU[0] = (float)shc(bU[0]);
          fU[1] = (float)shc(bU[1]);
#pragma unroll
          for (int hb = 0; hb < 4; ++hb) fS[hb] = (float)shc(bS[hb]);
          fpu = (float)shc(pu);
          fsame = (float)shc(1.0 + pu);
        }
#pragma unroll
        for (int ha = 0; ha < 2; ++ha) {
#pragma unroll
          for (int hb = 0; hb < 4; ++hb) {
            double v;
            if constexpr (sizeof(T) == 4 && !WMODE) {
              const float v32 = (ha == hb) ? fsame
                                           : (ta ? fmaxf(fU[ha], fS[hb])
                                                 : fmaxf(fmaxf(fU[ha], fS[hb]), fpu));
              v = (double)v32;  // exact; (T)v below gives v32 back
              if constexpr (OFS) omn32 = fminf(omn32, v32);
            } else if (ha == hb) {  // 1 + max(0, P): P is a mean of non-negative iterates, P >= 0
              v = 1.0 + pu;
            } else if (ta) {
              v = dmax(bU[ha], bS[hb]);  // two-array: no drop-both option (reading R20)
            } else {
              v = dmax(dmax(bU[ha], bS[hb]), pu);  // adv_b, adv_a, P
            }
            if constexpr (OFS && sizeof(T) == 8) {  // F - c (as the oracle: fp64), then the store
              v = v + osh;
              omn = dmin(omn, v);
            }
            const int hh = ha * 4 + hb;
            if (!WMODE) {
              // the head bits sit above the tail bits: | == +, so the row pointer is per unit
              if (g.p == 0) {
                drow[((uint64_t)ha << hbit_a) + ((uint64_t)hb << hbit_b)] = (T)v;
              } else {  // sharded: the owner of this (h_a, h_b) run (a peer: NVLink store)
                const uint64_t s0 =
                    ((uint64_t)ha << hbit_a) | ((uint64_t)hb << hbit_b) | (X << (4 * M));
                reinterpret_cast<T*>(a.dst_sh[q4_key(s0, g.ell, g.p)])[q4_local(s0, g.ell, g.p) +
                                                                       i] = (T)v;
              }
              if constexpr (!GR) {
                constexpr uint32_t NR1 = C::NR + 1;
                outs[(((uint32_t)k * 8 + hh) * 16 + (i & 15)) * NR1 + (i >> 4)] = (T)v;
              }
            } else {
              const T* uo = ubX + C::WIN + C::PR;
              wmax[m] = dmax(wmax[m], ((double)uo[hh * TT + i] + (ta ? R[m] : 2.0 * R[m])) - v);
            }
          }
        }
      }
    }
    __syncthreads();
    const bool early = (a.flags & kQ4EarlyIssue) != 0;
    if (early && tid == 0) {  // the input stage is consumed: refill it now
      q4_issue<T, M, S, WMODE>(g, pc, buf, &bars[s], metas + s * kMeta, g1, pin, a);
      if (pc < g.nunits) pc = q4_next(g, pc + G, G);
    }
    if (!WMODE) {
      // row means of the new table: output rows (h_a < 2, h_b, t >> 4) of the group's units, each
      // summed in Alg. 1's order over its 16 stored values
      constexpr uint32_t NR1 = C::NR + 1;
      // 8 NR = 128 rows per unit: threads 0-127 take the even units, 128-255 the odd ones
      static_assert(8 * C::NR * 2 == kThreads, "two units of rows per pass");
      const uint32_t jr = (uint32_t)tid % (8 * C::NR), odd = (uint32_t)tid / (8 * C::NR);
      const uint32_t hh = jr / C::NR, r = jr % C::NR;
      const uint64_t hx = ((uint64_t)(hh >> 2) << hbit_a) | ((uint64_t)(hh & 3) << hbit_b);
#pragma unroll
      for (int k2 = 0; k2 < kGroup; k2 += 2) {
        const uint32_t k = (uint32_t)k2 + odd;
        if ((int)k >= n) break;
        const uint64_t Uk = odd ? U[k2 + 1] : U[k2];
        double sum = 0.0;
        if constexpr (GR) {
          sum = row16_sum<T>(dst + (hx | (Uk << (4 * M))) + 16 * r);
        } else {
          const T* row = outs + ((k * 8 + hh) * 16) * NR1 + r;
#pragma unroll
          for (int c = 0; c < 16; ++c) sum = sum + (double)row[c * NR1];  // (+ 0.0: exact no-op)
        }
        const uint64_t row = ((hx | (Uk << (4 * M))) >> 4) | r;
        if (g.p == 0)
          pout[row] = 0.0625 * sum;
        else  // sharded: the shard of the items that read this row mean
          a.pout_sh[q4_mkey(row, g.ell, g.p)][q4_mlocal(row, g.ell, g.p)] = 0.0625 * sum;
      }
      __syncthreads();  // outs is reused by the next item
    }
    if (!early && tid == 0) {
      q4_issue<T, M, S, WMODE>(g, pc, buf, &bars[s], metas + s * kMeta, g1, pin, a);
      if (pc < g.nunits) pc = q4_next(g, pc + G, G);
    }
  }
  if (WMODE) block_max2_to(wmax[0], wmax[1], a.red_out);
  if constexpr (OFS) block_min_to(sizeof(T) == 4 ? (double)omn32 : omn, a.omin);
}

template <typename T, int M, int S, bool WMODE, bool GR = false, bool SH = false, bool OFS = false>
cudaError_t launch_q4_one(const Q4Args& a, cudaStream_t s, int sms) {
  using C = Q4Cfg<T, M, S, WMODE, GR>;
  static uint64_t cap = 0;
  if (cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(q4_kernel<T, M, S, WMODE, GR, SH, OFS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, q4_kernel<T, M, S, WMODE, GR, SH, OFS>,
                                                      kThreads, C::SMEM) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = (uint64_t)per_sm * sms;
  }
  const uint64_t nunits = 1ull << (4 * (a.ell - 1) - 4 * M);
  uint64_t blocks = cap < nunits ? cap : nunits;
  q4_kernel<T, M, S, WMODE, GR, SH, OFS><<<(unsigned)blocks, kThreads, C::SMEM, s>>>(a);
  return cudaGetLastError();
}
// sharded launches (a.p > 0) take the instantiation with the shard indexing compiled in
template <typename T, int M, int S, bool WMODE, bool GR = false>
cudaError_t launch_q4_t(const Q4Args& a, cudaStream_t s, int sms) {
  if (a.p > 0) return launch_q4_one<T, M, S, WMODE, false, true>(a, s, sms);
  return launch_q4_one<T, M, S, WMODE, GR, false>(a, s, sms);
}

}  // namespace

// the unit (16^2 tails) must leave at least one tail group above it (the folded row means are
// indexed by the first tail character)
int q4_min_ell() { return 4; }

static int q4_flags() {  // LCSB_Q4_FLAGS (A/B only): kQ4* bits, default both
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("LCSB_Q4_FLAGS");
    f = (e ? atoi(e) : (kQ4EarlyIssue | kQ4TailPerm)) & (kQ4EarlyIssue | kQ4TailPerm);
  }
  return f;
}

cudaError_t launch_q4_sweep(const Q4Args& a0, int dtype, cudaStream_t s, int sms) {
  static int variant = -1;  // LCSB_Q4_STAGES (A/B only): pipeline stages per CTA
  if (variant < 0) {
    const char* e = getenv("LCSB_Q4_STAGES");
    variant = e ? atoi(e) : 1;
  }
  Q4Args a = a0;
  a.flags = q4_flags() | (a0.flags & kQ4TwoArray);
  static int grows = -1;  // LCSB_Q4_GROWS (A/B): row means re-read from global, 4 CTAs/SM
  if (grows < 0) {
    const char* e = getenv("LCSB_Q4_GROWS");
    grows = e ? atoi(e) : 0;
  }
  if (a.ost) {  // integer offsets: the default pipeline (sharded: the shard indexing too)
    if (a.p > 0)
      return dtype == LCSB_F32 ? launch_q4_one<float, 2, 1, false, false, true, true>(a, s, sms)
                               : launch_q4_one<double, 2, 1, false, false, true, true>(a, s, sms);
    return dtype == LCSB_F32 ? launch_q4_one<float, 2, 1, false, false, false, true>(a, s, sms)
                             : launch_q4_one<double, 2, 1, false, false, false, true>(a, s, sms);
  }
  if (dtype == LCSB_F32) {
    if (variant == 2) return launch_q4_t<float, 2, 2, false>(a, s, sms);
    if (grows == 1) return launch_q4_t<float, 2, 1, false, true>(a, s, sms);
    if (grows == 2) return launch_q4_t<float, 2, 2, false, true>(a, s, sms);
    return launch_q4_t<float, 2, 1, false>(a, s, sms);
  }
  return launch_q4_t<double, 2, 1, false>(a, s, sms);
}
cudaError_t launch_q4_wpass(const Q4Args& a0, int dtype, cudaStream_t s, int sms) {
  Q4Args a = a0;
  a.flags = q4_flags() | (a0.flags & kQ4TwoArray);
  return dtype == LCSB_F32 ? launch_q4_t<float, 2, 1, true>(a, s, sms)
                           : launch_q4_t<double, 2, 1, true>(a, s, sms);
}

}  // namespace lcsbk
