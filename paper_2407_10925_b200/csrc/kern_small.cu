// kern_small.cu -- register-resident full-table sweep / W pass for small alphabets and string
// counts with sigma and d known at compile time (BASELINE config 2: sigma = 3, d = 3, fp64, KS;
// also (2,2), (3,2), (2,3)).  The same recurrence and Alg. 1 order as kern_generic.cu, but every
// per-string quantity lives in registers: the option masks are dispatched to compile-time
// instantiations whose appended-character loops are fully unrolled with constant offsets.
//
// Config 2's whole ring (4 x 4.05 MiB) is L2-resident, so the kernel is bound by L1/L2 gather
// throughput and launch latency rather than HBM; one thread per logical state, 32-bit indices.
//
// Pooled means (sweep only): an option that advances the strings in N (|N| = k >= 2) reads its
// generation only through the mean over N's appended characters, and those sigma^k entries lie
// in one "row" (the sigma^d states that differ only in the last character group) with the
// unchanged strings' last characters fixed.  So every sweep also writes, per row of the table it
// produces, those means for every mask of popcount k >= 2 and every value of the unchanged last
// characters (summed in Alg. 1's order from the stored values, staged in shared memory), and the
// options read one pooled value instead of sigma^k entries (config 2: ~35 gathers per state ->
// ~5).  The W pass adds a shift to every entry before summing (Alg. 2 line 6), so it keeps the
// raw gathers.
#include <math.h>

#include "lcsb_internal.cuh"

namespace lcsbk {
namespace {

template <int SIG, int D>
struct SmallConst {
  static constexpr uint32_t SIGD = [] {
    uint32_t v = 1;
    for (int i = 0; i < D; ++i) v *= SIG;
    return v;
  }();
};

// iterative (not recursive) so that calls with loop-variable exponents inline and fold once the
// loops are unrolled; the recursive form stayed a real CALL in SASS (a quarter of config 2's
// instructions)
__host__ __device__ __forceinline__ constexpr uint32_t ipow_c(uint32_t b, int e) {
  uint32_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// mean over the appended characters for the compile-time mask MASK (bit j = string j advances),
// reading `src` with `sh` added to each value, in Alg. 1's order (lexicographic, lowest string
// index most significant)
template <typename T, int SIG, int D, int MASK>
__device__ __forceinline__ double option_mean(const T* __restrict__ src, uint32_t base, double sh) {
  constexpr int K = __builtin_popcount(MASK);
  constexpr uint32_t COMBOS = ipow_c(SIG, K);
  double r = 0.0;
#pragma unroll
  for (uint32_t t = 0; t < COMBOS; ++t) {
    // decode t into c_q (q over the set bits of MASK, ascending j; last q fastest)
    uint32_t off = 0, tt = t;
#pragma unroll
    for (int j = D - 1; j >= 0; --j) {
      if (MASK & (1 << j)) {
        off += (tt % SIG) * ipow_c(SIG, D - 1 - j);
        tt /= SIG;
      }
    }
    r = r + ((double)__ldg(src + base + off) + sh);
  }
  const double inv = 1.0 / (double)COMBOS;  // sigma^{-|N|}, correctly rounded (constant-folded)
  return inv * r;
}

// ---- pooled-mean layout (per table, per k = |N| >= 2): per row, the masks of popcount k in
// increasing order, each with sigma^(d-k) values indexed by the unchanged strings' last
// characters (base sigma, string order)
__host__ __device__ __forceinline__ constexpr int popc_c(int m) {
  int c = 0;
  for (; m; m >>= 1) c += m & 1;
  return c;
}
__host__ __device__ __forceinline__ constexpr int mask_rank(int mask) {  // rank among masks of equal popcount
  int r = 0;
  for (int m = 0; m < mask; ++m)
    if (popc_c(m) == popc_c(mask)) ++r;
  return r;
}
__host__ __device__ __forceinline__ constexpr int nmasks(int d, int k) {
  int c = 0;
  for (int m = 0; m < (1 << d); ++m)
    if (popc_c(m) == k) ++c;
  return c;
}
template <int SIG, int D, int K>
struct PoolRow {  // pooled values per row for |N| = K
  static constexpr uint32_t PER_MASK = ipow_c(SIG, D - K);
  static constexpr uint32_t PER_ROW = (uint32_t)nmasks(D, K) * PER_MASK;
};
__host__ __device__ __forceinline__ constexpr uint32_t pool_per_row(int sig, int d, int k) {
  return (uint32_t)nmasks(d, k) * ipow_c((uint32_t)sig, d - k);
}

template <typename T, int SIG, int D, int MASK, bool POOL>
__device__ __forceinline__ double option_at(const T* const* src, const double* const* pin,
                                            const double* sh, const uint32_t* contrib,
                                            const uint32_t* head, uint32_t headw_top) {
  constexpr int K = __builtin_popcount(MASK);
  constexpr uint32_t SIGD = ipow_c(SIG, D);
  uint32_t base = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (MASK & (1 << j))
      base += (contrib[j] - head[j] * headw_top * ipow_c(SIG, D - 1 - j)) * SIGD;
    else
      base += contrib[j];
  }
  if constexpr (POOL && K >= 2) {
    // the unchanged strings' last characters (base % SIGD), in string order
    uint32_t fixed = 0;
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (!(MASK & (1 << j))) fixed = fixed * SIG + (base / ipow_c(SIG, D - 1 - j)) % SIG;
    using PR = PoolRow<SIG, D, K>;
    return pin[K - 1][(base / SIGD) * PR::PER_ROW + mask_rank(MASK) * PR::PER_MASK + fixed];
  } else {
    return option_mean<T, SIG, D, MASK>(src[K - 1], base, sh[K - 1]);
  }
}

template <typename T, int SIG, int D, bool POOL, int MASK = 1>
__device__ __forceinline__ double dispatch_mask(int mask, const T* const* src,
                                                const double* const* pin, const double* sh,
                                                const uint32_t* contrib, const uint32_t* head,
                                                uint32_t headw_top) {
  if constexpr (MASK < (1 << D)) {
    if (mask == MASK)
      return option_at<T, SIG, D, MASK, POOL>(src, pin, sh, contrib, head, headw_top);
    return dispatch_mask<T, SIG, D, POOL, MASK + 1>(mask, src, pin, sh, contrib, head, headw_top);
  } else {
    return 0.0;
  }
}

// F(src...)[x] (Eq. ineq3): b + max over the distinct option masks
template <typename T, int SIG, int D, bool POOL = false>
__device__ __forceinline__ double F_small(const T* const* src, const double* sh, uint32_t x,
                                          int ell, uint32_t headw_top,
                                          const double* const* pin = nullptr,
                                          bool two_array = false) {
  uint32_t contrib[D], head[D];
#pragma unroll
  for (int j = 0; j < D; ++j) contrib[j] = 0;
  uint32_t rem = x, pw = 1;
  for (int k = 0; k < ell; ++k) {  // groups from the last character up
#pragma unroll
    for (int j = D - 1; j >= 0; --j) {
      const uint32_t dig = rem % SIG;
      rem /= SIG;
      contrib[j] += dig * pw;
      head[j] = dig;  // the last group decoded is the heads
      pw *= SIG;
    }
  }
  int b = 1;
#pragma unroll
  for (int j = 1; j < D; ++j)
    if (head[j] != head[0]) b = 0;
  double best = -INFINITY;
  uint32_t seen = 0;
  int nseen = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const uint32_t hz = head[j];
    if (seen & (1u << hz)) continue;
    seen |= 1u << hz;
    ++nseen;
    int mask = 0;
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (head[i] != hz) mask |= 1 << i;
    const double cand =
        mask ? dispatch_mask<T, SIG, D, POOL>(mask, src, pin, sh, contrib, head, headw_top) : 0.0;
    if (cand > best) best = cand;
  }
  // some z is no string's head: N = all strings; the two-array form (d = 2) does not offer it
  // when the heads differ (drop-both, reading R20)
  if (nseen < SIG && !(two_array && !b)) {
    const double cand =
        option_at<T, SIG, D, (1 << D) - 1, POOL>(src, pin, sh, contrib, head, headw_top);
    if (cand > best) best = cand;
  }
  return (double)b + best;
}

template <typename T, int SIG, int D, bool WMODE>
__global__ void __launch_bounds__(256) small_kernel(GenericArgs a) {
  const T* src[D];
#pragma unroll
  for (int k = 0; k < D; ++k) src[k] = reinterpret_cast<const T*>(a.src[k]);
  const uint32_t headw_top = (uint32_t)a.headw_top;  // sigma^(d(l-1)), from the host
  const uint32_t n = (uint32_t)a.n;
  const uint32_t stride = gridDim.x * blockDim.x;
  const bool ta = (a.form == LCSB_FORM_TWO_ARRAY);
  if (!WMODE) {
    double zero[D];
#pragma unroll
    for (int k = 0; k < D; ++k) zero[k] = 0.0;
    T* dst = reinterpret_cast<T*>(a.dst);
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += stride)
      dst[x] = (T)F_small<T, SIG, D>(src, zero, x, a.ell, headw_top, nullptr, ta);
  } else {
    const double R0 = dec_ord(a.red_in[0]), R1 = dec_ord(a.red_in[1]);
    const bool ks = (a.form == LCSB_FORM_KS);
    double sh0[D], sh1[D];
#pragma unroll
    for (int k = 1; k <= D; ++k) {
      sh0[k - 1] = ks ? (double)(D - k) * R0 : 0.0;
      sh1[k - 1] = ks ? (double)(D - k) * R1 : 0.0;
    }
    const double dR0 = ks ? (double)D * R0 : R0, dR1 = ks ? (double)D * R1 : R1;
    const T* center = reinterpret_cast<const T*>(a.center);
    double w0 = -INFINITY, w1 = -INFINITY;
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += stride) {
      const double v = (double)center[x];
      const double F0 = F_small<T, SIG, D>(src, sh0, x, a.ell, headw_top, nullptr, ta);
      const double F1 = ks ? F_small<T, SIG, D>(src, sh1, x, a.ell, headw_top) : F0;
      w0 = dmax(w0, (v + dR0) - F0);
      w1 = dmax(w1, (v + dR1) - F1);
    }
    block_max2_to(w0, w1, a.red_out);
  }
}

// Pooled sweep: a CTA takes RPB consecutive rows (one thread per state), computes them with the
// pooled reads, stores them, stages them in shared memory and writes the pooled means of its rows
// for every k = 2..D.
template <int SIG, int D>
struct SmallPool {
  static constexpr uint32_t SIGD = ipow_c(SIG, D);
  static constexpr uint32_t RPB = 256 / SIGD;  // rows per CTA
  static constexpr uint32_t THREADS = RPB * SIGD;
  static constexpr uint32_t SUMS_PER_ROW = [] {
    uint32_t c = 0;
    for (int k = 2; k <= D; ++k) c += pool_per_row(SIG, D, k);
    return c;
  }();
};

template <typename T, int SIG, int D, int K, int MASK = 0>
__device__ __forceinline__ double pooled_sum(int maskidx, const T* row, uint32_t fixed) {
  // the mean over MASK's appended characters with the other strings' last characters = fixed,
  // in Alg. 1's order (lexicographic, lowest string index most significant)
  if constexpr (MASK < (1 << D)) {
    if constexpr (popc_c(MASK) == K) {
      if (mask_rank(MASK) == maskidx) {
        uint32_t foff = 0, ff = fixed;
#pragma unroll
        for (int j = D - 1; j >= 0; --j)
          if (!(MASK & (1 << j))) {
            foff += (ff % SIG) * ipow_c(SIG, D - 1 - j);
            ff /= SIG;
          }
        constexpr uint32_t COMBOS = ipow_c(SIG, K);
        double r = 0.0;
#pragma unroll
        for (uint32_t t = 0; t < COMBOS; ++t) {
          uint32_t off = 0, tt = t;
#pragma unroll
          for (int j = D - 1; j >= 0; --j) {
            if (MASK & (1 << j)) {
              off += (tt % SIG) * ipow_c(SIG, D - 1 - j);
              tt /= SIG;
            }
          }
          r = r + ((double)row[foff + off] + 0.0);
        }
        const double inv = 1.0 / (double)COMBOS;
        return inv * r;
      }
    }
    return pooled_sum<T, SIG, D, K, MASK + 1>(maskidx, row, fixed);
  } else {
    return 0.0;
  }
}

template <typename T, int SIG, int D>
__global__ void __launch_bounds__(SmallPool<SIG, D>::THREADS)
    small_pooled_kernel(GenericArgs a) {
  using SP = SmallPool<SIG, D>;
  constexpr uint32_t SIGD = SP::SIGD, RPB = SP::RPB;
  __shared__ T rows[RPB * SIGD];
  const T* src[D];
  const double* pin[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    src[k] = reinterpret_cast<const T*>(a.src[k]);
    pin[k] = a.pin[k];
  }
  const uint32_t headw_top = (uint32_t)a.headw_top;  // sigma^(d(l-1)), from the host
  const uint32_t nrows = (uint32_t)(a.n / SIGD);
  double zero[D];
#pragma unroll
  for (int k = 0; k < D; ++k) zero[k] = 0.0;
  T* dst = reinterpret_cast<T*>(a.dst);
  const uint32_t tid = threadIdx.x;
  for (uint32_t r0 = blockIdx.x * RPB; r0 < nrows; r0 += gridDim.x * RPB) {
    const uint32_t x = r0 * SIGD + tid;
    if (r0 + tid / SIGD < nrows) {
      const T v = (T)F_small<T, SIG, D, true>(src, zero, x, a.ell, headw_top, pin);
      dst[x] = v;
      rows[tid] = v;
    }
    __syncthreads();
    // pooled means of these rows for k = 2..D (SUMS_PER_ROW per row)
    for (uint32_t j = tid; j < RPB * SP::SUMS_PER_ROW; j += SP::THREADS) {
      const uint32_t rr = j / SP::SUMS_PER_ROW;
      if (r0 + rr >= nrows) continue;
      uint32_t q = j % SP::SUMS_PER_ROW;
      const T* row = rows + rr * SIGD;
#pragma unroll
      for (int k = 2; k <= D; ++k) {
        const uint32_t per = pool_per_row(SIG, D, k), pm = ipow_c(SIG, D - k);
        if (q < per) {
          double m = 0.0;
          if (k == 2) m = pooled_sum<T, SIG, D, 2>((int)(q / pm), row, q % pm);
          if (D >= 3 && k == 3) m = pooled_sum<T, SIG, D, (D >= 3 ? 3 : 2)>((int)(q / pm), row, q % pm);
          a.pout[k - 1][(uint64_t)(r0 + rr) * per + q] = m;
          break;
        }
        q -= per;
      }
    }
    __syncthreads();  // rows[] is reused
  }
}

template <typename T, int SIG, int D>
cudaError_t launch_small_pooled_t(const GenericArgs& a, cudaStream_t s, int sms) {
  using SP = SmallPool<SIG, D>;
  static uint64_t cap = 0;
  if (!cap) cap = resident_blocks(small_pooled_kernel<T, SIG, D>, SP::THREADS, sms);
  const uint64_t nrows = a.n / SP::SIGD;
  uint64_t blocks = (nrows + SP::RPB - 1) / SP::RPB;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  small_pooled_kernel<T, SIG, D><<<(unsigned)blocks, SP::THREADS, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int SIG, int D, bool WMODE>
cudaError_t launch_small_t(const GenericArgs& a, cudaStream_t s, int sms) {
  static uint64_t cap = 0;
  if (!cap) cap = resident_blocks(small_kernel<T, SIG, D, WMODE>, 256, sms);
  uint64_t blocks = (a.n + 255) / 256;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  small_kernel<T, SIG, D, WMODE><<<(unsigned)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

template <int SIG, int D>
cudaError_t launch_small_sd(const GenericArgs& a, int dtype, bool wpass, cudaStream_t s, int sms) {
  if (dtype == LCSB_F32)
    return wpass ? launch_small_t<float, SIG, D, true>(a, s, sms)
                 : launch_small_t<float, SIG, D, false>(a, s, sms);
  return wpass ? launch_small_t<double, SIG, D, true>(a, s, sms)
               : launch_small_t<double, SIG, D, false>(a, s, sms);
}

}  // namespace

// pooled sweeps: (sigma, d) with d = 3 (|N| = 2 and 3 pooled) or sigma^d >= 9 for d = 2
bool small_pooled_supported(int sigma, int d) {
  return (sigma == 3 && d == 3) || (sigma == 2 && d == 3) || (sigma == 3 && d == 2);
}
uint32_t small_pool_per_row(int sigma, int d, int k) { return pool_per_row(sigma, d, k); }

cudaError_t launch_small_pooled(const GenericArgs& a, int dtype, cudaStream_t s, int sms) {
#define LCSB_SP(SIG, D)                                                    \
  if (a.sigma == SIG && a.d == D)                                          \
    return dtype == LCSB_F32 ? launch_small_pooled_t<float, SIG, D>(a, s, sms) \
                             : launch_small_pooled_t<double, SIG, D>(a, s, sms);
  LCSB_SP(3, 3) LCSB_SP(2, 3) LCSB_SP(3, 2)
#undef LCSB_SP
  return cudaErrorInvalidValue;
}

bool small_supported(int sigma, int d, uint64_t n) {
  if (n >= (1ull << 31)) return false;
  return (sigma == 3 && d == 3) || (sigma == 2 && d == 2) || (sigma == 3 && d == 2) ||
         (sigma == 2 && d == 3);
}

cudaError_t launch_small(const GenericArgs& a, int dtype, bool wpass, cudaStream_t s, int sms) {
  if (a.sigma == 3 && a.d == 3) return launch_small_sd<3, 3>(a, dtype, wpass, s, sms);
  if (a.sigma == 2 && a.d == 2) return launch_small_sd<2, 2>(a, dtype, wpass, s, sms);
  if (a.sigma == 3 && a.d == 2) return launch_small_sd<3, 2>(a, dtype, wpass, s, sms);
  if (a.sigma == 2 && a.d == 3) return launch_small_sd<2, 3>(a, dtype, wpass, s, sms);
  return cudaErrorInvalidValue;
}

}  // namespace lcsbk
