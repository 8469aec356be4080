// kern_small.cu -- register-resident full-table sweep / W pass for small alphabets and string
// counts with sigma and d known at compile time (BASELINE config 2: sigma = 3, d = 3, fp64, KS;
// also (2,2), (3,2), (2,3)).  The same recurrence and Alg. 1 order as kern_generic.cu, but every
// per-string quantity lives in registers: the option masks are dispatched to compile-time
// instantiations whose appended-character loops are fully unrolled with constant offsets.
//
// Config 2's whole ring (4 x 4.05 MiB) is L2-resident, so the kernel is bound by L1/L2 gather
// throughput and launch latency rather than HBM; one thread per logical state, 32-bit indices.
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

__host__ __device__ constexpr uint32_t ipow_c(uint32_t b, int e) {
  return e == 0 ? 1u : b * ipow_c(b, e - 1);
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

template <typename T, int SIG, int D, int MASK>
__device__ __forceinline__ double option_at(const T* const* src, const double* sh,
                                            const uint32_t* contrib, const uint32_t* head,
                                            uint32_t headw_top) {
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
  return option_mean<T, SIG, D, MASK>(src[K - 1], base, sh[K - 1]);
}

template <typename T, int SIG, int D, int MASK = 1>
__device__ __forceinline__ double dispatch_mask(int mask, const T* const* src, const double* sh,
                                                const uint32_t* contrib, const uint32_t* head,
                                                uint32_t headw_top) {
  if constexpr (MASK < (1 << D)) {
    if (mask == MASK) return option_at<T, SIG, D, MASK>(src, sh, contrib, head, headw_top);
    return dispatch_mask<T, SIG, D, MASK + 1>(mask, src, sh, contrib, head, headw_top);
  } else {
    return 0.0;
  }
}

// F(src...)[x] (Eq. ineq3): b + max over the distinct option masks
template <typename T, int SIG, int D>
__device__ __forceinline__ double F_small(const T* const* src, const double* sh, uint32_t x,
                                          int ell, uint32_t headw_top) {
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
    const double cand = mask ? dispatch_mask<T, SIG, D>(mask, src, sh, contrib, head, headw_top) : 0.0;
    if (cand > best) best = cand;
  }
  if (nseen < SIG) {  // some z is no string's head: N = all strings
    const double cand = option_at<T, SIG, D, (1 << D) - 1>(src, sh, contrib, head, headw_top);
    if (cand > best) best = cand;
  }
  return (double)b + best;
}

template <typename T, int SIG, int D, bool WMODE>
__global__ void __launch_bounds__(256) small_kernel(GenericArgs a) {
  const T* src[D];
#pragma unroll
  for (int k = 0; k < D; ++k) src[k] = reinterpret_cast<const T*>(a.src[k]);
  uint32_t headw_top = 1;
  for (int i = 0; i < D * (a.ell - 1); ++i) headw_top *= SIG;
  const uint32_t n = (uint32_t)a.n;
  const uint32_t stride = gridDim.x * blockDim.x;
  if (!WMODE) {
    double zero[D];
#pragma unroll
    for (int k = 0; k < D; ++k) zero[k] = 0.0;
    T* dst = reinterpret_cast<T*>(a.dst);
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += stride)
      dst[x] = (T)F_small<T, SIG, D>(src, zero, x, a.ell, headw_top);
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
      const double F0 = F_small<T, SIG, D>(src, sh0, x, a.ell, headw_top);
      const double F1 = ks ? F_small<T, SIG, D>(src, sh1, x, a.ell, headw_top) : F0;
      w0 = fmax(w0, (v + dR0) - F0);
      w1 = fmax(w1, (v + dR1) - F1);
    }
    block_max2_to(w0, w1, a.red_out);
  }
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
