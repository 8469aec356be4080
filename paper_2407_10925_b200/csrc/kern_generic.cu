// kern_generic.cu -- full-table Feasible Triplet sweep for any (sigma, d, l), one thread per
// logical state.
//
//   v_new[A] = b(A) + max_{z in Sigma} F_z(v_{n-1}, ..., v_{n-d}, A)        Eq. (ineq3)
//   F_z      = sigma^{-|N|} * sum_{c in Sigma^{|N|}} v_{|N|}[A with s_j <- T(s_j) c_j, j in N]
//                                                                            Alg. 1
// with N = (j : h(a_j) != z), F_z = 0 for empty N (reading R3), and v_{|N|} the table |N| sweeps
// back (KS form, reading R1) or the previous sweep (two-array form; for sigma > 2,
// d = 2 without the drop-both option, reading R20).
//
// Index arithmetic (reading R14, heads in the top digit group): with contrib_j the part of x
// contributed by string j and W_j = sigma^(d(l-1) + (d-1-j)) the weight of its head, advancing
// the strings in mask M gives the row base
//     base_M = sum_{j not in M} contrib_j + sum_{j in M} (contrib_j - h_j W_j) * sigma^d
// and the sigma^{|M|} reads base_M + sum_q c_q sigma^(d-1-N[q]) all fall in ONE row of sigma^d
// consecutive entries (the bottom digit group).
//
// Floating point: every sum runs in fp64 in Alg. 1's order (c lexicographic, lowest string index
// most significant), then is multiplied by the correctly rounded 1/sigma^|N|; the library is
// compiled with -fmad=false so no product is fused into a later add.  Options z whose masks
// coincide (every z that is no string's head gives the full mask) are evaluated once: max is
// exact, so this changes no value.
#include <math.h>

#include "lcsb_internal.cuh"

namespace lcsbk {
namespace {

__device__ inline double dec_dev(unsigned long long u) {
  unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  return __longlong_as_double((long long)b);
}

template <typename T>
__device__ inline double ld(const void* p, uint64_t i) {
  return (double)__ldg(reinterpret_cast<const T*>(p) + i);
}

template <typename T, int S_, int D_>
struct Gen {
  int sigma, d, ell;
  uint64_t sig_d;        // sigma^d
  uint64_t headw_top;    // sigma^(d(l-1))
  uint64_t wts[kMaxD];   // sigma^(d-1-j)

  __device__ void init(const GenericArgs& a) {
    sigma = S_ ? S_ : a.sigma;
    d = D_ ? D_ : a.d;
    ell = a.ell;
    sig_d = 1;
    for (int i = 0; i < d; ++i) sig_d *= (uint64_t)sigma;
    headw_top = 1;
    for (int i = 0; i < d * (ell - 1); ++i) headw_top *= (uint64_t)sigma;
    uint64_t w = 1;
    for (int j = d - 1; j >= 0; --j) {
      wts[j] = w;
      w *= (uint64_t)sigma;
    }
  }

  // mean over the appended characters for mask `mask` (bit j = string j advances), reading
  // table src[popcount-1] with `shift[popcount-1]` added to each value (W pass); `post`
  // (KS integer offsets, reading R26; NULL = none): post[popcount] added to the mean.
  __device__ double option_mean(const GenericArgs& a, const uint64_t* contrib, const int* head,
                                unsigned mask, const double* shift,
                                const double* post = nullptr) const {
    int k = __popc(mask);
    uint64_t base = 0;
    uint64_t w[kMaxD];
    int q = 0;
#pragma unroll
    for (int j = 0; j < (D_ ? D_ : kMaxD); ++j) {
      if (j >= d) break;
      if (mask & (1u << j)) {
        uint64_t hw = headw_top * wts[j];
        base += (contrib[j] - (uint64_t)head[j] * hw) * sig_d;
        w[q++] = wts[j];
      } else {
        base += contrib[j];
      }
    }
    const void* src = a.src[k - 1];
    const double sh = shift[k - 1];
    uint64_t combos = 1;
    for (int i = 0; i < k; ++i) combos *= (uint64_t)sigma;
    int c[kMaxD];
    for (int i = 0; i < k; ++i) c[i] = 0;
    uint64_t off = 0;
    double r = 0.0;
    for (uint64_t t = 0; t < combos; ++t) {
      r = r + (ld<T>(src, base + off) + sh);
      // odometer: c_{k} (last position of N) runs fastest = lexicographic order
      int p = k - 1;
      c[p]++;
      off += w[p];
      while (c[p] == sigma && p > 0) {
        c[p] = 0;
        off -= (uint64_t)sigma * w[p];
        --p;
        c[p]++;
        off += w[p];
      }
    }
    double inv = 1.0 / (double)combos;  // sigma^{-|N|}, correctly rounded
    return post ? inv * r + post[k] : inv * r;
  }

  // F(src...)[x] with per-|N| shifts; also returns the decoded structure for reuse
  __device__ double F_at(const GenericArgs& a, uint64_t x, const double* shift,
                         const double* post = nullptr) const {
    uint64_t contrib[kMaxD];
    int head[kMaxD];
    for (int j = 0; j < d; ++j) contrib[j] = 0;
    uint64_t rem = x, pw = 1;
    const int nd = d * ell;
    for (int p = 0; p < nd; ++p) {
      uint64_t dig = rem % (uint64_t)sigma;
      rem /= (uint64_t)sigma;
      int j = d - 1 - (p % d);
      contrib[j] += dig * pw;
      if (p >= nd - d) head[j] = (int)dig;
      pw *= (uint64_t)sigma;
    }
    int b = 1;
    for (int j = 1; j < d; ++j)
      if (head[j] != head[0]) b = 0;
    double best = -INFINITY;
    unsigned long long seen = 0;
    int nseen = 0;
    const unsigned full = (d >= 32) ? 0xffffffffu : ((1u << d) - 1u);
    for (int j = 0; j < d; ++j) {
      int hz = head[j];
      if (seen & (1ull << hz)) continue;
      seen |= 1ull << hz;
      ++nseen;
      unsigned mask = 0;
      for (int i = 0; i < d; ++i)
        if (head[i] != hz) mask |= 1u << i;
      // |N| = 0: R3's 0 (offsets: in stored terms, post[0] = -o_n, reading R26)
      double cand = mask ? option_mean(a, contrib, head, mask, shift, post) : (post ? post[0] : 0.0);
      if (cand > best) best = cand;
    }
    // some z is no string's head: N = all strings; not offered by the two-array form (d = 2)
    // when the heads differ (drop-both, reading R20)
    if (nseen < sigma && !(a.form == LCSB_FORM_TWO_ARRAY && !b)) {
      double cand = option_mean(a, contrib, head, full, shift, post);
      if (cand > best) best = cand;
    }
    return (double)b + best;
  }
};

template <typename T, int S_, int D_>
__global__ void __launch_bounds__(256) generic_sweep_kernel(GenericArgs a) {
  Gen<T, S_, D_> g;
  g.init(a);
  double zero[kMaxD];
  for (int i = 0; i < kMaxD; ++i) zero[i] = 0.0;
  T* dst = reinterpret_cast<T*>(a.dst);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // integer offsets (reading R23): store round(F(s) + shift), reduce the min of the stored values;
  // KS (R26): gpost[k] added to the means over the table k back (0 in the two-array form)
  const double sh = a.ost ? a.ost->shift : 0.0;
  const double* gsh = a.ost ? a.ost->gpost : nullptr;
  double mn = INFINITY;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < a.n; x += stride) {
    double v = g.F_at(a, x, zero, gsh);
    if (a.ost) {
      const T st = (T)(v + sh);  // F(s) + (-c): exact in fp64 (c an integer), then the rounding
      dst[x] = st;
      mn = dmin(mn, (double)st);
    } else {
      dst[x] = (T)v;  // storage rounding: RNE for float
    }
  }
  if (a.ost) block_min_to(mn, a.omin);
}

__device__ inline void block_max2(double w0, double w1, unsigned long long* out) {
  __shared__ double s0[32], s1[32];
  for (int o = 16; o > 0; o >>= 1) {
    w0 = dmax(w0, __shfl_xor_sync(0xffffffffu, w0, o));
    w1 = dmax(w1, __shfl_xor_sync(0xffffffffu, w1, o));
  }
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s0[wid] = w0;
    s1[wid] = w1;
  }
  __syncthreads();
  if (wid == 0) {
    int nw = (blockDim.x + 31) >> 5;
    w0 = lane < nw ? s0[lane] : -INFINITY;
    w1 = lane < nw ? s1[lane] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      w0 = dmax(w0, __shfl_xor_sync(0xffffffffu, w0, o));
      w1 = dmax(w1, __shfl_xor_sync(0xffffffffu, w1, o));
    }
    if (lane == 0) {
      atomicMax(out + 0, ord_enc(w0));
      atomicMax(out + 1, ord_enc(w1));
    }
  }
}

// W pass (Alg. 2 line 6): W = (v + d R) - F(v + (d-1)R, ..., v + 0R)   (KS)
//                         W = (v + R)   - F(v, v)                      (two-array)
// for R = R_max and R = R_min; max over states into red_out[0..1].
template <typename T, int S_, int D_>
__global__ void __launch_bounds__(256) generic_wpass_kernel(GenericArgs a) {
  Gen<T, S_, D_> g;
  g.init(a);
  const double R0 = dec_dev(a.red_in[0]);
  const double R1 = dec_dev(a.red_in[1]);
  double sh0[kMaxD], sh1[kMaxD];
  const bool ks = (a.form == LCSB_FORM_KS);
  for (int k = 1; k <= g.d; ++k) {
    sh0[k - 1] = ks ? (double)(g.d - k) * R0 : 0.0;
    sh1[k - 1] = ks ? (double)(g.d - k) * R1 : 0.0;
  }
  const double dR0 = ks ? (double)g.d * R0 : R0;
  const double dR1 = ks ? (double)g.d * R1 : R1;
  double w0 = -INFINITY, w1 = -INFINITY;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < a.n; x += stride) {
    double v = ld<T>(a.center, x);
    double F0 = g.F_at(a, x, sh0);
    double F1 = ks ? g.F_at(a, x, sh1) : F0;
    w0 = dmax(w0, (v + dR0) - F0);
    w1 = dmax(w1, (v + dR1) - F1);
  }
  block_max2(w0, w1, a.red_out);
}

template <int S_, int D_>
cudaError_t launch_pair(const GenericArgs& a, int dtype, cudaStream_t s, int sms, bool wpass) {
  uint64_t blocks = (a.n + 255) / 256;
  static uint64_t caps[2][2] = {{0, 0}, {0, 0}};
  uint64_t& cap = caps[dtype == LCSB_F32][wpass];
  if (!cap)
    cap = dtype == LCSB_F32
              ? (wpass ? resident_blocks(generic_wpass_kernel<float, S_, D_>, 256, sms)
                       : resident_blocks(generic_sweep_kernel<float, S_, D_>, 256, sms))
              : (wpass ? resident_blocks(generic_wpass_kernel<double, S_, D_>, 256, sms)
                       : resident_blocks(generic_sweep_kernel<double, S_, D_>, 256, sms));
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (dtype == LCSB_F32) {
    if (wpass)
      generic_wpass_kernel<float, S_, D_><<<(unsigned)blocks, 256, 0, s>>>(a);
    else
      generic_sweep_kernel<float, S_, D_><<<(unsigned)blocks, 256, 0, s>>>(a);
  } else {
    if (wpass)
      generic_wpass_kernel<double, S_, D_><<<(unsigned)blocks, 256, 0, s>>>(a);
    else
      generic_sweep_kernel<double, S_, D_><<<(unsigned)blocks, 256, 0, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t dispatch(const GenericArgs& a, int dtype, cudaStream_t s, int sms, bool wpass) {
  if (a.sigma == 2 && a.d == 2) return launch_pair<2, 2>(a, dtype, s, sms, wpass);
  if (a.sigma == 3 && a.d == 3) return launch_pair<3, 3>(a, dtype, s, sms, wpass);
  if (a.sigma == 4 && a.d == 2) return launch_pair<4, 2>(a, dtype, s, sms, wpass);
  if (a.sigma == 3 && a.d == 2) return launch_pair<3, 2>(a, dtype, s, sms, wpass);
  if (a.sigma == 2 && a.d == 3) return launch_pair<2, 3>(a, dtype, s, sms, wpass);
  // compile-time alphabets for the larger Table-3 cells (digit arithmetic by constant divisors
  // instead of 64-bit division calls)
  if (a.d == 2) {
    switch (a.sigma) {
      case 5: return launch_pair<5, 2>(a, dtype, s, sms, wpass);
      case 6: return launch_pair<6, 2>(a, dtype, s, sms, wpass);
      case 7: return launch_pair<7, 2>(a, dtype, s, sms, wpass);
      case 8: return launch_pair<8, 2>(a, dtype, s, sms, wpass);
      case 9: return launch_pair<9, 2>(a, dtype, s, sms, wpass);
      case 10: return launch_pair<10, 2>(a, dtype, s, sms, wpass);
    }
  }
  if (a.sigma == 2 && a.d >= 4 && a.d <= 8) {
    switch (a.d) {
      case 8: return launch_pair<2, 8>(a, dtype, s, sms, wpass);
      case 4: return launch_pair<2, 4>(a, dtype, s, sms, wpass);
      case 5: return launch_pair<2, 5>(a, dtype, s, sms, wpass);
      case 6: return launch_pair<2, 6>(a, dtype, s, sms, wpass);
      case 7: return launch_pair<2, 7>(a, dtype, s, sms, wpass);
    }
  }
  if (a.sigma == 3 && a.d == 4) return launch_pair<3, 4>(a, dtype, s, sms, wpass);
  if (a.sigma == 4 && a.d == 3) return launch_pair<4, 3>(a, dtype, s, sms, wpass);
  if (a.sigma == 5 && a.d == 3) return launch_pair<5, 3>(a, dtype, s, sms, wpass);
  if (a.sigma == 6 && a.d == 3) return launch_pair<6, 3>(a, dtype, s, sms, wpass);
  if (a.sigma == 4 && a.d == 4) return launch_pair<4, 4>(a, dtype, s, sms, wpass);
  if (a.sigma == 3 && a.d == 8) return launch_pair<3, 8>(a, dtype, s, sms, wpass);
  return launch_pair<0, 0>(a, dtype, s, sms, wpass);
}

}  // namespace

cudaError_t launch_generic_sweep(const GenericArgs& a, int dtype, cudaStream_t s, int sms) {
  return dispatch(a, dtype, s, sms, false);
}
cudaError_t launch_generic_wpass(const GenericArgs& a, int dtype, cudaStream_t s, int sms) {
  return dispatch(a, dtype, s, sms, true);
}

}  // namespace lcsbk
