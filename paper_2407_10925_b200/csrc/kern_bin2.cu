// kern_bin2.cu -- binary (sigma = d = 2) two-array sweep on the complement-folded half table,
// reading every stored entry exactly once per sweep.
//
// Method (Eqs. F1/F0 PAPER.md:752-779), two-array form: every option
// reads the previous table g.  Stored entries are the logical pairs [0, H), H = 2^(2l-1) (head
// of a is 0); logical y >= H is read at 2^(2l) - 1 - y (Eq. comp_eq).
//   Q0 = [0, 2^(2l-2))  heads (0,0): v'[x] = 1 + 1/4 (g[4x] + g[4x+1] + g[4x+2] + g[4x+3])
//                                                           (Alg. 3 "SameFirstBit")
//   Q1 = [2^(2l-2), H)  heads (0,1): v'[x] = max(adv_b(x), adv_a(x))       (Alg. 4 and L10)
//        adv_b(x) = 1/2 (g[ib] + g[ib|1]), ib = a-bits | (b-bits without head) << 2
//        adv_a(x) = 1/2 (g[ia] + g[ia|2]), ia = b-bits | (a-bits) << 2   (folded if a_2 = 1)
//
// B200 design:
//  * A tile is an aligned block of T = 4^m consecutive Q1 outputs.  Its adv_b reads form ONE
//    contiguous window of 2T stored entries; the windows of all tiles
//    partition the stored table.  Within the window, output o reads the 8/16-byte pair
//    number pairswap(o) (the two bits of each bit pair exchanged).
//  * adv_a is not read from its own (strided, possibly folded) runs: with the string swap
//    W(a,b) = W(b,a) and the complement symmetry, adv_a(a,b) = adv_b(b~, a~) exactly (a sum of
//    two equal values, commutative in fp).  psi(a,b) = (b~, a~) maps Q1 tiles onto Q1 tiles, and
//    output o of tile t pairs with output pairswap(~o) of tile psi(t), whose adv_b pair sits at
//    window position T-1-o.  One CTA therefore takes the tile pair {t, psi(t)}, loads the two
//    windows once, and writes both tiles' final values.
//  * Each window of 2T entries also holds T/2 complete rows of 4: the Q0 output x = row and its
//    mirror 2^(2l-2)-1-row (which reads the same row reversed) are computed from the
//    same registers (partner lane exchange), in the oracle's summation order for each.
//  => per sweep every stored entry is read once and written once: 2 x table bytes (the
//     compulsory traffic of the two-array form).  All accesses are full 32-byte sectors.
#include <math.h>

#include "lcsb_internal.cuh"

namespace lcsbk {
namespace {

template <typename T>
struct V2T;
template <>
struct V2T<float> {
  using type = float2;
};
template <>
struct V2T<double> {
  using type = double2;
};

__device__ __forceinline__ uint64_t pairswap(uint64_t v) {
  return ((v & 0xAAAAAAAAAAAAAAAAull) >> 1) | ((v & 0x5555555555555555ull) << 1);
}

__device__ inline double dec_dev(unsigned long long u) {
  unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  return __longlong_as_double((long long)b);
}

template <typename V>
__device__ __forceinline__ V shfl_xor2(V v, int m) {
  V r;
  r.x = __shfl_xor_sync(0xffffffffu, v.x, m);
  r.y = __shfl_xor_sync(0xffffffffu, v.y, m);
  return r;
}

template <typename V>
__device__ __forceinline__ V ldg_stream(const V* p) {
  return __ldcs(p);  // read once: evict-first
}

// Q0 value 1 + max(0, 1/4 (((v0 + v1) + v2) + v3))  (Eq. ineq3 with z=0 empty -> 0)
// 1 + max(0, cand): the iterates are non-negative, so cand >= 0 and the max is cand (as kern_bin2q.cu)
__device__ __forceinline__ double q0_val(double v0, double v1, double v2, double v3) {
  const double r = ((v0 + v1) + v2) + v3;
  return 1.0 + 0.25 * r;
}

constexpr int kTPB = 256;

template <typename T, int M, bool WMODE>
__global__ void __launch_bounds__(kTPB) bin2_kernel(Bin2Args a) {
  using V2 = typename V2T<T>::type;
  constexpr uint64_t TT = 1ull << (2 * M);
  constexpr int NPT = (int)((TT + kTPB - 1) / kTPB);
  const int L = 2 * a.ell;
  const uint64_t lmask = (L >= 64) ? ~0ull : ((1ull << L) - 1);
  const uint64_t q1 = 1ull << (L - 2);
  const uint64_t amask = 0xAAAAAAAAAAAAAAAAull & lmask;
  const uint64_t bmask = 0x5555555555555555ull & lmask;
  const uint64_t ntiles = 1ull << (L - 2 - 2 * M);
  const T* src = reinterpret_cast<const T*>(a.src);
  T* dst = reinterpret_cast<T*>(a.dst);
  const int tid = threadIdx.x;

  double R0 = 0.0, R1 = 0.0, wm0 = -INFINITY, wm1 = -INFINITY;
  if (WMODE) {
    R0 = dec_dev(a.red_in[0]);
    R1 = dec_dev(a.red_in[1]);
  }

  for (uint64_t tau = blockIdx.x; tau < ntiles; tau += gridDim.x) {
    const uint64_t x0 = q1 + tau * TT;                     // first Q1 output of the tile
    const uint64_t p0 = pairswap(~x0 & lmask) & ~(TT - 1);  // first output of tile psi(tau)
    const uint64_t taup = (p0 - q1) >> (2 * M);
    if (taup < tau) continue;  // the pair is handled at its smaller tile
    const bool self = (taup == tau);
    const uint64_t wb = (x0 & amask) | ((x0 & bmask & ~q1) << 2);  // adv_b window of tau
    const uint64_t wp = (p0 & amask) | ((p0 & bmask & ~q1) << 2);  // adv_b window of psi(tau)
    const V2* W = reinterpret_cast<const V2*>(src + wb);
    const V2* Wp = reinterpret_cast<const V2*>(src + wp);

    V2 w[NPT], q[NPT];
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const uint64_t o = (uint64_t)i * kTPB + tid;
      if (o < TT) {
        w[i] = ldg_stream(W + pairswap(o));
        q[i] = ldg_stream(Wp + (TT - 1 - o));
      } else {
        w[i].x = w[i].y = (T)0;
        q[i].x = q[i].y = (T)0;
      }
    }
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const uint64_t o = (uint64_t)i * kTPB + tid;
      const bool act = o < TT;
      // ---- Q1: the pair (x, psi(x))
      const double bx = 0.5 * ((double)w[i].x + (double)w[i].y);  // adv_b(x)
      const double bp = 0.5 * ((double)q[i].x + (double)q[i].y);  // adv_b(psi x) = adv_a(x)
      double v = bx;
      if (bp > v) v = bp;
      const uint64_t xo = x0 + o;
      const uint64_t xp = p0 + pairswap(~o & (TT - 1));
      // ---- Q0 rows of window tau: partner holds the other half of the row (lane ^ 2)
      const uint64_t k = pairswap(o);
      const V2 wo = shfl_xor2(w[i], 2);
      const uint64_t row = (wb >> 2) + (k >> 1);
      double q0;
      uint64_t q0x;
      if ((k & 1) == 0) {
        q0 = q0_val(w[i].x, w[i].y, wo.x, wo.y);  // forward row, output x = row
        q0x = row;
      } else {
        q0 = q0_val(w[i].y, w[i].x, wo.y, wo.x);  // mirror output reads the row reversed
        q0x = (q1 - 1) - row;
      }
      // ---- Q0 rows of window psi(tau): partner is lane ^ 1 (position T-1-o)
      const uint64_t kp = TT - 1 - o;
      const V2 qo = shfl_xor2(q[i], 1);
      const uint64_t rowp = (wp >> 2) + (kp >> 1);
      double q0p;
      uint64_t q0px;
      if ((kp & 1) == 0) {
        q0p = q0_val(q[i].x, q[i].y, qo.x, qo.y);
        q0px = rowp;
      } else {
        q0p = q0_val(q[i].y, q[i].x, qo.y, qo.x);
        q0px = (q1 - 1) - rowp;
      }
      if (!act) continue;
      if (!WMODE) {
        dst[xo] = (T)v;
        if (!self) dst[xp] = (T)v;
        dst[q0x] = (T)q0;
        if (!self) dst[q0px] = (T)q0p;
      } else {
        // W = (u + R) - F'(u); u is the table itself.  W(psi x) = W(x) exactly (both entries
        // were written with the same value), so only x is evaluated for Q1.
        const double ux = (double)src[xo];
        wm0 = dmax(wm0, (ux + R0) - v);
        wm1 = dmax(wm1, (ux + R1) - v);
        const double uq = (double)src[q0x];
        wm0 = dmax(wm0, (uq + R0) - q0);
        wm1 = dmax(wm1, (uq + R1) - q0);
        if (!self) {
          const double uqp = (double)src[q0px];
          wm0 = dmax(wm0, (uqp + R0) - q0p);
          wm1 = dmax(wm1, (uqp + R1) - q0p);
        }
      }
    }
  }

  if (WMODE) {
    __shared__ double s0[kTPB / 32], s1[kTPB / 32];
    for (int o = 16; o > 0; o >>= 1) {
      wm0 = dmax(wm0, __shfl_xor_sync(0xffffffffu, wm0, o));
      wm1 = dmax(wm1, __shfl_xor_sync(0xffffffffu, wm1, o));
    }
    const int lane = tid & 31, wid = tid >> 5;
    if (lane == 0) {
      s0[wid] = wm0;
      s1[wid] = wm1;
    }
    __syncthreads();
    if (wid == 0) {
      wm0 = lane < kTPB / 32 ? s0[lane] : -INFINITY;
      wm1 = lane < kTPB / 32 ? s1[lane] : -INFINITY;
      for (int o = 16; o > 0; o >>= 1) {
        wm0 = dmax(wm0, __shfl_xor_sync(0xffffffffu, wm0, o));
        wm1 = dmax(wm1, __shfl_xor_sync(0xffffffffu, wm1, o));
      }
      if (lane == 0) {
        atomicMax(a.red_out + 0, ord_enc(wm0));
        atomicMax(a.red_out + 1, ord_enc(wm1));
      }
    }
  }
}

template <typename T, int M, bool WMODE>
cudaError_t launch_one(const Bin2Args& a, cudaStream_t s, int sms) {
  const int L = 2 * a.ell;
  const uint64_t ntiles = 1ull << (L - 2 - 2 * M);
  static uint64_t cap = 0;
  if (cap == 0) cap = resident_blocks(bin2_kernel<T, M, WMODE>, kTPB, sms);
  uint64_t blocks = a.grid_mult > 0 ? (uint64_t)a.grid_mult * sms : cap;
  if (blocks > ntiles) blocks = ntiles;
  if (blocks < 1) blocks = 1;
  bin2_kernel<T, M, WMODE><<<(unsigned)blocks, kTPB, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T, bool WMODE>
cudaError_t launch_m(const Bin2Args& a, cudaStream_t s, int sms) {
  switch (a.m) {
    case 1: return launch_one<T, 1, WMODE>(a, s, sms);
    case 2: return launch_one<T, 2, WMODE>(a, s, sms);
    case 3: return launch_one<T, 3, WMODE>(a, s, sms);
    case 4: return launch_one<T, 4, WMODE>(a, s, sms);
    case 5: return launch_one<T, 5, WMODE>(a, s, sms);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// register-kernel tile: 4^m outputs, small enough that small tables still give every SM work
// (at least ~2 x 148 tile pairs), at most 4^5
int bin2_tile_m(int ell) {
  int m = ell - 6;
  if (m > 5) m = 5;
  if (m < 1) m = 1;
  if (m > ell - 1) m = ell - 1;
  return m;
}

cudaError_t launch_bin2_sweep(const Bin2Args& a, int dtype, cudaStream_t s, int sms) {
  return dtype == LCSB_F32 ? launch_m<float, false>(a, s, sms) : launch_m<double, false>(a, s, sms);
}
cudaError_t launch_bin2_wpass(const Bin2Args& a, int dtype, cudaStream_t s, int sms) {
  return dtype == LCSB_F32 ? launch_m<float, true>(a, s, sms) : launch_m<double, true>(a, s, sms);
}

}  // namespace lcsbk
