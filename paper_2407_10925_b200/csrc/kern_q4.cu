// kern_q4.cu -- KS-form sweep (and W pass) for d = 2 strings over sigma = 4 (BASELINE config 3),
// full logical table, reading each input generation once per sweep.
//
// Recurrence (Eq. ineq3, Alg. 1, reading R1): for the pair
// (a, b) = (h_a alpha, h_b beta) with tails alpha, beta of length l-1,
//   h_a == h_b :  v' = 1 + max(0, P)                         (z = h: N empty -> 0; other z: P)
//   h_a != h_b :  v' = max(adv_b, adv_a, P)                  (z = h_a, z = h_b, the two other z)
//   P     = 1/16 sum_{c1,c2} g2[(alpha c1, beta c2)]          (|N| = 2 reads two sweeps back)
//   adv_b = 1/4  sum_c      g1[(h_a alpha, beta c)]           (|N| = 1 reads one sweep back)
//   adv_a = 1/4  sum_c      g1[(alpha c, h_b beta)]
// Layout (reading R14): x = h_a<<(4l-2) | h_b<<(4l-4) | t with t = interleave(alpha, beta), one
// 4-bit group (a digit, b digit) per character position.  The 16 entries read by P are the
// contiguous row t<<4 .. t<<4|15; adv_b's 4 entries are contiguous at
//   y = h_a<<(4l-2) | (t & A) | ((t & B) << 4) | c     (A / B = a / b digit bits of each group).
//
// B200 design: a unit is 16^M consecutive tails t for all 16 head pairs
// (16 x 16^M outputs).  For each h_a its adv_b reads are one contiguous window of 4 x 16^M
// entries of g1.  adv_a is taken from the string swap W(a,b) = W(b,a):
// adv_a(h_a,h_b,t) = adv_b(h_b,h_a,swap(t)), and swap maps the unit onto the unit of swapped
// tails (offset i -> ds(i), the two digits of every group exchanged).  One CTA takes the pair
// {unit, swap(unit)}, TMA bulk-loads it into shared memory (mbarrier-completed, S stages), and
// writes all 32 x 16^M outputs with coalesced stores.
//
// Pooled history: g2 (two sweeps back) is read ONLY through P, the mean of a 16-entry row, and
// P depends only on the tails t.  So every sweep also writes the row means of the table it
// produces (pout[x >> 4], fp64, N/16 entries: each output row of 16 is summed in Alg. 1's
// order from the stored -- rounded -- values, in shared memory), and the sweep two later reads
// those TT means per unit side instead of 16 TT entries of g2.  The full g2 table is never read,
// so the ring holds 2 full tables (+ 3 mean arrays): per sweep read g1 + means, write the new
// table + means = 2 x table + 2 x table/16 x 2 bytes ratio (9 B per state in fp32 instead of
// 12 for the three-table KS ring).
#include <math.h>
#include <stdlib.h>

#include "lcsb_internal.cuh"
#include "tma.cuh"

namespace lcsbk {
namespace {

constexpr int kThreads = 256;
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

template <typename T>
__device__ __forceinline__ double sum4(const T* p, double sh) {
  // r <- r + (v + shift), c = 0..3 in order (Alg. 1 line 8); p is 4-entry aligned
  const typename V4T<T>::type v = *reinterpret_cast<const typename V4T<T>::type*>(p);
  double r = 0.0;
  r = r + ((double)v.x + sh);
  r = r + ((double)v.y + sh);
  r = r + ((double)v.z + sh);
  r = r + ((double)v.w + sh);
  return r;
}

template <typename T, int M, int S, bool WMODE = false>
struct Q4Cfg {
  static constexpr uint32_t TT = 1u << (4 * M);  // tails per unit
  static constexpr uint32_t PR = TT * 8 / sizeof(T);  // the unit's TT row means (fp64), in T slots
  static constexpr uint32_t WB = 4 * TT;         // g1 entries per adv_b window
  static constexpr uint32_t UNIT = PR + 4 * WB;  // entries staged per unit
  // W pass: also u at the unit pair's 32 output runs (16 head pairs x T tails, per side)
  static constexpr uint32_t UOUT = WMODE ? 2 * 16 * TT : 0;
  static constexpr uint32_t STAGE = 2 * UNIT + UOUT;
  // sweep: the unit pair's outputs staged for the row means of the new table, transposed so a
  // row's 16 values are 16 "c-rows" apart: [side][head pair][c][NR + 1] (NR = TT/16 rows per
  // head pair, +1 pad: stores and in-order row reads are bank-conflict-free)
  static constexpr uint32_t NR = TT / 16;
  static constexpr uint32_t OUTS = WMODE ? 0 : 2 * 16 * 16 * (NR + 1);
  static constexpr size_t SMEM =
      (size_t)S * STAGE * sizeof(T) + (size_t)OUTS * sizeof(T) + (size_t)S * sizeof(uint64_t);
};

struct Q4Geo {
  int ell;
  uint32_t tail_bits;  // 4 (l - 1)
  uint64_t nunits;
};

// next unit >= c (step G) that is the smaller member of its swap pair
template <int M>
__device__ __forceinline__ uint64_t q4_next(const Q4Geo& g, uint64_t c, uint64_t G) {
  while (c < g.nunits) {
    if (digit_swap(c) >= c) return c;
    c += G;
  }
  return c;
}

template <typename T, int M, int S, bool WMODE>
__device__ __forceinline__ void q4_issue(const Q4Geo& g, uint64_t u, T* buf, uint64_t* bar,
                                         const T* g1, const double* pin) {
  using C = Q4Cfg<T, M, S, WMODE>;
  mbar_expect_tx(bar, C::STAGE * (uint32_t)sizeof(T));
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const uint64_t uu = side ? digit_swap(u) : u;
    const uint64_t t0 = uu << (4 * M);
    T* ub = buf + side * C::UNIT;
    tma_load_1d(ub, pin + t0, C::TT * sizeof(double), bar);
    const uint64_t low = (t0 & kA4) | ((t0 & kB4) << 4);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint64_t yb = ((uint64_t)h << (g.tail_bits + 2)) | low;
      tma_load_1d(ub + C::PR + h * C::WB, g1 + yb, C::WB * sizeof(T), bar);
    }
    if (WMODE) {  // u (= g1, the newest table) at the 16 output runs of this side
      T* uo = buf + 2 * C::UNIT + side * 16 * C::TT;
#pragma unroll
      for (int hh = 0; hh < 16; ++hh) {
        const uint64_t hx = ((uint64_t)(hh >> 2) << (g.tail_bits + 2)) |
                            ((uint64_t)(hh & 3) << g.tail_bits);
        tma_load_1d(uo + hh * C::TT, g1 + (hx | t0), C::TT * sizeof(T), bar);
      }
    }
  }
}

template <typename T, int M, int S, bool WMODE>
__global__ void __launch_bounds__(kThreads) q4_kernel(Q4Args a) {
  using C = Q4Cfg<T, M, S, WMODE>;
  constexpr uint32_t TT = C::TT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* in = reinterpret_cast<T*>(smem_raw);
  T* outs = in + (size_t)S * C::STAGE;  // Q4Cfg::OUTS layout (sweep only)
  uint64_t* bars = reinterpret_cast<uint64_t*>(outs + C::OUTS);

  Q4Geo g;
  g.ell = a.ell;
  g.tail_bits = 4u * (uint32_t)(a.ell - 1);
  g.nunits = 1ull << (g.tail_bits - 4 * M);
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
    pc = q4_next<M>(g, blockIdx.x, G);
    for (int s = 0; s < S && pc < g.nunits; ++s) {
      q4_issue<T, M, S, WMODE>(g, pc, in + (size_t)s * C::STAGE, &bars[s], g1, pin);
      pc = q4_next<M>(g, pc + G, G);
    }
  }

  uint32_t it = 0;
  for (uint64_t cu = q4_next<M>(g, blockIdx.x, G); cu < g.nunits; cu = q4_next<M>(g, cu + G, G), ++it) {
    const uint32_t s = it % S;
    T* buf = in + (size_t)s * C::STAGE;
    mbar_wait(&bars[s], (it / S) & 1u);
    __syncthreads();
    const uint64_t su = digit_swap(cu);
    const bool self = (su == cu);
    const uint64_t t0U = cu << (4 * M), t0S = su << (4 * M);
    const T* PU = buf;
    const T* WU = buf + C::PR;
    const T* PS = buf + C::UNIT;
    const T* WS = buf + C::UNIT + C::PR;

    for (uint32_t i = tid; i < TT; i += kThreads) {
      const uint32_t i2 = (uint32_t)digit_swap(i);       // the swapped tails' offset
      const uint32_t offU = (uint32_t)((i & kA4) | ((i & kB4) << 4));
      const uint32_t offS = (uint32_t)((i2 & kA4) | ((i2 & kB4) << 4));
      // P: mean of the 16-entry row of the table two sweeps back, |N| = 2 (shift (d-2) R = 0);
      // pooled when that table was written
      const double pu = reinterpret_cast<const double*>(PU)[i];
      const double ps = reinterpret_cast<const double*>(PS)[i2];
#pragma unroll
      for (int m = 0; m < (WMODE ? 2 : 1); ++m) {
        const double sh = WMODE ? R[m] : 0.0;  // |N| = 1: shift (d-1) R = R
        double bU[4], bS[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          bU[h] = 0.25 * sum4(WU + h * C::WB + offU, sh);
          bS[h] = 0.25 * sum4(WS + h * C::WB + offS, sh);
        }
#pragma unroll
        for (int ha = 0; ha < 4; ++ha) {
#pragma unroll
          for (int hb = 0; hb < 4; ++hb) {
            double vu, vs;
            if (ha == hb) {
              vu = 1.0 + fmax(0.0, pu);
              vs = 1.0 + fmax(0.0, ps);
            } else {
              vu = fmax(fmax(bU[ha], bS[hb]), pu);  // adv_b, adv_a (= adv_b of the swap), P
              vs = fmax(fmax(bS[ha], bU[hb]), ps);
            }
            const uint64_t hx = ((uint64_t)ha << hbit_a) | ((uint64_t)hb << hbit_b);
            const uint64_t xu = hx | (t0U + i), xs = hx | (t0S + i2);
            if (!WMODE) {
              dst[xu] = (T)vu;
              if (!self) dst[xs] = (T)vs;
              constexpr uint32_t NR1 = C::NR + 1;
              outs[((ha * 4 + hb) * 16 + (i & 15)) * NR1 + (i >> 4)] = (T)vu;
              outs[((16 + ha * 4 + hb) * 16 + (i2 & 15)) * NR1 + (i2 >> 4)] = (T)vs;
            } else {
              const double twoR = 2.0 * R[m];
              const T* uo = buf + 2 * C::UNIT;
              const double uu = (double)uo[(ha * 4 + hb) * TT + i];
              const double usv = (double)uo[16 * TT + (ha * 4 + hb) * TT + i2];
              wmax[m] = fmax(wmax[m], (uu + twoR) - vu);
              if (!self) wmax[m] = fmax(wmax[m], (usv + twoR) - vs);
              (void)xu;
              (void)xs;
            }
          }
        }
      }
    }
    __syncthreads();
    if (!WMODE) {
      // row means of the new table: output rows (h_a, h_b, t >> 4) of both sides, each summed
      // in Alg. 1's order over its 16 stored values (read all 16, then add in order)
      constexpr uint32_t RPS = 16 * C::NR, NR1 = C::NR + 1;  // rows per side
      for (uint32_t j = tid; j < (self ? 1u : 2u) * RPS; j += kThreads) {
        const uint32_t side = j / RPS, jr = j % RPS;
        const uint32_t hh = jr / C::NR, r = jr % C::NR;
        const T* row = outs + (side * 16 + hh) * 16 * NR1 + r;
        double sum = 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) sum = sum + ((double)row[k * NR1] + 0.0);
        const uint64_t hx = ((uint64_t)(hh >> 2) << hbit_a) | ((uint64_t)(hh & 3) << hbit_b);
        const uint64_t t0 = side ? t0S : t0U;
        pout[(hx | t0) >> 4 | r] = 0.0625 * sum;
      }
      __syncthreads();  // outs is reused by the next item
    }
    if (tid == 0 && pc < g.nunits) {
      q4_issue<T, M, S, WMODE>(g, pc, buf, &bars[s], g1, pin);
      pc = q4_next<M>(g, pc + G, G);
    }
  }
  if (WMODE) block_max2_to(wmax[0], wmax[1], a.red_out);
}

template <typename T, int M, int S, bool WMODE>
cudaError_t launch_q4_t(const Q4Args& a, cudaStream_t s, int sms) {
  using C = Q4Cfg<T, M, S, WMODE>;
  static uint64_t cap = 0;
  if (cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(q4_kernel<T, M, S, WMODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, q4_kernel<T, M, S, WMODE>, kThreads,
                                                      C::SMEM) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = (uint64_t)per_sm * sms;
  }
  const uint64_t nunits = 1ull << (4 * (a.ell - 1) - 4 * M);
  uint64_t blocks = cap < nunits ? cap : nunits;
  q4_kernel<T, M, S, WMODE><<<(unsigned)blocks, kThreads, C::SMEM, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

int q4_min_ell() { return 3; }  // the unit (16^2 tails) must fit in the 4^(2(l-1)) tail pairs

cudaError_t launch_q4_sweep(const Q4Args& a, int dtype, cudaStream_t s, int sms) {
  static int variant = -1;  // LCSB_Q4_STAGES (A/B only): pipeline stages per CTA
  if (variant < 0) {
    const char* e = getenv("LCSB_Q4_STAGES");
    variant = e ? atoi(e) : 1;
  }
  if (dtype == LCSB_F32) {
    if (variant == 2) return launch_q4_t<float, 2, 2, false>(a, s, sms);
    if (variant == 3) return launch_q4_t<float, 2, 3, false>(a, s, sms);
    return launch_q4_t<float, 2, 1, false>(a, s, sms);
  }
  return launch_q4_t<double, 2, 1, false>(a, s, sms);
}
cudaError_t launch_q4_wpass(const Q4Args& a, int dtype, cudaStream_t s, int sms) {
  return dtype == LCSB_F32 ? launch_q4_t<float, 2, 1, true>(a, s, sms)
                           : launch_q4_t<double, 2, 1, true>(a, s, sms);
}

}  // namespace lcsbk
