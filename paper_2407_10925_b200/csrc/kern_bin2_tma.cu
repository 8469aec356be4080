// kern_bin2_tma.cu -- the binary two-array half-table sweep (same arithmetic and tile pairing as
// kern_bin2.cu) with every byte moved by the Tensor Memory Accelerator:
//
//   * a persistent CTA walks its share of tile pairs {t, psi(t)} (kern_bin2.cu explains the
//     pairing); for each pair it bulk-copies (cp.async.bulk, 1-D TMA) the two contiguous adv_b
//     windows (2 x 2T entries) into an S-stage shared-memory ring completed by mbarrier
//     transaction counts, so S pairs of loads are in flight per CTA while it computes;
//   * the pair's outputs are assembled in shared memory as six contiguous runs -- Q1 tile t,
//     Q1 tile psi(t) (permuted in smem so the run is contiguous in HBM), and for each window its
//     Q0 rows and their mirrors (reversed in smem) -- and written back with bulk stores
//     (cp.async.bulk.global.shared::cta), double-buffered.
// HBM therefore sees one streaming read of every stored entry and full-line writes of every
// output; the SM only does the fp64 means/max in between.
#include <math.h>

#include "lcsb_internal.cuh"
#include "tma.cuh"

namespace lcsbk {
namespace {

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using v2 = float2;
  using v4 = float4;
};
template <>
struct Vec<double> {
  using v2 = double2;
  using v4 = double4;
};

__device__ __forceinline__ uint64_t pairswap(uint64_t v) {
  return ((v & 0xAAAAAAAAAAAAAAAAull) >> 1) | ((v & 0x5555555555555555ull) << 1);
}
__device__ __forceinline__ uint32_t pairswap32(uint32_t v) {
  return ((v & 0xAAAAAAAAu) >> 1) | ((v & 0x55555555u) << 1);
}

__device__ __forceinline__ double q0_val(double v0, double v1, double v2, double v3) {
  double r = ((v0 + v1) + v2) + v3;
  double cand = 0.25 * r;
  double best = 0.0;
  if (cand > best) best = cand;
  return 1.0 + best;
}

constexpr int kThreads = 256;

template <typename T, int M, int S, int OB>
struct TmaCfg {
  static constexpr uint32_t TT = 1u << (2 * M);   // Q1 outputs per tile
  static constexpr uint32_t WIN = 2 * TT;         // entries per adv_b window
  static constexpr uint32_t WIN_BYTES = WIN * sizeof(T);
  static constexpr uint32_t OUTN = 4 * TT;        // outputs per tile pair
  // OB = 0: outputs are stored straight from registers (sector-complete runs), no smem staging
  static constexpr size_t SMEM = (size_t)S * 2 * WIN * sizeof(T) + OB * (size_t)OUTN * sizeof(T) +
                                 (size_t)S * sizeof(uint64_t);
};

struct Geo {
  uint64_t q1, lmask, amask, bmask, ntiles;
};

__device__ __forceinline__ void tile_info(const Geo& g, uint64_t tau, uint32_t tt_log2,
                                          uint64_t& x0, uint64_t& p0, uint64_t& taup) {
  const uint64_t TT = 1ull << tt_log2;
  x0 = g.q1 + tau * TT;
  p0 = pairswap(~x0 & g.lmask) & ~(TT - 1);
  taup = (p0 - g.q1) >> tt_log2;
}

__device__ __forceinline__ uint64_t win_base(const Geo& g, uint64_t x) {
  return (x & g.amask) | ((x & g.bmask & ~g.q1) << 2);
}

// next tile >= c (stepping by G) that is the smaller member of its pair
__device__ __forceinline__ uint64_t next_item(const Geo& g, uint64_t c, uint64_t G,
                                              uint32_t tt_log2) {
  while (c < g.ntiles) {
    uint64_t x0, p0, taup;
    tile_info(g, c, tt_log2, x0, p0, taup);
    if (taup >= c) return c;
    c += G;
  }
  return c;
}

template <typename T, int M, int S, int OB>
__global__ void __launch_bounds__(kThreads) bin2_tma_kernel(Bin2Args a) {
  using C = TmaCfg<T, M, S, OB>;
  using V2 = typename Vec<T>::v2;
  constexpr uint32_t TT = C::TT, WIN = C::WIN, OUTN = C::OUTN;
  constexpr uint32_t LOG = 2 * M;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* in = reinterpret_cast<T*>(smem_raw);                 // [S][2][WIN]
  T* out = in + (size_t)S * 2 * WIN;                      // [OB][OUTN] (OB may be 0)
  uint64_t* bars = reinterpret_cast<uint64_t*>(out + OB * OUTN);

  const int L = 2 * a.ell;
  Geo g;
  g.lmask = (1ull << L) - 1;
  g.q1 = 1ull << (L - 2);
  g.amask = 0xAAAAAAAAAAAAAAAAull & g.lmask;
  g.bmask = 0x5555555555555555ull & g.lmask;
  g.ntiles = 1ull << (L - 2 - LOG);
  const T* src = reinterpret_cast<const T*>(a.src);
  T* dst = reinterpret_cast<T*>(a.dst);
  const int tid = threadIdx.x;
  const uint64_t G = gridDim.x;

  uint64_t pc = 0;  // producer cursor (thread 0 only)
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    pc = next_item(g, blockIdx.x, G, LOG);
    for (int s = 0; s < S && pc < g.ntiles; ++s) {
      uint64_t x0, p0, taup;
      tile_info(g, pc, LOG, x0, p0, taup);
      T* buf = in + (size_t)s * 2 * WIN;
      mbar_expect_tx(&bars[s], 2 * C::WIN_BYTES);
      tma_load_1d(buf, src + win_base(g, x0), C::WIN_BYTES, &bars[s]);
      tma_load_1d(buf + WIN, src + win_base(g, p0), C::WIN_BYTES, &bars[s]);
      pc = next_item(g, pc + G, G, LOG);
    }
  }

  uint32_t i = 0;
  for (uint64_t cc = next_item(g, blockIdx.x, G, LOG); cc < g.ntiles;
       cc = next_item(g, cc + G, G, LOG), ++i) {
    const uint32_t s = i % S;
    const uint32_t parity = (i / S) & 1u;
    T* buf = in + (size_t)s * 2 * WIN;
    T* ob = OB ? out + (size_t)(i % (OB ? OB : 1)) * OUTN : nullptr;
    if (OB && tid == 0) bulk_wait_read<(OB ? OB - 1 : 0)>();  // stores from ob OB items ago have read it
    mbar_wait(&bars[s], parity);
    __syncthreads();
    uint64_t x0, p0, taup;
    tile_info(g, cc, LOG, x0, p0, taup);
    const bool self = (taup == cc);
    const uint64_t wb = win_base(g, x0), wp = win_base(g, p0);

    const V2* W2 = reinterpret_cast<const V2*>(buf);
    const V2* P2 = reinterpret_cast<const V2*>(buf + WIN);
#pragma unroll
    for (uint32_t o = tid; o < TT; o += kThreads) {
      const V2 w = W2[pairswap32(o)];
      const V2 q = P2[TT - 1 - o];
      const double bx = 0.5 * ((double)w.x + (double)w.y);  // adv_b(x)
      const double bp = 0.5 * ((double)q.x + (double)q.y);  // adv_b(psi x) = adv_a(x)
      double v = bx;
      if (bp > v) v = bp;
      if (OB) {
        ob[o] = (T)v;
        ob[TT + pairswap32(~o & (TT - 1))] = (T)v;
      } else {
        dst[x0 + o] = (T)v;
        if (!self) dst[p0 + pairswap32(~o & (TT - 1))] = (T)v;
      }
    }
#pragma unroll
    for (uint32_t j = tid; j < TT; j += kThreads) {
      const uint32_t half = j / (TT / 2);        // 0: rows of window t, 1: of window psi(t)
      const uint32_t r = j % (TT / 2);
      const T* row = buf + half * WIN + 4 * r;
      const V2 lo = reinterpret_cast<const V2*>(row)[0];
      const V2 hi = reinterpret_cast<const V2*>(row)[1];
      const double fwd = q0_val(lo.x, lo.y, hi.x, hi.y);
      const double mir = q0_val(hi.y, hi.x, lo.y, lo.x);
      if (OB) {
        T* q0 = ob + 2 * TT + half * TT;
        q0[r] = (T)fwd;
        q0[TT / 2 + (TT / 2 - 1 - r)] = (T)mir;
      } else if (half == 0 || !self) {
        const uint64_t rb = (half ? wp : wb) >> 2;
        dst[rb + r] = (T)fwd;
        dst[(g.q1 - 1) - (rb + r)] = (T)mir;
      }
    }
    if (OB) fence_proxy_async_smem();
    __syncthreads();

    if (tid == 0) {
      if (OB) {
        constexpr uint32_t QB = TT * sizeof(T), HB = TT / 2 * sizeof(T);
        tma_store_1d(dst + x0, ob, QB);
        tma_store_1d(dst + (wb >> 2), ob + 2 * TT, HB);
        tma_store_1d(dst + (g.q1 - (wb >> 2) - TT / 2), ob + 2 * TT + TT / 2, HB);
        if (!self) {
          tma_store_1d(dst + p0, ob + TT, QB);
          tma_store_1d(dst + (wp >> 2), ob + 3 * TT, HB);
          tma_store_1d(dst + (g.q1 - (wp >> 2) - TT / 2), ob + 3 * TT + TT / 2, HB);
        }
        bulk_commit();
      }
      if (pc < g.ntiles) {  // refill the stage this item just vacated
        uint64_t px0, pp0, ptaup;
        tile_info(g, pc, LOG, px0, pp0, ptaup);
        mbar_expect_tx(&bars[s], 2 * C::WIN_BYTES);
        tma_load_1d(buf, src + win_base(g, px0), C::WIN_BYTES, &bars[s]);
        tma_load_1d(buf + WIN, src + win_base(g, pp0), C::WIN_BYTES, &bars[s]);
        pc = next_item(g, pc + G, G, LOG);
      }
    }
  }
  if (OB && tid == 0) bulk_wait<0>();
}

template <typename T, int M, int S, int OB>
cudaError_t launch_tma(const Bin2Args& a, cudaStream_t s, int sms) {
  using C = TmaCfg<T, M, S, OB>;
  static uint64_t cap = 0;
  if (cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(bin2_tma_kernel<T, M, S, OB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bin2_tma_kernel<T, M, S, OB>,
                                                      kThreads, C::SMEM) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = (uint64_t)per_sm * sms;
  }
  const uint64_t ntiles = 1ull << (2 * a.ell - 2 - 2 * M);
  uint64_t blocks = cap < ntiles ? cap : ntiles;
  bin2_tma_kernel<T, M, S, OB><<<(unsigned)blocks, kThreads, C::SMEM, s>>>(a);
  return cudaGetLastError();
}

struct VariantDesc {
  int m, s, ob;
};
// (M, S, OB) per variant id, fp32 and fp64 storage
constexpr VariantDesc kF32[] = {{0, 0, 0}, {5, 4, 2}, {4, 8, 2}, {5, 2, 2}, {4, 4, 2}, {0, 0, 0},
                                {5, 1, 2}, {5, 3, 2}, {4, 2, 2}, {5, 2, 1}, {5, 1, 1}, {6, 1, 1},
                                {6, 1, 0}, {6, 2, 0}, {5, 2, 0}, {5, 4, 0}, {6, 3, 0}};
constexpr VariantDesc kF64[] = {{0, 0, 0}, {4, 4, 2}, {4, 8, 2}, {4, 2, 2}, {3, 8, 2}, {0, 0, 0},
                                {4, 1, 2}, {4, 3, 2}, {5, 1, 1}, {4, 2, 1}, {4, 1, 1}, {3, 4, 2},
                                {5, 1, 0}, {5, 2, 0}, {4, 2, 0}, {4, 4, 0}, {5, 3, 0}};
constexpr int kNumVariants = 17;

}  // namespace

cudaError_t launch_bin2_tma_sweep(const Bin2Args& a, int dtype, int variant, cudaStream_t s,
                                  int sms) {
#define LCSB_V(T, M, S, OB) \
  if (d.m == M && d.s == S && d.ob == OB) return launch_tma<T, M, S, OB>(a, s, sms);
  if (variant <= 0 || variant >= kNumVariants) return cudaErrorInvalidValue;
  if (dtype == LCSB_F32) {
    const VariantDesc d = kF32[variant];
    LCSB_V(float, 5, 4, 2) LCSB_V(float, 4, 8, 2) LCSB_V(float, 5, 2, 2) LCSB_V(float, 4, 4, 2)
    LCSB_V(float, 5, 1, 2) LCSB_V(float, 5, 3, 2) LCSB_V(float, 4, 2, 2) LCSB_V(float, 5, 2, 1)
    LCSB_V(float, 5, 1, 1) LCSB_V(float, 6, 1, 1) LCSB_V(float, 6, 1, 0) LCSB_V(float, 6, 2, 0)
    LCSB_V(float, 5, 2, 0) LCSB_V(float, 5, 4, 0) LCSB_V(float, 6, 3, 0)
  } else {
    const VariantDesc d = kF64[variant];
    LCSB_V(double, 4, 4, 2) LCSB_V(double, 4, 8, 2) LCSB_V(double, 4, 2, 2) LCSB_V(double, 3, 8, 2)
    LCSB_V(double, 4, 1, 2) LCSB_V(double, 4, 3, 2) LCSB_V(double, 5, 1, 1) LCSB_V(double, 4, 2, 1)
    LCSB_V(double, 4, 1, 1) LCSB_V(double, 3, 4, 2) LCSB_V(double, 5, 1, 0) LCSB_V(double, 5, 2, 0)
    LCSB_V(double, 4, 2, 0) LCSB_V(double, 4, 4, 0) LCSB_V(double, 5, 3, 0)
  }
#undef LCSB_V
  return cudaErrorInvalidValue;
}

// smallest l whose Q1 has at least one tile of 4^M outputs (l - 1 >= M); 0 = not a TMA variant
int bin2_tma_min_ell(int dtype, int variant) {
  if (variant <= 0 || variant >= kNumVariants) return 0;
  const VariantDesc d = (dtype == LCSB_F32) ? kF32[variant] : kF64[variant];
  return d.m ? d.m + 1 : 0;
}

}  // namespace lcsbk
