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
#include <stdlib.h>

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

// 1 + max(0, cand): the iterates are non-negative, so cand >= 0 and the max is cand (as kern_bin2q.cu)
__device__ __forceinline__ double q0_val(double v0, double v1, double v2, double v3) {
  const double r = ((v0 + v1) + v2) + v3;
  return 1.0 + 0.25 * r;
}

constexpr int kThreads = 256;

template <typename T, int M, int S, int OB, bool WMODE = false>
struct TmaCfg {
  static constexpr uint32_t TT = 1u << (2 * M);   // Q1 outputs per tile
  static constexpr uint32_t WIN = 2 * TT;         // entries per adv_b window
  static constexpr uint32_t WIN_BYTES = WIN * sizeof(T);
  static constexpr uint32_t OUTN = 4 * TT;        // outputs per tile pair
  // W pass: the stage also holds u at the item's outputs (Q1 tile t, and the row / mirror runs of
  // both windows): 3T more entries
  static constexpr uint32_t STAGE = 2 * WIN + (WMODE ? 3 * TT : 0);
  // OB = 0: outputs are stored straight from registers (sector-complete runs), no smem staging
  static constexpr size_t SMEM = (size_t)S * STAGE * sizeof(T) + OB * (size_t)OUTN * sizeof(T) +
                                 (size_t)S * sizeof(uint64_t);
};

struct Geo {
  int L, p;
  uint32_t shard;
  uint64_t q1, lmask, amask, bmask;
  uint32_t h;       // tile-index pairs: the tile of 4^M outputs is fixed by h = l-1-M pairs
  uint64_t nloc;    // tiles owned by this shard: 4^h / 2^p
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

// j-th tile owned by this shard.  Tile index bits: pair i (i = 1..h, top first) = (a_i, b_i) of
// the tile's fixed characters.  Shard key kappa_i = a_i ^ b_i ^ 1 for i <= p, so
// the owned tiles have b_i = a_i ^ kappa_i ^ 1: j's top p bits are a_1..a_p, the rest free.
__device__ __forceinline__ uint64_t owned_tile(const Geo& g, uint64_t j) {
  if (g.p == 0) return j;
  const uint32_t rest = 2 * (g.h - g.p);
  uint64_t tau = j & ((1ull << rest) - 1);
  for (int i = 1; i <= g.p; ++i) {
    const uint64_t ai = (j >> (rest + g.p - i)) & 1ull;
    const uint64_t ki = (g.shard >> (g.p - i)) & 1u;
    const uint64_t bi = ai ^ ki ^ 1ull;
    tau |= ((ai << 1) | bi) << (2 * (g.h - i));
  }
  return tau;
}

// next owned item >= c (step G) whose tile is the smaller member of its psi pair; returns the
// enumeration index and the tile
__device__ __forceinline__ uint64_t next_item(const Geo& g, uint64_t c, uint64_t G,
                                              uint32_t tt_log2, uint64_t& tau_out) {
  while (c < g.nloc) {
    const uint64_t tau = owned_tile(g, c);
    uint64_t x0, p0, taup;
    tile_info(g, tau, tt_log2, x0, p0, taup);
    if (taup >= tau) {
      tau_out = tau;
      return c;
    }
    c += G;
  }
  return c;
}

template <typename T>
__device__ __forceinline__ T* out_ptr(const Geo& g, void* const* tabs, uint64_t global) {
  const uint32_t sh = shard_of_stored(global, g.L, g.p);
  return reinterpret_cast<T*>(tabs[sh]) + local_of_stored(global, g.L, g.p);
}

// Issue the TMA loads of one item into a stage (thread 0): the two adv_b windows and, for the
// W pass on an unsharded table, u at the item's outputs.
template <typename T, int M, int S, int OB, bool WMODE>
__device__ __forceinline__ void issue_item(const Geo& g, uint64_t tau, T* buf, uint64_t* bar,
                                           const T* src) {
  using C = TmaCfg<T, M, S, OB, WMODE>;
  constexpr uint32_t TT = C::TT, WIN = C::WIN;
  constexpr uint32_t LOG = 2 * M;
  uint64_t x0, p0, taup;
  tile_info(g, tau, LOG, x0, p0, taup);
  const uint64_t wb = win_base(g, x0), wp = win_base(g, p0);
  const bool with_u = WMODE && g.p == 0;
  const bool self = (taup == tau);
  uint32_t bytes = 2 * C::WIN_BYTES;
  if (with_u) bytes += (self ? 2 : 3) * TT * (uint32_t)sizeof(T);
  mbar_expect_tx(bar, bytes);
  tma_load_1d(buf, src + local_of_stored(wb, g.L, g.p), C::WIN_BYTES, bar);
  tma_load_1d(buf + WIN, src + local_of_stored(wp, g.L, g.p), C::WIN_BYTES, bar);
  if (with_u) {
    T* u = buf + 2 * WIN;
    constexpr uint32_t HB = TT / 2 * sizeof(T);
    tma_load_1d(u, src + x0, TT * sizeof(T), bar);
    tma_load_1d(u + TT, src + (wb >> 2), HB, bar);
    tma_load_1d(u + TT + TT / 2, src + (g.q1 - (wb >> 2) - TT / 2), HB, bar);
    if (!self) {
      tma_load_1d(u + 2 * TT, src + (wp >> 2), HB, bar);
      tma_load_1d(u + 2 * TT + TT / 2, src + (g.q1 - (wp >> 2) - TT / 2), HB, bar);
    }
  }
}

template <typename T, int M, int S, int OB, bool WMODE, int MINB = 1>
__global__ void __launch_bounds__(kThreads, MINB) bin2_tma_kernel(Bin2Args a) {
  using C = TmaCfg<T, M, S, OB, WMODE>;
  using V2 = typename Vec<T>::v2;
  constexpr uint32_t TT = C::TT, WIN = C::WIN, OUTN = C::OUTN;
  constexpr uint32_t LOG = 2 * M;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* in = reinterpret_cast<T*>(smem_raw);                 // [S][STAGE]
  T* out = in + (size_t)S * C::STAGE;                     // [OB][OUTN] (OB may be 0)
  uint64_t* bars = reinterpret_cast<uint64_t*>(out + OB * OUTN);

  Geo g;
  g.L = 2 * a.ell;
  g.p = a.shard_bits;
  g.shard = (uint32_t)a.shard;
  g.lmask = (1ull << g.L) - 1;
  g.q1 = 1ull << (g.L - 2);
  g.amask = 0xAAAAAAAAAAAAAAAAull & g.lmask;
  g.bmask = 0x5555555555555555ull & g.lmask;
  g.h = (uint32_t)(a.ell - 1 - M);
  g.nloc = (1ull << (2 * g.h)) >> g.p;
  const T* src = reinterpret_cast<const T*>(a.src);  // this shard's input table
  const int tid = threadIdx.x;
  const uint64_t G = gridDim.x;

  double R0 = 0.0, R1 = 0.0, wm0 = -INFINITY, wm1 = -INFINITY;
  if (WMODE) {
    R0 = dec_ord(a.red_in[0]);
    R1 = dec_ord(a.red_in[1]);
  }

  // shard table pointers in shared memory (a dynamic index into the kernel-parameter array
  // would force the parameter block through local memory)
  __shared__ void* s_tabs[kMaxShards];
  if (tid < kMaxShards)
    s_tabs[tid] = WMODE ? const_cast<void*>(a.src_shards[tid]) : a.dst_shards[tid];
  uint64_t pc = 0, ptau = 0;  // producer cursor (thread 0 only)
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    pc = next_item(g, blockIdx.x, G, LOG, ptau);
    for (int s = 0; s < S && pc < g.nloc; ++s) {
      issue_item<T, M, S, OB, WMODE>(g, ptau, in + (size_t)s * C::STAGE, &bars[s], src);
      pc = next_item(g, pc + G, G, LOG, ptau);
    }
  }

  uint32_t i = 0;
  uint64_t ctau = 0;
  for (uint64_t cc = next_item(g, blockIdx.x, G, LOG, ctau); cc < g.nloc;
       cc = next_item(g, cc + G, G, LOG, ctau), ++i) {
    const uint32_t s = i % S;
    const uint32_t parity = (i / S) & 1u;
    T* buf = in + (size_t)s * C::STAGE;
    const T* us = buf + 2 * WIN;  // W pass, unsharded: u at this item's outputs
    const bool u_in_smem = WMODE && g.p == 0;
    T* ob = OB ? out + (size_t)(i % (OB ? OB : 1)) * OUTN : nullptr;
    if (OB && tid == 0) bulk_wait_read<(OB ? OB - 1 : 0)>();  // stores from ob OB items ago have read it
    mbar_wait(&bars[s], parity);
    __syncthreads();
    uint64_t x0, p0, taup;
    tile_info(g, ctau, LOG, x0, p0, taup);
    const bool self = (taup == ctau);
    const uint64_t wb = win_base(g, x0), wp = win_base(g, p0);
    // the six output runs (each lies in one shard)
    void* const* tabs = s_tabs;
    T* runQ1 = out_ptr<T>(g, tabs, x0);
    T* runQ1p = out_ptr<T>(g, tabs, p0);
    T* runF = out_ptr<T>(g, tabs, wb >> 2);
    T* runM = out_ptr<T>(g, tabs, g.q1 - (wb >> 2) - TT / 2);
    T* runFp = out_ptr<T>(g, tabs, wp >> 2);
    T* runMp = out_ptr<T>(g, tabs, g.q1 - (wp >> 2) - TT / 2);

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
      if (WMODE) {
        // W = (u + R) - F'(u); W(psi x) = W(x) exactly (both entries hold the same value)
        const double ux = u_in_smem ? (double)us[o] : (double)runQ1[o];
        wm0 = dmax(wm0, (ux + R0) - v);
        wm1 = dmax(wm1, (ux + R1) - v);
      } else if (OB) {
        ob[o] = (T)v;
        ob[TT + pairswap32(~o & (TT - 1))] = (T)v;
      } else {
        runQ1[o] = (T)v;
        if (!self) runQ1p[pairswap32(~o & (TT - 1))] = (T)v;
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
      if (half == 1 && self) continue;
      T* rf = half ? runFp : runF;
      T* rm = half ? runMp : runM;
      if (WMODE) {
        const double uf = u_in_smem ? (double)us[TT + half * TT + r] : (double)rf[r];
        const double um = u_in_smem ? (double)us[TT + half * TT + TT / 2 + (TT / 2 - 1 - r)]
                                    : (double)rm[TT / 2 - 1 - r];
        wm0 = dmax(wm0, (uf + R0) - fwd);
        wm1 = dmax(wm1, (uf + R1) - fwd);
        wm0 = dmax(wm0, (um + R0) - mir);
        wm1 = dmax(wm1, (um + R1) - mir);
      } else if (OB) {
        T* q0 = ob + 2 * TT + half * TT;
        q0[r] = (T)fwd;
        q0[TT / 2 + (TT / 2 - 1 - r)] = (T)mir;
      } else {
        rf[r] = (T)fwd;
        rm[TT / 2 - 1 - r] = (T)mir;
      }
    }
    if (OB && !WMODE) fence_proxy_async_smem();
    __syncthreads();

    if (tid == 0) {
      if (OB && !WMODE) {  // OB > 0 only when unsharded (launcher enforces)
        constexpr uint32_t QB = TT * sizeof(T), HB = TT / 2 * sizeof(T);
        tma_store_1d(runQ1, ob, QB);
        tma_store_1d(runF, ob + 2 * TT, HB);
        tma_store_1d(runM, ob + 2 * TT + TT / 2, HB);
        if (!self) {
          tma_store_1d(runQ1p, ob + TT, QB);
          tma_store_1d(runFp, ob + 3 * TT, HB);
          tma_store_1d(runMp, ob + 3 * TT + TT / 2, HB);
        }
        bulk_commit();
      }
      if (pc < g.nloc) {  // refill the stage this item just vacated
        issue_item<T, M, S, OB, WMODE>(g, ptau, buf, &bars[s], src);
        pc = next_item(g, pc + G, G, LOG, ptau);
      }
    }
  }
  if (OB && !WMODE && tid == 0) bulk_wait<0>();
  if (!WMODE && g.p > 0) __threadfence_system();  // peer stores visible before the barrier
  if (WMODE) block_max2_to(wm0, wm1, a.red_out);
}

template <typename T, int M, int S, int OB, bool WMODE, int MINB = 1>
cudaError_t launch_tma(const Bin2Args& a, cudaStream_t s, int sms) {
  using C = TmaCfg<T, M, S, OB, WMODE>;
  static uint64_t cap = 0;
  if (cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(bin2_tma_kernel<T, M, S, OB, WMODE, MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm,
                                                      bin2_tma_kernel<T, M, S, OB, WMODE, MINB>,
                                                      kThreads, C::SMEM) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = (uint64_t)per_sm * sms;
  }
  if (!WMODE && OB > 0 && a.shard_bits > 0) return cudaErrorInvalidValue;
  const uint64_t nloc = (1ull << (2 * (a.ell - 1 - M))) >> a.shard_bits;
  uint64_t blocks = cap < nloc ? cap : nloc;
  if (blocks < 1) blocks = 1;
  bin2_tma_kernel<T, M, S, OB, WMODE, MINB><<<(unsigned)blocks, kThreads, C::SMEM, s>>>(a);
  return cudaGetLastError();
}

struct VariantDesc {
  int m, s, ob, mb;  // tile exponent, stages, out buffers, min CTAs/SM (register cap)
};
// (M, S, OB) per variant id, fp32 and fp64 storage
constexpr VariantDesc kF32[] = {{0, 0, 0, 1}, {5, 4, 2, 1}, {4, 8, 2, 1}, {5, 2, 2, 1},
                                {4, 4, 2, 1}, {0, 0, 0, 1}, {5, 1, 2, 1}, {5, 3, 2, 1},
                                {4, 2, 2, 1}, {5, 2, 1, 1}, {5, 1, 1, 1}, {6, 1, 1, 1},
                                {6, 1, 0, 2}, {6, 2, 0, 1}, {5, 2, 0, 1}, {5, 4, 0, 1},
                                {6, 3, 0, 1}, {4, 2, 0, 1}, {6, 1, 0, 3}, {5, 2, 0, 3},
                                {5, 1, 0, 4}, {6, 1, 0, 1}};
constexpr VariantDesc kF64[] = {{0, 0, 0, 1}, {4, 4, 2, 1}, {4, 8, 2, 1}, {4, 2, 2, 1},
                                {3, 8, 2, 1}, {0, 0, 0, 1}, {4, 1, 2, 1}, {4, 3, 2, 1},
                                {5, 1, 1, 1}, {4, 2, 1, 1}, {4, 1, 1, 1}, {3, 4, 2, 1},
                                {5, 1, 0, 1}, {5, 2, 0, 1}, {4, 2, 0, 1}, {4, 4, 0, 1},
                                {5, 3, 0, 1}, {3, 2, 0, 1}, {5, 1, 0, 3}, {4, 2, 0, 3},
                                {5, 1, 1, 3}, {5, 1, 1, 2}};
constexpr int kNumVariants = 22;

}  // namespace

cudaError_t launch_bin2_tma_sweep(const Bin2Args& a, int dtype, int variant, cudaStream_t s,
                                  int sms) {
#define LCSB_V(T, M, S, OB) \
  if (d.m == M && d.s == S && d.ob == OB && d.mb == 1) return launch_tma<T, M, S, OB, false>(a, s, sms);
#define LCSB_VB(T, M, S, OB, MB) \
  if (d.m == M && d.s == S && d.ob == OB && d.mb == MB) return launch_tma<T, M, S, OB, false, MB>(a, s, sms);
  if (variant <= 0 || variant >= kNumVariants) return cudaErrorInvalidValue;
  if (dtype == LCSB_F32) {
    const VariantDesc d = kF32[variant];
    LCSB_V(float, 5, 4, 2) LCSB_V(float, 4, 8, 2) LCSB_V(float, 5, 2, 2) LCSB_V(float, 4, 4, 2)
    LCSB_V(float, 5, 1, 2) LCSB_V(float, 5, 3, 2) LCSB_V(float, 4, 2, 2) LCSB_V(float, 5, 2, 1)
    LCSB_V(float, 5, 1, 1) LCSB_V(float, 6, 1, 1) LCSB_V(float, 6, 1, 0) LCSB_V(float, 6, 2, 0)
    LCSB_V(float, 5, 2, 0) LCSB_V(float, 5, 4, 0) LCSB_V(float, 6, 3, 0) LCSB_V(float, 4, 2, 0)
    LCSB_VB(float, 6, 1, 0, 3) LCSB_VB(float, 5, 2, 0, 3) LCSB_VB(float, 5, 1, 0, 4)
    LCSB_VB(float, 6, 1, 0, 2) LCSB_V(float, 6, 1, 0)
  } else {
    const VariantDesc d = kF64[variant];
    LCSB_V(double, 4, 4, 2) LCSB_V(double, 4, 8, 2) LCSB_V(double, 4, 2, 2) LCSB_V(double, 3, 8, 2)
    LCSB_V(double, 4, 1, 2) LCSB_V(double, 4, 3, 2) LCSB_V(double, 5, 1, 1) LCSB_V(double, 4, 2, 1)
    LCSB_V(double, 4, 1, 1) LCSB_V(double, 3, 4, 2) LCSB_V(double, 5, 1, 0) LCSB_V(double, 5, 2, 0)
    LCSB_V(double, 4, 2, 0) LCSB_V(double, 4, 4, 0) LCSB_V(double, 5, 3, 0) LCSB_V(double, 3, 2, 0)
    LCSB_VB(double, 5, 1, 0, 3) LCSB_VB(double, 4, 2, 0, 3) LCSB_VB(double, 5, 1, 1, 3)
    LCSB_VB(double, 5, 1, 1, 2)
  }
#undef LCSB_V
#undef LCSB_VB
  return cudaErrorInvalidValue;
}

// W pass on the same pipeline (no output staging); M = tile exponent.  Defaults from the A/B
// (tools/ab_wpass.py): fp32 M=6 single stage (2 CTAs/SM), fp64 M=5 two stages;
// LCSB_WPASS_STAGES=1/2 overrides the stage count.
cudaError_t launch_bin2_tma_wpass(const Bin2Args& a, int dtype, int M, cudaStream_t s, int sms) {
  static int stages = -1;
  if (stages < 0) {
    const char* e = getenv("LCSB_WPASS_STAGES");
    stages = e ? atoi(e) : 0;
  }
  const bool one_stage = stages == 1 || (stages == 0 && dtype == LCSB_F32);
  if (dtype == LCSB_F32) {
    if (M == 6) return one_stage ? launch_tma<float, 6, 1, 0, true, 2>(a, s, sms)
                                 : launch_tma<float, 6, 2, 0, true>(a, s, sms);
    if (M == 5) return one_stage ? launch_tma<float, 5, 1, 0, true, 3>(a, s, sms)
                                 : launch_tma<float, 5, 2, 0, true>(a, s, sms);
    if (M == 4) return launch_tma<float, 4, 2, 0, true>(a, s, sms);
    if (M == 3) return launch_tma<float, 3, 2, 0, true>(a, s, sms);
  } else {
    if (M == 5) return one_stage ? launch_tma<double, 5, 1, 0, true, 2>(a, s, sms)
                                 : launch_tma<double, 5, 2, 0, true>(a, s, sms);
    if (M == 4) return launch_tma<double, 4, 2, 0, true>(a, s, sms);
    if (M == 3) return launch_tma<double, 3, 2, 0, true>(a, s, sms);
  }
  return cudaErrorInvalidValue;
}
// largest W-pass tile exponent usable at this l and shard count (0 = none); LCSB_WPASS_M caps it
int bin2_tma_wpass_m(int dtype, int ell, int p) {
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("LCSB_WPASS_M");
    cap = e ? atoi(e) : 6;
  }
  const int ms32[] = {6, 5, 4, 3}, ms64[] = {5, 4, 3, 0};
  const int* ms = (dtype == LCSB_F32) ? ms32 : ms64;
  for (int i = 0; i < 4; ++i)
    if (ms[i] && ms[i] <= cap && ell >= ms[i] + 1 && p < ell - 1 - ms[i]) return ms[i];
  return 0;
}

// smallest l whose Q1 has at least one tile of 4^M outputs (l - 1 >= M); 0 = not a TMA variant
// tile exponent M of a variant (0 = not a TMA variant)
int bin2_tma_m(int dtype, int variant) {
  if (variant <= 0 || variant >= kNumVariants) return 0;
  return (dtype == LCSB_F32) ? kF32[variant].m : kF64[variant].m;
}
// does the variant store straight from registers (required when sharded)
int bin2_tma_direct(int dtype, int variant) {
  if (variant <= 0 || variant >= kNumVariants) return 0;
  const VariantDesc d = (dtype == LCSB_F32) ? kF32[variant] : kF64[variant];
  return d.m > 0 && d.ob == 0;
}

int bin2_tma_min_ell(int dtype, int variant) {
  if (variant <= 0 || variant >= kNumVariants) return 0;
  const VariantDesc d = (dtype == LCSB_F32) ? kF32[variant] : kF64[variant];
  return d.m ? d.m + 1 : 0;
}

}  // namespace lcsbk
