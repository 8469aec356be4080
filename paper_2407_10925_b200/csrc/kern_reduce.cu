// kern_reduce.cu -- bound reductions and table read-out.
//
//  rdiff:  R_max = max_j (v_new - v_prev)[j], R_min = min_j (...)   (Alg. 2 line 5, Alg. 5 line 7;
//          PAPER.md:705, 738; R_min per PAPER.md:694).  Over stored entries: with the
//          complement-folded table every logical entry equals a stored one, so the max/min are
//          the logical ones.  Differences are exact in fp64 for fp32 storage.
//          Grid-stride, 16-byte vector loads, warp shuffle + block reduction, one atomic per
//          block on order-preserving integer encodings (max/min are exact and order-free, so the
//          result is independent of the launch geometry).
//  expand: logical-order read-out, unfolding the complement symmetry and,
//          for the quarter table, the string swap (reading R19); widening to fp64.
#include <math.h>

#include "lcsb_internal.cuh"

namespace lcsbk {
namespace {

__global__ void red_init_kernel(unsigned long long* red, unsigned min_mask) {
  int i = threadIdx.x;
  if (i < kRedSlots) {
    // minima (slot 1 = R_min; slot 2 = min(F(u) - u) of the one-pass bound) start at +inf, the
    // maxima at -inf
    red[i] = ((min_mask >> i) & 1u) ? ord_enc(INFINITY) : ord_enc(-INFINITY);
  }
}

__global__ void offset_init_kernel(OffState* o) {
  const int i = threadIdx.x;
  if (i < kMaxGen) {
    o->off[i] = 0.0;
    o->mn[i] = ord_enc(0.0);
  }
  if (i <= kMaxD) o->gpost[i] = 0.0;
  if (i == 0) {
    o->shift = 0.0;
    o->quantum = 1.0;
  }
}

__global__ void offset_prep_kernel(OffState* o, int cur, int out, GenSlots g) {
  // KS (reading R26): generation k is read relative to o_n = off[cur] (integers: exact)
  o->gpost[0] = g.n > 0 ? -o->off[cur] : 0.0;
  for (int k = 1; k <= kMaxD; ++k)
    o->gpost[k] = k <= g.n ? o->off[g.slot[k - 1]] - o->off[cur] : 0.0;
  const double m = dec_ord(o->mn[cur]);
  // a multiple of the quantum (1, or 1/64 after a rebase): exact, and so is every shift by it
  const double q = o->quantum;
  const double c = floor(m / q) * q;
  o->off[out] = o->off[cur] + c;
  o->shift = -c;
  o->mn[out] = ord_enc(INFINITY);
}

// residual storage, rebase of a rebased table (reading R24): H' = round32(H + e) and
// e' = (H + e) - H' (exact: the rounding residual of a 35-bit value has <= 24 significant bits)
__global__ void rebase_fold_kernel(float* __restrict__ H, float* __restrict__ e, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = (double)H[i] + (double)e[i];
    const float h2 = (float)v;
    H[i] = h2;
    e[i] = (float)(v - (double)h2);
  }
}

__device__ __forceinline__ void acc(double dd, double& mx, double& mn) {
  mx = dmax(mx, dd);
  mn = dmin(mn, dd);
}

template <typename T>
__global__ void __launch_bounds__(256) rdiff_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                    uint64_t n, unsigned long long* red) {
  double mx = -INFINITY, mn = INFINITY;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sizeof(T) == 4) {
    const uint64_t nv = n / 4;
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    for (uint64_t i = t0; i < nv; i += stride) {
      float4 x = __ldcs(a4 + i), y = __ldcs(b4 + i);
      acc((double)x.x - (double)y.x, mx, mn);
      acc((double)x.y - (double)y.y, mx, mn);
      acc((double)x.z - (double)y.z, mx, mn);
      acc((double)x.w - (double)y.w, mx, mn);
    }
    for (uint64_t i = nv * 4 + t0; i < n; i += stride) acc((double)a[i] - (double)b[i], mx, mn);
  } else {
    const uint64_t nv = n / 2;
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* b2 = reinterpret_cast<const double2*>(b);
    for (uint64_t i = t0; i < nv; i += stride) {
      double2 x = __ldcs(a2 + i), y = __ldcs(b2 + i);
      acc((double)x.x - (double)y.x, mx, mn);
      acc((double)x.y - (double)y.y, mx, mn);
    }
    for (uint64_t i = nv * 2 + t0; i < n; i += stride) acc((double)a[i] - (double)b[i], mx, mn);
  }
  __shared__ double smx[8], smn[8];
  for (int o = 16; o > 0; o >>= 1) {
    mx = dmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = dmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    smx[wid] = mx;
    smn[wid] = mn;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    mx = lane < nw ? smx[lane] : -INFINITY;
    mn = lane < nw ? smn[lane] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      mx = dmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = dmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
      atomicMax(red + 0, ord_enc(mx));
      atomicMin(red + 1, ord_enc(mn));
    }
  }
}

struct ExpandTabs {
  const void* t[kMaxShards];
};

template <typename T>
__global__ void expand_kernel(ExpandTabs tabs, int p, int symmetric, int q4,
                              const double* __restrict__ add, const T* __restrict__ base,
                              uint64_t nlogical, int ell,
                              const uint32_t* __restrict__ qmap, int K, uint64_t first,
                              uint64_t count, const uint64_t* __restrict__ idx, double* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const double off = add ? *add : 0.0;  // integer offset of the generation (exact)
  const uint64_t half = symmetric ? nlogical / 2 : 0;
  const uint64_t top = symmetric ? nlogical - 1 : 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    uint64_t y = idx ? idx[i] : first + i;
    if (symmetric && y >= half) y = top - y;  // Eq. (comp_eq)
    if (qmap) {  // quarter table: the orbit representative under the string swap / psi
      const uint64_t q = qstored(qmap, y, K);
      // residual storage (R24): v = H + e + o, H + e exact in fp64
      const double hb = base ? (double)base[q] : 0.0;
      out[i] = (hb + (double)reinterpret_cast<const T*>(tabs.t[0])[q]) + off;
      continue;
    }
    if (q4) {  // sigma = 4 digit-key shards
      out[i] = (double)reinterpret_cast<const T*>(tabs.t[q4_key(y, ell, p)])[q4_local(y, ell, p)] +
               off;
      continue;
    }
    const uint32_t sh = shard_of_stored(y, 2 * ell, p);
    out[i] = (double)reinterpret_cast<const T*>(tabs.t[sh])[local_of_stored(y, 2 * ell, p)] + off;
  }
}

}  // namespace

cudaError_t launch_red_init(unsigned long long* red, cudaStream_t s, unsigned min_mask) {
  red_init_kernel<<<1, 32, 0, s>>>(red, min_mask);
  return cudaGetLastError();
}

cudaError_t launch_rdiff(const void* newest, const void* prev, uint64_t n, int dtype,
                         unsigned long long* red, cudaStream_t s, int sms) {
  uint64_t per = (dtype == LCSB_F32) ? 4 : 2;
  uint64_t blocks = (n / per + 255) / 256;
  static uint64_t cap_f = 0, cap_d = 0;
  if (!cap_f) cap_f = resident_blocks(rdiff_kernel<float>, 256, sms);
  if (!cap_d) cap_d = resident_blocks(rdiff_kernel<double>, 256, sms);
  const uint64_t cap = (dtype == LCSB_F32) ? cap_f : cap_d;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (dtype == LCSB_F32)
    rdiff_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)newest, (const float*)prev, n, red);
  else
    rdiff_kernel<double><<<(unsigned)blocks, 256, 0, s>>>((const double*)newest, (const double*)prev, n, red);
  return cudaGetLastError();
}

cudaError_t launch_offset_init(OffState* o, cudaStream_t s) {
  offset_init_kernel<<<1, 32, 0, s>>>(o);
  return cudaGetLastError();
}
cudaError_t launch_offset_prep(OffState* o, int cur, int out, cudaStream_t s,
                               const GenSlots* gens) {
  GenSlots g{};
  if (gens) g = *gens;
  offset_prep_kernel<<<1, 1, 0, s>>>(o, cur, out, g);
  return cudaGetLastError();
}

cudaError_t launch_rebase_fold(void* H, void* e, uint64_t n, cudaStream_t s, int sms) {
  uint64_t blocks = (n + 255) / 256;
  const uint64_t cap = (uint64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  rebase_fold_kernel<<<(unsigned)blocks, 256, 0, s>>>((float*)H, (float*)e, n);
  return cudaGetLastError();
}

cudaError_t launch_expand(const void* const* tabs, int p, int dtype, int symmetric, int q4,
                          const double* add, const void* base, uint64_t nlogical, int ell,
                          const uint32_t* qmap, int K, uint64_t first, uint64_t count,
                          const uint64_t* idx, double* out, cudaStream_t s) {
  uint64_t blocks = (count + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  ExpandTabs t;
  for (int k = 0; k < kMaxShards; ++k) t.t[k] = (k < (1 << p)) ? tabs[k] : nullptr;
  if (dtype == LCSB_F32)
    expand_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(t, p, symmetric, q4, add, (const float*)base, nlogical, ell, qmap, K, first, count, idx, out);
  else
    expand_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(t, p, symmetric, q4, add, (const double*)base, nlogical, ell, qmap, K, first, count, idx, out);
  return cudaGetLastError();
}

}  // namespace lcsbk
