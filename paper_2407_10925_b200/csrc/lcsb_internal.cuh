// lcsb_internal.cuh -- shared declarations of the B200 Feasible Triplet library.
// Product code: never includes or links anything under oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <math.h>

#include <vector>

#include "lcsb.h"

namespace lcsbk {

constexpr int kMaxD = 16;
constexpr int kMaxGen = kMaxD + 1;

// ordered encoding of doubles into uint64 so that unsigned integer max/min == fp max/min
__host__ __device__ inline unsigned long long ord_enc(double x) {
#ifdef __CUDA_ARCH__
  long long b = __double_as_longlong(x);
#else
  long long b;
  memcpy(&b, &x, sizeof b);
#endif
  return b < 0 ? ~(unsigned long long)b : ((unsigned long long)b | 0x8000000000000000ull);
}

inline double ord_dec(unsigned long long u) {
  unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  double x;
  memcpy(&x, &b, sizeof x);
  return x;
}

// Persistent grids: the number of CTAs that are co-resident (SMs x occupancy), so a static
// grid-stride partition has no partial second wave.  Cached per kernel by the caller.
template <typename K>
inline uint64_t resident_blocks(K kernel, int tpb, int sms) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, tpb, 0) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  return (uint64_t)per_sm * (uint64_t)sms;
}

// Integer-offset storage (lcsb_config.offset_policy, readings R23, R26):
// ring slot i holds s = v - off[i]; before each sweep (cur -> out) the prep kernel sets
// c = floor(min s[cur]) (mn[cur], ordered encoding), off[out] = off[cur] + c and shift = -c; the
// sweep stores round(F(s) + shift) and reduces the min of what it stores into mn[out].
// KS form (R26): gpost[k] = off[slot of the table k sweeps back] - off[cur] (an integer) is
// added to every option mean over that table, so F sees every generation relative to o_n, and
// gpost[0] = -off[cur] is the |N| = 0 option's 0 (R3) in stored terms; two-array: all 0.
struct OffState {
  double off[kMaxGen];
  unsigned long long mn[kMaxGen];
  double shift;
  double quantum;  // granularity of c: 1 (integer offsets), 1/64 with residual storage (R24)
  double gpost[kMaxD + 1];
};
// the ring slots of the tables 1..d sweeps back (KS form; the two-array form passes cur)
struct GenSlots {
  int n;
  int slot[kMaxD];
};

// Reduction slots (device, unsigned long long each):
//   0: R_max  1: R_min  2: max W at R_max  3: max W at R_min
constexpr int kRedSlots = 4;

struct GenericArgs {
  int sigma, d, ell;
  uint64_t n;                       // logical states
  const void* src[kMaxD];           // src[k-1]: table read when |N| = k
  void* dst;                        // output table (sweep mode)
  const void* center;               // W mode: the table v in W = (v + dR) - F(...)
  int form;                         // LCSB_FORM_KS / LCSB_FORM_TWO_ARRAY
  const unsigned long long* red_in; // W mode: encoded R_max, R_min
  unsigned long long* red_out;      // W mode: encoded max W slots
  // pooled small sweep (kern_small.cu): pin[k-1] = pooled means of the table read when
  // |N| = k (k >= 2); pout[k-1] = pooled means of the table written
  const double* pin[kMaxD];
  double* pout[kMaxD];
  uint64_t headw_top;               // sigma^(d(l-1)): weight of the head digit group
  // integer offsets (sweep mode): add ost->shift to every output before the storage rounding
  // and reduce the min of the stored values into *omin; NULL = off
  const OffState* ost;
  unsigned long long* omin;
};

constexpr int kMaxShards = 8;

struct Bin2Args {
  const void* src;  // this shard's input half table (unsharded: the whole stored table)
  void* dst;        // output half table (register kernel, unsharded)
  int ell;
  int m;            // register kernel: tile = 4^m Q1 outputs
  int grid_mult;    // register kernel: 0 = co-resident grid, k > 0 = k CTAs per SM
  int shard_bits;   // TMA kernel: 2^shard_bits shards (0 = unsharded)
  int shard;        // TMA kernel: this shard
  void* dst_shards[kMaxShards];        // output table of every shard (unsharded: [0] = dst)
  const void* src_shards[kMaxShards];  // input table of every shard (W pass reads u there)
  const unsigned long long* red_in;
  unsigned long long* red_out;
};

// Sharding of the binary complement-folded half table over 2^p shards.
// Stored index s (a_0 = 0): a_i at bit L-1-2i, b_i at bit L-2-2i.  Shard key
// kappa_i = a_i ^ b_{i-1} ^ 1 (i = 1..p), kappa_1 most significant.  Local index = s with the
// bits a_0..a_p removed (b_0..b_{p-1} become the top p bits).  Every adv_b window and every
// output run of the bin2 kernels lies in one shard, contiguously, when p < l - 1 - M.
__host__ __device__ inline uint32_t shard_of_stored(uint64_t s, int L, int p) {
  uint32_t k = 0;
  for (int i = 1; i <= p; ++i) {
    const uint32_t ai = (uint32_t)(s >> (L - 1 - 2 * i)) & 1u;
    const uint32_t bi1 = (uint32_t)(s >> (L - 2 * i)) & 1u;
    k = (k << 1) | (ai ^ bi1 ^ 1u);
  }
  return k;
}
__host__ __device__ inline uint64_t local_of_stored(uint64_t s, int L, int p) {
  if (p == 0) return s;
  const int lowbits = L - 1 - 2 * p;
  uint64_t top = 0;
  for (int i = 0; i < p; ++i) top = (top << 1) | ((s >> (L - 2 - 2 * i)) & 1ull);
  return (top << lowbits) | (s & ((1ull << lowbits) - 1));
}
__host__ __device__ inline uint64_t global_of_local(uint32_t shard, uint64_t loc, int L, int p) {
  if (p == 0) return loc;
  const int lowbits = L - 1 - 2 * p;
  uint64_t s = loc & ((1ull << lowbits) - 1);
  const uint64_t top = loc >> lowbits;
  for (int i = 0; i < p; ++i) {
    const uint64_t bi = (top >> (p - 1 - i)) & 1ull;
    const uint64_t k = (shard >> (p - 1 - i)) & 1u;
    s |= bi << (L - 2 - 2 * i);
    s |= (k ^ bi ^ 1ull) << (L - 3 - 2 * i);  // a_{i+1}
  }
  return s;
}

// Quarter table (kern_bin2q.cu): the half table cut into blocks of 4^K entries; map[block] =
// (slot << 2) | mode, mode 0 = stored here (canonical), else read from the block stored at
// `slot` through the in-block permutation of the symmetry that maps it there: 1 = string swap s
// (pairswap), 2 = psi = complement o swap (pairswap of the complement; for Q0 blocks the tail
// complement composed with s), 3 = tail complement t of a same-head block (complement).
struct Bin2QArgs {
  const void* src;  // input quarter table (bound pass: v_n)
  void* dst;        // output quarter table (sweep mode)
  const void* prev; // bound pass: v_{n-1}
  const uint32_t* map;
  int ell;
  int K;
  const unsigned long long* red_in;
  unsigned long long* red_out;
  // optional item order (the sweep of tile M == sched_m only): sched[c] = tile index of the c-th
  // tile pair; NULL = the natural order of the pair representatives
  const uint32_t* sched;
  uint64_t nitems;
  int sched_m;
  // optional work counter (zeroed before the launch): CTAs claim items in schedule order with an
  // atomic, so the items in flight stay within about one grid-width of the list; NULL = static
  // round-robin assignment
  unsigned long long* counter;
  int l2keep;  // policy of the pieces the schedule marks as reloaded soon: 0 normal, 1 evict-last
  // integer offsets (sweep mode, as GenericArgs); NULL = off
  const OffState* ost;
  unsigned long long* omin;
  // residual storage (reading R24): the fixed fp32 base H; the tables hold e = v - o - H
  const void* base;
  // set by the launcher: lmask, q1, a-bit mask, b-bit mask, block mask, tiles (kern_bin2q.cuh)
  uint64_t geo[6];
};
// schedule entries: tile index in the low bits, L2 hint bits (one per window piece) at the top
constexpr int kQHintShift = 28;
constexpr uint32_t kQTileMask = (1u << kQHintShift) - 1;

__host__ __device__ inline uint64_t pairswap_hd(uint64_t v) {
  return ((v & 0xAAAAAAAAAAAAAAAAull) >> 1) | ((v & 0x5555555555555555ull) << 1);
}
// Images of half-table block `beta` (prefix of PL = 2(l-K) bits, top bit a_0 = 0 implicit)
// under the symmetries the quarter table folds (reading R19, R18):
//   Q1 blocks (heads 01): psi = complement o swap (pairswap of the complement);
//   Q0 blocks (heads 00): the string swap s, the tail complement t (the same-head value depends
//   only on the tails and is complement-invariant: v'[00t] = v'[00t~]) and s t.
// qblock_image(beta, PL, g) for g = 1 (s), 2 (psi / s t), 3 (t); g = 1, 3 only for Q0 blocks.
__host__ __device__ inline uint64_t qblock_image(uint64_t beta, int PL, int g) {
  const uint64_t pm = (1ull << PL) - 1;
  const uint64_t tail = (1ull << (PL - 2)) - 1;  // every prefix digit but the heads
  const bool q1 = (beta >> (PL - 2)) & 1ull;
  if (q1) return pairswap_hd(~beta & pm) & pm;  // psi (heads 01 -> 01)
  if (g == 1) return pairswap_hd(beta) & pm;
  if (g == 3) return beta ^ tail;
  return pairswap_hd(beta ^ tail) & pm;  // s t
}
// stored index of half-table index s (map as above)
__host__ __device__ inline uint64_t qstored(const uint32_t* map, uint64_t s, int K) {
  const uint32_t m = map[s >> (2 * K)];
  const uint64_t kmask = (1ull << (2 * K)) - 1;
  uint64_t e = s & kmask;
  if ((m & 3u) == 1u) e = pairswap_hd(e) & kmask;
  else if ((m & 3u) == 2u) e = pairswap_hd(~e & kmask) & kmask;
  else if ((m & 3u) == 3u) e = ~e & kmask;
  return ((uint64_t)(m >> 2) << (2 * K)) | e;
}

// quarter_host.cu: the folded table's stored sizes, block map and item schedule
uint64_t quarter_map_entries(int ell, int K);  // half-table blocks of 4^K entries
uint64_t quarter_slots(int ell, int K);        // stored (canonical) blocks
bool build_quarter_map(int ell, int K, uint32_t* map);
bool quarter_schedule(int ell, int K, int M, const uint32_t* map, std::vector<uint32_t>& out);
bool quarter_schedule_cached(int ell, int K, int M, std::vector<uint32_t>& out);  // no build
// sharded quarter table: shard-major slots with a stride of the largest shard
// passes > 0: local-search refinement of the assignment (fewer NVLink bytes), deterministic
bool build_quarter_map_sharded(int ell, int K, int M, int p, int passes, uint32_t* map,
                               uint64_t* stride_slots);
uint64_t quarter_shard_maxslots(int ell, int K, int p);
void quarter_shard_items(int ell, int K, int M, const uint32_t* map, uint64_t maxslots, int shard,
                         const std::vector<uint32_t>& sched, std::vector<uint32_t>& out);
void quarter_shard_traffic(int ell, int K, int M, const uint32_t* map, uint64_t maxslots,
                           int shard, const std::vector<uint32_t>& items, uint64_t out[3]);

// vmm.cu: one virtual address range over the shards of a table (shard k at k * stride)
struct VmmTable {
  void* base;
  size_t stride;
  int P, device;
  unsigned long long handle[kMaxShards];
  int mapped[kMaxShards];
};
size_t vmm_granularity(int device);
bool vmm_reserve(VmmTable* t, int P, size_t stride, int device, char* why, size_t wl);
bool vmm_create_shard(VmmTable* t, int k, bool exportable, char* why, size_t wl);
bool vmm_export_fd(VmmTable* t, int k, int* fd, char* why, size_t wl);
bool vmm_import_fd(VmmTable* t, int k, int fd, char* why, size_t wl);
void vmm_release(VmmTable* t);
int fdx_listen(uint64_t token, int rank, char* why, size_t wl);
bool fdx_send(uint64_t token, int from, int to, const int* fds, int n, char* why, size_t wl);
bool fdx_recv(int lsock, int* from, int* fds, int n, char* why, size_t wl);

// Sharding of the sigma = 4, d = 2 complement-folded table over 2^p shards.
// State s: 4l bits, character group g (g = 0 the heads) at bits [4(l-1-g), 4(l-g)), the a digit
// in the top 2 bits of a group.  Key (p = 1, 2, 3): k = a_1 ^ b_0 (2 bits; p = 1: its top bit),
// p = 3 appends the top bit of a_2 ^ b_1.  Both windows of every unit of a q4 item group
// {u, su, cu, csu} have the key a_1 ^ b_1 (... a_2 ^ b_2) of the unit's first tail groups -- the
// digit swap and the complement d -> 3 - d = d ^ 3 leave a XOR of two digits unchanged -- so
// every sweep reads only its own shard; outputs and row means are pushed to their owners.
// Local index: the state with the a_1 digit (p = 1: its top bit) and, for p = 3, the top bit of
// a_2 removed.  Row means (index r = s >> 4 over stored rows, top group (a_0 < 2, b_0)): key
// r.a_0 ^ r.b_0 (p = 3: + top bit of r.a_1 ^ r.b_1) = the key of the items that read them; local
// row index: r with b_0 (p = 1: its top bit) and, for p = 3, the top bit of b_1 removed.
__host__ __device__ inline uint64_t del_bits(uint64_t x, int q, int n) {  // drop bits [q, q+n)
  return ((x >> (q + n)) << q) | (x & ((1ull << q) - 1));
}
// digit of group g (a: ab = 1, b: ab = 0) of an index of `bits` bits
__host__ __device__ inline uint32_t q4dig(uint64_t s, int bits, int g, int ab) {
  return (uint32_t)(s >> (bits - 4 * g - 4 + 2 * ab)) & 3u;
}
__host__ __device__ inline uint32_t q4_key(uint64_t s, int ell, int p) {  // stored state
  const int L = 4 * ell;
  if (p == 0) return 0;
  const uint32_t k1 = q4dig(s, L, 1, 1) ^ q4dig(s, L, 0, 0);
  if (p == 1) return k1 >> 1;
  if (p == 2) return k1;
  return (k1 << 1) | ((q4dig(s, L, 2, 1) ^ q4dig(s, L, 1, 0)) >> 1);
}
__host__ __device__ inline uint64_t q4_local(uint64_t s, int ell, int p) {
  const int L = 4 * ell;
  if (p == 0) return s;
  // higher bits first (deleting a bit shifts everything above it)
  s = p == 1 ? del_bits(s, L - 5, 1) : del_bits(s, L - 6, 2);  // a_1 (p = 1: its top bit)
  if (p == 3) s = del_bits(s, L - 9, 1);                      // top bit of a_2
  return s;
}
__host__ __device__ inline uint32_t q4_mkey(uint64_t r, int ell, int p) {  // row-mean index
  const int R = 4 * (ell - 1);
  if (p == 0) return 0;
  const uint32_t k1 = q4dig(r, R, 0, 1) ^ q4dig(r, R, 0, 0);
  if (p == 1) return k1 >> 1;
  if (p == 2) return k1;
  return (k1 << 1) | ((q4dig(r, R, 1, 1) ^ q4dig(r, R, 1, 0)) >> 1);
}
__host__ __device__ inline uint64_t q4_mlocal(uint64_t r, int ell, int p) {
  const int R = 4 * (ell - 1);
  if (p == 0) return r;
  r = p == 1 ? del_bits(r, R - 3, 1) : del_bits(r, R - 4, 2);  // b_0 (p = 1: its top bit)
  if (p == 3) r = del_bits(r, R - 7, 1);                      // top bit of b_1
  return r;
}

struct Q4Args {
  const void* g1;     // table one sweep back (W pass: the newest table); sharded: this shard's
  const double* pin;  // row means (x >> 4) of the table two sweeps back (W pass: of the newest)
  double* pout;       // sweep: row means of the table written
  void* dst;          // output (sweep mode)
  int ell;
  const unsigned long long* red_in;
  unsigned long long* red_out;
  int flags;          // kQ4TwoArray from the caller; kern_q4.cu adds its A/B bits
  // sharded (p > 0): this launch's shard, and every shard's output table / row means (sweep)
  // or newest table (W pass: u at the outputs)
  int p, shard;
  void* dst_sh[kMaxShards];
  double* pout_sh[kMaxShards];
  const void* g1_sh[kMaxShards];
  // integer offsets (sweep; readings R23, R26): P gets gpost[2] (KS: of the table two back),
  // outputs get shift before the storage rounding, the min of the stored values this launch
  // computes goes to omin (sharded: every shard's launch into the same min).  NULL = off
  const OffState* ost;
  unsigned long long* omin;
};
constexpr int kQ4TwoArray = 4;  // Q4Args::flags: two-array form (reading R20)

#ifdef __CUDACC__
// max / min by one compare and a select: the iterates and W values are never NaN, so the NaN
// handling of fmax/fmin (several extra instructions per call in SASS) is dead weight on hot paths
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double dec_ord(unsigned long long u) {
  unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  return __longlong_as_double((long long)b);
}

// block-wide max of two doubles, one atomicMax per block into out[0], out[1] (blockDim % 32 == 0)
__device__ __forceinline__ void block_max2_to(double w0, double w1, unsigned long long* out) {
  __shared__ double s0[32], s1[32];
  for (int o = 16; o > 0; o >>= 1) {
    w0 = dmax(w0, __shfl_xor_sync(0xffffffffu, w0, o));
    w1 = dmax(w1, __shfl_xor_sync(0xffffffffu, w1, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s0[wid] = w0;
    s1[wid] = w1;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
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

// block-wide min of v, one atomicMin (ordered encoding) into *out (blockDim % 32 == 0)
__device__ __forceinline__ void block_min_to(double v, unsigned long long* out) {
  __shared__ double sm[32];
  for (int o = 16; o > 0; o >>= 1) v = dmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? sm[lane] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = dmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) atomicMin(out, ord_enc(v));
  }
}

// block-wide (max a, min b, min c), one atomic each into out[0] (max), out[1], out[2] (min)
__device__ __forceinline__ void block_red3_to(double a, double b, double c,
                                              unsigned long long* out) {
  __shared__ double s0[32], s1[32], s2[32];
  for (int o = 16; o > 0; o >>= 1) {
    a = dmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = dmin(b, __shfl_xor_sync(0xffffffffu, b, o));
    c = dmin(c, __shfl_xor_sync(0xffffffffu, c, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s0[wid] = a;
    s1[wid] = b;
    s2[wid] = c;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    a = lane < nw ? s0[lane] : -INFINITY;
    b = lane < nw ? s1[lane] : INFINITY;
    c = lane < nw ? s2[lane] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      a = dmax(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = dmin(b, __shfl_xor_sync(0xffffffffu, b, o));
      c = dmin(c, __shfl_xor_sync(0xffffffffu, c, o));
    }
    if (lane == 0) {
      atomicMax(out + 0, ord_enc(a));
      atomicMin(out + 1, ord_enc(b));
      atomicMin(out + 2, ord_enc(c));
    }
  }
}
#endif

// launchers (return cudaError_t of the launch)
cudaError_t launch_generic_sweep(const GenericArgs& a, int dtype, cudaStream_t s, int sms);
cudaError_t launch_generic_wpass(const GenericArgs& a, int dtype, cudaStream_t s, int sms);
cudaError_t launch_bin2_sweep(const Bin2Args& a, int dtype, cudaStream_t s, int sms);
cudaError_t launch_bin2_wpass(const Bin2Args& a, int dtype, cudaStream_t s, int sms);
cudaError_t launch_bin2_tma_sweep(const Bin2Args& a, int dtype, int variant, cudaStream_t s,
                                  int sms);
int bin2_tma_min_ell(int dtype, int variant);
int bin2_tma_m(int dtype, int variant);
int bin2_tma_direct(int dtype, int variant);
cudaError_t launch_bin2_tma_wpass(const Bin2Args& a, int dtype, int M, cudaStream_t s, int sms);
int bin2_tma_wpass_m(int dtype, int ell, int p);
// variant 0: the default pipeline for tile 4^M; v > 0: the (M, stages, CTAs/SM) of table entry v
cudaError_t launch_bin2q_sweep(const Bin2QArgs& a, int dtype, int M, int variant, cudaStream_t s,
                               int sms);
int bin2q_variant_m(int dtype, int variant);
cudaError_t launch_bin2q_wpass(const Bin2QArgs& a, int dtype, int M, cudaStream_t s, int sms);
// the tracking sweep (kern_bin2q_diff.cu): the plain sweep that also reduces, against the table it
// reads at every stored output, R of the iterate it writes and D of the one it reads (red_out[0..2])
cudaError_t launch_bin2q_diff(const Bin2QArgs& a, int dtype, int M, cudaStream_t s, int sms);
// the sweep with integer offsets (a.ost) or residual storage (a.base): kern_bin2q_ext.cu
cudaError_t launch_bin2q_sweep_ext(const Bin2QArgs& a, int dtype, int M, cudaStream_t s, int sms);
cudaError_t launch_q4_sweep(const Q4Args& a, int dtype, cudaStream_t s, int sms);
cudaError_t launch_q4_wpass(const Q4Args& a, int dtype, cudaStream_t s, int sms);
int q4_min_ell();
bool small_supported(int sigma, int d, uint64_t n);
cudaError_t launch_small(const GenericArgs& a, int dtype, bool wpass, cudaStream_t s, int sms);
bool small_pooled_supported(int sigma, int d);
uint32_t small_pool_per_row(int sigma, int d, int k);  // pooled means per row for |N| = k
cudaError_t launch_small_pooled(const GenericArgs& a, int dtype, cudaStream_t s, int sms);
// slots whose bit is set in min_mask start at +inf (minima), the others at -inf (maxima)
cudaError_t launch_red_init(unsigned long long* red, cudaStream_t s, unsigned min_mask = 2u);
// integer offsets: zero every slot's offset, min(s) = 0 (the zero tables of W_0), shift 0
cudaError_t launch_offset_init(OffState* o, cudaStream_t s);
// before a sweep cur -> out: c = floor(min s[cur]), off[out] = off[cur] + c, shift = -c,
// mn[out] = +inf (the sweep reduces into it); gens->n > 0 (KS): gpost[0] = -off[cur] and
// gpost[k] = off[gens.slot[k-1]] - off[cur] for 1 <= k <= gens.n; otherwise all 0
cudaError_t launch_offset_prep(OffState* o, int cur, int out, cudaStream_t s,
                               const GenSlots* gens = nullptr);
// residual storage: H = round32(H + e), e = (H + e) - H (both fp32 arrays of n entries)
cudaError_t launch_rebase_fold(void* H, void* e, uint64_t n, cudaStream_t s, int sms);
cudaError_t launch_rdiff(const void* newest, const void* prev, uint64_t n, int dtype,
                         unsigned long long* red, cudaStream_t s, int sms);
// tabs[k]: the table of shard k (unsharded: tabs[0]); p = log2(shards); qmap != NULL: quarter
// table with blocks of 4^K
// symmetric: the table holds the logical states [0, nlogical/2); y >= nlogical/2 reads
// nlogical-1-y (the complement: Eq. comp_eq for sigma = 2, d -> 3-d for sigma = 4)
// q4: sigma = 4 digit-key shards (q4_key / q4_local) instead of the binary key
cudaError_t launch_expand(const void* const* tabs, int p, int dtype, int symmetric, int q4,
                          const double* add,  // integer offsets: added to every value (or NULL)
                          const void* base,   // residual storage: the base table (or NULL)
                          uint64_t nlogical, int ell,
                          const uint32_t* qmap, int K, uint64_t first, uint64_t count,
                          const uint64_t* idx, double* out, cudaStream_t s);

}  // namespace lcsbk
