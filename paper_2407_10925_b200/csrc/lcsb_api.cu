// lcsb_api.cu -- the C-ABI of include/lcsb.h: handle, table ring, shards, kernel dispatch and the
// bound bookkeeping.  Host code only enqueues work; the whole sweep / bound path runs in the
// kernels of kern_*.cu.  No CPU fallback exists: every entry point fails with LCSB_ECUDA when the
// device work cannot be enqueued.
#include <math.h>
#include <stddef.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <atomic>
#include <new>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler is attached

#include "lcsb_internal.cuh"

namespace lcsbk {
int bin2_tile_m(int ell);
}

using namespace lcsbk;

enum { MODE_SINGLE = 0, MODE_VIRTUAL = 1, MODE_PROCESS = 2 };

struct lcsb {
  lcsb_config cfg;
  int device;
  int sms;
  int form;       // resolved LCSB_FORM_KS / LCSB_FORM_TWO_ARRAY
  int symmetric;  // 1 complement-folded half table, 2 quarter table
  int kernel;     // 1 generic, 2 bin2, 3 q4, 4 small, 5 bin2q
  int qK, qM;     // quarter table: blocks of 4^qK, tiles of 4^qM
  uint32_t* qmap; // quarter table: device block map
  size_t qmap_bytes;
  uint32_t* qsched;  // quarter table: item order of the sweep (NULL = natural order)
  size_t qsched_bytes;
  uint64_t qsched_n;
  // sharded quarter table: each table is one virtual address range over the
  // shards (vt[ring slot]); shard k's items in their own list (the L2 order filtered by owner)
  int vmm;
  VmmTable vt[kMaxGen];
  uint64_t qmaxslots;  // stored blocks per shard stride
  uint64_t peer_read, peer_written, all_moved;  // per sweep, this rank's shards, entries
  uint32_t* qsched_sh[kMaxShards];
  size_t qsched_bytes_sh[kMaxShards];
  uint64_t qsched_n_sh[kMaxShards];
  unsigned long long* qcounter;  // quarter table: work counter of the scheduled kernels
  // the schedule is built on a host thread (lcsb_create returns without waiting for it); the
  // sweeps run in the natural item order -- identical results -- until install_schedule
  // uploads it at the start of a later call
  std::thread* qthread;
  std::atomic<int>* qready;
  std::vector<uint32_t>* qpending;
  int bin2_variant;  // 0 auto; see pick_bin2_variant
  int bin2q_variant; // 0 auto; LCSB_BIN2Q_VARIANT (A/B only)
  uint64_t n_logical;
  uint64_t n_stored;  // entries of the whole stored table
  uint64_t n_local;   // entries per shard
  size_t esize;
  int ntab;           // tables in the ring
  // kernel 3 (q4, pooled-history KS): ring of 3 row-mean arrays (fp64, n/16 entries each);
  // pools[k][pcur] holds the row means of the newest table (shard k's rows when sharded)
  double* pools[kMaxShards][3];
  size_t pool_bytes;  // per shard
  int pcur;
  // kernel 4 (small, KS, pooled sweep): spools[k][slot] = pooled means (|N| = k >= 2) of the
  // table in ring slot `slot` (kern_small.cu)
  int spooled;
  double* spools[kMaxD + 1][kMaxGen];
  size_t spool_bytes[kMaxD + 1];
  int p, P;           // shards: P = 2^p
  int mode;           // MODE_*
  int first, nown;    // owned shards [first, first + nown)
  void* tabs[kMaxShards][kMaxGen];
  size_t tab_bytes;   // bytes per shard table
  int cur;            // ring slot of the newest table
  unsigned long long* red;       // device reduction slots
  unsigned long long red_host[kRedSlots];  // pageable: a 32-byte read-back needs no pinning
  ncclComm_t comm;
  int* barrier_buf;
  // CUDA-graph replay of G consecutive sweeps for launch-latency-bound (small) tables
  cudaStream_t cap_stream;
  int cap_capturing;  // inside a graph capture: no allocation / upload may happen
  OffState* ost;      // integer offsets (reading R23): per-slot offsets, mins, shift; NULL = off
  void* base;         // residual storage (reading R24): the fixed fp32 base H; NULL = off
  int64_t rebase_sweep;  // sweeps_done at the rebase (the previous generation is invalid there)
  cudaGraphExec_t graph[kMaxGen];
  int graph_sweeps;
  int64_t sweeps_done;
  // tracking sweeps (quarter table, kern_bin2q_diff.cu): set j = k & 1 of the reduction slots
  // (red + kTrkSlot + 4 j: R_max, R_min of v_k - v_{k-1}, D = min(F(v_{k-1}) - v_{k-1})) holds
  // the values of sweep k = trk_at[j]; -1 = none
  int64_t trk_at[2];
  int64_t launches;
  double best_rho[2];
  int64_t best_sweep[2];
  char err[512];
};

static thread_local char g_err[512] = "";

// NVTX ranges (SURVEY §5 tracing): each public call, each sweep enqueue and each barrier shows
// up on an nsys / ncu timeline (host ranges; the kernels correlate through the CUDA API)
struct NvtxRange {
  explicit NvtxRange(const char* m) { nvtxRangePushA(m); }
  ~NvtxRange() { nvtxRangePop(); }
};

static int set_err(lcsb_t* h, int code, const char* fmt, ...) {
  char* buf = h ? h->err : g_err;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, 512, fmt, ap);
  va_end(ap);
  if (h) snprintf(g_err, sizeof g_err, "%s", h->err);
  return code;
}

#define CU(h, call)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return set_err((h), LCSB_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define NC(h, call)                                                                     \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      return set_err((h), LCSB_ENCCL, "%s failed: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

static bool mul_ok(uint64_t a, uint64_t b, uint64_t* out) {
  if (a != 0 && b > (~0ull) / a) return false;
  *out = a * b;
  return true;
}

extern "C" void lcsb_config_init(lcsb_config* c) {
  if (!c) return;
  memset(c, 0, sizeof *c);
  c->sigma = 2;
  c->d = 2;
  c->ell = 1;
  c->dtype = LCSB_F32;
  c->form = LCSB_FORM_AUTO;
  c->rmode = LCSB_R_MAX;
  c->symmetry = -1;
  c->kernel = LCSB_KERNEL_AUTO;
  c->shards = 1;
}

// ---------------------------------------------------------------- bin2 variant choice
// Auto choice of the bin2 sweep variant, from the A/B measurements on B200:
// fp32 -> (M=6, 1 stage, direct stores), 97% of the measured copy bandwidth at l=17;
// fp64 -> (M=5, 1 stage, smem-staged bulk stores, 3 CTAs/SM), 97% at l=16; smaller tiles for
// small l;
// the register kernel below that.  Sharded runs need direct stores (outputs go to peers) and
// a tile small enough that the shard key bits sit above it (p < l - 1 - M).
static int pick_bin2_variant(int dtype, int ell, int p) {
  static const int f32_chain[] = {12, 14, 8};
  static const int f64_chain[] = {20, 3, 4};
  static const int direct_chain[] = {12, 14, 17};
  const int* chain = p > 0 ? direct_chain : (dtype == LCSB_F32 ? f32_chain : f64_chain);
  for (int i = 0; i < 3; ++i) {
    const int v = chain[i];
    const int M = bin2_tma_m(dtype, v);
    // small tables: keep >= ~256 tile pairs so every SM has work (M <= l - 6)
    if (p == 0 && M > ell - 6) continue;
    if (M > 0 && ell >= M + 1 && p < ell - 1 - M) return v;
  }
  return p > 0 ? 0 : 5;  // 5 = register kernel (unsharded only); 0 = none
}

// ---------------------------------------------------------------- quarter table layout
// Auto choice: the quarter table from this l up, the half table below.
static const int kQuarterAutoEll = 12;
// (sizes, block map and item schedule: quarter_host.cu)

// ---------------------------------------------------------------- planning
struct Plan {
  int form, symmetric, kernel, ntab, p, P, mode, qK, qM, dtype_code, offsets;
  uint64_t n_logical, n_stored, n_local;
  size_t esize;
  uint64_t bytes;  // device bytes this handle allocates
};

static int log2_exact(int v) {
  int p = 0;
  while ((1 << p) < v) ++p;
  return (1 << p) == v ? p : -1;
}

static int plan_config(const lcsb_config* c, Plan* p, char* why, size_t whylen) {
  if (!c) {
    snprintf(why, whylen, "config is NULL");
    return LCSB_EINVAL;
  }
  if (c->sigma < 2 || c->sigma > 64 || c->d < 2 || c->d > kMaxD || c->ell < 1) {
    snprintf(why, whylen, "need 2 <= sigma <= 64, 2 <= d <= %d, ell >= 1 (got %d, %d, %d)", kMaxD,
             c->sigma, c->d, c->ell);
    return LCSB_EINVAL;
  }
  uint64_t n = 1;
  for (int i = 0; i < c->d * c->ell; ++i) {
    if (!mul_ok(n, (uint64_t)c->sigma, &n) || n >= (1ull << 62)) {
      snprintf(why, whylen, "sigma^(d*ell) must be < 2^62");
      return LCSB_EINVAL;
    }
  }
  if (c->dtype != LCSB_F32 && c->dtype != LCSB_F64) {
    snprintf(why, whylen, "dtype must be LCSB_F32 or LCSB_F64");
    return LCSB_EINVAL;
  }
  if (c->rmode != LCSB_R_MAX && c->rmode != LCSB_R_MIN) {
    snprintf(why, whylen, "rmode must be LCSB_R_MAX or LCSB_R_MIN");
    return LCSB_EINVAL;
  }
  const bool binary = (c->sigma == 2 && c->d == 2);
  int form = c->form;
  if (form == LCSB_FORM_AUTO) form = binary ? LCSB_FORM_TWO_ARRAY : LCSB_FORM_KS;
  if (form != LCSB_FORM_KS && form != LCSB_FORM_TWO_ARRAY) {
    snprintf(why, whylen, "unknown form %d", c->form);
    return LCSB_EINVAL;
  }
  if (form == LCSB_FORM_TWO_ARRAY && c->d != 2) {
    snprintf(why, whylen,
             "the two-array form is defined for d = 2 only (PAPER.md:400; sigma > 2: reading R20)");
    return LCSB_EINVAL;
  }
  if (c->kernel != LCSB_KERNEL_AUTO && c->kernel != LCSB_KERNEL_GENERIC) {
    snprintf(why, whylen, "unknown kernel %d", c->kernel);
    return LCSB_EINVAL;
  }
  const bool sym_ok =
      binary && (form == LCSB_FORM_TWO_ARRAY) && c->ell >= 2 && c->kernel == LCSB_KERNEL_AUTO;
  const int P = c->shards < 1 ? 1 : c->shards;
  const bool has_comm = c->nccl_id || c->comm;
  if (c->comm && (!c->comm->allgather || !c->comm->barrier || !c->comm->allreduce_max_u64)) {
    snprintf(why, whylen, "comm hooks need allgather, barrier and allreduce_max_u64");
    return LCSB_EINVAL;
  }
  const bool sharded = P > 1 || (has_comm && !c->virtual_shards);
  const int lp0 = log2_exact(P);
  // quarter table geometry: blocks of 4^K, tiles of 4^M (M <= K - 1)
  int qK = c->block_log4;
  if (qK <= 0) {
    qK = c->ell - 5;
    const int kmax = (c->dtype == LCSB_F32) ? 7 : 6;
    if (qK > kmax) qK = kmax;
    if (qK < 2) qK = 2;
  }
  const int qM = qK - 1 < ((c->dtype == LCSB_F32) ? 6 : 5) ? qK - 1 : ((c->dtype == LCSB_F32) ? 6 : 5);
  // the item schedule packs a tile index into kQHintShift bits, so the tiles of 4^qM must number
  // at most 2^kQHintShift (larger counts would alias tiles)
  // sharded (§9c): the shard key needs p non-head pairs in a block prefix (l - K - 1 >= p)
  const bool quarter_ok = sym_ok && qK >= 2 && qK <= c->ell - 1 && c->ell - qK <= 16 &&
                          2 * (c->ell - 1 - qM) <= kQHintShift &&
                          (!sharded || (lp0 >= 0 && c->ell - qK - 1 >= lp0));
  // integer offsets (readings R23, R26): unsharded; the quarter table (two-array binary) or the
  // generic kernel (either form; KS with per-generation offsets) carry the shift and min
  const int ofs = c->offset_policy;
  if (ofs != 0 && ofs != 1) {
    snprintf(why, whylen, "offset_policy must be 0 or 1");
    return LCSB_EINVAL;
  }
  // sharded: the quarter table and sigma = 4, d = 2 (their kernels carry the offsets; the min
  // crosses the ranks before each sweep's prep), not the half table
  const bool ofs_shard_ok = (c->sigma == 4 && c->d == 2) ||
                            (c->sigma == 2 && c->d == 2 && form == LCSB_FORM_TWO_ARRAY &&
                             (c->symmetry == 2 || c->symmetry == -1));
  if (ofs && ((sharded && !ofs_shard_ok) || c->symmetry == 1 ||
              (form != LCSB_FORM_TWO_ARRAY && c->symmetry == 2))) {
    snprintf(why, whylen,
             "integer offsets need symmetry -1, 0 or 2 (2: the two-array form) and, sharded, the "
             "quarter table or sigma = 4, d = 2");
    return LCSB_EINVAL;
  }
  int sym = c->symmetry;
  if (sym < 0 && ofs) sym = quarter_ok ? 2 : 0;
  if (sym < 0) sym = (quarter_ok && c->ell >= kQuarterAutoEll) ? 2 : (sym_ok ? 1 : 0);
  if (sym == 1 && !sym_ok) {
    snprintf(why, whylen,
             "the complement-folded table needs the two-array binary form, ell >= 2 and the "
             "AUTO kernel");
    return LCSB_EINVAL;
  }
  if (sym == 2 && !quarter_ok) {
    snprintf(why, whylen,
             "the quarter table needs the two-array binary form, the AUTO kernel, "
             "2 <= block_log4 <= ell - 1 (ell - block_log4 <= 16, at most 2^28 tiles of "
             "4^(block_log4 - 1)) and, sharded, ell - block_log4 - 1 >= log2(shards)");
    return LCSB_EINVAL;
  }
  if (sym < 0 || sym > 2) {
    snprintf(why, whylen, "symmetry must be -1, 0, 1 or 2");
    return LCSB_EINVAL;
  }
  const int lp = log2_exact(P);
  if (lp < 0 || P > kMaxShards) {
    snprintf(why, whylen, "shards must be 1, 2, 4 or 8");
    return LCSB_EINVAL;
  }
  // sigma = 4, d = 2 (q4) shards by a digit key of the first characters: the
  // unit of 16^2 tails must leave the key's tail groups above it (one group for p <= 2, two for
  // p = 3)
  const bool q4_shard = c->sigma == 4 && c->d == 2 && c->kernel == LCSB_KERNEL_AUTO &&
                        c->ell >= q4_min_ell() && c->ell >= (lp == 3 ? 5 : 4);
  if (sharded && q4_shard) {
    if (!c->virtual_shards && (c->shard < 0 || c->shard >= P)) {
      snprintf(why, whylen, "shard must be in [0, %d)", P);
      return LCSB_EINVAL;
    }
    if (!c->virtual_shards && !has_comm) {
      snprintf(why, whylen, "process-sharded mode needs nccl_id or comm hooks");
      return LCSB_EINVAL;
    }
  } else if (sharded && sym == 2) {  // the sharded quarter table (§9c)
    if (!c->virtual_shards && (c->shard < 0 || c->shard >= P)) {
      snprintf(why, whylen, "shard must be in [0, %d)", P);
      return LCSB_EINVAL;
    }
    if (!c->virtual_shards && !has_comm) {
      snprintf(why, whylen, "process-sharded mode needs nccl_id or comm hooks");
      return LCSB_EINVAL;
    }
  } else if (sharded) {
    if (!sym) {
      snprintf(why, whylen,
               "sharding needs the complement-folded binary two-array table or sigma = 4, "
               "d = 2 (l >= 4; l >= 5 for 8 shards)");
      return LCSB_EINVAL;
    }
    if (pick_bin2_variant(c->dtype, c->ell, lp) == 0 ||
        bin2_tma_wpass_m(c->dtype, c->ell, lp) == 0) {
      snprintf(why, whylen, "ell = %d is too small for %d shards", c->ell, P);
      return LCSB_EINVAL;
    }
    if (!c->virtual_shards) {
      if (c->shard < 0 || c->shard >= P) {
        snprintf(why, whylen, "shard must be in [0, %d)", P);
        return LCSB_EINVAL;
      }
      if (!has_comm) {
        snprintf(why, whylen, "process-sharded mode needs nccl_id or comm hooks");
        return LCSB_EINVAL;
      }
    }
  }
  p->form = form;
  p->dtype_code = c->dtype;
  p->symmetric = sym;
  p->qK = (sym == 2) ? qK : 0;
  p->qM = (sym == 2) ? qM : 0;
  p->kernel = sym == 2 ? 5 : (sym ? 2 : 1);
  p->offsets = ofs;
  if (!sym && c->sigma == 4 && c->d == 2 && c->ell >= q4_min_ell() &&
      c->kernel == LCSB_KERNEL_AUTO)
    p->kernel = 3;  // sigma = 4, d = 2 swap-paired TMA kernel (kern_q4.cu; offsets too)
  else if (ofs) {
    // the quarter table (binary) or the generic full-table kernel: no small kernel
  } else if (p->kernel == 1 && c->kernel == LCSB_KERNEL_AUTO && small_supported(c->sigma, c->d, n))
    p->kernel = 4;  // register-resident compile-time (sigma, d) kernel (kern_small.cu)
  p->ntab = (form == LCSB_FORM_KS) ? c->d + 1 : 2;  // Alg. 2: d+1 rows; two-array: 2
  // q4: v_{n-2} is only read through its row means (kern_q4.cu): 2 full tables + 3 mean arrays
  if (p->kernel == 3) p->ntab = 2;
  p->P = P;
  p->p = lp;
  // process mode also with a single rank when an NCCL id is given (exercises the communicator,
  // the IPC exchange and the collective barrier/bound path on one GPU)
  p->mode = c->virtual_shards ? (P == 1 ? MODE_SINGLE : MODE_VIRTUAL)
                              : ((P > 1 || has_comm) ? MODE_PROCESS : MODE_SINGLE);
  p->n_logical = n;
  // q4: complement-folded table (heads h_a < 2 stored, kern_q4.cu)
  p->n_stored = (sym == 2) ? quarter_slots(c->ell, qK) << (2 * qK)
                           : ((sym || p->kernel == 3) ? n / 2 : n);
  p->n_local = p->n_stored / (uint64_t)P;
  if (sym == 2 && P > 1) {  // shard-major slots with the stride of the largest shard (§9c)
    const uint64_t mx = quarter_shard_maxslots(c->ell, qK, lp);
    if (!mx) {
      snprintf(why, whylen, "no shard map for ell = %d, block_log4 = %d, %d shards", c->ell, qK, P);
      return LCSB_EINVAL;
    }
    p->n_local = mx << (2 * qK);
  }
  p->esize = (c->dtype == LCSB_F32) ? 4 : 8;
  const uint64_t owned = (p->mode == MODE_PROCESS) ? 1 : (uint64_t)P;
  uint64_t tb, all;
  if (!mul_ok(p->n_local, p->esize, &tb) || !mul_ok(tb, (uint64_t)p->ntab, &all) ||
      !mul_ok(all, owned, &p->bytes)) {
    snprintf(why, whylen, "table size overflows");
    return LCSB_EINVAL;
  }
  p->bytes += 256;
  if (p->kernel == 3) p->bytes += 3 * (n / 32 / (uint64_t)P) * owned * sizeof(double);
  if (p->kernel == 4 && form == LCSB_FORM_KS && small_pooled_supported(c->sigma, c->d)) {
    uint64_t sigd = 1;
    for (int j = 0; j < c->d; ++j) sigd *= (uint64_t)c->sigma;
    for (int k = 2; k <= c->d; ++k)
      p->bytes += (uint64_t)p->ntab * (n / sigd) * small_pool_per_row(c->sigma, c->d, k) *
                  sizeof(double);
  }
  if (sym == 2) p->bytes += quarter_map_entries(c->ell, qK) * sizeof(uint32_t);
  if (ofs) p->bytes += 512;  // OffState
  return LCSB_OK;
}

extern "C" uint64_t lcsb_required_bytes(const lcsb_config* c) {
  Plan p;
  char why[256];
  if (plan_config(c, &p, why, sizeof why) != LCSB_OK) return 0;
  return p.bytes;
}

extern "C" int lcsb_shard_locate(int32_t ell, int32_t shards, uint64_t logical, int32_t* shard,
                                 uint64_t* local) {
  const int p = log2_exact(shards);
  if (ell < 2 || ell > 31 || p < 0 || shards > kMaxShards || !shard || !local)
    return set_err(nullptr, LCSB_EINVAL, "bad arguments to lcsb_shard_locate");
  const int L = 2 * ell;
  if (logical >= (1ull << L)) return set_err(nullptr, LCSB_EINVAL, "logical index out of range");
  uint64_t s = logical;
  if (s >= (1ull << (L - 1))) s = ((1ull << L) - 1) - s;  // Eq. (comp_eq)
  *shard = (int32_t)shard_of_stored(s, L, p);
  *local = local_of_stored(s, L, p);
  return LCSB_OK;
}

extern "C" int lcsb_shard_locate_sigma4(int32_t ell, int32_t shards, uint64_t logical,
                                        int32_t* shard, uint64_t* local) {
  const int p = log2_exact(shards);
  if (ell < 1 || ell > 15 || p < 0 || shards > kMaxShards || !shard || !local ||
      (p > 0 && ell < (p == 3 ? 5 : 4)))
    return set_err(nullptr, LCSB_EINVAL, "bad arguments to lcsb_shard_locate_sigma4");
  const int L = 4 * ell;
  if (logical >> L) return set_err(nullptr, LCSB_EINVAL, "logical index out of range");
  uint64_t s = logical;
  if (s >= (1ull << (L - 1))) s = ((1ull << L) - 1) - s;  // complement d -> 3 - d (kern_q4.cu)
  *shard = (int32_t)q4_key(s, ell, p);
  *local = q4_local(s, ell, p);
  return LCSB_OK;
}

extern "C" int lcsb_quarter_locate(int32_t ell, int32_t block_log4, uint64_t logical,
                                   uint64_t* stored, uint64_t* n_stored) {
  const int K = block_log4;
  if (ell < 3 || ell > 31 || K < 2 || K > ell - 1 || ell - K > 12 || !stored || !n_stored)
    return set_err(nullptr, LCSB_EINVAL, "bad arguments to lcsb_quarter_locate");
  const int L = 2 * ell;
  if (logical >= (1ull << L)) return set_err(nullptr, LCSB_EINVAL, "logical index out of range");
  static thread_local int cached_ell = 0, cached_K = 0;
  static thread_local uint32_t* cached = nullptr;
  if (cached_ell != ell || cached_K != K) {
    free(cached);
    cached = (uint32_t*)malloc(quarter_map_entries(ell, K) * sizeof(uint32_t));
    if (!cached || !build_quarter_map(ell, K, cached)) {
      cached_ell = 0;
      return set_err(nullptr, LCSB_EINVAL, "quarter map construction failed");
    }
    cached_ell = ell;
    cached_K = K;
  }
  uint64_t s = logical;
  if (s >= (1ull << (L - 1))) s = ((1ull << L) - 1) - s;  // Eq. (comp_eq)
  *stored = qstored(cached, s, K);
  *n_stored = quarter_slots(ell, K) << (2 * K);
  return LCSB_OK;
}

extern "C" int lcsb_quarter_shard_plan(int32_t ell, int32_t dtype, int32_t shards,
                                       int32_t passes, uint64_t* items, uint64_t* peer_read,
                                       uint64_t* peer_written) {
  if (!items || !peer_read || !peer_written || passes < 0)
    return set_err(nullptr, LCSB_EINVAL, "bad arguments to lcsb_quarter_shard_plan");
  lcsb_config c;
  lcsb_config_init(&c);
  c.sigma = 2, c.d = 2, c.ell = ell, c.dtype = dtype, c.symmetry = 2, c.shards = shards;
  c.virtual_shards = 1;
  Plan p;
  char why[256];
  if (plan_config(&c, &p, why, sizeof why) != LCSB_OK || p.symmetric != 2 || p.P < 2)
    return set_err(nullptr, LCSB_EINVAL, "no sharded quarter table for this configuration");
  std::vector<uint32_t> map(quarter_map_entries(ell, p.qK));
  uint64_t maxslots = 0;
  if (!build_quarter_map_sharded(ell, p.qK, p.qM, p.p, passes, map.data(), &maxslots))
    return set_err(nullptr, LCSB_EINVAL, "sharded quarter map construction failed");
  const std::vector<uint32_t> none;
  std::vector<uint32_t> mine;
  for (int k = 0; k < p.P; ++k) {
    quarter_shard_items(ell, p.qK, p.qM, map.data(), maxslots, k, none, mine);
    uint64_t tr[3];
    quarter_shard_traffic(ell, p.qK, p.qM, map.data(), maxslots, k, mine, tr);
    items[k] = mine.size();
    peer_read[k] = tr[0];
    peer_written[k] = tr[1];
  }
  return LCSB_OK;
}

extern "C" int lcsb_nccl_unique_id(void* out, size_t len) {
  if (!out || len < sizeof(ncclUniqueId))
    return set_err(nullptr, LCSB_EINVAL, "need a %zu-byte buffer", sizeof(ncclUniqueId));
  ncclUniqueId id;
  NC(nullptr, ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return LCSB_OK;
}

// ---------------------------------------------------------------- memory
static void* dev_alloc(lcsb_t* h, size_t bytes) {
  void* p = nullptr;
  if (h->mode == MODE_PROCESS) {  // IPC-exportable allocations
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return p;
  }
  if (h->cfg.alloc) return h->cfg.alloc(bytes, h->cfg.stream, h->cfg.alloc_ctx);
  if (cudaMallocAsync(&p, bytes, (cudaStream_t)h->cfg.stream) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

static void dev_free(lcsb_t* h, void* p, size_t bytes) {
  if (!p) return;
  if (h->mode == MODE_PROCESS)
    cudaFree(p);
  else if (h->cfg.free_)
    h->cfg.free_(p, bytes, h->cfg.stream, h->cfg.alloc_ctx);
  else
    cudaFreeAsync(p, (cudaStream_t)h->cfg.stream);
}

static bool owns(const lcsb_t* h, int k) { return k >= h->first && k < h->first + h->nown; }

// the device buffers of shard k a peer needs: the table ring, then (q4) the row-mean ring
static int ipc_nbuf(const lcsb_t* h) { return h->ntab + (h->kernel == 3 ? 3 : 0); }
static void** ipc_buf(lcsb_t* h, int k, int i) {
  return i < h->ntab ? &h->tabs[k][i] : reinterpret_cast<void**>(&h->pools[k][i - h->ntab]);
}


static const lcsb_comm_hooks* hooks(const lcsb_t* h) {
  return h->mode == MODE_PROCESS ? h->cfg.comm : nullptr;
}

static int barrier(lcsb_t* h) {  // process mode: every rank's preceding work is complete
  if (h->mode != MODE_PROCESS) return LCSB_OK;
  NvtxRange r("lcsb barrier");
  if (const lcsb_comm_hooks* c = hooks(h)) {  // host hooks: drain the stream, then meet
    CU(h, cudaStreamSynchronize((cudaStream_t)h->cfg.stream));
    if (c->barrier(c->ctx) != 0) return set_err(h, LCSB_ENCCL, "comm hook barrier failed");
    return LCSB_OK;
  }
  NC(h, ncclAllReduce(h->barrier_buf, h->barrier_buf, 1, ncclInt32, ncclSum, h->comm,
                      (cudaStream_t)h->cfg.stream));
  return LCSB_OK;
}

// process mode: element-wise max over the ranks of device reduction slots [first, first + n)
// (slot 1 = R_min is a minimum: the NCCL path reduces it with ncclMin, the hook path by a max of
// the complemented encoding)
// process mode: element-wise max (bit i of min_mask: min) over the ranks of n ordered-encoded
// device values at d, in place, stream-ordered
static int allreduce_dev(lcsb_t* h, unsigned long long* d, int n, unsigned min_mask) {
  if (h->mode != MODE_PROCESS) return LCSB_OK;
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  if (const lcsb_comm_hooks* c = hooks(h)) {
    unsigned long long v[kRedSlots];
    if (n > kRedSlots) return set_err(h, LCSB_EINVAL, "allreduce of %d values", n);
    CU(h, cudaMemcpyAsync(v, d, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CU(h, cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i)
      if ((min_mask >> i) & 1u) v[i] = ~v[i];
    if (c->allreduce_max_u64(reinterpret_cast<uint64_t*>(v), n, c->ctx) != 0)
      return set_err(h, LCSB_ENCCL, "comm hook allreduce_max_u64 failed");
    for (int i = 0; i < n; ++i)
      if ((min_mask >> i) & 1u) v[i] = ~v[i];
    CU(h, cudaMemcpyAsync(d, v, n * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
    CU(h, cudaStreamSynchronize(s));
    return LCSB_OK;
  }
  for (int i = 0; i < n; ++i)
    NC(h, ncclAllReduce(d + i, d + i, 1, ncclUint64, ((min_mask >> i) & 1u) ? ncclMin : ncclMax,
                        h->comm, s));
  return LCSB_OK;
}

static int allreduce_slots(lcsb_t* h, int first, int n, unsigned min_mask) {
  return allreduce_dev(h, h->red + first, n, min_mask >> first);
}

// integer offsets, sharded process mode: every rank's sweep reduced the min of the outputs it
// computed into its own mn[cur]; the global min before the prep kernel derives c from it
static int offsets_global_min(lcsb_t* h) {
  if (!h->ost || h->mode != MODE_PROCESS) return LCSB_OK;
  return allreduce_dev(h, &h->ost->mn[h->cur], 1, 1u);
}

extern "C" void lcsb_destroy(lcsb_t* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  cudaStreamSynchronize(s);
  if (h->mode == MODE_PROCESS && (h->comm || hooks(h))) {
    barrier(h);  // no peer may still be writing into our tables
    cudaStreamSynchronize(s);
    for (int k = 0; k < h->P && !h->vmm; ++k)
      if (!owns(h, k))
        for (int i = 0; i < ipc_nbuf(h); ++i)
          if (*ipc_buf(h, k, i)) cudaIpcCloseMemHandle(*ipc_buf(h, k, i));
  }
  if (h->vmm) {
    for (int i = 0; i < h->ntab; ++i) vmm_release(&h->vt[i]);
  } else {
    for (int k = 0; k < h->P; ++k)
      if (owns(h, k))
        for (int i = 0; i < h->ntab; ++i) dev_free(h, h->tabs[k][i], h->tab_bytes);
  }
  for (int k = 0; k < kMaxShards; ++k) dev_free(h, h->qsched_sh[k], h->qsched_bytes_sh[k]);
  dev_free(h, h->red, 256);
  dev_free(h, h->ost, 512);
  dev_free(h, h->base, h->tab_bytes);
  dev_free(h, h->qmap, h->qmap_bytes);
  if (h->qthread) {  // a schedule still being built is not needed any more
    h->qthread->join();
    delete h->qthread;
  }
  delete h->qready;
  delete h->qpending;
  dev_free(h, h->qsched, h->qsched_bytes);
  dev_free(h, h->qcounter, 256);
  for (int k = 0; k < h->P; ++k)
    if (owns(h, k))
      for (int i = 0; i < 3; ++i) dev_free(h, h->pools[k][i], h->pool_bytes);
  for (int k = 0; k <= kMaxD; ++k)
    for (int i = 0; i < kMaxGen; ++i) dev_free(h, h->spools[k][i], h->spool_bytes[k]);
  if (h->barrier_buf) cudaFree(h->barrier_buf);
  for (int i = 0; i < kMaxGen; ++i)
    if (h->graph[i]) cudaGraphExecDestroy(h->graph[i]);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->comm) ncclCommDestroy(h->comm);
  cudaStreamSynchronize(s);
  delete h;
}

static int exchange_ipc(lcsb_t* h) {
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  const int nbuf = ipc_nbuf(h);
  const size_t mine = hb * (size_t)nbuf;
  char host_mine[sizeof(cudaIpcMemHandle_t) * (kMaxGen + 3)];
  for (int i = 0; i < nbuf; ++i)
    CU(h, cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(host_mine + i * hb),
                              *ipc_buf(h, h->first, i)));
  char* dbuf = nullptr;
  char* host_all = (char*)malloc(mine * (size_t)h->P);
  int rc = LCSB_OK;
  cudaError_t e = cudaSuccess;
  if (const lcsb_comm_hooks* c = hooks(h)) {  // host hooks: the handles are plain bytes
    if (c->allgather(host_mine, host_all, mine, c->ctx) != 0)
      rc = set_err(h, LCSB_ENCCL, "comm hook allgather of the IPC handles failed");
  } else {
    CU(h, cudaMalloc(&dbuf, mine * (size_t)(h->P + 1)));
    e = cudaMemcpyAsync(dbuf + mine * h->P, host_mine, mine, cudaMemcpyHostToDevice, s);
    ncclResult_t r = ncclSuccess;
    if (e == cudaSuccess)
      r = ncclAllGather(dbuf + mine * h->P, dbuf, mine, ncclUint8, h->comm, s);
    if (e == cudaSuccess && r == ncclSuccess)
      e = cudaMemcpyAsync(host_all, dbuf, mine * h->P, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (r != ncclSuccess)
      rc = set_err(h, LCSB_ENCCL, "IPC handle all-gather: %s", ncclGetErrorString(r));
    else if (e != cudaSuccess)
      rc = set_err(h, LCSB_ECUDA, "IPC handle exchange: %s", cudaGetErrorString(e));
  }
  for (int k = 0; rc == LCSB_OK && k < h->P; ++k) {
    if (owns(h, k)) continue;
    for (int i = 0; i < nbuf && rc == LCSB_OK; ++i) {
      cudaIpcMemHandle_t mh;
      memcpy(&mh, host_all + (size_t)k * mine + i * hb, hb);
      e = cudaIpcOpenMemHandle(ipc_buf(h, k, i), mh, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess)
        rc = set_err(h, LCSB_ECUDA, "cudaIpcOpenMemHandle(shard %d): %s", k, cudaGetErrorString(e));
    }
  }
  free(host_all);
  if (dbuf) cudaFree(dbuf);
  return rc;
}

static int install_schedule(lcsb_t* h, bool wait);

// passes of the shard-assignment refinement of the sharded quarter table (§9c); LCSB_QSHARD_PASSES
// (A/B): 0 = the xor key alone
static int shard_refine_passes() {
  static const int n = getenv("LCSB_QSHARD_PASSES") ? atoi(getenv("LCSB_QSHARD_PASSES")) : 24;
  return n;
}

// LCSB_DEBUG: a SIGSEGV handler that prints the native backtrace (diagnosis only)
#include <execinfo.h>
#include <signal.h>
static void segv_backtrace(int sig) {
  void* fr[64];
  const int n = backtrace(fr, 64);
  fprintf(stderr, "[lcsb] signal %d, native backtrace:\n", sig);
  backtrace_symbols_fd(fr, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
static void debug_hooks() {
  static bool done = false;
  if (!done && getenv("LCSB_DEBUG")) {
    signal(SIGSEGV, segv_backtrace);
    done = true;
  }
}

// process mode: every rank's bytes (n each, host memory) in rank order, through the comm hooks or
// the library's NCCL communicator
static int allgather_host(lcsb_t* h, const void* mine, void* all, size_t n) {
  if (const lcsb_comm_hooks* c = hooks(h)) {
    if (c->allgather(mine, all, n, c->ctx) != 0)
      return set_err(h, LCSB_ENCCL, "comm hook allgather failed");
    return LCSB_OK;
  }
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  char* d = nullptr;
  CU(h, cudaMalloc(&d, n * (size_t)(h->P + 1)));
  cudaError_t e = cudaMemcpyAsync(d + n * h->P, mine, n, cudaMemcpyHostToDevice, s);
  ncclResult_t r = ncclSuccess;
  if (e == cudaSuccess) r = ncclAllGather(d + n * h->P, d, n, ncclUint8, h->comm, s);
  if (e == cudaSuccess && r == ncclSuccess)
    e = cudaMemcpyAsync(all, d, n * h->P, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d);
  if (r != ncclSuccess) return set_err(h, LCSB_ENCCL, "allgather: %s", ncclGetErrorString(r));
  if (e != cudaSuccess) return set_err(h, LCSB_ECUDA, "allgather: %s", cudaGetErrorString(e));
  return LCSB_OK;
}

// process mode, sharded quarter table (§9c): map every peer's shard allocations into this
// process's table ranges -- POSIX fds of the allocations over Unix sockets (vmm.cu)
static int exchange_vmm(lcsb_t* h) {
  static const bool dbg = getenv("LCSB_DEBUG") != nullptr;
#define VDBG(...) do { if (dbg) { fprintf(stderr, "[lcsb r%d] ", h->cfg.shard); fprintf(stderr, __VA_ARGS__); fprintf(stderr, "\n"); } } while (0)
  uint64_t tok[kMaxShards];
  uint64_t mine = ((uint64_t)getpid() << 20) ^ (uint64_t)(uintptr_t)h ^ (uint64_t)h->cfg.shard;
  int rc = allgather_host(h, &mine, tok, sizeof mine);
  if (rc != LCSB_OK) return rc;
  const uint64_t token = tok[0];  // rank 0's: one name space per handle
  char why[256];
  VDBG("token %llx", (unsigned long long)token);
  const int ls = fdx_listen(token, h->cfg.shard, why, sizeof why);
  VDBG("listening %d", ls);
  if (ls < 0) return set_err(h, LCSB_ECUDA, "sharded quarter table: %s", why);
  int fds[kMaxGen];
  int nf = 0;
  rc = barrier(h);  // every rank listens (the NCCL barrier completes on the stream: wait for it)
  if (rc == LCSB_OK && cudaStreamSynchronize((cudaStream_t)h->cfg.stream) != cudaSuccess)
    rc = set_err(h, LCSB_ECUDA, "sharded quarter table: stream synchronisation failed");
  for (int i = 0; rc == LCSB_OK && i < h->ntab; ++i, ++nf)
    if (!vmm_export_fd(&h->vt[i], h->cfg.shard, &fds[i], why, sizeof why))
      rc = set_err(h, LCSB_ECUDA, "sharded quarter table: %s", why);
  VDBG("exported %d fds rc %d", nf, rc);
  for (int k = 0; rc == LCSB_OK && k < h->P; ++k)
    if (k != h->cfg.shard && !fdx_send(token, h->cfg.shard, k, fds, h->ntab, why, sizeof why))
      rc = set_err(h, LCSB_ECUDA, "sharded quarter table: %s", why);
  VDBG("sent rc %d", rc);
  for (int i = 0; i < nf; ++i) close(fds[i]);
  for (int got = 0; rc == LCSB_OK && got < h->P - 1; ++got) {
    int from = -1, in[kMaxGen];
    if (!fdx_recv(ls, &from, in, h->ntab, why, sizeof why)) {
      rc = set_err(h, LCSB_ECUDA, "sharded quarter table: %s", why);
      break;
    }
    for (int i = 0; i < h->ntab; ++i) {
      if (rc == LCSB_OK && (from < 0 || from >= h->P || from == h->cfg.shard ||
                            !vmm_import_fd(&h->vt[i], from, in[i], why, sizeof why)))
        rc = set_err(h, LCSB_ECUDA, "sharded quarter table (shard %d): %s", from, why);
      close(in[i]);
    }
    VDBG("imported from %d rc %d", from, rc);
  }
  close(ls);
#undef VDBG
  return rc;
}

extern "C" int lcsb_create_ex(const lcsb_config* cfg, lcsb_t** out) {
  if (!out) return set_err(nullptr, LCSB_EINVAL, "out is NULL");
  debug_hooks();
  *out = nullptr;
  Plan p;
  char why[256];
  int rc = plan_config(cfg, &p, why, sizeof why);
  if (rc != LCSB_OK) return set_err(nullptr, rc, "%s", why);

  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess)
    return set_err(nullptr, LCSB_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
  size_t free_b = 0, total_b = 0;
  e = cudaMemGetInfo(&free_b, &total_b);
  if (e != cudaSuccess)
    return set_err(nullptr, LCSB_ECUDA, "cudaMemGetInfo failed: %s", cudaGetErrorString(e));
  if (!cfg->alloc && p.bytes > free_b)
    return set_err(nullptr, LCSB_ECAPACITY,
                   "needs %llu bytes of device memory for %d tables of %llu entries, %llu free",
                   (unsigned long long)p.bytes, p.ntab, (unsigned long long)p.n_local,
                   (unsigned long long)free_b);

  lcsb_t* h = new (std::nothrow) lcsb();
  if (!h) return set_err(nullptr, LCSB_ECAPACITY, "host allocation failed");
  memset(h, 0, sizeof *h);
  h->cfg = *cfg;
  h->device = dev;
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev);
  if (const char* e = getenv("LCSB_SMS")) {  // A/B only: persistent grids on fewer SMs
    const int k = atoi(e);
    if (k > 0 && k < h->sms) h->sms = k;
  }
  h->form = p.form;
  h->symmetric = p.symmetric;
  h->kernel = p.kernel;
  h->qK = p.qK;
  h->qM = p.qM;
  h->n_logical = p.n_logical;
  h->n_stored = p.n_stored;
  h->n_local = p.n_local;
  h->esize = p.esize;
  h->ntab = p.ntab;
  h->p = p.p;
  h->P = p.P;
  h->mode = p.mode;
  h->first = (p.mode == MODE_PROCESS) ? cfg->shard : 0;
  h->nown = (p.mode == MODE_PROCESS) ? 1 : p.P;
  h->tab_bytes = (size_t)(p.n_local * p.esize);
  h->bin2_variant = 0;  // auto (pick_bin2_variant)
  if (const char* v = getenv("LCSB_BIN2_VARIANT")) h->bin2_variant = atoi(v);
  if (const char* v = getenv("LCSB_BIN2Q_VARIANT")) h->bin2q_variant = atoi(v);
  if (h->bin2q_variant > 0 && h->symmetric == 2) {
    const int vm = bin2q_variant_m(p.dtype_code, h->bin2q_variant);
    if (vm <= 0 || vm > h->qK - 1 || vm > cfg->ell - 2) {
      lcsb_destroy(h);
      return set_err(nullptr, LCSB_EINVAL, "LCSB_BIN2Q_VARIANT %d does not fit block_log4 %d",
                     h->bin2q_variant, p.qK);
    }
  }
  cudaStream_t s = (cudaStream_t)cfg->stream;

  if (h->mode == MODE_PROCESS && !cfg->comm) {
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&h->comm, h->P, id, cfg->shard);
    if (r != ncclSuccess) {
      h->comm = nullptr;
      lcsb_destroy(h);
      return set_err(nullptr, LCSB_ENCCL, "ncclCommInitRank failed: %s", ncclGetErrorString(r));
    }
    if (cudaMalloc(&h->barrier_buf, 256) != cudaSuccess) {
      lcsb_destroy(h);
      return set_err(nullptr, LCSB_ECAPACITY, "barrier buffer allocation failed");
    }
    cudaMemsetAsync(h->barrier_buf, 0, 256, s);
  }
  static const bool cdbg = getenv("LCSB_DEBUG") != nullptr;
  if (cdbg) fprintf(stderr, "[lcsb] create: tables (mode %d, P %d, sym %d)\n", h->mode, h->P, h->symmetric);
  h->vmm = h->symmetric == 2 && h->P > 1;
  if (h->vmm) {  // sharded quarter table: one VA range per ring slot, shard k at k * stride
    const size_t g = vmm_granularity(dev);
    h->tab_bytes = (h->tab_bytes + g - 1) / g * g;
    char why2[256];
    for (int i = 0; i < h->ntab; ++i) {
      bool ok = vmm_reserve(&h->vt[i], h->P, h->tab_bytes, dev, why2, sizeof why2);
      for (int k = h->first; ok && k < h->first + h->nown; ++k)
        ok = vmm_create_shard(&h->vt[i], k, h->mode == MODE_PROCESS, why2, sizeof why2);
      if (!ok) {
        lcsb_destroy(h);
        return set_err(nullptr, LCSB_ECAPACITY, "sharded quarter table: %s", why2);
      }
      for (int k = 0; k < h->P; ++k)
        h->tabs[k][i] = (char*)h->vt[i].base + (size_t)k * h->tab_bytes;
    }
    if (cdbg) fprintf(stderr, "[lcsb] create: vmm tables mapped\n");
  }
  for (int k = h->first; !h->vmm && k < h->first + h->nown; ++k) {
    for (int i = 0; i < h->ntab; ++i) {
      h->tabs[k][i] = dev_alloc(h, h->tab_bytes);
      if (!h->tabs[k][i]) {
        int code = set_err(nullptr, LCSB_ECAPACITY,
                           "device allocation of table %d (%llu bytes) failed; %llu bytes needed",
                           i, (unsigned long long)h->tab_bytes, (unsigned long long)p.bytes);
        lcsb_destroy(h);
        return code;
      }
    }
  }
  h->red = (unsigned long long*)dev_alloc(h, 256);
  if (!h->red) {
    lcsb_destroy(h);
    return set_err(nullptr, LCSB_ECAPACITY, "scratch allocation failed");
  }
  static_assert(sizeof(OffState) <= 512, "plan_config reserves 512 bytes for the offset state");
  if (p.offsets) {  // W_0 = 0 with offset 0; min of the zero table = 0
    h->ost = (OffState*)dev_alloc(h, 512);
    if (!h->ost || launch_offset_init(h->ost, s) != cudaSuccess) {
      lcsb_destroy(h);
      return set_err(nullptr, LCSB_ECAPACITY, "offset state allocation failed");
    }
  }
  if (h->kernel == 3) {  // row-mean ring of the pooled-history KS sweep, zero (W_0 = 0)
    // rows of stored states, split evenly over the shards
    h->pool_bytes = (size_t)(h->n_logical / 32 / (uint64_t)h->P) * sizeof(double);
    for (int k = h->first; k < h->first + h->nown; ++k)
      for (int i = 0; i < 3; ++i) {
        h->pools[k][i] = (double*)dev_alloc(h, h->pool_bytes);
        if (!h->pools[k][i] ||
            cudaMemsetAsync(h->pools[k][i], 0, h->pool_bytes, s) != cudaSuccess) {
          lcsb_destroy(h);
          return set_err(nullptr, LCSB_ECAPACITY, "row-mean array allocation failed");
        }
      }
  }
  if (h->kernel == 4 && h->form == LCSB_FORM_KS && small_pooled_supported(cfg->sigma, cfg->d) &&
      !getenv("LCSB_NO_SMALL_POOL")) {  // pooled means of every ring slot, zero (W_0 = 0)
    h->spooled = 1;
    uint64_t sigd = 1;
    for (int j = 0; j < cfg->d; ++j) sigd *= (uint64_t)cfg->sigma;
    for (int k = 2; k <= cfg->d; ++k) {
      h->spool_bytes[k] = (size_t)(h->n_logical / sigd) *
                          small_pool_per_row(cfg->sigma, cfg->d, k) * sizeof(double);
      for (int i = 0; i < h->ntab; ++i) {
        h->spools[k][i] = (double*)dev_alloc(h, h->spool_bytes[k]);
        if (!h->spools[k][i] ||
            cudaMemsetAsync(h->spools[k][i], 0, h->spool_bytes[k], s) != cudaSuccess) {
          lcsb_destroy(h);
          return set_err(nullptr, LCSB_ECAPACITY, "pooled-mean array allocation failed");
        }
      }
    }
  }
  if (cdbg) fprintf(stderr, "[lcsb] create: map\n");
  if (h->symmetric == 2) {  // quarter table block map (host-built, uploaded once)
    const uint64_t nb = quarter_map_entries(cfg->ell, h->qK);
    h->qmap_bytes = nb * sizeof(uint32_t);
    uint32_t* hm = (uint32_t*)malloc(h->qmap_bytes);
    h->qmap = (uint32_t*)dev_alloc(h, h->qmap_bytes);
    const bool ok = hm && h->qmap &&
                    (h->vmm ? build_quarter_map_sharded(cfg->ell, h->qK, h->qM, h->p,
                                                        shard_refine_passes(), hm, &h->qmaxslots)
                            : build_quarter_map(cfg->ell, h->qK, hm));
    e = ok ? cudaMemcpyAsync(h->qmap, hm, h->qmap_bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
    if (e == cudaSuccess && ok) e = cudaStreamSynchronize(s);
    if (ok && e == cudaSuccess && h->vmm) {
      // sharded (§9c): the items of each owned shard -- the L2 order filtered by owner (built
      // here, synchronously: every rank derives the same lists), dynamic claiming per launch
      std::vector<uint32_t> sched, mine;
      if (cdbg) fprintf(stderr, "[lcsb] create: schedule (maxslots %llu)\n", (unsigned long long)h->qmaxslots);
      if (!getenv("LCSB_NO_QSCHED") && cfg->ell - h->qM - 1 >= 4) {
        // the L2 order depends only on which items share stored blocks: built (and cached) on
        // the unsharded slot numbering, whose slot count sizes its arrays
        std::vector<uint32_t> plain(nb);
        if (!build_quarter_map(cfg->ell, h->qK, plain.data()) ||
            !quarter_schedule(cfg->ell, h->qK, h->qM, plain.data(), sched))
          sched.clear();
      }
      if (cdbg) fprintf(stderr, "[lcsb] create: schedule %zu\n", sched.size());
      for (int k = h->first; k < h->first + h->nown && e == cudaSuccess; ++k) {
        quarter_shard_items(cfg->ell, h->qK, h->qM, hm, h->qmaxslots, k, sched, mine);
        if (cdbg) fprintf(stderr, "[lcsb] create: shard %d items %zu\n", k, mine.size());
        uint64_t tr[3];
        quarter_shard_traffic(cfg->ell, h->qK, h->qM, hm, h->qmaxslots, k, mine, tr);
        h->peer_read += tr[0];
        h->peer_written += tr[1];
        h->all_moved += tr[2];
        h->qsched_n_sh[k] = mine.size();
        h->qsched_bytes_sh[k] = (mine.size() ? mine.size() : 1) * sizeof(uint32_t);
        h->qsched_sh[k] = (uint32_t*)dev_alloc(h, h->qsched_bytes_sh[k]);
        if (!h->qsched_sh[k]) {
          e = cudaErrorMemoryAllocation;
          break;
        }
        if (!mine.empty())
          e = cudaMemcpyAsync(h->qsched_sh[k], mine.data(), mine.size() * sizeof(uint32_t),
                              cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      }
      if (e == cudaSuccess && h->qM >= 6 && !getenv("LCSB_QSTATIC")) {
        h->qcounter = (unsigned long long*)dev_alloc(h, 256);
        if (!h->qcounter) e = cudaErrorMemoryAllocation;
      }
    } else if (ok && e == cudaSuccess && !getenv("LCSB_NO_QSCHED") &&
               cfg->ell - h->qM - 1 >= 4) {
      // the L2 item order of the sweep (large tables), built on a host thread: it changes only
      // the order of the items, never a value (every output is written once from the previous
      // table), so the first sweeps may run without it
      h->qpending = new (std::nothrow) std::vector<uint32_t>();
      h->qready = new (std::nothrow) std::atomic<int>(0);
      if (h->qpending && h->qready &&
          quarter_schedule_cached(cfg->ell, h->qK, h->qM, *h->qpending)) {
        h->qready->store(1);  // built before in this process: installed right below
        h->qthread = new (std::nothrow) std::thread([] {});
      } else if (h->qpending && h->qready) {
        std::vector<uint32_t> mcopy(hm, hm + nb);
        const int ell = cfg->ell, K = h->qK, M = h->qM;
        std::vector<uint32_t>* pend = h->qpending;
        std::atomic<int>* rdy = h->qready;
        h->qthread = new (std::nothrow) std::thread([ell, K, M, pend, rdy, m = std::move(mcopy)]() {
          if (!quarter_schedule(ell, K, M, m.data(), *pend)) pend->clear();
          rdy->store(1, std::memory_order_release);
        });
      }
    }
    free(hm);
    if (!ok || e != cudaSuccess) {
      lcsb_destroy(h);
      return set_err(nullptr, ok ? LCSB_ECUDA : LCSB_ECAPACITY, "quarter map setup failed");
    }
  }
  // W_0 = 0: every generation the first sweep reads starts at zero.  The
  // slot the first sweep writes, (cur + 1) % ntab with cur = 0, is overwritten entirely (every
  // stored entry is written once per sweep) before anything reads it; generations older than
  // the start read out as W_0 = 0 (readout).
  for (int k = h->first; k < h->first + h->nown; ++k)
    for (int i = 0; i < h->ntab; ++i) {
      if (i == 1 % h->ntab && h->ntab > 1) continue;
      e = cudaMemsetAsync(h->tabs[k][i], 0, h->tab_bytes, s);
      if (e != cudaSuccess) {
        lcsb_destroy(h);
        return set_err(nullptr, LCSB_ECUDA, "cudaMemsetAsync failed: %s", cudaGetErrorString(e));
      }
    }
  if (cdbg) fprintf(stderr, "[lcsb] create: exchange\n");
  if (h->mode == MODE_PROCESS) {
    rc = h->vmm ? exchange_vmm(h) : exchange_ipc(h);
    if (rc == LCSB_OK) rc = barrier(h);
    if (rc != LCSB_OK) {
      char msg[512];
      snprintf(msg, sizeof msg, "%s", h->err);
      lcsb_destroy(h);
      return set_err(nullptr, rc, "%s", msg);
    }
  }
  h->cur = 0;
  const bool sync = getenv("LCSB_QSCHED_SYNC") ||
                    (h->qready && h->qready->load(std::memory_order_acquire));
  if (sync && install_schedule(h, true) != LCSB_OK) {  // ready (cached) or A/B: no overlap
    char msg[512];
    snprintf(msg, sizeof msg, "%s", h->err);
    lcsb_destroy(h);
    return set_err(nullptr, LCSB_ECAPACITY, "%s", msg);
  }
  *out = h;
  return LCSB_OK;
}

extern "C" int lcsb_create(int32_t sigma, int32_t d, int32_t ell, int32_t dtype, lcsb_t** out) {
  lcsb_config c;
  lcsb_config_init(&c);
  c.sigma = sigma;
  c.d = d;
  c.ell = ell;
  c.dtype = dtype;
  return lcsb_create_ex(&c, out);
}

extern "C" int lcsb_reset(lcsb_t* h) {
  if (!h) return set_err(nullptr, LCSB_EINVAL, "handle is NULL");
  NvtxRange r("lcsb_reset");
  CU(h, cudaSetDevice(h->device));
  int rc = barrier(h);  // nobody is still sweeping into our tables
  if (rc != LCSB_OK) return rc;
  // zero the generations the first sweep reads (cur = 0); its output slot 1 is overwritten
  // entirely by that sweep (see lcsb_create)
  for (int k = h->first; k < h->first + h->nown; ++k)
    for (int i = 0; i < h->ntab; ++i)
      if (!(i == 1 % h->ntab && h->ntab > 1))
        CU(h, cudaMemsetAsync(h->tabs[k][i], 0, h->tab_bytes, (cudaStream_t)h->cfg.stream));
  rc = barrier(h);  // everyone's tables are zero before anyone sweeps into them
  if (rc != LCSB_OK) return rc;
  for (int k = h->first; k < h->first + h->nown; ++k)
    for (int i = 0; i < 3; ++i)
      if (h->pools[k][i])
        CU(h, cudaMemsetAsync(h->pools[k][i], 0, h->pool_bytes, (cudaStream_t)h->cfg.stream));
  for (int k = 0; k <= kMaxD; ++k)
    for (int i = 0; i < kMaxGen; ++i)
      if (h->spools[k][i])
        CU(h, cudaMemsetAsync(h->spools[k][i], 0, h->spool_bytes[k], (cudaStream_t)h->cfg.stream));
  if (h->ost) CU(h, launch_offset_init(h->ost, (cudaStream_t)h->cfg.stream));
  if (h->base) {  // back to plain storage (W_0 = 0 needs no base)
    dev_free(h, h->base, h->tab_bytes);
    h->base = nullptr;
    for (int i = 0; i < kMaxGen; ++i)
      if (h->graph[i]) {
        cudaGraphExecDestroy(h->graph[i]);
        h->graph[i] = nullptr;
      }
  }
  h->cur = 0;
  h->pcur = 0;
  h->sweeps_done = 0;
  h->trk_at[0] = h->trk_at[1] = -1;
  h->best_rho[0] = h->best_rho[1] = 0.0;
  h->best_sweep[0] = h->best_sweep[1] = 0;
  return LCSB_OK;
}

static inline int slot_back(const lcsb_t* h, int k) {  // table k sweeps back from the newest
  return ((h->cur - k) % h->ntab + h->ntab) % h->ntab;
}

static void fill_generic(const lcsb_t* h, GenericArgs* a) {
  memset(a, 0, sizeof *a);
  a->sigma = h->cfg.sigma;
  a->d = h->cfg.d;
  a->ell = h->cfg.ell;
  a->n = h->n_logical;
  a->form = h->form;
  a->headw_top = 1;
  for (int i = 0; i < a->d * (a->ell - 1); ++i) a->headw_top *= (uint64_t)a->sigma;
}

static void fill_bin2(const lcsb_t* h, Bin2Args* a, int shard, int in_slot, int out_slot) {
  memset(a, 0, sizeof *a);
  a->src = h->tabs[shard][in_slot];
  a->dst = out_slot >= 0 ? h->tabs[shard][out_slot] : nullptr;
  a->ell = h->cfg.ell;
  a->m = bin2_tile_m(h->cfg.ell);
  a->shard_bits = h->p;
  a->shard = shard;
  for (int k = 0; k < h->P; ++k) {
    a->src_shards[k] = h->tabs[k][in_slot];
    a->dst_shards[k] = out_slot >= 0 ? h->tabs[k][out_slot] : nullptr;
  }
}

// Upload the quarter table's item schedule once its host thread has finished (wait: block until
// then).  Graphs captured before use the natural order: they are dropped and re-captured.
static int install_schedule(lcsb_t* h, bool wait) {
  if (!h->qthread) return LCSB_OK;
  if (!wait && !h->qready->load(std::memory_order_acquire)) return LCSB_OK;
  h->qthread->join();
  delete h->qthread;
  h->qthread = nullptr;
  std::vector<uint32_t>& sched = *h->qpending;
  if (!sched.empty()) {
    cudaStream_t s = (cudaStream_t)h->cfg.stream;
    const size_t bytes = sched.size() * sizeof(uint32_t);
    uint32_t* d = (uint32_t*)dev_alloc(h, bytes);
    if (!d) return set_err(h, LCSB_ECAPACITY, "schedule allocation failed");
    // pageable source: the call returns once the bytes are staged, so `sched` may be freed
    CU(h, cudaMemcpyAsync(d, sched.data(), bytes, cudaMemcpyHostToDevice, s));
    // dynamic claiming (one work counter): 20.7 vs 26.6 GB read at l = 17 fp32.  For the 4x
    // more, smaller items of fp64 (4^5 tiles) it paid only once the producer was pipelined
    // (kern_bin2q.cuh DEPTH 3; l = 17 fp64: 12.56 vs 13.05 ms static, before 3.99 vs 3.28 at
    // l = 16).  LCSB_QSTATIC (A/B): static round-robin claims
    if (!getenv("LCSB_QSTATIC")) {
      h->qcounter = (unsigned long long*)dev_alloc(h, 256);
      if (!h->qcounter) return set_err(h, LCSB_ECAPACITY, "counter allocation failed");
    }
    h->qsched = d;
    h->qsched_bytes = bytes;
    h->qsched_n = sched.size();
    for (int i = 0; i < kMaxGen; ++i)
      if (h->graph[i]) {
        cudaGraphExecDestroy(h->graph[i]);
        h->graph[i] = nullptr;
      }
  }
  sched.clear();
  sched.shrink_to_fit();
  return LCSB_OK;
}

extern "C" int32_t lcsb_ready(lcsb_t* h, int32_t wait) {
  if (!h) return set_err(nullptr, LCSB_EINVAL, "handle is NULL"), -1;
  if (install_schedule(h, wait != 0) != LCSB_OK) return -1;
  return h->qthread ? 0 : 1;
}

static void fill_bin2q(const lcsb_t* h, Bin2QArgs* a, int in_slot, int out_slot) {
  memset(a, 0, sizeof *a);
  a->src = h->tabs[0][in_slot];
  a->dst = out_slot >= 0 ? h->tabs[0][out_slot] : nullptr;
  a->map = h->qmap;
  a->ell = h->cfg.ell;
  a->K = h->qK;
  a->sched = h->qsched;
  a->nitems = h->qsched_n;
  a->sched_m = h->qM;
  static const int l2keep = getenv("LCSB_QKEEP") ? atoi(getenv("LCSB_QKEEP")) : 0;  // A/B
  a->l2keep = l2keep;
  a->counter = h->qcounter;
  a->base = h->base;
}

static int enqueue_sweeps(lcsb_t* h, int64_t n, cudaStream_t s, int64_t track = 0);

// Small tables are launch-latency bound: replay a captured graph of G sweeps (G a multiple of
// the ring length, so the ring slots are the same before and after) instead of G launches.
static bool graph_worthy(const lcsb_t* h) {
  return h->mode == MODE_SINGLE && (uint64_t)h->tab_bytes <= (64ull << 20);
}

static int sweep_graph(lcsb_t* h, cudaStream_t s) {
  const int start = h->cur + h->ntab * h->pcur;  // ring state (both rings line up after G)
  if (!h->graph[start]) {
    if (!h->cap_stream) CU(h, cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    const int64_t done = h->sweeps_done, launches = h->launches;
    CU(h, cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    h->cap_capturing = 1;
    int rc = enqueue_sweeps(h, h->graph_sweeps, h->cap_stream);
    h->cap_capturing = 0;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    if (rc != LCSB_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return set_err(h, LCSB_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&h->graph[start], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      h->graph[start] = nullptr;
      return set_err(h, LCSB_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    }
    h->sweeps_done = done;  // the capture only recorded the sweeps
    h->launches = launches;
    h->cur = start % h->ntab;
    h->pcur = start / h->ntab;
  }
  CU(h, cudaGraphLaunch(h->graph[start], s));
  h->sweeps_done += h->graph_sweeps;
  h->launches += h->graph_sweeps;
  return LCSB_OK;
}

// the tracking sweep applies (quarter table, plain storage)
static bool can_track(const lcsb_t* h) { return h->kernel == 5 && !h->ost && !h->base; }
constexpr int kTrkSlot = 8;  // red[8..15]: the two tracking sets (h->red holds 32 slots)
static unsigned long long* trk_slots(lcsb_t* h, int64_t k) { return h->red + kTrkSlot + 4 * (k & 1); }

static int sweep_impl(lcsb_t* h, int64_t n, int64_t track);

extern "C" int lcsb_sweep(lcsb_t* h, int64_t n) {
  if (!h) return set_err(nullptr, LCSB_EINVAL, "handle is NULL");
  NvtxRange r("lcsb_sweep");
  return sweep_impl(h, n, 0);
}

extern "C" int lcsb_sweep_ex(lcsb_t* h, int64_t n, uint32_t flags) {
  if (!h) return set_err(nullptr, LCSB_EINVAL, "handle is NULL");
  NvtxRange r("lcsb_sweep_ex");
  if (flags & ~(uint32_t)LCSB_SWEEP_TRACK2) return set_err(h, LCSB_EINVAL, "unknown flags %u", flags);
  const int64_t t = (flags & LCSB_SWEEP_TRACK2) == LCSB_SWEEP_TRACK2 ? 2 : (flags & 1u) ? 1 : 0;
  return sweep_impl(h, n, t);
}

// n sweeps; the last min(track, n) of them are tracking sweeps where the layout has them
static int sweep_impl(lcsb_t* h, int64_t n, int64_t track) {
  if (n < 0) return set_err(h, LCSB_EINVAL, "n must be >= 0");
  if (track > n) track = n;
  if (!can_track(h)) track = 0;
  const int64_t total = n;
  n -= track;  // the plain sweeps (graphs, ...) first, the tracked ones at the end
  CU(h, cudaSetDevice(h->device));
  {
    int rc = install_schedule(h, false);
    if (rc != LCSB_OK) return rc;
  }
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  if (total > 0 && h->mode == MODE_PROCESS) {
    // every rank is done with the tables (e.g. a rank-local lcsb_table read since the last
    // collective call) before anyone overwrites the oldest generation in the peers' memory
    int rc = barrier(h);
    if (rc != LCSB_OK) return rc;
  }
  if (graph_worthy(h) && !getenv("LCSB_NO_GRAPHS")) {
    if (!h->graph_sweeps) {
      const int period = (h->kernel == 3) ? 6 : h->ntab;  // q4: lcm(2 tables, 3 mean arrays)
      h->graph_sweeps = period;
      while (h->graph_sweeps < 32) h->graph_sweeps += period;
    }
    if (h->sweeps_done == 0 && n > 0) {  // one plain sweep first (initialises launch caches)
      int rc = enqueue_sweeps(h, 1, s);
      if (rc != LCSB_OK) return rc;
      --n;
    }
    while (n >= h->graph_sweeps) {
      int rc = sweep_graph(h, s);
      if (rc != LCSB_OK) return rc;
      n -= h->graph_sweeps;
    }
  }
  return enqueue_sweeps(h, n + track, s, track);
}

static int enqueue_sweeps(lcsb_t* h, int64_t n, cudaStream_t s, int64_t track) {
  for (int64_t it = 0; it < n; ++it) {
    const bool trk = it >= n - track;  // a tracking sweep (can_track checked by the caller)
    NvtxRange r("sweep");
    if (h->qthread && !h->cap_capturing) {  // the schedule finished during a long call
      int rc = install_schedule(h, false);
      if (rc != LCSB_OK) return rc;
    }
    const int out = (h->cur + 1) % h->ntab;  // the slot of the oldest table
    cudaError_t e = cudaSuccess;
    if (h->kernel == 2) {
      const int v = h->bin2_variant ? h->bin2_variant
                                    : pick_bin2_variant(h->cfg.dtype, h->cfg.ell, h->p);
      const int M = bin2_tma_m(h->cfg.dtype, v);
      const bool tma_ok = M > 0 && h->cfg.ell >= M + 1 && h->p < h->cfg.ell - 1 - M &&
                          (h->p == 0 || bin2_tma_direct(h->cfg.dtype, v));
      if (!tma_ok && h->p > 0)
        return set_err(h, LCSB_EINVAL, "variant %d cannot run sharded at ell = %d", v,
                       h->cfg.ell);
      for (int k = h->first; k < h->first + h->nown && e == cudaSuccess; ++k) {
        Bin2Args a;
        fill_bin2(h, &a, k, h->cur, out);
        if (tma_ok) {
          e = launch_bin2_tma_sweep(a, h->cfg.dtype, v, s, h->sms);
        } else {
          a.grid_mult = (v == 5) ? 8 : 0;
          e = launch_bin2_sweep(a, h->cfg.dtype, s, h->sms);
        }
        h->launches += 1;
      }
    } else if (h->kernel == 5) {
      Bin2QArgs a;
      fill_bin2q(h, &a, h->cur, out);
      if (h->ost) {  // integer offsets: c = floor(min s) of the table read, then the sweep
        int rc = offsets_global_min(h);
        if (rc != LCSB_OK) return rc;
        e = launch_offset_prep(h->ost, h->cur, out, s);
        h->launches += 1;
        a.ost = h->ost;
        a.omin = &h->ost->mn[out];
      }
      if (trk) {  // the tracking set of this sweep: R_max, R_min at -inf / +inf, D at +inf
        a.red_out = trk_slots(h, h->sweeps_done + 1);
        h->trk_at[(h->sweeps_done + 1) & 1] = -1;
        e = launch_red_init(a.red_out, s, 6u);
        h->launches += 1;
      }
      // sharded (§9c): one launch per owned shard over its item list; the table pointers span
      // every shard (reads of other shards' windows and stores of their outputs go to peers)
      for (int k = h->first; k < h->first + h->nown && e == cudaSuccess; ++k) {
        if (h->vmm) {
          a.sched = h->qsched_sh[k];
          a.nitems = h->qsched_n_sh[k];
        }
        if (a.counter) e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), s);
        if (e == cudaSuccess)
          e = trk ? launch_bin2q_diff(a, h->cfg.dtype, h->qM, s, h->sms)
                  : launch_bin2q_sweep(a, h->cfg.dtype, h->qM, h->bin2q_variant, s, h->sms);
        h->launches += 1;
        if (!h->vmm) break;
      }
    } else if (h->kernel == 3) {
      // row means of v_{n-2} (KS) / of v_{n-1}, the table this sweep reads (two-array)
      const int pin = (h->form == LCSB_FORM_KS) ? (h->pcur + 2) % 3 : h->pcur;
      const int pout = (h->pcur + 1) % 3;  // row means of the table written now
      if (h->ost) {  // integer offsets (R23; KS: the row means read are of the table two back)
        int rc = offsets_global_min(h);
        if (rc != LCSB_OK) return rc;
        GenSlots gs{};
        if (h->form == LCSB_FORM_KS) {
          gs.n = 2;
          gs.slot[0] = slot_back(h, 0);
          gs.slot[1] = slot_back(h, 1);  // = out (ring of 2): read before prep overwrites it
        }
        e = launch_offset_prep(h->ost, h->cur, out, s, &gs);
        h->launches += 1;
      }
      for (int k = h->first; k < h->first + h->nown && e == cudaSuccess; ++k) {
        Q4Args a;
        memset(&a, 0, sizeof a);
        a.g1 = h->tabs[k][slot_back(h, 0)];
        a.pin = h->pools[k][pin];
        a.flags = (h->form == LCSB_FORM_TWO_ARRAY) ? kQ4TwoArray : 0;
        a.pout = h->pools[k][pout];
        a.dst = h->tabs[k][out];
        a.ell = h->cfg.ell;
        a.p = h->p;
        a.shard = k;
        for (int j = 0; j < h->P; ++j) {  // sharded: outputs and row means go to their owners
          a.dst_sh[j] = h->tabs[j][out];
          a.pout_sh[j] = h->pools[j][pout];
        }
        if (h->ost) {  // every shard's launch reduces into the same min (virtual shards)
          a.ost = h->ost;
          a.omin = &h->ost->mn[out];
        }
        e = launch_q4_sweep(a, h->cfg.dtype, s, h->sms);
        h->launches += 1;
      }
      h->pcur = (h->pcur + 1) % 3;
    } else {
      GenericArgs a;
      fill_generic(h, &a);
      for (int k = 1; k <= h->cfg.d; ++k)
        a.src[k - 1] = (h->form == LCSB_FORM_KS) ? h->tabs[0][slot_back(h, k - 1)]
                                                 : h->tabs[0][h->cur];
      a.dst = h->tabs[0][out];
      if (h->spooled) {  // the table k back is read through its pooled means (k >= 2)
        for (int k = 2; k <= h->cfg.d; ++k) {
          a.pin[k - 1] = h->spools[k][slot_back(h, k - 1)];
          a.pout[k - 1] = h->spools[k][out];
        }
        e = launch_small_pooled(a, h->cfg.dtype, s, h->sms);
      } else {
        if (h->ost) {  // integer offsets (generic kernel; KS: per-generation shifts, R26)
          GenSlots gs{};
          if (h->form == LCSB_FORM_KS) {
            gs.n = h->cfg.d;
            for (int k = 1; k <= h->cfg.d; ++k) gs.slot[k - 1] = slot_back(h, k - 1);
          }
          e = launch_offset_prep(h->ost, h->cur, out, s, &gs);
          h->launches += 1;
          a.ost = h->ost;
          a.omin = &h->ost->mn[out];
        }
        if (e == cudaSuccess)
          e = (h->kernel == 4) ? launch_small(a, h->cfg.dtype, false, s, h->sms)
                               : launch_generic_sweep(a, h->cfg.dtype, s, h->sms);
      }
      h->launches += 1;
    }
    if (e != cudaSuccess)
      return set_err(h, LCSB_ECUDA, "sweep launch failed: %s", cudaGetErrorString(e));
    int rc = barrier(h);  // every shard's outputs are in place before the next sweep reads them
    if (rc != LCSB_OK) return rc;
    h->cur = out;
    h->sweeps_done += 1;
    if (trk) h->trk_at[h->sweeps_done & 1] = h->sweeps_done;
  }
  return LCSB_OK;
}

static double bound_from(const lcsb_t* h, double rho) {
  if (h->form == LCSB_FORM_KS) return (double)h->cfg.d * rho;  // Eq. (lwrbound)
  return rho > 0.0 ? 2.0 * rho / (1.0 + rho) : 0.0;           // reading R10
}

// the tracking set of sweep k (process mode: reduced over the ranks first) -> v[0..2]
static int read_trk(lcsb_t* h, int64_t k, unsigned long long* v) {
  const int first = kTrkSlot + 4 * (int)(k & 1);
  int rc = allreduce_slots(h, first, 3, (6u << first));
  if (rc != LCSB_OK) return rc;
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  CU(h, cudaMemcpyAsync(v, h->red + first, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        s));
  CU(h, cudaStreamSynchronize(s));
  return LCSB_OK;
}

// E, the bound for both R and the best-so-far update (Alg. 2 lines 7-10) of the iterate after
// `u_sweeps` sweeps, from R and max W
static int finish_bound(lcsb_t* h, const double (&R)[2], const double (&Wm)[2], int64_t u_sweeps,
                        lcsb_bound_t* out) {
  double E[2], B[2];
  for (int i = 0; i < 2; ++i) {
    E[i] = Wm[i] > 0.0 ? Wm[i] : 0.0;  // E = max(0, max W)
    B[i] = bound_from(h, R[i] - E[i]);
    if (R[i] - E[i] >= h->best_rho[i]) {  // Alg. 2 line 8
      h->best_rho[i] = R[i] - E[i];
      h->best_sweep[i] = u_sweeps;
    }
  }
  const int m = h->cfg.rmode;
  out->R_max = R[0];
  out->R_min = R[1];
  out->E_at_Rmax = E[0];
  out->E_at_Rmin = E[1];
  out->bound_at_Rmax = B[0];
  out->bound_at_Rmin = B[1];
  out->bound = B[m];
  out->best_bound = bound_from(h, h->best_rho[m]);
  out->sweeps_done = u_sweeps;
  out->best_sweep = h->best_sweep[m];
  return LCSB_OK;
}


extern "C" int lcsb_bound(lcsb_t* h, lcsb_bound_t* out) {
  if (!h || !out) return set_err(h, LCSB_EINVAL, "NULL argument");
  NvtxRange r("lcsb_bound");
  if (h->sweeps_done < 1) return set_err(h, LCSB_ESTATE, "lcsb_bound needs at least one sweep");
  if (h->base && h->sweeps_done <= h->rebase_sweep)
    return set_err(h, LCSB_ESTATE, "lcsb_bound needs a sweep after lcsb_rebase");
  CU(h, cudaSetDevice(h->device));
  {
    int rc = install_schedule(h, false);
    if (rc != LCSB_OK) return rc;
  }
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  const int prev = slot_back(h, 1);
  // quarter table (two-array binary): ONE pass gives R_max, R_min and D = min(F(u,u) - u); then
  // E = max(0, max W) = max(0, R - D) for both R (reading R21).  Other kernels: the R
  // reduction, then the W pass at the known R.
  const bool one_pass = h->kernel == 5;
  // the last sweep tracked R of this iterate (lcsb_sweep_ex): the pass needs only D, so it does
  // not read v_{n-1} at all (reading R25)
  const bool dpass = can_track(h) && h->trk_at[h->sweeps_done & 1] == h->sweeps_done;
  // integer offsets: v_n - v_{n-1} = s_n - s_{n-1} + (o_n - o_{n-1})  (reading R23)
  double cofs = 0.0;
  if (h->ost) {
    double offs[kMaxGen];
    CU(h, cudaMemcpyAsync(offs, h->ost->off, sizeof offs, cudaMemcpyDeviceToHost, s));
    CU(h, cudaStreamSynchronize(s));
    cofs = offs[h->cur] - offs[prev];
  }
  CU(h, launch_red_init(h->red, s, one_pass ? 6u : 2u));
  h->launches += 1;
  for (int k = h->first; !one_pass && k < h->first + h->nown; ++k) {
    CU(h, launch_rdiff(h->tabs[k][h->cur], h->tabs[k][prev], h->n_local, h->cfg.dtype, h->red, s,
                       h->sms));
    h->launches += 1;
  }
  if (!one_pass) {
    int rc = allreduce_slots(h, 0, 2, 2u);  // the global R before the W pass
    if (rc != LCSB_OK) return rc;
    if (h->ost) {  // the W pass reads R from the device: add the offset step there
      unsigned long long r[2];
      CU(h, cudaMemcpyAsync(r, h->red, sizeof r, cudaMemcpyDeviceToHost, s));
      CU(h, cudaStreamSynchronize(s));
      for (int i = 0; i < 2; ++i) r[i] = ord_enc(ord_dec(r[i]) + cofs);
      CU(h, cudaMemcpyAsync(h->red, r, sizeof r, cudaMemcpyHostToDevice, s));
    }
  }
  if (h->kernel == 2) {
    const int M = bin2_tma_wpass_m(h->cfg.dtype, h->cfg.ell, h->p);
    for (int k = h->first; k < h->first + h->nown; ++k) {
      Bin2Args a;
      fill_bin2(h, &a, k, h->cur, -1);
      a.red_in = h->red;
      a.red_out = h->red + 2;
      if (M > 0)
        CU(h, launch_bin2_tma_wpass(a, h->cfg.dtype, M, s, h->sms));
      else
        CU(h, launch_bin2_wpass(a, h->cfg.dtype, s, h->sms));
      h->launches += 1;
    }
  } else if (h->kernel == 5) {
    Bin2QArgs a;
    fill_bin2q(h, &a, h->cur, -1);
    a.prev = dpass ? nullptr : h->tabs[0][prev];
    a.red_out = h->red;
    for (int k = h->first; k < h->first + h->nown; ++k) {  // sharded: each owned shard's items
      if (h->vmm) {
        a.sched = h->qsched_sh[k];
        a.nitems = h->qsched_n_sh[k];
      }
      if (a.counter) CU(h, cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), s));
      CU(h, launch_bin2q_wpass(a, h->cfg.dtype, h->qM, s, h->sms));
      h->launches += 1;
      if (!h->vmm) break;
    }
  } else if (h->kernel == 3) {
    for (int k = h->first; k < h->first + h->nown; ++k) {
      Q4Args a;
      memset(&a, 0, sizeof a);
      a.g1 = h->tabs[k][h->cur];
      a.pin = h->pools[k][h->pcur];  // |N| = 2 reads v_n itself in the W pass (shift 0)
      a.flags = (h->form == LCSB_FORM_TWO_ARRAY) ? kQ4TwoArray : 0;
      a.ell = h->cfg.ell;
      a.red_in = h->red;
      a.red_out = h->red + 2;
      a.p = h->p;
      a.shard = k;
      for (int j = 0; j < h->P; ++j) a.g1_sh[j] = h->tabs[j][h->cur];  // u at the outputs
      CU(h, launch_q4_wpass(a, h->cfg.dtype, s, h->sms));
      h->launches += 1;
    }
  } else {
    GenericArgs a;
    fill_generic(h, &a);
    for (int k = 1; k <= h->cfg.d; ++k) a.src[k - 1] = h->tabs[0][h->cur];
    a.center = h->tabs[0][h->cur];
    a.red_in = h->red;
    a.red_out = h->red + 2;
    if (h->kernel == 4)
      CU(h, launch_small(a, h->cfg.dtype, true, s, h->sms));
    else
      CU(h, launch_generic_wpass(a, h->cfg.dtype, s, h->sms));
    h->launches += 1;
  }
  {
    int rc = one_pass ? allreduce_slots(h, 0, 3, 6u) : allreduce_slots(h, 2, 2, 0u);
    if (rc != LCSB_OK) return rc;
  }
  unsigned long long trk[4] = {0, 0, 0, 0};
  if (dpass) {
    int rc = read_trk(h, h->sweeps_done, trk);
    if (rc != LCSB_OK) return rc;
  }
  CU(h, cudaMemcpyAsync(h->red_host, h->red, kRedSlots * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, s));
  CU(h, cudaStreamSynchronize(s));
  if (dpass) {  // R of this iterate from its tracking sweep
    h->red_host[0] = trk[0];
    h->red_host[1] = trk[1];
  }
  // (generic two-pass with offsets: red[0..1] already hold the shifted R)
  const double radd = (one_pass && h->ost) ? cofs : 0.0;
  const double R[2] = {ord_dec(h->red_host[0]) + radd, ord_dec(h->red_host[1]) + radd};
  double Wm[2] = {ord_dec(h->red_host[2]), ord_dec(h->red_host[3])};
  if (one_pass) {  // max W = max(u + R - F(u,u)) = R - min(F(u,u) - u)   (reading R21)
    const double D = ord_dec(h->red_host[2]);
    Wm[0] = R[0] - D;
    Wm[1] = R[1] - D;
  }
  return finish_bound(h, R, Wm, h->sweeps_done, out);
}

// n sweeps and the bound of the iterate BEFORE the last of them (reading R25): Alg. 2's W of
// iterate u = v_{N-1} needs F(u,u), which the two-array form computes as sweep N anyway, so the
// last two sweeps track (R of v_{N-1} against v_{N-2}; D = min(F(u,u) - u)) and no pass over the
// table is added.  Layouts without tracking sweeps (and n = 1 after an untracked sweep): the
// same result from sweeps, lcsb_bound and one more sweep.
extern "C" int lcsb_sweep_bound(lcsb_t* h, int64_t n, lcsb_bound_t* out) {
  if (!h || !out) return set_err(h, LCSB_EINVAL, "NULL argument");
  NvtxRange r("lcsb_sweep_bound");
  if (n < 1) return set_err(h, LCSB_EINVAL, "n must be >= 1");
  const int64_t N = h->sweeps_done + n;
  if (N - 1 < 1) return set_err(h, LCSB_ESTATE, "the bounded iterate needs at least one sweep");
  if (h->base && N - 1 <= h->rebase_sweep)
    return set_err(h, LCSB_ESTATE, "lcsb_bound needs a sweep after lcsb_rebase");
  const bool fused = can_track(h) && (n >= 2 || h->trk_at[h->sweeps_done & 1] == h->sweeps_done);
  if (!fused) {
    int rc = sweep_impl(h, n - 1, 0);
    if (rc == LCSB_OK) rc = lcsb_bound(h, out);
    if (rc == LCSB_OK) rc = sweep_impl(h, 1, 0);
    return rc;
  }
  int rc = sweep_impl(h, n, 2);
  if (rc != LCSB_OK) return rc;
  if (h->trk_at[(N - 1) & 1] != N - 1 || h->trk_at[N & 1] != N)
    return set_err(h, LCSB_ESTATE, "tracking sets missing");
  unsigned long long tr[4], td[4];
  rc = read_trk(h, N - 1, tr);
  if (rc == LCSB_OK) rc = read_trk(h, N, td);
  if (rc != LCSB_OK) return rc;
  const double R[2] = {ord_dec(tr[0]), ord_dec(tr[1])};
  const double D = ord_dec(td[2]);  // min(F(v_{N-1}) - v_{N-1})
  const double Wm[2] = {R[0] - D, R[1] - D};  // max W = R - D (reading R21)
  return finish_bound(h, R, Wm, N - 1, out);
}

static int readout(lcsb_t* h, int which, uint64_t first, uint64_t count, const uint64_t* host_idx,
                   double* host_dst) {
  if (!h) return set_err(nullptr, LCSB_EINVAL, "handle is NULL");
  if (!host_dst && count) return set_err(h, LCSB_EINVAL, "host_dst is NULL");
  const int maxback = (h->form == LCSB_FORM_KS) ? h->cfg.d - 1 : 1;
  if (which < 0 || which > maxback)
    return set_err(h, LCSB_EINVAL, "which must be in [0, %d]", maxback);
  if (!host_idx && (first > h->n_logical || count > h->n_logical - first))
    return set_err(h, LCSB_EINVAL, "range [%llu, +%llu) outside the %llu states",
                   (unsigned long long)first, (unsigned long long)count,
                   (unsigned long long)h->n_logical);
  if (host_idx)
    for (uint64_t i = 0; i < count; ++i)
      if (host_idx[i] >= h->n_logical)
        return set_err(h, LCSB_EINVAL, "index %llu out of range", (unsigned long long)host_idx[i]);
  if (count == 0) return LCSB_OK;
  if (h->base && which > 0 && h->sweeps_done - which < h->rebase_sweep)
    return set_err(h, LCSB_ESTATE, "the generation before lcsb_rebase is not kept");
  if (which > h->sweeps_done) {  // a generation before the start: W_0 = 0 (never stored)
    memset(host_dst, 0, count * sizeof(double));
    return LCSB_OK;
  }
  CU(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  const int slot = slot_back(h, which);
  const void* tabs[kMaxShards];
  for (int k = 0; k < h->P; ++k) tabs[k] = h->tabs[k][slot];
  const uint64_t chunk = 1ull << 22;
  const uint64_t c0 = count < chunk ? count : chunk;
  double* dbuf = (double*)dev_alloc(h, c0 * sizeof(double));
  uint64_t* ibuf = host_idx ? (uint64_t*)dev_alloc(h, c0 * sizeof(uint64_t)) : nullptr;
  if (!dbuf || (host_idx && !ibuf)) {
    dev_free(h, dbuf, c0 * sizeof(double));
    dev_free(h, ibuf, c0 * sizeof(uint64_t));
    return set_err(h, LCSB_ECAPACITY, "staging allocation failed");
  }
  int rc = LCSB_OK;
  for (uint64_t off = 0; off < count && rc == LCSB_OK; off += c0) {
    const uint64_t c = (count - off) < c0 ? (count - off) : c0;
    cudaError_t e = cudaSuccess;
    if (host_idx)
      e = cudaMemcpyAsync(ibuf, host_idx + off, c * sizeof(uint64_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = launch_expand(tabs, h->p, h->cfg.dtype, h->symmetric != 0 || h->kernel == 3,
                        h->kernel == 3, h->ost ? &h->ost->off[slot] : nullptr, h->base,
                        h->n_logical, h->cfg.ell, h->qmap, h->qK,
                        first + off, c, host_idx ? ibuf : nullptr, dbuf, s);
    if (e == cudaSuccess) {
      h->launches += 1;
      e = cudaMemcpyAsync(host_dst + off, dbuf, c * sizeof(double), cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess)
      rc = set_err(h, LCSB_ECUDA, "table read-out failed: %s", cudaGetErrorString(e));
  }
  dev_free(h, dbuf, c0 * sizeof(double));
  dev_free(h, ibuf, c0 * sizeof(uint64_t));
  return rc;
}

extern "C" int lcsb_table(lcsb_t* h, int32_t which, uint64_t first, uint64_t count,
                          double* host_dst) {
  return readout(h, which, first, count, nullptr, host_dst);
}

extern "C" int lcsb_table_gather(lcsb_t* h, int32_t which, const uint64_t* host_idx, uint64_t n,
                                 double* host_dst) {
  if (!host_idx && n) return set_err(h, LCSB_EINVAL, "host_idx is NULL");
  return readout(h, which, 0, n, host_idx, host_dst);
}

// ---------------------------------------------------------------- residual storage (R24)
extern "C" int lcsb_rebase(lcsb_t* h) {
  if (!h) return set_err(nullptr, LCSB_EINVAL, "handle is NULL");
  if (h->kernel != 5 || h->cfg.dtype != LCSB_F32 || !h->ost || h->mode != MODE_SINGLE)
    return set_err(h, LCSB_EINVAL,
                   "lcsb_rebase needs the quarter table with fp32 storage and offset_policy = 1");
  NvtxRange r("lcsb_rebase");
  CU(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  if (h->base) {
    // already rebased: fold the residual into the base, H := round32(H + e), e := the exact
    // rounding residual -- the iterate (H + e) is unchanged and e shrinks back to ~ulp(H)
    CU(h, launch_rebase_fold(h->base, h->tabs[0][h->cur], h->n_stored, s, h->sms));
    h->launches += 1;
  } else {
    h->base = dev_alloc(h, h->tab_bytes);
    if (!h->base)
      return set_err(h, LCSB_ECAPACITY, "base table allocation (%llu bytes) failed",
                     (unsigned long long)h->tab_bytes);
    // H := the newest stored table s (v = s + o), e := 0; mn[cur] = min(s) = min(H + e) holds
    CU(h, cudaMemcpyAsync(h->base, h->tabs[0][h->cur], h->tab_bytes, cudaMemcpyDeviceToDevice, s));
    CU(h, cudaMemsetAsync(h->tabs[0][h->cur], 0, h->tab_bytes, s));
  }
  static const double q = 1.0 / 64.0;  // finer offsets: the residual stays below one sweep's growth
  CU(h, cudaMemcpyAsync(&h->ost->quantum, &q, sizeof q, cudaMemcpyHostToDevice, s));
  CU(h, cudaStreamSynchronize(s));
  for (int i = 0; i < kMaxGen; ++i)  // captured sweeps know no base
    if (h->graph[i]) {
      cudaGraphExecDestroy(h->graph[i]);
      h->graph[i] = nullptr;
    }
  h->rebase_sweep = h->sweeps_done;
  h->trk_at[0] = h->trk_at[1] = -1;
  return LCSB_OK;
}

// ---------------------------------------------------------------- checkpoint / resume
// File: a header (the run's identity and its scalar state), then every device buffer the next
// sweep or bound reads, in a fixed order: the table ring, the q4 row-mean ring, the small
// kernel's pooled means, the offset state.  Raw stored entries (the layout is a function of the
// config), so a checkpoint restores into a handle created with the same config.
struct CkptHeader {
  char magic[8];  // "LCSBCKP1"
  int32_t sigma, d, ell, dtype, form, symmetric, kernel, qK, ntab, offsets, spooled, based;
  uint64_t n_stored, tab_bytes, pool_bytes;
  int32_t cur, pcur;
  int64_t sweeps_done;
  double best_rho[2];
  int64_t best_sweep[2];
  int64_t rebase_sweep;
};

template <typename F>
static int for_each_buffer(lcsb_t* h, F f) {  // (device pointer, bytes) in the file's order
  for (int i = 0; i < h->ntab; ++i) {
    int rc = f(h->tabs[0][i], h->tab_bytes);
    if (rc != LCSB_OK) return rc;
  }
  for (int i = 0; i < 3; ++i)
    if (h->pools[0][i]) {
      int rc = f(h->pools[0][i], h->pool_bytes);
      if (rc != LCSB_OK) return rc;
    }
  for (int k = 0; k <= kMaxD; ++k)
    for (int i = 0; i < kMaxGen; ++i)
      if (h->spools[k][i]) {
        int rc = f(h->spools[k][i], h->spool_bytes[k]);
        if (rc != LCSB_OK) return rc;
      }
  if (h->base) {
    int rc = f(h->base, h->tab_bytes);
    if (rc != LCSB_OK) return rc;
  }
  if (h->ost) return f(h->ost, sizeof(OffState));
  return LCSB_OK;
}

static CkptHeader ckpt_header(const lcsb_t* h) {
  CkptHeader c;
  memset(&c, 0, sizeof c);
  memcpy(c.magic, "LCSBCKP1", 8);
  c.sigma = h->cfg.sigma;
  c.d = h->cfg.d;
  c.ell = h->cfg.ell;
  c.dtype = h->cfg.dtype;
  c.form = h->form;
  c.symmetric = h->symmetric;
  c.kernel = h->kernel;
  c.qK = h->qK;
  c.ntab = h->ntab;
  c.offsets = h->ost != nullptr;
  c.spooled = h->spooled;
  c.based = h->base != nullptr;
  c.n_stored = h->n_stored;
  c.tab_bytes = h->tab_bytes;
  c.pool_bytes = h->pool_bytes;
  return c;
}

extern "C" int lcsb_save(lcsb_t* h, const char* path) {
  if (!h || !path) return set_err(h, LCSB_EINVAL, "NULL argument");
  if (h->mode != MODE_SINGLE)
    return set_err(h, LCSB_EINVAL, "checkpoints are per handle of one GPU (unsharded)");
  CU(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  CU(h, cudaStreamSynchronize(s));
  FILE* f = fopen(path, "wb");
  if (!f) return set_err(h, LCSB_EINVAL, "cannot open %s for writing", path);
  CkptHeader c = ckpt_header(h);
  c.cur = h->cur;
  c.pcur = h->pcur;
  c.sweeps_done = h->sweeps_done;
  c.best_rho[0] = h->best_rho[0];
  c.best_rho[1] = h->best_rho[1];
  c.best_sweep[0] = h->best_sweep[0];
  c.best_sweep[1] = h->best_sweep[1];
  c.rebase_sweep = h->rebase_sweep;
  const size_t chunk = 64ull << 20;
  char* buf = (char*)malloc(chunk);
  int rc = (buf && fwrite(&c, sizeof c, 1, f) == 1) ? LCSB_OK
                                                    : set_err(h, LCSB_EINVAL, "write failed");
  if (rc == LCSB_OK)
    rc = for_each_buffer(h, [&](void* d, size_t bytes) -> int {
      for (size_t o = 0; o < bytes; o += chunk) {
        const size_t n = bytes - o < chunk ? bytes - o : chunk;
        cudaError_t e = cudaMemcpy(buf, (char*)d + o, n, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess)
          return set_err(h, LCSB_ECUDA, "checkpoint read-back: %s", cudaGetErrorString(e));
        if (fwrite(buf, 1, n, f) != n) return set_err(h, LCSB_EINVAL, "write to %s failed", path);
      }
      return LCSB_OK;
    });
  free(buf);
  if (fclose(f) != 0 && rc == LCSB_OK) rc = set_err(h, LCSB_EINVAL, "closing %s failed", path);
  return rc;
}

extern "C" int lcsb_load(lcsb_t* h, const char* path) {
  if (!h || !path) return set_err(h, LCSB_EINVAL, "NULL argument");
  if (h->mode != MODE_SINGLE)
    return set_err(h, LCSB_EINVAL, "checkpoints are per handle of one GPU (unsharded)");
  CU(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  CU(h, cudaStreamSynchronize(s));
  FILE* f = fopen(path, "rb");
  if (!f) return set_err(h, LCSB_EINVAL, "cannot open %s", path);
  CkptHeader c, want = ckpt_header(h);
  int rc = LCSB_OK;
  if (fread(&c, sizeof c, 1, f) != 1 || memcmp(c.magic, "LCSBCKP1", 8) != 0)
    rc = set_err(h, LCSB_EINVAL, "%s is not an lcsb checkpoint", path);
  else if (memcmp(&c.sigma, &want.sigma, offsetof(CkptHeader, cur) - offsetof(CkptHeader, sigma)))
    rc = set_err(h, LCSB_EINVAL,
                 "checkpoint %s was written by a handle of another config or layout", path);
  else if (c.cur < 0 || c.cur >= h->ntab || c.pcur < 0 || c.pcur > 2 || c.sweeps_done < 0)
    rc = set_err(h, LCSB_EINVAL, "checkpoint %s has a corrupt header", path);
  const size_t chunk = 64ull << 20;
  char* buf = rc == LCSB_OK ? (char*)malloc(chunk) : nullptr;
  if (rc == LCSB_OK && !buf) rc = set_err(h, LCSB_ECAPACITY, "host buffer allocation failed");
  if (rc == LCSB_OK)
    rc = for_each_buffer(h, [&](void* d, size_t bytes) -> int {
      for (size_t o = 0; o < bytes; o += chunk) {
        const size_t n = bytes - o < chunk ? bytes - o : chunk;
        if (fread(buf, 1, n, f) != n) return set_err(h, LCSB_EINVAL, "%s is truncated", path);
        cudaError_t e = cudaMemcpy((char*)d + o, buf, n, cudaMemcpyHostToDevice);
        if (e != cudaSuccess)
          return set_err(h, LCSB_ECUDA, "checkpoint upload: %s", cudaGetErrorString(e));
      }
      return LCSB_OK;
    });
  free(buf);
  fclose(f);
  if (rc != LCSB_OK) return rc;
  h->cur = c.cur;
  h->pcur = c.pcur;
  h->sweeps_done = c.sweeps_done;
  h->best_rho[0] = c.best_rho[0];
  h->best_rho[1] = c.best_rho[1];
  h->best_sweep[0] = c.best_sweep[0];
  h->best_sweep[1] = c.best_sweep[1];
  h->rebase_sweep = c.rebase_sweep;
  h->trk_at[0] = h->trk_at[1] = -1;
  return LCSB_OK;
}

extern "C" int64_t lcsb_sweeps_done(const lcsb_t* h) { return h ? h->sweeps_done : -1; }
extern "C" int32_t lcsb_num_shards(const lcsb_t* h) { return h ? h->P : 0; }
extern "C" uint64_t lcsb_num_states(const lcsb_t* h) { return h ? h->n_logical : 0; }
extern "C" uint64_t lcsb_stored_states(const lcsb_t* h) { return h ? h->n_stored : 0; }
extern "C" uint64_t lcsb_device_bytes(const lcsb_t* h) {
  if (!h) return 0;
  uint64_t b = (uint64_t)h->tab_bytes * ((uint64_t)h->ntab * (uint64_t)h->nown + (h->base ? 1 : 0)) + 256 +
               h->qmap_bytes + h->qsched_bytes + 3 * (uint64_t)h->pool_bytes * (uint64_t)h->nown;
  for (int k = 0; k <= kMaxD; ++k)
    for (int i = 0; i < kMaxGen; ++i)
      if (h->spools[k][i]) b += h->spool_bytes[k];
  return b;
}
extern "C" int32_t lcsb_kernel_in_use(const lcsb_t* h) { return h ? h->kernel : 0; }
extern "C" int lcsb_shard_traffic(const lcsb_t* h, uint64_t* peer_read_bytes,
                                  uint64_t* peer_written_bytes, uint64_t* requested_bytes) {
  if (!h || !peer_read_bytes || !peer_written_bytes || !requested_bytes)
    return set_err(nullptr, LCSB_EINVAL, "NULL argument");
  if (!h->vmm) return set_err(nullptr, LCSB_EINVAL, "not a sharded quarter table");
  *peer_read_bytes = h->peer_read * h->esize;
  *peer_written_bytes = h->peer_written * h->esize;
  *requested_bytes = h->all_moved * h->esize;
  return LCSB_OK;
}
extern "C" int64_t lcsb_launch_count(const lcsb_t* h) { return h ? h->launches : 0; }
extern "C" const char* lcsb_last_error(const lcsb_t* h) { return h ? h->err : g_err; }
