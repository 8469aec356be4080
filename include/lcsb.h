/*
 * lcsb.h -- C-ABI of the B200 Feasible Triplet library (liblcsb.so).
 *
 * The library computes the value-iteration sweep of the Feasible Triplet recurrence of
 * arXiv 2407.10925 (Kiwi-Soto's F; Alg. 1; Alg. 2
 * PAPER.md:696-717; binary Alg. 5 PAPER.md:728-750 with F_0/F_1 of PAPER.md:752-779) and the
 * bound reduction that turns the swept table into a certified lower bound on the
 * Chvatal-Sankoff constant gamma_{sigma,d} (Lemma 1).
 *
 * A "state" is a d-tuple of length-l strings over {0..sigma-1}; a table holds one real per
 * state, sigma^(d l) of them.  Logical state order (reading R14):
 *     idx = sum_{k<l} sum_{j<d} A_j[k] * sigma^(d(l-1-k) + (d-1-j))
 * i.e. the heads are the most significant digit group and string 0 is the most significant
 * digit of each group.  For sigma = d = 2 this is the paper's interleaved pair
 * (a = 1011, b = 0010 -> 142).
 *
 * Every pointer argument is a HOST pointer unless stated otherwise; the library owns all of
 * its device memory.  Functions return LCSB_OK (0) or an error code and never abort; the
 * message of the last failure is available from lcsb_last_error().  A handle is not
 * thread-safe; distinct handles are independent.
 */
#ifndef LCSB_H
#define LCSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lcsb lcsb_t; /* opaque; owns every device table and scratch buffer */

/* STORAGE dtype of the tables.  Arithmetic is always fp64 (BASELINE.json: "fp32 storage with
 * fp64 accumulation"); LCSB_F32 rounds every stored value to nearest-even fp32. */
enum { LCSB_F64 = 0, LCSB_F32 = 1 };

/* Recurrence form.
 *   KS:        Alg. 2 / Alg. 5 -- an option that advances k strings reads the table k sweeps
 *              back (reading R1); d+1 tables live.
 *   TWO_ARRAY: Lueker's two-array form for sigma = d = 2 ("storing only two arrays",
 *              PAPER.md:400): every option reads the previous sweep; 2 tables live; the bound
 *              is 2 rho / (1 + rho) with rho = R - E (reading R10).  Also accepted for d = 2
 *              and any sigma (beyond the paper, reading R20): the option that drops
 *              both heads when they differ is not offered.  d > 2 is rejected (LCSB_EINVAL).
 *   AUTO:      TWO_ARRAY for sigma = d = 2, KS otherwise. */
enum { LCSB_FORM_AUTO = 0, LCSB_FORM_KS = 1, LCSB_FORM_TWO_ARRAY = 2 };

/* Which R the headline bound uses (reading R5).  Both are always computed:
 *   R_MAX = max(v_new - v_prev) (Alg. 2 line 5), R_MIN = min(...). */
enum { LCSB_R_MAX = 0, LCSB_R_MIN = 1 };

/* Kernel selection: AUTO picks the specialised kernel for the shape; GENERIC forces the
 * full-table one-thread-per-state kernel (used as a cross-check). */
enum { LCSB_KERNEL_AUTO = 0, LCSB_KERNEL_GENERIC = 1 };

/* Status codes. */
enum {
  LCSB_OK = 0,
  LCSB_EINVAL = 1,    /* bad argument or unsupported combination */
  LCSB_ECAPACITY = 2, /* not enough device memory; lcsb_last_error() states the bytes needed */
  LCSB_ESTATE = 3,    /* call not valid in the handle's state (e.g. bound before any sweep) */
  LCSB_ECUDA = 4,     /* a CUDA runtime call failed */
  LCSB_ENCCL = 5      /* a communication call of the sharded process mode failed (NCCL, or a
                         comm hook returned non-zero) */
};

/* Device allocation hooks (optional).  alloc returns a device pointer of >= bytes, 256-B
 * aligned, usable on `stream`, or NULL; free_ releases it.  NULL hooks -> cudaMallocAsync /
 * cudaFreeAsync on the handle's stream.  The Python binding passes the PyTorch caching
 * allocator here. */
typedef void* (*lcsb_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*lcsb_free_fn)(void* ptr, size_t bytes, void* stream, void* ctx);

/* Host communication hooks of the process-sharded mode (optional).  When lcsb_config.comm is
 * non-NULL the library uses these instead of NCCL: the CUDA IPC handles of the tables are
 * exchanged with allgather, the per-sweep barrier is "synchronise this handle's stream, then
 * barrier()" (so lcsb_sweep becomes synchronous), and the bound's 4 reduction scalars cross the
 * ranks through allreduce_max_u64 (the library encodes minima so that a max serves).  No kernel
 * ever waits on another rank, so several processes may share one GPU (how the multi-process
 * path is tested on one device: DESIGN.md §9).  Each hook returns 0 on success; a non-zero return
 * fails the call with LCSB_ENCCL.  The hooks are called only from the calling thread, inside
 * collective library calls. */
typedef struct {
  /* every rank passes `bytes` bytes at `mine`; on return `all` holds the P contributions in rank
   * order (P * bytes, host memory) */
  int (*allgather)(const void* mine, void* all, size_t bytes, void* ctx);
  /* returns once every rank has entered it */
  int (*barrier)(void* ctx);
  /* element-wise maximum over the ranks of n unsigned 64-bit values, in place (host memory) */
  int (*allreduce_max_u64)(uint64_t* vals, int32_t n, void* ctx);
  void* ctx;
} lcsb_comm_hooks;

typedef struct {
  int32_t sigma;    /* alphabet size, >= 2 */
  int32_t d;        /* number of strings, 2..16 */
  int32_t ell;      /* string-length parameter l >= 1; sigma^(d l) must be < 2^62 */
  int32_t dtype;    /* LCSB_F64 / LCSB_F32 */
  int32_t form;     /* LCSB_FORM_* */
  int32_t rmode;    /* LCSB_R_* : which R gives lcsb_bound_t.bound / best_bound */
  int32_t symmetry; /* -1 auto; 0 full logical table; 1 complement-folded half table
                       (two-array binary only, l >= 2); 2 symmetry-folded
                       ("quarter") table: one entry per orbit of {id, complement, string swap,
                       both}, same-head states also folded under the tail complement
                       (v'[00t] = v'[00t~]): 3/16 of the states (two-array
                       binary, unsharded, l >= block_log4 + 1; string swap = reading R19 of
                       DESIGN.md, implied by "if symmetry is fully exploited").
                       AUTO = 2 for l >= 12 unsharded, 1 otherwise when allowed, else 0. */
  int32_t kernel;   /* LCSB_KERNEL_* */
  void* stream;     /* cudaStream_t every kernel and copy is enqueued on; NULL = legacy default */
  lcsb_alloc_fn alloc;
  lcsb_free_fn free_;
  void* alloc_ctx;
  /* ---- sharding of the complement-folded binary half table (two-array form) ----
   * The stored table is split over `shards` = P in {1, 2, 4, 8} shards by a key on the first
   * characters of both strings; every sweep reads only the shard's own table and writes its
   * outputs into the owners' tables (peer stores over NVLink).  Two modes:
   *   virtual_shards = 1: this handle holds all P shards on its own GPU (one-GPU mode, used to
   *                       test the sharded kernels; no communication library involved);
   *   virtual_shards = 0, P > 1: one process per GPU, this process owns shard `shard`; either
   *                       all P processes pass the same 128-byte ncclUniqueId in nccl_id (from
   *                       lcsb_nccl_unique_id on one rank) -- the library builds its own NCCL
   *                       communicator, exchanges CUDA IPC handles of the tables through it, and
   *                       uses NCCL all-reduces on the stream for the per-sweep barrier and the
   *                       bound -- or all pass comm hooks (below; no NCCL involved).  Every
   *                       process must call create / reset / sweep / bound / destroy collectively. */
  int32_t shards;
  int32_t shard;
  int32_t virtual_shards;
  const void* nccl_id;
  /* quarter table only: the table is cut into blocks of 4^block_log4 entries that are stored
   * whole or read through the swap permutation; 0 = auto (min(7, l-5) for F32, min(6, l-5)
   * for F64, at least 2).  Must satisfy 2 <= block_log4 <= l - 1. */
  int32_t block_log4;
  /* process-sharded mode: host communication hooks instead of NCCL (see lcsb_comm_hooks); the
   * struct must stay valid until lcsb_destroy returns.  NULL = NCCL (nccl_id). */
  const lcsb_comm_hooks* comm;
  /* integer-offset storage (readings R23, R26):
   *   0 = none (default);
   *   1 = each table holds s = v - o with an integer o: before every sweep c = floor(min s) of
   *       the table it reads, and the sweep stores round(F(s) - c) (F(v + c) = F(v) + c,
   *       translation invariance, Lemma 1 (2)), so stored magnitudes stay small and
   *       fp32 storage drifts less.  Values read out (lcsb_table) and the bound are those of v.
   *       Two-array form: binary on the quarter table (l >= 3) or, below that, the generic
   *       kernel; other sigma (d = 2): the generic kernel (q4 for sigma = 4, l >= 4).  KS form
   *       (any sigma, d; R26): the generic kernel or q4 (sigma = 4, d = 2); every generation
   *       keeps its own o and the means over the table k sweeps back get o_{n+1-k} - o_n added.
   *       The half table and sharding: LCSB_EINVAL. */
  int32_t offset_policy;
} lcsb_config;

/* Fill *cfg with defaults: sigma=2,d=2,ell=1, F32, AUTO form, R_MAX, symmetry auto, AUTO
 * kernel, NULL stream and hooks, 1 shard. */
void lcsb_config_init(lcsb_config* cfg);

/* Device bytes a handle with this config would own (tables + scratch).  0 on bad config. */
uint64_t lcsb_required_bytes(const lcsb_config* cfg);

/* Create a handle and zero every live table: W_0 = 0, the (d+1) x sigma^(d l) zero matrix of
 * Alg. 2 line 2 / v_0 = v_1 = 0 of Alg. 5.
 * Errors: EINVAL (bad parameters), ECAPACITY (device memory), ECUDA. */
int lcsb_create(int32_t sigma, int32_t d, int32_t ell, int32_t dtype, lcsb_t** out);
int lcsb_create_ex(const lcsb_config* cfg, lcsb_t** out);

/* Restart the run without reallocating: zero every live table again (W_0 = 0), reset the sweep
 * count and the best-so-far triplet.  Asynchronous.  Errors: ECUDA. */
int lcsb_reset(lcsb_t* h);

/* Enqueue n >= 0 sweeps on the handle's stream and return (asynchronous).  One sweep computes
 * v_new = F(v_{n-1}, ..., v_{n-d}) at every state (Eq. ineq3) and rotates the
 * generations (Alg. 2 line 11).  Process-sharded mode: collective; a barrier precedes the first
 * sweep (so rank-local table reads made since the last collective call are complete before any
 * rank overwrites a generation) and follows every sweep.  Errors: EINVAL (n < 0), ECUDA (launch
 * failure), ENCCL. */
int lcsb_sweep(lcsb_t* h, int64_t n);

/* lcsb_sweep_ex flags (round 2, reading R25).  A TRACKING sweep v_k = F(v_{k-1}) also reads
 * v_{k-1} at every stored output and reduces R_max, R_min of v_k - v_{k-1} (Alg. 5 line 7,
 * PAPER.md:738, the R of the iterate it writes) and D = min(F(v_{k-1}) - v_{k-1}) (F in fp64
 * before the storage rounding; max W = R - D, reading R21, for the iterate it reads) into device
 * slots kept with the handle.  TRACK: the last sweep of the call tracks; TRACK2: the last two.
 * Only the binary quarter table with plain storage has tracking sweeps; elsewhere the flags are
 * accepted and ignored (the sweeps are plain). */
#define LCSB_SWEEP_TRACK 1u
#define LCSB_SWEEP_TRACK2 3u

/* lcsb_sweep with flags (above).  A tracked last sweep lets the next lcsb_bound skip the read of
 * v_{n-1} (it evaluates only D at the current iterate, with R from the tracking sweep); values,
 * R and the bound are identical to the untracked path.  Errors: as lcsb_sweep; EINVAL (unknown
 * flag bits). */
int lcsb_sweep_ex(lcsb_t* h, int64_t n, uint32_t flags);

typedef struct {
  double R_max, R_min;         /* max / min over states of v_new - v_prev */
  double E_at_Rmax, E_at_Rmin; /* E = max(0, max W) for each R (Alg. 2 lines 6-7) */
  double bound_at_Rmax, bound_at_Rmin; /* KS: d (R - E); two-array: 2 rho/(1+rho), rho = R-E */
  double bound;                /* bound_at_R<rmode> */
  double best_bound;           /* best over every lcsb_bound call so far for rmode, starting
                                  from the triplet (v_0, 0, 0) (Alg. 2 lines 2, 8-10) */
  int64_t sweeps_done;         /* sweeps of the iterate u the bound certifies (lcsb_bound: the
                                  handle's sweep count; lcsb_sweep_bound: that count - 1) */
  int64_t best_sweep;          /* sweeps_done at the best evaluation (0 = initial triplet) */
} lcsb_bound_t;

/* Evaluate the bound at the current iterate (Alg. 2 lines 5-10) for both R readings.
 * Synchronises the handle's stream; the only host round-trip of the path.
 * Errors: ESTATE (no sweep yet), ECUDA. */
int lcsb_bound(lcsb_t* h, lcsb_bound_t* out);

/* Enqueue n >= 1 sweeps and evaluate the bound (Alg. 2 lines 5-10, both R readings, best-so-far
 * update) of the iterate BEFORE the last of them, u = v_{N-1} with N = sweeps after the call
 * (reading R25): in the two-array form Alg. 2's W needs F(u,u) = v_N, i.e. exactly the last
 * sweep, so on the quarter table the last two sweeps are tracking sweeps and no pass over the
 * table is added (R of u from sweep N-1, D of u from sweep N).  Other layouts give the same values
 * by lcsb_sweep(n-1), lcsb_bound, lcsb_sweep(1).  out->sweeps_done = N - 1.  Synchronises the
 * stream.  Errors: EINVAL (n < 1), ESTATE (N - 1 < 1, or no sweep after lcsb_rebase), ECUDA,
 * ENCCL. */
int lcsb_sweep_bound(lcsb_t* h, int64_t n, lcsb_bound_t* out);

/* Copy count table entries, logical indices [first, first+count), of generation `which`
 * (0 = newest, 1 = one sweep back, ... up to d-1 for KS / 1 for two-array) into host_dst,
 * unfolded (complement symmetry applied) and widened to fp64.  Synchronous.
 * Errors: EINVAL (range / which), ECUDA. */
int lcsb_table(lcsb_t* h, int32_t which, uint64_t first, uint64_t count, double* host_dst);

/* Same for n arbitrary logical indices host_idx[0..n) -> host_dst[0..n).  Synchronous. */
int lcsb_table_gather(lcsb_t* h, int32_t which, const uint64_t* host_idx, uint64_t n,
                      double* host_dst);

/* Write a fresh ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128) into out[0..len); for sharded
 * process mode, called on one rank and broadcast to the others by the caller.  Errors: EINVAL
 * (len < 128), ENCCL. */
int lcsb_nccl_unique_id(void* out, size_t len);

/* Host-only sharding plan (no GPU needed): the shard and shard-local index holding logical
 * state `logical` of the binary (sigma = d = 2) complement-folded table of length-ell strings
 * split over `shards` shards.  Errors: EINVAL. */
int lcsb_shard_locate(int32_t ell, int32_t shards, uint64_t logical, int32_t* shard,
                      uint64_t* local);

/* Host-only sharding plan (no GPU needed) of the sigma = 4, d = 2 complement-folded table (the
 * q4 kernel): shard and shard-local index of logical state `logical` for
 * `shards` in {1, 2, 4, 8} (l >= 4; l >= 5 for 8 shards).  Errors: EINVAL. */
int lcsb_shard_locate_sigma4(int32_t ell, int32_t shards, uint64_t logical, int32_t* shard,
                             uint64_t* local);

/* Host-only layout query (no GPU needed): the stored index of logical state `logical` in the
 * quarter table (symmetry = 2) of the binary two-array form with length-ell strings and blocks
 * of 4^block_log4 entries, and the number of stored entries.  Every stored entry holds states
 * of ONE class -- an orbit of {id, complement, string swap, both}, for same-head states joined
 * with its tail complement -- so sharing it is exact; every stored entry is used; a class
 * occupies two entries only inside the few blocks that a symmetry maps onto themselves.  Requires 3 <= ell <= 31, 2 <= block_log4 <= ell - 1,
 * ell - block_log4 <= 12.  Errors: EINVAL. */
int lcsb_quarter_locate(int32_t ell, int32_t block_log4, uint64_t logical, uint64_t* stored,
                        uint64_t* n_stored);

/* Host-only plan query (no GPU needed) of the sharded quarter table of the
 * binary two-array form, length-ell strings, storage `dtype`, `shards` = 2, 4 or 8 GPUs and
 * `passes` passes of the placement search (as lcsb_create would build it): per shard k, the
 * items (tile pairs) it runs, and the table ENTRIES one sweep of those items reads from other
 * shards' memory (windows) and stores into them (output runs).  The arrays hold `shards`
 * values.  Deterministic; takes seconds at ell = 18.  Errors: EINVAL (no sharded quarter table
 * for the configuration: ell too small for the key, other shard counts). */
int lcsb_quarter_shard_plan(int32_t ell, int32_t dtype, int32_t shards, int32_t passes,
                            uint64_t* items, uint64_t* peer_read, uint64_t* peer_written);

/* Host preparations that affect only speed -- the quarter table's L2 item schedule, which
 * lcsb_create builds on a host thread so that it returns without waiting (about 0.4-1.5 s at
 * l = 17) -- are installed by the first lcsb_sweep / lcsb_bound after they are ready; sweeps
 * before that run the natural item order, with bit-identical results.  lcsb_ready installs them
 * if ready and returns 1 (0 = still being built; wait != 0 blocks until they are).  -1 on error. */
int32_t lcsb_ready(lcsb_t* h, int32_t wait);

/* Residual storage (reading R24; quarter table, fp32, offset_policy = 1): the newest
 * stored table becomes a fixed base H (one more table of device memory), the tables hold the
 * residual e = v - o - H from then on (e := 0 now), the offset steps become multiples of 1/64,
 * and every sweep stores round_fp32((F(H + e) - c) - H): H + e is exact in fp64 and the residual
 * stays below one sweep's growth, so the iterate carries ~64x the precision of fp32 values --
 * fp64-quality bounds at 12 instead of 16 bytes per stored entry (l = 18 on one B200).  The
 * generation before the rebase is dropped: lcsb_bound and lcsb_table(which >= 1) need a sweep
 * after it (LCSB_ESTATE).  Calling it again on a rebased handle folds the residual into the
 * base (H := round32(H + e), e := the exact rounding residual; the iterate is unchanged) -- for
 * when the iterate's shape has moved away from H.  lcsb_reset returns to plain storage.  To
 * resume a rebased checkpoint, call lcsb_rebase on the fresh handle before lcsb_load.
 * Errors: EINVAL (not that layout), ECAPACITY, ECUDA. */
int lcsb_rebase(lcsb_t* h);

/* Checkpoint / resume (long converging runs): lcsb_save writes every buffer the next
 * sweep or bound reads (the table ring, row-mean rings, offsets) and the run's scalar state
 * (sweeps done, ring positions, best-so-far triplet) to a file at `path`; lcsb_load restores it
 * into a handle created with the same config (same sigma, d, l, dtype, form, layout), after
 * which sweeps continue bit-identically to an uninterrupted run.  Synchronous.  Unsharded
 * handles only.  Errors: EINVAL (path, config mismatch, corrupt or truncated file), ECUDA. */
int lcsb_save(lcsb_t* h, const char* path);
int lcsb_load(lcsb_t* h, const char* path);

int64_t lcsb_sweeps_done(const lcsb_t* h);
int32_t lcsb_num_shards(const lcsb_t* h);   /* P (1 when unsharded) */
uint64_t lcsb_num_states(const lcsb_t* h);   /* logical states sigma^(d l) */
uint64_t lcsb_stored_states(const lcsb_t* h);/* entries per stored table */
uint64_t lcsb_device_bytes(const lcsb_t* h); /* device bytes owned */
int32_t lcsb_kernel_in_use(const lcsb_t* h);
/* Sharded quarter table: the bytes one sweep of this handle's shards moves over
 * NVLink -- windows read from another shard's memory, outputs stored into another shard's --
 * and all the bytes it requests (windows + stored outputs), counted at creation from the item
 * geometry.  Errors: EINVAL (another layout). */
int lcsb_shard_traffic(const lcsb_t* h, uint64_t* peer_read_bytes, uint64_t* peer_written_bytes,
                       uint64_t* requested_bytes); /* 1 generic, 2 binary half-table paired,
                                                3 sigma=4 d=2 KS swap-paired,
                                                4 register-resident small (sigma, d),
                                                5 binary quarter-table paired */

/* Launches of the library's own kernels enqueued by this handle so far (for bench accounting). */
int64_t lcsb_launch_count(const lcsb_t* h);

/* Message of the last failure on this handle (h != NULL) or of the last failed create on
 * this thread (h == NULL).  Never NULL. */
const char* lcsb_last_error(const lcsb_t* h);

/* Free every device buffer (through free_ when hooks were given).  Safe on NULL. */
void lcsb_destroy(lcsb_t* h);

#ifdef __cplusplus
}
#endif
#endif /* LCSB_H */
