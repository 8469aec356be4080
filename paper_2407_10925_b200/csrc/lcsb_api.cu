// lcsb_api.cu -- the C-ABI of include/lcsb.h: handle, table ring, kernel dispatch, bound
// bookkeeping.  Host code only enqueues work; the whole sweep / bound path runs in the kernels
// of kern_*.cu.  No CPU fallback exists: every entry point fails with LCSB_ECUDA when the
// device work cannot be enqueued.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>

#include "lcsb_internal.cuh"

namespace lcsbk {
int bin2_tile_m(int ell);
}

using namespace lcsbk;

struct lcsb {
  lcsb_config cfg;
  int device;
  int sms;
  int form;       // resolved LCSB_FORM_KS / LCSB_FORM_TWO_ARRAY
  int symmetric;  // complement-folded half table
  int kernel;     // 1 generic, 2 bin2
  int bin2_variant;  // 0 register kernel, 5 register kernel 8 CTAs/SM, 1..4 TMA pipelines
  uint64_t n_logical;
  uint64_t n_stored;
  size_t esize;
  int ntab;                 // tables in the ring
  void* tab[kMaxGen];
  size_t tab_bytes;
  int cur;                  // ring slot of the newest table
  unsigned long long* red;  // device reduction slots
  unsigned long long* red_host;  // pinned
  int64_t sweeps_done;
  int64_t launches;
  double best_rho[2];
  int64_t best_sweep[2];
  char err[512];
};

static thread_local char g_err[512] = "";

static int set_err(lcsb_t* h, int code, const char* fmt, ...) {
  char* buf = h ? h->err : g_err;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, 512, fmt, ap);
  va_end(ap);
  if (!h) return code;
  snprintf(g_err, sizeof g_err, "%s", h->err);
  return code;
}

#define CU(h, call)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return set_err((h), LCSB_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
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
}

struct Plan {
  int form, symmetric, kernel, ntab;
  uint64_t n_logical, n_stored;
  size_t esize;
  uint64_t bytes;
};

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
  if (form == LCSB_FORM_TWO_ARRAY && !binary) {
    snprintf(why, whylen, "the two-array form is defined for sigma = d = 2 only (PAPER.md:400)");
    return LCSB_EINVAL;
  }
  if (c->kernel != LCSB_KERNEL_AUTO && c->kernel != LCSB_KERNEL_GENERIC) {
    snprintf(why, whylen, "unknown kernel %d", c->kernel);
    return LCSB_EINVAL;
  }
  const bool sym_ok = (form == LCSB_FORM_TWO_ARRAY) && c->ell >= 2 && c->kernel == LCSB_KERNEL_AUTO;
  int sym = c->symmetry;
  if (sym < 0) sym = sym_ok ? 1 : 0;
  if (sym == 1 && !sym_ok) {
    snprintf(why, whylen,
             "the complement-folded table needs the two-array binary form, ell >= 2 and the "
             "AUTO kernel");
    return LCSB_EINVAL;
  }
  if (sym != 0 && sym != 1) {
    snprintf(why, whylen, "symmetry must be -1, 0 or 1");
    return LCSB_EINVAL;
  }
  p->form = form;
  p->symmetric = sym;
  p->kernel = sym ? 2 : 1;
  if (!sym && c->sigma == 4 && c->d == 2 && form == LCSB_FORM_KS && c->ell >= 3 &&
      c->kernel == LCSB_KERNEL_AUTO)
    p->kernel = 3;  // sigma = 4, d = 2 swap-paired TMA kernel (kern_q4.cu)
  p->ntab = (form == LCSB_FORM_KS) ? c->d + 1 : 2;  // Alg. 2: d+1 rows; two-array: 2
  p->n_logical = n;
  p->n_stored = sym ? n / 2 : n;
  p->esize = (c->dtype == LCSB_F32) ? 4 : 8;
  uint64_t tb;
  if (!mul_ok(p->n_stored, p->esize, &tb) || !mul_ok(tb, (uint64_t)p->ntab, &p->bytes)) {
    snprintf(why, whylen, "table size overflows");
    return LCSB_EINVAL;
  }
  p->bytes += 256;
  return LCSB_OK;
}

extern "C" uint64_t lcsb_required_bytes(const lcsb_config* c) {
  Plan p;
  char why[256];
  if (plan_config(c, &p, why, sizeof why) != LCSB_OK) return 0;
  return p.bytes;
}

static void* dev_alloc(lcsb_t* h, size_t bytes) {
  if (h->cfg.alloc) return h->cfg.alloc(bytes, h->cfg.stream, h->cfg.alloc_ctx);
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, (cudaStream_t)h->cfg.stream) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

static void dev_free(lcsb_t* h, void* p, size_t bytes) {
  if (!p) return;
  if (h->cfg.free_)
    h->cfg.free_(p, bytes, h->cfg.stream, h->cfg.alloc_ctx);
  else
    cudaFreeAsync(p, (cudaStream_t)h->cfg.stream);
}

extern "C" void lcsb_destroy(lcsb_t* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize((cudaStream_t)h->cfg.stream);
  for (int i = 0; i < h->ntab; ++i) dev_free(h, h->tab[i], h->tab_bytes);
  dev_free(h, h->red, 256);
  if (h->red_host) cudaFreeHost(h->red_host);
  if (!h->cfg.free_) cudaStreamSynchronize((cudaStream_t)h->cfg.stream);
  delete h;
}

extern "C" int lcsb_create_ex(const lcsb_config* cfg, lcsb_t** out) {
  if (!out) return set_err(nullptr, LCSB_EINVAL, "out is NULL");
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
                   (unsigned long long)p.bytes, p.ntab, (unsigned long long)p.n_stored,
                   (unsigned long long)free_b);

  lcsb_t* h = new (std::nothrow) lcsb();
  if (!h) return set_err(nullptr, LCSB_ECAPACITY, "host allocation failed");
  memset(h, 0, sizeof *h);
  h->cfg = *cfg;
  h->device = dev;
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev);
  h->form = p.form;
  h->symmetric = p.symmetric;
  h->kernel = p.kernel;
  h->n_logical = p.n_logical;
  h->n_stored = p.n_stored;
  h->esize = p.esize;
  h->ntab = p.ntab;
  h->tab_bytes = (size_t)(p.n_stored * p.esize);
  cudaStream_t s = (cudaStream_t)cfg->stream;

  for (int i = 0; i < h->ntab; ++i) {
    h->tab[i] = dev_alloc(h, h->tab_bytes);
    if (!h->tab[i]) {
      int code = set_err(nullptr, LCSB_ECAPACITY,
                         "device allocation of table %d (%llu bytes) failed; %llu bytes needed",
                         i, (unsigned long long)h->tab_bytes, (unsigned long long)p.bytes);
      lcsb_destroy(h);
      return code;
    }
  }
  h->red = (unsigned long long*)dev_alloc(h, 256);
  if (!h->red || cudaMallocHost(&h->red_host, 256) != cudaSuccess) {
    lcsb_destroy(h);
    return set_err(nullptr, LCSB_ECAPACITY, "scratch allocation failed");
  }
  // W_0 = 0: every live generation starts at zero
  for (int i = 0; i < h->ntab; ++i) {
    e = cudaMemsetAsync(h->tab[i], 0, h->tab_bytes, s);
    if (e != cudaSuccess) {
      lcsb_destroy(h);
      return set_err(nullptr, LCSB_ECUDA, "cudaMemsetAsync failed: %s", cudaGetErrorString(e));
    }
  }
  h->cur = 0;
  h->bin2_variant = 0;  // auto: the measured-best TMA variant that fits ell (pick_bin2_variant)
  if (const char* v = getenv("LCSB_BIN2_VARIANT")) h->bin2_variant = atoi(v);
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
  CU(h, cudaSetDevice(h->device));
  for (int i = 0; i < h->ntab; ++i)
    CU(h, cudaMemsetAsync(h->tab[i], 0, h->tab_bytes, (cudaStream_t)h->cfg.stream));
  h->cur = 0;
  h->sweeps_done = 0;
  h->best_rho[0] = h->best_rho[1] = 0.0;
  h->best_sweep[0] = h->best_sweep[1] = 0;
  return LCSB_OK;
}

// Auto choice of the bin2 sweep variant, from the A/B measurements on B200:
// fp32 -> (M=6, 2 stages, direct stores) 97% of the measured copy bandwidth at l=17;
// fp64 -> (M=5, 1 stage, smem-staged bulk stores) 97% at l=16; smaller tiles for small l,
// and the register kernel below l=4.
static int pick_bin2_variant(int dtype, int ell) {
  static const int f32_chain[] = {13, 6, 8};
  static const int f64_chain[] = {8, 3, 4};
  const int* chain = (dtype == LCSB_F32) ? f32_chain : f64_chain;
  for (int i = 0; i < 3; ++i)
    if (ell >= bin2_tma_min_ell(dtype, chain[i])) return chain[i];
  return 5;  // register kernel
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
}

extern "C" int lcsb_sweep(lcsb_t* h, int64_t n) {
  if (!h) return set_err(nullptr, LCSB_EINVAL, "handle is NULL");
  if (n < 0) return set_err(h, LCSB_EINVAL, "n must be >= 0");
  CU(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  for (int64_t it = 0; it < n; ++it) {
    const int out = (h->cur + 1) % h->ntab;  // the slot of the oldest table
    cudaError_t e;
    if (h->kernel == 2) {
      Bin2Args a;
      memset(&a, 0, sizeof a);
      a.src = h->tab[h->cur];
      a.dst = h->tab[out];
      a.ell = h->cfg.ell;
      a.m = bin2_tile_m(h->cfg.ell);
      const int v = h->bin2_variant ? h->bin2_variant : pick_bin2_variant(h->cfg.dtype, h->cfg.ell);
      const int min_ell = bin2_tma_min_ell(h->cfg.dtype, v);
      if (min_ell > 0 && h->cfg.ell >= min_ell) {
        e = launch_bin2_tma_sweep(a, h->cfg.dtype, v, s, h->sms);
      } else {
        a.grid_mult = (v == 5) ? 8 : 0;
        e = launch_bin2_sweep(a, h->cfg.dtype, s, h->sms);
      }
    } else if (h->kernel == 3) {
      Q4Args a;
      memset(&a, 0, sizeof a);
      a.g1 = h->tab[slot_back(h, 0)];
      a.g2 = h->tab[slot_back(h, 1)];
      a.dst = h->tab[out];
      a.ell = h->cfg.ell;
      e = launch_q4_sweep(a, h->cfg.dtype, s, h->sms);
    } else {
      GenericArgs a;
      fill_generic(h, &a);
      for (int k = 1; k <= h->cfg.d; ++k)
        a.src[k - 1] = (h->form == LCSB_FORM_KS) ? h->tab[slot_back(h, k - 1)] : h->tab[h->cur];
      a.dst = h->tab[out];
      e = launch_generic_sweep(a, h->cfg.dtype, s, h->sms);
    }
    if (e != cudaSuccess)
      return set_err(h, LCSB_ECUDA, "sweep launch failed: %s", cudaGetErrorString(e));
    h->launches += 1;
    h->cur = out;
    h->sweeps_done += 1;
  }
  return LCSB_OK;
}

static double bound_from(const lcsb_t* h, double rho) {
  if (h->form == LCSB_FORM_KS) return (double)h->cfg.d * rho;  // Eq. (lwrbound)
  return rho > 0.0 ? 2.0 * rho / (1.0 + rho) : 0.0;           // reading R10
}

extern "C" int lcsb_bound(lcsb_t* h, lcsb_bound_t* out) {
  if (!h || !out) return set_err(h, LCSB_EINVAL, "NULL argument");
  if (h->sweeps_done < 1) return set_err(h, LCSB_ESTATE, "lcsb_bound needs at least one sweep");
  CU(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  const void* newest = h->tab[h->cur];
  const void* prev = h->tab[slot_back(h, 1)];
  CU(h, launch_red_init(h->red, s));
  CU(h, launch_rdiff(newest, prev, h->n_stored, h->cfg.dtype, h->red, s, h->sms));
  if (h->kernel == 2) {
    Bin2Args a;
    memset(&a, 0, sizeof a);
    a.src = newest;
    a.ell = h->cfg.ell;
    a.m = bin2_tile_m(h->cfg.ell);
    a.red_in = h->red;
    a.red_out = h->red + 2;
    CU(h, launch_bin2_wpass(a, h->cfg.dtype, s, h->sms));
  } else if (h->kernel == 3) {
    Q4Args a;
    memset(&a, 0, sizeof a);
    a.g1 = newest;
    a.g2 = newest;
    a.ell = h->cfg.ell;
    a.red_in = h->red;
    a.red_out = h->red + 2;
    CU(h, launch_q4_wpass(a, h->cfg.dtype, s, h->sms));
  } else {
    GenericArgs a;
    fill_generic(h, &a);
    for (int k = 1; k <= h->cfg.d; ++k) a.src[k - 1] = newest;
    a.center = newest;
    a.red_in = h->red;
    a.red_out = h->red + 2;
    CU(h, launch_generic_wpass(a, h->cfg.dtype, s, h->sms));
  }
  h->launches += 3;
  CU(h, cudaMemcpyAsync(h->red_host, h->red, kRedSlots * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, s));
  CU(h, cudaStreamSynchronize(s));
  const double R[2] = {ord_dec(h->red_host[0]), ord_dec(h->red_host[1])};
  const double Wm[2] = {ord_dec(h->red_host[2]), ord_dec(h->red_host[3])};
  double E[2], B[2];
  for (int i = 0; i < 2; ++i) {
    E[i] = Wm[i] > 0.0 ? Wm[i] : 0.0;  // E = max(0, max W)
    B[i] = bound_from(h, R[i] - E[i]);
    if (R[i] - E[i] >= h->best_rho[i]) {  // Alg. 2 line 8
      h->best_rho[i] = R[i] - E[i];
      h->best_sweep[i] = h->sweeps_done;
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
  out->sweeps_done = h->sweeps_done;
  out->best_sweep = h->best_sweep[m];
  return LCSB_OK;
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
  CU(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)h->cfg.stream;
  const void* tab = h->tab[slot_back(h, which)];
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
      e = launch_expand(tab, h->cfg.dtype, h->symmetric, h->cfg.ell, first + off, c,
                        host_idx ? ibuf : nullptr, dbuf, s);
    if (e == cudaSuccess) {
      h->launches += 1;
      e = cudaMemcpyAsync(host_dst + off, dbuf, c * sizeof(double), cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = set_err(h, LCSB_ECUDA, "table read-out failed: %s", cudaGetErrorString(e));
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

extern "C" int64_t lcsb_sweeps_done(const lcsb_t* h) { return h ? h->sweeps_done : -1; }
extern "C" uint64_t lcsb_num_states(const lcsb_t* h) { return h ? h->n_logical : 0; }
extern "C" uint64_t lcsb_stored_states(const lcsb_t* h) { return h ? h->n_stored : 0; }
extern "C" uint64_t lcsb_device_bytes(const lcsb_t* h) {
  return h ? (uint64_t)h->tab_bytes * (uint64_t)h->ntab + 256 : 0;
}
extern "C" int32_t lcsb_kernel_in_use(const lcsb_t* h) { return h ? h->kernel : 0; }
extern "C" int64_t lcsb_launch_count(const lcsb_t* h) { return h ? h->launches : 0; }
extern "C" const char* lcsb_last_error(const lcsb_t* h) { return h ? h->err : g_err; }
