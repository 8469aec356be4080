// quarter_host.cu -- host side of the symmetry-folded ("quarter") binary table (kern_bin2q.cu,
// DESIGN.md §6): stored sizes, the block map, and the L2 item schedule of the sweep.
#include <stdlib.h>

#include <stdio.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "lcsb_internal.cuh"

namespace lcsbk {

// blocks of the half table: 2^(2(l-K)-1), m = l-K-1 non-head prefix digits each.  Stored
// (canonical) blocks, by Burnside: Q1 under {id, psi}: (4^m + 2^m) / 2 (psi fixes prefixes with
// every digit in {01, 10}); Q0 under {id, s, t, s t}: (4^m + 2^m + 0 + 2^m) / 4 (s fixes digits
// in {00, 11}, s t those in {01, 10}, t none).
uint64_t quarter_map_entries(int ell, int K) { return 1ull << (2 * (ell - K) - 1); }
uint64_t quarter_slots(int ell, int K) {
  const int m = ell - K - 1;
  if (m == 0) return 2;  // the two head blocks
  return ((1ull << (2 * m)) + (1ull << m)) / 2 + ((1ull << (2 * m)) + (2ull << m)) / 4;
}
// map[beta] = (slot << 2) | mode; slots numbered in increasing order of canonical beta (the
// smallest prefix of its orbit); mode = the symmetry mapping the canonical block to beta
bool build_quarter_map(int ell, int K, uint32_t* map) {
  const int PL = 2 * (ell - K);
  const uint64_t nb = quarter_map_entries(ell, K);
  uint64_t next = 0;
  std::vector<uint64_t> canon(nb);
  std::vector<int> how(nb);
  for (uint64_t b = 0; b < nb; ++b) {
    const bool q1 = (b >> (PL - 2)) & 1ull;
    uint64_t c = b;
    int g = 0;
    for (int gg = 1; gg <= 3; ++gg) {
      if (q1 && gg != 2) continue;
      const uint64_t im = qblock_image(b, PL, gg);
      if (im < c) {
        c = im;
        g = gg;  // b = g(c): every g here is an involution
      }
    }
    canon[b] = c;
    how[b] = g;
  }
  for (uint64_t b = 0; b < nb; ++b)
    if (canon[b] == b) map[b] = (uint32_t)(next++ << 2);
  for (uint64_t b = 0; b < nb; ++b)
    if (canon[b] != b) map[b] = (map[canon[b]] & ~3u) | (uint32_t)how[b];
  return next == quarter_slots(ell, K);
}

// ---- sharded quarter table.  Shard of a canonical block: the xor key of the
// first p non-head character pairs of its prefix, x_i = a_i ^ b_i -- invariant under the block
// symmetries (swap, psi, tail complement), so a block and its images agree.  Slots are renumbered
// shard-major with a fixed stride of `maxslots` per shard (the largest shard), so the slot of a
// block also names its shard (slot / maxslots) and its place in that shard's memory.
static uint32_t qblock_key(uint64_t beta, int PL, int p) {
  uint32_t k = 0;
  for (int i = 1; i <= p; ++i) {
    const uint32_t pair = (uint32_t)(beta >> (PL - 2 - 2 * i)) & 3u;
    k = (k << 1) | ((pair >> 1) ^ (pair & 1u));
  }
  return k;
}

// Shard sizes: every shard gets the same stride of slots -- the largest shard of the xor key, or
// 2 % above the mean if that is larger (the room the refinement below may use).
static uint64_t shard_stride(const std::vector<uint64_t>& cnt, uint64_t total) {
  uint64_t mx = 0;
  for (uint64_t c : cnt) mx = c > mx ? c : mx;
  const uint64_t room = total / cnt.size() + total / cnt.size() / 50 + 1;
  return mx > room ? mx : room;
}

// Owner of an item (the shard whose launch runs it) in the sharded quarter table: the kernel
// addresses every window and output run through the one virtual range, so any shard may run any
// item.  Default: the shard holding most of the item's entries (both windows, 2 T each, and its
// stored output runs), ties to the first window's shard; LCSB_QOWNER_FIRST=1 (A/B): always the
// first window's shard (round 2's first rule).  `sh` holds the shard of each part.
static bool owner_first() {
  static const bool f = getenv("LCSB_QOWNER_FIRST") != nullptr;
  return f;
}
static uint32_t item_owner(int n, const uint32_t* sh, const uint32_t* len) {
  if (owner_first()) return sh[0];
  uint64_t loc[kMaxShards] = {0};
  for (int k = 0; k < n; ++k) loc[sh[k]] += len[k];
  uint32_t best = sh[0];
  for (uint32_t s = 0; s < (uint32_t)kMaxShards; ++s)
    if (loc[s] > loc[best]) best = s;
  return best;
}
// the parts of item tau: both windows (2 T entries each) and its stored output runs, as block
// indices of the half table (`blk`) and lengths; returns the count
static int item_parts(uint64_t tau, uint64_t q1, uint64_t lmask, uint64_t amask, uint64_t bmask,
                      int M, int K, const uint32_t* map, uint64_t* blk, uint32_t* len) {
  const uint64_t T = 1ull << (2 * M);
  const int sh = 2 * K;
  const uint64_t x0 = q1 + tau * T, p0 = pairswap_hd(~x0 & lmask) & ~(T - 1);
  const bool self = ((p0 - q1) >> (2 * M)) == tau;
  auto win = [&](uint64_t x) { return (x & amask) | ((x & bmask & ~q1) << 2); };
  const uint64_t wb = win(x0), wp = win(p0), yf = wb >> 2, ypf = wp >> 2;
  int n = 0;
  blk[n] = wb >> sh, len[n++] = (uint32_t)(2 * T);
  blk[n] = wp >> sh, len[n++] = (uint32_t)(2 * T);
  const uint64_t runs[6] = {x0, p0, yf, q1 - yf - T / 2, ypf, q1 - ypf - T / 2};
  for (int r = 0; r < 6; ++r) {
    if (self && (r == 1 || r >= 4)) continue;
    if ((map[runs[r] >> sh] & 3u) != 0) continue;
    blk[n] = runs[r] >> sh, len[n++] = (uint32_t)(r < 2 ? T : T / 2);
  }
  return n;
}

// Refinement of the block -> shard assignment (round 2): the key places each block by its own
// prefix, but an item's two windows and its output runs sit in blocks whose prefixes are
// shifted against each other, so most of them land on other shards.  Any assignment is correct
// (a slot is a global address), so a local search moves each block to the shard that minimises
// the NVLink entries of the items touching it -- the psi window read when not on the item's
// owner (the shard of its first window) and every output run stored elsewhere -- within the
// stride.  The de Bruijn dependency graph has small-cut partitions: at l = 18 this cuts the
// cross-shard bytes 2.7x at 8 shards and to a third at 2.  Sequential and
// deterministic: every rank derives the same assignment.
static void refine_shards(int ell, int K, int M, const uint32_t* map, uint32_t P, uint64_t stride,
                          int passes, std::vector<uint32_t>& shard_of_slot) {
  const int L = 2 * ell;
  const uint64_t lmask = (1ull << L) - 1, q1 = 1ull << (L - 2);
  const uint64_t amask = 0xAAAAAAAAAAAAAAAAull & lmask, bmask = 0x5555555555555555ull & lmask;
  const uint64_t T = 1ull << (2 * M);
  const int sh = 2 * K;
  const uint64_t ns = shard_of_slot.size();
  auto win = [&](uint64_t x) { return (x & amask) | ((x & bmask & ~q1) << 2); };
  // items: [w1, w2, nr, (run slot, run length)...] flattened
  std::vector<uint32_t> it;
  std::vector<uint64_t> ioff;
  const uint64_t ntiles = 1ull << (2 * (ell - 1 - M));
  for (uint64_t tau = 0; tau < ntiles; ++tau) {
    const uint64_t x0 = q1 + tau * T, p0 = pairswap_hd(~x0 & lmask) & ~(T - 1);
    const uint64_t taup = (p0 - q1) >> (2 * M);
    if (taup < tau) continue;
    const bool self = taup == tau;
    const uint64_t wb = win(x0), wp = win(p0), yf = wb >> 2, ypf = wp >> 2;
    ioff.push_back(it.size());
    it.push_back(map[wb >> sh] >> 2);
    it.push_back(map[wp >> sh] >> 2);
    const size_t nrpos = it.size();
    it.push_back(0);
    const uint64_t runs[6] = {x0, p0, yf, q1 - yf - T / 2, ypf, q1 - ypf - T / 2};
    for (int r = 0; r < 6; ++r) {
      if (self && (r == 1 || r >= 4)) continue;
      if ((map[runs[r] >> sh] & 3u) != 0) continue;
      it.push_back(map[runs[r] >> sh] >> 2);
      it.push_back(r < 2 ? (uint32_t)T : (uint32_t)(T / 2));
      ++it[nrpos];
    }
  }
  const uint64_t E = ioff.size();
  ioff.push_back(it.size());
  // slot -> items (CSR, each item once per slot)
  std::vector<uint64_t> aoff(ns + 1, 0);
  std::vector<uint32_t> last(ns, ~0u);
  auto each_slot = [&](uint64_t e, auto&& fn) {
    const uint32_t* r = it.data() + ioff[e];
    fn(r[0]);
    fn(r[1]);
    for (uint32_t k = 0; k < r[2]; ++k) fn(r[3 + 2 * k]);
  };
  for (uint64_t e = 0; e < E; ++e)
    each_slot(e, [&](uint32_t s) {
      if (last[s] != (uint32_t)e) {
        last[s] = (uint32_t)e;
        ++aoff[s + 1];
      }
    });
  for (uint64_t s = 0; s < ns; ++s) aoff[s + 1] += aoff[s];
  std::vector<uint32_t> adj(aoff[ns]);
  std::vector<uint64_t> fillp(aoff.begin(), aoff.end() - 1);
  std::fill(last.begin(), last.end(), ~0u);
  for (uint64_t e = 0; e < E; ++e)
    each_slot(e, [&](uint32_t s) {
      if (last[s] != (uint32_t)e) {
        last[s] = (uint32_t)e;
        adj[fillp[s]++] = (uint32_t)e;
      }
    });
  // NVLink entries of item e: every part not on the item's owner (item_owner's rule)
  auto cost = [&](uint64_t e) -> uint64_t {
    const uint32_t* r = it.data() + ioff[e];
    uint32_t shv[8], lenv[8];
    int n = 0;
    shv[n] = shard_of_slot[r[0]], lenv[n++] = (uint32_t)(2 * T);
    shv[n] = shard_of_slot[r[1]], lenv[n++] = (uint32_t)(2 * T);
    for (uint32_t k = 0; k < r[2]; ++k) shv[n] = shard_of_slot[r[3 + 2 * k]], lenv[n++] = r[4 + 2 * k];
    const uint32_t o = item_owner(n, shv, lenv);
    uint64_t c = 0;
    for (int k = 0; k < n; ++k) c += shv[k] != o ? lenv[k] : 0;
    return c;
  };
  std::vector<uint64_t> size(P, 0);
  for (uint32_t k : shard_of_slot) ++size[k];
  for (int pass = 0; pass < passes; ++pass) {
    uint64_t moves = 0;
    for (uint64_t b = 0; b < ns; ++b) {
      const uint32_t from = shard_of_slot[b];
      uint64_t before = 0;
      for (uint64_t a = aoff[b]; a < aoff[b + 1]; ++a) before += cost(adj[a]);
      uint32_t best = from;
      uint64_t best_c = before;
      for (uint32_t to = 0; to < P; ++to) {
        if (to == from || size[to] >= stride) continue;
        shard_of_slot[b] = to;
        uint64_t after = 0;
        for (uint64_t a = aoff[b]; a < aoff[b + 1] && after < best_c; ++a) after += cost(adj[a]);
        if (after < best_c) {
          best_c = after;
          best = to;
        }
      }
      shard_of_slot[b] = best;
      if (best != from) {
        --size[from];
        ++size[best];
        ++moves;
      }
    }
    if (!moves) break;
  }
}

static bool build_quarter_map_sharded_nocache(int ell, int K, int M, int p, int passes,
                                              uint32_t* map, uint64_t* stride_slots);

bool build_quarter_map_sharded(int ell, int K, int M, int p, int passes, uint32_t* map,
                               uint64_t* stride_slots) {
  // the last map of this process is kept: repeated creates of one config skip the search
  static std::mutex cmu;
  static int ck[5] = {0, 0, 0, -1, -1};
  static std::vector<uint32_t> cmap;
  static uint64_t cstride = 0;
  const uint64_t nb0 = quarter_map_entries(ell, K);
  {
    std::lock_guard<std::mutex> lock(cmu);
    if (ck[0] == ell && ck[1] == K && ck[2] == M && ck[3] == p && ck[4] == passes &&
        cmap.size() == nb0) {
      std::copy(cmap.begin(), cmap.end(), map);
      *stride_slots = cstride;
      return true;
    }
  }
  bool ok = build_quarter_map_sharded_nocache(ell, K, M, p, passes, map, stride_slots);
  if (ok) {
    std::lock_guard<std::mutex> lock(cmu);
    cmap.assign(map, map + nb0);
    cstride = *stride_slots;
    ck[0] = ell, ck[1] = K, ck[2] = M, ck[3] = p, ck[4] = passes;
  }
  return ok;
}

static bool build_quarter_map_sharded_nocache(int ell, int K, int M, int p, int passes,
                                              uint32_t* map, uint64_t* stride_slots) {
  if (!build_quarter_map(ell, K, map)) return false;
  const int PL = 2 * (ell - K);
  if (p < 0 || ell - K - 1 < p) return false;
  const uint64_t nb = quarter_map_entries(ell, K), ns = quarter_slots(ell, K);
  const uint32_t P = 1u << p;
  std::vector<uint32_t> shard(ns);
  std::vector<uint64_t> cnt(P, 0);
  for (uint64_t b = 0; b < nb; ++b)  // canonical blocks: the xor key of their prefix
    if ((map[b] & 3u) == 0) {
      shard[map[b] >> 2] = qblock_key(b, PL, p);
      ++cnt[shard[map[b] >> 2]];
    }
  const uint64_t stride = shard_stride(cnt, ns);
  if (stride * P >= (1ull << 30)) return false;  // map entries hold slot << 2 in 32 bits
  if (P > 1 && passes > 0) {
    // hierarchical: refine 2 shards (the key's first bit), split each by the next bit and refine
    // again, ... -- at 8 shards 20 % fewer NVLink bytes (27 % on the busiest GPU) than refining
    // the 3-bit key at once
    const std::vector<uint32_t> key(shard);
    for (int q = 1; q <= p; ++q) {
      const uint32_t Pq = 1u << q;
      for (uint64_t s = 0; s < ns; ++s)
        shard[s] = (q == 1 ? 0u : 2 * shard[s]) + ((key[s] >> (p - q)) & 1u);
      std::vector<uint64_t> cq(Pq, 0);
      for (uint64_t s = 0; s < ns; ++s) ++cq[shard[s]];
      refine_shards(ell, K, M, map, Pq, q == p ? stride : shard_stride(cq, ns), passes, shard);
    }
  }
  std::vector<uint32_t> newslot(ns);
  std::fill(cnt.begin(), cnt.end(), 0);
  for (uint64_t s = 0; s < ns; ++s) newslot[s] = (uint32_t)(shard[s] * stride + cnt[shard[s]]++);
  for (uint64_t b = 0; b < nb; ++b) map[b] = (newslot[map[b] >> 2] << 2) | (map[b] & 3u);
  *stride_slots = stride;
  return true;
}

uint64_t quarter_shard_maxslots(int ell, int K, int p) {
  // the stride depends on the key's counts only (the refinement stays within it)
  std::vector<uint32_t> map(quarter_map_entries(ell, K));
  if (!build_quarter_map(ell, K, map.data()) || p < 0 || ell - K - 1 < p) return 0;
  const int PL = 2 * (ell - K);
  std::vector<uint64_t> cnt(1u << p, 0);
  for (uint64_t b = 0; b < map.size(); ++b)
    if ((map[b] & 3u) == 0) ++cnt[qblock_key(b, PL, p)];
  const uint64_t stride = shard_stride(cnt, quarter_slots(ell, K));
  return stride * (1u << p) >= (1ull << 30) ? 0 : stride;
}

// The items (tile pairs) of one shard -- those whose first window (tile t's adv_b window) lies in
// the shard -- in the order of `sched` (entries with hint bits) or, if empty, in tile order.
void quarter_shard_items(int ell, int K, int M, const uint32_t* map, uint64_t maxslots,
                         int shard, const std::vector<uint32_t>& sched, std::vector<uint32_t>& out) {
  const int L = 2 * ell;
  const uint64_t lmask = (1ull << L) - 1, q1 = 1ull << (L - 2);
  const uint64_t amask = 0xAAAAAAAAAAAAAAAAull & lmask, bmask = 0x5555555555555555ull & lmask;
  const uint64_t T = 1ull << (2 * M);
  auto owner = [&](uint64_t tau) {
    uint64_t blk[8];
    uint32_t len[8], shv[8];
    const int n = item_parts(tau, q1, lmask, amask, bmask, M, K, map, blk, len);
    for (int k = 0; k < n; ++k) shv[k] = (uint32_t)((map[blk[k]] >> 2) / maxslots);
    return (int)item_owner(n, shv, len);
  };
  out.clear();
  if (!sched.empty()) {
    for (uint32_t e : sched)
      if (owner(e & kQTileMask) == shard) out.push_back(e);
    return;
  }
  const uint64_t ntiles = 1ull << (2 * (ell - 1 - M));
  for (uint64_t tau = 0; tau < ntiles; ++tau) {
    const uint64_t x0 = q1 + tau * T;
    const uint64_t p0 = pairswap_hd(~x0 & lmask) & ~(T - 1);
    if (((p0 - q1) >> (2 * M)) < tau) continue;  // the pair is an item at its smaller tile
    if (owner(tau) == shard) out.push_back((uint32_t)tau | (0xFu << kQHintShift));
  }
}

// Entries one shard's sweep moves over NVLink (sharded quarter table): for each of its items,
// the psi window when another shard stores it (read) and every stored output run another shard
// owns (written) -- the same geometry as the kernel's qissue / qrun.  out[0] = entries read,
// out[1] = entries written remotely, out[2] = entries read + written in total (local + remote).
void quarter_shard_traffic(int ell, int K, int M, const uint32_t* map, uint64_t maxslots,
                           int shard, const std::vector<uint32_t>& items, uint64_t out[3]) {
  const int L = 2 * ell;
  const uint64_t lmask = (1ull << L) - 1, q1 = 1ull << (L - 2);
  const uint64_t amask = 0xAAAAAAAAAAAAAAAAull & lmask, bmask = 0x5555555555555555ull & lmask;
  out[0] = out[1] = out[2] = 0;
  for (uint32_t ent : items) {  // the items this shard runs: every part elsewhere crosses NVLink
    uint64_t blk[8];
    uint32_t len[8];
    const int n = item_parts(ent & kQTileMask, q1, lmask, amask, bmask, M, K, map, blk, len);
    for (int k = 0; k < n; ++k) {
      out[2] += len[k];
      if ((int)((map[blk[k]] >> 2) / maxslots) != shard) out[k < 2 ? 0 : 1] += len[k];
    }
  }
}

// Item order of the quarter sweep ("L2 schedule").  Block graph: nodes = stored
// blocks, edges = tile pairs {t, psi t} joining the stored blocks of their two adv_b windows;
// every block has four window ends (two per logical image).  A 2-colouring that cuts most edges
// (BFS colouring + local search) gives a side A whose blocks have their tile pairs mostly on
// the other side; listing each A-block's tile pairs consecutively makes them run concurrently on
// neighbouring CTAs, so the block's four windows -- its two logical images -- come from DRAM once
// and from L2 after.  The order is a permutation of the pair representatives; the arithmetic of
// every item is unchanged.  Cached per (l, K, M): it depends on nothing else.
static std::mutex g_mu;
static int c_ell = 0, c_K = 0, c_M = 0;  // (A/B: LCSB_QSCHED=1 / 2 is read once per process)
static std::vector<uint32_t> g_cache;

bool quarter_schedule_cached(int ell, int K, int M, std::vector<uint32_t>& out) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (c_ell == ell && c_K == K && c_M == M) {
    out = g_cache;
    return true;
  }
  return false;
}

bool quarter_schedule(int ell, int K, int M, const uint32_t* map,
                             std::vector<uint32_t>& out) {
  std::vector<uint32_t>& cache = g_cache;
  std::lock_guard<std::mutex> lock(g_mu);
  // entries hold the tile index in kQHintShift bits (plan_config rejects larger tile counts)
  if (2 * (ell - 1 - M) > kQHintShift) return false;
  if (c_ell == ell && c_K == K && c_M == M) {
    out = cache;
    return true;
  }
  const int L = 2 * ell;
  const uint64_t lmask = (1ull << L) - 1, q1 = 1ull << (L - 2);
  const uint64_t amask = 0xAAAAAAAAAAAAAAAAull & lmask, bmask = 0x5555555555555555ull & lmask;
  const uint64_t T = 1ull << (2 * M);
  const uint64_t ntiles = 1ull << (2 * (ell - 1 - M));
  const uint64_t nslots = quarter_slots(ell, K);
  auto win = [&](uint64_t x) { return (x & amask) | ((x & bmask & ~q1) << 2); };
  std::vector<uint32_t> etau, eu, ev;
  for (uint64_t tau = 0; tau < ntiles; ++tau) {
    const uint64_t x0 = q1 + tau * T;
    const uint64_t p0 = pairswap_hd(~x0 & lmask) & ~(T - 1);
    if (((p0 - q1) >> (2 * M)) < tau) continue;  // the pair is an item at its smaller tile
    etau.push_back((uint32_t)tau);
    eu.push_back(map[win(x0) >> (2 * K)] >> 2);
    ev.push_back(map[win(p0) >> (2 * K)] >> 2);
  }
  const size_t E = etau.size();
  std::vector<uint32_t> off(nslots + 1, 0);
  for (size_t e = 0; e < E; ++e) {
    off[eu[e] + 1]++;
    if (ev[e] != eu[e]) off[ev[e] + 1]++;
  }
  for (uint64_t v = 0; v < nslots; ++v) off[v + 1] += off[v];
  std::vector<uint32_t> adj(off[nslots]), fill(off.begin(), off.end() - 1);
  for (size_t e = 0; e < E; ++e) {
    adj[fill[eu[e]]++] = (uint32_t)e;
    if (ev[e] != eu[e]) adj[fill[ev[e]]++] = (uint32_t)e;
  }
  auto other = [&](uint32_t e, uint32_t v) { return eu[e] == v ? ev[e] : eu[e]; };
  std::vector<int8_t> col(nslots, -1);
  std::vector<uint32_t> order;
  order.reserve(nslots);
  for (uint64_t s0 = 0; s0 < nslots; ++s0) {
    if (col[s0] >= 0) continue;
    col[s0] = 0;
    size_t head = order.size();
    order.push_back((uint32_t)s0);
    while (head < order.size()) {
      const uint32_t u = order[head++];
      for (uint32_t i = off[u]; i < off[u + 1]; ++i) {
        const uint32_t w = other(adj[i], u);
        if (col[w] < 0) {
          col[w] = (int8_t)(1 - col[u]);
          order.push_back(w);
        }
      }
    }
  }
  for (int pass = 0; pass < 16; ++pass) {  // local search: fewer same-coloured edges
    size_t flips = 0;
    for (uint64_t v = 0; v < nslots; ++v) {
      int same = 0, diff = 0;
      for (uint32_t i = off[v]; i < off[v + 1]; ++i) {
        const uint32_t w = other(adj[i], (uint32_t)v);
        if (w == v) continue;
        if (col[w] == col[v]) ++same; else ++diff;
      }
      if (same > diff) {
        col[v] ^= 1;
        ++flips;
      }
    }
    if (!flips) break;
  }
  std::vector<uint8_t> done(E, 0), grouped(nslots, 0);
  out.clear();
  out.reserve(E);
  auto emit_group = [&](uint32_t v) {  // an A-block's not yet listed tile pairs, consecutively
    grouped[v] = 1;
    for (uint32_t i = off[v]; i < off[v + 1]; ++i)
      if (!done[adj[i]]) {
        done[adj[i]] = 1;
        out.push_back(etau[adj[i]]);
      }
  };
  // v2 (default): walking the BFS order, a B-block emits the groups of all its A-neighbours
  // together, so its own windows (read by those groups) are consumed close in time as well
  static const int version = getenv("LCSB_QSCHED") ? atoi(getenv("LCSB_QSCHED")) : 4;
  for (uint32_t v : order) {
    if (col[v] == 0) {
      if (!grouped[v]) emit_group(v);
    } else if (version >= 2) {
      for (uint32_t i = off[v]; i < off[v + 1]; ++i) {
        const uint32_t w = other(adj[i], v);
        if (col[w] == 0 && !grouped[w]) emit_group(w);
      }
    }
  }
  for (size_t e = 0; e < E; ++e)
    if (!done[e]) out.push_back(etau[e]);
  if (out.size() != E) return false;
  if (version >= 4) {
    // v4 (default): re-cut the v2 order into waves of `kWave` items (about one wave of the
    // persistent grid: its items run concurrently, so a stored quarter-block loaded in a wave is
    // in L2 for the rest of it).  A wave grows greedily: always the item with the most of its
    // (<= 4) quarter-block pieces already loaded by the wave; a new seed comes from the v2 order.
    static const int kWave = getenv("LCSB_QWAVE") ? atoi(getenv("LCSB_QWAVE")) : 444;
    std::vector<uint32_t> idx_of_tau(ntiles, 0);
    for (size_t e = 0; e < E; ++e) idx_of_tau[etau[e]] = (uint32_t)e;
    const uint64_t kmask = (1ull << (2 * K)) - 1;
    auto window_pieces = [&](uint64_t w, uint32_t* pc) {  // the 2 stored quarter-blocks of w
      const uint32_t m = map[w >> (2 * K)];
      const uint64_t slot = m >> 2, e = w & kmask;
      uint64_t o0, o1;
      if ((m & 3u) == 0) {
        o0 = e;
        o1 = e + T;
      } else if ((m & 3u) == 3u) {
        o0 = (~e & kmask) & ~(2 * T - 1);
        o1 = o0 + T;
      } else {
        const uint64_t f = ((m & 3u) == 1u) ? (pairswap_hd(e) & kmask) : (pairswap_hd(~e & kmask) & kmask);
        o0 = (f & ~(4 * T - 1)) | (f & T);
        o1 = o0 + 2 * T;
      }
      pc[0] = (uint32_t)((slot << 2) | ((o0 / T) & 3));
      pc[1] = (uint32_t)((slot << 2) | ((o1 / T) & 3));
    };
    std::vector<uint32_t> pcs(4 * E);
    std::vector<uint8_t> npc(E);
    const uint64_t npieces = nslots * 4;
    std::vector<uint32_t> poff(npieces + 1, 0);
    for (size_t e = 0; e < E; ++e) {
      const uint64_t x0 = q1 + (uint64_t)etau[e] * T;
      const uint64_t p0 = pairswap_hd(~x0 & lmask) & ~(T - 1);
      uint32_t q[4];
      window_pieces(win(x0), q);
      window_pieces(win(p0), q + 2);
      int n = 0;
      for (int k = 0; k < 4; ++k) {
        bool dup = false;
        for (int j = 0; j < n; ++j) dup = dup || pcs[4 * e + j] == q[k];
        if (!dup) pcs[4 * e + n++] = q[k];
      }
      npc[e] = (uint8_t)n;
      for (int k = 0; k < n; ++k) poff[pcs[4 * e + k] + 1]++;
    }
    for (uint64_t q = 0; q < npieces; ++q) poff[q + 1] += poff[q];
    std::vector<uint32_t> pinv(poff[npieces]), pfill(poff.begin(), poff.end() - 1);
    for (size_t e = 0; e < E; ++e)
      for (int k = 0; k < npc[e]; ++k) pinv[pfill[pcs[4 * e + k]]++] = (uint32_t)e;
    std::vector<uint32_t> v2(out);  // seeds, in v2 order
    std::vector<uint8_t> taken(E, 0), score(E, 0);
    std::vector<uint32_t> pwave(npieces, ~0u), touched;
    std::vector<uint32_t> bucket[5];
    out.clear();
    size_t seed = 0;
    for (uint32_t wave = 0; out.size() < E; ++wave) {
      int cnt = 0;
      for (auto& b : bucket) b.clear();
      for (uint32_t j : touched) score[j] = 0;
      touched.clear();
      auto add = [&](uint32_t i) {
        taken[i] = 1;
        out.push_back(etau[i]);
        ++cnt;
        for (int k = 0; k < npc[i]; ++k) {
          const uint32_t q = pcs[4 * i + k];
          if (pwave[q] == wave) continue;
          pwave[q] = wave;
          for (uint32_t t = poff[q]; t < poff[q + 1]; ++t) {
            const uint32_t j = pinv[t];
            if (taken[j]) continue;
            if (!score[j]) touched.push_back(j);
            bucket[++score[j]].push_back(j);
          }
        }
      };
      while (cnt < kWave && out.size() < E) {
        int pick = -1;
        for (int sc = 4; sc >= 1 && pick < 0; --sc)
          while (!bucket[sc].empty()) {
            const uint32_t j = bucket[sc].back();
            bucket[sc].pop_back();
            if (!taken[j] && score[j] == sc) {
              pick = (int)j;
              break;
            }
          }
        if (pick < 0) {
          while (seed < E && taken[idx_of_tau[v2[seed]]]) ++seed;
          if (seed >= E) break;
          pick = (int)idx_of_tau[v2[seed]];
        }
        add((uint32_t)pick);
      }
    }
    if (out.size() != E) return false;
    // model cost of an order (LCSB_QSCHED_MODEL=1, offline harness only): pieces loaded per
    // wave of kWave items (carry 0), and with a sliding window of W waves (a piece loaded again
    // only if its previous use is more than W kWave positions back).  At l = 17 the v4 order
    // costs 20.50 GB per sweep by waves (measured: 20.66 GB), 20.43 / 20.36 / 19.99 / 18.60 GB
    // with windows of 1 / 8 / 32 / 128 waves: nearly all reuse is inside a wave.  Measured in
    // the model and dropped (round 2): a local search moving items between waves (20.54 GB) and
    // a greedy over a sliding window of 0.5-2 waves instead of hard waves (20.42-20.37 GB).
    static const bool model = getenv("LCSB_QSCHED_MODEL") != nullptr;
    auto report = [&](const char* tag) {
      if (!model) return;
      std::vector<uint32_t> seen(npieces, ~0u), last(npieces, ~0u);
      uint64_t waves = 0, win1 = 0, win2 = 0;
      for (size_t c = 0; c < E; ++c) {
        const uint32_t e = idx_of_tau[out[c] & kQTileMask];
        const uint32_t wv = (uint32_t)(c / (size_t)kWave);
        for (int k = 0; k < npc[e]; ++k) {
          const uint32_t q = pcs[4 * e + k];
          if (seen[q] != wv) { seen[q] = wv; ++waves; }
          if (last[q] == ~0u || c - last[q] > (size_t)kWave) ++win1;
          if (last[q] == ~0u || c - last[q] > 2 * (size_t)kWave) ++win2;
          last[q] = (uint32_t)c;
        }
      }
      const double gb = (double)T * 4.0 / 1e9;  // fp32 piece bytes
      fprintf(stderr, "[qsched %s] pieces %llu: waves %.2f GB, window %.2f GB, 2 windows %.2f GB\n",
              tag, (unsigned long long)npieces, waves * gb, win1 * gb, win2 * gb);
      for (size_t W : {1, 2, 4, 8, 16, 32, 64, 128}) {
        std::vector<uint32_t> lst(npieces, ~0u);
        uint64_t n = 0;
        for (size_t c = 0; c < E; ++c) {
          const uint32_t e = idx_of_tau[out[c] & kQTileMask];
          for (int k = 0; k < npc[e]; ++k) {
            const uint32_t q = pcs[4 * e + k];
            if (lst[q] == ~0u || c - lst[q] > W * (size_t)kWave) ++n;
            lst[q] = (uint32_t)c;
          }
        }
        fprintf(stderr, "   window %zu waves: %.2f GB\n", W, n * gb);
      }
    };
    report("v4");
    // LCSB_QSPREAD=P (A/B): permute each wave by j -> (j P) mod kWave, so the items that share a
    // piece (adjacent after the greedy growth) are claimed apart in time instead of together
    static const long spread = getenv("LCSB_QSPREAD") ? atol(getenv("LCSB_QSPREAD")) : 0;
    if (spread > 1) {
      std::vector<uint32_t> w(kWave);
      for (size_t w0 = 0; w0 + (size_t)kWave <= E; w0 += (size_t)kWave) {
        for (int j = 0; j < kWave; ++j) w[(size_t)((long)j * spread % kWave)] = out[w0 + j];
        std::copy(w.begin(), w.end(), out.begin() + (long)w0);
      }
    }
  }
  // L2 eviction hints (bits kQHintShift.. of each entry; see kern_bin2q.cu qissue): for each of
  // the item's 4 window pieces, set = the piece is loaded again within the next kQHintDist items
  // of the order (keep it in L2), clear = it is not (load it evict-first, so it does not push out
  // pieces that will be reused).  Default off (every bit set): measured at l = 17 fp32, the
  // evict-first loads RAISE the DRAM reads (20.65 -> 21.9 GB) and the sweep time (5.13 -> 5.32 ms)
  // for every distance tried (800, 1500, 3000; with evict-last for the kept pieces 5.25 ms).
  // LCSB_QHINT=<distance> (A/B) turns them on.
  {
    static const long hint_dist = getenv("LCSB_QHINT") ? atol(getenv("LCSB_QHINT")) : 0;
    const uint64_t ntiles_all = 1ull << (2 * (ell - 1 - M));
    const uint64_t kmask = (1ull << (2 * K)) - 1;
    if (ntiles_all <= (1ull << kQHintShift)) {
      auto pieces = [&](uint64_t w, uint32_t* pc) {  // as window_pieces above (any version)
        const uint32_t m = map[w >> (2 * K)];
        const uint64_t slot = m >> 2, e = w & kmask;
        uint64_t o0;
        uint64_t step = T;
        if ((m & 3u) == 0) {
          o0 = e;
        } else if ((m & 3u) == 3u) {
          o0 = (~e & kmask) & ~(2 * T - 1);
        } else {
          const uint64_t f = ((m & 3u) == 1u) ? (pairswap_hd(e) & kmask) : (pairswap_hd(~e & kmask) & kmask);
          o0 = (f & ~(4 * T - 1)) | (f & T);
          step = 2 * T;
        }
        pc[0] = (uint32_t)((slot << 2) | ((o0 / T) & 3));
        pc[1] = (uint32_t)((slot << 2) | (((o0 + step) / T) & 3));
      };
      std::vector<uint32_t> next_seen(nslots * 4, ~0u);
      for (size_t c = E; c-- > 0;) {
        const uint64_t tau = out[c];
        const uint64_t x0 = q1 + tau * T;
        const uint64_t p0 = pairswap_hd(~x0 & lmask) & ~(T - 1);
        uint32_t q[4];
        pieces(win(x0), q);
        pieces(win(p0), q + 2);
        uint32_t bits = 0;
        for (int k = 0; k < 4; ++k)
          if (hint_dist <= 0 || (next_seen[q[k]] != ~0u && (long)(next_seen[q[k]] - c) <= hint_dist))
            bits |= 1u << k;
        for (int k = 0; k < 4; ++k) next_seen[q[k]] = (uint32_t)c;
        out[c] = (uint32_t)tau | (bits << kQHintShift);
      }
    }
  }
  cache = out;
  c_ell = ell;
  c_K = K;
  c_M = M;
  return true;
}

}  // namespace lcsbk
