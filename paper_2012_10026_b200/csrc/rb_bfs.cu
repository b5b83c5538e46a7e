// rb_bfs.cu -- direction-optimizing BFS for sm_100a (B200).
//
// Replaces the reference level loop BfsEngine.run (engine.py:518-604) and its
// step kernels td_plain / td_striped / bu_range / bu_steal / bu_reduced
// (_kernels.py:57-293).  The whole traversal of one root is ONE cooperative
// persistent launch: levels are separated by a grid barrier, the direction
// policy (update_traversal_policy, engine.py:215-228) is evaluated by every
// block from the same device counters, so no host round trip happens between
// levels.
//
// State (all HBM, n_dev = non-isolated prefix of the RCM graph):
//   vis[]          uint32 words: vertices of levels < L (plus isolated/padding)
//   fb[3][]        frontier bitmaps, rotated: fcur = fb[L%3], fnext = fb[(L+1)%3],
//                  fb[(L+2)%3] is zeroed during level L (it is fnext of L+1)
//   lq[2], hq[2]   queue form of the frontier: light (deg <= kHubDeg) vertices
//                  and hubs; hubs carry a running edge-chunk base so a hub is
//                  split across many warps (degree-binned top-down)
//   parent, level  int32 per vertex
// Invariant at level L: visited = vis | fcur.  Each level ORs its own
// frontier into vis, so no separate "publish" pass is needed.
//
// Top-down: warps pull work items (32 light frontier vertices, or one
// kHubChunk-edge slice of a hub); inside a light item the 32 rows are
// edge-balanced with a warp prefix sum.  A neighbour is claimed with one
// atomicOr on the next-frontier bitmap word (the visited test filters first);
// the winner writes parent/level and appends to the next queue with a
// warp-aggregated atomic.
// Bottom-up: a warp owns a 1024-vertex tile (32 words).  Unvisited vertices
// of the tile are compacted across the warp's lanes; each lane checks up to
// kLight neighbours from the scan start (reverse row order by default: RCM ids
// ascend with degree, so the end of a row holds the likely frontier hubs);
// vertices still unresolved are finished by the whole warp, 32 neighbours per
// step with ballot early exit.  The warp owns its tile's words, so visited and
// next-frontier words are written with plain stores.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>

#include "rb_common.cuh"
#include "rb_error.h"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kHubDeg = 256;      // deg > kHubDeg -> hub queue
constexpr uint32_t kHubChunk = 1024;   // edges per hub work item
constexpr int kLight = 4;              // per-lane bottom-up checks before the warp takes over
constexpr int kCountShift = 37;        // hub packing: count << 37 | chunk total
constexpr uint64_t kChunkMask = (1ull << kCountShift) - 1;
constexpr int64_t kRecCap = 4096;      // level records per launch

struct Slot {  // per-level counters, triple-buffered by level % 3
  unsigned long long n_next;
  unsigned long long deg_next;
  unsigned long long scanned;
  unsigned long long lq_count;   // light queue entries for the NEXT level
  unsigned long long hq_packed;  // hubs for the NEXT level: count << 37 | chunk total
  unsigned long long items;      // dynamic work cursor (top-down items)
  unsigned long long pad0, pad1;
};

struct Final {  // state after a launch (continuation for very deep graphs)
  long long levels_done;
  long long L;
  long long dir;
  long long need_compact;
  long long nf, mf, mu;
  long long pad;
};

struct KParams {
  const int64_t* rs;
  const int32_t* col;
  const int32_t* col_bu;
  const int32_t* deg;
  int64_t n_dev;
  int64_t n_words;  // multiple of 32
  uint32_t* vis;
  uint32_t* fb0;
  uint32_t* fb1;
  uint32_t* fb2;
  int32_t* lq0;
  int32_t* lq1;
  int32_t* hq0;
  int32_t* hq1;
  int64_t* hb0;
  int64_t* hb1;
  int32_t* parent;
  int32_t* level;
  Slot* slots;
  uint32_t* bar;
  rb_level_record* rec;
  Final* fin;
  int alpha, beta, hybrid, pad_;
  int64_t n_policy;
  // start state
  int64_t level0;
  int64_t dir0;
  int64_t need_compact0;
  int64_t max_levels;
  int64_t nf0, mf0, mu0;  // mf0 < 0: derive m_f / m_u from deg(src)
  int64_t src;
  int64_t m_directed;
};

__device__ __forceinline__ uint32_t* fb_of(const KParams& p, int64_t i) {
  int64_t r = i % 3;
  return r == 0 ? p.fb0 : (r == 1 ? p.fb1 : p.fb2);
}

__device__ __forceinline__ uint32_t nth_set_bit(uint32_t x, uint32_t k) {  // 0-based, LSB first
  uint32_t pos = 0, c;
  c = __popc(x & 0xffffu); if (k >= c) { k -= c; x >>= 16; pos += 16; }
  c = __popc(x & 0xffu);   if (k >= c) { k -= c; x >>= 8;  pos += 8; }
  c = __popc(x & 0xfu);    if (k >= c) { k -= c; x >>= 4;  pos += 4; }
  c = __popc(x & 0x3u);    if (k >= c) { k -= c; x >>= 2;  pos += 2; }
  c = x & 1u;              if (k >= c) { pos += 1; }
  return pos;
}

__device__ __forceinline__ bool test_bit(const uint32_t* words, int32_t v) {
  return (__ldcg(words + (v >> 5)) >> (v & 31)) & 1u;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// top-down

struct TdOut {
  Slot* out;
  int32_t* lq_out;
  int32_t* hq_out;
  int64_t* hb_out;
};

// Warp-collective: every lane calls, act marks lanes with an edge (v -> w).
__device__ __forceinline__ void td_visit(const KParams& p, int64_t L, bool act, int32_t v, int32_t w,
                                         const uint32_t* fcur, uint32_t* fnext, const TdOut& o,
                                         unsigned long long& my_n, unsigned long long& my_deg) {
  const uint32_t lane = rb::lane_id();
  bool claim = false;
  uint32_t dw = 0;
  if (act) {
    const int32_t wi = w >> 5;
    const uint32_t bit = 1u << (w & 31);
    const uint32_t seen = __ldcg(p.vis + wi) | __ldcg(fcur + wi);
    if (!(seen & bit)) {
      const uint32_t old = atomicOr(fnext + wi, bit);
      if (!(old & bit)) {
        claim = true;
        p.parent[w] = v;
        p.level[w] = (int32_t)(L + 1);
        dw = (uint32_t)rb::ldg_i32(p.deg + w);
      }
    }
  }
  const bool hub = claim && dw > kHubDeg;
  if (hub) {  // rare: one 64-bit atomic reserves the slot and the chunk range
    const unsigned long long inc =
        (1ull << kCountShift) | (unsigned long long)((dw + kHubChunk - 1) / kHubChunk);
    const unsigned long long old = atomicAdd(&o.out->hq_packed, inc);
    const uint64_t slot = old >> kCountShift;
    o.hq_out[slot] = w;
    o.hb_out[slot] = (int64_t)(old & kChunkMask);
  }
  const bool light = claim && !hub;
  const uint32_t lm = __ballot_sync(RB_FULL, light);
  if (lm) {
    const uint32_t leader = __ffs(lm) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(&o.out->lq_count, (unsigned long long)__popc(lm));
    base = __shfl_sync(RB_FULL, base, leader);
    if (light) o.lq_out[base + __popc(lm & ((1u << lane) - 1u))] = w;
  }
  if (claim) {
    my_n += 1;
    my_deg += dw;
  }
}

__device__ void td_level(const KParams& p, int64_t L, const uint32_t* fcur, uint32_t* fnext,
                         const int32_t* lq_in, const int32_t* hq_in, const int64_t* hb_in, uint64_t nl,
                         uint64_t nh, uint64_t nchunks, const TdOut& o, unsigned long long& my_n,
                         unsigned long long& my_deg, unsigned long long& my_scan) {
  const uint32_t lane = rb::lane_id();
  const uint64_t nb = (nl + 31) / 32;
  const uint64_t total = nb + nchunks;
  while (true) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(&o.out->items, 1ull);
    item = __shfl_sync(RB_FULL, item, 0);
    if (item >= total) break;
    if (item < nb) {
      const uint64_t idx = item * 32 + lane;
      const bool valid = idx < nl;
      int32_t v = 0;
      int64_t s = 0;
      uint32_t d = 0;
      if (valid) {
        v = __ldcg(lq_in + idx);
        s = rb::ldg_i64(p.rs + v);
        d = (uint32_t)(rb::ldg_i64(p.rs + v + 1) - s);
        atomicOr(p.vis + (v >> 5), 1u << (v & 31));
      }
      const uint32_t incl = rb::warp_incl_scan(d);
      const uint32_t tot = __shfl_sync(RB_FULL, incl, 31);
      const uint32_t excl = incl - d;
      my_scan += d;
      for (uint32_t base = 0; base < tot; base += 32) {
        const uint32_t e = base + lane;
        const bool act = e < tot;
        const uint32_t j = rb::warp_upper_bound(incl, act ? e : tot - 1);
        const int32_t vj = __shfl_sync(RB_FULL, v, j);
        const int64_t sj = rb::shfl_i64(s, j);
        const uint32_t exj = __shfl_sync(RB_FULL, excl, j);
        const int32_t w = act ? rb::ldg_i32(p.col + sj + (e - exj)) : 0;
        td_visit(p, L, act, vj, w, fcur, fnext, o, my_n, my_deg);
      }
    } else {
      const uint64_t c = item - nb;
      uint64_t lo = 0, hi = nh;  // last hub whose chunk base <= c
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldcg(hb_in + mid) <= c) lo = mid; else hi = mid;
      }
      const int32_t v = __ldcg(hq_in + lo);
      const int64_t s = rb::ldg_i64(p.rs + v);
      const int64_t e = rb::ldg_i64(p.rs + v + 1);
      const uint64_t local = c - (uint64_t)__ldcg(hb_in + lo);
      const int64_t a = s + (int64_t)(local * kHubChunk);
      const int64_t b = min(e, a + (int64_t)kHubChunk);
      if (local == 0 && lane == 0) atomicOr(p.vis + (v >> 5), 1u << (v & 31));
      if (lane == 0) my_scan += (unsigned long long)(b - a);
      for (int64_t j0 = a; j0 < b; j0 += 32) {
        const int64_t j = j0 + lane;
        const bool act = j < b;
        const int32_t w = act ? rb::ldg_i32(p.col + j) : 0;
        td_visit(p, L, act, v, w, fcur, fnext, o, my_n, my_deg);
      }
    }
  }
}

// Bitmap -> queues (light / hub split) at a bottom-up -> top-down switch.
__device__ void compact_level(const KParams& p, const uint32_t* fcur, Slot* in, int32_t* lq, int32_t* hq,
                              int64_t* hb) {
  const uint32_t lane = rb::lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  const uint64_t gw = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t ntiles = (uint64_t)p.n_words / 32;
  for (uint64_t tile = gw; tile < ntiles; tile += nwarps) {
    const uint64_t wi = tile * 32 + lane;
    const uint32_t x = __ldcg(fcur + wi);
    uint32_t hubmask = 0, cnt = 0;
    for (uint32_t y = x; y; y &= y - 1) {
      const int b = __ffs(y) - 1;
      const int32_t v = (int32_t)(wi * 32 + b);
      const uint32_t d = (uint32_t)rb::ldg_i32(p.deg + v);
      if (d > kHubDeg) {
        hubmask |= 1u << b;
        const unsigned long long inc =
            (1ull << kCountShift) | (unsigned long long)((d + kHubChunk - 1) / kHubChunk);
        const unsigned long long old = atomicAdd(&in->hq_packed, inc);
        const uint64_t slot = old >> kCountShift;
        hq[slot] = v;
        hb[slot] = (int64_t)(old & kChunkMask);
      } else {
        ++cnt;
      }
    }
    const uint32_t incl = rb::warp_incl_scan(cnt);
    const uint32_t tot = __shfl_sync(RB_FULL, incl, 31);
    if (tot == 0) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&in->lq_count, (unsigned long long)tot);
    base = __shfl_sync(RB_FULL, base, 0);
    unsigned long long pos = base + incl - cnt;
    for (uint32_t y = x & ~hubmask; y; y &= y - 1) {
      const int b = __ffs(y) - 1;
      lq[pos++] = (int32_t)(wi * 32 + b);
    }
  }
}

// ---------------------------------------------------------------------------
// bottom-up

template <bool kRev>
__device__ void bu_level(const KParams& p, int64_t L, const uint32_t* fcur, uint32_t* fnext, uint32_t* s_found,
                         unsigned long long& my_n, unsigned long long& my_deg, unsigned long long& my_scan) {
  const uint32_t lane = rb::lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  const uint64_t gw = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t ntiles = (uint64_t)p.n_words / 32;
  for (uint64_t tile = gw; tile < ntiles; tile += nwarps) {
    const uint64_t wi = tile * 32 + lane;
    const uint32_t vw = __ldcg(p.vis + wi);
    const uint32_t fw = __ldcg(fcur + wi);
    if (fw) p.vis[wi] = vw | fw;  // publish this level's frontier (warp owns the word)
    const uint32_t unv = ~(vw | fw);
    const uint32_t cnt = __popc(unv);
    const uint32_t incl = rb::warp_incl_scan(cnt);
    const uint32_t U = __shfl_sync(RB_FULL, incl, 31);
    const uint32_t excl = incl - cnt;
    s_found[lane] = 0;
    __syncwarp();
    for (uint32_t b0 = 0; b0 < U; b0 += 32) {
      const uint32_t t = b0 + lane;
      const bool act = t < U;
      const uint32_t j = rb::warp_upper_bound(incl, act ? t : U - 1);
      const uint32_t unvj = __shfl_sync(RB_FULL, unv, j);
      const uint32_t exj = __shfl_sync(RB_FULL, excl, j);
      const uint32_t bitpos = nth_set_bit(unvj, act ? t - exj : 0);
      const int64_t v = (int64_t)(tile * 32 + j) * 32 + bitpos;
      bool found = false, heavy = false;
      int64_t s = 0, e = 0;
      int32_t par = -1;
      uint32_t checks = 0;
      if (act) {
        s = rb::ldg_i64(p.rs + v);
        e = rb::ldg_i64(p.rs + v + 1);
        const int64_t d = e - s;
        int32_t u[kLight];
#pragma unroll
        for (int k = 0; k < kLight; ++k)
          u[k] = (k < d) ? rb::ldg_i32(p.col_bu + (kRev ? e - 1 - k : s + k)) : -1;
        uint32_t hit = 0;
#pragma unroll
        for (int k = 0; k < kLight; ++k)
          if (u[k] >= 0 && test_bit(fcur, u[k])) hit |= 1u << k;
        if (hit) {
          const int k = __ffs(hit) - 1;
          found = true;
          par = u[k];
          checks = k + 1;
        } else {
          checks = (uint32_t)(d < kLight ? d : kLight);
          heavy = d > kLight;
        }
      }
      uint32_t hm = __ballot_sync(RB_FULL, heavy);
      while (hm) {  // warp-cooperative finish of long rows
        const int h = __ffs(hm) - 1;
        hm &= hm - 1;
        const int64_t hs = rb::shfl_i64(s, h);
        const int64_t he = rb::shfl_i64(e, h);
        const int64_t len = he - hs - kLight;
        int32_t hpar = -1;
        int64_t hchecks = len;
        for (int64_t r = 0; r < len; r += 32) {
          const int64_t k = r + lane;
          bool hit = false;
          int32_t uu = 0;
          if (k < len) {
            uu = rb::ldg_i32(p.col_bu + (kRev ? he - kLight - 1 - k : hs + kLight + k));
            hit = test_bit(fcur, uu);
          }
          const uint32_t hb = __ballot_sync(RB_FULL, hit);
          if (hb) {
            const int f = __ffs(hb) - 1;
            hpar = __shfl_sync(RB_FULL, uu, f);
            hchecks = r + f + 1;
            break;
          }
        }
        if ((int)lane == h) {
          checks += (uint32_t)hchecks;
          if (hpar >= 0) {
            found = true;
            par = hpar;
          }
        }
      }
      if (found) {
        p.parent[v] = par;
        p.level[v] = (int32_t)(L + 1);
        atomicOr(s_found + j, 1u << bitpos);
        my_n += 1;
        my_deg += (unsigned long long)(e - s);
      }
      my_scan += checks;
    }
    __syncwarp();
    fnext[wi] = s_found[lane];  // full-word store: also clears stale bits
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------

__device__ __forceinline__ void block_add3(unsigned long long* red, unsigned long long a, unsigned long long b,
                                           unsigned long long c, Slot* out) {
  a = rb::warp_sum_u64(a);
  b = rb::warp_sum_u64(b);
  c = rb::warp_sum_u64(c);
  const uint32_t w = threadIdx.x >> 5;
  if (rb::lane_id() == 0) {
    red[w * 3 + 0] = a;
    red[w * 3 + 1] = b;
    red[w * 3 + 2] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long A = 0, B = 0, C = 0;
    for (int i = 0; i < kWarps; ++i) {
      A += red[i * 3];
      B += red[i * 3 + 1];
      C += red[i * 3 + 2];
    }
    if (A) atomicAdd(&out->n_next, A);
    if (B) atomicAdd(&out->deg_next, B);
    if (C) atomicAdd(&out->scanned, C);
  }
}

template <bool kRev>
__global__ void __launch_bounds__(kThreads) bfs_persistent(KParams p) {
  __shared__ uint32_t s_found_all[kWarps][32];
  __shared__ unsigned long long s_red[kWarps * 3];
  uint32_t* s_found = s_found_all[threadIdx.x >> 5];
  const uint32_t nblocks = gridDim.x;
  const uint64_t gtid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const uint64_t gthreads = (uint64_t)nblocks * kThreads;

  int64_t L = p.level0;
  int dir = (int)p.dir0;
  int need_compact = (int)p.need_compact0;
  int64_t nf = p.nf0, mf = p.mf0, mu = p.mu0;
  if (mf < 0) {  // engine.py:536-538
    mf = rb::ldg_i64(p.rs + p.src + 1) - rb::ldg_i64(p.rs + p.src);
    mu = p.m_directed - mf;
  }
  int64_t done = 0;
  uint64_t t_prev = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) t_prev = globaltimer();

  while (done < p.max_levels && nf > 0) {
    Slot* out = p.slots + (L % 3);
    Slot* in = p.slots + ((L + 2) % 3);
    const uint32_t* fcur = fb_of(p, L);
    uint32_t* fnext = fb_of(p, L + 1);
    uint32_t* fzero = fb_of(p, L + 2);
    // zero ahead: next level's fnext bitmap and the counter slot of level L+1
    for (uint64_t i = gtid; i < (uint64_t)p.n_words; i += gthreads) fzero[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x < sizeof(Slot) / 8)
      reinterpret_cast<unsigned long long*>(p.slots + ((L + 1) % 3))[threadIdx.x] = 0ull;

    unsigned long long my_n = 0, my_deg = 0, my_scan = 0;
    if (dir == 0) {
      int32_t* lq_in = (L & 1) ? p.lq1 : p.lq0;
      int32_t* hq_in = (L & 1) ? p.hq1 : p.hq0;
      int64_t* hb_in = (L & 1) ? p.hb1 : p.hb0;
      if (need_compact) {
        compact_level(p, fcur, in, lq_in, hq_in, hb_in);
        rb::grid_barrier(p.bar, nblocks);
      }
      const uint64_t nl = rb::ld_relaxed_u64(&in->lq_count);
      const uint64_t hp = rb::ld_relaxed_u64(&in->hq_packed);
      TdOut o;
      o.out = out;
      o.lq_out = (L & 1) ? p.lq0 : p.lq1;
      o.hq_out = (L & 1) ? p.hq0 : p.hq1;
      o.hb_out = (L & 1) ? p.hb0 : p.hb1;
      td_level(p, L, fcur, fnext, lq_in, hq_in, hb_in, nl, hp >> kCountShift, hp & kChunkMask, o, my_n,
               my_deg, my_scan);
    } else {
      bu_level<kRev>(p, L, fcur, fnext, s_found, my_n, my_deg, my_scan);
    }
    block_add3(s_red, my_n, my_deg, my_scan, out);
    rb::grid_barrier(p.bar, nblocks);

    const int64_t n_next = (int64_t)rb::ld_relaxed_u64(&out->n_next);
    const int64_t deg_next = (int64_t)rb::ld_relaxed_u64(&out->deg_next);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const uint64_t t_now = globaltimer();
      rb_level_record r;
      r.level = L;
      r.direction = dir;
      r.n_f = nf;
      r.m_f = mf;
      r.m_u = mu;
      r.scanned_edges = (int64_t)rb::ld_relaxed_u64(&out->scanned);
      r.t_ns = (int64_t)(t_now - t_prev);
      r.n_next = n_next;
      p.rec[done] = r;
      t_prev = t_now;
    }
    // engine.py:587-596
    mu -= deg_next;
    mf = deg_next;
    nf = n_next;
    int ndir = 0;
    if (p.hybrid) {
      if (dir == 0)
        ndir = ((double)mf > (double)mu / (double)p.alpha) ? 1 : 0;
      else
        ndir = ((double)nf < (double)p.n_policy / (double)p.beta) ? 0 : 1;
    }
    need_compact = (dir == 1 && ndir == 0);
    dir = ndir;
    ++L;
    ++done;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.fin->levels_done = done;
    p.fin->L = L;
    p.fin->dir = dir;
    p.fin->need_compact = need_compact;
    p.fin->nf = nf;
    p.fin->mf = mf;
    p.fin->mu = mu;
  }
}

// Per-root reset tail: source seeds (engine.py:526-539).
__global__ void bfs_seed(KParams p, int64_t src) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  p.parent[src] = (int32_t)src;
  p.level[src] = 0;
  p.fb0[src >> 5] |= 1u << (src & 31);
  const int64_t d = p.rs[src + 1] - p.rs[src];
  Slot* in = p.slots + 2;  // inputs of level 0 = outputs of "level -1"
  if (d > (int64_t)kHubDeg) {
    p.hq0[0] = (int32_t)src;
    p.hb0[0] = 0;
    in->hq_packed = (1ull << kCountShift) | (unsigned long long)((d + kHubChunk - 1) / kHubChunk);
  } else {
    p.lq0[0] = (int32_t)src;
    in->lq_count = 1;
  }
}

__global__ void words_or3(const uint32_t* a, const uint32_t* b, const uint32_t* c, uint32_t* out, int64_t n,
                          const uint32_t* mask_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (a[i] | b[i] | c[i]) & ~mask_out[i];
}

__global__ void words_or(uint32_t* dst, const uint32_t* src, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] |= src[i];
}

__global__ void make_pad_mask(uint32_t* m, int64_t n_dev, int64_t n_words) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_words; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = i * 32;
    uint32_t x;
    if (lo >= n_dev) x = RB_FULL;
    else if (lo + 32 <= n_dev) x = 0u;
    else x = RB_FULL << (uint32_t)(n_dev - lo);
    m[i] = x;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

struct rb_bfs {
  KParams kp;
  rb_bfs_params prm;
  int64_t n_dev;
  int64_t n_words;
  uint32_t* vis_template;  // isolated + padding premarked
  uint32_t* pad_mask;      // padding bits only
  int blocks;
  int sms;
  int bu_reverse;
  int64_t source;
  std::vector<rb_level_record> recs;
  bool launched;
  void* stream;
};

static int alloc_dev(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    rb_set_error("cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    return RB_ERR_OOM;
  }
  return RB_OK;
}

extern "C" int rb_bfs_create(const int64_t* d_row_starts, const int32_t* d_col, const int32_t* d_col_bu,
                             const int32_t* d_degrees, int64_t n_dev, const uint32_t* d_isolated_words,
                             const rb_bfs_params* params, rb_bfs** out) {
  if (!out || !params || n_dev <= 0 || !d_row_starts || !d_col || !d_degrees) {
    rb_set_error("rb_bfs_create: invalid argument");
    return RB_ERR_ARG;
  }
  if (n_dev >= (1ll << 31)) {
    rb_set_error("rb_bfs_create: n_dev %lld exceeds int32 vertex ids", (long long)n_dev);
    return RB_ERR_ARG;
  }
  rb_bfs* h = new rb_bfs();
  memset(&h->kp, 0, sizeof(h->kp));
  h->prm = *params;
  h->n_dev = n_dev;
  h->n_words = ((n_dev + 1023) / 1024) * 32;
  h->bu_reverse = params->bu_reverse;
  h->launched = false;
  KParams& k = h->kp;
  k.rs = d_row_starts;
  k.col = d_col;
  k.col_bu = d_col_bu ? d_col_bu : d_col;
  k.deg = d_degrees;
  k.n_dev = n_dev;
  k.n_words = h->n_words;
  const size_t wb = (size_t)h->n_words * 4;
  int rc = RB_OK;
#define RB_ALLOC(ptr, bytes)                               \
  if (rc == RB_OK) rc = alloc_dev((void**)&(ptr), (bytes));
  RB_ALLOC(k.vis, wb);
  RB_ALLOC(k.fb0, wb);
  RB_ALLOC(k.fb1, wb);
  RB_ALLOC(k.fb2, wb);
  RB_ALLOC(h->vis_template, wb);
  RB_ALLOC(h->pad_mask, wb);
  RB_ALLOC(k.lq0, (size_t)n_dev * 4);
  RB_ALLOC(k.lq1, (size_t)n_dev * 4);
  const size_t nhub = (size_t)n_dev + 2;
  RB_ALLOC(k.hq0, nhub * 4);
  RB_ALLOC(k.hq1, nhub * 4);
  RB_ALLOC(k.hb0, nhub * 8);
  RB_ALLOC(k.hb1, nhub * 8);
  RB_ALLOC(k.parent, (size_t)n_dev * 4);
  RB_ALLOC(k.level, (size_t)n_dev * 4);
  RB_ALLOC(k.slots, 3 * sizeof(Slot));
  RB_ALLOC(k.bar, 64);
  RB_ALLOC(k.rec, kRecCap * sizeof(rb_level_record));
  RB_ALLOC(k.fin, sizeof(Final));
#undef RB_ALLOC
  if (rc != RB_OK) {
    rb_bfs_destroy(h);
    return rc;
  }
  k.alpha = params->alpha;
  k.beta = params->beta;
  k.hybrid = params->hybrid;
  k.n_policy = params->n_policy;

  make_pad_mask<<<256, 256>>>(h->pad_mask, n_dev, h->n_words);
  if (cudaMemcpy(h->vis_template, h->pad_mask, wb, cudaMemcpyDeviceToDevice) != cudaSuccess) {
    rb_set_error("rb_bfs_create: template copy failed");
    rb_bfs_destroy(h);
    return RB_ERR_CUDA;
  }
  if (d_isolated_words) words_or<<<256, 256>>>(h->vis_template, d_isolated_words, (n_dev + 31) / 32);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    rb_set_error("rb_bfs_create: %s", cudaGetErrorString(e));
    rb_bfs_destroy(h);
    return RB_ERR_CUDA;
  }
  int dev = 0, nb = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev);
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) {
    rb_set_error("rb_bfs_create: device lacks cooperative launch");
    rb_bfs_destroy(h);
    return RB_ERR_CUDA;
  }
  if (h->bu_reverse)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bfs_persistent<true>, kThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bfs_persistent<false>, kThreads, 0);
  if (nb < 1) nb = 1;
  h->blocks = nb * h->sms;
  *out = h;
  return RB_OK;
}

extern "C" int rb_bfs_destroy(rb_bfs* h) {
  if (!h) return RB_OK;
  KParams& k = h->kp;
  void* ptrs[] = {k.vis, k.fb0, k.fb1, k.fb2, h->vis_template, h->pad_mask, k.lq0, k.lq1, k.hq0, k.hq1,
                  k.hb0, k.hb1, k.parent, k.level, k.slots, k.bar, k.rec, k.fin};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete h;
  return RB_OK;
}

extern "C" int32_t* rb_bfs_parent_ptr(rb_bfs* h) { return h ? h->kp.parent : nullptr; }
extern "C" int32_t* rb_bfs_level_ptr(rb_bfs* h) { return h ? h->kp.level : nullptr; }
extern "C" int rb_bfs_grid(rb_bfs* h, int* blocks, int* threads) {
  if (!h) return RB_ERR_ARG;
  if (blocks) *blocks = h->blocks;
  if (threads) *threads = kThreads;
  return RB_OK;
}

static int reset_common(rb_bfs* h, cudaStream_t s) {
  KParams& k = h->kp;
  const size_t wb = (size_t)h->n_words * 4;
  RB_CUDA_TRY(cudaMemsetAsync(k.parent, 0xff, (size_t)h->n_dev * 4, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.level, 0xff, (size_t)h->n_dev * 4, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.fb0, 0, wb, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.fb1, 0, wb, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.slots, 0, 3 * sizeof(Slot), s));
  RB_CUDA_TRY(cudaMemsetAsync(k.bar, 0, 64, s));
  return RB_OK;
}

extern "C" int rb_bfs_reset(rb_bfs* h, int64_t source, void* stream) {
  if (!h) return RB_ERR_ARG;
  if (source < 0 || source >= h->n_dev) {
    rb_set_error("source %lld out of range for n_dev=%lld", (long long)source, (long long)h->n_dev);
    return RB_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_common(h, s);
  if (rc) return rc;
  RB_CUDA_TRY(cudaMemcpyAsync(h->kp.vis, h->vis_template, (size_t)h->n_words * 4, cudaMemcpyDeviceToDevice, s));
  bfs_seed<<<1, 32, 0, s>>>(h->kp, source);
  RB_CUDA_TRY(cudaGetLastError());
  h->source = source;
  h->recs.clear();
  return RB_OK;
}

static int launch(rb_bfs* h, cudaStream_t s, int64_t level0, int64_t dir0, int64_t need_compact0, int64_t max_levels,
                  int64_t nf0, int64_t mf0, int64_t mu0) {
  KParams kp = h->kp;
  kp.level0 = level0;
  kp.dir0 = dir0;
  kp.need_compact0 = need_compact0;
  kp.max_levels = max_levels;
  kp.nf0 = nf0;
  kp.mf0 = mf0;
  kp.mu0 = mu0;
  kp.src = h->source;
  kp.m_directed = h->prm.m_directed;
  void* args[] = {&kp};
  cudaError_t e;
  if (h->bu_reverse)
    e = cudaLaunchCooperativeKernel((const void*)bfs_persistent<true>, dim3(h->blocks), dim3(kThreads), args, 0, s);
  else
    e = cudaLaunchCooperativeKernel((const void*)bfs_persistent<false>, dim3(h->blocks), dim3(kThreads), args, 0, s);
  if (e != cudaSuccess) {
    rb_set_error("cooperative launch failed: %s", cudaGetErrorString(e));
    return RB_ERR_CUDA;
  }
  return RB_OK;
}

extern "C" int rb_bfs_traverse(rb_bfs* h, void* stream) {
  if (!h) return RB_ERR_ARG;
  h->launched = true;
  h->stream = stream;
  return launch(h, (cudaStream_t)stream, 0, 0, 0, kRecCap, 1, -1, 0);
}

extern "C" int rb_bfs_results(rb_bfs* h, int32_t* parent_out, int32_t* level_out, rb_level_record* h_records,
                              int64_t cap, int64_t* n_records, void* stream) {
  if (!h) return RB_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (h->launched) {
    // drain: copy records, continue very deep traversals
    while (true) {
      Final f;
      RB_CUDA_TRY(cudaMemcpyAsync(&f, h->kp.fin, sizeof(Final), cudaMemcpyDeviceToHost, s));
      RB_CUDA_TRY(cudaStreamSynchronize(s));
      size_t old = h->recs.size();
      h->recs.resize(old + (size_t)f.levels_done);
      if (f.levels_done)
      {
        RB_CUDA_TRY(cudaMemcpyAsync(h->recs.data() + old, h->kp.rec,
                                    (size_t)f.levels_done * sizeof(rb_level_record), cudaMemcpyDeviceToHost, s));
        RB_CUDA_TRY(cudaStreamSynchronize(s));
      }
      if (f.nf <= 0) break;
      int rc = launch(h, s, f.L, f.dir, f.need_compact, kRecCap, f.nf, f.mf, f.mu);
      if (rc) return rc;
    }
    h->launched = false;
  }
  if (parent_out)
    RB_CUDA_TRY(cudaMemcpyAsync(parent_out, h->kp.parent, (size_t)h->n_dev * 4, cudaMemcpyDefault, s));
  if (level_out)
    RB_CUDA_TRY(cudaMemcpyAsync(level_out, h->kp.level, (size_t)h->n_dev * 4, cudaMemcpyDefault, s));
  int64_t nr = (int64_t)h->recs.size();
  if (h_records) {
    int64_t c = nr < cap ? nr : cap;
    memcpy(h_records, h->recs.data(), (size_t)c * sizeof(rb_level_record));
  }
  if (n_records) *n_records = nr;
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  return RB_OK;
}

extern "C" int rb_bfs_step(rb_bfs* h, int direction, const uint32_t* d_visited_words,
                           const uint32_t* d_frontier_words, const int32_t* d_parent_in, uint32_t* d_visited_out,
                           uint32_t* d_next_out, int32_t* d_parent_out, int64_t* h_counters, void* stream) {
  if (!h || (direction != 0 && direction != 1)) {
    rb_set_error("rb_bfs_step: invalid argument");
    return RB_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  KParams& k = h->kp;
  const int64_t nw_in = (h->n_dev + 31) / 32;
  int rc = reset_common(h, s);
  if (rc) return rc;
  RB_CUDA_TRY(cudaMemcpyAsync(k.vis, h->pad_mask, (size_t)h->n_words * 4, cudaMemcpyDeviceToDevice, s));
  words_or<<<256, 256, 0, s>>>(k.vis, d_visited_words, nw_in);
  RB_CUDA_TRY(cudaMemcpyAsync(k.fb0, d_frontier_words, (size_t)nw_in * 4, cudaMemcpyDeviceToDevice, s));
  RB_CUDA_TRY(cudaMemcpyAsync(k.parent, d_parent_in, (size_t)h->n_dev * 4, cudaMemcpyDeviceToDevice, s));
  rc = launch(h, s, 0, direction, direction == 0 ? 1 : 0, 1, 1, 0, 0);
  if (rc) return rc;
  words_or3<<<256, 256, 0, s>>>(k.vis, k.fb0, k.fb1, d_visited_out, nw_in, h->pad_mask);
  RB_CUDA_TRY(cudaMemcpyAsync(d_next_out, k.fb1, (size_t)nw_in * 4, cudaMemcpyDeviceToDevice, s));
  RB_CUDA_TRY(cudaMemcpyAsync(d_parent_out, k.parent, (size_t)h->n_dev * 4, cudaMemcpyDeviceToDevice, s));
  Slot sl;
  RB_CUDA_TRY(cudaMemcpyAsync(&sl, k.slots, sizeof(Slot), cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  if (h_counters) {
    h_counters[0] = (int64_t)sl.n_next;
    h_counters[1] = (int64_t)sl.deg_next;
    h_counters[2] = (int64_t)sl.scanned;
  }
  return RB_OK;
}
