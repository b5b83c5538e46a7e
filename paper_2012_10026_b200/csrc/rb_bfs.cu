// rb_bfs.cu -- direction-optimizing BFS for sm_100a (B200).
//
// Replaces the reference level loop BfsEngine.run (engine.py:518-604) and its
// step kernels td_plain / td_striped / bu_range / bu_steal / bu_reduced
// (_kernels.py:57-293).  The whole traversal of one root is ONE cooperative
// persistent launch: levels are separated by a grid barrier and the direction
// policy (update_traversal_policy, engine.py:215-228) is evaluated by every
// block from the same device counters, so no host round trip happens between
// levels.
//
// State (HBM; n_dev = non-isolated prefix of the RCM graph):
//   vis[]        uint32 words: vertices of levels < L (+ isolated, padding)
//   fb[3][]      frontier bitmaps, rotated: fcur = fb[L%3], fnext = fb[(L+1)%3];
//                fb[(L+2)%3] is zeroed during level L (it is fnext of L+1)
//   lq[2]        light frontier vertices (deg <= kLightDeg), int32
//   hq[2]        hub work items (chunk << 32 | v): one entry per kChunk-edge
//                slice of a hub row, so hubs spread over many warps
//   parent, level  int32 per vertex
// Invariant: vis holds every vertex discovered so far (the current frontier
// included), so a top-down claim is one atomicOr on vis and a bottom-up
// step tests ~vis directly.
//
// The path is latency-bound integer work, so both directions are written for
// memory-level parallelism: every lane keeps several independent loads in
// flight (unrolled edge / vertex groups), work items are sized so the whole
// grid is busy, and there is no per-item atomic work fetching.
//
// Top-down: warps take items statically (light batches of 32 rows that are
// edge-balanced with a warp prefix sum, processed 128 edges per step; or one
// 256-edge hub slice, 8 edges per lane).  A neighbour is claimed with one
// atomicOr on its visited word; the winner sets the next-frontier bit (RED),
// writes parent / level and appends to the next queue (warp-aggregated).
// Bottom-up: a warp owns kUB consecutive bitmap words (kUB*32 vertices), so
// its visited / next-frontier words are written with plain stores.  Each lane
// checks its unvisited vertices' rows from the scan start kK1 neighbours at a
// time (reverse row order by default: RCM ids ascend with degree, so the end
// of a row holds the likely frontier hubs), continuing up to kK2 checks;
// longer rows are finished by the whole warp 256 neighbours per step with a
// ballot early exit.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>

#include "rb_common.cuh"
#include "rb_error.h"

namespace {

constexpr int kThreads = 1024;
#ifndef RB_MINB
#define RB_MINB 1
#endif
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kLightDeg = 32;  // deg <= kLightDeg -> light queue
constexpr int kChunkPerLane = 8;
constexpr uint32_t kChunk = 32 * kChunkPerLane;  // edges per hub work item
constexpr int kTdUnroll = 4;                     // light batch: edges per lane per step
constexpr int kUB = 4;                           // compaction: words per warp step
constexpr int kBU = 8;                           // bottom-up: words per warp step
constexpr int kK1 = 2;                           // bottom-up: first-round checks per vertex
constexpr int kK2 = 10;                          // bottom-up: per-lane checks before the warp takes over
constexpr int kHeavyPerLane = 8;                 // warp-cooperative bottom-up: neighbours per lane per step
constexpr int64_t kRecCap = 4096;                // level records per launch

// Queue entry: a light frontier row (d <= kLightDeg) or one hub slice
// (columns [s, s+d), d <= kChunk).  Carrying the offsets saves the dependent
// row_starts load in the consuming level.
struct __align__(16) QEnt {
  long long s;
  int32_t v;
  int32_t d;
};

struct Slot {  // per-level counters, triple-buffered by level % 3
  unsigned long long n_next;
  unsigned long long deg_next;
  unsigned long long scanned;
  unsigned long long lq_count;  // light queue entries for the NEXT level
  unsigned long long hq_count;  // hub slices for the NEXT level
  unsigned long long pad0, pad1, pad2;
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
  const int2* hot;  // per vertex: the first two neighbours in bottom-up scan order (-1 = none)
  int64_t n_dev;
  int64_t n_words;  // multiple of 32 * kUB
  uint32_t* vis;
  uint32_t* fb0;
  uint32_t* fb1;
  uint32_t* fb2;
  uint32_t* nz0;   // bit i: fb0 word i is nonzero -- lets the queue build skip empty words
  uint32_t* nz1;
  uint32_t* nz2;
  QEnt* lq0;
  QEnt* lq1;
  QEnt* hq0;
  QEnt* hq1;
  int32_t* parent;
  int32_t* level;
  Slot* slots;
  uint32_t* bar;
  rb_level_record* rec;
  Final* fin;
  int alpha, beta, hybrid, debug;
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
  const int64_t r = i % 3;
  return r == 0 ? p.fb0 : (r == 1 ? p.fb1 : p.fb2);
}

__device__ __forceinline__ uint32_t* nz_of(const KParams& p, int64_t i) {
  const int64_t r = i % 3;
  return r == 0 ? p.nz0 : (r == 1 ? p.nz1 : p.nz2);
}

// Frontier / visited bits: written before the last grid barrier and not
// modified during this level (the barrier invalidates L1), so L1 may cache.
__device__ __forceinline__ uint32_t ld_bits(const uint32_t* p) { return __ldca(p); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Acc {
  unsigned long long n, deg, scan;
};

// Global warp index, interleaved across blocks: consecutive work items go to
// different SMs, so a small level is not concentrated on a few SMs' LSU/L1.
__device__ __forceinline__ uint64_t warp_slot() {
  return (uint64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
}

struct TdCtx {
  const KParams* p;
  int64_t L;
  const uint32_t* fcur;
  uint32_t* fnext;
  uint32_t* nznext;
  Slot* out;
};

__device__ __forceinline__ QEnt ld_qent(const QEnt* q) {
  const int4 x = __ldcg(reinterpret_cast<const int4*>(q));
  QEnt e;
  e.s = (long long)(((unsigned long long)(uint32_t)x.y << 32) | (uint32_t)x.x);
  e.v = x.z;
  e.d = x.w;
  return e;
}

// Warp-aggregated append of frontier rows: light rows to lq, hubs as
// kChunk-edge slices to hq.  One atomic per queue per warp (issued by two
// lanes so they overlap).  Hub slices are written by all 32 lanes in
// parallel, so a lane holding a huge row does not serialize the warp.
template <int KU>
__device__ __forceinline__ void warp_append(QEnt* lq, unsigned long long* lq_count, QEnt* hq,
                                            unsigned long long* hq_count, const int32_t (&w)[KU],
                                            const int64_t (&s)[KU], const uint32_t (&d)[KU], const bool (&on)[KU]) {
  uint32_t nl = 0, nh = 0;
  uint32_t nk[KU];
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    nk[k] = 0;
    if (!on[k]) continue;
    if (d[k] > kLightDeg) nk[k] = (d[k] + kChunk - 1) / kChunk;
    else ++nl;
    nh += nk[k];
  }
  const uint32_t il = rb::warp_incl_scan(nl);
  const uint32_t ih = rb::warp_incl_scan(nh);
  const uint32_t tl = __shfl_sync(RB_FULL, il, 31);
  const uint32_t th = __shfl_sync(RB_FULL, ih, 31);
  if ((tl | th) == 0) return;
  const uint32_t lane = rb::lane_id();
  unsigned long long b = 0;
  if (lane == 31 && tl) b = atomicAdd(lq_count, (unsigned long long)tl);
  if (lane == 30 && th) b = atomicAdd(hq_count, (unsigned long long)th);
  const unsigned long long bl = __shfl_sync(RB_FULL, b, 31);
  const unsigned long long bh = __shfl_sync(RB_FULL, b, 30);
  unsigned long long pl = bl + il - nl;
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    if (on[k] && d[k] <= kLightDeg) {
      QEnt e;
      e.s = s[k];
      e.v = w[k];
      e.d = (int32_t)d[k];
      lq[pl++] = e;
    }
  }
  for (uint32_t r = 0; r < th; r += 32) {
    const uint32_t idx = r + lane;
    const bool act = idx < th;
    const uint32_t j = rb::warp_upper_bound(ih, act ? idx : th - 1);
    uint32_t local = (act ? idx : th - 1) - (__shfl_sync(RB_FULL, ih, j) - __shfl_sync(RB_FULL, nh, j));
    int32_t ew = 0;
    int64_t es = 0;
    uint32_t ed = 0;
    bool got = false;
#pragma unroll
    for (int k = 0; k < KU; ++k) {
      const uint32_t c = __shfl_sync(RB_FULL, nk[k], j);
      const int32_t wk = __shfl_sync(RB_FULL, w[k], j);
      const int64_t sk = rb::shfl_i64(s[k], j);
      const uint32_t dk = __shfl_sync(RB_FULL, d[k], j);
      if (!got && local < c) {
        got = true;
        ew = wk;
        es = sk + (int64_t)local * kChunk;
        ed = min(kChunk, dk - local * kChunk);
      } else if (!got) {
        local -= c;
      }
    }
    if (act) {
      QEnt e;
      e.s = es;
      e.v = ew;
      e.d = (int32_t)ed;
      hq[bh + idx] = e;
    }
  }
}


// Warp-collective claim of KU edges per lane (v[k] -> w[k], act[k]).
template <int KU>
__device__ __forceinline__ void td_claim(const TdCtx& c, const int32_t (&v)[KU], const int32_t (&w)[KU],
                                         const bool (&act)[KU], Acc& acc) {
  const KParams& p = *c.p;
  // claim = first to set the visited bit (vis holds every discovered vertex)
  bool claim[KU];
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    claim[k] = false;
    if (act[k]) {
      const uint32_t bit = 1u << (w[k] & 31);
      const uint32_t old = atomicOr(p.vis + (w[k] >> 5), bit);
      claim[k] = !(old & bit);
    }
  }
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    if (!claim[k]) continue;
    p.parent[w[k]] = v[k];
    p.level[w[k]] = (int32_t)(c.L + 1);
    const uint32_t old = atomicOr(c.fnext + (w[k] >> 5), 1u << (w[k] & 31));
    if (old == 0u) atomicOr(c.nznext + (w[k] >> 10), 1u << ((w[k] >> 5) & 31));
  }
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    if (claim[k]) {
      acc.n += 1;
      acc.deg += (uint32_t)rb::ldg_i32(p.deg + w[k]);
    }
  }
}

__device__ void td_level(const TdCtx& c, const QEnt* lq_in, const QEnt* hq_in, uint64_t nl,
                         uint64_t nh, Acc& acc) {
  const KParams& p = *c.p;
  const uint32_t lane = rb::lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  const uint64_t gw = warp_slot();
  const uint64_t nb = (nl + 31) / 32;
  const uint64_t total = nb + nh;
  // hub slices first (uniform size), then light batches
  for (uint64_t item = gw; item < total; item += nwarps) {
    if (item < nh) {
      const QEnt ent = ld_qent(hq_in + item);
      const int32_t v = ent.v;
      const int64_t a = ent.s;
      const int64_t b = a + ent.d;
      if (lane == 0) acc.scan += (unsigned long long)(b - a);
      int32_t vv[kChunkPerLane], w[kChunkPerLane];
      bool act[kChunkPerLane];
#pragma unroll
      for (int k = 0; k < kChunkPerLane; ++k) {
        const int64_t j = a + lane + 32 * k;
        act[k] = j < b;
        vv[k] = v;
        w[k] = act[k] ? rb::ldg_i32(p.col + j) : 0;
      }
      td_claim<kChunkPerLane>(c, vv, w, act, acc);
    } else {
      const uint64_t idx = (item - nh) * 32 + lane;
      int32_t v = 0;
      int64_t s = 0;
      uint32_t d = 0;
      if (idx < nl) {
        const QEnt ent = ld_qent(lq_in + idx);
        v = ent.v;
        s = ent.s;
        d = (uint32_t)ent.d;
      }
      const uint32_t incl = rb::warp_incl_scan(d);
      const uint32_t tot = __shfl_sync(RB_FULL, incl, 31);
      const uint32_t excl = incl - d;
      acc.scan += d;
      for (uint32_t base = 0; base < tot; base += 32 * kTdUnroll) {
        int32_t vv[kTdUnroll], w[kTdUnroll];
        bool act[kTdUnroll];
#pragma unroll
        for (int k = 0; k < kTdUnroll; ++k) {
          const uint32_t e = base + lane + 32 * k;
          act[k] = e < tot;
          const uint32_t j = rb::warp_upper_bound(incl, act[k] ? e : tot - 1);
          vv[k] = __shfl_sync(RB_FULL, v, j);
          const int64_t sj = rb::shfl_i64(s, j);
          const uint32_t exj = __shfl_sync(RB_FULL, excl, j);
          w[k] = act[k] ? rb::ldg_i32(p.col + sj + (e - exj)) : 0;
        }
        td_claim<kTdUnroll>(c, vv, w, act, acc);
      }
    }
  }
}

// Bitmap -> queues at a bottom-up -> top-down switch.  Same lane mapping as
// the bottom-up step (lane l <-> bit l of kUB consecutive words): one degree
// load per set bit, kUB independent loads per lane, warp-aggregated appends.
__device__ void compact_level(const KParams& p, const uint32_t* fcur, const uint32_t* nzcur, Slot* in, QEnt* lq,
                              QEnt* hq) {
  const uint32_t lane = rb::lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  const uint64_t gw = warp_slot();
  const uint64_t nw = (uint64_t)p.n_words;
  for (uint64_t w0 = gw * kUB; w0 < nw; w0 += nwarps * kUB) {
    const uint32_t nzb = (ld_bits(nzcur + (w0 >> 5)) >> (w0 & 31)) & ((1u << kUB) - 1u);
    if (!nzb) continue;  // no frontier vertex in these kUB words
    const uint32_t x = (lane < kUB && ((nzb >> lane) & 1u)) ? __ldcg(fcur + w0 + lane) : 0u;
    int32_t v[kUB];
    int64_t s0[kUB];
    uint32_t d[kUB];
    bool on[kUB];
#pragma unroll
    for (int k = 0; k < kUB; ++k) {
      on[k] = (__shfl_sync(RB_FULL, x, k) >> lane) & 1u;
      v[k] = (int32_t)((w0 + k) * 32 + lane);
      s0[k] = 0;
      d[k] = 0;
      if (on[k]) {
        s0[k] = rb::ldg_i64(p.rs + v[k]);
        d[k] = (uint32_t)(rb::ldg_i64(p.rs + v[k] + 1) - s0[k]);
      }
    }
    warp_append<kUB>(lq, &in->lq_count, hq, &in->hq_count, v, s0, d, on);
  }
}

// ---------------------------------------------------------------------------
// bottom-up

template <bool kRev>
__device__ __forceinline__ int64_t bu_idx(int64_t s, int64_t e, int64_t k) {
  return kRev ? e - 1 - k : s + k;
}

// Warp-cooperative finish of one long row (rank h of the warp): checks
// [t0, d) in scan order, kHeavyPerLane * 32 neighbours per step, ballot
// early exit.  Returns the parent (or -1); *checks gets the checks done.
template <bool kRev>
__device__ __forceinline__ int32_t bu_heavy(const KParams& p, const uint32_t* fcur, int64_t hs, int64_t he,
                                            int64_t t0, int64_t* checks) {
  const uint32_t lane = rb::lane_id();
  const int64_t len = he - hs;
  for (int64_t r = t0; r < len; r += 32 * kHeavyPerLane) {
    int32_t uu[kHeavyPerLane];
    uint32_t bb[kHeavyPerLane];
#pragma unroll
    for (int t = 0; t < kHeavyPerLane; ++t) {
      const int64_t q = r + lane * kHeavyPerLane + t;  // lane-major: scan order preserved per lane
      uu[t] = q < len ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(hs, he, q)) : -1;
    }
#pragma unroll
    for (int t = 0; t < kHeavyPerLane; ++t) bb[t] = uu[t] >= 0 ? ld_bits(fcur + (uu[t] >> 5)) : 0u;
    int first = -1;
    int32_t fu = -1;
#pragma unroll
    for (int t = kHeavyPerLane - 1; t >= 0; --t)
      if (uu[t] >= 0 && ((bb[t] >> (uu[t] & 31)) & 1u)) {
        first = t;
        fu = uu[t];
      }
    const uint32_t hit = __ballot_sync(RB_FULL, first >= 0);
    if (hit) {
      const int f = __ffs(hit) - 1;  // lowest lane = earliest in scan order
      const int ft = __shfl_sync(RB_FULL, first, f);
      *checks = (r - t0) + f * kHeavyPerLane + ft + 1;
      return __shfl_sync(RB_FULL, fu, f);
    }
  }
  *checks = len - t0;
  return -1;
}

template <bool kRev>
__device__ void bu_level(const KParams& p, int64_t L, const uint32_t* fcur, uint32_t* fnext, uint32_t* nznext,
                         Acc& acc, uint32_t* s_found, uint32_t* s_pair) {
  const uint32_t lane = rb::lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  const uint64_t gw = warp_slot();
  const uint64_t nw = (uint64_t)p.n_words;
  const uint64_t stride = nwarps * kBU;
  // software pipeline: the visited words of the next step are in flight while
  // this step works (fnext is pre-zeroed, so fully visited words need no store)
  uint64_t w0 = gw * kBU;
  uint32_t vw_next = (w0 < nw && lane < kBU) ? __ldcg(p.vis + w0 + lane) : 0xffffffffu;
  for (; w0 < nw; w0 += stride) {
    const uint32_t vw = vw_next;
    vw_next = (w0 + stride < nw && lane < kBU) ? __ldcg(p.vis + w0 + stride + lane) : 0xffffffffu;
    // lane l owns vertex (w0 + k) * 32 + l of each of the kBU words
    uint32_t actm = 0;
#pragma unroll
    for (int k = 0; k < kBU; ++k) actm |= ((~__shfl_sync(RB_FULL, vw, k) >> lane) & 1u) << k;
    if (!__any_sync(RB_FULL, actm != 0)) continue;
    const int64_t vbase = (int64_t)w0 * 32 + lane;
    // round 1: the two scan-first neighbours from the compact `hot` side
    // array (8 B per vertex, coalesced) -- all kBU loads in flight
    int2 hv[kBU];
    uint32_t dg[kBU];
#pragma unroll
    for (int k = 0; k < kBU; ++k) {
      hv[k] = make_int2(-1, -1);
      dg[k] = 0;
      if ((actm >> k) & 1u) {
        hv[k] = __ldg(p.hot + vbase + 32 * k);
        dg[k] = (uint32_t)rb::ldg_i32(p.deg + vbase + 32 * k);
      }
    }
    uint32_t hb0[kBU], hb1[kBU];
#pragma unroll
    for (int k = 0; k < kBU; ++k) {
      hb0[k] = hv[k].x >= 0 ? ld_bits(fcur + (hv[k].x >> 5)) : 0u;
      hb1[k] = hv[k].y >= 0 ? ld_bits(fcur + (hv[k].y >> 5)) : 0u;
    }
    uint32_t foundm = 0, needm = 0, checks = 0;
#pragma unroll
    for (int k = 0; k < kBU; ++k) {
      if (!((actm >> k) & 1u)) continue;
      int32_t par = -1;
      if (hv[k].x >= 0 && ((hb0[k] >> (hv[k].x & 31)) & 1u)) {
        par = hv[k].x;
        checks += 1;
      } else if (hv[k].y >= 0 && ((hb1[k] >> (hv[k].y & 31)) & 1u)) {
        par = hv[k].y;
        checks += 2;
      } else {
        checks += dg[k] < 2u ? dg[k] : 2u;
        if (dg[k] > 2u) needm |= 1u << k;
      }
      if (par >= 0) {
        foundm |= 1u << k;
        p.parent[vbase + 32 * k] = par;
        p.level[vbase + 32 * k] = (int32_t)(L + 1);
        acc.n += 1;
        acc.deg += dg[k];
      }
    }
    // Longer rows that did not hit: the (lane, k) pairs are compacted across
    // the warp through shared memory so every lane continues one row (up to
    // kK2 checks, 4 per step); rows longer still are finished by the whole warp.
    uint32_t* fm_s = s_found;  // kBU words: found bits per word
#pragma unroll
    for (int k = 0; k < kBU; ++k) {
      const uint32_t fm = __ballot_sync(RB_FULL, (foundm >> k) & 1u);
      if (lane == 0) fm_s[k] = fm;
    }
    const uint32_t np = __popc(needm);
    const uint32_t incl = rb::warp_incl_scan(np);
    const uint32_t npairs = __shfl_sync(RB_FULL, incl, 31);
    if (npairs) {
      uint32_t pos = incl - np;
      for (uint32_t m = needm; m; m &= m - 1) {
        const uint32_t k = __ffs(m) - 1;
        s_pair[pos] = (min(dg[k], 0xffffffu) << 8) | (k << 5) | lane;  // degree saturates at 2^24-1
        ++pos;
      }
      __syncwarp();
      for (uint32_t base = 0; base < npairs; base += 32) {
        const bool mine = base + lane < npairs;
        uint32_t idx = 0, d = 0;
        int64_t s0 = 0;
        int32_t par = -1;
        if (mine) {
          const uint32_t ent = s_pair[base + lane];
          idx = ent & 0xffu;
          d = ent >> 8;
          if (d == 0xffffffu) d = (uint32_t)rb::ldg_i32(p.deg + (int64_t)w0 * 32 + idx);
          s0 = rb::ldg_i64(p.rs + (int64_t)w0 * 32 + idx);
          const int64_t e0 = s0 + d;
          const int64_t lim = d < (uint32_t)kK2 ? d : kK2;
          for (int64_t t0 = 2; par < 0 && t0 < lim; t0 += 4) {
            int32_t uu[4];
            uint32_t bb[4];
#pragma unroll
            for (int t = 0; t < 4; ++t)
              uu[t] = (t0 + t < lim) ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(s0, e0, t0 + t)) : -1;
#pragma unroll
            for (int t = 0; t < 4; ++t) bb[t] = uu[t] >= 0 ? ld_bits(fcur + (uu[t] >> 5)) : 0u;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              if (par < 0 && uu[t] >= 0) {
                ++checks;
                if ((bb[t] >> (uu[t] & 31)) & 1u) par = uu[t];
              }
            }
          }
        }
        uint32_t hm = __ballot_sync(RB_FULL, mine && par < 0 && d > (uint32_t)kK2);
        while (hm) {
          const int h = __ffs(hm) - 1;
          hm &= hm - 1;
          const int64_t hs = rb::shfl_i64(s0, h);
          const int64_t he = hs + __shfl_sync(RB_FULL, d, h);
          int64_t hc = 0;
          const int32_t hp = bu_heavy<kRev>(p, fcur, hs, he, kK2, &hc);
          if ((int)lane == h) {
            checks += (uint32_t)hc;
            par = hp;
          }
        }
        if (mine && par >= 0) {
          const int64_t v = (int64_t)w0 * 32 + idx;
          p.parent[v] = par;
          p.level[v] = (int32_t)(L + 1);
          acc.n += 1;
          acc.deg += d;
          atomicOr(fm_s + (idx >> 5), 1u << (idx & 31));
        }
      }
      __syncwarp();
    }
    // next-frontier words (pre-zeroed) and visited words: the warp owns them
    uint32_t nzmask = 0;
#pragma unroll
    for (int k = 0; k < kBU; ++k) {
      const uint32_t fm = fm_s[k];
      nzmask |= (fm != 0u) << k;
      if (lane == (uint32_t)k && fm) {
        fnext[w0 + k] = fm;
        p.vis[w0 + k] = vw | fm;
      }
    }
    __syncwarp();
    if (lane == 0 && nzmask) atomicOr(nznext + (w0 >> 5), nzmask << (w0 & 31));
    acc.scan += checks;
  }
}

// ---------------------------------------------------------------------------

__device__ __forceinline__ void block_add3(unsigned long long* red, const Acc& a, Slot* out) {
  const unsigned long long A = rb::warp_sum_u64(a.n);
  const unsigned long long B = rb::warp_sum_u64(a.deg);
  const unsigned long long C = rb::warp_sum_u64(a.scan);
  const uint32_t w = threadIdx.x >> 5;
  if (rb::lane_id() == 0) {
    red[w * 3 + 0] = A;
    red[w * 3 + 1] = B;
    red[w * 3 + 2] = C;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    unsigned long long s = 0;
    for (int i = 0; i < kWarps; ++i) s += red[i * 3 + threadIdx.x];
    if (s) atomicAdd(threadIdx.x == 0 ? &out->n_next : (threadIdx.x == 1 ? &out->deg_next : &out->scanned), s);
  }
}

template <bool kRev>
__global__ void __launch_bounds__(kThreads, RB_MINB) bfs_persistent(KParams p) {
  __shared__ unsigned long long s_red[kWarps * 3];
  __shared__ uint32_t s_bu_found[kWarps][kBU];
  __shared__ uint32_t s_bu_pair[kWarps][32 * kBU];
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
  uint32_t epoch = 0;
  uint64_t t_prev = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) t_prev = globaltimer();

  while (done < p.max_levels && nf > 0) {
    Slot* out = p.slots + (L % 3);
    Slot* in = p.slots + ((L + 2) % 3);
    const uint32_t* fcur = fb_of(p, L);
    uint32_t* fnext = fb_of(p, L + 1);
    uint32_t* fzero = fb_of(p, L + 2);
    uint32_t* nzzero = nz_of(p, L + 2);
    // zero ahead: next level's fnext bitmap (+ summary) and the counter slot of level L+1
    for (uint64_t i = gtid; i < (uint64_t)p.n_words / 4; i += gthreads)
      reinterpret_cast<uint4*>(fzero)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (uint64_t i = gtid; i < (uint64_t)p.n_words / 32; i += gthreads) nzzero[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x < sizeof(Slot) / 8)
      reinterpret_cast<unsigned long long*>(p.slots + ((L + 1) % 3))[threadIdx.x] = 0ull;

    Acc acc{0, 0, 0};
    if (dir == 0) {
      QEnt* lq_in = (L & 1) ? p.lq1 : p.lq0;
      QEnt* hq_in = (L & 1) ? p.hq1 : p.hq0;
      if (need_compact) {
        compact_level(p, fcur, nz_of(p, L), in, lq_in, hq_in);
        rb::grid_barrier(p.bar, nblocks, epoch);
      }
      TdCtx c;
      c.p = &p;
      c.L = L;
      c.fcur = fcur;
      c.fnext = fnext;
      c.nznext = nz_of(p, L + 1);
      c.out = out;
      td_level(c, lq_in, hq_in, rb::ld_relaxed_u64(&in->lq_count), rb::ld_relaxed_u64(&in->hq_count), acc);
    } else {
      const uint32_t wib = threadIdx.x >> 5;
      bu_level<kRev>(p, L, fcur, fnext, nz_of(p, L + 1), acc, s_bu_found[wib], s_bu_pair[wib]);
    }
    block_add3(s_red, acc, out);
    rb::grid_barrier(p.bar, nblocks, epoch);

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
    need_compact = ndir == 0;  // queues are always rebuilt from the frontier bitmap
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
  p.nz0[src >> 10] |= 1u << ((src >> 5) & 31);
  p.vis[src >> 5] |= 1u << (src & 31);
  const int64_t s0 = p.rs[src];
  const uint32_t d = (uint32_t)(p.rs[src + 1] - s0);
  Slot* in = p.slots + 2;  // inputs of level 0 = outputs of "level -1"
  if (d > kLightDeg) {
    uint32_t c = 0;
    for (; c * kChunk < d; ++c) {
      QEnt e;
      e.s = s0 + (long long)c * kChunk;
      e.v = (int32_t)src;
      e.d = (int32_t)min(kChunk, d - c * kChunk);
      p.hq0[c] = e;
    }
    in->hq_count = c;
  } else {
    QEnt e;
    e.s = s0;
    e.v = (int32_t)src;
    e.d = (int32_t)d;
    p.lq0[0] = e;
    in->lq_count = 1;
  }
}

// hot[v] = the first two neighbours of v in bottom-up scan order (-1 if absent)
__global__ void make_hot(const int64_t* rs, const int32_t* col, int64_t n, int reverse, int2* hot) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = rs[v], e = rs[v + 1];
    const int64_t d = e - s;
    int2 h = make_int2(-1, -1);
    if (d > 0) h.x = reverse ? col[e - 1] : col[s];
    if (d > 1) h.y = reverse ? col[e - 2] : col[s + 1];
    hot[v] = h;
  }
}

// nz[j] bit i <=> words[32*j + i] != 0
__global__ void make_nz(const uint32_t* words, uint32_t* nz, int64_t n_nz) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_nz; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t f = 0;
    for (int i = 0; i < 32; ++i) f |= (words[j * 32 + i] != 0u ? 1u : 0u) << i;
    nz[j] = f;
  }
}

// Diagnostics: cost of the grid barrier alone (same grid as the traversal).
__global__ void __launch_bounds__(kThreads, 1) barrier_probe(uint32_t* bar, int iters) {
  uint32_t epoch = 0;
  for (int i = 0; i < iters; ++i) rb::grid_barrier(bar, gridDim.x, epoch);
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
  uint32_t* vis_template;   // isolated + padding premarked
  uint32_t* pad_mask;       // padding bits only
  int2* hot;
  int64_t n_full;  // words of a nonzero-summary bitmap (n_words / 32)
  int blocks;
  int sms;
  int bu_reverse;
  int64_t source;
  std::vector<rb_level_record> recs;
  int64_t levels_per_launch;  // kRecCap; RB_LEVELS_PER_LAUNCH=1 gives one launch per level (profiling)
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
  const int64_t tile = 32 * 32 * kBU;  // vertex alignment of the word arrays
  h->n_words = ((n_dev + tile - 1) / tile) * (tile / 32);
  h->bu_reverse = params->bu_reverse;
  h->launched = false;
  h->levels_per_launch = kRecCap;
  if (const char* env = getenv("RB_DEBUG")) h->kp.debug = atoi(env);
  if (const char* env = getenv("RB_LEVELS_PER_LAUNCH")) {
    const long long v = atoll(env);
    if (v >= 1 && v <= kRecCap) h->levels_per_launch = v;
  }
  KParams& k = h->kp;
  k.rs = d_row_starts;
  k.col = d_col;
  k.col_bu = d_col_bu ? d_col_bu : d_col;
  k.deg = d_degrees;
  k.n_dev = n_dev;
  k.n_words = h->n_words;
  const size_t wb = (size_t)h->n_words * 4;
  // hub-slice queue capacity: sum over vertices of ceil(deg / kChunk)
  const size_t nhub = (size_t)n_dev + (size_t)(params->m_directed / kChunk) + 64;
  int rc = RB_OK;
#define RB_ALLOC(ptr, bytes) \
  if (rc == RB_OK) rc = alloc_dev((void**)&(ptr), (bytes));
  RB_ALLOC(k.vis, wb);
  RB_ALLOC(k.fb0, wb);
  RB_ALLOC(k.fb1, wb);
  RB_ALLOC(k.fb2, wb);
  RB_ALLOC(h->vis_template, wb);
  RB_ALLOC(h->pad_mask, wb);
  h->n_full = h->n_words / 32;
  RB_ALLOC(k.nz0, (size_t)h->n_full * 4);
  RB_ALLOC(k.nz1, (size_t)h->n_full * 4);
  RB_ALLOC(k.nz2, (size_t)h->n_full * 4);
  RB_ALLOC(k.lq0, (size_t)n_dev * sizeof(QEnt));
  RB_ALLOC(k.lq1, (size_t)n_dev * sizeof(QEnt));
  RB_ALLOC(k.hq0, nhub * sizeof(QEnt));
  RB_ALLOC(k.hq1, nhub * sizeof(QEnt));
  RB_ALLOC(k.parent, (size_t)n_dev * 4);
  RB_ALLOC(h->hot, (size_t)n_dev * sizeof(int2));
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
  make_hot<<<1024, 256>>>(d_row_starts, k.col_bu, n_dev, params->bu_reverse, h->hot);
  k.hot = h->hot;
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
                  k.parent, k.level, k.slots, k.bar, k.rec, k.fin, k.nz0, k.nz1, k.nz2, h->hot};
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
  RB_CUDA_TRY(cudaMemsetAsync(k.nz0, 0, (size_t)h->n_full * 4, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.nz1, 0, (size_t)h->n_full * 4, s));
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
  return launch(h, (cudaStream_t)stream, 0, 0, 0, h->levels_per_launch, 1, -1, 0);
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
      if (f.levels_done) {
        RB_CUDA_TRY(cudaMemcpyAsync(h->recs.data() + old, h->kp.rec,
                                    (size_t)f.levels_done * sizeof(rb_level_record), cudaMemcpyDeviceToHost, s));
        RB_CUDA_TRY(cudaStreamSynchronize(s));
      }
      if (f.nf <= 0) break;
      RB_CUDA_TRY(cudaMemsetAsync(h->kp.bar, 0, 64, s));
      int rc = launch(h, s, f.L, f.dir, f.need_compact, h->levels_per_launch, f.nf, f.mf, f.mu);
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
  words_or<<<256, 256, 0, s>>>(k.vis, d_frontier_words, nw_in);
  RB_CUDA_TRY(cudaMemcpyAsync(k.fb0, d_frontier_words, (size_t)nw_in * 4, cudaMemcpyDeviceToDevice, s));
  make_nz<<<256, 256, 0, s>>>(k.fb0, k.nz0, h->n_full);
  RB_CUDA_TRY(cudaMemcpyAsync(k.parent, d_parent_in, (size_t)h->n_dev * 4, cudaMemcpyDeviceToDevice, s));
  h->source = 0;
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

extern "C" int rb_bfs_barrier_probe(rb_bfs* h, int iters, double* ns_per_barrier, void* stream) {
  if (!h || iters <= 0) return RB_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  RB_CUDA_TRY(cudaMemsetAsync(h->kp.bar, 0, 64, s));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  uint32_t* bar = h->kp.bar;
  void* args[] = {&bar, &iters};
  RB_CUDA_TRY(cudaEventRecord(a, s));
  RB_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)barrier_probe, dim3(h->blocks), dim3(kThreads), args, 0, s));
  RB_CUDA_TRY(cudaEventRecord(b, s));
  RB_CUDA_TRY(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  RB_CUDA_TRY(cudaMemsetAsync(h->kp.bar, 0, 64, s));
  *ns_per_barrier = 1e6 * (double)ms / iters;
  return RB_OK;
}
