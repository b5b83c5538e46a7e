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
// State (HBM; n_dev = non-isolated prefix of the RCM graph, word arrays
// padded to whole 8192-vertex tiles):
//   vis[]        uint32 words: every discovered vertex (+ isolated, padding)
//   fb[3][]      frontier bitmaps, rotated: fcur = fb[L%3], fnext = fb[(L+1)%3];
//                fb[(L+2)%3] is zeroed during level L (it is fnext of L+1)
//   nz[3][]      one byte per bitmap word: 1 = "word nonzero" (rotated with fb;
//                plain byte stores, no atomics)
//   hq[2], hs[2] hub rows {row start, vertex, degree} and the first index of
//                their 256-edge slices (phase B deals slices over all warps)
//   vinfo[]      16-B row record {40-bit row start, degree, first two neighbours}
//   hot[]        int2 per vertex: the first two neighbours in bottom-up order
//   parent[]     int32; level[] only when the caller asks for it
//   ul[2]        sparse bottom-up: the vertices still unvisited (tail levels)
//   solo_q       the frontier the solo start levels hand to the grid
// Invariant: vis holds every vertex discovered so far (the current frontier
// included), so a top-down claim is one atomicOr on vis and a bottom-up step
// tests ~vis directly.
//
// The path is latency-bound integer work, so both directions are written for
// memory-level parallelism: every lane keeps several independent loads in
// flight and work is dealt so that the whole grid is busy.
//
// Levels: CTA 0 runs the first small top-down levels alone (solo_levels,
// frontier in shared memory, no grid barrier).  Every level keeps the
// reference policy's direction label but executes the cheaper way (early
// crossover m_f <= m_u / 11, a latency cost model late).
// Top-down, phase A (td_rows_*): frontier rows from a list (after the solo
// levels), from bitmap words dealt over all warps (dense frontiers) or from
// the nonzero summary (sparse ones); row records are loaded 4 per lane.  Rows
// of degree <= 2 claim the neighbours held in the record, rows of degree <= 32
// are edge-balanced across the warp, longer rows are published as hub rows
// (one entry each) whose 256-edge slices every warp shares after a grid
// barrier (phase B, td_hubs: a contiguous slice range per warp, columns of
// the next slice in flight).  A claim is one atomicOr on the visited word
// (probe first on late or big levels); the winner sets the next-frontier bit,
// the summary byte and the parent.  Levels with >= 2^20 frontier edges are
// deferred: racing parent stores + fire-and-forget visited reds, the next
// frontier and its counters computed afterwards (count_next).
// Bottom-up (bu_level): a warp owns KB consecutive bitmap words (4 up to 2^23
// vertices, else 8), lane l bit l of each, so visited / next-frontier words
// are written with plain stores.  Round 1 checks the two scan-first neighbours
// from hot[] (reverse row order by default: RCM ids ascend with degree, so
// the end of a row holds the likely frontier hubs); rows still open are
// queued per warp and continued 32 at a time, 8 neighbours per lane per step
// up to kK2 checks; longer rows are finished by the whole warp 256 neighbours
// per step with a ballot early exit.  Late levels of large graphs with few
// unvisited vertices run over a list of them (bu_sparse_pass).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "rb_common.cuh"
#include "rb_error.h"

namespace {

#ifndef RB_THREADS
#define RB_THREADS 768  // 24 warps x 80 registers: measured best (1024 x 64 spills in the bottom-up loop; s22 -8%, s26 -6%, Chung-Lu -9%)
#endif
constexpr int kThreads = RB_THREADS;
#ifndef RB_SPARSE_ALL
#define RB_SPARSE_ALL 0  // sparse bottom-up also in the small-graph (4-word step) build
#endif
#ifndef RB_BU_PREFETCH
#define RB_BU_PREFETCH 1  // bottom-up: L2 prefetch of the next step's records while most vertices are unvisited
#endif
#ifndef RB_BU_REQUEUE
#define RB_BU_REQUEUE 1  // bottom-up (large-graph build): continued rows advance one 8-neighbour chunk per batch and are re-queued
#endif
#ifndef RB_BU_DEFER_CONT
#define RB_BU_DEFER_CONT 1  // bottom-up: continuation rows queued per warp and run 32 at a time
#endif
#define RB_LEVEL_FN __device__  // (tried __noinline__ level bodies: call-ABI spills, s26 +35%)
#ifndef RB_MINB
#define RB_MINB 1
#endif
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kLightDeg = 32;  // deg <= kLightDeg -> light queue
constexpr uint32_t kTinyDeg = 2;    // deg <= kTinyDeg -> tiny queue (neighbours inline)
constexpr int kChunkPerLane = 8;
constexpr uint32_t kChunk = 32 * kChunkPerLane;  // edges per hub work item
constexpr unsigned long long kSliceMask = (1ull << 40) - 1;  // hq_count: rows << 40 | slices
constexpr int kTdUnroll = 4;                     // light batch: edges per lane per step
constexpr int kUB = 4;                           // top-down: rows per lane per round
#ifndef RB_DENSE_NF
#define RB_DENSE_NF 1024  // measured: 256 / 1024 / 8192 -> s22 95.8 / 95.9 / 96.7 us, s26 433 / 433 / 434
#endif
constexpr int64_t kDenseFrontier = RB_DENSE_NF;
constexpr int64_t kLightToB = 1024;              // top-down: small hub levels claim light rows in phase B         // top-down: word-granular dealing from this frontier size
constexpr int kBU = 8;                           // bottom-up: max words per warp step (template KB <= kBU)
constexpr int64_t kSmallGraph = 1ll << 23;       // n_dev up to this: 4-word bottom-up steps (shorter chains)
constexpr int kList = 256;                       // top-down: rows per warp list round
constexpr int64_t kExecAlpha = 11;               // execution: early bottom-up only if m_f > m_u / 11 (measured crossover, s22 and s26)
// late-level execution cost model (picoseconds; measured level times at s22 / s26)
constexpr int64_t kTdFixPs = 8000000;   // a top-down level: summary walk + barriers
constexpr int64_t kTdRowPs = 80;        // per frontier row (bitmap walk, record load, list)
constexpr int64_t kTdEdgePs = 7;        // per frontier edge (probe / claim)
constexpr int64_t kBuFixPs = 3000000;   // a bottom-up level: zeroing + barrier
constexpr int64_t kBuStepPs = 650000;   // per warp step of the bitmap pass (dependent chain)
constexpr int64_t kBuVertPs = 5;        // per unvisited vertex
constexpr int64_t kBuCheckPs = 1;       // per neighbour check (bounded by 8 per unvisited vertex)
constexpr int64_t kBuSparsePs = 2000000; // sparse bottom-up: the list pass (+ collection barrier)
constexpr int64_t kSparseRatio = 256;   // sparse bottom-up when at most one vertex in 256 is unvisited
constexpr int64_t kListRatio = 16;      // a bitmap bottom-up level lists its survivors from one in 16 (list capacity)
constexpr int kK2 = 258;                         // bottom-up: per-lane checks before the warp takes over
constexpr int kPairCap = 32 * kBU + 64;           // bottom-up: queued continuation rows per warp
// per-warp scratch: the row queue (or a top-down row list), then one progress byte per queued row
constexpr int kPairWords = (kPairCap > kList ? kPairCap : kList) + kPairCap / 4;
constexpr int kHeavyPerLane = 8;                 // warp-cooperative bottom-up: neighbours per lane per step
constexpr uint64_t kDbgWarpBase = 65536;  // RB_DEBUG_TS buffer: per-block stamps, then per-warp stamps
constexpr uint64_t kDbgPhase = 60000;     // RB_DEBUG_TS: CTA 0 phase stamps, 8 per level (top-down sub-phases)
constexpr uint64_t kDbgWarpA = kDbgWarpBase + 64ull * 256 * 32;  // RB_DEBUG_TS: per-warp end of top-down phase A
constexpr uint64_t kDbgWarpB = kDbgWarpA + 64ull * 256 * 32;     // RB_DEBUG_TS: per-warp end of top-down phase B
constexpr int64_t kRecCap = 4096;                // level records per launch

// Queue entry: a light frontier row (d <= kLightDeg) or one hub slice
// (columns [s, s+d), d <= kChunk).  Carrying the offsets saves the dependent
// row_starts load in the consuming level.
struct __align__(16) QEnt {
  long long s;
  int32_t v;
  int32_t d;
};

struct __align__(16) VInfo {  // top-down row record (see ld_vinfo)
  uint32_t s_lo;               // row start, low 32 bits
  uint32_t sd;                 // row start bits 32..39 << 24 | degree (kVdSat: read the row starts)
  int32_t n0;                  // first two neighbours (-1: none)
  int32_t n1;
};
constexpr uint32_t kVdSat = 0xFFFFFFu;

struct Slot {  // per-level counters, triple-buffered by level % 3
  unsigned long long n_next;
  unsigned long long deg_next;
  unsigned long long scanned;
  unsigned long long hq_count;  // hub rows << 40 | their 256-edge slices, appended by phase A of the NEXT level
  unsigned long long maxdeg;    // max degree of the next frontier (hub slices needed?)
  unsigned long long ul_count;  // sparse bottom-up: 1 << 40 (a list was written) | vertices listed by this level
  unsigned long long pad2;
  unsigned long long pad3;
};

struct Final {  // state after a launch (continuation for very deep graphs)
  long long levels_done;
  long long L;
  long long dir;
  long long need_compact;
  long long nf, mf, mu;
  long long pad;
  long long reached;  // vertices discovered so far (frontier included)
  long long pad2;
};

struct KParams {
  const int64_t* rs;
  const int32_t* col;
  const int32_t* col_bu;
  const int32_t* deg;
  const int2* hot;  // per vertex: the first two neighbours in bottom-up scan order (-1 = none)
  const uint8_t* deg8;  // min(degree, 255) per vertex, zero-padded to n_words * 32 (count_next)
  int64_t n_dev;
  int64_t n_words;  // multiple of 32 * kUB
  uint32_t* vis;
  uint32_t* fb0;
  uint32_t* fb1;
  uint32_t* fb2;
  uint8_t* nz0;  // byte i: fb0 word i is nonzero -- lets sparse top-down levels skip empty words
  uint8_t* nz1;
  uint8_t* nz2;
  const VInfo* vinfo;  // top-down row records (single GPU: of the graph itself)
  // 1D partition (multi-GPU): this engine owns global vertices [v_lo, v_lo + n_dev);
  // top-down expands every GLOBAL frontier vertex through the transpose slice
  // (td_vinfo / td_col: the owned neighbours of each global vertex).  Single
  // GPU: v_lo = 0, td_* = the graph, n_words_glob = n_words.
  int64_t v_lo;
  int64_t n_words_glob;
  const VInfo* td_vinfo;
  const int64_t* td_rs;  // row starts of the top-down rows (records saturate the degree at 2^24 - 1)
  const int32_t* td_col;
  const uint32_t* fcur_ext;   // if set: the (all-gathered) global frontier bitmap of this level
  const uint8_t* nzcur_ext;  // and its nonzero summary (one byte per word)
  int64_t hubs0;              // -1: derive from deg(src); 0 / 1: forced (distributed levels)
  QEnt* hq0;           // hub rows of the current top-down level (alternating)
  QEnt* hq1;
  uint32_t* hs0;       // first slice index of each hub row (ascending)
  uint32_t* hs1;
  int32_t* parent;
  int32_t* level;
  Slot* slots;
  uint32_t* bar;
  rb_level_record* rec;
  Final* fin;
  int alpha, beta, hybrid, debug;
  unsigned long long* dbg;
  int64_t n_policy;
  // start state
  int64_t level0;
  int64_t dir0;
  int64_t need_compact0;
  int64_t max_levels;
  int64_t nf0, mf0, mu0;  // mf0 < 0: derive m_f / m_u from deg(src)
  int64_t from_fin;       // 1: traversal start; CTA 0 runs the first small levels alone (solo_levels)
  int64_t exec_opt;       // pick the executed direction by cost (see kExecAlpha)
  int64_t probe_mf;       // top-down: probe before claiming from this many frontier edges
  int64_t defer_mf;       // top-down: fire-and-forget claims + count_next from this many frontier edges
  int64_t td_m;           // entries of td_col
  int64_t exec_alpha;     // early levels labelled bottom-up run top-down if m_f * exec_alpha <= m_u
  int64_t bu_sparse;      // late bottom-up levels with few unvisited vertices run over a list
  uint32_t* solo_q;       // the frontier the solo start levels hand to the grid (kSoloCap entries)
  uint32_t* ul0;          // unvisited-vertex lists (alternating by level parity)
  uint32_t* ul1;
  int64_t src;
  int64_t m_directed;
  int64_t n_active;  // non-isolated vertices in [0, n_dev) (executed-direction cost model)
  int64_t reached0;  // vertices discovered before this launch
  // partitioned modes (rb_bfs_set_partitions): pass-1 hit count, live bounds
  int64_t count_p1;            // bottom-up: count vertices found by their first scanned neighbour
  int64_t n_parts;             // > 0: live_vertices per bottom-up level (partition.py shrink rule)
  int64_t n_full;              // g.n: the reference's bitmap size (isolated tail included)
  const int32_t* part_blk;     // n_parts + 1 partition bounds in 512-vertex blocks (last: ceil(n_full / 512))
  int32_t* part_first;         // per partition: first / last block that is not all visited (reset to
  int32_t* part_last;          //   INT_MAX / -1 after every use)
};

__device__ __forceinline__ uint32_t* fb_of(const KParams& p, int r) {  // r = level % 3
  return r == 0 ? p.fb0 : (r == 1 ? p.fb1 : p.fb2);
}

__device__ __forceinline__ uint8_t* nz_of(const KParams& p, int r) {
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
  uint32_t maxdeg;
};

// Global warp index, interleaved across blocks: consecutive work items go to
// different SMs, so a small level is not concentrated on a few SMs' LSU/L1.
__device__ __forceinline__ uint64_t warp_slot() {
  return (uint64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
}

__device__ __forceinline__ void red_or(uint32_t* a, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

struct TdCtx {
  const KParams* p;
  int64_t L;
  const uint32_t* fcur;
  uint32_t* fnext;
  uint8_t* nznext;
  bool probe;  // probe visited bits before the atomic (most targets visited)
  bool defer;  // fire-and-forget claims; the next frontier is counted after the level (count_next)
  uint32_t hub_min;  // rows longer than this go to phase B (kLightDeg; kTinyDeg on small hub levels)
};

__device__ __forceinline__ QEnt ld_qent(const QEnt* q) {
  const int4 x = __ldcg(reinterpret_cast<const int4*>(q));
  QEnt e;
  e.s = (long long)(((unsigned long long)(uint32_t)x.y << 32) | (uint32_t)x.x);
  e.v = x.z;
  e.d = x.w;
  return e;
}

// Top-down row record: 16 bytes per vertex (row start, degree and the first
// two neighbours) -- one load per row, two rows per sector in the dense
// regions of a clustered frontier.
__device__ __forceinline__ void ld_vinfo(const KParams& p, int64_t v, int64_t& s, uint32_t& d, int32_t& n0,
                                         int32_t& n1) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(p.td_vinfo + v));
  s = (int64_t)(((uint64_t)((uint32_t)a.y >> 24) << 32) | (uint32_t)a.x);
  d = (uint32_t)a.y & kVdSat;
  if (d == kVdSat) d = (uint32_t)(rb::ldg_i64(p.td_rs + v + 1) - s);  // degree >= 2^24: rare
  n0 = a.z;
  n1 = a.w;
}

// Deferred claim of KU edges per lane given the probed visited words.
// Big levels: no atomic return trip and no per-winner degree load.  Every
// frontier vertex adjacent to an unvisited w is a valid parent of w, so
// concurrent writers of parent[w] may race -- the last store stands.  Only
// the visited bit is set (fire-and-forget red; it also stops later probes
// of this level): the next frontier is vis minus the copy of vis taken at
// the level start (held in fnext), and its summary and exact counters
// (n_next, deg_next, max degree) come from one pass over it (count_next).
template <int KU>
__device__ __forceinline__ void td_claim_deferred(const TdCtx& c, const int32_t (&v)[KU], const int32_t (&wl)[KU],
                                                  const bool (&act)[KU], const uint32_t (&seen)[KU]) {
  const KParams& p = *c.p;
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    const uint32_t bit = 1u << (wl[k] & 31);
    if (act[k] && !(seen[k] & bit)) {
      p.parent[wl[k]] = v[k];
      if (p.level) p.level[wl[k]] = (int32_t)(c.L + 1);
      red_or(p.vis + (wl[k] >> 5), bit);
    }
  }
}

// Warp-collective claim of KU edges per lane (v[k] -> w[k], act[k]).
template <int KU>
__device__ __forceinline__ void td_claim(const TdCtx& c, const int32_t (&v)[KU], const int32_t (&w)[KU],
                                         const bool (&act)[KU], Acc& acc) {
  const KParams& p = *c.p;
  // targets are global ids of OWNED vertices; local index = w - v_lo
  int32_t wl[KU];
#pragma unroll
  for (int k = 0; k < KU; ++k) wl[k] = w[k] - (int32_t)p.v_lo;
  if (c.defer) {
    uint32_t seen[KU];
#pragma unroll
    for (int k = 0; k < KU; ++k) seen[k] = act[k] ? ld_bits(p.vis + (wl[k] >> 5)) : 0u;
    td_claim_deferred<KU>(c, v, wl, act, seen);
    return;
  }
  // claim = first to set the visited bit (vis holds every discovered vertex).
  // Late levels (most targets already visited) first probe with a plain,
  // L1-cacheable load -- bits only ever get set, so a stale probe can only
  // cost an extra atomic; early levels go straight to the atomic.
  uint32_t seen[KU];
#pragma unroll
  for (int k = 0; k < KU; ++k) seen[k] = (act[k] && c.probe) ? ld_bits(p.vis + (wl[k] >> 5)) : 0u;
  bool claim[KU];
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    claim[k] = false;
    const uint32_t bit = 1u << (wl[k] & 31);
    if (act[k] && !(seen[k] & bit)) {
      const uint32_t old = atomicOr(p.vis + (wl[k] >> 5), bit);
      claim[k] = !(old & bit);
    }
  }
  // the degree loads of the winners are issued before the frontier atomics
  uint32_t dw[KU];
#pragma unroll
  for (int k = 0; k < KU; ++k) dw[k] = claim[k] ? (uint32_t)rb::ldg_i32(p.deg + wl[k]) : 0u;
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    if (!claim[k]) continue;
    p.parent[wl[k]] = v[k];
    if (p.level) p.level[wl[k]] = (int32_t)(c.L + 1);
    red_or(c.fnext + (wl[k] >> 5), 1u << (wl[k] & 31));  // fire-and-forget: no return trip
    c.nznext[wl[k] >> 5] = 1u;
  }
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    if (claim[k]) {
      acc.n += 1;
      acc.deg += dw[k];
      acc.maxdeg = max(acc.maxdeg, dw[k]);
    }
  }
}

// Warp-aggregated append of hub rows (deg > kLightDeg): one entry per row
// {row start, vertex, degree} plus its first slice index.  One 64-bit atomic
// per warp reserves rows and slices together (rows << 40 | slices), so the
// slice starts ascend with the row index and phase B maps a slice to its row
// by search; a row of a million edges costs one entry, not 4000.
template <int KU>
__device__ __forceinline__ void warp_push_rows(QEnt* hq, uint32_t* hs, unsigned long long* count,
                                               const int32_t (&w)[KU], const int64_t (&s)[KU],
                                               const uint32_t (&d)[KU], const bool (&hub)[KU]) {
  uint32_t nr = 0, ns = 0;
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    nr += hub[k] ? 1u : 0u;
    ns += hub[k] ? (d[k] + kChunk - 1) / kChunk : 0u;
  }
  const uint32_t ir = rb::warp_incl_scan(nr);
  const uint32_t tr = __shfl_sync(RB_FULL, ir, 31);
  if (tr == 0) return;
  const uint32_t is = rb::warp_incl_scan(ns);
  const uint32_t ts = __shfl_sync(RB_FULL, is, 31);
  unsigned long long b = 0;
  if (rb::lane_id() == 31) b = atomicAdd(count, ((unsigned long long)tr << 40) | ts);
  b = __shfl_sync(RB_FULL, b, 31);
  uint64_t r = (b >> 40) + ir - nr;
  uint32_t sl = (uint32_t)(b & kSliceMask) + is - ns;
#pragma unroll
  for (int k = 0; k < KU; ++k) {
    if (!hub[k]) continue;
    QEnt e;
    e.s = s[k];
    e.v = w[k];
    e.d = (int32_t)d[k];
    hq[r] = e;
    hs[r] = sl;
    ++r;
    sl += (d[k] + kChunk - 1) / kChunk;
  }
}

// The hub row holding slice i (warp-uniform i < total slices): the last row
// whose first slice <= i, by a 32-ary warp search over hs.  The final step
// loads the candidate rows' entries together with their first slices, so a
// level with <= 32 hub rows pays one round trip.  Returns the row entry and
// sets *first to its first slice and *r to its index.
__device__ __forceinline__ QEnt row_of_slice(const QEnt* hq, const uint32_t* hs, uint64_t nrows, uint64_t i,
                                             uint32_t* first, uint64_t* r) {
  const uint32_t lane = rb::lane_id();
  uint64_t lo = 0, hi = nrows;
  while (hi - lo > 32) {
    const uint64_t step = (hi - lo + 31) / 32;
    const uint64_t idx = lo + lane * step;
    const bool le = idx < hi && (uint64_t)__ldcg(hs + idx) <= i;
    const uint32_t m = __ballot_sync(RB_FULL, le);  // lane 0 always qualifies
    lo += (uint64_t)(31 - __clz(m)) * step;
    hi = min(lo + step, hi);
  }
  const uint64_t idx = lo + lane;
  const bool in = idx < hi;
  const uint32_t h = in ? __ldcg(hs + idx) : 0xffffffffu;
  const int4 q = in ? __ldcg(reinterpret_cast<const int4*>(hq + idx)) : make_int4(0, 0, 0, 0);
  const uint32_t m = __ballot_sync(RB_FULL, in && (uint64_t)h <= i);
  const int j = 31 - __clz(m);
  *first = __shfl_sync(RB_FULL, h, j);
  *r = lo + j;
  QEnt e;
  e.s = (long long)(((unsigned long long)(uint32_t)__shfl_sync(RB_FULL, q.y, j) << 32) |
                    (uint32_t)__shfl_sync(RB_FULL, q.x, j));
  e.v = __shfl_sync(RB_FULL, q.z, j);
  e.d = __shfl_sync(RB_FULL, q.w, j);
  return e;
}

// Top-down phase A: the frontier rows straight from the bitmap.  Rows with
// deg <= 2 claim their inline neighbours directly, rows with deg <= 32 are
// edge-balanced across the warp (4 edges per lane per step), hub rows are
// appended as 256-edge slices for phase B.
// The rows of a warp's shared-memory list lst[0, tot), 4 per lane per round.
__device__ __forceinline__ void td_list(const TdCtx& c, const uint32_t* lst, uint32_t tot, QEnt* hq, uint32_t* hs,
                                        unsigned long long* hq_count, Acc& acc) {
  const KParams& p = *c.p;
  const uint32_t lane = rb::lane_id();
  for (uint32_t r = 0; r < tot; r += 32 * kUB) {
    int32_t v[kUB];
    int64_t s0[kUB];
    uint32_t d[kUB];
    int32_t n0[kUB], n1[kUB];
    bool on[kUB], hub[kUB];
#pragma unroll
    for (int k = 0; k < kUB; ++k) {
      const uint32_t t = r + 32 * k + lane;
      on[k] = t < tot;
      v[k] = on[k] ? (int32_t)lst[t] : 0;
      s0[k] = 0;
      d[k] = 0;
      n0[k] = n1[k] = 0;
      if (on[k]) ld_vinfo(p, v[k], s0[k], d[k], n0[k], n1[k]);
    }
    // rows with deg <= 2: neighbours are in the record
    {
      int32_t tv[2 * kUB], tw[2 * kUB];
      bool ta[2 * kUB];
#pragma unroll
      for (int k = 0; k < kUB; ++k) {
        const bool tiny = on[k] && d[k] >= 1 && d[k] <= kTinyDeg;
        tv[2 * k] = tv[2 * k + 1] = v[k];
        tw[2 * k] = n0[k];
        tw[2 * k + 1] = n1[k];
        ta[2 * k] = tiny;
        ta[2 * k + 1] = tiny && d[k] == 2;
        hub[k] = on[k] && d[k] > c.hub_min;
        if (on[k] && !hub[k]) acc.scan += d[k];
      }
      td_claim<2 * kUB>(c, tv, tw, ta, acc);
    }
    // rows with 2 < deg <= 32: edge-balanced over the warp
    uint32_t ld[kUB], lsum = 0;
#pragma unroll
    for (int k = 0; k < kUB; ++k) {
      ld[k] = (on[k] && d[k] > kTinyDeg && d[k] <= c.hub_min) ? d[k] : 0u;
      lsum += ld[k];
    }
    const uint32_t li = rb::warp_incl_scan(lsum);
    const uint32_t lt = __shfl_sync(RB_FULL, li, 31);
    for (uint32_t base = 0; base < lt; base += 32 * kTdUnroll) {
      int32_t vv[kTdUnroll], w[kTdUnroll];
      bool act[kTdUnroll];
#pragma unroll
      for (int q = 0; q < kTdUnroll; ++q) {
        const uint32_t e = base + 32 * q + lane;
        act[q] = e < lt;
        const uint32_t ec = act[q] ? e : lt - 1;
        const uint32_t o = rb::warp_upper_bound(li, ec);
        uint32_t local = ec - (__shfl_sync(RB_FULL, li, o) - __shfl_sync(RB_FULL, lsum, o));
        int32_t rv = 0;
        int64_t rs0 = 0;
        bool got = false;
#pragma unroll
        for (int k = 0; k < kUB; ++k) {
          const uint32_t dk = __shfl_sync(RB_FULL, ld[k], o);
          const int32_t vk = __shfl_sync(RB_FULL, v[k], o);
          const int64_t sk = rb::shfl_i64(s0[k], o);
          if (!got && local < dk) {
            got = true;
            rv = vk;
            rs0 = sk + local;
          } else if (!got) {
            local -= dk;
          }
        }
        vv[q] = rv;
        w[q] = act[q] ? rb::ldg_i32(p.td_col + rs0) : 0;
      }
      td_claim<kTdUnroll>(c, vv, w, act, acc);
    }
    warp_push_rows<kUB>(hq, hs, hq_count, v, s0, d, hub);
  }
}

// Top-down phase A, dense frontiers: batch q (of Q = nw / 32) holds the
// bitmap words q + l * Q, one per lane, so consecutive words fall in
// consecutive batches and a dense region of a clustered (RCM) frontier
// spreads over every CTA and warp 32 vertices at a time.  CTA b owns batches
// b, b + gridDim.x, ...; its warps claim them from a shared counter (one
// batch ahead, its words in flight).  The nonzero words of a batch are
// compacted into the warp's shared-memory list, at most 256 rows per round
// (popc + warp scan + a loop over each lane's set bits).
RB_LEVEL_FN void td_rows_words_small(const TdCtx& c, QEnt* hq, uint32_t* hs, unsigned long long* hq_count, Acc& acc,
                               uint32_t* lst,
                              uint32_t* s_next) {
  const KParams& p = *c.p;
  const uint32_t lane = rb::lane_id();
  const uint64_t nw = (uint64_t)p.n_words_glob;
  const uint64_t Q = (nw + 31) / 32;
  auto claim = [&]() -> uint64_t {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(s_next, 1u);
    k = __shfl_sync(RB_FULL, k, 0);
    return (uint64_t)blockIdx.x + (uint64_t)k * gridDim.x;
  };
  uint64_t q_nx = claim();
  uint64_t w_nx = q_nx + (uint64_t)lane * Q;
  uint32_t x_nx = (q_nx < Q && w_nx < nw) ? __ldcg(c.fcur + w_nx) : 0u;
  while (q_nx < Q) {
    uint32_t x = x_nx;
    const uint32_t vb = (uint32_t)(w_nx * 32);
    q_nx = claim();
    w_nx = q_nx + (uint64_t)lane * Q;
    x_nx = (q_nx < Q && w_nx < nw) ? __ldcg(c.fcur + w_nx) : 0u;
    while (__any_sync(RB_FULL, x != 0u)) {
      // take a prefix of the lanes whose rows fit the 256-entry list
      const uint32_t cnt = __popc(x);
      const uint32_t incl = rb::warp_incl_scan(cnt);
      const bool take = incl <= (uint32_t)kList;
      const uint32_t tot = __reduce_max_sync(RB_FULL, take ? incl : 0u);
      __syncwarp();
      if (take) {
        uint32_t pos = incl - cnt;
        for (uint32_t y = x; y; y &= y - 1) lst[pos++] = vb + (__ffs(y) - 1);
        x = 0u;
      }
      __syncwarp();
      td_list(c, lst, tot, hq, hs, hq_count, acc);
    }
  }
}

RB_LEVEL_FN void td_rows_words_big(const TdCtx& c, QEnt* hq, uint32_t* hs, unsigned long long* hq_count, Acc& acc,
                               uint32_t* lst,
                              uint32_t* s_next) {
  // A warp claims kG batches per shared-counter add and has their words in
  // flight together; the rows of the whole group go through ONE list round when
  // they fit (one record-load latency and one hub-row append per group instead
  // of per batch: phase A of a 5 K-row frontier at scale 26 took 9+ dependent
  // claim / load / append rounds per warp, 17.6 us; 13 us with groups).
  constexpr int kG = 2;  // (4 / 8: more spills, s26 -0.4 % / -1.3 %)
  static_assert(32 * kG <= kList, "a lane's rows must fit one list round");
  const KParams& p = *c.p;
  const uint32_t lane = rb::lane_id();
  const uint64_t nw = (uint64_t)p.n_words_glob;
  const uint64_t Q = (nw + 31) / 32;
  // (groups only when every warp has several batches to do: a scale-22 bitmap is one batch per warp)
  const uint32_t g = Q >= 2ull * kG * gridDim.x * kWarps ? (uint32_t)kG : 1u;
  while (true) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(s_next, g);
    k = __shfl_sync(RB_FULL, k, 0);
    if ((uint64_t)blockIdx.x + (uint64_t)k * gridDim.x >= Q) break;
    uint32_t x[kG], vb[kG];
    uint32_t cnt;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const uint64_t q = (uint64_t)blockIdx.x + (uint64_t)(k + j) * gridDim.x;
      const uint64_t w = q + (uint64_t)lane * Q;
      x[j] = ((uint32_t)j < g && q < Q && w < nw) ? __ldcg(c.fcur + w) : 0u;
      vb[j] = (uint32_t)(w * 32);
    }
    while (true) {
      // the rows of a prefix of the lanes that fits the 256-entry list (a lane
      // holds at most 32 kG <= kList rows, so every round makes progress)
      cnt = 0;
#pragma unroll
      for (int j = 0; j < kG; ++j) cnt += __popc(x[j]);
      const uint32_t incl = rb::warp_incl_scan(cnt);
      const bool take = incl <= (uint32_t)kList;
      const uint32_t tot = __reduce_max_sync(RB_FULL, take ? incl : 0u);
      if (tot == 0) break;
      __syncwarp();
      if (take) {
        uint32_t pos = incl - cnt;
#pragma unroll
        for (int j = 0; j < kG; ++j) {
          for (uint32_t y = x[j]; y; y &= y - 1) lst[pos++] = vb[j] + (__ffs(y) - 1);
          x[j] = 0u;
        }
      }
      __syncwarp();
      td_list(c, lst, tot, hq, hs, hq_count, acc);
    }
  }
}

// Small graphs (4-word bottom-up build) keep the one-batch-ahead loop: their
// bitmap is about one batch per warp, and the grouped loop measured 2 % slower
// at scale 22.
template <bool kBig>
__device__ __forceinline__ void td_rows_words(const TdCtx& c, QEnt* hq, uint32_t* hs, unsigned long long* hq_count,
                                              Acc& acc, uint32_t* lst, uint32_t* s_next) {
  if constexpr (kBig)
    td_rows_words_big(c, hq, hs, hq_count, acc, lst, s_next);
  else
    td_rows_words_small(c, hq, hs, hq_count, acc, lst, s_next);
}

// Top-down phase A from a frontier list (the one the solo levels leave):
// warp slot s takes entries [32 s, 32 s + 32).
__device__ void td_rows_list(const TdCtx& c, const uint32_t* q, uint32_t n, QEnt* hq, uint32_t* hs,
                             unsigned long long* hq_count, Acc& acc, uint32_t* lst) {
  const uint32_t lane = rb::lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t b = warp_slot() * 32; b < n; b += nwarps * 32) {
    const uint32_t tot = (uint32_t)min((uint64_t)32, n - b);
    __syncwarp();
    if (lane < tot) lst[lane] = __ldcg(q + b + lane);
    __syncwarp();
    td_list(c, lst, tot, hq, hs, hq_count, acc);
  }
}

// Top-down phase A, sparse frontiers: the lanes of a warp check 32 bytes of
// the nonzero summary (each bit covers one bitmap word, a byte one 256-vertex
// item) strided over the whole range, so one load skips 32 empty items; a
// nonzero item is compacted into the warp's list (lane l owns byte l).
RB_LEVEL_FN void td_rows_items(const TdCtx& c, const uint8_t* nzcur, QEnt* hq, uint32_t* hs,
                               unsigned long long* hq_count,
                              Acc& acc, uint32_t* lst) {
  const KParams& p = *c.p;
  const uint32_t lane = rb::lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  const uint64_t n_items = (uint64_t)p.n_words_glob / 8;
  for (uint64_t i0 = warp_slot(); i0 < n_items; i0 += nwarps * 32) {
    const uint64_t ime = i0 + (uint64_t)lane * nwarps;
    uint32_t nzb = 0u;  // bit j: word 8 * ime + j is nonzero
    if (ime < n_items) {
      const uint2 b = __ldcg(reinterpret_cast<const uint2*>(nzcur + ime * 8));
      nzb = (b.x & 1u) | ((b.x >> 7) & 2u) | ((b.x >> 14) & 4u) | ((b.x >> 21) & 8u) | ((b.y & 1u) << 4) |
            ((b.y >> 3) & 32u) | ((b.y >> 10) & 64u) | ((b.y >> 17) & 128u);
    }
    for (uint32_t mask = __ballot_sync(RB_FULL, nzb != 0u); mask; mask &= mask - 1) {
      const uint32_t il = __ffs(mask) - 1;
      const uint64_t wbase = (i0 + (uint64_t)il * nwarps) * 8;  // first bitmap word of this item
      const uint32_t bits = __shfl_sync(RB_FULL, nzb, il);
      const uint32_t wi = lane >> 2;
      const uint32_t x = ((bits >> wi) & 1u) ? __ldcg(c.fcur + wbase + wi) : 0u;
      uint32_t byte = (x >> (8 * (lane & 3))) & 0xffu;
      const uint32_t cnt = __popc(byte);
      const uint32_t incl = rb::warp_incl_scan(cnt);
      const uint32_t tot = __shfl_sync(RB_FULL, incl, 31);
      uint32_t pos = incl - cnt;
      const uint32_t vb = (uint32_t)(wbase * 32) + lane * 8;
      __syncwarp();
      while (byte) {
        lst[pos++] = vb + (__ffs(byte) - 1);
        byte &= byte - 1;
      }
      __syncwarp();
      td_list(c, lst, tot, hq, hs, hq_count, acc);
    }
  }
}

// End of a deferred top-down level: fnext (holding vis as it was at the
// level start) becomes the next frontier vis & ~fnext, with its nonzero
// summary; counters n_next = popcount, deg_next = sum of the degrees of the
// new bits, max degree.  Streaming passes instead of per-claim random traffic.
struct CnArgs {  // the fields count_next reads
  const uint32_t* vis;
  const uint8_t* deg8;
  const int32_t* deg;
  uint64_t n_words;
  int64_t n_dev;
};
__device__ __forceinline__ Acc count_next_fn(const CnArgs p, uint32_t* fnext, uint8_t* nznext) {
  Acc acc{0, 0, 0, 0u};
  // Lane l owns word w0 + l: its next-frontier bits, and -- if any -- the 32
  // degrees of that word from the saturating 8-bit copy deg8 (ONE sector per
  // word, two 16-B loads; the int32 degrees cost four sectors and made this
  // pass read the whole 4 n_dev-byte array on every deferred level).  Bits are
  // spread to byte masks by a carry-free multiply, selected bytes summed with
  // dp4a; a selected byte of 255 (degree >= 255: the high-id hub region only)
  // reads the exact degree.
  // kCN words per lane per round, every load of a round in flight together
  // (the pass is a chain of dependent round trips per warp, not bandwidth).
  constexpr int kCN = 4;
  const uint32_t lane = rb::lane_id();
  const uint64_t nw = (uint64_t)p.n_words;
  const uint64_t stride = (uint64_t)gridDim.x * kWarps * 32;
  for (uint64_t w0 = warp_slot() * 32; w0 < nw; w0 += kCN * stride) {
    uint32_t x[kCN];
#pragma unroll
    for (int r = 0; r < kCN; ++r) {
      const uint64_t w = w0 + r * stride + lane;
      x[r] = w < nw ? (__ldcg(p.vis + w) & ~__ldcg(fnext + w)) : 0u;
    }
    uint4 qa[kCN], qb[kCN];
#pragma unroll
    for (int r = 0; r < kCN; ++r) {
      const uint64_t w = w0 + r * stride + lane;
      qa[r] = qb[r] = make_uint4(0u, 0u, 0u, 0u);
      if (x[r]) {  // (deg8 is padded to n_words * 32)
        const uint4* dp = reinterpret_cast<const uint4*>(p.deg8 + (int64_t)w * 32);
        qa[r] = __ldg(dp);
        qb[r] = __ldg(dp + 1);
      }
    }
#pragma unroll
    for (int r = 0; r < kCN; ++r) {
      const uint64_t w = w0 + r * stride + lane;
      if (w < nw) {
        fnext[w] = x[r];
        nznext[w] = x[r] != 0u ? 1u : 0u;
      }
      acc.n += __popc(x[r]);
      const uint32_t q[8] = {qa[r].x, qa[r].y, qa[r].z, qa[r].w, qb[r].x, qb[r].y, qb[r].z, qb[r].w};
      uint32_t sum = 0, mx = 0, sat = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        // bits 4j .. 4j+3 of x -> 0xFF in bytes 0 .. 3 (bit k lands on bit 8k: k + 7k, no carries)
        const uint32_t m = ((((x[r] >> (4 * j)) & 0xFu) * 0x00204081u) & 0x01010101u) * 0xFFu;
        const uint32_t sel = q[j] & m;
        sum = __dp4a(sel, 0x01010101u, sum);
        mx = __vmaxu4(mx, sel);
        sat |= __vcmpeq4(sel, 0xFFFFFFFFu);
      }
      uint32_t dmax = max(max(mx & 0xFFu, (mx >> 8) & 0xFFu), max((mx >> 16) & 0xFFu, mx >> 24));
      if (sat) {  // a selected degree >= 255 (hub region): the word's exact degrees, all loads in flight
        sum = 0;
        dmax = 0;
        if ((int64_t)(w + 1) * 32 <= p.n_dev) {
          const int4* dq = reinterpret_cast<const int4*>(p.deg + (int64_t)w * 32);
          int4 f[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) f[j] = __ldg(dq + j);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t dv[4] = {(uint32_t)f[j].x, (uint32_t)f[j].y, (uint32_t)f[j].z, (uint32_t)f[j].w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const uint32_t d = ((x[r] >> (4 * j + t)) & 1u) ? dv[t] : 0u;
              sum += d;
              dmax = max(dmax, d);
            }
          }
        } else {  // the word holding the end of the vertex range: no reads past deg[n_dev)
          for (uint32_t y = x[r]; y; y &= y - 1) {
            const uint32_t d = (uint32_t)rb::ldg_i32(p.deg + (int64_t)w * 32 + (__ffs(y) - 1));
            sum += d;
            dmax = max(dmax, d);
          }
        }
      }
      acc.deg += sum;
      acc.maxdeg = max(acc.maxdeg, dmax);
    }
  }
  return acc;
}

__device__ __forceinline__ void count_next_small(const KParams& p, uint32_t* fnext, uint8_t* nznext, Acc& acc) {
  // Lane l owns word w0 + l: its next-frontier bits, and -- if any -- the 32
  // degrees of that word as eight 16-B loads, all in flight together (one
  // round trip per 32 words instead of one per 4 nonzero words).
  const uint32_t lane = rb::lane_id();
  const uint64_t nw = (uint64_t)p.n_words;
  const uint64_t stride = (uint64_t)gridDim.x * kWarps * 32;
  for (uint64_t w0 = warp_slot() * 32; w0 < nw; w0 += stride) {
    const uint64_t w = w0 + lane;
    const uint32_t x = __ldcg(p.vis + w) & ~__ldcg(fnext + w);
    fnext[w] = x;
    nznext[w] = x != 0u ? 1u : 0u;
    acc.n += __popc(x);
    if (!x) continue;
    if ((int64_t)(w + 1) * 32 <= p.n_dev) {
      const int4* dp = reinterpret_cast<const int4*>(p.deg + (int64_t)w * 32);
      int4 q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = __ldg(dp + j);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t dv[4] = {(uint32_t)q[j].x, (uint32_t)q[j].y, (uint32_t)q[j].z, (uint32_t)q[j].w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t d = ((x >> (4 * j + c)) & 1u) ? dv[c] : 0u;
          acc.deg += d;
          acc.maxdeg = max(acc.maxdeg, d);
        }
      }
    } else {  // the word holding the end of the vertex range: no reads past deg[n_dev)
      for (uint32_t y = x; y; y &= y - 1) {
        const uint32_t d = (uint32_t)rb::ldg_i32(p.deg + (int64_t)w * 32 + (__ffs(y) - 1));
        acc.deg += d;
        acc.maxdeg = max(acc.maxdeg, d);
      }
    }
  }
}

template <bool kBig>
__device__ __forceinline__ void count_next(const KParams& p, uint32_t* fnext, uint8_t* nznext, Acc& acc) {
  if constexpr (kBig) {
    const CnArgs a{p.vis, p.deg8, p.deg, (uint64_t)p.n_words, p.n_dev};
    const Acc r = count_next_fn(a, fnext, nznext);
    acc.n += r.n;
    acc.deg += r.deg;
    acc.maxdeg = max(acc.maxdeg, r.maxdeg);
  } else {
    count_next_small(p, fnext, nznext, acc);  // (one round per warp at scale 22: the exact degrees in one round trip)
  }
}

// Top-down phase B: hub slices, one warp item each (8 edges per lane).
#ifndef RB_TD_DYN_MINK
#define RB_TD_DYN_MINK 16  // slices per warp from which the tail of phase B is dealt dynamically
#endif
#ifndef RB_TD_DYN_NUM
#define RB_TD_DYN_NUM 3    // static share of phase B: RB_TD_DYN_NUM / 4 of the slices
#endif
#ifndef RB_TD_DYN_CHUNK
#define RB_TD_DYN_CHUNK 8  // slices per dynamic claim (4: the row search per claim ate the gain)
#endif
RB_LEVEL_FN void td_hubs(const TdCtx& c, const QEnt* hq, const uint32_t* hs, uint64_t nrows, uint64_t nh,
                         unsigned long long* dyn, Acc& acc) {
  // Warp g takes the contiguous slices [g*K, (g+1)*K): one row search per
  // warp, then the rows are walked in order (each warp streams its own part
  // of the column array).  Software-pipelined: the columns of the next slice
  // are in flight while the current one is probed and claimed.
  // Big levels (dyn set, >= RB_TD_DYN_MINK slices per warp): equal slice counts
  // do not finish together -- the warps of a scale-26 deferred level ended
  // between 120 and 176 us (claim density and L1 hits differ by row) and the
  // grid waited for the last one.  There only the first 3/4 of the slices are
  // dealt statically; the rest is claimed in chunks of RB_TD_DYN_CHUNK slices
  // from a level counter, the next claim in flight while a chunk is processed.
  const KParams& p = *c.p;
  const uint32_t lane = rb::lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  uint64_t K = (nh + nwarps - 1) / nwarps;
  uint64_t dyn0 = nh;  // first dynamically dealt slice
  if (dyn && nh / nwarps >= (uint64_t)RB_TD_DYN_MINK) {
    K = (nh / nwarps) * RB_TD_DYN_NUM / 4;
    dyn0 = K * nwarps;
  }
  unsigned long long ticket = 0;
  if (dyn0 < nh && lane == 0) ticket = atomicAdd(dyn, (unsigned long long)RB_TD_DYN_CHUNK);
  auto columns = [&](const QEnt& e, int32_t (&x)[kChunkPerLane]) {
#pragma unroll
    for (int k = 0; k < kChunkPerLane; ++k) {
      const int32_t j = (int32_t)lane + 32 * k;
      x[k] = j < e.d ? rb::ldg_i32(p.td_col + e.s + j) : -1;
    }
  };
  uint64_t i0 = warp_slot() * K;
  uint32_t left = i0 < dyn0 ? (uint32_t)min(K, dyn0 - i0) : 0u;  // slices still to process
  while (true) {
    if (left > 0) {
      // current slice: row entry `row` (index r), edges [row.s + o, row.s + o + 256) of it
      int32_t w[kChunkPerLane];
      // the row's remaining edges after the current slice, and the next row index
      int64_t rest;   // edges of the current row after this slice
      uint64_t rnext;  // index of the next row
      QEnt cur;
      {
        uint32_t first;
        uint64_t r0;
        const QEnt row = row_of_slice(hq, hs, nrows, i0, &first, &r0);
        const int64_t off = (int64_t)(i0 - first) * kChunk;
        cur.s = row.s + off;
        cur.v = row.v;
        cur.d = (int32_t)min((int64_t)kChunk, (int64_t)row.d - off);
        rest = (int64_t)row.d - off - cur.d;
        rnext = r0 + 1;
      }
      columns(cur, w);
      while (true) {
        // descriptor of the next slice (same row, or the start of the next row)
        QEnt nx;
        nx.s = 0;
        nx.v = 0;
        nx.d = 0;
        int64_t nrest = 0;
        if (left > 1) {
          if (rest > 0) {
            nx.s = cur.s + cur.d;
            nx.v = cur.v;
            nx.d = (int32_t)min((int64_t)kChunk, rest);
            nrest = rest - nx.d;
          } else {
            const QEnt row = ld_qent(hq + rnext);
            ++rnext;
            nx.s = row.s;
            nx.v = row.v;
            nx.d = min((int32_t)kChunk, row.d);
            nrest = (int64_t)row.d - nx.d;
          }
        }
        int32_t w2[kChunkPerLane];
        columns(nx, w2);
        if (lane == 0) acc.scan += (unsigned long long)cur.d;
        int32_t vv[kChunkPerLane];
        bool act[kChunkPerLane];
#pragma unroll
        for (int k = 0; k < kChunkPerLane; ++k) {
          vv[k] = cur.v;
          act[k] = w[k] >= 0;
        }
        td_claim<kChunkPerLane>(c, vv, w, act, acc);
        if (--left == 0) break;
        cur = nx;
        rest = nrest;
#pragma unroll
        for (int k = 0; k < kChunkPerLane; ++k) w[k] = w2[k];
      }
    }
    if (dyn0 >= nh) break;
    i0 = dyn0 + __shfl_sync(RB_FULL, ticket, 0);
    if (i0 >= nh) break;
    if (lane == 0) ticket = atomicAdd(dyn, (unsigned long long)RB_TD_DYN_CHUNK);
    left = (uint32_t)min((uint64_t)RB_TD_DYN_CHUNK, nh - i0);
  }
}

// ---------------------------------------------------------------------------
// bottom-up

// First frontier neighbour among 8 probed ones (absent: u = -1 with b = 0, a
// prefix-valid chunk): sets par to it and returns the checks the scan order
// spends on the chunk -- up to the hit, else every valid entry.  Branch-free
// (a mask, predicated moves) instead of a dependent per-entry chain.
__device__ __forceinline__ uint32_t chunk_first_hit(const int32_t (&u)[8], const uint32_t (&b)[8], int32_t& par) {
  uint32_t hm = 0, nv = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    hm |= ((b[t] >> (u[t] & 31)) & 1u) << t;
    nv += u[t] >= 0 ? 1u : 0u;
  }
  int32_t first = -1;
#pragma unroll
  for (int t = 7; t >= 0; --t)
    if ((hm >> t) & 1u) first = u[t];
  if (hm) par = first;
  return hm ? (uint32_t)__ffs(hm) : nv;
}

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

// Offset in a bottom-up warp step (KB words) of lane l's k-th vertex: lane l
// owns bit l of every word, so each of the step's loads is one coalesced
// warp access.  (Measured and rejected: lane l owning KB consecutive
// vertices with 16-byte loads -- s26 bottom-up 265 -> 311 us/root, four times
// the L1 wavefronts.)
template <int KB>
__device__ __forceinline__ uint32_t step_off_t(uint32_t lane, uint32_t k) {
  return (k << 5) | lane;
}

template <bool kRev, int KB, bool kCollect, bool kP1 = false>
RB_LEVEL_FN void bu_level(const KParams& p, int64_t L, const uint32_t* fcur, uint32_t* fnext, uint8_t* nznext,
                         Acc& acc, uint32_t* s_found, uint32_t* s_pair, uint32_t* s_next, uint32_t* ulist,
                         unsigned long long* ulist_count, uint32_t* s_p1, bool pf = false) {
  const uint32_t lane = rb::lane_id();
  const uint64_t nw = (uint64_t)p.n_words;
  int32_t* const level_out = p.level;
  auto step_off = [](uint32_t l, uint32_t k) { return step_off_t<KB>(l, k); };
  // CTA b owns the steps b, b + gridDim.x, ... (KB words each); its warps
  // take them in order from a shared-memory counter, so a warp that meets
  // long rows does not hold up the CTA.  Software pipeline: the next step
  // is claimed and its visited words are in flight while this step works
  // (fnext is pre-zeroed, so fully visited words need no store).
  auto claim_step = [&]() -> uint64_t {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(s_next, 1u);
    k = __shfl_sync(RB_FULL, k, 0);
    return ((uint64_t)blockIdx.x + (uint64_t)k * gridDim.x) * KB;
  };
#if RB_BU_DEFER_CONT
  // Deferred continuation: rows that miss both hot checks are queued per warp
  // (s_pair, global vertex ids) and continued 32 at a time, one per lane, so a
  // step's round 1 does not wait on a few rows' dependent row-start / column
  // loads and continuation batches run with every lane busy.  Found vertices
  // set their (already written) words with reds.
  uint32_t npend = 0;
  auto continue_batch = [&](uint32_t nb, const uint32_t* q) {
    const bool mine = lane < nb;
    int64_t v = 0, s0 = 0;
    uint32_t d = 0;
    int32_t par = -1;
    uint32_t chk = 0;
    if (mine) {
      v = (int64_t)q[lane];
      d = (uint32_t)rb::ldg_i32(p.deg + v);
      s0 = rb::ldg_i64(p.rs + v);
      const int64_t e0 = s0 + d;
      const int64_t lim = d < (uint32_t)kK2 ? d : kK2;
      for (int64_t t0 = 2; par < 0 && t0 < lim; t0 += 8) {
        int32_t uu[8];
        uint32_t bb[8];
#pragma unroll
        for (int t = 0; t < 8; ++t)
          uu[t] = (t0 + t < lim) ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(s0, e0, t0 + t)) : -1;
#pragma unroll
        for (int t = 0; t < 8; ++t) bb[t] = uu[t] >= 0 ? ld_bits(fcur + (uu[t] >> 5)) : 0u;
        chk += chunk_first_hit(uu, bb, par);
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
        chk += (uint32_t)hc;
        par = hp;
      }
    }
    acc.scan += chk;
    if (mine && par >= 0) {
      const uint32_t bit = 1u << (v & 31);
      p.parent[v] = par;
      if (p.level) p.level[v] = (int32_t)(L + 1);
      red_or(fnext + (v >> 5), bit);
      red_or(p.vis + (v >> 5), bit);
      nznext[v >> 5] = 1u;
      acc.n += 1;
      acc.deg += d;
      acc.maxdeg = max(acc.maxdeg, d);
    }
  };
#endif
#if RB_BU_DEFER_CONT
  // Large-graph build: two queued rows per lane (64 per batch), both rows'
  // neighbour chunks in flight together (s26 -2%; neutral at s22).
  auto found_one = [&](int64_t v, int32_t par, uint32_t d) {
    const uint32_t bit = 1u << (v & 31);
    p.parent[v] = par;
    if (p.level) p.level[v] = (int32_t)(L + 1);
    red_or(fnext + (v >> 5), bit);
    red_or(p.vis + (v >> 5), bit);
    nznext[v >> 5] = 1u;
    acc.n += 1;
    acc.deg += d;
    acc.maxdeg = max(acc.maxdeg, d);
  };
  auto continue_batch2 = [&](const uint32_t* q) {
    const int64_t va = (int64_t)q[lane], vb = (int64_t)q[lane + 32];
    const uint32_t da = (uint32_t)rb::ldg_i32(p.deg + va), db = (uint32_t)rb::ldg_i32(p.deg + vb);
    const int64_t sa = rb::ldg_i64(p.rs + va), sb = rb::ldg_i64(p.rs + vb);
    const int64_t la = da < (uint32_t)kK2 ? da : kK2, lb = db < (uint32_t)kK2 ? db : kK2;
    int32_t pa = -1, pb = -1;
    uint32_t chk = 0;
    for (int64_t t0 = 2; (pa < 0 && t0 < la) || (pb < 0 && t0 < lb); t0 += 8) {
      int32_t ua[8], ub[8];
      uint32_t xa[8], xb[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        ua[t] = (pa < 0 && t0 + t < la) ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(sa, sa + da, t0 + t)) : -1;
        ub[t] = (pb < 0 && t0 + t < lb) ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(sb, sb + db, t0 + t)) : -1;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        xa[t] = ua[t] >= 0 ? ld_bits(fcur + (ua[t] >> 5)) : 0u;
        xb[t] = ub[t] >= 0 ? ld_bits(fcur + (ub[t] >> 5)) : 0u;
      }
      chk += chunk_first_hit(ua, xa, pa);  // (a row already found loaded no entries: 0 checks)
      chk += chunk_first_hit(ub, xb, pb);
    }
    for (int r = 0; r < 2; ++r) {
      const int64_t s0 = r ? sb : sa;
      const uint32_t d = r ? db : da;
      int32_t& par = r ? pb : pa;
      uint32_t hm = __ballot_sync(RB_FULL, par < 0 && d > (uint32_t)kK2);
      while (hm) {
        const int h = __ffs(hm) - 1;
        hm &= hm - 1;
        const int64_t hs = rb::shfl_i64(s0, h);
        const int64_t he = hs + __shfl_sync(RB_FULL, d, h);
        int64_t hc = 0;
        const int32_t hp = bu_heavy<kRev>(p, fcur, hs, he, kK2, &hc);
        if ((int)lane == h) {
          chk += (uint32_t)hc;
          par = hp;
        }
      }
    }
    acc.scan += chk;
    if (pa >= 0) found_one(va, pa, da);
    if (pb >= 0) found_one(vb, pb, db);
  };
  // One 8-neighbour chunk for each of the top nb (<= 64) queued rows, two per
  // lane; rows still open afterwards go back on the queue with their progress
  // (one byte per entry behind the queue), so every batch runs with all lanes
  // busy -- scanning a row to its end inside the batch kept the warp for the
  // longest of its 64 rows (35 % of the big level's stall samples sat in that
  // loop).  Same scan order per row, same checks.  Returns the rows re-queued.
  uint8_t* const s_prog = reinterpret_cast<uint8_t*>(s_pair + (kPairWords - kPairCap / 4));
  auto continue_chunk = [&](uint32_t nb) -> uint32_t {
    const uint32_t base = npend - nb;
    const bool oa = lane < nb, ob = lane + 32 < nb;
    const int64_t va = oa ? (int64_t)s_pair[base + lane] : 0, vb = ob ? (int64_t)s_pair[base + lane + 32] : 0;
    const uint32_t ga = oa ? s_prog[base + lane] : 0u, gb = ob ? s_prog[base + lane + 32] : 0u;
    __syncwarp();  // every entry is read before survivors are written back
    const uint32_t da = oa ? (uint32_t)rb::ldg_i32(p.deg + va) : 0u, db = ob ? (uint32_t)rb::ldg_i32(p.deg + vb) : 0u;
    const int64_t sa = oa ? rb::ldg_i64(p.rs + va) : 0, sb = ob ? rb::ldg_i64(p.rs + vb) : 0;
    const int64_t la = da < (uint32_t)kK2 ? da : kK2, lb = db < (uint32_t)kK2 ? db : kK2;
    const int64_t ta = 2 + 8 * (int64_t)ga, tb = 2 + 8 * (int64_t)gb;
    int32_t pa = -1, pb = -1;
    uint32_t chk = 0;
    {
      int32_t ua[8], ub[8];
      uint32_t xa[8], xb[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        ua[t] = (oa && ta + t < la) ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(sa, sa + da, ta + t)) : -1;
        ub[t] = (ob && tb + t < lb) ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(sb, sb + db, tb + t)) : -1;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        xa[t] = ua[t] >= 0 ? ld_bits(fcur + (ua[t] >> 5)) : 0u;
        xb[t] = ub[t] >= 0 ? ld_bits(fcur + (ub[t] >> 5)) : 0u;
      }
      chk += chunk_first_hit(ua, xa, pa);
      chk += chunk_first_hit(ub, xb, pb);
    }
    const bool ra = oa && pa < 0 && ta + 8 < la, rb_ = ob && pb < 0 && tb + 8 < lb;  // more chunks to go
    for (int r = 0; r < 2; ++r) {  // rows past kK2 checks: the whole warp finishes them now
      const int64_t s0 = r ? sb : sa;
      const uint32_t d = r ? db : da;
      int32_t& par = r ? pb : pa;
      const bool open = r ? (ob && !rb_) : (oa && !ra);
      uint32_t hm = __ballot_sync(RB_FULL, open && par < 0 && d > (uint32_t)kK2);
      while (hm) {
        const int h = __ffs(hm) - 1;
        hm &= hm - 1;
        const int64_t hs = rb::shfl_i64(s0, h);
        const int64_t he = hs + __shfl_sync(RB_FULL, d, h);
        int64_t hc = 0;
        const int32_t hp = bu_heavy<kRev>(p, fcur, hs, he, kK2, &hc);
        if ((int)lane == h) {
          chk += (uint32_t)hc;
          par = hp;
        }
      }
    }
    acc.scan += chk;
    if (pa >= 0) found_one(va, pa, da);
    if (pb >= 0) found_one(vb, pb, db);
    const uint32_t ma = __ballot_sync(RB_FULL, ra), mb = __ballot_sync(RB_FULL, rb_);
    const uint32_t lt = (1u << lane) - 1u;
    if (ra) {
      const uint32_t pos = base + __popc(ma & lt);
      s_pair[pos] = (uint32_t)va;
      s_prog[pos] = (uint8_t)(ga + 1);
    }
    if (rb_) {
      const uint32_t pos = base + __popc(ma) + __popc(mb & lt);
      s_pair[pos] = (uint32_t)vb;
      s_prog[pos] = (uint8_t)(gb + 1);
    }
    __syncwarp();
    return (uint32_t)(__popc(ma) + __popc(mb));
  };
#endif
  auto load_vis = [&](uint64_t w) -> uint32_t {
    return (w < nw && lane < KB) ? __ldcg(p.vis + w + lane) : 0xffffffffu;
  };
  // lane l owns vertex (w + k) * 32 + l of each of the step's KB words: bit k = that vertex is unvisited
  auto act_of = [&](uint32_t vwx) -> uint32_t {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < KB; ++k) m |= ((~__shfl_sync(RB_FULL, vwx, k) >> lane) & 1u) << k;
    return m;
  };
  // round-1 records of a step: the two scan-first neighbours and the degree, coalesced, all loads in flight
  auto load_rec = [&](uint64_t w, uint32_t m, int2 (&hvx)[KB], uint32_t (&dgx)[KB]) {
    const int64_t vb = (int64_t)w * 32 + lane;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      hvx[k] = make_int2(-1, -1);
      dgx[k] = 0;
      if ((m >> k) & 1u) {
        hvx[k] = __ldg(p.hot + vb + 32 * k);
        dgx[k] = (uint32_t)rb::ldg_i32(p.deg + vb + 32 * k);
      }
    }
  };
  // Levels with most vertices still unvisited (pf): the next step's hot pairs
  // and degrees (KB * 32 consecutive vertices: 2 KB + 1 KB at KB = 8) are
  // prefetched into L2 one step ahead, one 128-byte line per lane, so round 1
  // pays an L2 hit instead of a DRAM round trip (s26 bottom-up 237.4 -> 234.0
  // us/root; also prefetching the row starts, which only continued rows read,
  // costs 250 us: the level is sensitive to every extra DRAM byte).
  auto prefetch_step = [&](uint64_t w) {
#if RB_BU_PREFETCH
    if (pf && (int64_t)(w + KB) * 32 <= p.n_dev) {
      constexpr uint32_t kHotLines = KB * 32 * 8 / 128, kDegLines = KB * 32 * 4 / 128;
      const char* a = nullptr;
      if (lane < kHotLines)
        a = reinterpret_cast<const char*>(p.hot + w * 32) + lane * 128;
      else if (lane < kHotLines + kDegLines)
        a = reinterpret_cast<const char*>(p.deg + w * 32) + (lane - kHotLines) * 128;
      if (a) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
#endif
  };
  uint64_t w_nx = claim_step();
  uint32_t vw_nx = load_vis(w_nx);
  while (w_nx < nw) {
    const uint64_t w0 = w_nx;
    const uint32_t vw = vw_nx;
    w_nx = claim_step();
    vw_nx = load_vis(w_nx);
    prefetch_step(w_nx);
    const uint32_t actm = act_of(vw);
    if (!__any_sync(RB_FULL, actm != 0)) continue;
    int2 hv[KB];
    uint32_t dg[KB];
    load_rec(w0, actm, hv, dg);
    const int64_t vbase = (int64_t)w0 * 32 + lane;
    uint32_t hb0[KB], hb1[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      hb0[k] = hv[k].x >= 0 ? ld_bits(fcur + (hv[k].x >> 5)) : 0u;
      hb1[k] = hv[k].y >= 0 ? ld_bits(fcur + (hv[k].y >> 5)) : 0u;
    }
    // branch-free resolution, 32-bit step-local counters
    uint32_t foundm = 0, needm = 0, checks = 0, dsum = 0, dmax = 0, h0m = 0;
    int32_t* const par_out = p.parent + vbase;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      // inactive vertices (and missing neighbours) hold hv = -1, hb = 0 and dg = 0,
      // so no activity test is needed: a -1 neighbour tests bit 31 of a zero word
      const bool h0 = (hb0[k] >> (hv[k].x & 31)) & 1u;
      const bool h1 = !h0 && ((hb1[k] >> (hv[k].y & 31)) & 1u);
      const bool found = h0 || h1;
      if (kP1) h0m += h0 ? 1u : 0u;
      checks += h0 ? 1u : min(dg[k], 2u);  // (a second-neighbour hit implies dg >= 2)
      rb::st_if(par_out + 32 * k, h0 ? hv[k].x : hv[k].y, found);  // predicated store, no branch
      foundm |= (uint32_t)found << k;
      needm |= (uint32_t)(!found && dg[k] > 2u) << k;
      dsum += found ? dg[k] : 0u;
      dmax = max(dmax, found ? dg[k] : 0u);
    }
    constexpr int kFirst = 2;
    if (foundm && level_out) {
#pragma unroll
      for (int k = 0; k < KB; ++k) rb::st_if(level_out + vbase + 32 * k, (int32_t)(L + 1), (foundm >> k) & 1u);
    }
    acc.n += __popc(foundm);
    acc.deg += dsum;
    acc.maxdeg = max(acc.maxdeg, dmax);
    if (kP1 && s_p1) {  // partitioned modes: first-neighbour hits (bu_reduced pass 1)
      const uint32_t c = __reduce_add_sync(RB_FULL, h0m);
      if (lane == 0 && c) atomicAdd(s_p1, c);
    }
    uint32_t* fm_s = s_found;  // KB words: found bits per word (the non-deferred path)
    uint32_t my_fm = 0;         // lane k < KB: the found bits of word k
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const uint32_t fm = __ballot_sync(RB_FULL, (foundm >> k) & 1u);
      if (lane == (uint32_t)k) my_fm = fm;
      if ((kCollect || !RB_BU_DEFER_CONT) && lane == 0) fm_s[k] = fm;
    }
    // Longer rows that did not hit: the (lane, k) pairs are compacted across
    // the warp through shared memory so every lane continues one row (up to
    // kK2 checks, 4 per step); rows longer still are finished by the whole warp.
    const uint32_t np = __popc(needm);
    const uint32_t incl = rb::warp_incl_scan(np);
    const uint32_t npairs = __shfl_sync(RB_FULL, incl, 31);
#if RB_BU_DEFER_CONT
    if (!kCollect) {
      if (npairs) {  // queue the rows (global ids) behind the pending ones
        uint32_t pos = npend + incl - np;
#pragma unroll
        for (int k = 0; k < KB; ++k) {  // (unrolled, predicated: no divergent loop)
          const bool q = (needm >> k) & 1u;
          if (q) {
            s_pair[pos] = (uint32_t)(w0 * 32 + step_off(lane, k));
            s_prog[pos] = 0;
          }
          pos += q ? 1u : 0u;
        }
        npend += npairs;
      }
      __syncwarp();
      if (lane < (uint32_t)KB && my_fm) {  // round-1 results: the warp owns these words
        fnext[w0 + lane] = my_fm;
        nznext[w0 + lane] = 1u;
        p.vis[w0 + lane] = vw | my_fm;
      }
      __syncwarp();
      if constexpr (KB == 8 && RB_BU_REQUEUE) {
        while (npend >= 64) npend = npend - 64 + continue_chunk(64);  // two rows per lane, one chunk each
      } else if constexpr (KB == 8) {
        while (npend >= 64) {  // two rows per lane
          npend -= 64;
          continue_batch2(s_pair + npend);
          __syncwarp();
        }
      } else {
        while (npend >= 32) {  // full batches from the top of the queue
          npend -= 32;
          continue_batch(32, s_pair + npend);
          __syncwarp();
        }
      }
      acc.scan += checks;
      continue;
    }
#endif
    if (npairs) {
      uint32_t pos = incl - np;
      for (uint32_t m = needm; m; m &= m - 1) {
        const uint32_t k = __ffs(m) - 1;
        s_pair[pos] = (min(dg[k], 0xffffffu) << 8) | step_off(lane, k);  // degree saturates at 2^24-1
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
          // contiguous 8-neighbour chunks of the row: one sector per lane per step
          for (int64_t t0 = kFirst; par < 0 && t0 < lim; t0 += 8) {
            int32_t uu[8];
            uint32_t bb[8];
#pragma unroll
            for (int t = 0; t < 8; ++t)
              uu[t] = (t0 + t < lim) ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(s0, e0, t0 + t)) : -1;
#pragma unroll
            for (int t = 0; t < 8; ++t) bb[t] = uu[t] >= 0 ? ld_bits(fcur + (uu[t] >> 5)) : 0u;
            checks += chunk_first_hit(uu, bb, par);
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
          if (p.level) p.level[v] = (int32_t)(L + 1);
          acc.n += 1;
          acc.deg += d;
          acc.maxdeg = max(acc.maxdeg, d);
          atomicOr(fm_s + (idx >> 5), 1u << (idx & 31));
        }
      }
      __syncwarp();
    }
    // next-frontier words (pre-zeroed), their summary bytes and the visited
    // words: the warp owns them; lane k < KB writes word k (it holds vis word k)
    __syncwarp();  // lane 0's (and the continuation's) fm_s updates are visible
    if (lane < (uint32_t)KB) {
      const uint32_t fm = fm_s[lane];
      if (fm) {
        fnext[w0 + lane] = fm;
        nznext[w0 + lane] = 1u;
        p.vis[w0 + lane] = vw | fm;
      }
    }
    if (kCollect) {  // the vertices still unvisited after this level: the next level's sparse list
      const uint32_t un = lane < (uint32_t)KB ? ~(vw | fm_s[lane]) : 0u;
      const uint32_t c = __popc(un);
      const uint32_t incl = rb::warp_incl_scan(c);
      const uint32_t tot = __shfl_sync(RB_FULL, incl, 31);
      if (tot) {
        unsigned long long b = 0;
        if (lane == 31) b = atomicAdd(ulist_count, (unsigned long long)tot) & kSliceMask;
        uint32_t pos = (uint32_t)__shfl_sync(RB_FULL, b, 31) + incl - c;
        for (uint32_t y = un; y; y &= y - 1) ulist[pos++] = (uint32_t)((w0 + lane) * 32 + (__ffs(y) - 1));
      }
    }
    __syncwarp();
    acc.scan += checks;
  }
#if RB_BU_DEFER_CONT
  if constexpr (KB == 8 && RB_BU_REQUEUE && !kCollect) {
    while (npend) {
      const uint32_t nb = npend < 64u ? npend : 64u;
      npend = npend - nb + continue_chunk(nb);
    }
  } else {
    if (!kCollect && npend > 32) {
      npend -= 32;
      continue_batch(32, s_pair + npend);
      __syncwarp();
    }
    if (!kCollect && npend) continue_batch(npend, s_pair);
  }
#endif
}

// Sparse bottom-up (late levels, at most one unvisited vertex in 256): the
// unvisited vertices are kept in a list (written by the bitmap level before,
// bu_level<.., kCollect>; each sparse level rewrites its survivors) and
// checked one per lane -- the hot pair, then the rest of the row in scan
// order, 8 neighbours per step.  Found vertices set their bits with reds
// (words are shared between threads here).  Replaces the 8-word warp steps
// of bu_level, whose bitmap pass costs ~20 us at scale 26 however few
// vertices are left.

// Check the listed vertices (one per lane); survivors go to `lout`.  Rows
// are scanned per lane up to kK2 checks, longer ones by the whole warp
// (bu_heavy), as in bu_level.
template <bool kRev>
__device__ void bu_sparse_pass(const KParams& p, int64_t L, const uint32_t* fcur, uint32_t* fnext, uint8_t* nznext,
                               const uint32_t* lin, uint64_t n, uint32_t* lout, unsigned long long* lcount, Acc& acc) {
  const uint32_t lane = rb::lane_id();
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads + (threadIdx.x & ~31u); base < n; base += stride) {
    const uint64_t t = base + lane;
    int32_t v = -1, par = -1;
    uint32_t d = 0, checks = 0;
    bool live = false;
    int64_t s0 = 0;
    if (t < n) {
      v = (int32_t)__ldcg(lin + t);
      if (!((ld_bits(p.vis + (v >> 5)) >> (v & 31)) & 1u)) {  // (a top-down level may have found it since)
        live = true;
        const int2 h = __ldg(p.hot + v);
        d = (uint32_t)rb::ldg_i32(p.deg + v);
        const uint32_t b0 = h.x >= 0 ? ld_bits(fcur + (h.x >> 5)) : 0u;
        const uint32_t b1 = h.y >= 0 ? ld_bits(fcur + (h.y >> 5)) : 0u;
        if (h.x >= 0 && ((b0 >> (h.x & 31)) & 1u)) {
          par = h.x;
          checks = 1;
        } else if (h.y >= 0 && ((b1 >> (h.y & 31)) & 1u)) {
          par = h.y;
          checks = 2;
        } else {
          checks = min(d, 2u);
          if (d > 2u) {
            s0 = rb::ldg_i64(p.rs + v);
            const int64_t e0 = s0 + d;
            const int64_t lim = d < (uint32_t)kK2 ? d : kK2;
            for (int64_t t0 = 2; par < 0 && t0 < lim; t0 += 8) {
              int32_t uu[8];
              uint32_t bb[8];
#pragma unroll
              for (int k = 0; k < 8; ++k)
                uu[k] = (t0 + k < lim) ? rb::ldg_i32(p.col_bu + bu_idx<kRev>(s0, e0, t0 + k)) : -1;
#pragma unroll
              for (int k = 0; k < 8; ++k) bb[k] = uu[k] >= 0 ? ld_bits(fcur + (uu[k] >> 5)) : 0u;
              checks += chunk_first_hit(uu, bb, par);
            }
          }
        }
      }
    }
    uint32_t hm = __ballot_sync(RB_FULL, live && par < 0 && d > (uint32_t)kK2);
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
    const bool keep = live && par < 0;
    if (par >= 0) {
      const uint32_t bit = 1u << (v & 31);
      p.parent[v] = par;
      if (p.level) p.level[v] = (int32_t)(L + 1);
      red_or(p.vis + (v >> 5), bit);
      red_or(fnext + (v >> 5), bit);
      nznext[v >> 5] = 1u;
      acc.n += 1;
      acc.deg += d;
      acc.maxdeg = max(acc.maxdeg, d);
    }
    acc.scan += checks;
    const uint32_t km = __ballot_sync(RB_FULL, keep);
    if (km) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(lcount, (unsigned long long)__popc(km)) & kSliceMask;  // (bit 40: list valid)
      b = __shfl_sync(RB_FULL, b, 0);
      if (keep) lout[b + __popc(km & ((1u << lane) - 1u))] = (uint32_t)v;
    }
  }
}

// ---------------------------------------------------------------------------

// Block reduction of the level counters: warp partials go to shared memory,
// warp 0 combines them with shuffles and one lane per counter issues the
// global atomic (fire-and-forget).  The caller's grid barrier follows.
__device__ __forceinline__ void block_add3(unsigned long long* red, const Acc& a, Slot* out) {
  const unsigned long long A = rb::warp_sum_u64(a.n);
  const unsigned long long B = rb::warp_sum_u64(a.deg);
  const unsigned long long C = rb::warp_sum_u64(a.scan);
  const uint32_t M = __reduce_max_sync(RB_FULL, a.maxdeg);
  const uint32_t w = threadIdx.x >> 5, lane = rb::lane_id();
  if (lane == 0) {
    red[w * 4 + 0] = A;
    red[w * 4 + 1] = B;
    red[w * 4 + 2] = C;
    red[w * 4 + 3] = M;
  }
  __syncthreads();
  if (w == 0) {
    const unsigned long long sa = rb::warp_sum_u64(lane < kWarps ? red[lane * 4 + 0] : 0ull);
    const unsigned long long sb = rb::warp_sum_u64(lane < kWarps ? red[lane * 4 + 1] : 0ull);
    const unsigned long long sc = rb::warp_sum_u64(lane < kWarps ? red[lane * 4 + 2] : 0ull);
    const uint32_t sm = __reduce_max_sync(RB_FULL, lane < kWarps ? (uint32_t)red[lane * 4 + 3] : 0u);
    if (lane == 0 && sa) atomicAdd(&out->n_next, sa);
    if (lane == 1 && sb) atomicAdd(&out->deg_next, sb);
    if (lane == 2 && sc) atomicAdd(&out->scanned, sc);
    if (lane == 3 && sm) atomicMax(&out->maxdeg, (unsigned long long)sm);
  }
}


// ---------------------------------------------------------------------------
// Partition live bounds (partition.py:143-171 shrink_bounds, applied by
// bu_reduced before and after each pass; the bounds persist within a
// traversal).  Shrinking is monotone in the visited set, so the bounds after
// a bottom-up level equal one shrink of the partition's full range against
// the visited bitmap after the level: lo = the first 512-vertex block that is
// not all visited, hi = the end of the last one (aligned ends; the final,
// unaligned end stays).  Blocks past n_dev are isolated (premarked visited)
// and the block holding the reference bitmap's padding (n_full % 512 != 0)
// is never full; both are settled in live_total.

__device__ void live_pass(const KParams& p) {
  const uint32_t lane = rb::lane_id();
  const int64_t nb = (p.n_dev + 511) / 512;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t b0 = (uint64_t)blockIdx.x * kThreads + (threadIdx.x & ~31u); b0 < (uint64_t)nb; b0 += stride) {
    const int64_t b = (int64_t)(b0 + lane);
    bool nonfull = false;
    if (b < nb) {
      const uint4* w = reinterpret_cast<const uint4*>(p.vis + b * 16);
      const uint4 a = __ldcg(w), c = __ldcg(w + 1), d = __ldcg(w + 2), e = __ldcg(w + 3);
      nonfull = (a.x & a.y & a.z & a.w & c.x & c.y & c.z & c.w & d.x & d.y & d.z & d.w & e.x & e.y & e.z & e.w) !=
                0xffffffffu;
    }
    // partition of block b: last bound <= b (bounds ascending, n_parts small)
    int32_t part = -1;
    if (nonfull) {
      int32_t lo = 0, hi = (int32_t)p.n_parts;  // part_blk[lo] <= b < part_blk[hi]
      while (hi - lo > 1) {
        const int32_t mid = (lo + hi) >> 1;
        if (__ldg(p.part_blk + mid) <= b) lo = mid; else hi = mid;
      }
      part = lo;
    }
    const uint32_t m = __ballot_sync(RB_FULL, nonfull);
    if (!m) continue;
    const int32_t p0 = __shfl_sync(RB_FULL, part, __ffs(m) - 1);
    if (__all_sync(RB_FULL, !nonfull || part == p0)) {  // one partition: one min / max per warp
      if ((int)lane == __ffs(m) - 1) atomicMin(p.part_first + p0, (int32_t)b);
      if ((int)lane == 31 - __clz(m)) atomicMax(p.part_last + p0, (int32_t)b);
    } else if (nonfull) {
      atomicMin(p.part_first + part, (int32_t)b);
      atomicMax(p.part_last + part, (int32_t)b);
    }
  }
}

// One warp (CTA 0): sum of the shrunk partition sizes; re-arms first / last.
__device__ void live_total(const KParams& p, long long* s_out) {
  const uint32_t lane = rb::lane_id();
  const int64_t tail = (p.n_full % 512) ? (p.n_full - 1) / 512 : -1;  // never-full padding block
  const int64_t nb_dev = (p.n_dev + 511) / 512;
  long long sum = 0;
  for (int64_t q = lane; q < p.n_parts; q += 32) {
    const int64_t b0 = p.part_blk[q], b1 = p.part_blk[q + 1];
    int64_t f = __ldcg(p.part_first + q), l = __ldcg(p.part_last + q);
    if (f == INT32_MAX) f = INT64_MAX;
    // blocks [nb_dev, b1) hold only isolated vertices (full); the block with the
    // reference bitmap's zero padding is never full, wherever n_dev ends
    (void)nb_dev;
    if (tail >= b0 && tail < b1) {
      f = min(f, tail);
      l = max(l, tail);
    }
    const bool last = q == p.n_parts - 1;
    const int64_t end = last ? p.n_full : b1 * 512;
    if (end % 512 == 0)
      sum += (l >= 0) ? (l + 1 - f) * 512 : 0;
    else
      sum += end - f * 512;  // the unaligned final end never moves (and its block is never full)
    p.part_first[q] = INT32_MAX;
    p.part_last[q] = -1;
  }
  sum = (long long)rb::warp_sum_u64((unsigned long long)sum);
  if (lane == 0) *s_out = sum;
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Solo levels: the first top-down levels of a traversal usually hold a
// handful of rows (the source, then its neighbours).  A whole-grid level
// costs a full pass of scans plus a grid barrier (~7 us); CTA 0 instead runs
// such levels alone with its frontier in shared memory and __syncthreads as
// the level barrier, while the other CTAs wait at one grid barrier.  The
// bitmaps end up exactly as the grid path leaves them: claims set the
// next-frontier bits (+ summary), and the buffer the grid would zero ahead
// holds exactly the frontier of level L-1, whose bits are cleared from its
// list.  Entry only at the start of a traversal (level 0, frontier {src}).

constexpr int kSoloCap = kThreads < 1024 ? kThreads : 1024;  // frontier vertices held in shared memory (one row per thread)
constexpr int64_t kSoloMf = 4096;  // frontier edges of a solo level

struct SoloShared {
  unsigned long long deg;  // deg_next
  unsigned int nn, maxd;   // n_next, max degree of the next frontier
  unsigned int total;      // edges of the current frontier
};

// Block-wide exclusive scan of one value per thread (kThreads <= 1024).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* warp_tot, uint32_t* total) {
  const uint32_t lane = rb::lane_id(), w = threadIdx.x >> 5;
  const uint32_t incl = rb::warp_incl_scan(x);
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    const uint32_t t = lane < (uint32_t)kWarps ? warp_tot[lane] : 0u;
    const uint32_t ti = rb::warp_incl_scan(t);
    warp_tot[lane] = ti - t;
    if (lane == 31) *total = ti;
  }
  __syncthreads();
  return warp_tot[w] + incl - x;
}

// Runs in CTA 0 only, with the frontier of level L listed in smem[kSoloCap,
// kSoloCap + nf) and the buffer fb[(L+2)%3] zero.  On return the state
// variables describe the first level that is not run solo (or the end of
// the traversal).  (Tried: re-entering solo mode for the tail levels of a
// traversal -- their cost is the same chain of dependent misses either way,
// so the entry pass and barrier made them slower.)
__device__ __forceinline__ void solo_levels(const KParams& p, uint32_t* smem, SoloShared* sh, uint32_t* warp_tot, int64_t& L,
                            int& dir, int64_t& nf, int64_t& mf, int64_t& mu, int64_t& done, bool& hubs,
                            uint64_t& t_prev, int64_t& reached) {
  const uint32_t tid = threadIdx.x;
  uint32_t* qp = smem;                 // frontier of level L-1
  uint32_t* qc = smem + kSoloCap;      // frontier of level L
  uint32_t* qn = smem + 2 * kSoloCap;  // frontier of level L+1
  uint32_t* sOff = smem + 3 * kSoloCap;
  int64_t* sS = reinterpret_cast<int64_t*>(smem + 4 * kSoloCap);
  uint32_t np = 0, nc = (uint32_t)nf;
  __syncthreads();
  while (true) {
    const int r0 = (int)(L % 3), r1 = (r0 + 1) % 3, r2 = (r0 + 2) % 3;
    uint32_t* fnext = fb_of(p, r1);
    uint8_t* nznext = nz_of(p, r1);
    uint32_t* fold = fb_of(p, r2);
    uint8_t* nzold = nz_of(p, r2);
    if (tid == 0) {
      sh->nn = 0u;
      sh->deg = 0ull;
      sh->maxd = 0u;
    }
    if (tid < sizeof(Slot) / 8) reinterpret_cast<unsigned long long*>(p.slots + r1)[tid] = 0ull;
    // rows of the current frontier
    uint32_t d = 0;
    if (tid < nc) {
      int64_t s0;
      int32_t n0, n1;
      ld_vinfo(p, qc[tid], s0, d, n0, n1);
      sS[tid] = s0;
    }
    const uint32_t off = block_excl_scan(tid < nc ? d : 0u, warp_tot, &sh->total);
    const uint32_t total = sh->total;
    if (tid < nc) sOff[tid] = off;
    __syncthreads();
    // clear the frontier of level L-1 (the buffer the grid would zero ahead)
    for (uint32_t i = tid; i < np; i += kThreads) {
      const uint32_t u = qp[i];
      atomicAnd(fold + (u >> 5), ~(1u << (u & 31)));
      nzold[u >> 5] = 0u;  // the word holds only level L-1 bits: it is zero now
    }
    __syncthreads();
    // edges, block-balanced: edge e belongs to the last row with sOff <= e
    const bool probe = 2 * mu < p.m_directed;
    for (uint32_t e0 = 0; e0 < total; e0 += kThreads) {  // same trip count for every lane
      const uint32_t e = e0 + tid;
      bool won = false;
      int32_t w = 0;
      uint32_t dw = 0;
      if (e < total) {
        uint32_t lo = 0, hi = nc;  // upper_bound(sOff, e) - 1
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (sOff[mid] <= e)
            lo = mid;
          else
            hi = mid;
        }
        const int32_t v = (int32_t)qc[lo];
        w = rb::ldg_i32(p.td_col + sS[lo] + (e - sOff[lo]));
        const uint32_t bit = 1u << (w & 31);
        if (!(probe && (ld_bits(p.vis + (w >> 5)) & bit))) {
          dw = (uint32_t)rb::ldg_i32(p.deg + w);
          won = !(atomicOr(p.vis + (w >> 5), bit) & bit);
          if (won) {
            p.parent[w] = v;
            if (p.level) p.level[w] = (int32_t)(L + 1);
            red_or(fnext + (w >> 5), bit);
            nznext[w >> 5] = 1u;
          }
        }
      }
      // warp-aggregated queue append and counters (one shared atomic per warp)
      const uint32_t lane = rb::lane_id();
      const uint32_t wm = __ballot_sync(RB_FULL, won);
      if (wm) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&sh->nn, (uint32_t)__popc(wm));
        base = __shfl_sync(RB_FULL, base, 0);
        const uint32_t pos = base + __popc(wm & ((1u << lane) - 1u));
        if (won && pos < (uint32_t)kSoloCap) qn[pos] = (uint32_t)w;
        const unsigned long long ds = rb::warp_sum_u64(won ? dw : 0u);
        const uint32_t dm = __reduce_max_sync(RB_FULL, won ? dw : 0u);
        if (lane == 0) {
          atomicAdd(&sh->deg, ds);
          atomicMax(&sh->maxd, dm);
        }
      }
    }
    __syncthreads();
    // counters, record, policy (engine.py:587-596) -- same as the grid path
    const int64_t n_next = (int64_t)sh->nn;
    const int64_t deg_next = (int64_t)sh->deg;
    hubs = sh->maxd > kLightDeg;
    if (tid == 32) {
      const uint64_t t_now = globaltimer();
      rb_level_record r;
      r.level = L;
      r.direction = dir;
      r.n_f = nf;
      r.m_f = mf;
      r.m_u = mu;
      r.scanned_edges = (int64_t)total;
      r.t_ns = (int64_t)(t_now - t_prev);
      r.n_next = n_next;
      r.t_queue_ns = 0;
      r.reserved = 0;  // executed direction (solo levels: top-down)
      r.pass1_hits = -1;
      r.live_vertices = -1;
      r.claimed = -1;
      r.reserved2 = 0;
      p.rec[done] = r;
      t_prev = t_now;
    }
    mu -= deg_next;
    mf = deg_next;
    nf = n_next;
    reached += n_next;
    int ndir = 0;
    if (p.hybrid) {
      if (dir == 0)
        ndir = (mf * (int64_t)p.alpha > mu) ? 1 : 0;
      else
        ndir = (nf * (int64_t)p.beta < p.n_policy) ? 0 : 1;
    }
    dir = ndir;
    ++L;
    ++done;
    __syncthreads();  // everyone has read sh before the next level resets it
    if (!(nf > 0 && dir == 0 && nf <= kSoloCap && mf <= kSoloMf && done < p.max_levels)) {
      // hand the next frontier to the grid as a list (its first level then
      // skips the summary walk): complete when it fits the shared buffer
      for (int64_t i = tid; i < nf && nf <= kSoloCap; i += kThreads) p.solo_q[i] = qn[i];
      break;
    }
    uint32_t* t = qp;
    qp = qc;
    qc = qn;
    qn = t;
    np = nc;
    nc = (uint32_t)nf;
  }
}

// kPart: the partitioned modes' record fields (pass-1 hits, live bounds);
// a separate instantiation so the fast kernels carry none of that code.
template <bool kRev, int KB, bool kPart>
__global__ void __launch_bounds__(kThreads, RB_MINB) bfs_persistent(KParams p) {
  // Sparse bottom-up lists only in the large-graph build (8-word steps): at
  // scale 22 the tail levels are latency floors either way and the extra
  // code costs the small-graph kernel ~2% (measured).
  constexpr bool kSparseOK = RB_SPARSE_ALL || KB == 8;
  __shared__ unsigned long long s_red[kWarps * 4];
  __shared__ unsigned long long s_ctr[5];  // [4]: the unvisited list of the last level (bit 40: valid | count)
  __shared__ uint32_t s_bu_found[kWarps][kBU];
  __shared__ uint32_t s_bu_pair[kWarps][kPairWords];
  __shared__ uint32_t s_bu_next[2];  // bottom-up: next step of this CTA (level parity)
  __shared__ SoloShared s_solo;
  __shared__ uint32_t s_wtot[32];
  __shared__ uint32_t s_p1;          // first-neighbour hits of this CTA in the current bottom-up level
  __shared__ long long s_live;       // live_vertices of the current level (CTA 0)
  if (p.dbg && threadIdx.x == 0 && blockIdx.x == 0) p.dbg[kDbgPhase + 63 * 8 + 0] = globaltimer();  // kernel entry
  __shared__ long long s_mf0;  // deg(src) at a traversal start (one load per CTA, not per thread)
  if (threadIdx.x == 0) {
    s_bu_next[0] = s_bu_next[1] = 0u;
    s_p1 = 0u;
    s_ctr[4] = 0ull;  // no unvisited list yet
    if (p.mf0 < 0) s_mf0 = (long long)rb::ld_relaxed_u64((const unsigned long long*)&p.fin->mf);
  }
  __syncthreads();
  const uint32_t nblocks = gridDim.x;
  const uint64_t gtid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const uint64_t gthreads = (uint64_t)nblocks * kThreads;

  int64_t L = p.level0;
  int dir = (int)p.dir0;
  int need_compact = (int)p.need_compact0;
  int64_t nf = p.nf0, mf = p.mf0, mu = p.mu0;
  if (mf < 0) {  // engine.py:536-538; deg(src) was stored by the reset kernel
    mf = (int64_t)s_mf0;
    mu = p.m_directed - mf;
  }
  int64_t done = 0;
  int64_t reached = p.reached0;
  uint32_t epoch = 0;
  bool solo_hubs = false;
  __shared__ unsigned long long s_fin[9];  // the state after the solo levels ([8]: frontier list length)
  if (threadIdx.x == 0) s_fin[0] = ~0ull, s_fin[8] = 0ull;
  __syncthreads();
  if (p.from_fin && mf <= kSoloMf) {
    // traversal start with a small frontier: CTA 0 runs the first levels
    // alone, the grid waits at one barrier and picks up the state
    if (blockIdx.x == 0) {
      uint64_t t0 = globaltimer();
      bool h = false;
      if (threadIdx.x == 0) (&s_bu_pair[0][0])[kSoloCap] = (uint32_t)p.src;  // the level-0 frontier list
      solo_levels(p, &s_bu_pair[0][0], &s_solo, s_wtot, L, dir, nf, mf, mu, done, h, t0, reached);
      if (threadIdx.x == 0) {
        p.fin->reached = reached;
        p.fin->levels_done = done;
        p.fin->L = L;
        p.fin->dir = dir;
        p.fin->nf = nf;
        p.fin->mf = mf;
        p.fin->mu = mu;
        p.fin->pad = h ? 1 : 0;
        p.fin->pad2 = (nf > 0 && nf <= kSoloCap) ? nf : 0;  // p.solo_q holds the frontier
      }
    }
    {
      // the state after the solo levels: thread 0 of each CTA fetches it
      // into shared memory (all threads loading it would queue on one line)
      const unsigned long long* const src[9] = {
          (const unsigned long long*)&p.fin->levels_done, (const unsigned long long*)&p.fin->L,
          (const unsigned long long*)&p.fin->dir,         (const unsigned long long*)&p.fin->nf,
          (const unsigned long long*)&p.fin->mf,          (const unsigned long long*)&p.fin->mu,
          (const unsigned long long*)&p.fin->pad,         (const unsigned long long*)&p.fin->reached,
          (const unsigned long long*)&p.fin->pad2};
      rb::grid_barrier_fetch<9>(p.bar, nblocks, epoch, src, s_fin);
      done = (int64_t)s_fin[0];
      L = (int64_t)s_fin[1];
      dir = (int)s_fin[2];
      nf = (int64_t)s_fin[3];
      mf = (int64_t)s_fin[4];
      mu = (int64_t)s_fin[5];
      solo_hubs = s_fin[6] != 0;
      reached = (int64_t)s_fin[7];
    }
    need_compact = dir == 0;
  }
  int r0 = (int)(L % 3);
  // does the current frontier hold a row longer than kLightDeg?  Level 0: the
  // source's degree; a continuation launch conservatively assumes yes.
  bool hubs = p.hubs0 >= 0 ? p.hubs0 != 0 : ((p.mf0 < 0) ? (mf > (int64_t)kLightDeg) : true);
  if (p.from_fin && done > 0) hubs = solo_hubs;
  uint64_t t_prev = 0, t_queue = 0;
  if (blockIdx.x == 0 && threadIdx.x == 32) t_prev = globaltimer();

  while (done < p.max_levels && nf > 0) {
    // rotating buffers: r0 = L % 3 (kept incrementally, no 64-bit modulo)
    const int r1 = r0 == 2 ? 0 : r0 + 1, r2 = r1 == 2 ? 0 : r1 + 1;
    Slot* out = p.slots + r0;
    Slot* in = p.slots + r2;
    const uint32_t* fcur = p.fcur_ext ? p.fcur_ext : fb_of(p, r0);
    uint32_t* fnext = fb_of(p, r1);
    uint32_t* fzero = fb_of(p, r2);
    uint8_t* nzzero = nz_of(p, r2);
    // zero ahead: next level's fnext bitmap (+ summary) and the counter slot of level L+1
    const uint64_t tA = globaltimer();
    for (uint64_t i = gtid; i < (uint64_t)p.n_words / 4; i += gthreads)
      reinterpret_cast<uint4*>(fzero)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (uint64_t i = gtid; i < (uint64_t)p.n_words / 16; i += gthreads)
      reinterpret_cast<uint4*>(nzzero)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (blockIdx.x == 0 && threadIdx.x < sizeof(Slot) / 8)
      reinterpret_cast<unsigned long long*>(p.slots + r1)[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) s_bu_next[(L + 1) & 1] = 0u;  // the next level's counter (idle during this one)

    // Execution direction.  The level keeps the reference policy's label
    // (records, next decisions); the work is done the cheaper way.  Same next
    // frontier either way; any frontier neighbour is a valid parent.
    //  * early (most edges unvisited), labelled bottom-up: executed top-down
    //    when the frontier edges are few against the unvisited ones (m_f <=
    //    m_u / kExecAlpha) -- most bottom-up scans would run to the row end;
    //  * late (most edges visited), either label: a latency cost model in
    //    picoseconds -- top-down pays per frontier row and edge, bottom-up
    //    pays a bitmap pass (step chain per warp) plus per unvisited vertex.
    //    After the big bottom-up levels the frontier is millions of leaves
    //    but only thousands of vertices are still unvisited: bottom-up wins
    //    5x; the tail frontiers of a few thousand rows go top-down.
    int xdir = dir;
    bool sparse = false;   // few unvisited vertices left: sparse bottom-up over the previous level's list
    bool collect = false;  // bitmap bottom-up that lists the survivors (the next level may go sparse)
    const unsigned long long ul_code = s_ctr[4];  // from the previous level's closing fetch
    if (p.exec_opt) {
      if (2 * mu > p.m_directed) {
        if (dir == 1 && mf * p.exec_alpha <= mu) xdir = 0;
      } else {
        const int64_t U = p.n_active > reached ? p.n_active - reached : 0;
        const int64_t t_td = kTdFixPs + nf * kTdRowPs + mf * kTdEdgePs;
        if constexpr (kSparseOK) {
          sparse = p.bu_sparse && (ul_code >> 40) && U * kSparseRatio <= p.n_dev;
          collect = p.bu_sparse && !sparse && U * kListRatio <= p.n_dev;
        }
        const int64_t t_bu = kBuFixPs +
                             (sparse ? kBuSparsePs : (p.n_words / KB) * kBuStepPs / ((int64_t)nblocks * kWarps)) +
                             U * kBuVertPs + min(mu, 8 * U) * kBuCheckPs;
        xdir = t_td <= t_bu ? 0 : 1;
      }
    }
    Acc acc{0, 0, 0, 0u};
    if (xdir == 0) {
      QEnt* hq = (L & 1) ? p.hq1 : p.hq0;
      uint32_t* hs = (L & 1) ? p.hs1 : p.hs0;
      TdCtx c;
      c.p = &p;
      c.L = L;
      c.fcur = fcur;
      c.fnext = fnext;
      c.nznext = nz_of(p, r1);
      // probe the visited word before the atomic when most targets are
      // already taken: late levels, or big levels whose frontier rows share
      // many neighbours (RB_PROBE_MF: from this many frontier edges)
      c.probe = 2 * mu < p.m_directed || mf >= p.probe_mf;
      c.defer = mf >= p.defer_mf;
      // a small frontier with hub rows: its light rows join phase B too, so
      // phase A (which ends at a grid barrier) is only find rows + publish
      c.hub_min = (hubs && nf <= kLightToB) ? kTinyDeg : kLightDeg;
      if (c.defer) {  // snapshot of vis at the level start (see count_next)
        for (uint64_t i = gtid; i < (uint64_t)p.n_words / 4; i += gthreads)
          reinterpret_cast<uint4*>(fnext)[i] = __ldcg(reinterpret_cast<const uint4*>(p.vis) + i);
        rb::grid_barrier(p.bar, nblocks, epoch);
        if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0 && done < 64) p.dbg[kDbgPhase + done * 8 + 0] = globaltimer();
      }
      // phase A: frontier rows from the bitmap; hub rows become slices in hq
      if (s_fin[8] && done == (int64_t)s_fin[0])  // the first grid level after the solo levels
        td_rows_list(c, p.solo_q, (uint32_t)s_fin[8], hq, hs, &in->hq_count, acc, s_bu_pair[threadIdx.x >> 5]);
      else if (nf >= kDenseFrontier)
        td_rows_words<KB == 8>(c, hq, hs, &in->hq_count, acc, s_bu_pair[threadIdx.x >> 5], &s_bu_next[L & 1]);
      else
        td_rows_items(c, p.nzcur_ext ? p.nzcur_ext : nz_of(p, r0), hq, hs, &in->hq_count, acc,
                      s_bu_pair[threadIdx.x >> 5]);
      if (p.dbg && (threadIdx.x & 31) == 0 && done < 64)
        p.dbg[kDbgWarpA + ((uint64_t)done * gridDim.x + blockIdx.x) * kWarps + (threadIdx.x >> 5)] = globaltimer();
      if (hubs) {  // phase B only if some frontier row has more than kLightDeg edges
        {
          const unsigned long long* const src[1] = {&in->hq_count};
          rb::grid_barrier_fetch<1>(p.bar, nblocks, epoch, src, s_ctr);
        }
        if (blockIdx.x == 0 && threadIdx.x == 32) t_queue = globaltimer() - t_prev;
        if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0 && done < 64) p.dbg[kDbgPhase + done * 8 + 1] = globaltimer();
        td_hubs(c, hq, hs, s_ctr[0] >> 40, s_ctr[0] & kSliceMask, RB_TD_DYN_MINK > 0 ? &in->pad2 : nullptr, acc);
        if (p.dbg && (threadIdx.x & 31) == 0 && done < 64)
          p.dbg[kDbgWarpB + ((uint64_t)done * gridDim.x + blockIdx.x) * kWarps + (threadIdx.x >> 5)] = globaltimer();
      }
      if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0 && done < 64) p.dbg[kDbgPhase + done * 8 + 2] = globaltimer();
      if (c.defer) {
        rb::grid_barrier(p.bar, nblocks, epoch);  // every claim of the level has landed
        if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0 && done < 64) p.dbg[kDbgPhase + done * 8 + 3] = globaltimer();
        count_next<KB == 8>(p, fnext, nz_of(p, r1), acc);
        if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0 && done < 64) p.dbg[kDbgPhase + done * 8 + 4] = globaltimer();
      }
    } else {
      const uint32_t wib = threadIdx.x >> 5;
      uint32_t* const lout = (L & 1) ? p.ul1 : p.ul0;  // the list this level leaves for the next
      if (kSparseOK && sparse) {  // over the list the previous level left (its survivors go to lout)
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&out->ul_count, 1ull << 40);  // list valid flag
        bu_sparse_pass<kRev>(p, L, fcur, fnext, nz_of(p, r1), (L & 1) ? p.ul0 : p.ul1, ul_code & kSliceMask, lout,
                             &out->ul_count, acc);
      } else if (kSparseOK && collect) {  // bitmap pass that also lists the vertices left unvisited
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&out->ul_count, 1ull << 40);
        bu_level<kRev, KB, true>(p, L, fcur, fnext, nz_of(p, r1), acc, s_bu_found[wib], s_bu_pair[wib],
                                 &s_bu_next[L & 1], lout, &out->ul_count, nullptr);
      } else
        bu_level<kRev, KB, false, kPart>(p, L, fcur, fnext, nz_of(p, r1), acc, s_bu_found[wib], s_bu_pair[wib],
                                         &s_bu_next[L & 1], nullptr, nullptr, (kPart && p.count_p1) ? &s_p1 : nullptr,
                                         !kPart && 2 * reached < p.n_active);
    }
    if (p.dbg && (threadIdx.x & 31) == 0 && done < 64)  // RB_DEBUG_TS: per-warp end of work
      p.dbg[kDbgWarpBase + ((uint64_t)done * gridDim.x + blockIdx.x) * kWarps + (threadIdx.x >> 5)] = globaltimer();
    block_add3(s_red, acc, out);  // (its __syncthreads also orders the CTA's s_p1 updates)
    if (kPart && threadIdx.x == 0 && s_p1) {  // re-armed here: the next adds follow the closing grid barrier
      atomicAdd(&out->pad3, (unsigned long long)s_p1);
      s_p1 = 0u;
    }
    const uint64_t tB = globaltimer();
    {
      if constexpr (kSparseOK) {
        const unsigned long long* const src[5] = {&out->n_next, &out->deg_next, &out->maxdeg, &out->scanned,
                                                  &out->ul_count};
        rb::grid_barrier_fetch<5>(p.bar, nblocks, epoch, src, s_ctr);
      } else {
        const unsigned long long* const src[4] = {&out->n_next, &out->deg_next, &out->maxdeg, &out->scanned};
        rb::grid_barrier_fetch<4>(p.bar, nblocks, epoch, src, s_ctr);
      }
    }
    if (p.dbg && threadIdx.x == 0 && done < 64) {  // RB_DEBUG_TS: per-block phase timestamps
      const uint64_t tC = globaltimer();
      unsigned long long* d = p.dbg + ((uint64_t)done * gridDim.x + blockIdx.x) * 4;
      d[0] = tA;
      d[1] = tB;
      d[2] = tC;
    }

    const int64_t n_next = (int64_t)s_ctr[0];
    const int64_t deg_next = (int64_t)s_ctr[1];
    hubs = s_ctr[2] > kLightDeg;
    if (kPart && p.n_parts > 0 && xdir == 1) {  // PartitionSet.live_total() after this bottom-up level
      live_pass(p);
      rb::grid_barrier(p.bar, nblocks, epoch);
      if (blockIdx.x == 0 && (threadIdx.x >> 5) == 1) live_total(p, &s_live);
    }
    if (p.dbg && threadIdx.x == 0 && done < 64) p.dbg[((uint64_t)done * gridDim.x + blockIdx.x) * 4 + 3] = globaltimer() + (uint64_t)(n_next & 0) + (uint64_t)(deg_next & 0) + (hubs ? 0 : 0);
    if (blockIdx.x == 0 && threadIdx.x == 32) {
      const uint64_t t_now = globaltimer();
      rb_level_record r;
      r.level = L;
      r.direction = dir;
      r.n_f = nf;
      r.m_f = mf;
      r.m_u = mu;
      r.scanned_edges = (int64_t)s_ctr[3];
      r.t_ns = (int64_t)(t_now - t_prev);
      r.n_next = n_next;
      r.t_queue_ns = (int64_t)t_queue;
      r.reserved = xdir;  // executed direction
      r.pass1_hits = (kPart && p.count_p1 && xdir == 1) ? (int64_t)rb::ld_relaxed_u64(&out->pad3) : -1;
      r.live_vertices = (kPart && p.n_parts > 0 && xdir == 1) ? (int64_t)s_live : -1;
      r.claimed = -1;
      r.reserved2 = 0;
      p.rec[done] = r;
      t_queue = 0;
      t_prev = t_now;
    }
    // engine.py:587-596
    mu -= deg_next;
    mf = deg_next;
    nf = n_next;
    reached += n_next;
    int ndir = 0;
    if (p.hybrid) {
      if (dir == 0)
        ndir = (mf * (int64_t)p.alpha > mu) ? 1 : 0;  // == (m_f > m_u / alpha) exactly for m_u < 2^46
      else
        ndir = (nf * (int64_t)p.beta < p.n_policy) ? 0 : 1;  // == (n_f < n / beta)
    }
    need_compact = ndir == 0;  // queues are always rebuilt from the frontier bitmap
    dir = ndir;
    ++L;
    ++done;
    r0 = r0 == 2 ? 0 : r0 + 1;
  }
  if (p.dbg && threadIdx.x == 0 && blockIdx.x == 0) p.dbg[kDbgPhase + 63 * 8 + 1] = globaltimer();  // kernel exit
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.fin->levels_done = done;
    p.fin->L = L;
    p.fin->dir = dir;
    p.fin->need_compact = need_compact;
    p.fin->nf = nf;
    p.fin->mf = mf;
    p.fin->mu = mu;
    p.fin->reached = reached;
  }
}

// Per-root reset in one launch (engine.py:526-539): parents (and levels)
// -1, frontier bitmaps and summaries 0, visited = the isolated/padding
// template, counters 0, and the source seeded by the thread that owns it.
__global__ void bfs_reset_all(KParams p, const uint32_t* vis_template, int64_t src) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < p.n_dev; i += stride) {
    p.parent[i] = i == src ? (int32_t)src : -1;
    if (p.level) p.level[i] = i == src ? 0 : -1;
  }
  const int64_t sw = src >> 5;
  const uint32_t sb = 1u << (src & 31);
  for (int64_t i = t0; i < p.n_words; i += stride) {
    p.fb0[i] = i == sw ? sb : 0u;
    p.fb1[i] = 0u;
    p.fb2[i] = 0u;
    p.nz0[i] = i == sw ? 1u : 0u;
    p.nz1[i] = 0u;
    p.nz2[i] = 0u;
    p.vis[i] = __ldg(vis_template + i) | (i == sw ? sb : 0u);
  }
  if (t0 < (int64_t)(3 * sizeof(Slot) / 8)) reinterpret_cast<unsigned long long*>(p.slots)[t0] = 0ull;
  if (t0 < 16) p.bar[t0] = 0u;
  if (t0 == 0) p.fin->mf = (long long)(p.rs[src + 1] - p.rs[src]);  // deg(src) for the traversal's first level
}

// Per-root reset tail: source seeds (engine.py:526-539).
__global__ void bfs_seed(KParams p, int64_t src) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  p.parent[src] = (int32_t)src;
  if (p.level) p.level[src] = 0;
  p.fb0[src >> 5] |= 1u << (src & 31);
  p.nz0[src >> 5] = 1u;
  p.vis[src >> 5] |= 1u << (src & 31);
}

// vinfo[v] = {row start, degree, first two neighbours} (top-down row record)
__global__ void make_vinfo(const int64_t* rs, const int32_t* col, int64_t n, VInfo* vi) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = rs[v], e = rs[v + 1];
    const uint64_t d = (uint64_t)(e - s);
    VInfo r;
    r.s_lo = (uint32_t)s;
    r.sd = ((uint32_t)((uint64_t)s >> 32) << 24) | (uint32_t)(d < kVdSat ? d : kVdSat);
    r.n0 = d > 0 ? col[s] : -1;
    r.n1 = d > 1 ? col[s + 1] : -1;
    vi[v] = r;
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

// deg8[v] = min(deg[v], 255) for v < n, 0 up to n_pad
__global__ void make_deg8(const int32_t* deg, int64_t n, int64_t n_pad, uint8_t* deg8) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_pad; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = v < n ? deg[v] : 0;
    deg8[v] = (uint8_t)(d < 255 ? d : 255);
  }
}

// *out += number of zero bits of words[0, n) (unvisited-at-start vertices)
__global__ void count_zero_bits(const uint32_t* words, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += (unsigned long long)__popc(~words[i]);
  c = rb::warp_sum_u64(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// nz[i] = words[i] != 0
__global__ void make_nz(const uint32_t* words, uint8_t* nz, int64_t n_words) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_words; j += (int64_t)gridDim.x * blockDim.x)
    nz[j] = words[j] != 0u ? 1u : 0u;
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


// ---------------------------------------------------------------------------
// 1D-partitioned traversal with the exchange on the device.
//
// Rank r owns global vertices [v_lo, v_lo + n_dev): its CSR rows (global
// column ids; bottom-up), the transpose slice (the owned neighbours of every
// global vertex; top-down), its visited words and parents -- exactly the
// rb_bfs_create_part engine.  Instead of the host driving one launch per
// level, ONE persistent launch per rank runs the whole level loop:
//   1. the level's local work (top-down claims through the transpose slice or
//      bottom-up finds over the owned rows, both against the GLOBAL frontier
//      bitmap xg[L % 3]) into the local next-frontier words;
//   2. publish: the nonzero local next-frontier words (and their summary
//      bytes) are stored straight into EVERY rank's xg[(L + 1) % 3] at this
//      rank's word offset -- peer memory over NVLink (CUDA IPC mappings) --
//      and the level totals {n_next, deg_next, maxdeg, scanned} into every
//      rank's counter slot [L & 1][r];
//   3. one cross-GPU barrier (system-scope release adds on every peer's
//      counter, acquire spin on the own one), then every rank sums the slots:
//      the same global counters drive update_traversal_policy on all ranks.
// xg is triple-buffered: during level L a rank zeroes its xg[(L + 2) % 3],
// which nobody reads any more (level L - 1's frontier) and nobody writes
// before the barrier that ends level L.  No host round trip per level.
//
// Emulation (one GPU, the profiling guide's rule for fewer GPUs than ranks):
// bfs_dist_emu runs all ranks' data in ONE cooperative launch, the ranks'
// level work one after the other with the whole grid, the publish identical,
// and the cross-rank barrier a grid barrier.

constexpr int kMaxWorld = 8;

struct XParams {
  int32_t world, rank;
  int64_t n_words_glob;
  int64_t w_lo;                                // this rank's first global word (v_lo / 32)
  uint32_t* xg[3];                             // own global frontier bitmaps
  uint8_t* xnz[3];                             // their summaries (one byte per word)
  unsigned long long* slot;                    // own counter slots [2][kMaxWorld][4]
  uint32_t* xbar;                              // own cross-rank barrier counter (never reset)
  uint32_t* peer_xg[kMaxWorld][3];             // every rank's xg / xnz / slot / xbar as seen from here
  uint8_t* peer_xnz[kMaxWorld][3];
  unsigned long long* peer_slot[kMaxWorld];
  uint32_t* peer_xbar[kMaxWorld];
  uint32_t xepoch0;                            // cross barriers completed before this launch
};

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct DistShared {
  unsigned long long red[kWarps * 4];
  unsigned long long ctr[5];
  uint32_t bu_found[kWarps][kBU];
  uint32_t bu_pair[kWarps][kPairWords];
  uint32_t next_step;
};

// One rank's work of level L (local claims / finds), ending with a grid
// barrier that leaves this rank's level totals in sm.ctr[0..3] (n_next,
// deg_next, maxdeg, scanned).  nblocks = the grid; epoch = its barrier count.
template <bool kRev, int KB>
__device__ void dist_body(const KParams& p, const XParams& x, int64_t L, int xdir, bool hubs, int64_t nf,
                          int64_t mf, int64_t mu, uint32_t& epoch, DistShared& sm) {
  const int r0 = (int)(L % 3), r1 = (r0 + 1) % 3, r2 = (r0 + 2) % 3;
  const uint32_t nblocks = gridDim.x;
  const uint64_t gtid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const uint64_t gthreads = (uint64_t)nblocks * kThreads;
  Slot* out = p.slots + r0;
  Slot* in = p.slots + r2;
  const uint32_t* fcur = x.xg[r0];
  uint32_t* fnext = fb_of(p, r1);
  // zero ahead: the local fnext of level L+1, the global frontier of level L+2, the next counter slot
  for (uint64_t i = gtid; i < (uint64_t)p.n_words / 4; i += gthreads) {
    reinterpret_cast<uint4*>(fb_of(p, r2))[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (uint64_t i = gtid; i < (uint64_t)p.n_words / 16; i += gthreads)
    reinterpret_cast<uint4*>(nz_of(p, r2))[i] = make_uint4(0u, 0u, 0u, 0u);
  for (uint64_t i = gtid; i < (uint64_t)x.n_words_glob / 4; i += gthreads)
    reinterpret_cast<uint4*>(x.xg[r2])[i] = make_uint4(0u, 0u, 0u, 0u);
  for (uint64_t i = gtid; i < (uint64_t)x.n_words_glob / 16; i += gthreads)
    reinterpret_cast<uint4*>(x.xnz[r2])[i] = make_uint4(0u, 0u, 0u, 0u);
  if (blockIdx.x == 0 && threadIdx.x < sizeof(Slot) / 8)
    reinterpret_cast<unsigned long long*>(p.slots + r1)[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) sm.next_step = 0u;
  __syncthreads();
  Acc acc{0, 0, 0, 0u};
  if (xdir == 0) {
    QEnt* hq = (L & 1) ? p.hq1 : p.hq0;
    uint32_t* hs = (L & 1) ? p.hs1 : p.hs0;
    TdCtx c;
    c.p = &p;
    c.L = L;
    c.fcur = fcur;
    c.fnext = fnext;
    c.nznext = nz_of(p, r1);
    c.probe = 2 * mu < p.m_directed || mf >= p.probe_mf;
    c.defer = mf >= p.defer_mf;
    c.hub_min = (hubs && nf <= kLightToB) ? kTinyDeg : kLightDeg;
    if (c.defer) {
      for (uint64_t i = gtid; i < (uint64_t)p.n_words / 4; i += gthreads)
        reinterpret_cast<uint4*>(fnext)[i] = __ldcg(reinterpret_cast<const uint4*>(p.vis) + i);
      rb::grid_barrier(p.bar, nblocks, epoch);
    }
    if (nf >= kDenseFrontier)
      td_rows_words<KB == 8>(c, hq, hs, &in->hq_count, acc, sm.bu_pair[threadIdx.x >> 5], &sm.next_step);
    else
      td_rows_items(c, x.xnz[r0], hq, hs, &in->hq_count, acc, sm.bu_pair[threadIdx.x >> 5]);
    if (hubs) {
      const unsigned long long* const src[1] = {&in->hq_count};
      rb::grid_barrier_fetch<1>(p.bar, nblocks, epoch, src, sm.ctr);
      td_hubs(c, hq, hs, sm.ctr[0] >> 40, sm.ctr[0] & kSliceMask, nullptr, acc);
    }
    if (c.defer) {
      rb::grid_barrier(p.bar, nblocks, epoch);
      count_next<KB == 8>(p, fnext, nz_of(p, r1), acc);
    }
  } else {
    const uint32_t wib = threadIdx.x >> 5;
    bu_level<kRev, KB, false>(p, L, fcur, fnext, nz_of(p, r1), acc, sm.bu_found[wib], sm.bu_pair[wib],
                              &sm.next_step, nullptr, nullptr, nullptr);
  }
  block_add3(sm.red, acc, out);
  const unsigned long long* const src[4] = {&out->n_next, &out->deg_next, &out->maxdeg, &out->scanned};
  rb::grid_barrier_fetch<4>(p.bar, nblocks, epoch, src, sm.ctr);
}

// Publish this rank's level-L results to every rank (peer stores; see above).
__device__ void dist_publish(const KParams& p, const XParams& x, int64_t L, const unsigned long long* tot) {
  const int r1 = (int)((L + 1) % 3);
  const uint32_t* fnext = fb_of(p, r1);
  const uint64_t gtid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const uint64_t gthreads = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = gtid; i < (uint64_t)p.n_words / 4; i += gthreads) {
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(fnext) + i);
    if (!(v.x | v.y | v.z | v.w)) continue;  // the targets are zeroed ahead
    const uint32_t nzb = (v.x ? 1u : 0u) | (v.y ? 0x100u : 0u) | (v.z ? 0x10000u : 0u) | (v.w ? 0x1000000u : 0u);
    const uint64_t gw = (uint64_t)x.w_lo + 4 * i;  // w_lo % 4 == 0: 16-byte chunks never straddle two ranks
    for (int q = 0; q < x.world; ++q) {
      reinterpret_cast<uint4*>(x.peer_xg[q][r1] + gw)[0] = v;
      reinterpret_cast<uint32_t*>(x.peer_xnz[q][r1] + gw)[0] = nzb;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 4 * (uint32_t)x.world) {
    const int q = threadIdx.x >> 2, k = threadIdx.x & 3;
    x.peer_slot[q][((L & 1) * kMaxWorld + x.rank) * 4 + k] = tot[k];
  }
}

// Global level totals: sum (max for maxdeg) of every rank's slot [L & 1].
__device__ __forceinline__ void dist_totals(const XParams& x, int64_t L, unsigned long long* out4) {
  unsigned long long a = 0, b = 0, m = 0, c = 0;
  for (int q = 0; q < x.world; ++q) {
    const unsigned long long* sl = x.slot + ((L & 1) * kMaxWorld + q) * 4;
    a += rb::ld_relaxed_u64(sl + 0);
    b += rb::ld_relaxed_u64(sl + 1);
    m = max(m, (unsigned long long)rb::ld_relaxed_u64(sl + 2));
    c += rb::ld_relaxed_u64(sl + 3);
  }
  out4[0] = a;
  out4[1] = b;
  out4[2] = m;
  out4[3] = c;
}

// Grid barrier whose release waits for every rank (real multi-GPU): CTA 0
// arrives last, after the cross-rank barrier.  All CTAs fenced their peer
// stores at system scope before arriving.
__device__ void grid_barrier_cross(const XParams& x, uint32_t* bar, uint32_t nblocks, uint32_t& epoch,
                                   uint32_t& xepoch) {
  ++epoch;
  ++xepoch;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t target = epoch * nblocks;
    if (blockIdx.x == 0) {
      while ((int32_t)(rb::ld_relaxed_u32(bar) - (target - 1)) < 0) {
      }
      __threadfence_system();
      for (int q = 0; q < x.world; ++q) red_release_sys_add(x.peer_xbar[q], 1u);
      const uint32_t xt = xepoch * (uint32_t)x.world;
      while ((int32_t)(ld_acquire_sys_u32(x.xbar) - xt) < 0) {
      }
      rb::red_release_add(bar, 1u);
    } else {
      rb::red_release_add(bar, 1u);
      while ((int32_t)(rb::ld_relaxed_u32(bar) - target) < 0) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Level record + policy (engine.py:587-596), identical on every rank.
struct DistState {
  int64_t L, nf, mf, mu, done;
  int dir;
  bool hubs;
  uint64_t t_prev;
};

__device__ __forceinline__ void dist_advance(const KParams& p, bool write_rec, int xdir, const unsigned long long* g,
                                             DistState& st) {
  const int64_t n_next = (int64_t)g[0], deg_next = (int64_t)g[1];
  if (write_rec && blockIdx.x == 0 && threadIdx.x == 32) {
    const uint64_t t_now = globaltimer();
    rb_level_record r;
    r.level = st.L;
    r.direction = st.dir;
    r.n_f = st.nf;
    r.m_f = st.mf;
    r.m_u = st.mu;
    r.scanned_edges = (int64_t)g[3];
    r.t_ns = (int64_t)(t_now - st.t_prev);
    r.n_next = n_next;
    r.t_queue_ns = 0;
    r.reserved = xdir;
    r.pass1_hits = -1;
    r.live_vertices = -1;
    r.claimed = -1;
    r.reserved2 = 0;
    p.rec[st.done] = r;
    st.t_prev = t_now;
  }
  st.mu -= deg_next;
  st.mf = deg_next;
  st.nf = n_next;
  st.hubs = g[2] > kLightDeg;
  int ndir = 0;
  if (p.hybrid) {
    if (st.dir == 0)
      ndir = (st.mf * (int64_t)p.alpha > st.mu) ? 1 : 0;
    else
      ndir = (st.nf * (int64_t)p.beta < p.n_policy) ? 0 : 1;
  }
  st.dir = ndir;
  ++st.L;
  ++st.done;
}

__device__ __forceinline__ int dist_exec_dir(const KParams& p, const DistState& st) {
  // early levels labelled bottom-up with few frontier edges run top-down (the
  // single-GPU crossover, every input global so all ranks agree)
  if (p.exec_opt && st.dir == 1 && 2 * st.mu > p.m_directed && st.mf * p.exec_alpha <= st.mu) return 0;
  return st.dir;
}

__device__ __forceinline__ void dist_finish(const KParams& p, const DistState& st, uint32_t xepoch) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.fin->levels_done = st.done;
    p.fin->L = st.L;
    p.fin->dir = st.dir;
    p.fin->nf = st.nf;
    p.fin->mf = st.mf;
    p.fin->mu = st.mu;
    p.fin->pad = xepoch;  // cross barriers completed (the next launch's xepoch0)
  }
}

// Real multi-GPU: one launch per rank, the whole level loop on the device.
template <bool kRev, int KB>
__global__ void __launch_bounds__(kThreads, 1) bfs_dist(KParams p, XParams x) {
  __shared__ DistShared sm;
  __shared__ unsigned long long s_tot[4];
  uint32_t epoch = 0, xepoch = x.xepoch0;
  DistState st{0, 1, p.mf0, p.mu0, 0, 0, p.mf0 > (int64_t)kLightDeg, 0};
  if (blockIdx.x == 0 && threadIdx.x == 32) st.t_prev = globaltimer();
  // every rank's reset (its xg[1] zeroed, its seed) is done before anyone publishes
  grid_barrier_cross(x, p.bar, gridDim.x, epoch, xepoch);
  while (st.done < p.max_levels && st.nf > 0) {
    const int xdir = dist_exec_dir(p, st);
    dist_body<kRev, KB>(p, x, st.L, xdir, st.hubs, st.nf, st.mf, st.mu, epoch, sm);
    dist_publish(p, x, st.L, sm.ctr);
    grid_barrier_cross(x, p.bar, gridDim.x, epoch, xepoch);
    if (threadIdx.x == 0) dist_totals(x, st.L, s_tot);
    __syncthreads();
    dist_advance(p, x.rank == 0, xdir, s_tot, st);
  }
  dist_finish(p, st, xepoch);
}

// One GPU: the ranks' data in one cooperative launch (ranks run in turn).
struct EmuParams {
  int32_t world;
  const KParams* kp;  // device arrays of world entries
  const XParams* xp;
};

template <bool kRev, int KB>
__global__ void __launch_bounds__(kThreads, 1) bfs_dist_emu(EmuParams e) {
  __shared__ DistShared sm;
  __shared__ unsigned long long s_tot[4];
  uint32_t epoch = 0;
  const KParams& p0 = e.kp[0];
  DistState st{0, 1, p0.mf0, p0.mu0, 0, 0, p0.mf0 > (int64_t)kLightDeg, 0};
  if (blockIdx.x == 0 && threadIdx.x == 32) st.t_prev = globaltimer();
  while (st.done < p0.max_levels && st.nf > 0) {
    const int xdir = dist_exec_dir(p0, st);
    for (int g = 0; g < e.world; ++g) {
      dist_body<kRev, KB>(e.kp[g], e.xp[g], st.L, xdir, st.hubs, st.nf, st.mf, st.mu, epoch, sm);
      dist_publish(e.kp[g], e.xp[g], st.L, sm.ctr);
    }
    rb::grid_barrier(p0.bar, gridDim.x, epoch);  // the cross-rank barrier of the emulation
    if (threadIdx.x == 0) dist_totals(e.xp[0], st.L, s_tot);
    __syncthreads();
    dist_advance(p0, true, xdir, s_tot, st);
  }
  for (int g = 0; g < e.world; ++g) dist_finish(e.kp[g], st, 0);
}

// Per-root reset of the exchange buffers: xg[0] = the source bit, summary;
// xg[1], xg[2], summaries and the slots zero.
__global__ void dist_reset_x(XParams x, int64_t src_glob) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t sw = src_glob >> 5;
  for (int64_t i = t0; i < x.n_words_glob; i += stride) {
    x.xg[0][i] = i == sw ? (1u << (src_glob & 31)) : 0u;
    x.xg[1][i] = 0u;
    x.xg[2][i] = 0u;
    x.xnz[0][i] = i == sw ? 1u : 0u;
    x.xnz[1][i] = 0u;
    x.xnz[2][i] = 0u;
  }
  if (t0 < 2 * kMaxWorld * 4) x.slot[t0] = 0ull;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

constexpr int kMaxChunks = 32;  // async result path: parent copy chunks

struct rb_bfs {
  KParams kp;
  rb_bfs_params prm;
  int64_t n_dev;
  int64_t n_words;
  uint32_t* vis_template;   // isolated + padding premarked
  uint32_t* pad_mask;       // padding bits only
  int2* hot;
  uint8_t* deg8;
  VInfo* vinfo;
  VInfo* td_vinfo;  // partitioned engines only
  int64_t n_glob;
  int blocks;
  int sms;
  int bu_reverse;
  int64_t source;
  std::vector<rb_level_record> recs;
  int64_t levels_per_launch;  // kRecCap; RB_LEVELS_PER_LAUNCH=1 gives one launch per level (profiling)
  cudaEvent_t ev_start, ev_end;  // bracket all launches of one traversal
  cudaEvent_t ev_chunk[kMaxChunks + 1];  // async result path: parent chunks, then the small copies
  bool launched;
  bool solo;      // run the first small levels in one CTA (solo_levels); RB_SOLO=0 disables
  bool exec_opt;  // executed direction by cost; RB_EXEC_OPT=0 disables
  int64_t probe_mf;
  int64_t defer_mf;
  void* stream;
  bool exact;            // RB_PART_EXACT: run the labelled direction every level
  int32_t* part_dev;     // [n_parts + 1 block bounds | first | last]
  // device-side exchange (rb_bfs_xchg_*): partitioned engines only
  XParams x;
  void* xblock;                    // xg[3] | xnz[3] | slots | xbar, one allocation (IPC-exported)
  size_t xbytes;
  std::vector<void*> x_opened;     // peers' blocks mapped with cudaIpcOpenMemHandle
  int64_t src_deg;                 // deg(source) of the current distributed traversal
};

// The traversal kernel of an engine: scan direction x bottom-up step width.
static const void* bfs_kernel(const rb_bfs* h) {
  bool small = h->n_dev <= kSmallGraph;
  if (const char* env = getenv("RB_KB")) small = atoi(env) == 4;  // tuning override
  if (h->bu_reverse)
    return small ? (const void*)bfs_persistent<true, 4, false> : (const void*)bfs_persistent<true, 8, false>;
  if (h->kp.count_p1 || h->kp.n_parts)  // partitioned modes: pass-1 hits / live bounds in the records
    return small ? (const void*)bfs_persistent<false, 4, true> : (const void*)bfs_persistent<false, 8, true>;
  return small ? (const void*)bfs_persistent<false, 4, false> : (const void*)bfs_persistent<false, 8, false>;
}

// RB_ERR_ARG with a message for a null handle / argument (every ARG path sets the error text)
static int rb_null_handle(const char* fn) {
  rb_set_error("%s: invalid (null) handle or argument", fn);
  return RB_ERR_ARG;
}

static int alloc_dev(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    rb_set_error("cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    return RB_ERR_OOM;
  }
  return RB_OK;
}

extern "C" int rb_bfs_create_part(const int64_t* d_row_starts, const int32_t* d_col, const int32_t* d_col_bu,
                                  const int32_t* d_degrees, int64_t n_dev, const uint32_t* d_isolated_words,
                                  const rb_bfs_params* params, const rb_bfs_partition* part, rb_bfs** out) {
  if (!out || !params || n_dev <= 0 || !d_row_starts || !d_col || !d_degrees) {
    rb_set_error("rb_bfs_create: invalid argument");
    return RB_ERR_ARG;
  }
  if (params->m_directed >= (1ll << 40)) {
    rb_set_error("rb_bfs_create: m_directed %lld exceeds the 40-bit row offsets of the row records",
                 (long long)params->m_directed);
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
  h->solo = true;
  if (const char* env = getenv("RB_SOLO")) h->solo = atoi(env) != 0;
  h->exec_opt = true;
  if (const char* env = getenv("RB_EXEC_OPT")) h->exec_opt = atoi(env) != 0;
  h->probe_mf = 1ll << 16;
  if (const char* env = getenv("RB_PROBE_MF")) h->probe_mf = atoll(env);
  h->defer_mf = 1ll << 20;
  if (const char* env = getenv("RB_DEFER_MF")) h->defer_mf = atoll(env);
  h->kp.probe_mf = h->probe_mf;  // also seen by rb_bfs_dist_level (which copies kp)
  h->kp.defer_mf = h->defer_mf;
  h->kp.exec_alpha = kExecAlpha;
  if (const char* env = getenv("RB_EXEC_ALPHA")) h->kp.exec_alpha = atoll(env);
  h->kp.bu_sparse = 1;
  if (const char* env = getenv("RB_BU_SPARSE")) h->kp.bu_sparse = atoll(env);
  cudaEventCreate(&h->ev_start);
  cudaEventCreate(&h->ev_end);
  for (int i = 0; i <= kMaxChunks; ++i) cudaEventCreateWithFlags(&h->ev_chunk[i], cudaEventDisableTiming);
  if (const char* env = getenv("RB_DEBUG")) h->kp.debug = atoi(env);
  h->kp.dbg = nullptr;
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
  // hub-row queue capacity (one entry per frontier row longer than kLightDeg):
  // single GPU n_dev rows (+ slack); a partition expands GLOBAL rows of the
  // transpose slice, of which fewer than td_m / kLightDeg are that long
  size_t nhub = (size_t)n_dev + (size_t)(params->m_directed / kChunk) + 64;
  if (part) {
    int64_t td_m = 0;
    if (cudaMemcpy(&td_m, part->d_td_row_starts + part->n_glob, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
      rb_set_error("rb_bfs_create: reading the transpose slice size failed");
      rb_bfs_destroy(h);
      return RB_ERR_CUDA;
    }
    nhub = std::max((size_t)n_dev, (size_t)(td_m / kLightDeg)) + (size_t)(td_m / kChunk) + 64;
  }
  int rc = RB_OK;
#define RB_ALLOC(ptr, bytes) \
  if (rc == RB_OK) rc = alloc_dev((void**)&(ptr), (bytes));
  RB_ALLOC(k.vis, wb);
  RB_ALLOC(k.fb0, wb);
  RB_ALLOC(k.fb1, wb);
  RB_ALLOC(k.fb2, wb);
  RB_ALLOC(h->vis_template, wb);
  RB_ALLOC(h->pad_mask, wb);
  RB_ALLOC(k.nz0, (size_t)h->n_words);
  RB_ALLOC(k.nz1, (size_t)h->n_words);
  RB_ALLOC(k.nz2, (size_t)h->n_words);
  RB_ALLOC(h->vinfo, (size_t)n_dev * sizeof(VInfo));
  RB_ALLOC(k.hq0, nhub * sizeof(QEnt));
  RB_ALLOC(k.hq1, nhub * sizeof(QEnt));
  RB_ALLOC(k.hs0, nhub * sizeof(uint32_t));
  RB_ALLOC(k.hs1, nhub * sizeof(uint32_t));
  RB_ALLOC(k.solo_q, kSoloCap * sizeof(uint32_t));
  RB_ALLOC(k.ul0, ((size_t)n_dev / kListRatio + 1024) * sizeof(uint32_t));
  RB_ALLOC(k.ul1, ((size_t)n_dev / kListRatio + 1024) * sizeof(uint32_t));

  RB_ALLOC(k.parent, (size_t)n_dev * 4);
  RB_ALLOC(h->hot, (size_t)n_dev * sizeof(int2));
  RB_ALLOC(h->deg8, (size_t)h->n_words * 32);
  if (params->record_levels) RB_ALLOC(k.level, (size_t)n_dev * 4);
  RB_ALLOC(k.slots, 3 * sizeof(Slot));
  RB_ALLOC(k.bar, 64);
  RB_ALLOC(k.rec, kRecCap * sizeof(rb_level_record));
  RB_ALLOC(k.fin, sizeof(Final));
  if (getenv("RB_DEBUG_TS")) RB_ALLOC(k.dbg, ((size_t)kDbgWarpBase + (size_t)64 * 1024 * kWarps) * 8);
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
  make_deg8<<<1024, 256>>>(d_degrees, n_dev, h->n_words * 32, h->deg8);
  k.deg8 = h->deg8;
  make_vinfo<<<1024, 256>>>(d_row_starts, d_col, n_dev, h->vinfo);
  k.vinfo = h->vinfo;
  k.hubs0 = -1;
  if (part) {
    const int64_t tile_g = 32 * 32 * kBU;
    k.v_lo = part->v_lo;
    k.n_words_glob = ((part->n_glob + tile_g - 1) / tile_g) * (tile_g / 32);
    if (alloc_dev((void**)&h->td_vinfo, (size_t)part->n_glob * sizeof(VInfo)) != RB_OK) {
      rb_bfs_destroy(h);
      return RB_ERR_OOM;
    }
    make_vinfo<<<1024, 256>>>(part->d_td_row_starts, part->d_td_col, part->n_glob, h->td_vinfo);
    k.td_vinfo = h->td_vinfo;
    k.td_col = part->d_td_col;
    if (cudaMemcpy(&k.td_m, part->d_td_row_starts + part->n_glob, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
      rb_set_error("rb_bfs_create: reading the transpose slice size failed");
      rb_bfs_destroy(h);
      return RB_ERR_CUDA;
    }
    k.td_rs = part->d_td_row_starts;
    h->n_glob = part->n_glob;
  } else {
    k.v_lo = 0;
    k.n_words_glob = h->n_words;
    k.td_vinfo = h->vinfo;
    k.td_col = d_col;
    k.td_m = params->m_directed;
    k.td_rs = d_row_starts;
    h->n_glob = n_dev;
  }
  if (cudaMemcpy(h->vis_template, h->pad_mask, wb, cudaMemcpyDeviceToDevice) != cudaSuccess) {
    rb_set_error("rb_bfs_create: template copy failed");
    rb_bfs_destroy(h);
    return RB_ERR_CUDA;
  }
  if (d_isolated_words) words_or<<<256, 256>>>(h->vis_template, d_isolated_words, (n_dev + 31) / 32);
  // non-isolated vertices of [0, n_dev): zero bits of the template (slot 0 is scratch here)
  cudaMemset(k.slots, 0, sizeof(Slot));
  count_zero_bits<<<256, 256>>>(h->vis_template, h->n_words, &k.slots->n_next);
  unsigned long long n_active = 0;
  cudaMemcpy(&n_active, &k.slots->n_next, 8, cudaMemcpyDeviceToHost);
  k.n_active = (int64_t)n_active;
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
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bfs_kernel(h), kThreads, 0);
  if (nb < 1) nb = 1;
  h->blocks = nb * h->sms;
  *out = h;
  return RB_OK;
}

extern "C" int rb_bfs_destroy(rb_bfs* h) {
  if (!h) return RB_OK;
  KParams& k = h->kp;
  void* ptrs[] = {k.vis, k.fb0, k.fb1, k.fb2, h->vis_template, h->pad_mask, k.hq0, k.hq1, k.hs0, k.hs1, k.ul0, k.ul1, k.solo_q, k.parent,
                  k.level, k.slots, k.bar, k.rec, k.fin, k.nz0, k.nz1, k.nz2, h->hot, h->deg8, h->vinfo, k.dbg, h->td_vinfo,
                  h->part_dev};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (void* b : h->x_opened) cudaIpcCloseMemHandle(b);
  if (h->xblock) cudaFree(h->xblock);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  for (int i = 0; i <= kMaxChunks; ++i)
    if (h->ev_chunk[i]) cudaEventDestroy(h->ev_chunk[i]);
  if (h->ev_end) cudaEventDestroy(h->ev_end);
  delete h;
  return RB_OK;
}

__global__ void part_init(int32_t* first, int32_t* last, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    first[i] = INT32_MAX;
    last[i] = -1;
  }
}

extern "C" int rb_bfs_set_partitions(rb_bfs* h, const int64_t* h_bounds, int64_t n_parts, int64_t n_full,
                                     int32_t flags) {
  if (!h || n_parts < 0 || (n_parts > 0 && !h_bounds) || n_full < h->n_dev) {
    rb_set_error("rb_bfs_set_partitions: invalid argument");
    return RB_ERR_ARG;
  }
  KParams& k = h->kp;
  if (h->part_dev) cudaFree(h->part_dev);
  h->part_dev = nullptr;
  k.n_parts = 0;
  k.part_blk = nullptr;
  k.part_first = k.part_last = nullptr;
  h->exact = (flags & RB_PART_EXACT) != 0;
  k.count_p1 = (flags & RB_PART_COUNT_PASS1) ? 1 : 0;
  k.n_full = n_full;
  if (n_parts == 0 || !(flags & RB_PART_SHRINK)) return RB_OK;
  std::vector<int32_t> blk((size_t)n_parts + 1);
  int64_t prev = 0;
  for (int64_t i = 0; i <= n_parts; ++i) {
    const int64_t b = i < n_parts ? h_bounds[i] : n_full;
    const bool bad = (i < n_parts && b % 512) || b < prev || b > n_full || (i == 0 && b != 0);
    prev = b;
    if (bad) {
      rb_set_error("rb_bfs_set_partitions: partition starts must ascend and be 512-aligned");
      return RB_ERR_ARG;
    }
    blk[(size_t)i] = (int32_t)((b + 511) / 512);
  }
  int rc = alloc_dev((void**)&h->part_dev, (size_t)(3 * n_parts + 1) * sizeof(int32_t));
  if (rc) return rc;
  RB_CUDA_TRY(cudaMemcpy(h->part_dev, blk.data(), blk.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  k.part_blk = h->part_dev;
  k.part_first = h->part_dev + n_parts + 1;
  k.part_last = k.part_first + n_parts;
  part_init<<<64, 256>>>(k.part_first, k.part_last, n_parts);
  RB_CUDA_TRY(cudaDeviceSynchronize());
  k.n_parts = n_parts;
  return RB_OK;
}

extern "C" int32_t* rb_bfs_parent_ptr(rb_bfs* h) { return h ? h->kp.parent : nullptr; }
extern "C" int32_t* rb_bfs_level_ptr(rb_bfs* h) { return h ? h->kp.level : nullptr; }
extern "C" int rb_bfs_grid(rb_bfs* h, int* blocks, int* threads) {
  if (!h) return rb_null_handle(__func__);
  if (blocks) *blocks = h->blocks;
  if (threads) *threads = kThreads;
  return RB_OK;
}

static int reset_common(rb_bfs* h, cudaStream_t s) {
  KParams& k = h->kp;
  const size_t wb = (size_t)h->n_words * 4;
  RB_CUDA_TRY(cudaMemsetAsync(k.parent, 0xff, (size_t)h->n_dev * 4, s));
  if (k.level) RB_CUDA_TRY(cudaMemsetAsync(k.level, 0xff, (size_t)h->n_dev * 4, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.fb0, 0, wb, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.fb1, 0, wb, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.fb2, 0, wb, s));  // solo levels rely on all three (see solo_levels)
  RB_CUDA_TRY(cudaMemsetAsync(k.nz0, 0, (size_t)h->n_words, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.nz1, 0, (size_t)h->n_words, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.nz2, 0, (size_t)h->n_words, s));
  RB_CUDA_TRY(cudaMemsetAsync(k.slots, 0, 3 * sizeof(Slot), s));
  RB_CUDA_TRY(cudaMemsetAsync(k.bar, 0, 64, s));
  return RB_OK;
}

extern "C" int rb_bfs_reset(rb_bfs* h, int64_t source, void* stream) {
  if (!h) return rb_null_handle(__func__);
  if (source < 0 || source >= h->n_dev) {
    rb_set_error("source %lld out of range for n_dev=%lld", (long long)source, (long long)h->n_dev);
    return RB_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  bfs_reset_all<<<h->sms * 4, 512, 0, s>>>(h->kp, h->vis_template, source);
  RB_CUDA_TRY(cudaGetLastError());
  h->source = source;
  h->recs.clear();
  return RB_OK;
}

static int launch(rb_bfs* h, cudaStream_t s, int64_t level0, int64_t dir0, int64_t need_compact0, int64_t max_levels,
                  int64_t nf0, int64_t mf0, int64_t mu0, int64_t from_fin = 0, int64_t reached0 = 1,
                  bool exec = true) {
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
  kp.from_fin = from_fin;
  // the cost-model execution (a level may run the other way) only in hybrid
  // modes: level_sync / sequential are top-down only (engine.py use_dir)
  kp.exec_opt = (exec && h->exec_opt && h->prm.hybrid && !h->exact) ? 1 : 0;
  kp.reached0 = reached0;
  kp.probe_mf = h->probe_mf;
  kp.defer_mf = h->defer_mf;
  kp.exec_alpha = h->kp.exec_alpha;
  kp.bu_sparse = h->kp.bu_sparse;
  void* args[] = {&kp};
  cudaError_t e;
  e = cudaLaunchCooperativeKernel(bfs_kernel(h), dim3(h->blocks), dim3(kThreads), args, 0, s);
  if (e != cudaSuccess) {
    rb_set_error("cooperative launch failed: %s", cudaGetErrorString(e));
    return RB_ERR_CUDA;
  }
  return RB_OK;
}

extern "C" int rb_bfs_traverse(rb_bfs* h, void* stream) {
  if (!h) return rb_null_handle(__func__);
  h->launched = true;
  h->stream = stream;
  RB_CUDA_TRY(cudaEventRecord(h->ev_start, (cudaStream_t)stream));
  int rc = launch(h, (cudaStream_t)stream, 0, 0, 0, h->levels_per_launch, 1, -1, 0, h->solo ? 1 : 0);
  if (rc) return rc;
  RB_CUDA_TRY(cudaEventRecord(h->ev_end, (cudaStream_t)stream));
  return RB_OK;
}

extern "C" int rb_bfs_results(rb_bfs* h, int32_t* parent_out, int32_t* level_out, rb_level_record* h_records,
                              int64_t cap, int64_t* n_records, void* stream) {
  if (!h) return rb_null_handle(__func__);
  if (level_out && !h->kp.level) {
    rb_set_error("rb_bfs_results: engine created without record_levels");
    return RB_ERR_ARG;
  }
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
      int rc = launch(h, s, f.L, f.dir, f.need_compact, h->levels_per_launch, f.nf, f.mf, f.mu, 0, f.reached);
      if (rc) return rc;
      RB_CUDA_TRY(cudaEventRecord(h->ev_end, s));
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

// Asynchronous result path (BfsEngine.run): enqueue the copies of the launch
// state and the first `cap` level records into caller-owned (pinned) host
// memory behind the traversal; nothing waits.  After the caller has
// synchronized the stream, rb_bfs_complete() accepts the host copies when the
// single launch finished the traversal (returns 0) -- else it returns 1 and
// the caller drains with rb_bfs_results (very deep graphs: continuations).
extern "C" int rb_bfs_results_async(rb_bfs* h, void* h_state, rb_level_record* h_records, int64_t cap,
                                    int32_t* h_parent, int32_t chunks, void* stream) {
  if (!h || !h_state || (cap > 0 && !h_records) || chunks < 0 || chunks > kMaxChunks) {
    rb_set_error("rb_bfs_results_async: invalid argument (chunks %d, allowed 0..%d)", (int)chunks, kMaxChunks);
    return RB_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  RB_CUDA_TRY(cudaMemcpyAsync(h_state, h->kp.fin, sizeof(Final), cudaMemcpyDeviceToHost, s));
  if (cap > 0)
    RB_CUDA_TRY(cudaMemcpyAsync(h_records, h->kp.rec, (size_t)(cap < kRecCap ? cap : kRecCap) * sizeof(rb_level_record),
                                cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaEventRecord(h->ev_chunk[kMaxChunks], s));  // the small copies
  if (h_parent && chunks > 0) {  // parents [0, n_dev) in `chunks` pieces, an event behind each
    const int64_t step = (h->n_dev + chunks - 1) / chunks;
    for (int32_t i = 0; i < chunks; ++i) {
      const int64_t a = i * step, b = a + step < h->n_dev ? a + step : h->n_dev;
      if (b > a)
        RB_CUDA_TRY(cudaMemcpyAsync(h_parent + a, h->kp.parent + a, (size_t)(b - a) * 4, cudaMemcpyDeviceToHost, s));
      RB_CUDA_TRY(cudaEventRecord(h->ev_chunk[i], s));
    }
  }
  return RB_OK;
}

// Wait for the async result copies: what = -1 the launch state + records,
// what = i the parent chunk i.
extern "C" int rb_bfs_wait(rb_bfs* h, int32_t what) {
  if (!h || what < -1 || what >= kMaxChunks) {
    rb_set_error("rb_bfs_wait: invalid argument (what %d, allowed -1..%d)", (int)what, kMaxChunks - 1);
    return RB_ERR_ARG;
  }
  RB_CUDA_TRY(cudaEventSynchronize(h->ev_chunk[what < 0 ? kMaxChunks : what]));
  return RB_OK;
}

extern "C" int rb_bfs_complete(rb_bfs* h, const void* h_state, const rb_level_record* h_records, int64_t cap,
                               int64_t* n_records) {
  if (!h || !h_state || !n_records) {
    rb_set_error("rb_bfs_complete: invalid argument");
    return RB_ERR_ARG;
  }
  Final f;
  memcpy(&f, h_state, sizeof(Final));
  if (!h->launched || f.nf > 0 || f.levels_done > cap) return 1;
  h->recs.assign(h_records, h_records + f.levels_done);
  h->launched = false;
  *n_records = f.levels_done;
  return RB_OK;
}

extern "C" size_t rb_bfs_state_bytes(void) { return sizeof(Final); }

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
  make_nz<<<256, 256, 0, s>>>(k.fb0, k.nz0, h->n_words);
  RB_CUDA_TRY(cudaMemcpyAsync(k.parent, d_parent_in, (size_t)h->n_dev * 4, cudaMemcpyDeviceToDevice, s));
  h->source = 0;
  rc = launch(h, s, 0, direction, direction == 0 ? 1 : 0, 1, 1, 0, 0, 0, 1, false);  // the direction asked for
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
  if (!h || iters <= 0) return rb_null_handle(__func__);
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

extern "C" int rb_bfs_debug_timestamps(rb_bfs* h, uint64_t* out, int64_t cap, int* blocks) {
  if (!h || !h->kp.dbg) return rb_null_handle(__func__);
  const int64_t n = (int64_t)kDbgWarpBase + (int64_t)64 * 1024 * kWarps;  // the whole buffer (see kDbgWarpBase / A / B)
  RB_CUDA_TRY(cudaMemcpy(out, h->kp.dbg, (size_t)(n < cap ? n : cap) * 8, cudaMemcpyDeviceToHost));
  *blocks = h->blocks;
  return RB_OK;
}

extern "C" int rb_bfs_elapsed(rb_bfs* h, double* seconds) {
  if (!h || !seconds) return rb_null_handle(__func__);
  float ms = 0.f;
  RB_CUDA_TRY(cudaEventSynchronize(h->ev_end));
  RB_CUDA_TRY(cudaEventElapsedTime(&ms, h->ev_start, h->ev_end));
  *seconds = 1e-3 * (double)ms;
  return RB_OK;
}

extern "C" int rb_bfs_create(const int64_t* d_row_starts, const int32_t* d_col, const int32_t* d_col_bu,
                             const int32_t* d_degrees, int64_t n_dev, const uint32_t* d_isolated_words,
                             const rb_bfs_params* params, rb_bfs** out) {
  return rb_bfs_create_part(d_row_starts, d_col, d_col_bu, d_degrees, n_dev, d_isolated_words, params, nullptr, out);
}

// ---- 1D-partition levels: the host drives the level loop and the exchange ----

extern "C" int rb_bfs_reset_part(rb_bfs* h, int64_t source_global, void* stream) {
  if (!h) return rb_null_handle(__func__);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_common(h, s);
  if (rc) return rc;
  RB_CUDA_TRY(cudaMemcpyAsync(h->kp.vis, h->vis_template, (size_t)h->n_words * 4, cudaMemcpyDeviceToDevice, s));
  const int64_t local = source_global - h->kp.v_lo;
  if (local >= 0 && local < h->n_dev) {
    bfs_seed<<<1, 32, 0, s>>>(h->kp, local);
    RB_CUDA_TRY(cudaGetLastError());
  }
  h->source = local;
  h->recs.clear();
  h->launched = false;
  return RB_OK;
}

extern "C" int rb_bfs_dist_level(rb_bfs* h, int64_t level, int direction, int hubs, const uint32_t* d_fcur_glob,
                                 const uint8_t* d_nz_glob, uint32_t** d_next_local, int64_t* h_counters,
                                 void* stream) {
  if (!h || !d_fcur_glob || !d_nz_glob || (direction != 0 && direction != 1)) {
    rb_set_error("rb_bfs_dist_level: invalid argument");
    return RB_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  RB_CUDA_TRY(cudaMemsetAsync(h->kp.bar, 0, 64, s));
  KParams kp = h->kp;
  kp.level0 = level;
  kp.dir0 = direction;
  kp.need_compact0 = 0;
  kp.max_levels = 1;
  kp.nf0 = 1;
  kp.mf0 = 0;
  kp.mu0 = 0;
  kp.src = 0;
  kp.m_directed = h->prm.m_directed;
  kp.fcur_ext = d_fcur_glob;
  kp.nzcur_ext = d_nz_glob;
  kp.hubs0 = hubs ? 1 : 0;
  void* args[] = {&kp};
  cudaError_t e;
  e = cudaLaunchCooperativeKernel(bfs_kernel(h), dim3(h->blocks), dim3(kThreads), args, 0, s);
  if (e != cudaSuccess) {
    rb_set_error("cooperative launch failed: %s", cudaGetErrorString(e));
    return RB_ERR_CUDA;
  }
  Slot sl;
  RB_CUDA_TRY(cudaMemcpyAsync(&sl, h->kp.slots + (level % 3), sizeof(Slot), cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  if (h_counters) {
    h_counters[0] = (int64_t)sl.n_next;
    h_counters[1] = (int64_t)sl.deg_next;
    h_counters[2] = (int64_t)sl.maxdeg;
    h_counters[3] = (int64_t)sl.scanned;
  }
  if (d_next_local) {
    const int64_t r = (level + 1) % 3;
    *d_next_local = r == 0 ? h->kp.fb0 : (r == 1 ? h->kp.fb1 : h->kp.fb2);
  }
  return RB_OK;
}


// ---------------------------------------------------------------------------
// Device-side exchange for the 1D partition (see bfs_dist)

static size_t xblock_layout(int64_t nwg, size_t off[5]) {
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 255) & ~(size_t)255; return r; };
  off[0] = take((size_t)3 * nwg * 4);                 // xg[3]
  off[1] = take((size_t)3 * nwg);                     // xnz[3]
  off[2] = take((size_t)2 * kMaxWorld * 4 * 8);       // slots
  off[3] = take(64);                                  // xbar
  off[4] = o;
  return o;
}

static void xparams_self(rb_bfs* h) {
  XParams& x = h->x;
  size_t off[5];
  xblock_layout(x.n_words_glob, off);
  char* b = (char*)h->xblock;
  for (int r = 0; r < 3; ++r) {
    x.xg[r] = (uint32_t*)(b + off[0]) + (size_t)r * x.n_words_glob;
    x.xnz[r] = (uint8_t*)(b + off[1]) + (size_t)r * x.n_words_glob;
  }
  x.slot = (unsigned long long*)(b + off[2]);
  x.xbar = (uint32_t*)(b + off[3]);
}

static void xparams_peer(rb_bfs* h, int q, char* b) {
  XParams& x = h->x;
  size_t off[5];
  xblock_layout(x.n_words_glob, off);
  for (int r = 0; r < 3; ++r) {
    x.peer_xg[q][r] = (uint32_t*)(b + off[0]) + (size_t)r * x.n_words_glob;
    x.peer_xnz[q][r] = (uint8_t*)(b + off[1]) + (size_t)r * x.n_words_glob;
  }
  x.peer_slot[q] = (unsigned long long*)(b + off[2]);
  x.peer_xbar[q] = (uint32_t*)(b + off[3]);
}

extern "C" int rb_bfs_xchg_alloc(rb_bfs* h, int32_t world, int32_t rank) {
  if (!h || !h->td_vinfo || world < 1 || world > kMaxWorld || rank < 0 || rank >= world || (h->kp.v_lo % 128)) {
    rb_set_error("rb_bfs_xchg_alloc: needs a partitioned engine with v_lo %% 128 == 0, 1 <= world <= %d, "
                 "0 <= rank < world", kMaxWorld);
    return RB_ERR_ARG;
  }
  if (h->xblock) return RB_OK;
  XParams& x = h->x;
  memset(&x, 0, sizeof(x));
  x.world = world;
  x.rank = rank;
  x.n_words_glob = h->kp.n_words_glob;
  x.w_lo = h->kp.v_lo / 32;
  size_t off[5];
  h->xbytes = xblock_layout(x.n_words_glob, off);
  int rc = alloc_dev(&h->xblock, h->xbytes);
  if (rc) return rc;
  RB_CUDA_TRY(cudaMemset(h->xblock, 0, h->xbytes));
  xparams_self(h);
  xparams_peer(h, rank, (char*)h->xblock);
  return RB_OK;
}

extern "C" size_t rb_bfs_xchg_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

extern "C" int rb_bfs_xchg_handle(rb_bfs* h, void* out) {
  if (!h || !h->xblock || !out) return rb_null_handle(__func__);
  cudaIpcMemHandle_t m;
  RB_CUDA_TRY(cudaIpcGetMemHandle(&m, h->xblock));
  memcpy(out, &m, sizeof(m));
  return RB_OK;
}

// handles: world IPC handles (rank order, rb_bfs_xchg_handle of every rank).
extern "C" int rb_bfs_xchg_open(rb_bfs* h, const void* handles) {
  if (!h || !h->xblock || !handles) return rb_null_handle(__func__);
  for (int q = 0; q < h->x.world; ++q) {
    if (q == h->x.rank) continue;
    cudaIpcMemHandle_t m;
    memcpy(&m, (const char*)handles + (size_t)q * sizeof(m), sizeof(m));
    void* b = nullptr;
    RB_CUDA_TRY(cudaIpcOpenMemHandle(&b, m, cudaIpcMemLazyEnablePeerAccess));
    h->x_opened.push_back(b);
    xparams_peer(h, q, (char*)b);
  }
  return RB_OK;
}

// One process, several engines (the emulation on one GPU): peers are plain pointers.
extern "C" int rb_bfs_xchg_connect_local(rb_bfs* const* hs, int32_t world) {
  if (!hs || world < 1 || world > kMaxWorld) return rb_null_handle(__func__);
  for (int r = 0; r < world; ++r)
    if (!hs[r] || !hs[r]->xblock || hs[r]->x.world != world || hs[r]->x.rank != r) return rb_null_handle(__func__);
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q) xparams_peer(hs[r], q, (char*)hs[q]->xblock);
  return RB_OK;
}

// Per-root reset of a distributed traversal (engine.py:526-532): local state,
// the exchange buffers (xg[0] = {source}), the source seeded by its owner.
extern "C" int rb_bfs_dist_reset(rb_bfs* h, int64_t source_global, int64_t deg_source, void* stream) {
  if (!h || !h->xblock || source_global < 0 || source_global >= h->n_glob) {
    rb_set_error("rb_bfs_dist_reset: invalid argument (source %lld, n %lld)", (long long)source_global,
                 (long long)h->n_glob);
    return RB_ERR_ARG;
  }
  {
    const cudaError_t prior = cudaGetLastError();
    if (prior != cudaSuccess) {
      rb_set_error("rb_bfs_dist_reset: pending CUDA error before the reset: %s", cudaGetErrorString(prior));
      return RB_ERR_CUDA;
    }
  }
  int rc = rb_bfs_reset_part(h, source_global, stream);
  if (rc) return rc;
  dist_reset_x<<<h->sms * 2, 256, 0, (cudaStream_t)stream>>>(h->x, source_global);
  RB_CUDA_TRY(cudaGetLastError());
  h->src_deg = deg_source;
  return RB_OK;
}

static KParams dist_kparams(const rb_bfs* h) {
  KParams kp = h->kp;
  kp.level0 = 0;
  kp.dir0 = 0;
  kp.need_compact0 = 0;
  kp.max_levels = kRecCap;
  kp.nf0 = 1;
  kp.mf0 = h->src_deg;
  kp.mu0 = h->prm.m_directed - h->src_deg;
  kp.m_directed = h->prm.m_directed;
  kp.from_fin = 0;
  kp.exec_opt = (h->exec_opt && h->prm.hybrid) ? 1 : 0;
  kp.fcur_ext = nullptr;
  kp.nzcur_ext = nullptr;
  return kp;
}

static const void* dist_kernel(const rb_bfs* h, bool emu) {
  const bool small = h->n_dev <= kSmallGraph;
  if (emu) return small ? (const void*)bfs_dist_emu<true, 4> : (const void*)bfs_dist_emu<true, 8>;
  return small ? (const void*)bfs_dist<true, 4> : (const void*)bfs_dist<true, 8>;
}

// The whole traversal of this rank: one persistent launch (every rank launches).
extern "C" int rb_bfs_dist_traverse(rb_bfs* h, void* stream) {
  if (!h || !h->xblock) return rb_null_handle(__func__);
  cudaStream_t s = (cudaStream_t)stream;
  KParams kp = dist_kparams(h);
  XParams x = h->x;
  void* args[] = {&kp, &x};
  RB_CUDA_TRY(cudaEventRecord(h->ev_start, s));
  cudaError_t e =
      cudaLaunchCooperativeKernel(dist_kernel(h, false), dim3(h->blocks), dim3(kThreads), args, 0, s);
  if (e != cudaSuccess) {
    rb_set_error("distributed launch failed: %s", cudaGetErrorString(e));
    return RB_ERR_CUDA;
  }
  RB_CUDA_TRY(cudaEventRecord(h->ev_end, s));
  h->launched = true;
  h->recs.clear();
  return RB_OK;
}

// One GPU: all ranks' traversal in one cooperative launch (engines of one
// process, rb_bfs_xchg_connect_local'ed, each reset with rb_bfs_dist_reset).
extern "C" int rb_bfs_dist_traverse_emu(rb_bfs* const* hs, int32_t world, void* stream) {
  if (!hs || world < 1 || world > kMaxWorld || !hs[0]) return rb_null_handle(__func__);
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<KParams> kps((size_t)world);
  std::vector<XParams> xps((size_t)world);
  for (int r = 0; r < world; ++r) {
    kps[(size_t)r] = dist_kparams(hs[r]);
    kps[(size_t)r].bar = hs[0]->kp.bar;  // one grid, one barrier counter
    xps[(size_t)r] = hs[r]->x;
  }
  // (the parameter arrays live in rank 0's slot area tail: a small device scratch)
  static thread_local void* scratch = nullptr;
  static thread_local size_t scratch_bytes = 0;
  const size_t need = (sizeof(KParams) + sizeof(XParams)) * (size_t)world;
  if (scratch_bytes < need) {
    if (scratch) cudaFree(scratch);
    RB_CUDA_TRY(cudaMalloc(&scratch, need));
    scratch_bytes = need;
  }
  RB_CUDA_TRY(cudaMemcpyAsync(scratch, kps.data(), sizeof(KParams) * world, cudaMemcpyHostToDevice, s));
  RB_CUDA_TRY(cudaMemcpyAsync((char*)scratch + sizeof(KParams) * world, xps.data(), sizeof(XParams) * world,
                              cudaMemcpyHostToDevice, s));
  EmuParams ep{world, (const KParams*)scratch, (const XParams*)((char*)scratch + sizeof(KParams) * world)};
  void* args[] = {&ep};
  rb_bfs* h0 = hs[0];
  RB_CUDA_TRY(cudaMemsetAsync(h0->kp.bar, 0, 64, s));
  RB_CUDA_TRY(cudaEventRecord(h0->ev_start, s));
  cudaError_t e =
      cudaLaunchCooperativeKernel(dist_kernel(h0, true), dim3(h0->blocks), dim3(kThreads), args, 0, s);
  if (e != cudaSuccess) {
    rb_set_error("emulated distributed launch failed: %s", cudaGetErrorString(e));
    return RB_ERR_CUDA;
  }
  RB_CUDA_TRY(cudaEventRecord(h0->ev_end, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));  // (the parameter scratch is reused by the next call)
  for (int r = 0; r < world; ++r) {
    hs[r]->launched = true;
    hs[r]->recs.clear();
  }
  return RB_OK;
}

// After a distributed traversal: level records (rank 0's engine holds them),
// elapsed device time, and the cross-barrier count carried to the next launch.
extern "C" int rb_bfs_dist_results(rb_bfs* h, rb_level_record* h_records, int64_t cap, int64_t* n_records,
                                   double* elapsed_s, void* stream) {
  if (!h || !h->xblock) return rb_null_handle(__func__);
  cudaStream_t s = (cudaStream_t)stream;
  Final f;
  RB_CUDA_TRY(cudaMemcpyAsync(&f, h->kp.fin, sizeof(Final), cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  if (f.nf > 0) {
    rb_set_error("distributed traversal deeper than %lld levels", (long long)kRecCap);
    return RB_ERR_CUDA;
  }
  h->x.xepoch0 = (uint32_t)f.pad;
  h->launched = false;
  const int64_t nr = f.levels_done;
  if (h_records && nr > 0) {
    std::vector<rb_level_record> tmp((size_t)nr);
    RB_CUDA_TRY(cudaMemcpy(tmp.data(), h->kp.rec, (size_t)nr * sizeof(rb_level_record), cudaMemcpyDeviceToHost));
    memcpy(h_records, tmp.data(), (size_t)(nr < cap ? nr : cap) * sizeof(rb_level_record));
  }
  if (n_records) *n_records = nr;
  if (elapsed_s) {  // (emulation: only the first rank's engine recorded the launch events)
    float ms = 0.f;
    RB_CUDA_TRY(cudaEventSynchronize(h->ev_end));
    RB_CUDA_TRY(cudaEventElapsedTime(&ms, h->ev_start, h->ev_end));
    *elapsed_s = 1e-3 * (double)ms;
  }
  return RB_OK;
}

extern "C" int rb_bfs_words(rb_bfs* h, int64_t* n_words_local, int64_t* n_words_glob) {
  if (!h) return rb_null_handle(__func__);
  if (n_words_local) *n_words_local = h->n_words;
  if (n_words_glob) *n_words_glob = h->kp.n_words_glob;
  return RB_OK;
}

extern "C" int rb_make_nz(const uint32_t* d_words, int64_t n_words, uint8_t* d_nz, void* stream) {
  if (n_words % 32) {
    rb_set_error("rb_make_nz: n_words must be a multiple of 32");
    return RB_ERR_ARG;
  }
  make_nz<<<256, 256, 0, (cudaStream_t)stream>>>(d_words, d_nz, n_words);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}
