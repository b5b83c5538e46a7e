/*
 * oracle.c -- CPU restatement of the rcmbfs hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker for the B200 implementation.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it; the product package never links or calls it.
 *
 * Every function restates one piece of the reference package `rcmbfs`
 * (/root/reference/pkg/src/rcmbfs/...) and cites the lines it follows.  The
 * restatement is pinned against the reference's own golden vectors and
 * against fixtures produced by running the reference (tests/golden/).
 *
 * Conventions: vertex ids uint32, row offsets int64, bitmaps are uint64 words
 * with bit i in word i>>6 at position i&63 (bitmap.py:1-24).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* LSD radix sort of uint64 keys (optionally with a uint32 payload).        */
/* Stable; 11-bit digits; passes whose digit is constant are skipped.       */

static void radix_sort_u64(uint64_t* keys, uint32_t* vals, int64_t n, int bits) {
  if (n <= 1) return;
  uint64_t* tk = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
  uint32_t* tv = vals ? (uint32_t*)malloc((size_t)n * sizeof(uint32_t)) : NULL;
  const int D = 11, R = 1 << D;
  int64_t* cnt = (int64_t*)malloc(R * sizeof(int64_t));
  uint64_t *ks = keys, *kd = tk;
  uint32_t *vs = vals, *vd = tv;
  for (int shift = 0; shift < bits; shift += D) {
    memset(cnt, 0, R * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[(ks[i] >> shift) & (R - 1)]++;
    int trivial = 0;
    for (int r = 0; r < R; ++r)
      if (cnt[r] == n) trivial = 1;
    if (trivial) continue;
    int64_t s = 0;
    for (int r = 0; r < R; ++r) { int64_t c = cnt[r]; cnt[r] = s; s += c; }
    for (int64_t i = 0; i < n; ++i) {
      int64_t p = cnt[(ks[i] >> shift) & (R - 1)]++;
      kd[p] = ks[i];
      if (vs) vd[p] = vs[i];
    }
    uint64_t* t = ks; ks = kd; kd = t;
    uint32_t* u = vs; vs = vd; vd = u;
  }
  if (ks != keys) {
    memcpy(keys, ks, (size_t)n * sizeof(uint64_t));
    if (vals) memcpy(vals, vs, (size_t)n * sizeof(uint32_t));
  }
  free(tk); free(tv); free(cnt);
}

static int bits_for(uint64_t x) { int b = 0; while (b < 64 && (x >> b)) ++b; return b; }

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

/* ------------------------------------------------------------------------ */
/* build_csr -- graph.py:85-120.                                             */
/* Returns m_directed, or -1 with *bad_index set on an out-of-range edge.    */
/* dst must hold 2*m entries.                                               */

EXPORT int64_t or_build_csr(int64_t n, int64_t m, const uint32_t* edges,
                            int64_t* row_starts, uint32_t* dst, int32_t* degrees,
                            int64_t* bad_index) {
  /* graph.py:103-108: first out-of-range edge by input index */
  for (int64_t i = 0; i < m; ++i) {
    if ((int64_t)edges[2 * i] >= n || (int64_t)edges[2 * i + 1] >= n) {
      *bad_index = i;
      return -1;
    }
  }
  uint64_t* keys = (uint64_t*)malloc((size_t)(2 * m + 1) * sizeof(uint64_t));
  int64_t k = 0;
  for (int64_t i = 0; i < m; ++i) {
    uint64_t u = edges[2 * i], v = edges[2 * i + 1];
    if (u == v) continue; /* graph.py:110-111 self-loops dropped */
    keys[k++] = (u << 32) | v; /* (u, v) lexicographic == u*n+v order (graph.py:114) */
    keys[k++] = (v << 32) | u;
  }
  radix_sort_u64(keys, NULL, k, 32 + bits_for((uint64_t)(n > 0 ? n - 1 : 0)));
  int64_t md = 0;
  for (int64_t i = 0; i < k; ++i)
    if (md == 0 || keys[i] != keys[md - 1]) keys[md++] = keys[i]; /* np.unique dedup */
  memset(degrees, 0, (size_t)n * sizeof(int32_t));
  for (int64_t i = 0; i < md; ++i) {
    dst[i] = (uint32_t)(keys[i] & 0xffffffffu);
    degrees[keys[i] >> 32]++; /* graph.py:117 bincount */
  }
  row_starts[0] = 0; /* graph.py:118-119 int64 cumsum */
  for (int64_t v = 0; v < n; ++v) row_starts[v + 1] = row_starts[v] + degrees[v];
  free(keys);
  return md;
}

/* ------------------------------------------------------------------------ */
/* degree_sort_adjacency -- reorder.py:151-166, 181-195.                     */
/* key = d*n + w (asc) or (2^31 - d)*n + w (desc); ties by ascending id.     */

EXPORT void or_degree_sort_rows(int64_t n, const int64_t* rs, const uint32_t* dst,
                                const int32_t* deg, uint32_t* out, int descending) {
  uint64_t* keys = NULL;
  int64_t cap = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t a = rs[v], b = rs[v + 1], d = b - a;
    if (d > cap) { cap = d; keys = (uint64_t*)realloc(keys, (size_t)cap * sizeof(uint64_t)); }
    for (int64_t j = 0; j < d; ++j) {
      uint64_t w = dst[a + j];
      uint64_t dd = descending ? ((1ull << 31) - (uint64_t)deg[w]) : (uint64_t)deg[w];
      keys[j] = (dd << 32) | w; /* same order as dd*n + w since w < n <= 2^32 */
    }
    if (d > 1) qsort(keys, (size_t)d, sizeof(uint64_t), cmp_u64);
    for (int64_t j = 0; j < d; ++j) out[a + j] = (uint32_t)(keys[j] & 0xffffffffu);
  }
  free(keys);
}

/* ------------------------------------------------------------------------ */
/* rcm -- reorder.py:198-237 with _rcm_walk reorder.py:106-148.              */
/* perm[new] = old.  comp_starts (capacity n+1) gets discovery-order          */
/* component starts; returns the number of components.  *n_plus = |V+|.     */

EXPORT int64_t or_rcm(int64_t n, const int64_t* rs, const uint32_t* dst, const int32_t* deg,
                      uint32_t* perm, int64_t* comp_starts, int64_t* n_plus_out) {
  /* vplus: V+ sorted by (degree, id) -- reorder.py:202-203 (stable counting sort) */
  int32_t maxd = 0;
  for (int64_t v = 0; v < n; ++v) if (deg[v] > maxd) maxd = deg[v];
  int64_t* bucket = (int64_t*)calloc((size_t)maxd + 2, sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) bucket[deg[v] + 1]++;
  for (int32_t d = 0; d <= maxd; ++d) bucket[d + 1] += bucket[d];
  uint32_t* by_deg = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(uint32_t));
  for (int64_t v = 0; v < n; ++v) by_deg[bucket[deg[v]]++] = (uint32_t)v;
  free(bucket);
  int64_t iso = 0;
  for (int64_t v = 0; v < n; ++v) if (deg[v] == 0) ++iso;
  int64_t k = n - iso;
  const uint32_t* vplus = by_deg + iso; /* degree-0 vertices sort first */
  *n_plus_out = k;

  /* ascending (deg, id) adjacency -- reorder.py:216 */
  int64_t m = n ? rs[n] : 0;
  uint32_t* asc = (uint32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint32_t));
  or_degree_sort_rows(n, rs, dst, deg, asc, 0);

  /* the walk -- reorder.py:115-148 */
  uint32_t* order = (uint32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(uint32_t));
  uint8_t* placed = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  int64_t n_comp = 0, slow = 0, fast = 0, seed_scan = 0;
  while (slow < k) {
    if (slow == fast) {
      while (placed[vplus[seed_scan]]) ++seed_scan;
      uint32_t s = vplus[seed_scan];
      comp_starts[n_comp++] = fast;
      placed[s] = 1;
      order[fast++] = s;
    }
    uint32_t v = order[slow++];
    for (int64_t j = rs[v]; j < rs[v + 1]; ++j) {
      uint32_t w = asc[j];
      if (!placed[w]) { placed[w] = 1; order[fast++] = w; }
    }
  }
  /* perm = concat(order[::-1], remaining(empty for full RCM), isolated asc) -- reorder.py:219-220 */
  for (int64_t i = 0; i < k; ++i) perm[i] = order[k - 1 - i];
  for (int64_t i = 0; i < iso; ++i) perm[k + i] = by_deg[i]; /* by_deg[0:iso] is ascending id */
  free(order); free(placed); free(asc); free(by_deg);
  return n_comp;
}

/* ------------------------------------------------------------------------ */
/* apply_permutation -- reorder.py:169-178, 254-271.                          */

EXPORT void or_apply_permutation(int64_t n, const int64_t* rs, const uint32_t* dst,
                                 const int32_t* deg, const uint32_t* perm, const uint32_t* inv,
                                 int64_t* rs_out, uint32_t* dst_out, int32_t* deg_out) {
  rs_out[0] = 0;
  for (int64_t nv = 0; nv < n; ++nv) {
    deg_out[nv] = deg[perm[nv]];
    rs_out[nv + 1] = rs_out[nv] + deg_out[nv];
  }
  for (int64_t nv = 0; nv < n; ++nv) {
    uint32_t ov = perm[nv];
    int64_t o0 = rs[ov], cnt = rs[ov + 1] - o0, b = rs_out[nv];
    for (int64_t j = 0; j < cnt; ++j) dst_out[b + j] = inv[dst[o0 + j]];
    if (cnt > 1) qsort(dst_out + b, (size_t)cnt, sizeof(uint32_t), cmp_u32);
  }
}

/* ------------------------------------------------------------------------ */
/* Sequential BFS -- _kernels.py:26-54 (parent = first discoverer in scan    */
/* order).  Also emits levels (-1 unreached).  Returns the level count.      */

EXPORT int64_t or_seq_bfs(int64_t n, const int64_t* rs, const uint32_t* dst, int64_t source,
                          int32_t* parent, int32_t* level, uint32_t* queue, int64_t* bounds) {
  for (int64_t v = 0; v < n; ++v) { parent[v] = -1; level[v] = -1; }
  parent[source] = (int32_t)source;
  level[source] = 0;
  queue[0] = (uint32_t)source;
  bounds[0] = 0;
  int64_t n_levels = 0, ls = 0, le = 1, tail = 1;
  while (ls < le) {
    ++n_levels;
    bounds[n_levels] = le;
    for (int64_t i = ls; i < le; ++i) {
      uint32_t v = queue[i];
      for (int64_t j = rs[v]; j < rs[v + 1]; ++j) {
        uint32_t w = dst[j];
        if (parent[w] < 0) {
          parent[w] = (int32_t)v;
          level[w] = level[v] + 1;
          queue[tail++] = w;
        }
      }
    }
    ls = le;
    le = tail;
  }
  return n_levels;
}

/* ------------------------------------------------------------------------ */
/* Single steps for random-state parity (criterion 2, test_acceptance.py:   */
/* 117-164).  td: _kernels.py:57-87 (td_plain, 1 thread).  bu:               */
/* _kernels.py:144-173 (bu_range over [0,n)).  Both update visited/parent     */
/* in place.  out[0..2] = (n_next, deg_next, scanned).                       */

EXPORT void or_td_step(int64_t n, const int64_t* rs, const uint32_t* dst,
                       const uint32_t* frontier, int64_t nf, int32_t* parent,
                       uint64_t* visited, uint32_t* next_q, int64_t* out) {
  int64_t cnt = 0, degsum = 0, scanned = 0;
  (void)n;
  for (int64_t i = 0; i < nf; ++i) {
    uint32_t v = frontier[i];
    for (int64_t j = rs[v]; j < rs[v + 1]; ++j) {
      uint32_t w = dst[j];
      ++scanned;
      uint64_t m = 1ull << (w & 63);
      if (!(visited[w >> 6] & m)) {
        visited[w >> 6] |= m;
        parent[w] = (int32_t)v;
        next_q[cnt++] = w;
        degsum += rs[w + 1] - rs[w];
      }
    }
  }
  out[0] = cnt; out[1] = degsum; out[2] = scanned;
}

EXPORT void or_bu_step(int64_t n, const int64_t* rs, const uint32_t* dst,
                       const uint64_t* fcur, uint64_t* fnext, uint64_t* visited,
                       int32_t* parent, int64_t* out) {
  int64_t cnt = 0, degsum = 0, checks = 0;
  for (int64_t v = 0; v < n; ++v) {
    uint64_t mv = 1ull << (v & 63);
    if (visited[v >> 6] & mv) continue;
    int64_t a = rs[v], b = rs[v + 1];
    for (int64_t j = a; j < b; ++j) {
      uint32_t u = dst[j];
      ++checks;
      if (fcur[u >> 6] & (1ull << (u & 63))) {
        parent[v] = (int32_t)u;
        visited[v >> 6] |= mv;
        fnext[v >> 6] |= mv;
        ++cnt;
        degsum += b - a;
        break;
      }
    }
  }
  out[0] = cnt; out[1] = degsum; out[2] = checks;
}

/* ------------------------------------------------------------------------ */
/* Hybrid BFS -- BfsEngine.run, engine.py:518-604, mode "hybrid" (or         */
/* "level_sync" when hybrid==0), with td_plain (_kernels.py:57-87) over       */
/* contiguous frontier chunks (engine.py:248-249, 270-276) and bu_range over */
/* block-aligned static ranges (engine.py:355-370).  Multithreaded with      */
/* OpenMP; atomics as in _atomics.py.  This is the CPU baseline arm.         */
/*                                                                          */
/* rec (capacity rec_cap rows of 6 int64): level, direction (0 TD, 1 BU),    */
/* n_f, m_f, m_u, scanned.  Returns the level count; *elapsed = seconds of   */
/* the level loop (engine.py:534-598, reset excluded).                       */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

EXPORT int64_t or_hybrid_bfs(int64_t n, const int64_t* rs, const uint32_t* dst,
                             const int32_t* deg, int64_t source, int alpha, int beta,
                             int hybrid, int threads, int32_t* parent, int64_t* rec,
                             int64_t rec_cap, double* elapsed) {
  int64_t nw = ((n + 511) / 512) * 8; /* whole 512-bit blocks (bitmap.py:21-24) */
  if (nw == 0) nw = 8;
  uint64_t* visited = (uint64_t*)calloc((size_t)nw, 8);
  uint64_t* fcur = (uint64_t*)calloc((size_t)nw, 8);
  uint64_t* fnext = (uint64_t*)calloc((size_t)nw, 8);
  uint32_t* q = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * 4);
  uint32_t* nq = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * 4);
#ifdef _OPENMP
  if (threads < 1) threads = omp_get_max_threads();
#else
  threads = 1;
#endif
  /* reset (not timed): engine.py:526-532 */
  for (int64_t v = 0; v < n; ++v) {
    parent[v] = -1;
    if (deg[v] == 0) visited[v >> 6] |= 1ull << (v & 63); /* engine.py:432-437 */
  }
  parent[source] = (int32_t)source;
  visited[source >> 6] |= 1ull << (source & 63);

  double t0 = now_s();
  int64_t m_directed = rs[n];
  int64_t nf = 1, m_f = deg[source], m_u = m_directed - deg[source];
  int q_valid = 1, bits_valid = 0; /* which frontier forms are present */
  q[0] = (uint32_t)source;
  int dir = 0, level = 0;
  int64_t nblocks = (n + 511) / 512;
  while (nf > 0) {
    int use = hybrid ? dir : 0;
    int64_t n_next = 0, deg_next = 0, scanned = 0;
    if (use == 0) {
      if (!q_valid) { /* Frontier.to_queue_form: Bitmap.to_indices (bitmap.py:122-125) */
        int64_t c = 0;
        for (int64_t w = 0; w < nw; ++w) {
          uint64_t x = fcur[w];
          while (x) { int b = __builtin_ctzll(x); q[c++] = (uint32_t)(w * 64 + b); x &= x - 1; }
        }
        q_valid = 1;
      }
      int64_t cursor = 0;
#pragma omp parallel num_threads(threads) reduction(+ : deg_next, scanned)
      {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num(); T = omp_get_num_threads();
#endif
        int64_t lo = nf * t / T, hi = nf * (t + 1) / T; /* _chunk_bounds */
        for (int64_t i = lo; i < hi; ++i) {
          uint32_t v = q[i];
          for (int64_t j = rs[v]; j < rs[v + 1]; ++j) {
            uint32_t w = dst[j];
            ++scanned;
            uint64_t mk = 1ull << (w & 63);
            if (!(__atomic_load_n(&visited[w >> 6], __ATOMIC_RELAXED) & mk)) {
              uint64_t old = __atomic_fetch_or(&visited[w >> 6], mk, __ATOMIC_RELAXED);
              if (!(old & mk)) {
                parent[w] = (int32_t)v;
                int64_t pos = __atomic_fetch_add(&cursor, 1, __ATOMIC_RELAXED);
                nq[pos] = w;
                deg_next += deg[w];
              }
            }
          }
        }
      }
      n_next = cursor;
      uint32_t* t = q; q = nq; nq = t;
      q_valid = 1; bits_valid = 0;
    } else {
      if (!bits_valid) { /* Frontier.to_bitmap_form: queue_to_bits (_kernels.py:296-301) */
        memset(fcur, 0, (size_t)nw * 8);
        for (int64_t i = 0; i < nf; ++i) fcur[q[i] >> 6] |= 1ull << (q[i] & 63);
        bits_valid = 1;
      }
      memset(fnext, 0, (size_t)nw * 8); /* fresh Bitmap(n) per step (engine.py:356) */
#pragma omp parallel num_threads(threads) reduction(+ : n_next, deg_next, scanned)
      {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num(); T = omp_get_num_threads();
#endif
        int64_t lo = (nblocks * t / T) * 512, hi = (nblocks * (t + 1) / T) * 512;
        if (lo > n) lo = n;
        if (hi > n || t == T - 1) hi = n;
        for (int64_t v = lo; v < hi; ++v) {
          uint64_t mv = 1ull << (v & 63);
          if (visited[v >> 6] & mv) continue;
          int64_t a = rs[v], b = rs[v + 1];
          for (int64_t j = a; j < b; ++j) {
            uint32_t u = dst[j];
            ++scanned;
            if (fcur[u >> 6] & (1ull << (u & 63))) {
              parent[v] = (int32_t)u;
              visited[v >> 6] |= mv;
              fnext[v >> 6] |= mv;
              ++n_next;
              deg_next += b - a;
              break;
            }
          }
        }
      }
      uint64_t* t = fcur; fcur = fnext; fnext = t;
      bits_valid = 1; q_valid = 0;
    }
    if (level < rec_cap) {
      int64_t* r = rec + 6 * level;
      r[0] = level; r[1] = use; r[2] = nf; r[3] = m_f; r[4] = m_u; r[5] = scanned;
    }
    m_u -= deg_next; /* engine.py:587-589 */
    m_f = deg_next;
    nf = n_next;
    if (hybrid) { /* update_traversal_policy, engine.py:215-228 (n = g.n) */
      if (use == 0) dir = ((double)m_f > (double)m_u / (double)alpha) ? 1 : 0;
      else dir = ((double)nf < (double)n / (double)beta) ? 0 : 1;
    }
    ++level;
  }
  *elapsed = now_s() - t0;
  free(visited); free(fcur); free(fnext); free(q); free(nq);
  return level;
}

/* ------------------------------------------------------------------------ */
/* Validator -- validate.py:123-225.  Five rules; derived levels out.        */
/* ok[0..4] = rule pass flags.  labels: component label per vertex (caller   */
/* computes from raw edges with or_components).  Returns 1 iff all pass.     */

EXPORT void or_components(int64_t n, int64_t m, const uint32_t* us, int64_t su,
                          const uint32_t* vs, int64_t sv, int64_t* root) {
  /* _uf_components, validate.py:63-86 (path halving, min-id root) */
  for (int64_t v = 0; v < n; ++v) root[v] = v;
  for (int64_t e = 0; e < m; ++e) {
    int64_t a = us[e * su], b = vs[e * sv];
    while (root[a] != a) { root[a] = root[root[a]]; a = root[a]; }
    while (root[b] != b) { root[b] = root[root[b]]; b = root[b]; }
    if (a != b) { if (a < b) root[b] = a; else root[a] = b; }
  }
  for (int64_t v = 0; v < n; ++v) {
    int64_t r = v;
    while (root[r] != r) r = root[r];
    root[v] = r;
  }
}

static int has_edge(const int64_t* rs, const uint32_t* dst, int64_t v, int64_t p) {
  /* binary search in the (ascending) row of v -- validate.py:146-153 uses
     sorted (u*n+v) keys; rows are ascending for build_csr/apply_permutation */
  int64_t lo = rs[v], hi = rs[v + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)dst[mid] < p) lo = mid + 1; else hi = mid;
  }
  return lo < rs[v + 1] && (int64_t)dst[lo] == p;
}

EXPORT int or_validate(int64_t n, const int64_t* rs, const uint32_t* dst, const int64_t* labels,
                       int64_t source, const int32_t* parent, int64_t* levels, int* ok) {
  /* rule 1 */
  ok[0] = parent[source] == source;
  /* rule 2: tree edges exist (rows must be ascending) */
  ok[1] = 1;
  for (int64_t v = 0; v < n && ok[1]; ++v) {
    if (v == source || parent[v] < 0) continue;
    int64_t p = parent[v];
    if (p >= n || !has_edge(rs, dst, v, p)) ok[1] = 0;
  }
  /* rule 3: levels from parent chains (validate.py:169-190) */
  for (int64_t v = 0; v < n; ++v) levels[v] = -1;
  levels[source] = 0;
  int64_t* stack = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  ok[2] = 1;
  for (int64_t v = 0; v < n; ++v) {
    if (parent[v] < 0 || levels[v] >= 0) continue;
    int64_t sp = 0, u = v, bad = 0;
    while (levels[u] < 0) {
      /* a chain longer than n vertices is a cycle */
      if (sp >= n || parent[u] < 0 || parent[u] >= n) { bad = 1; break; }
      stack[sp++] = u;
      u = parent[u];
    }
    if (bad) { ok[2] = 0; continue; }
    int64_t base = levels[u];
    while (sp > 0) levels[stack[--sp]] = ++base;
  }
  free(stack);
  /* cycles leave chains unresolved: validator semantics mark them -1 */
  /* rule 4: edges span at most one level among reached endpoints */
  ok[3] = 1;
  for (int64_t v = 0; v < n && ok[3]; ++v) {
    if (levels[v] < 0) continue;
    for (int64_t j = rs[v]; j < rs[v + 1]; ++j) {
      int64_t lw = levels[dst[j]];
      if (lw >= 0 && (lw - levels[v] > 1 || levels[v] - lw > 1)) { ok[3] = 0; break; }
    }
  }
  /* rule 5: reached iff same component as source */
  ok[4] = 1;
  for (int64_t v = 0; v < n; ++v)
    if ((labels[v] == labels[source]) != (parent[v] >= 0)) { ok[4] = 0; break; }
  return ok[0] && ok[1] && ok[2] && ok[3] && ok[4];
}
