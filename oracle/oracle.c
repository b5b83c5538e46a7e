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

static int bits_for(uint64_t x) { int b = 0; while (b < 64 && (x >> b)) ++b; return b; }

static void radix_sort_u64_buf(uint64_t* a, int64_t n, uint64_t* tmp) {
  /* LSD, 11-bit digits over the bits where the keys differ (a row's keys) */
  uint64_t diff = 0;
  for (int64_t i = 1; i < n; ++i) diff |= a[i] ^ a[0];
  const int bits = bits_for(diff);
  uint64_t *src = a, *dstb = tmp;
  int64_t cnt[2048];
  for (int shift = 0; shift < bits; shift += 11) {
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < n; ++i) cnt[(src[i] >> shift) & 2047]++;
    int64_t s0 = 0;
    for (int r = 0; r < 2048; ++r) { int64_t c = cnt[r]; cnt[r] = s0; s0 += c; }
    for (int64_t i = 0; i < n; ++i) dstb[cnt[(src[i] >> shift) & 2047]++] = src[i];
    uint64_t* t = src; src = dstb; dstb = t;
  }
  if (src != a) memcpy(a, src, (size_t)n * 8);
}


/* ------------------------------------------------------------------------ */
/* Row sorts used by the CSR build, the relabel and the degree sort.         */
/* Short rows: insertion sort; long rows: LSD radix sort (11-bit digits,     */
/* only as many passes as the largest key needs) through a caller scratch.   */

static void sort_u32(uint32_t* a, int64_t n, uint32_t* tmp) {
  if (n <= 48) {
    for (int64_t i = 1; i < n; ++i) {
      uint32_t x = a[i];
      int64_t j = i - 1;
      while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
      a[j + 1] = x;
    }
    return;
  }
  uint32_t mx = 0;
  for (int64_t i = 0; i < n; ++i) if (a[i] > mx) mx = a[i];
  int bits = bits_for(mx);
  uint32_t *src = a, *dstb = tmp;
  int64_t cnt[2048];
  for (int shift = 0; shift < bits; shift += 11) {
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < n; ++i) cnt[(src[i] >> shift) & 2047]++;
    int64_t s0 = 0;
    for (int r = 0; r < 2048; ++r) { int64_t c = cnt[r]; cnt[r] = s0; s0 += c; }
    for (int64_t i = 0; i < n; ++i) dstb[cnt[(src[i] >> shift) & 2047]++] = src[i];
    uint32_t* t = src; src = dstb; dstb = t;
  }
  if (src != a) memcpy(a, src, (size_t)n * 4);
}

static void sort_u64(uint64_t* a, int64_t n, uint64_t* tmp) {
  if (n <= 48) {
    for (int64_t i = 1; i < n; ++i) {
      uint64_t x = a[i];
      int64_t j = i - 1;
      while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
      a[j + 1] = x;
    }
    return;
  }
  radix_sort_u64_buf(a, n, tmp);
}

static int nthreads_of(int threads) {
#ifdef _OPENMP
  return threads > 0 ? threads : omp_get_max_threads();
#else
  (void)threads;
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* build_csr -- graph.py:85-120.                                             */
/* Two calls: or_build_csr_begin validates, buckets both orientations of    */
/* every non-self-loop pair by source (counting sort), sorts and dedups each */
/* row -- exactly np.unique over u*n+v keys, graph.py:110-116 -- and keeps   */
/* the result in a handle; or_build_csr_take copies it out and frees it.    */
/* Returns m_directed, or -1 with *bad_index set on an out-of-range edge.    */

typedef struct {
  int64_t n, md;
  int64_t* rs;
  uint32_t* dst;
  int32_t* deg;
} csr_handle;

EXPORT int64_t or_build_csr_begin(int64_t n, int64_t m, const uint32_t* edges, int threads, int64_t* bad_index,
                                  void** handle) {
  int T = nthreads_of(threads);
  /* graph.py:103-108: first out-of-range edge by input index */
  int64_t bad = m;
#pragma omp parallel for num_threads(T) reduction(min : bad) schedule(static)
  for (int64_t i = 0; i < m; ++i)
    if ((int64_t)edges[2 * i] >= n || (int64_t)edges[2 * i + 1] >= n) if (i < bad) bad = i;
  if (bad < m) { *bad_index = bad; return -1; }
  int64_t* rs = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  /* per-source counts of both orientations, self-loops dropped (graph.py:110-111) */
#pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    uint32_t u = edges[2 * i], v = edges[2 * i + 1];
    if (u == v) continue;
    __atomic_fetch_add(&rs[u + 1], 1, __ATOMIC_RELAXED);
    __atomic_fetch_add(&rs[v + 1], 1, __ATOMIC_RELAXED);
  }
  for (int64_t v = 0; v < n; ++v) rs[v + 1] += rs[v];
  int64_t tot = rs[n];
  uint32_t* raw = (uint32_t*)malloc((size_t)(tot > 0 ? tot : 1) * 4);
  int64_t* cur = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  memcpy(cur, rs, (size_t)n * sizeof(int64_t));
#pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    uint32_t u = edges[2 * i], v = edges[2 * i + 1];
    if (u == v) continue;
    raw[__atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED)] = v;
    raw[__atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED)] = u;
  }
  /* each row: ascending, duplicates removed (np.unique); cur[v] = new degree */
#pragma omp parallel num_threads(T)
  {
    int64_t cap = 0;
    uint32_t* tmp = NULL;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; ++v) {
      int64_t a = rs[v], d = rs[v + 1] - a;
      if (d > cap) { cap = d; tmp = (uint32_t*)realloc(tmp, (size_t)cap * 4); }
      sort_u32(raw + a, d, tmp);
      int64_t k = 0;
      for (int64_t j = 0; j < d; ++j)
        if (k == 0 || raw[a + j] != raw[a + k - 1]) raw[a + k++] = raw[a + j];
      cur[v] = k;
    }
    free(tmp);
  }
  csr_handle* h = (csr_handle*)calloc(1, sizeof(csr_handle));
  h->n = n;
  h->deg = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * 4);
  h->rs = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  h->rs[0] = 0; /* graph.py:117-119: bincount + int64 cumsum */
  for (int64_t v = 0; v < n; ++v) { h->deg[v] = (int32_t)cur[v]; h->rs[v + 1] = h->rs[v] + cur[v]; }
  h->md = h->rs[n];
  h->dst = (uint32_t*)malloc((size_t)(h->md > 0 ? h->md : 1) * 4);
#pragma omp parallel for num_threads(T) schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; ++v) memcpy(h->dst + h->rs[v], raw + rs[v], (size_t)cur[v] * 4);
  free(raw); free(cur); free(rs);
  *handle = h;
  return h->md;
}

EXPORT void or_build_csr_take(void* handle, int64_t* row_starts, uint32_t* dst, int32_t* degrees) {
  csr_handle* h = (csr_handle*)handle;
  memcpy(row_starts, h->rs, (size_t)(h->n + 1) * sizeof(int64_t));
  memcpy(dst, h->dst, (size_t)h->md * 4);
  memcpy(degrees, h->deg, (size_t)h->n * 4);
  free(h->rs); free(h->dst); free(h->deg); free(h);
}

/* ------------------------------------------------------------------------ */
/* degree_sort_adjacency -- reorder.py:151-166, 181-195.                     */
/* key = d*n + w (asc) or (2^31 - d)*n + w (desc); ties by ascending id.     */

EXPORT void or_degree_sort_rows(int64_t n, const int64_t* rs, const uint32_t* dst,
                                const int32_t* deg, uint32_t* out, int descending) {
#pragma omp parallel
  {
    uint64_t *keys = NULL, *tmp = NULL;
    int64_t cap = 0;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; ++v) {
      int64_t a = rs[v], b = rs[v + 1], d = b - a;
      if (d > cap) {
        cap = d;
        keys = (uint64_t*)realloc(keys, (size_t)cap * sizeof(uint64_t));
        tmp = (uint64_t*)realloc(tmp, (size_t)cap * sizeof(uint64_t));
      }
      for (int64_t j = 0; j < d; ++j) {
        uint64_t w = dst[a + j];
        uint64_t dd = descending ? ((1ull << 31) - (uint64_t)deg[w]) : (uint64_t)deg[w];
        keys[j] = (dd << 32) | w; /* same order as dd*n + w since w < n <= 2^32 */
      }
      sort_u64(keys, d, tmp);
      for (int64_t j = 0; j < d; ++j) out[a + j] = (uint32_t)(keys[j] & 0xffffffffu);
    }
    free(keys); free(tmp);
  }
}

/* ------------------------------------------------------------------------ */
/* rcm / partial_rcm -- reorder.py:198-251 with _rcm_walk reorder.py:106-148. */
/* perm[new] = old.  comp_starts (capacity n+1) gets discovery-order          */
/* component starts; returns the number of components.  *n_plus = |V+|.     */
/* k_req < 0: full RCM (k = |V+|); else the walk stops after k_req labels    */
/* (partial_rcm, reorder.py:240-251) and the unlabelled non-isolated         */
/* vertices follow the reversed prefix in ascending id (reorder.py:219-220). */

EXPORT int64_t or_rcm_k(int64_t n, const int64_t* rs, const uint32_t* dst, const int32_t* deg, int64_t k_req,
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
  const int64_t n_plus = n - iso;
  const uint32_t* vplus = by_deg + iso; /* degree-0 vertices sort first */
  *n_plus_out = n_plus;
  const int64_t k = (k_req < 0 || k_req > n_plus) ? n_plus : k_req;
  uint8_t* placed = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  uint32_t* order = (uint32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(uint32_t));
  int64_t n_comp = 0;
  if (k > 0) {
    /* ascending (deg, id) adjacency -- reorder.py:216 */
    int64_t m = n ? rs[n] : 0;
    uint32_t* asc = (uint32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint32_t));
    or_degree_sort_rows(n, rs, dst, deg, asc, 0);
    /* the walk -- reorder.py:115-148, stopping at k labels */
    int64_t slow = 0, fast = 0, seed_scan = 0;
    while (slow < k && fast < k) {
      if (slow == fast) {
        while (placed[vplus[seed_scan]]) ++seed_scan;
        uint32_t s0 = vplus[seed_scan];
        comp_starts[n_comp++] = fast;
        placed[s0] = 1;
        order[fast++] = s0;
        if (fast == k) break;
      }
      uint32_t v = order[slow++];
      for (int64_t j = rs[v]; j < rs[v + 1] && fast < k; ++j) {
        uint32_t w = asc[j];
        if (!placed[w]) { placed[w] = 1; order[fast++] = w; }
      }
    }
    free(asc);
  }
  /* perm = concat(order[::-1], remaining, isolated asc) -- reorder.py:219-220 */
  int64_t o = 0;
  for (int64_t i = 0; i < k; ++i) perm[o++] = order[k - 1 - i];
  if (k == 0) { /* reorder.py:208-213: non-isolated ascending, then isolated */
    for (int64_t v = 0; v < n; ++v) if (deg[v] > 0) perm[o++] = (uint32_t)v;
  } else {
    for (int64_t v = 0; v < n; ++v) if (deg[v] > 0 && !placed[v]) perm[o++] = (uint32_t)v;
  }
  for (int64_t i = 0; i < iso; ++i) perm[o++] = by_deg[i]; /* by_deg[0:iso] is ascending id */
  free(order); free(placed); free(by_deg);
  return n_comp;
}

EXPORT int64_t or_rcm(int64_t n, const int64_t* rs, const uint32_t* dst, const int32_t* deg,
                      uint32_t* perm, int64_t* comp_starts, int64_t* n_plus_out) {
  return or_rcm_k(n, rs, dst, deg, -1, perm, comp_starts, n_plus_out);
}

/* ------------------------------------------------------------------------ */
/* apply_permutation -- reorder.py:169-178, 254-271.                          */

EXPORT void or_apply_permutation(int64_t n, const int64_t* rs, const uint32_t* dst,
                                 const int32_t* deg, const uint32_t* perm, const uint32_t* inv,
                                 int64_t* rs_out, uint32_t* dst_out, int32_t* deg_out) {
  rs_out[0] = 0; /* reorder.py:262-264: new_degrees = deg[perm], int64 cumsum */
  for (int64_t nv = 0; nv < n; ++nv) {
    deg_out[nv] = deg[perm[nv]];
    rs_out[nv + 1] = rs_out[nv] + deg_out[nv];
  }
#pragma omp parallel
  {
    uint32_t* tmp = NULL;
    int64_t cap = 0;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t nv = 0; nv < n; ++nv) { /* _permute_rows, reorder.py:169-178 */
      uint32_t ov = perm[nv];
      int64_t o0 = rs[ov], cnt = rs[ov + 1] - o0, b = rs_out[nv];
      if (cnt > cap) { cap = cnt; tmp = (uint32_t*)realloc(tmp, (size_t)cap * 4); }
      for (int64_t j = 0; j < cnt; ++j) dst_out[b + j] = inv[dst[o0 + j]];
      sort_u32(dst_out + b, cnt, tmp);
    }
    free(tmp);
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
/* BfsEngine.run -- engine.py:478-604, every mode except "sequential":       */
/*   mode 0 level_sync       td_plain over contiguous frontier chunks        */
/*   mode 1 hybrid           td_plain + bu_range (512-aligned static ranges) */
/*   mode 2 hybrid_balanced  td_striped + bu_steal (work-stealing partitions)*/
/*   mode 3 hybrid_reduced   td_striped + bu_reduced (Alg. 6 two-pass on the */
/*                           descending-degree adjacency dst_desc, shrinking */
/*                           live bounds, deferred visited publish)          */
/* Kernels: _kernels.py:57-293; partitions: partition.py:67-157; atomics as  */
/* _atomics.py (fetch_or / fetch_add).  OpenMP threads = params.threads, so  */
/* the partition count is partition_factor * threads like the reference.    */
/* This is also the CPU baseline arm (bench.py --impl reference).           */
/*                                                                          */
/* rec (rec_cap rows of 9 int64): level, direction (0 TD / 1 BU), n_f, m_f,  */
/* m_u, scanned, pass1_hits, live_vertices, claimed (-1 = None, as the       */
/* reference's LevelRecord).  level (optional): BFS level per vertex.        */
/* Returns the level count; *elapsed = seconds of the level loop            */
/* (engine.py:534-598: frontier conversions included, reset excluded).      */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* partition.py:77-95 _descending_block_counts */
static void descending_block_counts(int64_t b, int64_t s, int64_t* counts) {
  if (s == 1) { counts[0] = b; return; }
  int64_t num0 = (2 * b - s) * (s - 1), step = 2 * b - 2 * s, den = s * (s - 1), sum = 0;
  for (int64_t i = 0; i < s; ++i) {
    int64_t x = num0 - i * step; /* floor division as Python's // */
    int64_t q = x / den;
    if ((x % den != 0) && ((x < 0) != (den < 0))) --q;
    counts[i] = q;
    sum += q;
  }
  for (int64_t i = 0; i < b - sum; ++i) counts[i] += 1;
}

/* partition.py:98-140 get_partitions: returns the partition count */
EXPORT int64_t or_get_partitions(int64_t n, int64_t factor, int64_t threads, int64_t* starts, int64_t* ends) {
  int64_t total = (n + 511) / 512, req = factor * threads;
  int64_t np_ = req < total ? req : total;
  int64_t* counts = (int64_t*)malloc((size_t)(np_ > 0 ? np_ : 1) * sizeof(int64_t));
  descending_block_counts(total, np_, counts);
  int64_t be = 0;
  for (int64_t i = 0; i < np_; ++i) {
    starts[i] = i == 0 ? 0 : ends[i - 1];
    be += counts[i];
    ends[i] = be * 512 < n ? be * 512 : n;
  }
  free(counts);
  return np_;
}

/* partition.py:143-171 shrink_bounds over vis | ext (uint64 words) */
static void shrink_bounds(const uint64_t* vis, const uint64_t* ext, int64_t* plo, int64_t* phi) {
  int64_t lo = *plo, hi = *phi;
  while (hi - lo >= 512) {
    int64_t w0 = lo >> 6, ok = 1;
    for (int j = 0; j < 8; ++j) if ((vis[w0 + j] | ext[w0 + j]) != ~0ull) { ok = 0; break; }
    if (!ok) break;
    lo += 512;
  }
  while (hi - lo >= 512 && (hi & 511) == 0) {
    int64_t w0 = (hi >> 6) - 8, ok = 1;
    for (int j = 0; j < 8; ++j) if ((vis[w0 + j] | ext[w0 + j]) != ~0ull) { ok = 0; break; }
    if (!ok) break;
    hi -= 512;
  }
  *plo = lo;
  *phi = hi;
}

EXPORT void or_shrink_bounds(const uint64_t* vis, const uint64_t* ext, int64_t* lo, int64_t* hi) {
  shrink_bounds(vis, ext, lo, hi);
}

#define TD_CLAIM(w, v)                                                                    \
  do {                                                                                    \
    uint64_t mk_ = 1ull << ((w) & 63);                                                    \
    if (!(__atomic_load_n(&visited[(w) >> 6], __ATOMIC_RELAXED) & mk_)) {                 \
      uint64_t old_ = __atomic_fetch_or(&visited[(w) >> 6], mk_, __ATOMIC_RELAXED);       \
      if (!(old_ & mk_)) {                                                                \
        parent[w] = (int32_t)(v);                                                         \
        if (level) level[w] = (int32_t)(L + 1);                                           \
        nq[__atomic_fetch_add(&cursor, 1, __ATOMIC_RELAXED)] = (w);                       \
        deg_next += deg[w];                                                               \
      }                                                                                   \
    }                                                                                     \
  } while (0)

EXPORT int64_t or_bfs_run(int64_t n, const int64_t* rs, const uint32_t* dst, const uint32_t* dst_desc,
                          const int32_t* deg, int64_t source, int alpha, int beta, int mode, int factor,
                          int threads, int32_t* parent, int32_t* level, int64_t* rec, int64_t rec_cap,
                          double* elapsed) {
  int64_t nw = ((n + 511) / 512) * 8; /* whole 512-bit blocks (bitmap.py:21-24) */
  if (nw == 0) nw = 8;
  const int T = nthreads_of(threads);
  uint64_t* visited = (uint64_t*)calloc((size_t)nw, 8);
  uint64_t* fcur = (uint64_t*)calloc((size_t)nw, 8);
  uint64_t* fnext = (uint64_t*)calloc((size_t)nw, 8);
  uint32_t* q = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * 4);
  uint32_t* nq = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * 4);
  const int partitioned = mode >= 2; /* engine.py:67, 499-500 */
  int64_t *pst = NULL, *pen = NULL, *plo = NULL, *phi = NULL, n_parts = 0;
  if (partitioned && n >= 1) {
    int64_t cap = factor * (int64_t)T;
    pst = (int64_t*)malloc((size_t)cap * 8); pen = (int64_t*)malloc((size_t)cap * 8);
    plo = (int64_t*)malloc((size_t)cap * 8); phi = (int64_t*)malloc((size_t)cap * 8);
    n_parts = or_get_partitions(n, factor, T, pst, pen);
    memcpy(plo, pst, (size_t)n_parts * 8); /* ps.reset(): engine.py:530-531 */
    memcpy(phi, pen, (size_t)n_parts * 8);
  }
  /* reset (not timed): engine.py:526-532 */
  for (int64_t v = 0; v < n; ++v) {
    parent[v] = -1;
    if (level) level[v] = -1;
    if (deg[v] == 0) visited[v >> 6] |= 1ull << (v & 63); /* engine.py:432-437 */
  }
  parent[source] = (int32_t)source;
  if (level) level[source] = 0;
  visited[source >> 6] |= 1ull << (source & 63);

  double t0 = now_s();
  const int64_t m_directed = rs[n];
  int64_t nf = 1, m_f = deg[source], m_u = m_directed - deg[source];
  int q_valid = 1, bits_valid = 0; /* which frontier forms are present */
  q[0] = (uint32_t)source;
  int dir = 0;
  int64_t L = 0;
  const int64_t nblocks = (n + 511) / 512;
  const int hybrid = mode != 0;
  while (nf > 0) {
    const int use = hybrid ? dir : 0;
    int64_t n_next = 0, deg_next = 0, scanned = 0, pass1 = -1, live = -1, claimed = -1;
    if (use == 0) {
      if (!q_valid) { /* Frontier.to_queue_form: Bitmap.to_indices (bitmap.py:122-125) */
        int64_t c = 0;
        for (int64_t w = 0; w < nw; ++w) {
          uint64_t x = fcur[w];
          while (x) { int b0 = __builtin_ctzll(x); q[c++] = (uint32_t)(w * 64 + b0); x &= x - 1; }
        }
        q_valid = 1;
      }
      int64_t cursor = 0;
#pragma omp parallel num_threads(T) reduction(+ : deg_next, scanned)
      {
        int t = 0, TT = 1;
#ifdef _OPENMP
        t = omp_get_thread_num(); TT = omp_get_num_threads();
#endif
        if (!partitioned) { /* td_plain over _chunk_bounds */
          int64_t lo = nf * t / TT, hi = nf * (t + 1) / TT;
          for (int64_t i = lo; i < hi; ++i) {
            uint32_t v = q[i];
            for (int64_t j = rs[v]; j < rs[v + 1]; ++j) {
              uint32_t w = dst[j];
              ++scanned;
              TD_CLAIM(w, v);
            }
          }
        } else { /* td_striped (_kernels.py:90-141) */
          for (int64_t idx = 0; idx < nf; ++idx) {
            uint32_t v = q[idx];
            int64_t base = rs[v], d = rs[v + 1] - base, wl = d / TT;
            for (int64_t j = base + t * wl; j < base + (t + 1) * wl; ++j) {
              uint32_t w = dst[j];
              ++scanned;
              TD_CLAIM(w, v);
            }
            if (idx % TT == t)
              for (int64_t j = base + TT * wl; j < base + d; ++j) {
                uint32_t w = dst[j];
                ++scanned;
                TD_CLAIM(w, v);
              }
          }
        }
      }
      n_next = cursor;
      uint32_t* tq = q; q = nq; nq = tq;
      q_valid = 1; bits_valid = 0;
    } else {
      if (!bits_valid) { /* Frontier.to_bitmap_form: queue_to_bits (_kernels.py:296-301) */
        memset(fcur, 0, (size_t)nw * 8);
        for (int64_t i = 0; i < nf; ++i) fcur[q[i] >> 6] |= 1ull << (q[i] & 63);
        bits_valid = 1;
      }
      memset(fnext, 0, (size_t)nw * 8); /* fresh Bitmap(n) per step (engine.py:356) */
      const uint32_t* bdst = mode == 3 ? dst_desc : dst;
      int64_t pcur = 0, p1 = 0, cl = 0;
#pragma omp parallel num_threads(T) reduction(+ : n_next, deg_next, scanned, p1, cl)
      {
        int t = 0, TT = 1;
#ifdef _OPENMP
        t = omp_get_thread_num(); TT = omp_get_num_threads();
#endif
        if (mode <= 1) { /* bu_range over block-aligned static ranges (engine.py:355-370) */
          int64_t lo = (nblocks * t / TT) * 512, hi = (nblocks * (t + 1) / TT) * 512;
          if (lo > n) lo = n;
          if (hi > n || t == TT - 1) hi = n;
          for (int64_t v = lo; v < hi; ++v) {
            uint64_t mv = 1ull << (v & 63);
            if (visited[v >> 6] & mv) continue;
            int64_t a = rs[v], b = rs[v + 1];
            for (int64_t j = a; j < b; ++j) {
              uint32_t u = bdst[j];
              ++scanned;
              if (fcur[u >> 6] & (1ull << (u & 63))) {
                parent[v] = (int32_t)u;
                if (level) level[v] = (int32_t)(L + 1);
                visited[v >> 6] |= mv;
                fnext[v >> 6] |= mv;
                ++n_next;
                deg_next += b - a;
                break;
              }
            }
          }
        } else {
          while (1) {
            int64_t p = __atomic_fetch_add(&pcur, 1, __ATOMIC_RELAXED);
            if (p >= n_parts) break;
            ++cl;
            if (mode == 2) { /* bu_steal: live bounds read, not shrunk */
              for (int64_t v = plo[p]; v < phi[p]; ++v) {
                uint64_t mv = 1ull << (v & 63);
                if (visited[v >> 6] & mv) continue;
                int64_t a = rs[v], b = rs[v + 1];
                for (int64_t j = a; j < b; ++j) {
                  uint32_t u = bdst[j];
                  ++scanned;
                  if (fcur[u >> 6] & (1ull << (u & 63))) {
                    parent[v] = (int32_t)u;
                    if (level) level[v] = (int32_t)(L + 1);
                    visited[v >> 6] |= mv;
                    fnext[v >> 6] |= mv;
                    ++n_next;
                    deg_next += b - a;
                    break;
                  }
                }
              }
              continue;
            }
            /* bu_reduced (_kernels.py:217-293) */
            int64_t lo = plo[p], hi = phi[p];
            shrink_bounds(visited, fnext, &lo, &hi);
            const int64_t lo1 = lo, hi1 = hi;
            for (int64_t v = lo; v < hi; ++v) { /* pass 1: highest-degree neighbour only */
              uint64_t mv = 1ull << (v & 63);
              if ((visited[v >> 6] | fnext[v >> 6]) & mv) continue;
              int64_t a = rs[v];
              if (rs[v + 1] == a) continue;
              uint32_t u = bdst[a];
              ++scanned;
              if (fcur[u >> 6] & (1ull << (u & 63))) {
                parent[v] = (int32_t)u;
                if (level) level[v] = (int32_t)(L + 1);
                fnext[v >> 6] |= mv;
                ++n_next; ++p1;
                deg_next += rs[v + 1] - a;
              }
            }
            shrink_bounds(visited, fnext, &lo, &hi);
            for (int64_t v = lo; v < hi; ++v) { /* pass 2: the rest, early break */
              uint64_t mv = 1ull << (v & 63);
              if ((visited[v >> 6] | fnext[v >> 6]) & mv) continue;
              int64_t a = rs[v], b = rs[v + 1];
              for (int64_t j = a + 1; j < b; ++j) {
                uint32_t u = bdst[j];
                ++scanned;
                if (fcur[u >> 6] & (1ull << (u & 63))) {
                  parent[v] = (int32_t)u;
                  if (level) level[v] = (int32_t)(L + 1);
                  fnext[v >> 6] |= mv;
                  ++n_next;
                  deg_next += b - a;
                  break;
                }
              }
            }
            shrink_bounds(visited, fnext, &lo, &hi);
            plo[p] = lo;
            phi[p] = hi;
            for (int64_t w = lo1 >> 6; w < (hi1 + 63) >> 6; ++w) visited[w] |= fnext[w]; /* publish */
          }
        }
      }
      if (mode >= 2) claimed = cl;
      if (mode == 3) pass1 = p1;
      if (partitioned) { /* ps.live_total() (partition.py:70-72) */
        live = 0;
        for (int64_t p = 0; p < n_parts; ++p) live += phi[p] - plo[p];
      }
      uint64_t* tb = fcur; fcur = fnext; fnext = tb;
      bits_valid = 1; q_valid = 0;
    }
    if (L < rec_cap) {
      int64_t* r = rec + 9 * L;
      r[0] = L; r[1] = use; r[2] = nf; r[3] = m_f; r[4] = m_u; r[5] = scanned;
      r[6] = pass1; r[7] = live; r[8] = claimed;
    }
    m_u -= deg_next; /* engine.py:587-589 */
    m_f = deg_next;
    nf = n_next;
    if (hybrid) { /* update_traversal_policy, engine.py:215-228 (n = g.n) */
      if (use == 0) dir = ((double)m_f > (double)m_u / (double)alpha) ? 1 : 0;
      else dir = ((double)nf < (double)n / (double)beta) ? 0 : 1;
    }
    ++L;
  }
  *elapsed = now_s() - t0;
  free(visited); free(fcur); free(fnext); free(q); free(nq);
  free(pst); free(pen); free(plo); free(phi);
  return L;
}

/* ------------------------------------------------------------------------ */
/* Generators (BASELINE inputs) -- generator.py:74-148 with numpy's Philox  */
/* bit generator (philox4x64-10: counter incremented before each block, so  */
/* block b of a stream has counter b + 1; Generator.random() = (x>>11)*2^-53)*/

static inline void philox_block(uint64_t ctr0, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
  for (int r = 0; r < 10; ++r) {
    const __uint128_t p0 = (__uint128_t)0xD2E7470EE14C6C93ull * c0;
    const __uint128_t p1 = (__uint128_t)0xCA5A826395121157ull * c2;
    const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static uint64_t splitmix64(uint64_t x) { /* generator.py:74-79 */
  x = x + 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* kronecker_generate (generator.py:114-148): 65,536-edge chunks, chunk c a  */
/* Generator(Philox(key=[seed, c])), count x scale doubles row-major, column */
/* 0 the most significant level; ids scrambled (generator.py:82-111).       */
EXPORT void or_kronecker_generate(int scale, int64_t edgefactor, uint64_t seed, double a, double b, double c,
                                  int threads, uint32_t* out) {
  const int64_t m = ((int64_t)1 << scale) * edgefactor, CH = 1 << 16;
  const double t1 = a, t2 = a + b, t3 = a + b + c;
  const uint64_t mask = ((uint64_t)1 << scale) - 1;
  uint64_t mult[3], add[3];
  int shift[3] = {scale / 2 > 1 ? scale / 2 : 1, scale / 3 > 1 ? scale / 3 : 1,
                  (2 * scale) / 3 > 1 ? (2 * scale) / 3 : 1};
  uint64_t x = seed ^ 0xD6E8FEB86659FD93ull;
  for (int r = 0; r < 3; ++r) {
    x = splitmix64(x);
    mult[r] = x | 1;
    x = splitmix64(x);
    add[r] = x & mask;
  }
  const int64_t chunks = (m + CH - 1) / CH;
#pragma omp parallel for num_threads(nthreads_of(threads)) schedule(dynamic, 1)
  for (int64_t ch = 0; ch < chunks; ++ch) {
    const int64_t lo = ch * CH, hi = lo + CH < m ? lo + CH : m;
    uint64_t words[4];
    int64_t j = 0; /* draw index inside the chunk */
    for (int64_t e = lo; e < hi; ++e) {
      uint64_t src = 0, dstv = 0;
      for (int t = 0; t < scale; ++t, ++j) {
        if ((j & 3) == 0) philox_block((uint64_t)(j >> 2) + 1, seed, (uint64_t)ch, words);
        const double u = (double)(words[j & 3] >> 11) * (1.0 / 9007199254740992.0);
        const int qd = (u >= t1) + (u >= t2) + (u >= t3);
        src = (src << 1) | (uint64_t)((qd >> 1) & 1);
        dstv = (dstv << 1) | (uint64_t)(qd & 1);
      }
      for (int r = 0; r < 3; ++r) {
        src = (src * mult[r]) & mask; src ^= src >> shift[r]; src = (src + add[r]) & mask;
        dstv = (dstv * mult[r]) & mask; dstv ^= dstv >> shift[r]; dstv = (dstv + add[r]) & mask;
      }
      out[2 * e] = (uint32_t)src;
      out[2 * e + 1] = (uint32_t)dstv;
    }
  }
}

/* Chung-Lu endpoint sampling (configs[4]; the recipe of                    */
/* paper_2012_10026_b200/generator.py ChungLuParams, steps 3): pair j uses   */
/* raw words 2i, 2i+1 (i = j mod 65536) of Philox(key=[seed, 2^32 + j/65536])*/
/* and picks the first vertex whose inclusive weight prefix exceeds          */
/* floor(x * T / 2^64).  The float step (weights) stays in numpy.           */
EXPORT void or_chunglu_sample(const int64_t* prefix, int64_t n, int64_t m, uint64_t seed, int threads, uint32_t* out) {
  const uint64_t T = (uint64_t)prefix[n - 1], CH = 1 << 16;
  const int64_t chunks = (m + (int64_t)CH - 1) / (int64_t)CH;
#pragma omp parallel for num_threads(nthreads_of(threads)) schedule(dynamic, 1)
  for (int64_t ch = 0; ch < chunks; ++ch) {
    const int64_t lo = ch * (int64_t)CH, hi = lo + (int64_t)CH < m ? lo + (int64_t)CH : m;
    uint64_t words[4];
    for (int64_t jj = lo; jj < hi; ++jj) {
      const int64_t i = jj - lo;
      if (((2 * i) & 3) == 0) philox_block((uint64_t)((2 * i) >> 2) + 1, seed, (1ull << 32) + (uint64_t)ch, words);
      for (int t = 0; t < 2; ++t) {
        const uint64_t r = (uint64_t)(((__uint128_t)words[(2 * i + t) & 3] * T) >> 64);
        int64_t a0 = 0, b0 = n - 1; /* searchsorted(prefix, r, side="right") */
        while (a0 < b0) {
          const int64_t mid = (a0 + b0) >> 1;
          if ((uint64_t)prefix[mid] > r) b0 = mid; else a0 = mid + 1;
        }
        out[2 * jj + t] = (uint32_t)a0;
      }
    }
  }
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
