// rb_prep.cu -- graph preprocessing on device: CSR build, RCM relabelling,
// permutation apply and degree-sorted adjacency.
//
// build_csr (graph.py:85-120): both orientations of every non-loop pair become
// 64-bit keys (u << 32 | v); one radix sort over the significant bits plus a
// unique pass yields exactly the reference's np.unique order (CSR order), row
// offsets are filled from the key boundaries.
//
// rcm (reorder.py:198-237): the reference's sequential Cuthill-McKee walk
// (_rcm_walk, reorder.py:106-148) is reproduced bit-exactly by a
// level-synchronous multi-source BFS:
//   * rank[v]  = position of v in V+ sorted by (degree, id)   (stable radix sort)
//   * components by union-find in rank space, hooking to the smaller rank, so
//     each root is the component's minimum-rank vertex = the walk's seed;
//     components are laid out in seed-rank order (prefix sum of sizes)
//   * per level, every newly reached w gets key (min CM position of a
//     frontier neighbour, rank[w]); sorting the level by that key and
//     numbering consecutively inside each component reproduces the walk
//     (parents are processed in position order, rows in (deg,id) order).
// perm = reverse(CM order) ++ isolated ascending.
//
// apply_permutation (reorder.py:254-271): degrees gathered through perm,
// int64 exclusive scan, rows gathered and mapped through inv, then a segmented
// sort makes every row ascending.
//
// Sorting/scanning building blocks come from CUB (ships with the CUDA
// toolkit); the graph kernels around them are hand-written.
#include <cub/cub.cuh>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "rb_common.cuh"
#include "rb_error.h"

namespace {

constexpr uint64_t kSentinel = ~0ull;
constexpr uint32_t kUnset = 0xffffffffu;

inline int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

struct Carver {  // carve a caller workspace into aligned pieces
  char* base;
  size_t off = 0;
  size_t cap;
  Carver(void* b, size_t c) : base((char*)b), cap(c) {}
  template <class T>
  T* take(size_t count) {
    size_t o = align_up(off);
    off = o + count * sizeof(T);
    return base ? (T*)(base + o) : nullptr;
  }
};

int grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (int)b;
}

struct MaxOp {
  __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

// ---------------------------------------------------------------------------
// CSR build

__global__ void csr_make_keys(const uint32_t* __restrict__ edges, int64_t m, int64_t n, uint64_t* __restrict__ keys,
                              unsigned long long* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint2 e = reinterpret_cast<const uint2*>(edges)[i];
    uint64_t k0 = kSentinel, k1 = kSentinel;
    if ((int64_t)e.x >= n || (int64_t)e.y >= n) {
      atomicMin(bad, (unsigned long long)i);
    } else if (e.x != e.y) {
      k0 = ((uint64_t)e.x << 32) | e.y;
      k1 = ((uint64_t)e.y << 32) | e.x;
    }
    keys[2 * i] = k0;
    keys[2 * i + 1] = k1;
  }
}

// row_starts from sorted unique keys: every boundary i fills rs[prev_src+1 .. src]
__global__ void csr_emit(const uint64_t* __restrict__ keys, int64_t md, int64_t n, int64_t* __restrict__ rs,
                         int32_t* __restrict__ col) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= md; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = (i < md) ? (int64_t)(keys[i] >> 32) : n;
    const int64_t ps = (i > 0) ? (int64_t)(keys[i - 1] >> 32) : -1;
    for (int64_t v = ps + 1; v <= s; ++v) rs[v] = i;
    if (i < md) col[i] = (int32_t)(keys[i] & 0xffffffffu);
  }
}

__global__ void degrees_from_rs(const int64_t* __restrict__ rs, int64_t n, int32_t* __restrict__ deg) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    deg[v] = (int32_t)(rs[v + 1] - rs[v]);
}

struct CsrHeader {
  int64_t m_directed;
  int64_t result_off;  // byte offset of the unique keys inside the workspace
  int64_t pad[6];
};

size_t csr_ws(int64_t m_raw, int64_t n, void* ws, size_t cap, uint64_t** A, uint64_t** B, void** temp,
              size_t* temp_bytes, unsigned long long** bad, int64_t** nsel) {
  const int64_t nk = 2 * m_raw;
  Carver c(ws, cap);
  c.take<CsrHeader>(1);
  *A = c.take<uint64_t>(nk > 0 ? nk : 1);
  *B = c.take<uint64_t>(nk > 0 ? nk : 1);
  *bad = c.take<unsigned long long>(1);
  *nsel = c.take<int64_t>(1);
  size_t t1 = 0, t2 = 0;
  cub::DoubleBuffer<uint64_t> db(*A, *B);
  cub::DeviceRadixSort::SortKeys(nullptr, t1, db, nk, 0, 64);
  cub::DeviceSelect::Unique(nullptr, t2, *A, *B, *nsel, nk);
  *temp_bytes = std::max(t1, t2);
  *temp = c.take<char>(*temp_bytes);
  return c.off + 256;
}

// ---------------------------------------------------------------------------
// RCM kernels

__global__ void iota_u32(uint32_t* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

__global__ void copy_deg_u32(const int32_t* deg, uint32_t* out, int64_t n, unsigned long long* iso) {
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = (uint32_t)deg[i];
    local += deg[i] == 0;
  }
  local = rb::warp_sum_u64(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(iso, local);
}

// rank[v] = index of v in V+ (sorted by (deg,id)); isolated get kUnset
__global__ void set_rank(const uint32_t* sorted_ids, int64_t iso, int64_t n, uint32_t* rank) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = sorted_ids[i];
    rank[v] = i < iso ? kUnset : (uint32_t)(i - iso);
  }
}

__device__ __forceinline__ int32_t uf_rep(int32_t* uf, int32_t x) {
  int32_t cur = __ldcg(uf + x);
  if (cur != x) {
    int32_t prev = x, next;
    while (cur > (next = __ldcg(uf + cur))) {
      uf[prev] = next;  // path halving; values only decrease (benign race)
      prev = cur;
      cur = next;
    }
  }
  return cur;
}

__device__ __forceinline__ void uf_hook(int32_t* uf, int32_t a, int32_t b) {
  int32_t ra = uf_rep(uf, a), rb_ = uf_rep(uf, b);
  while (ra != rb_) {
    if (ra < rb_) {
      const int32_t ret = atomicCAS(uf + rb_, rb_, ra);
      if (ret == rb_) break;
      rb_ = uf_rep(uf, ret);
    } else {
      const int32_t ret = atomicCAS(uf + ra, ra, rb_);
      if (ret == ra) break;
      ra = uf_rep(uf, ret);
    }
  }
}

// union-find over edges in rank space; light rows thread-per-row, heavy rows warp-per-row
__global__ void cc_hook_light(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                              const uint32_t* __restrict__ rank, int64_t n, int32_t* uf) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = rs[v], e = rs[v + 1];
    if (e - s > 32 || e == s) continue;
    const int32_t rv = (int32_t)rank[v];
    for (int64_t j = s; j < e; ++j) {
      const int32_t rw = (int32_t)rank[col[j]];
      if (rw < rv) uf_hook(uf, rv, rw);
    }
  }
}

__global__ void cc_hook_heavy(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                              const uint32_t* __restrict__ rank, int64_t n, int32_t* uf) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int64_t s = rs[v], e = rs[v + 1];
    if (e - s <= 32) continue;
    const int32_t rv = (int32_t)rank[v];
    for (int64_t j = s + lane; j < e; j += 32) {
      const int32_t rw = (int32_t)rank[col[j]];
      if (rw < rv) uf_hook(uf, rv, rw);
    }
  }
}

// Afforest-style components (rank space, root = min rank): every vertex first
// hooks its first kSample neighbours (short chains, spread over all roots);
// after compression the most frequent root is the giant component's, and the
// full edge pass skips every vertex already in it -- an edge leaving the
// giant set is still seen from its other endpoint, whose row is processed
// (the CSR holds both directions).  Replaces hooking all 2m edges, which
// hot-spots atomics on the giant component's root.
constexpr int kSample = 2;

__global__ void cc_sample(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                          const uint32_t* __restrict__ rank, int64_t n, int32_t* uf) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = rs[v], e = rs[v + 1];
    if (e == s) continue;
    const int32_t rv = (int32_t)rank[v];
    for (int64_t j = s; j < e && j < s + kSample; ++j) {
      const int32_t rw = (int32_t)rank[col[j]];
      if (rw != rv) uf_hook(uf, rv, rw);
    }
  }
}

__global__ void cc_compress(int32_t* uf, int64_t k) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x)
    uf[r] = uf_rep(uf, (int32_t)r);
}

// the root of sample i (i < 1024): ranks spread evenly over [0, k)
__global__ void cc_probe_roots(const int32_t* uf, int64_t k, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 1024) out[i] = uf_rep(const_cast<int32_t*>(uf), (int32_t)(((int64_t)i * k) / 1024));
}

__global__ void cc_hook_rest_light(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                                   const uint32_t* __restrict__ rank, int64_t n, int32_t giant, int32_t* uf) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = rs[v] + kSample, e = rs[v + 1];
    if (e - s > 32 || e <= s) continue;
    const int32_t rv = (int32_t)rank[v];
    if (uf_rep(uf, rv) == giant) continue;
    for (int64_t j = s; j < e; ++j) {
      const int32_t rw = (int32_t)rank[col[j]];
      if (rw != rv) uf_hook(uf, rv, rw);
    }
  }
}

__global__ void cc_hook_rest_heavy(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                                   const uint32_t* __restrict__ rank, int64_t n, int32_t giant, int32_t* uf) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int64_t s = rs[v] + kSample, e = rs[v + 1];
    if (e - s <= 32) continue;
    const int32_t rv = (int32_t)rank[v];
    if (uf_rep(uf, rv) == giant) continue;  // (warp-uniform)
    for (int64_t j = s + lane; j < e; j += 32) {
      const int32_t rw = (int32_t)rank[col[j]];
      if (rw != rv) uf_hook(uf, rv, rw);
    }
  }
}

__global__ void cc_finalize(int32_t* uf, int64_t k, uint32_t* comp_size) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x) {
    int32_t x = (int32_t)r;
    while (true) {
      const int32_t p = __ldcg(uf + x);
      if (p == x) break;
      x = p;
    }
    uf[r] = x;
  }
}

__global__ void cc_sizes(const int32_t* uf, int64_t k, uint32_t* comp_size) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k + 31; r += (int64_t)gridDim.x * blockDim.x) {
    // whole warps participate (loop bound padded) so match_any is safe
    const bool act = r < k;
    const int32_t c = act ? uf[r] : -1;
    const uint32_t peers = __match_any_sync(__activemask(), c);
    const int leader = __ffs(peers) - 1;
    if (act && (int)(threadIdx.x & 31) == leader) atomicAdd(comp_size + c, (uint32_t)__popc(peers));
  }
}

__global__ void root_flags(const int32_t* uf, int64_t k, uint32_t* flag) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x)
    flag[r] = uf[r] == (int32_t)r;
}

// seeds: frontier[idx] = vplus[root], pos/cursor, component ranges (ascending start)
__global__ void seed_components(const int32_t* uf, const uint32_t* comp_off, const uint32_t* comp_size,
                                const uint32_t* root_idx, const uint32_t* vplus, int64_t k, int64_t nc,
                                uint32_t* pos, uint32_t* cursor, uint32_t* frontier, int64_t* ranges) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x) {
    if (uf[r] != (int32_t)r) continue;
    const uint32_t v = vplus[r];
    const uint32_t o = comp_off[r];
    pos[v] = o;
    cursor[r] = o + 1;
    const uint32_t idx = root_idx[r];
    frontier[idx] = v;
    const int64_t sz = comp_size[r];
    // discovery range [o, o+sz) -> new ids [k-o-sz, k-o); listed ascending by start
    ranges[2 * (nc - 1 - idx)] = k - (int64_t)o - sz;
    ranges[2 * (nc - 1 - idx) + 1] = k - (int64_t)o;
  }
}

// expand one CM level: warp per frontier vertex
__global__ void rcm_expand(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                           const uint32_t* __restrict__ frontier, int64_t nf, const uint32_t* pos, uint32_t* minpos,
                           uint32_t* next, unsigned long long* next_count) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (int64_t i = warp; i < nf; i += nwarps) {
    const uint32_t v = frontier[i];
    const uint32_t p = pos[v];
    const int64_t s = rs[v], e = rs[v + 1];
    for (int64_t j0 = s; j0 < e; j0 += 32) {
      const int64_t j = j0 + lane;
      bool fresh = false;
      uint32_t w = 0;
      if (j < e) {
        w = (uint32_t)col[j];
        if (__ldcg(pos + w) == kUnset) {
          const uint32_t old = atomicMin(minpos + w, p);
          fresh = old == kUnset;
        }
      }
      const uint32_t fm = __ballot_sync(RB_FULL, fresh);
      if (fm) {
        const int leader = __ffs(fm) - 1;
        unsigned long long base = 0;
        if ((int)lane == leader) base = atomicAdd(next_count, (unsigned long long)__popc(fm));
        base = __shfl_sync(RB_FULL, base, leader);
        if (fresh) next[base + __popc(fm & ((1u << lane) - 1u))] = w;
      }
    }
  }
}

__global__ void rcm_keys(const uint32_t* next, int64_t cnt, const uint32_t* minpos, const uint32_t* rank, int b,
                         uint64_t* keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w = next[i];
    keys[i] = ((uint64_t)minpos[w] << b) | rank[w];
  }
}

// sorted keys -> vertices + group heads (component boundaries)
__global__ void rcm_heads(const uint64_t* keys, int64_t cnt, int b, const uint32_t* vplus, const int32_t* uf,
                          uint32_t* verts, int64_t* head) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(keys[i] & mask);
    verts[i] = vplus[r];
    bool h = i == 0;
    if (!h) h = uf[(uint32_t)(keys[i - 1] & mask)] != uf[r];
    head[i] = h ? i : 0;
  }
}

__global__ void rcm_assign(const uint64_t* keys, int64_t cnt, int b, const int32_t* uf, const int64_t* gstart,
                           const uint32_t* verts, uint32_t* pos, uint32_t* cursor) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(keys[i] & mask);
    const int32_t c = uf[r];
    pos[verts[i]] = cursor[c] + (uint32_t)(i - gstart[i]);
  }
}

// after rcm_assign: the last vertex of each component group advances its cursor
__global__ void rcm_advance(const uint64_t* keys, int64_t cnt, int b, const int32_t* uf, const uint32_t* verts,
                            const uint32_t* pos, uint32_t* cursor) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = uf[(uint32_t)(keys[i] & mask)];
    const bool last = (i + 1 == cnt) || uf[(uint32_t)(keys[i + 1] & mask)] != c;
    if (last) cursor[c] = pos[verts[i]] + 1;  // next level of this component continues here
  }
}

__global__ void rcm_perm(const uint32_t* pos, const uint32_t* sorted_ids, const uint32_t* rank, int64_t n, int64_t iso,
                         int64_t k, uint32_t* perm, uint32_t* inv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = sorted_ids[i];
    uint32_t nv;
    if (i < iso) nv = (uint32_t)(k + i);              // isolated, ascending id (stable sort)
    else nv = (uint32_t)(k - 1 - (int64_t)pos[v]);    // reversed CM position
    perm[nv] = v;
    inv[v] = nv;
  }
}

// ---------------------------------------------------------------------------
// permutation apply / degree sort

__global__ void gather_deg(const int32_t* deg, const uint32_t* perm, int64_t n, int32_t* deg_out, int64_t* deg64) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = deg[perm[i]];
    deg_out[i] = d;
    deg64[i] = d;
  }
}

__global__ void gather_rows(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                            const uint32_t* __restrict__ perm, const uint32_t* __restrict__ inv,
                            const int64_t* __restrict__ rs_new, int64_t n, int32_t* __restrict__ out) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t nv = warp; nv < n; nv += nwarps) {
    const uint32_t ov = perm[nv];
    const int64_t s = rs[ov], e = rs[ov + 1], b = rs_new[nv];
    for (int64_t j = s + lane; j < e; j += 32) out[b + (j - s)] = (int32_t)inv[col[j]];
  }
}

// Relabel by transposition (undirected graphs: every edge is stored in both
// directions).  New row nv = old row perm[nv]; its entries are emitted as pairs
// (key = the neighbour's new id, value = nv) in new-row order.  A STABLE sort by
// key then lists, for every new vertex x, the new ids of the vertices adjacent
// to it in ascending order -- by symmetry exactly row x of the relabelled graph
// -- so the sorted values ARE the new column array: log2(n) key bits of one
// radix sort instead of a sort inside every row (the segmented sort of the hub
// rows was the largest preprocessing cost at scale 26).
__global__ void relabel_pairs(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                              const uint32_t* __restrict__ perm, const uint32_t* __restrict__ inv,
                              const int64_t* __restrict__ rs_new, int64_t n, uint32_t* __restrict__ keys,
                              uint32_t* __restrict__ vals) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t nv = warp; nv < n; nv += nwarps) {
    const uint32_t ov = perm[nv];
    const int64_t s = rs[ov], e = rs[ov + 1], b = rs_new[nv];
    for (int64_t j = s + lane; j < e; j += 32) {
      keys[b + (j - s)] = inv[col[j]];
      vals[b + (j - s)] = (uint32_t)nv;
    }
  }
}

// The sorted keys must fill every new row exactly (key x on [rs_new[x], rs_new[x+1])):
// true for a symmetric graph; *bad counts the rows where it fails.
__global__ void relabel_check(const uint32_t* __restrict__ keys, const int64_t* __restrict__ rs_new, int64_t n,
                              unsigned long long* __restrict__ bad) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = rs_new[v], e = rs_new[v + 1];
    if (e > s && (keys[s] != (uint32_t)v || keys[e - 1] != (uint32_t)v)) atomicAdd(bad, 1ull);
  }
}

__global__ void degree_keys(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ deg, int64_t n, int descending, uint64_t* __restrict__ keys) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int64_t s = rs[v], e = rs[v + 1];
    for (int64_t j = s + lane; j < e; j += 32) {
      const uint32_t w = (uint32_t)col[j];
      const uint64_t d = (uint64_t)deg[w];
      const uint64_t dd = descending ? ((1ull << 31) - d) : d;  // reorder.py:160-163
      keys[j] = (dd << 32) | w;
    }
  }
}

__global__ void keys_low32(const uint64_t* keys, int64_t m, int32_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)(keys[i] & 0xffffffffu);
}

__global__ void rel_offsets(const int64_t* rs, int64_t v0, int64_t nseg, int32_t* out) {
  const int64_t base = rs[v0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nseg; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)(rs[v0 + i] - base);
}

// Row batches with <= kBatchItems entries so CUB's int item counts never overflow.
constexpr int64_t kBatchItems = 1ll << 30;

std::vector<std::pair<int64_t, int64_t>> row_batches(const int64_t* d_rs, int64_t n, int64_t m, cudaStream_t s) {
  std::vector<std::pair<int64_t, int64_t>> out;
  if (m <= kBatchItems) {
    out.push_back({0, n});
    return out;
  }
  std::vector<int64_t> h(n + 1);
  cudaMemcpyAsync(h.data(), d_rs, (n + 1) * 8, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  int64_t v0 = 0;
  while (v0 < n) {
    int64_t v1 = v0 + 1;
    // largest v1 with h[v1]-h[v0] <= kBatchItems (at least one row)
    int64_t lo = v0 + 1, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) / 2;
      if (h[mid] - h[v0] <= kBatchItems) lo = mid; else hi = mid - 1;
    }
    v1 = std::max(lo, v0 + 1);
    out.push_back({v0, v1});
    v0 = v1;
  }
  return out;
}

template <class K>
size_t segsort_temp_bytes(int64_t n, int64_t m) {
  size_t t = 0;
  const int items = (int)std::min<int64_t>(std::max<int64_t>(m, 1), kBatchItems);
  const int segs = (int)std::min<int64_t>(std::max<int64_t>(n, 1), (int64_t)INT32_MAX - 1);
  cub::DeviceSegmentedSort::SortKeys((void*)nullptr, t, (const K*)nullptr, (K*)nullptr, items, segs,
                                     (const int32_t*)nullptr, (const int32_t*)nullptr);
  return t;
}

// Sort every row of keys_in[rs[v]..rs[v+1]) into keys_out (batched over rows).
template <class K>
int segmented_sort_rows(const int64_t* d_rs, int64_t n, int64_t m, const K* in, K* out, void* temp, size_t temp_bytes,
                        int32_t* rel, cudaStream_t s) {
  if (m == 0 || n == 0) return RB_OK;
  for (auto [v0, v1] : row_batches(d_rs, n, m, s)) {
    const int64_t nseg = v1 - v0;
    rel_offsets<<<grid_for(nseg + 1), 256, 0, s>>>(d_rs, v0, nseg, rel);
    int64_t base = 0, end = 0;
    RB_CUDA_TRY(cudaMemcpyAsync(&base, d_rs + v0, 8, cudaMemcpyDeviceToHost, s));
    RB_CUDA_TRY(cudaMemcpyAsync(&end, d_rs + v1, 8, cudaMemcpyDeviceToHost, s));
    RB_CUDA_TRY(cudaStreamSynchronize(s));
    size_t tb = temp_bytes;
    RB_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(temp, tb, in + base, out + base, (int)(end - base), (int)nseg, rel,
                                                   rel + 1, s));
  }
  return RB_OK;
}

}  // namespace

// ===========================================================================
// C ABI

extern "C" size_t rb_csr_workspace_bytes(int64_t m_raw, int64_t n) {
  uint64_t *A, *B;
  void* temp;
  size_t tb;
  unsigned long long* bad;
  int64_t* nsel;
  return csr_ws(m_raw, n, nullptr, SIZE_MAX, &A, &B, &temp, &tb, &bad, &nsel);
}

extern "C" int rb_csr_build(const uint32_t* d_edges, int64_t m_raw, int64_t n, void* d_ws, size_t ws_bytes,
                            int64_t* m_directed, int64_t* bad_index, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0 || m_raw < 0 || !d_ws) {
    rb_set_error("rb_csr_build: invalid argument");
    return RB_ERR_ARG;
  }
  if (n >= (1ll << 31)) {
    rb_set_error("rb_csr_build: n=%lld exceeds int32 column ids", (long long)n);
    return RB_ERR_ARG;
  }
  uint64_t *A, *B;
  void* temp;
  size_t tb;
  unsigned long long* bad;
  int64_t* nsel;
  size_t need = csr_ws(m_raw, n, d_ws, ws_bytes, &A, &B, &temp, &tb, &bad, &nsel);
  if (need > ws_bytes) {
    rb_set_error("rb_csr_build: workspace too small (%zu < %zu)", ws_bytes, need);
    return RB_ERR_ARG;
  }
  CsrHeader hdr{};
  const int64_t nk = 2 * m_raw;
  if (m_raw == 0) {
    hdr.m_directed = 0;
    hdr.result_off = (char*)A - (char*)d_ws;
    RB_CUDA_TRY(cudaMemcpyAsync(d_ws, &hdr, sizeof(hdr), cudaMemcpyHostToDevice, s));
    RB_CUDA_TRY(cudaStreamSynchronize(s));
    *m_directed = 0;
    return RB_OK;
  }
  RB_CUDA_TRY(cudaMemsetAsync(bad, 0xff, 8, s));
  csr_make_keys<<<grid_for(m_raw), 256, 0, s>>>(d_edges, m_raw, n, A, bad);
  RB_CUDA_TRY(cudaGetLastError());
  unsigned long long hbad = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad != ~0ull) {
    *bad_index = (int64_t)hbad;
    rb_set_error("edge %lld out of range for n=%lld", (long long)hbad, (long long)n);
    return RB_ERR_ARG;
  }
  const int end_bit = 32 + std::max(1, bits_for((uint64_t)(n > 0 ? n - 1 : 0)));
  cub::DoubleBuffer<uint64_t> db(A, B);
  size_t t = tb;
  RB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(temp, t, db, nk, 0, end_bit, s));
  uint64_t* sorted = db.Current();
  uint64_t* uniq = db.Alternate();
  t = tb;
  RB_CUDA_TRY(cub::DeviceSelect::Unique(temp, t, sorted, uniq, nsel, nk, s));
  int64_t nu = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&nu, nsel, 8, cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  uint64_t last = 0;
  if (nu > 0) {
    RB_CUDA_TRY(cudaMemcpyAsync(&last, uniq + nu - 1, 8, cudaMemcpyDeviceToHost, s));
    RB_CUDA_TRY(cudaStreamSynchronize(s));
  }
  const int64_t md = (nu > 0 && last == kSentinel) ? nu - 1 : nu;
  hdr.m_directed = md;
  hdr.result_off = (char*)uniq - (char*)d_ws;
  RB_CUDA_TRY(cudaMemcpyAsync(d_ws, &hdr, sizeof(hdr), cudaMemcpyHostToDevice, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  *m_directed = md;
  return RB_OK;
}

extern "C" int rb_csr_emit(const void* d_ws, int64_t m_directed, int64_t n, int64_t* d_row_starts, int32_t* d_col,
                           int32_t* d_degrees, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CsrHeader hdr;
  RB_CUDA_TRY(cudaMemcpyAsync(&hdr, d_ws, sizeof(hdr), cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  if (hdr.m_directed != m_directed) {
    rb_set_error("rb_csr_emit: m_directed mismatch (%lld vs %lld)", (long long)m_directed,
                 (long long)hdr.m_directed);
    return RB_ERR_ARG;
  }
  const uint64_t* keys = (const uint64_t*)((const char*)d_ws + hdr.result_off);
  csr_emit<<<grid_for(m_directed + 1), 256, 0, s>>>(keys, m_directed, n, d_row_starts, d_col);
  RB_CUDA_TRY(cudaGetLastError());
  if (n > 0) degrees_from_rs<<<grid_for(n), 256, 0, s>>>(d_row_starts, n, d_degrees);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

// ---------------------------------------------------------------------------

namespace {
struct RcmWs {
  uint32_t *deg_a, *deg_b, *ids_a, *ids_b, *rank, *pos, *minpos, *comp_size, *comp_off, *rflag, *ridx, *cursor;
  uint32_t *lst_a, *lst_b, *verts;
  int32_t* uf;
  uint64_t *keys_a, *keys_b;
  int64_t *head, *gstart;
  unsigned long long* ctr;
  void* temp;
  size_t temp_bytes;
  size_t total;
};

RcmWs rcm_ws(int64_t n, int64_t m, void* base, size_t cap) {
  RcmWs w{};
  Carver c(base, cap);
  const size_t N = (size_t)std::max<int64_t>(n, 1);
  w.deg_a = c.take<uint32_t>(N);
  w.deg_b = c.take<uint32_t>(N);
  w.ids_a = c.take<uint32_t>(N);
  w.ids_b = c.take<uint32_t>(N);
  w.rank = c.take<uint32_t>(N);
  w.pos = c.take<uint32_t>(N);
  w.minpos = c.take<uint32_t>(N);
  w.comp_size = c.take<uint32_t>(N);
  w.comp_off = c.take<uint32_t>(N);
  w.rflag = c.take<uint32_t>(N);
  w.ridx = c.take<uint32_t>(N);
  w.cursor = c.take<uint32_t>(N);
  w.lst_a = c.take<uint32_t>(N);
  w.lst_b = c.take<uint32_t>(N);
  w.verts = c.take<uint32_t>(N);
  w.uf = c.take<int32_t>(N);
  w.keys_a = c.take<uint64_t>(N);
  w.keys_b = c.take<uint64_t>(N);
  w.head = c.take<int64_t>(N);
  w.gstart = c.take<int64_t>(N);
  w.ctr = c.take<unsigned long long>(8);
  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  {
    cub::DoubleBuffer<uint32_t> dk(w.deg_a, w.deg_b), dv(w.ids_a, w.ids_b);
    cub::DeviceRadixSort::SortPairs(nullptr, t1, dk, dv, (int64_t)N, 0, 32);
    cub::DoubleBuffer<uint64_t> kk(w.keys_a, w.keys_b);
    cub::DeviceRadixSort::SortKeys(nullptr, t2, kk, (int64_t)N, 0, 64);
    cub::DeviceScan::ExclusiveSum(nullptr, t3, w.comp_size, w.comp_off, (int64_t)N);
    cub::DeviceScan::InclusiveScan(nullptr, t4, w.head, w.gstart, MaxOp(), (int64_t)N);
  }
  w.temp_bytes = std::max(std::max(t1, t2), std::max(t3, t4));
  w.temp = c.take<char>(w.temp_bytes);
  w.total = c.off + 256;
  (void)m;
  return w;
}
}  // namespace

extern "C" size_t rb_rcm_workspace_bytes(int64_t n, int64_t m_directed) {
  return rcm_ws(n, m_directed, nullptr, SIZE_MAX).total;
}

extern "C" int rb_rcm(const int64_t* d_rs, const int32_t* d_col, const int32_t* d_deg, int64_t n, void* d_ws,
                      size_t ws_bytes, uint32_t* d_perm, uint32_t* d_inv, int64_t* n_plus, int64_t* d_ranges,
                      int64_t* n_components, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0 || n >= (1ll << 31)) {
    rb_set_error("rb_rcm: invalid n=%lld", (long long)n);
    return RB_ERR_ARG;
  }
  RcmWs w = rcm_ws(n, 0, d_ws, ws_bytes);
  if (w.total > ws_bytes) {
    rb_set_error("rb_rcm: workspace too small (%zu < %zu)", ws_bytes, w.total);
    return RB_ERR_ARG;
  }
  *n_plus = 0;
  *n_components = 0;
  if (n == 0) return RB_OK;
  // 1. V+ by (degree, id): stable radix sort of (deg, id) pairs (reorder.py:202-203)
  RB_CUDA_TRY(cudaMemsetAsync(w.ctr, 0, 64, s));
  copy_deg_u32<<<grid_for(n), 256, 0, s>>>(d_deg, w.deg_a, n, w.ctr);
  iota_u32<<<grid_for(n), 256, 0, s>>>(w.ids_a, n);
  cub::DoubleBuffer<uint32_t> dk(w.deg_a, w.deg_b), dv(w.ids_a, w.ids_b);
  size_t t = w.temp_bytes;
  RB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.temp, t, dk, dv, n, 0, 32, s));
  const uint32_t* sorted_ids = dv.Current();
  unsigned long long iso = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&iso, w.ctr, 8, cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t k = n - (int64_t)iso;
  *n_plus = k;
  const uint32_t* vplus = sorted_ids + iso;
  set_rank<<<grid_for(n), 256, 0, s>>>(sorted_ids, (int64_t)iso, n, w.rank);
  RB_CUDA_TRY(cudaGetLastError());
  if (k == 0) {
    rcm_perm<<<grid_for(n), 256, 0, s>>>(w.pos, sorted_ids, w.rank, n, (int64_t)iso, 0, d_perm, d_inv);
    RB_CUDA_TRY(cudaGetLastError());
    return RB_OK;
  }
  // 2. components in rank space (root = min rank = the walk's seed)
  iota_u32<<<grid_for(k), 256, 0, s>>>((uint32_t*)w.uf, k);
  if (getenv("RB_CC_FULL")) {  // (A/B reference: hook every edge)
    cc_hook_light<<<grid_for(n), 256, 0, s>>>(d_rs, d_col, w.rank, n, w.uf);
    cc_hook_heavy<<<grid_for(n * 32), 256, 0, s>>>(d_rs, d_col, w.rank, n, w.uf);
  } else {
    cc_sample<<<grid_for(n), 256, 0, s>>>(d_rs, d_col, w.rank, n, w.uf);
    cc_compress<<<grid_for(k), 256, 0, s>>>(w.uf, k);
    int32_t* probe = reinterpret_cast<int32_t*>(w.keys_a);  // (scratch: the level keys are unused yet)
    cc_probe_roots<<<4, 256, 0, s>>>(w.uf, k, probe);
    std::vector<int32_t> h(1024);
    RB_CUDA_TRY(cudaMemcpyAsync(h.data(), probe, 1024 * 4, cudaMemcpyDeviceToHost, s));
    RB_CUDA_TRY(cudaStreamSynchronize(s));
    std::sort(h.begin(), h.end());
    int32_t giant = h[0];
    for (size_t i = 0, best = 0; i < h.size();) {  // most frequent sampled root
      size_t j = i;
      while (j < h.size() && h[j] == h[i]) ++j;
      if (j - i > best) {
        best = j - i;
        giant = h[i];
      }
      i = j;
    }
    cc_hook_rest_light<<<grid_for(n), 256, 0, s>>>(d_rs, d_col, w.rank, n, giant, w.uf);
    cc_hook_rest_heavy<<<grid_for(n * 32), 256, 0, s>>>(d_rs, d_col, w.rank, n, giant, w.uf);
  }
  cc_finalize<<<grid_for(k), 256, 0, s>>>(w.uf, k, w.comp_size);
  RB_CUDA_TRY(cudaMemsetAsync(w.comp_size, 0, (size_t)k * 4, s));
  cc_sizes<<<grid_for(k + 31), 256, 0, s>>>(w.uf, k, w.comp_size);
  root_flags<<<grid_for(k), 256, 0, s>>>(w.uf, k, w.rflag);
  t = w.temp_bytes;
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.temp, t, w.comp_size, w.comp_off, k, s));
  t = w.temp_bytes;
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.temp, t, w.rflag, w.ridx, k, s));
  uint32_t last_idx = 0, last_flag = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&last_idx, w.ridx + k - 1, 4, cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaMemcpyAsync(&last_flag, w.rflag + k - 1, 4, cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t nc = (int64_t)last_idx + last_flag;
  *n_components = nc;
  // 3. level-synchronous CM walk
  RB_CUDA_TRY(cudaMemsetAsync(w.pos, 0xff, (size_t)n * 4, s));
  RB_CUDA_TRY(cudaMemsetAsync(w.minpos, 0xff, (size_t)n * 4, s));
  seed_components<<<grid_for(k), 256, 0, s>>>(w.uf, w.comp_off, w.comp_size, w.ridx, vplus, k, nc, w.pos, w.cursor,
                                              w.lst_a, d_ranges);
  RB_CUDA_TRY(cudaGetLastError());
  const int b = std::max(1, bits_for((uint64_t)k));
  uint32_t* frontier = w.lst_a;
  uint32_t* next = w.lst_b;
  int64_t nf = nc;
  int64_t placed = nc;
  while (nf > 0) {
    RB_CUDA_TRY(cudaMemsetAsync(w.ctr, 0, 8, s));
    rcm_expand<<<grid_for(nf * 32), 256, 0, s>>>(d_rs, d_col, frontier, nf, w.pos, w.minpos, next, w.ctr);
    RB_CUDA_TRY(cudaGetLastError());
    unsigned long long cnt = 0;
    RB_CUDA_TRY(cudaMemcpyAsync(&cnt, w.ctr, 8, cudaMemcpyDeviceToHost, s));
    RB_CUDA_TRY(cudaStreamSynchronize(s));
    if (cnt == 0) break;
    rcm_keys<<<grid_for(cnt), 256, 0, s>>>(next, cnt, w.minpos, w.rank, b, w.keys_a);
    cub::DoubleBuffer<uint64_t> kk(w.keys_a, w.keys_b);
    t = w.temp_bytes;
    RB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(w.temp, t, kk, (int64_t)cnt, 0, 2 * b, s));
    const uint64_t* sk = kk.Current();
    rcm_heads<<<grid_for(cnt), 256, 0, s>>>(sk, cnt, b, vplus, w.uf, frontier /*reuse as verts*/, w.head);
    t = w.temp_bytes;
    RB_CUDA_TRY(cub::DeviceScan::InclusiveScan(w.temp, t, w.head, w.gstart, MaxOp(), (int64_t)cnt, s));
    rcm_assign<<<grid_for(cnt), 256, 0, s>>>(sk, cnt, b, w.uf, w.gstart, frontier, w.pos, w.cursor);
    rcm_advance<<<grid_for(cnt), 256, 0, s>>>(sk, cnt, b, w.uf, frontier, w.pos, w.cursor);
    RB_CUDA_TRY(cudaGetLastError());
    // frontier now holds this level's vertices in CM order; next is scratch
    placed += cnt;
    nf = (int64_t)cnt;
  }
  if (placed != k) {
    rb_set_error("rb_rcm: internal error, placed %lld of %lld", (long long)placed, (long long)k);
    return RB_ERR_CUDA;
  }
  rcm_perm<<<grid_for(n), 256, 0, s>>>(w.pos, sorted_ids, w.rank, n, (int64_t)iso, k, d_perm, d_inv);
  RB_CUDA_TRY(cudaGetLastError());
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  return RB_OK;
}

// ---------------------------------------------------------------------------

namespace {
size_t pair_sort_temp_bytes(int64_t m) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int64_t)std::max<int64_t>(m, 1), 0, 32);
  return t;
}
}  // namespace

extern "C" size_t rb_permute_workspace_bytes(int64_t n, int64_t m) {
  Carver c(nullptr, SIZE_MAX);
  c.take<int64_t>((size_t)n + 1);                   // deg64 / rs scan input
  c.take<uint64_t>((size_t)std::max<int64_t>(m, 1));  // gathered rows (int32) or degree keys (uint64)
  c.take<uint64_t>((size_t)std::max<int64_t>(m, 1));  // sorted degree keys
  c.take<int32_t>((size_t)n + 2);                   // relative offsets
  size_t t1 = segsort_temp_bytes<int32_t>(n, m), t2 = segsort_temp_bytes<uint64_t>(n, m), t3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t3, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)n + 1);
  c.take<char>(std::max(std::max(std::max(t1, t2), t3), pair_sort_temp_bytes(m)));
  return c.off + 256;
}

extern "C" int rb_apply_permutation(const int64_t* d_rs, const int32_t* d_col, const int32_t* d_deg, int64_t n,
                                    int64_t m, const uint32_t* d_perm, const uint32_t* d_inv, void* d_ws,
                                    size_t ws_bytes, int64_t* d_rs_out, int32_t* d_col_out, int32_t* d_deg_out,
                                    void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (rb_permute_workspace_bytes(n, m) > ws_bytes) {
    rb_set_error("rb_apply_permutation: workspace too small");
    return RB_ERR_ARG;
  }
  Carver c(d_ws, ws_bytes);
  int64_t* deg64 = c.take<int64_t>((size_t)n + 1);
  uint64_t* area_a = c.take<uint64_t>((size_t)std::max<int64_t>(m, 1));
  uint64_t* area_b = c.take<uint64_t>((size_t)std::max<int64_t>(m, 1));
  int32_t* gathered = (int32_t*)area_a;
  int32_t* rel = c.take<int32_t>((size_t)n + 2);
  size_t t1 = segsort_temp_bytes<int32_t>(n, m), t2 = segsort_temp_bytes<uint64_t>(n, m), t3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t3, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)n + 1);
  const size_t tb = std::max(std::max(std::max(t1, t2), t3), pair_sort_temp_bytes(m));
  void* temp = c.take<char>(tb);
  if (n == 0) {
    RB_CUDA_TRY(cudaMemsetAsync(d_rs_out, 0, 8, s));
    return RB_OK;
  }
  RB_CUDA_TRY(cudaMemsetAsync(deg64 + n, 0, 8, s));
  gather_deg<<<grid_for(n), 256, 0, s>>>(d_deg, d_perm, n, d_deg_out, deg64);
  size_t t = tb;
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(temp, t, deg64, d_rs_out, n + 1, s));
  const char* mode = getenv("RB_RELABEL");  // "segsort": always sort inside the rows (tuning / A-B)
  if (m > 0 && !(mode && strcmp(mode, "segsort") == 0)) {
    // undirected graph: pairs (new neighbour id, new row) in new-row order, one stable radix sort by key
    uint32_t* keys_in = reinterpret_cast<uint32_t*>(area_a);
    uint32_t* vals_in = keys_in + m;
    uint32_t* keys_out = reinterpret_cast<uint32_t*>(area_b);
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(deg64);  // (the scan input is free again)
    relabel_pairs<<<grid_for(n * 32), 256, 0, s>>>(d_rs, d_col, d_perm, d_inv, d_rs_out, n, keys_in, vals_in);
    RB_CUDA_TRY(cudaGetLastError());
    t = tb;
    const int bits = std::max(1, bits_for((uint64_t)(n > 0 ? n - 1 : 0)));
    RB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, t, (const uint32_t*)keys_in, keys_out, (const uint32_t*)vals_in,
                                                reinterpret_cast<uint32_t*>(d_col_out), m, 0, bits, s));
    RB_CUDA_TRY(cudaMemsetAsync(bad, 0, 8, s));
    relabel_check<<<grid_for(n), 256, 0, s>>>(keys_out, d_rs_out, n, bad);
    unsigned long long h_bad = 0;
    RB_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, 8, cudaMemcpyDeviceToHost, s));
    RB_CUDA_TRY(cudaStreamSynchronize(s));
    if (h_bad == 0) return RB_OK;
    // not symmetric (the transposed rows do not fit): fall through to the general path
  }
  gather_rows<<<grid_for(n * 32), 256, 0, s>>>(d_rs, d_col, d_perm, d_inv, d_rs_out, n, gathered);
  RB_CUDA_TRY(cudaGetLastError());
  int rc = segmented_sort_rows<int32_t>(d_rs_out, n, m, gathered, d_col_out, temp, tb, rel, s);
  if (rc) return rc;
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  return RB_OK;
}

extern "C" int rb_degree_sort_adjacency(const int64_t* d_rs, const int32_t* d_col, const int32_t* d_deg, int64_t n,
                                        int64_t m, int descending, void* d_ws, size_t ws_bytes, int32_t* d_col_out,
                                        void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (rb_permute_workspace_bytes(n, m) > ws_bytes) {
    rb_set_error("rb_degree_sort_adjacency: workspace too small");
    return RB_ERR_ARG;
  }
  if (n == 0 || m == 0) return RB_OK;
  Carver c(d_ws, ws_bytes);
  c.take<int64_t>((size_t)n + 1);
  uint64_t* keys = c.take<uint64_t>((size_t)m);
  uint64_t* sorted = c.take<uint64_t>((size_t)m);
  int32_t* rel = c.take<int32_t>((size_t)n + 2);
  size_t t1 = segsort_temp_bytes<int32_t>(n, m), t2 = segsort_temp_bytes<uint64_t>(n, m), t3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t3, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)n + 1);
  const size_t tb = std::max(std::max(t1, t2), t3);
  void* temp = c.take<char>(tb);
  degree_keys<<<grid_for(n * 32), 256, 0, s>>>(d_rs, d_col, d_deg, n, descending, keys);
  RB_CUDA_TRY(cudaGetLastError());
  int rc = segmented_sort_rows<uint64_t>(d_rs, n, m, keys, sorted, temp, tb, rel, s);
  if (rc) return rc;
  keys_low32<<<grid_for(m), 256, 0, s>>>(sorted, m, d_col_out);
  RB_CUDA_TRY(cudaGetLastError());
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  return RB_OK;
}

// ---------------------------------------------------------------------------
// transpose slice of a 1D partition: for every global u, its owned neighbours

namespace {
__global__ void transpose_keys(const int64_t* __restrict__ rs, const int32_t* __restrict__ col, int64_t n_local,
                               int64_t v_lo, uint64_t* __restrict__ keys) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t w = warp; w < n_local; w += nwarps) {
    const int64_t s = rs[w], e = rs[w + 1];
    const uint64_t owner = (uint64_t)(v_lo + w);
    for (int64_t j = s + lane; j < e; j += 32) keys[j] = ((uint64_t)(uint32_t)col[j] << 32) | owner;
  }
}

size_t transpose_ws(int64_t m_local, uint64_t** A, uint64_t** B, void* base, size_t cap, void** temp,
                    size_t* temp_bytes) {
  Carver c(base, cap);
  *A = c.take<uint64_t>((size_t)std::max<int64_t>(m_local, 1));
  *B = c.take<uint64_t>((size_t)std::max<int64_t>(m_local, 1));
  size_t t = 0;
  cub::DoubleBuffer<uint64_t> db(*A, *B);
  cub::DeviceRadixSort::SortKeys(nullptr, t, db, std::max<int64_t>(m_local, 1), 0, 64);
  *temp_bytes = t;
  *temp = c.take<char>(t);
  return c.off + 256;
}
}  // namespace

extern "C" size_t rb_transpose_workspace_bytes(int64_t m_local, int64_t n_glob) {
  uint64_t *A, *B;
  void* temp;
  size_t tb;
  (void)n_glob;
  return transpose_ws(m_local, &A, &B, nullptr, SIZE_MAX, &temp, &tb);
}

extern "C" int rb_transpose_rows(const int64_t* d_rs, const int32_t* d_col, int64_t n_local, int64_t v_lo,
                                 int64_t m_local, int64_t n_glob, void* d_ws, size_t ws_bytes, int64_t* d_td_rs,
                                 int32_t* d_td_col, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t *A, *B;
  void* temp;
  size_t tb;
  if (transpose_ws(m_local, &A, &B, d_ws, ws_bytes, &temp, &tb) > ws_bytes) {
    rb_set_error("rb_transpose_rows: workspace too small");
    return RB_ERR_ARG;
  }
  if (m_local == 0) {
    RB_CUDA_TRY(cudaMemsetAsync(d_td_rs, 0, (size_t)(n_glob + 1) * 8, s));
    return RB_OK;
  }
  transpose_keys<<<grid_for(n_local * 32), 256, 0, s>>>(d_rs, d_col, n_local, v_lo, A);
  RB_CUDA_TRY(cudaGetLastError());
  cub::DoubleBuffer<uint64_t> db(A, B);
  const int end_bit = 32 + std::max(1, bits_for((uint64_t)(n_glob > 0 ? n_glob - 1 : 0)));
  size_t t = tb;
  RB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(temp, t, db, m_local, 0, end_bit, s));
  csr_emit<<<grid_for(m_local + 1), 256, 0, s>>>(db.Current(), m_local, n_glob, d_td_rs, d_td_col);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

// ---------------------------------------------------------------------------
// Sharded CSR build / relabel building blocks (configs[3]: the graph is split
// over the ranks by vertex block; see paper_2012_10026_b200/sharded.py)

namespace {
__global__ void relabel_keys(const int64_t* __restrict__ rs, const int32_t* __restrict__ col, int64_t n_local,
                             int64_t v_lo, const uint32_t* __restrict__ inv, uint64_t* __restrict__ keys) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t base = rs[0];
  for (int64_t v = warp; v < n_local; v += nwarps) {
    const uint64_t nv = inv[v_lo + v];
    for (int64_t j = rs[v] + lane; j < rs[v + 1]; j += 32) keys[j - base] = (nv << 32) | inv[col[j]];
  }
}

__global__ void keys_rows(const uint64_t* __restrict__ keys, int64_t m, int64_t v_lo, int64_t n_local,
                          int64_t* __restrict__ rs, int32_t* __restrict__ col) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = (i < m) ? (int64_t)(keys[i] >> 32) - v_lo : n_local;
    const int64_t ps = (i > 0) ? (int64_t)(keys[i - 1] >> 32) - v_lo : -1;
    for (int64_t v = ps + 1; v <= s; ++v) rs[v] = i;
    if (i < m) col[i] = (int32_t)(keys[i] & 0xffffffffu);
  }
}
}  // namespace

// The sorted unique keys (u << 32 | v) rb_csr_build left in its workspace.
extern "C" int rb_csr_keys(const void* d_ws, const uint64_t** d_keys, int64_t* m_directed) {
  if (!d_ws || !d_keys || !m_directed) {
    rb_set_error("rb_csr_keys: invalid argument");
    return RB_ERR_ARG;
  }
  CsrHeader hdr;
  RB_CUDA_TRY(cudaMemcpy(&hdr, d_ws, sizeof(hdr), cudaMemcpyDeviceToHost));
  *d_keys = (const uint64_t*)((const char*)d_ws + hdr.result_off);
  *m_directed = hdr.m_directed;
  return RB_OK;
}

extern "C" size_t rb_keys_workspace_bytes(int64_t m) {
  size_t t1 = 0, t2 = 0;
  const int64_t k = m > 0 ? m : 1;
  cub::DoubleBuffer<uint64_t> db(nullptr, nullptr);
  cub::DeviceRadixSort::SortKeys(nullptr, t1, db, k, 0, 64);
  cub::DeviceSelect::Unique(nullptr, t2, (uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t*)nullptr, k);
  return (size_t)k * 8 + 256 + std::max(t1, t2) + 256;
}

// Sort keys[0, m) (low end_bit bits significant) and drop duplicates, in place.
extern "C" int rb_keys_sort_unique(uint64_t* d_keys, int64_t m, int end_bit, void* d_ws, size_t ws_bytes,
                                   int64_t* m_out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (m < 0 || !m_out || end_bit < 1 || end_bit > 64 || (m > 0 && (!d_keys || ws_bytes < rb_keys_workspace_bytes(m)))) {
    rb_set_error("rb_keys_sort_unique: invalid argument");
    return RB_ERR_ARG;
  }
  *m_out = 0;
  if (m == 0) return RB_OK;
  Carver c(d_ws, ws_bytes);
  uint64_t* alt = c.take<uint64_t>((size_t)m);
  int64_t* nsel = c.take<int64_t>(1);
  size_t t1 = 0, t2 = 0;
  cub::DoubleBuffer<uint64_t> db(d_keys, alt);
  cub::DeviceRadixSort::SortKeys(nullptr, t1, db, m, 0, end_bit);
  cub::DeviceSelect::Unique(nullptr, t2, (uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t*)nullptr, m);
  size_t tb = std::max(t1, t2);
  void* temp = c.take<char>(tb);
  RB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(temp, tb, db, m, 0, end_bit, s));
  tb = std::max(t1, t2);
  uint64_t* sorted = db.Current();
  uint64_t* out = sorted == d_keys ? alt : d_keys;
  RB_CUDA_TRY(cub::DeviceSelect::Unique(temp, tb, sorted, out, nsel, m, s));
  int64_t nu = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&nu, nsel, 8, cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  if (out != d_keys) RB_CUDA_TRY(cudaMemcpyAsync(d_keys, out, (size_t)nu * 8, cudaMemcpyDeviceToDevice, s));
  *m_out = nu;
  return RB_OK;
}

// Local CSR of the vertex block [v_lo, v_lo + n_local) from its sorted unique
// keys (u << 32 | v): row starts (n_local + 1), columns (global ids), degrees.
extern "C" int rb_keys_to_csr(const uint64_t* d_keys, int64_t m, int64_t v_lo, int64_t n_local, int64_t* d_rs,
                              int32_t* d_col, int32_t* d_deg, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (m < 0 || n_local < 0 || v_lo < 0 || !d_rs || (n_local > 0 && !d_deg)) {
    rb_set_error("rb_keys_to_csr: invalid argument");
    return RB_ERR_ARG;
  }
  if (m == 0) {
    RB_CUDA_TRY(cudaMemsetAsync(d_rs, 0, (size_t)(n_local + 1) * 8, s));
  } else {
    keys_rows<<<grid_for(m + 1), 256, 0, s>>>(d_keys, m, v_lo, n_local, d_rs, d_col);
    RB_CUDA_TRY(cudaGetLastError());
  }
  if (n_local > 0) degrees_from_rs<<<grid_for(n_local), 256, 0, s>>>(d_rs, n_local, d_deg);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

// Keys (inv[v] << 32 | inv[w]) of every entry of a local block's rows: the
// relabelled graph, ready to be routed to the owners of the new ids.
extern "C" int rb_relabel_keys(const int64_t* d_rs, const int32_t* d_col, int64_t n_local, int64_t v_lo,
                               const uint32_t* d_inv, uint64_t* d_keys, void* stream) {
  if (n_local < 0 || !d_rs || !d_inv || !d_keys) {
    rb_set_error("rb_relabel_keys: invalid argument");
    return RB_ERR_ARG;
  }
  if (n_local == 0) return RB_OK;
  relabel_keys<<<grid_for(n_local * 32), 256, 0, (cudaStream_t)stream>>>(d_rs, d_col, n_local, v_lo, d_inv, d_keys);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}
