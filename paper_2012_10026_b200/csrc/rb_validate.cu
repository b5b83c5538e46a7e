// GPU BFS-tree validator + level oracle.
//
// Restates the five rules of validate.py:123-225 over device arrays so that
// trees can be checked at sizes where the CPU Validator's int64 edge keys do
// not fit (~17 B keys at scale 29):
//   1 parent[source] == source                                  (validate.py:143-150)
//   2 every tree edge (v, parent(v)) exists                       (validate.py:155-174)
//   3 parent chains reach the source; derived level = chain length (validate.py:176-200)
//   4 no graph edge spans more than one level                     (validate.py:202-215)
//   5 reached <=> same component as the source                    (validate.py:217-227)
// Component labels (validate.py:63-84: union-find, root = min id) come from a
// device union-find over the CSR or over the raw edge list.
//
// Each rule reports its first counterexample (min vertex / CSR edge index),
// the same one the reference names.  Rule 3 uses pointer jumping on packed
// (ancestor, distance) pairs instead of the reference's level-by-level sweep;
// both give the chain length to the source, or -1 if the chain never gets there.

#include <cstdint>
#include <cuda_runtime.h>

#include "rb_common.cuh"
#include "rb_error.h"

namespace {

constexpr int kT = 256;

int grid_for(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  if (b < 1) b = 1;
  if (b > 148 * 64) b = 148 * 64;
  return (int)b;
}

__device__ __forceinline__ int32_t uf_find(int32_t* uf, int32_t x) {
  int32_t cur = __ldcg(uf + x);
  if (cur != x) {
    int32_t prev = x, next;
    while (cur > (next = __ldcg(uf + cur))) {
      uf[prev] = next;  // path halving; values only decrease
      prev = cur;
      cur = next;
    }
  }
  return cur;
}

// hook the larger root under the smaller: the final root is the min id (validate.py:74-77)
__device__ __forceinline__ void uf_union(int32_t* uf, int32_t a, int32_t b) {
  int32_t ra = uf_find(uf, a), rb_ = uf_find(uf, b);
  while (ra != rb_) {
    if (ra < rb_) {
      const int32_t ret = atomicCAS(uf + rb_, rb_, ra);
      if (ret == rb_) break;
      rb_ = uf_find(uf, ret);
    } else {
      const int32_t ret = atomicCAS(uf + ra, ra, rb_);
      if (ret == ra) break;
      ra = uf_find(uf, ret);
    }
  }
}

__global__ void uf_init(int32_t* uf, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    uf[v] = (int32_t)v;
}

// CSR route: warp per row (rows of any length), edges with w < v only
__global__ void uf_csr(const int64_t* __restrict__ rs, const int32_t* __restrict__ col, int64_t n, int32_t* uf) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int64_t s = rs[v], e = rs[v + 1];
    for (int64_t j = s + lane; j < e; j += 32) {
      const int32_t w = col[j];
      if (w < (int32_t)v) uf_union(uf, (int32_t)v, w);
    }
  }
}

// raw edge-list route (validate.py:108-113): duplicates / self loops are harmless
__global__ void uf_edges(const uint32_t* __restrict__ edges, int64_t m, int64_t n, int32_t* uf) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = edges[2 * i], b = edges[2 * i + 1];
    if (a != b && a < (uint64_t)n && b < (uint64_t)n) uf_union(uf, (int32_t)a, (int32_t)b);
  }
}

__global__ void uf_flatten(int32_t* uf, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    int32_t x = (int32_t)v;
    while (true) {
      const int32_t p = __ldcg(uf + x);
      if (p == x) break;
      x = p;
    }
    uf[v] = x;
  }
}

struct VCtr {
  unsigned long long bad1, bad2_oor, bad2_missing, bad3, bad4, bad5, changed, pad;
};

__device__ __forceinline__ bool row_has(const int64_t* rs, const int32_t* col, int64_t v, int32_t p) {
  int64_t lo = rs[v], hi = rs[v + 1];
  const int64_t s = lo, e = hi;
  while (lo < hi) {  // rows of build_csr / apply_permutation are ascending
    const int64_t mid = (lo + hi) >> 1;
    if (col[mid] < p)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < e && col[lo] == p) return true;
  for (int64_t j = s; j < e; ++j)  // unsorted rows (degree-sorted adjacency): exact scan
    if (col[j] == p) return true;
  return false;
}

// rules 1, 2, 5 + pointer-jumping init (packed: ancestor in the low 32 bits,
// distance in the high 32 bits; ancestor -1 = dead end)
__global__ void v_rules(const int64_t* __restrict__ rs, const int32_t* __restrict__ col, int64_t n,
                        const int32_t* __restrict__ labels, int64_t src, const int32_t* __restrict__ parent,
                        unsigned long long* P, VCtr* c) {
  const int32_t lsrc = labels[src];
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = parent[v];
    const bool reached = p >= 0;
    uint32_t anc = 0xffffffffu, dist = 0;
    if (v == src) {
      anc = (uint32_t)src;
      if (p != (int32_t)src) atomicMin(&c->bad1, (unsigned long long)v);
    } else if (reached) {
      if ((int64_t)p >= n) {
        atomicMin(&c->bad2_oor, (unsigned long long)v);
      } else {
        anc = (uint32_t)p;
        dist = 1;
        if (!row_has(rs, col, v, p)) atomicMin(&c->bad2_missing, (unsigned long long)v);
      }
    }
    if ((labels[v] == lsrc) != reached) atomicMin(&c->bad5, (unsigned long long)v);
    P[v] = ((unsigned long long)dist << 32) | anc;
  }
}

__global__ void v_jump(unsigned long long* P, int64_t n, int64_t src, VCtr* c) {
  bool changed = false;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = __ldcg(P + v);
    const uint32_t a = (uint32_t)x;
    if (a == 0xffffffffu || (int64_t)a == src) continue;
    const unsigned long long y = __ldcg(P + a);
    const uint32_t a2 = (uint32_t)y;
    unsigned long long nx;
    if (a2 == 0xffffffffu)
      nx = 0xffffffffull;  // the chain ends at an unreached vertex
    else
      nx = ((unsigned long long)((uint32_t)(x >> 32) + (uint32_t)(y >> 32)) << 32) | a2;
    if (nx != x) {
      P[v] = nx;
      changed = true;
    }
  }
  if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) c->changed = 1;
}

__global__ void v_levels(const unsigned long long* P, int64_t n, int64_t src, const int32_t* parent,
                         int32_t* levels, VCtr* c) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = P[v];
    int32_t lv = -1;
    if (v == src)
      lv = 0;
    else if ((int64_t)(uint32_t)x == src)
      lv = (int32_t)(x >> 32);
    levels[v] = lv;
    if (lv < 0 && parent[v] >= 0) atomicMin(&c->bad3, (unsigned long long)v);
  }
}

// rule 4 over every stored directed edge; warp per row
__global__ void v_edges(const int64_t* __restrict__ rs, const int32_t* __restrict__ col, int64_t n,
                        const int32_t* __restrict__ levels, VCtr* c) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int32_t lv = levels[v];
    if (lv < 0) continue;
    const int64_t s = rs[v], e = rs[v + 1];
    for (int64_t j = s + lane; j < e; j += 32) {
      const int32_t lw = levels[col[j]];
      if (lw >= 0 && (lw - lv > 1 || lv - lw > 1)) {
        atomicMin(&c->bad4, (unsigned long long)j);
        break;
      }
    }
  }
}

}  // namespace

extern "C" size_t rb_validate_workspace_bytes(int64_t n) { return (size_t)(n > 0 ? n : 1) * 8 + 256; }

extern "C" int rb_components(const int64_t* d_rs, const int32_t* d_col, int64_t n, const uint32_t* d_edges,
                             int64_t m_raw, int32_t* d_labels, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0 || n >= (1ll << 31) || !d_labels || (!d_edges && (!d_rs || !d_col))) {
    rb_set_error("rb_components: invalid argument");
    return RB_ERR_ARG;
  }
  if (n == 0) return RB_OK;
  uf_init<<<grid_for(n), kT, 0, s>>>(d_labels, n);
  if (d_edges) {
    if (m_raw > 0) uf_edges<<<grid_for(m_raw), kT, 0, s>>>(d_edges, m_raw, n, d_labels);
  } else {
    uf_csr<<<grid_for(n * 32), kT, 0, s>>>(d_rs, d_col, n, d_labels);
  }
  uf_flatten<<<grid_for(n), kT, 0, s>>>(d_labels, n);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

extern "C" int rb_validate(const int64_t* d_rs, const int32_t* d_col, int64_t n, const int32_t* d_labels,
                           int64_t source, const int32_t* d_parent, void* d_ws, size_t ws_bytes,
                           int32_t* d_levels, int64_t* h_first_bad, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0 || n >= (1ll << 31) || !d_rs || !d_col || !d_labels || !d_parent || !d_levels || !h_first_bad) {
    rb_set_error("rb_validate: invalid argument");
    return RB_ERR_ARG;
  }
  if (source < 0 || source >= n) {
    rb_set_error("source %lld out of range for n=%lld", (long long)source, (long long)n);
    return RB_ERR_ARG;
  }
  if (ws_bytes < rb_validate_workspace_bytes(n)) {
    rb_set_error("rb_validate: workspace too small");
    return RB_ERR_ARG;
  }
  unsigned long long* P = reinterpret_cast<unsigned long long*>(d_ws);
  VCtr* c = reinterpret_cast<VCtr*>(reinterpret_cast<char*>(d_ws) + (size_t)n * 8);
  RB_CUDA_TRY(cudaMemsetAsync(c, 0xff, sizeof(VCtr), s));
  v_rules<<<grid_for(n), kT, 0, s>>>(d_rs, d_col, n, d_labels, source, d_parent, P, c);
  // pointer jumping: ceil(log2(depth)) + 1 rounds for a tree; cycles never
  // settle, so the loop is capped (2^40 > any chain)
  for (int round = 0; round < 40; ++round) {
    unsigned long long zero = 0;
    RB_CUDA_TRY(cudaMemcpyAsync(&c->changed, &zero, 8, cudaMemcpyHostToDevice, s));
    v_jump<<<grid_for(n), kT, 0, s>>>(P, n, source, c);
    unsigned long long changed = 0;
    RB_CUDA_TRY(cudaMemcpyAsync(&changed, &c->changed, 8, cudaMemcpyDeviceToHost, s));
    RB_CUDA_TRY(cudaStreamSynchronize(s));
    if (!changed) break;
  }
  v_levels<<<grid_for(n), kT, 0, s>>>(P, n, source, d_parent, d_levels, c);
  v_edges<<<grid_for(n * 32), kT, 0, s>>>(d_rs, d_col, n, d_levels, c);
  RB_CUDA_TRY(cudaGetLastError());
  VCtr h;
  RB_CUDA_TRY(cudaMemcpyAsync(&h, c, sizeof(VCtr), cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  auto first = [](unsigned long long x) -> int64_t { return x == ~0ull ? -1 : (int64_t)x; };
  h_first_bad[0] = first(h.bad1);
  // the reference names an out-of-range parent first, then a missing edge
  h_first_bad[1] = h.bad2_oor != ~0ull ? (int64_t)h.bad2_oor : first(h.bad2_missing);
  h_first_bad[2] = first(h.bad3);
  h_first_bad[3] = first(h.bad4);
  h_first_bad[4] = first(h.bad5);
  return RB_OK;
}
