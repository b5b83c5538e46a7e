// First-discoverer parents of a queue BFS, from the level array of a
// level-synchronous traversal (bfs_sequential; reference _kernels.py:26-54).
//
// The reference's sequential BFS pops vertices in discovery order and gives w
// the parent v that reaches it first: the frontier vertex with the smallest
// queue position among w's neighbours in the level above, and -- positions
// being the order of (parent position, index in the parent's row) -- the next
// level is queued in the order of those pairs.  So, level by level:
//   expand : every frontier row v (queue position pos[v]) offers each
//            neighbour w one level down the key pos[v] << 32 | j (j = index
//            of w in row v) with a 64-bit atomicMin;
//   order  : the vertices of the next level sorted by their key are the next
//            stretch of the queue; parent[w] = queue[key >> 32].
// Keys are unique ((v, j) names one CSR entry), so the result is the
// reference's parent array bit for bit, for any row order (ascending or
// degree-sorted).  Vertices are grouped by level once (one radix sort); the
// per-level sorts are CUB radix sorts on 32 + log2(max degree) key bits.

#include <cstdint>
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <vector>

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

// level keys for the grouping sort: unreached vertices (level < 0) last
__global__ void seq_level_keys(const int32_t* level, int64_t n, uint32_t* key, uint32_t* id) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = level[v];
    key[v] = l < 0 ? 0xffffffffu : (uint32_t)l;
    id[v] = (uint32_t)v;
  }
}

// off[l] = first index of level l in the level-sorted order, for l in [0, n_levels]
// (off[n_levels] = the number of reached vertices)
__global__ void seq_level_offsets(const uint32_t* sorted_level, int64_t n, int64_t n_levels, int64_t* off) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l <= n_levels;
       l += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)sorted_level[mid] < l)
        lo = mid + 1;
      else
        hi = mid;
    }
    off[l] = lo;
  }
}

__global__ void seq_init(int32_t* parent, unsigned long long* key, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    parent[v] = -1;
    key[v] = ~0ull;
  }
}

__global__ void seq_seed(int32_t* parent, uint32_t* queue, int64_t source) {
  parent[source] = (int32_t)source;
  queue[0] = (uint32_t)source;
}

// one warp per frontier vertex (queue positions [q0, q1)): offer the keys
__global__ void seq_expand(const int64_t* __restrict__ rs, const int32_t* __restrict__ col,
                           const int32_t* __restrict__ level, const uint32_t* __restrict__ queue, int64_t q0,
                           int64_t q1, int32_t next_level, unsigned long long* key) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (int64_t q = q0 + warp; q < q1; q += nwarps) {
    const uint32_t v = queue[q];
    const int64_t s = rs[v], e = rs[v + 1];
    for (int64_t j = s + lane; j < e; j += 32) {
      const int32_t w = col[j];
      if (level[w] == next_level)
        atomicMin(key + w, ((unsigned long long)q << 32) | (unsigned long long)(j - s));
    }
  }
}

// the keys of the next level's vertices (by_level order), for the sort
__global__ void seq_gather(const uint32_t* by_level, int64_t a, int64_t b, const unsigned long long* key,
                           unsigned long long* seg_key) {
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x)
    seg_key[i - a] = key[by_level[i]];
}

// sorted (key, vertex) pairs -> queue stretch [a, b) and parents
__global__ void seq_assign(const unsigned long long* sorted_key, const uint32_t* sorted_id, int64_t a, int64_t b,
                           uint32_t* queue, int32_t* parent) {
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w = sorted_id[i - a];
    queue[i] = w;
    parent[w] = (int32_t)queue[sorted_key[i - a] >> 32];  // (a position of the level above: already final)
  }
}

struct Bufs {
  void* p[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  ~Bufs() {
    for (void* q : p)
      if (q) cudaFree(q);
  }
};

}  // namespace

extern "C" int rb_bfs_first_parents(const int64_t* d_rs, const int32_t* d_col, int64_t n, const int32_t* d_level,
                                    int64_t source, int64_t n_levels, int32_t* d_parent, void* stream) {
  if (!d_rs || !d_col || !d_level || !d_parent || n <= 0 || source < 0 || source >= n || n_levels < 1 ||
      n >= (1ll << 32)) {
    rb_set_error("rb_bfs_first_parents: bad argument (n=%lld source=%lld levels=%lld)", (long long)n,
                 (long long)source, (long long)n_levels);
    return RB_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  Bufs bf;
  uint32_t *lvl_key, *lvl_key2, *ids, *by_level, *queue, *seg_id;
  unsigned long long *key, *seg_key, *seg_key2;
  int64_t* d_off;
  // by_level doubles as the sort's value output; seg buffers sized for the largest level (<= n)
  size_t tmp_bytes = 0, tmp2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, 32, s);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp2, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, 64, s);
  if (tmp2 > tmp_bytes) tmp_bytes = tmp2;
  const size_t n4 = ((size_t)n * 4 + 255) & ~(size_t)255, n8 = ((size_t)n * 8 + 255) & ~(size_t)255;
  const size_t offb = (((size_t)n_levels + 2) * 8 + 255) & ~(size_t)255;
  RB_CUDA_TRY(cudaMalloc(&bf.p[0], 6 * n4 + 3 * n8 + offb));
  RB_CUDA_TRY(cudaMalloc(&bf.p[1], tmp_bytes));
  char* base = (char*)bf.p[0];
  lvl_key = (uint32_t*)base, base += n4;
  lvl_key2 = (uint32_t*)base, base += n4;
  ids = (uint32_t*)base, base += n4;
  by_level = (uint32_t*)base, base += n4;
  queue = (uint32_t*)base, base += n4;
  seg_id = (uint32_t*)base, base += n4;
  key = (unsigned long long*)base, base += n8;
  seg_key = (unsigned long long*)base, base += n8;
  seg_key2 = (unsigned long long*)base, base += n8;
  d_off = (int64_t*)base;

  seq_level_keys<<<grid_for(n), kT, 0, s>>>(d_level, n, lvl_key, ids);
  // (unreached = 0xffffffff sorts last: all 32 key bits)
  RB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(bf.p[1], tmp_bytes, lvl_key, lvl_key2, ids, by_level, n, 0, 32, s));
  seq_level_offsets<<<grid_for(n_levels + 1), kT, 0, s>>>(lvl_key2, n, n_levels, d_off);
  seq_init<<<grid_for(n), kT, 0, s>>>(d_parent, key, n);
  seq_seed<<<1, 1, 0, s>>>(d_parent, queue, source);
  std::vector<int64_t> off((size_t)n_levels + 1);
  RB_CUDA_TRY(cudaMemcpyAsync(off.data(), d_off, ((size_t)n_levels + 1) * 8, cudaMemcpyDeviceToHost, s));
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  if (off[0] != 0 || (n_levels >= 1 && off[1] != 1)) {
    rb_set_error("rb_bfs_first_parents: level array does not start at the source (level 0 holds %lld vertices)",
                 (long long)(n_levels >= 1 ? off[1] : -1));
    return RB_ERR_ARG;
  }
  for (int64_t l = 0; l + 1 < n_levels; ++l) {
    const int64_t q0 = off[l], q1 = off[l + 1], a = off[l + 1], b = off[l + 2];
    if (b <= a) break;
    const int64_t rows = q1 - q0;
    seq_expand<<<grid_for(rows * 32), kT, 0, s>>>(d_rs, d_col, d_level, queue, q0, q1, (int32_t)(l + 1), key);
    seq_gather<<<grid_for(b - a), kT, 0, s>>>(by_level, a, b, key, seg_key);
    RB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(bf.p[1], tmp_bytes, seg_key, seg_key2, by_level + a, seg_id, b - a, 0,
                                                64, s));
    seq_assign<<<grid_for(b - a), kT, 0, s>>>(seg_key2, seg_id, a, b, queue, d_parent);
  }
  RB_CUDA_TRY(cudaGetLastError());
  RB_CUDA_TRY(cudaStreamSynchronize(s));
  return RB_OK;
}
