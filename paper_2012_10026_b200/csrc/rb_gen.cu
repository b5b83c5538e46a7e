// rb_gen.cu -- Kronecker (R-MAT) edge generator on device, byte-identical
// with the reference kronecker_generate (generator.py:114-148).
//
// The reference draws, per 65,536-edge chunk c, a numpy Generator over
// Philox4x64-10 keyed (seed, c) and takes count x scale doubles row-major:
// draw j of a chunk is word j mod 4 of the Philox block whose 256-bit
// counter is j/4 + 1 (numpy increments the counter before each block), and
// Generator.random() maps a raw word x to (x >> 11) * 2^-53.  Each draw picks
// the quadrant q = (u >= a) + (u >= a+b) + (u >= a+b+c); bit q>>1 goes to the
// source, bit q&1 to the destination, column 0 being the most significant
// level.  Ids are then scrambled by three rounds of
//   x = (x * mult) & mask;  x ^= x >> shift;  x = (x + add) & mask
// with constants from splitmix64 of the seed (generator.py:74-111).
// One thread per edge: scale/4 Philox blocks, all arithmetic in registers.
#include <stdint.h>

#include <cub/cub.cuh>

#include "rb_common.cuh"
#include "rb_error.h"

namespace {

constexpr int64_t kChunkEdges = 1 << 16;

struct GenParams {
  int scale;
  int64_t m;
  uint64_t seed;
  double t1, t2, t3;
  uint64_t mask;
  uint64_t mult[3], add[3];
  int shift[3];
};

__device__ __forceinline__ void philox4x64_10(uint64_t ctr[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * ctr[0];
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ull, ctr[0]);
    const uint64_t lo1 = 0xCA5A826395121157ull * ctr[2];
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ull, ctr[2]);
    const uint64_t n0 = hi1 ^ ctr[1] ^ k0;
    const uint64_t n2 = hi0 ^ ctr[3] ^ k1;
    ctr[0] = n0;
    ctr[1] = lo1;
    ctr[2] = n2;
    ctr[3] = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
}

__device__ __forceinline__ uint64_t scramble(uint64_t x, const GenParams& g) {
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    x = (x * g.mult[r]) & g.mask;
    x ^= x >> g.shift[r];
    x = (x + g.add[r]) & g.mask;
  }
  return x;
}

__global__ void kron_kernel(GenParams g, int64_t e_lo, int64_t e_hi, uint2* __restrict__ out) {
  for (int64_t e = e_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e_hi; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t chunk = (uint64_t)(e / kChunkEdges);
    const int64_t i = e % kChunkEdges;  // edge index inside the chunk
    uint64_t src = 0, dst = 0;
    int64_t j = i * g.scale;  // first draw of this edge
    uint64_t cur_block = ~0ull;
    uint64_t words[4];
    for (int t = 0; t < g.scale; ++t, ++j) {
      const uint64_t blk = (uint64_t)(j >> 2);
      if (blk != cur_block) {
        words[0] = blk + 1;  // numpy's counter starts at 1
        words[1] = 0;
        words[2] = 0;
        words[3] = 0;
        philox4x64_10(words, g.seed, chunk);
        cur_block = blk;
      }
      const uint64_t raw = words[j & 3];
      const double u = (double)(raw >> 11) * (1.0 / 9007199254740992.0);
      const int q = (u >= g.t1) + (u >= g.t2) + (u >= g.t3);
      src = (src << 1) | (uint64_t)((q >> 1) & 1);
      dst = (dst << 1) | (uint64_t)(q & 1);
    }
    out[e - e_lo] = make_uint2((uint32_t)scramble(src, g), (uint32_t)scramble(dst, g));
  }
}

// Chung-Lu endpoint sampling (BASELINE configs[4]; recipe in generator.py):
// pair j takes raw words 2i, 2i+1 (i = j mod 65536) of the Philox stream
// keyed (seed, 2^32 + j / 65536) -- numpy's Philox(key=[seed, 2^32 + c])
// .random_raw() order -- maps each to r = floor(x * T / 2^64) over the total
// integer weight T, and picks the first vertex whose inclusive weight prefix
// exceeds r.  All integer: byte-identical with the numpy restatement.
__global__ void chunglu_kernel(const int64_t* __restrict__ prefix, int64_t n, int64_t m, uint64_t seed,
                               uint2* __restrict__ out) {
  const uint64_t T = (uint64_t)prefix[n - 1];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t chunk = (1ull << 32) + (uint64_t)(j / kChunkEdges);
    const int64_t i = j % kChunkEdges;
    uint64_t words[4] = {(uint64_t)((2 * i) >> 2) + 1, 0, 0, 0};  // words 2i, 2i+1 share one block
    philox4x64_10(words, seed, chunk);
    uint32_t ends[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint64_t r = __umul64hi(words[(2 * i + t) & 3], T);
      int64_t lo = 0, hi = n - 1;  // first idx with prefix[idx] > r (exists: r < T)
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(prefix + mid) > r)
          hi = mid;
        else
          lo = mid + 1;
      }
      ends[t] = (uint32_t)lo;
    }
    out[j] = make_uint2(ends[0], ends[1]);
  }
}

uint64_t splitmix64(uint64_t x) {
  x = x + 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" int rb_kronecker_generate_range(int scale, int64_t edgefactor, uint64_t seed, double a, double b,
                                           double c, int64_t e_lo, int64_t e_hi, uint32_t* d_edges, void* stream) {
  if (scale < 1 || scale > 30 || edgefactor < 1 || (!d_edges && e_hi > e_lo) || e_lo < 0 ||
      e_hi > ((int64_t)1 << scale) * edgefactor || e_hi < e_lo) {
    rb_set_error("rb_kronecker_generate: invalid argument");
    return RB_ERR_ARG;
  }
  GenParams g{};
  g.scale = scale;
  g.m = ((int64_t)1 << scale) * edgefactor;
  g.seed = seed;
  g.t1 = a;  // generator.py:117: t1, t2, t3 = a, a + b, a + b + c (double arithmetic)
  g.t2 = a + b;
  g.t3 = a + b + c;
  g.mask = ((uint64_t)1 << scale) - 1;
  // _scramble_constants (generator.py:82-93)
  uint64_t x = seed ^ 0xD6E8FEB86659FD93ull;
  const int shifts[3] = {scale / 2 > 1 ? scale / 2 : 1, scale / 3 > 1 ? scale / 3 : 1,
                         (2 * scale) / 3 > 1 ? (2 * scale) / 3 : 1};
  for (int r = 0; r < 3; ++r) {
    x = splitmix64(x);
    g.mult[r] = x | 1;
    x = splitmix64(x);
    g.add[r] = x & g.mask;
    g.shift[r] = shifts[r];
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (e_hi == e_lo) return RB_OK;
  int64_t blocks = (e_hi - e_lo + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  kron_kernel<<<(int)blocks, 256, 0, s>>>(g, e_lo, e_hi, reinterpret_cast<uint2*>(d_edges));
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

extern "C" int rb_kronecker_generate(int scale, int64_t edgefactor, uint64_t seed, double a, double b, double c,
                                     uint32_t* d_edges, void* stream) {
  if (scale < 1 || scale > 30 || edgefactor < 1 || !d_edges) {
    rb_set_error("rb_kronecker_generate: invalid argument");
    return RB_ERR_ARG;
  }
  return rb_kronecker_generate_range(scale, edgefactor, seed, a, b, c, 0, ((int64_t)1 << scale) * edgefactor, d_edges,
                                     stream);
}

extern "C" size_t rb_chunglu_workspace_bytes(int64_t n) {
  size_t t = 0;
  cub::DeviceScan::InclusiveSum(nullptr, t, (const int64_t*)nullptr, (int64_t*)nullptr, (int)(n > 0 ? n : 1));
  return (size_t)(n > 0 ? n : 1) * 8 + 256 + t;
}

extern "C" int rb_chunglu_generate(const int64_t* d_weights, int64_t n, int64_t m_pairs, uint64_t seed, void* d_ws,
                                   size_t ws_bytes, uint32_t* d_edges, void* stream) {
  if (n < 1 || n >= (1ll << 31) || m_pairs < 0 || !d_weights || !d_edges || ws_bytes < rb_chunglu_workspace_bytes(n)) {
    rb_set_error("rb_chunglu_generate: invalid argument");
    return RB_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* prefix = reinterpret_cast<int64_t*>(d_ws);
  void* temp = reinterpret_cast<char*>(d_ws) + (((size_t)n * 8 + 255) & ~(size_t)255);
  size_t t = ws_bytes - (((size_t)n * 8 + 255) & ~(size_t)255);
  RB_CUDA_TRY(cub::DeviceScan::InclusiveSum(temp, t, d_weights, prefix, (int)n, s));
  if (m_pairs == 0) return RB_OK;
  int64_t blocks = (m_pairs + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  chunglu_kernel<<<(int)blocks, 256, 0, s>>>(prefix, n, m_pairs, seed, reinterpret_cast<uint2*>(d_edges));
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}
