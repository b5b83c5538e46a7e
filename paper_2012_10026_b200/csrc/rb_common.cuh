// rb_common.cuh -- shared device helpers for the B200 RCM + BFS kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define RB_FULL 0xffffffffu

namespace rb {

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Read-only (for the whole launch) streaming loads of graph structure.
__device__ __forceinline__ int32_t ldg_i32(const int32_t* p) { return __ldg(p); }
__device__ __forceinline__ int64_t ldg_i64(const int64_t* p) { return __ldg(p); }

// Grid-wide barrier for a cooperative (co-resident) launch.  bar[0] is a
// monotonically increasing arrival counter (zeroed before the launch); the
// e-th barrier of a launch completes when it reaches e * nblocks.  One
// fire-and-forget release add per block, a relaxed spin, one acquire fence --
// no counter reset, no generation word.
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t nblocks, uint32_t& epoch) {
  ++epoch;
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_add(bar, 1u);
    const uint32_t target = epoch * nblocks;
    while ((int32_t)(ld_relaxed_u32(bar) - target) < 0) {
    }
    __threadfence();  // acquire side (also invalidates this SM's L1)
  }
  __syncthreads();
}

// Grid barrier that also fetches K 64-bit words written before it (counters
// reduced by atomics): thread 0 loads them once per block and shares them
// through shared memory -- if every thread loaded them, thousands of warps
// would queue on one L2 line.
template <int K>
__device__ __forceinline__ void grid_barrier_fetch(uint32_t* bar, uint32_t nblocks, uint32_t& epoch,
                                                   const unsigned long long* const (&src)[K],
                                                   unsigned long long* s_out) {
  ++epoch;
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_add(bar, 1u);
    const uint32_t target = epoch * nblocks;
    while ((int32_t)(ld_relaxed_u32(bar) - target) < 0) {
    }
    __threadfence();
#pragma unroll
    for (int k = 0; k < K; ++k) s_out[k] = ld_relaxed_u64(src[k]);
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// *p |= v (fire-and-forget) if c, predicated.
__device__ __forceinline__ void red_or_if(uint32_t* p, uint32_t v, bool c) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.relaxed.gpu.global.or.b32 [%0], %1;\n\t}" ::"l"(p),
               "r"(v), "r"((uint32_t)c)
               : "memory");
}

// *p = v if c, as one predicated store (no branch around it).
__device__ __forceinline__ void st_if(int32_t* p, int32_t v, bool c) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.b32 [%0], %1;\n\t}" ::"l"(p), "r"(v),
               "r"((uint32_t)c)
               : "memory");
}

// Warp inclusive scan (32-bit).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(RB_FULL, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(RB_FULL, x, o);
  return x;
}

// First lane j whose inclusive prefix incl[j] > e (incl nondecreasing, e < incl[31]).
__device__ __forceinline__ uint32_t warp_upper_bound(uint32_t incl, uint32_t e) {
  uint32_t j = 0;
#pragma unroll
  for (uint32_t s = 16; s >= 1; s >>= 1) {
    uint32_t v = __shfl_sync(RB_FULL, incl, j + s - 1);
    if (v <= e) j += s;
  }
  return j;
}

__device__ __forceinline__ int64_t shfl_i64(int64_t v, int src) {
  return (int64_t)__shfl_sync(RB_FULL, (long long)v, src);
}

}  // namespace rb

#define RB_CUDA_TRY(x)                                  \
  do {                                                  \
    cudaError_t _e = (x);                               \
    if (_e != cudaSuccess) {                            \
      rb_set_error("%s:%d %s: %s", __FILE__, __LINE__,  \
                   #x, cudaGetErrorString(_e));         \
      return RB_ERR_CUDA;                               \
    }                                                   \
  } while (0)
