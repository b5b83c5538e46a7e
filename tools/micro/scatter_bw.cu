// Micro-benchmark: how fast can one B200 do the scattered WRITES of a top-down
// claim?  The deferred top-down level of the BFS does, per newly found vertex,
// one 4-byte parent store into a 131 MB array and one red.or into a 4 MB
// bitmap (scale 26).  Measured here: random 4-byte stores, random red.or, both
// together, and 1-byte stores into a byte map, with every lane or only a
// fraction of the lanes active, 8 writes per lane per step (as td_claim).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scatter_bw.cu -o scatter_bw
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// mode bit 0: parent store, bit 1: red.or on the bitmap, bit 2: byte store
// pct: share of lanes (0..256) that write at all
template <int MODE>
__global__ void __launch_bounds__(768, 1) scatter(int32_t* parent, uint32_t* vis, uint8_t* visb, uint32_t n,
                                                  uint64_t total, uint32_t pct) {
  const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = gt * 8; i0 < total; i0 += nt * 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t h = mix((uint32_t)(i0 + k) * 2654435761u + 12345u);
      const uint32_t w = h % n;
      if ((mix(h) & 255u) < pct) {
        if (MODE & 1) parent[w] = (int32_t)i0;
        if (MODE & 2) asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(vis + (w >> 5)), "r"(1u << (w & 31)) : "memory");
        if (MODE & 4) visb[w] = 1;
      }
    }
  }
}

template <int MODE>
static void run(const char* name, int32_t* parent, uint32_t* vis, uint8_t* visb, uint32_t n, uint64_t total,
                uint32_t pct) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int it = 0; it < 4; ++it) {
    cudaMemset(vis, 0, (size_t)(n / 32 + 1) * 4);
    cudaEventRecord(a);
    scatter<MODE><<<148, 768>>>(parent, vis, visb, n, total, pct);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double writes = (double)total * pct / 256.0;
  printf("%-28s pct %3u/256: %8.1f us for %6.1f M target vertices -> %6.1f G vertices/s\n", name, pct, best * 1e3,
         writes / 1e6, writes / (best * 1e-3) / 1e9);
}

int main() {
  const uint32_t n = 32804088u;  // scale 26: non-isolated vertices
  int32_t* parent;
  uint32_t* vis;
  uint8_t* visb;
  cudaMalloc(&parent, (size_t)n * 4);
  cudaMalloc(&vis, (size_t)(n / 32 + 1) * 4);
  cudaMalloc(&visb, (size_t)n);
  cudaMemset(parent, 0xff, (size_t)n * 4);
  cudaMemset(visb, 0, n);
  for (uint32_t pct : {256u, 36u}) {  // every lane / 14 % of the lanes (the s26 deferred level)
    const uint64_t total = pct == 256u ? 8100000ull : 57500000ull;
    run<0>("loop only", parent, vis, visb, n, total, pct);
    run<1>("parent store", parent, vis, visb, n, total, pct);
    run<2>("red.or bitmap", parent, vis, visb, n, total, pct);
    run<3>("parent store + red.or", parent, vis, visb, n, total, pct);
    run<4>("byte store", parent, vis, visb, n, total, pct);
    run<5>("parent store + byte store", parent, vis, visb, n, total, pct);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
