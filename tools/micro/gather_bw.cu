// Micro-benchmark: achievable HBM read bandwidth for the access shapes of the
// BFS kernels (sequential stream vs 1 KB chunks at random offsets, scalar vs
// 16-B loads, chunks in flight per warp).  nvcc -O3 -arch=sm_100a gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void seq_read(const int4* a, size_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 x = __ldcg(a + i);
    s += x.x ^ x.w;
  }
  if (s == 42) *out = s;
}

// warp per chunk of 256 ints at offset off[c]; K chunks per warp iteration
template <int K, bool VEC>
__global__ void chunk_read(const int* a, const long long* off, size_t nchunks, unsigned long long* out) {
  const unsigned lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long s = 0;
  for (size_t c0 = warp * K; c0 < nchunks; c0 += nw * K) {
    int v[K][8];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const size_t c = c0 + k;
      const long long o = c < nchunks ? off[c] : 0;
      if (VEC) {
        const int4* p = reinterpret_cast<const int4*>(a + o);
        int4 x = __ldg(p + lane), y = __ldg(p + 32 + lane);
        v[k][0] = x.x; v[k][1] = x.y; v[k][2] = x.z; v[k][3] = x.w; v[k][4] = y.x; v[k][5] = y.y; v[k][6] = y.z; v[k][7] = y.w;
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) v[k][t] = __ldg(a + o + lane + 32 * t);
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int t = 0; t < 8; ++t) s += v[k][t];
  }
  if (s == 42) *out = s;
}

int main() {
  const size_t bytes = 8ull << 30;  // 8 GiB array (like s26 col)
  const size_t n = bytes / 4;
  int* a;
  cudaMalloc(&a, bytes);
  cudaMemset(a, 1, bytes);
  const size_t nch = 547000;  // chunks of 1 KB (s26 BT level: 140M edges)
  long long* off;
  cudaMalloc(&off, nch * 8);
  long long* h = new long long[nch];
  unsigned long long x = 88172645463325252ull;
  for (size_t i = 0; i < nch; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = (long long)((x % (n / 256 - 1)) * 256);  // 1 KB aligned
  }
  cudaMemcpy(off, h, nch * 8, cudaMemcpyHostToDevice);
  unsigned long long* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto timeit = [&](const char* name, auto launch, double mb) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.1f us  %7.0f GB/s\n", name, ms * 1000 / 5, mb * 5 / (ms * 1e-3) / 1e9);
  };
  const int G = 148;
  timeit("seq 560MB int4 148x1024", [&] { seq_read<<<G, 1024>>>((const int4*)a, 560000000 / 16, out); }, 560e6);
  timeit("seq 560MB int4 592x1024", [&] { seq_read<<<G * 4, 1024>>>((const int4*)a, 560000000 / 16, out); }, 560e6);
  timeit("chunk K=1 scalar", [&] { chunk_read<1, false><<<G, 1024>>>(a, off, nch, out); }, nch * 1024.0);
  timeit("chunk K=2 scalar", [&] { chunk_read<2, false><<<G, 1024>>>(a, off, nch, out); }, nch * 1024.0);
  timeit("chunk K=4 scalar", [&] { chunk_read<4, false><<<G, 1024>>>(a, off, nch, out); }, nch * 1024.0);
  timeit("chunk K=1 vec", [&] { chunk_read<1, true><<<G, 1024>>>(a, off, nch, out); }, nch * 1024.0);
  timeit("chunk K=2 vec", [&] { chunk_read<2, true><<<G, 1024>>>(a, off, nch, out); }, nch * 1024.0);
  timeit("chunk K=4 vec", [&] { chunk_read<4, true><<<G, 1024>>>(a, off, nch, out); }, nch * 1024.0);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
