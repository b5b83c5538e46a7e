// Micro-benchmark: event-timed cost of an (almost) empty persistent launch
// (148 x 768 threads, ~26 KB static smem) after a big memset kernel, normal
// vs cooperative launch.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(768, 1) persist(int* out, int iters) {
  __shared__ int buf[6500];
  buf[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (iters < 0) out[blockIdx.x] = buf[(threadIdx.x + 1) % 768];
}

__global__ void fill(int4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_int4(0, 0, 0, 0);
}

int main() {
  int* out;
  cudaMalloc(&out, 4096);
  int4* flush;
  const size_t fb = 256u << 20;
  cudaMalloc(&flush, fb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 148;
  for (int coop = 0; coop < 2; ++coop)
    for (int withflush = 0; withflush < 2; ++withflush) {
      float tot = 0;
      for (int r = 0; r < 22; ++r) {
        if (withflush) fill<<<592, 512>>>(flush, fb / 16);
        cudaEventRecord(a);
        int it = 0;
        void* args[] = {&out, &it};
        if (coop)
          cudaLaunchCooperativeKernel((const void*)persist, dim3(sms), dim3(768), args, 0, 0);
        else
          persist<<<sms, 768>>>(out, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 2) tot += ms;
      }
      printf("coop=%d flush_before=%d: %.2f us per launch (event to event)\n", coop, withflush, tot * 1000 / 20);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
