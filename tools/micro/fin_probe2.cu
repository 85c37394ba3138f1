#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512) k(const float *x, float *partial, unsigned *counter, float *out, long long *tm,
                                         int C, int useD) {
  __shared__ bool is_last;
  if (threadIdx.x < C) partial[blockIdx.x * 2 * C + threadIdx.x] = x[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  long long t0 = clock64();
  double a = 0; float af = 0;
  float v[160];
#pragma unroll
  for (int j = 0; j < 148; ++j) v[j] = partial[j * 2 * C + threadIdx.x % C];
  long long t1 = clock64();
  if (useD) {
#pragma unroll
    for (int j = 0; j < 148; ++j) a += v[j];
  } else {
#pragma unroll
    for (int j = 0; j < 148; ++j) af += v[j];
    a = af;
  }
  long long t2 = clock64();
  out[threadIdx.x] = (float)a;
  if (threadIdx.x == 0) { tm[0] = t1 - t0; tm[1] = t2 - t1; *counter = 0; }
}
int main() {
  float *x, *p, *o; unsigned *c; long long *tm;
  cudaMalloc(&x, 1 << 24); cudaMemset(x, 0, 1 << 24);
  cudaMalloc(&p, 1 << 22); cudaMalloc(&o, 4096); cudaMalloc(&c, 4); cudaMemset(c, 0, 4); cudaMalloc(&tm, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int useD : {0, 1}) {
    for (int r = 0; r < 3; ++r) k<<<148, 512>>>(x, p, c, o, tm, 512, useD);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) k<<<148, 512>>>(x, p, c, o, tm, 512, useD);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long h[2]; cudaMemcpy(h, tm, 16, cudaMemcpyDeviceToHost);
    printf("useD %d: %.2f us/launch; last block: loads %lld cyc, adds %lld cyc  %s\n", useD, ms * 1000 / 20, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
}
