// Micro-benchmark: cost of the pieces of a last-block-finalize reduction
// (ticket fence/atomic, partial reads, fp64 finalize) on a tiny tensor.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512) k(const float *x, int64_t n, float *partial, unsigned *counter, float *out,
                                         int mode, int C) {
  __shared__ bool is_last;
  float s = 0.f;
  for (int64_t i = blockIdx.x * 512 + threadIdx.x; i < n; i += gridDim.x * 512) s += x[i];
  if (threadIdx.x < C) partial[blockIdx.x * 2 * C + threadIdx.x] = s;
  if (mode == 0) return;
  if (mode == 1) __threadfence();
  if (mode == 4) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  if (mode == 1) __threadfence();
  if (mode == 4) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  if (mode >= 2) {
    double a = 0;
    for (int k0 = 0; k0 < (int)gridDim.x; k0 += 8) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float *src = mode == 5 ? x : partial;
        v[j] = k0 + j < (int)gridDim.x ? (mode == 2 ? __ldcg(src + (k0 + j) * 2 * C + threadIdx.x % C) : src[(k0 + j) * 2 * C + threadIdx.x % C]) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) a += v[j];
    }
    if (mode == 3) a = 1.0 / sqrt(a + 1e-5);
    if (threadIdx.x < C) out[threadIdx.x] = (float)a;
  }
  if (threadIdx.x == 0) *counter = 0;
}
int main() {
  float *x, *p, *o;
  unsigned *c;
  cudaMalloc(&x, 1 << 24); cudaMemset(x, 0, 1 << 24);
  cudaMalloc(&p, 1 << 22); cudaMalloc(&o, 4096); cudaMalloc(&c, 4); cudaMemset(c, 0, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {36, 148})
    for (int mode : {0, 1, 4, 2, 3, 5, 6}) {
      for (int r = 0; r < 3; ++r) k<<<blocks, 512>>>(x, 147456, p, c, o, mode, 512);
      cudaEventRecord(a);
      for (int r = 0; r < 50; ++r) k<<<blocks, 512>>>(x, 147456, p, c, o, mode, 512);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("blocks %3d mode %d (%s): %.2f us\n", blocks, mode,
             mode == 0 ? "reduce only" : mode == 1 ? "+threadfence ticket" : mode == 4 ? "+fence.acq_rel ticket" : mode == 2 ? "+ticket(no fence)+partial ldcg reads" : mode == 3 ? "+plain reads +fp64 finalize" : mode == 5 ? "plain reads of x (not written)" : "plain reads, no fence",
             ms * 1000 / 50);
    }
}
