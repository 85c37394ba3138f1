// Micro-benchmark: throughput of the legacy warp-level mma.sync.m16n8k16 (bf16 -> fp32)
// on sm_100a, 8 independent accumulator chains per warp, W warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 hmma_rate.cu -o hmma_rate
#include <cstdio>
#include <cstdint>
__global__ void k(float *out, int iters) {
  uint32_t a[4] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u}, b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  float d[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void kf(float *out, int iters) {
  float d[8] = {1, 2, 3, 4, 5, 6, 7, 8}, x = out[0] + 1.0001f;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 64; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) d[c] = fmaf(d[c], x, 0.5f);
  float s = 0;
  for (int c = 0; c < 8; ++c) s += d[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}
int main() {
  float *o;
  cudaMalloc(&o, 4096);
  cudaMemset(o, 0, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  for (int w : {4, 8, 16, 32}) {
    int iters = 4096;
    k<<<sms, w * 32>>>(o, 16);
    cudaEventRecord(e0);
    k<<<sms, w * 32>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * w * sms;
    printf("mma.sync m16n8k16 bf16: %2d warps/SM  %.1f TFLOP/s  (%.1f cycles per mma per SMSP at 1.9 GHz)\n", w,
           flops / ms / 1e9, ms * 1e-3 * 1.9e9 / (8.0 * iters * w / 4));
  }
  for (int w : {8, 32}) {
    int iters = 256;
    kf<<<sms, w * 32>>>(o, 4);
    cudaEventRecord(e0);
    kf<<<sms, w * 32>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * 8 * iters * w * 32.0 * sms;
    printf("fp32 FFMA: %2d warps/SM  %.1f TFLOP/s\n", w, flops / ms / 1e9);
  }
  return 0;
}
