// Micro-benchmark: the BN statistics reduce+finalize kernel (k_elem.cu) in
// isolation, CUDA-event timed, for the r18 tensor shapes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2104_05035_b200/csrc red_probe.cu ../../paper_2104_05035_b200/librn.so -o red_probe -lcuda
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "kernels.h"
using namespace rn;

int main() {
  struct S { int64_t V; int C; const char *name; } shapes[] = {
      {931040, 64, "stem 8x46x55x46x64"}, {118496, 64, "s1 8x23x28x23x64"}, {16128, 128, "s2 8x12x14x12x128"},
      {2016, 256, "s3 8x6x7x6x256"}, {288, 512, "s4 8x3x4x3x512"}};
  void *x;
  cudaMalloc(&x, 931040LL * 64 * 2);
  cudaMemset(x, 0x3c, 931040LL * 64 * 2);
  float *part, *prm;
  unsigned *cnt;
  cudaMalloc(&part, 1 << 22);
  cudaMalloc(&prm, 16 * 512 * 4);
  cudaMemset(prm, 0, 16 * 512 * 4);
  cudaMalloc(&cnt, 256);
  cudaMemset(cnt, 0, 256);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto &s : shapes) {
    for (int rep = 0; rep < 3; ++rep)
      bn_stats_finalize(DT_BF16, x, s.V, s.C, part, cnt, prm, prm + 512, prm + 1024, prm + 1536, prm + 2048,
                        prm + 2560, prm + 3072, prm + 3584, 0.1f, 1e-5f, st);
    cudaEventRecord(a, st);
    const int R = 20;
    for (int rep = 0; rep < R; ++rep)
      bn_stats_finalize(DT_BF16, x, s.V, s.C, part, cnt, prm, prm + 512, prm + 1024, prm + 1536, prm + 2048,
                        prm + 2560, prm + 3072, prm + 3584, 0.1f, 1e-5f, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = 1000.0 * ms / R;
    printf("%-22s blocks=%3d  %7.2f us  %6.0f GB/s   %s\n", s.name, chan_fin_blocks(s.V, s.C), us,
           s.V * s.C * 2 / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    // plain apply pass for comparison
    cudaEventRecord(a, st);
    for (int rep = 0; rep < R; ++rep)
      bn_apply(DT_BF16, x, s.V, s.C, prm, prm + 512, nullptr, nullptr, nullptr, true, (char *)x, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("%-22s apply          %7.2f us  %6.0f GB/s\n", s.name, 1000.0 * ms / R, 2.0 * s.V * s.C * 2 / (1000.0 * ms / R) / 1e3);
  }
}
