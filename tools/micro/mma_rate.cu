// Micro-benchmark: issue rate of back-to-back tcgen05.mma (SS, bf16, M=128) for
// several N, from one CTA per SM, operands resident in smem (no TMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2104_05035_b200/csrc mma_rate.cu
#include <cstdio>
#include <cuda.h>
#include "tc_ptx.cuh"
using namespace rn;

template <int N>
__global__ void __launch_bounds__(128, 1) k(long long *out, int iters, int kstep, int aoff, int asbo, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (200 + N) * 128 / 4; i += blockDim.x) ((uint32_t *)s)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&bar2, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc<256>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = slot;
  if (warp == 0) {
    const uint32_t a = tc::smem_u32(s), b = a + 200 * 128;
    constexpr uint32_t ID = tc::idesc_bf16(128, N);
    long long t0 = clock64();
    if (mode == 4) {   // whole warp runs the loop (uniform values), elect.sync inside the asm
      for (int i = 0; i < iters; ++i) {
        const int k = i & 3;
        const uint64_t ad = tc::smem_desc(a + aoff + k * kstep, 16, asbo, 2), bd = tc::smem_desc(b + k * kstep, 16, 1024, 2);
        asm volatile("{\n.reg .pred p, q;\nelect.sync _|p, 0xffffffff;\nsetp.ne.b32 q, %4, 0;\n"
                     "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n}\n"
                     :: "r"(tb), "l"(ad), "l"(bd), "r"(ID), "r"((uint32_t)(i != 0)) : "memory");
        if ((i & 7) == 7) asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" :: "r"(tc::smem_u32(&bar2)) : "memory");
      }
      asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" :: "r"(tc::smem_u32(&bar)) : "memory");
    } else if (threadIdx.x == 0) {
      for (int i = 0; i < iters; ++i) {
        const int k = i & 3;
        tc::mma_bf16(tb, tc::smem_desc(a + aoff + k * kstep, 16, asbo, 2), tc::smem_desc(b + k * kstep, 16, 1024, 2), ID, i != 0);
        if (mode == 1 && (i & 7) == 7) tc::tc_fence_after();
        if (mode == 2 && (i & 7) == 7) tc::mma_commit(&bar2);
        if (mode == 3 && (i & 7) == 7) { tc::mma_commit(&bar2); tc::tc_fence_after(); }
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tb);
}

template <int N>
void run(long long *d, int iters, int grid, int aoff = 0, int asbo = 1024, int mode = 0) {
  const int smem = (200 + N) * 128 + 2048;
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<N><<<grid, 128, smem>>>(d, iters, 32, aoff, asbo, mode);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("mode=%d aoff=%4d sbo=%4d N=%3d grid=%3d iters=%5d: %.1f cycles/MMA  (%.0f FLOP/cycle/SM)\n", mode, aoff, asbo, N, grid, iters, (double)mx / iters,
         2.0 * 128 * N * 16 / ((double)mx / iters));
}

int main() {
  long long *d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int m : {0, 3, 4}) run<64>(d, 4096, 148, 0, 1024, m);
  for (int m : {0, 4}) run<128>(d, 4096, 148, 0, 1024, m);
  for (int m : {0, 4}) run<256>(d, 4096, 148, 0, 1024, m);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
