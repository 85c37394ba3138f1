// Micro-benchmark (B200): tcgen05.mma issue rate for operand layouts the conv
// kernels could use, 1-CTA and 2-CTA (cta_group::2).  Operands sit in smem (no
// TMA); the numbers are cycles per MMA, M=128 (1-CTA) or 256 (pair), K=16.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2104_05035_b200/csrc tc_probe.cu -o tc_probe
#include <cstdio>
#include <cuda.h>
#include "tc_ptx.cuh"
using namespace rn;

struct Cfg {
  int layout;        // 2 = SW128, 0 = no swizzle (interleave)
  int aoff, alo, asbo;  // A start offset (B), LBO, SBO
  int blo, bsbo;
  int amn, bmn;      // MN-major flags
  int astep;         // per-MMA A advance (bytes) cycling over 4
  int bstep;
};

__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p, q;\nelect.sync _|p, 0xffffffff;\nsetp.ne.b32 q, %4, 0;\n"
               "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, q;\n}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

template <int N, int CG>
__global__ void __launch_bounds__(128, 1) k(long long *out, int iters, Cfg c) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t *)s)[i] = 0x3c003c00u;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) {
    if (CG == 1) tc::tmem_alloc<256>(&slot);
    else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(tc::smem_u32(&slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc::tc_fence_before();
  if (CG == 2) { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
  else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = slot;
  if (warp == 0 && rank == 0) {
    const uint32_t a = tc::smem_u32(s) + c.aoff, b = tc::smem_u32(s) + 96 * 1024;
    const uint32_t ID = tc::idesc_bf16(CG == 2 ? 256 : 128, N, c.amn, c.bmn);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      const uint64_t ad = tc::smem_desc(a + kk * c.astep, c.alo, c.asbo, c.layout);
      const uint64_t bd = tc::smem_desc(b + kk * c.bstep, c.blo, c.bsbo, c.layout);
      if (CG == 1) tc::mma_bf16_warp(tb, ad, bd, ID, i != 0);
      else mma2(tb, ad, bd, ID, i != 0);
    }
    if (CG == 1) tc::mma_commit_warp(&bar);
    else asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n"
                      :: "r"(tc::smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if (warp == 0 && CG == 2) {
    tc::mbar_wait(&bar, 0);
  }
  tc::tc_fence_before();
  if (CG == 2) { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
  else __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    if (CG == 1) tc::tmem_dealloc<256>(tb);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tb) : "memory");
  }
}

template <int N, int CG>
void run(const char *name, long long *d, Cfg c, int iters = 4096) {
  const int smem = 160 * 1024 + 2048;
  cudaFuncSetAttribute(k<N, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int grid = 148;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaMemset(d, 0, 148 * sizeof(long long));
  cudaError_t e = cudaLaunchKernelEx(&cfg, k<N, CG>, d, iters, c);
  cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cyc = (double)mx / iters;
  const double flop_sm = 2.0 * (CG == 2 ? 256 : 128) * N * 16 / cyc / CG;
  printf("%-44s N=%3d cg=%d: %6.1f cyc/MMA  %5.0f FLOP/cyc/SM (%3.0f%% of 8192)  %s\n", name, N, CG, cyc, flop_sm,
         100 * flop_sm / 8192, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long *d;
  cudaMalloc(&d, 148 * sizeof(long long));
  // K-major SW128 (the current kernels): A rows 128 B, 8-row groups at SBO
  Cfg sw = {2, 0, 16, 1024, 16, 1024, 0, 0, 32, 32};
  run<64, 1>("SW128 K-major aligned", d, sw);
  run<128, 1>("SW128 K-major aligned", d, sw);
  run<256, 1>("SW128 K-major aligned", d, sw);
  Cfg swo = sw; swo.aoff = 128; swo.asbo = 1280;
  run<64, 1>("SW128 K-major A +1 row, SBO 10 rows (halo)", d, swo);
  run<128, 1>("SW128 K-major A +1 row, SBO 10 rows (halo)", d, swo);
  Cfg swo2 = sw; swo2.aoff = 0; swo2.asbo = 1280;
  run<64, 1>("SW128 K-major A SBO 10 rows", d, swo2);
  Cfg swo3 = sw; swo3.aoff = 128;
  run<64, 1>("SW128 K-major A +1 row, SBO 8 rows", d, swo3);
  // no swizzle K-major: core matrix 8 rows x 16 B contiguous; LBO = K-chunk stride, SBO = 8-row group stride
  Cfg ns = {0, 0, 180 * 16, 128, 64 * 16, 128, 0, 0, 2 * 180 * 16, 2 * 64 * 16};
  run<64, 1>("NOSWZ K-major aligned (SBO 128)", d, ns);
  run<128, 1>("NOSWZ K-major aligned (SBO 128)", d, ns);
  Cfg ns1 = ns; ns1.aoff = 16; ns1.asbo = 160;
  run<64, 1>("NOSWZ K-major A +16B, SBO 160 (halo rows)", d, ns1);
  run<128, 1>("NOSWZ K-major A +16B, SBO 160 (halo rows)", d, ns1);
  Cfg ns2 = ns; ns2.aoff = 48; ns2.asbo = 160; ns2.alo = 181 * 16;
  run<64, 1>("NOSWZ K-major A +48B, SBO 160, LBO odd", d, ns2);
  // MN-major (wgrad): SW128 and no-swizzle
  Cfg mn = {2, 0, 16384, 1024, 16384, 1024, 1, 1, 2048, 2048};
  run<64, 1>("SW128 MN-major aligned", d, mn);
  run<128, 1>("SW128 MN-major aligned", d, mn);
  Cfg mno = mn; mno.aoff = 128; mno.asbo = 1280;
  run<64, 1>("SW128 MN-major A +1 row (haloed wgrad)", d, mno);
  Cfg mnh = {2, 128 * 7, 128 * 37, 1280, 16384, 1024, 1, 1, 2560, 2048};
  run<64, 1>("SW128 MN-major A haloed (+7 rows, LBO 37 rows, SBO 10 rows)", d, mnh);
  Cfg mnh2 = mnh; mnh2.aoff = 0; mnh2.alo = 128 * 40; mnh2.asbo = 1280;
  run<64, 1>("SW128 MN-major A (LBO 40 rows, SBO 10 rows)", d, mnh2);
  Cfg mnh3 = mnh; mnh3.aoff = 0; mnh3.alo = 16384; mnh3.asbo = 1280;
  run<64, 1>("SW128 MN-major A (LBO 16K, SBO 10 rows)", d, mnh3);
  Cfg mnh4 = mnh; mnh4.aoff = 128 * 3; mnh4.alo = 16384; mnh4.asbo = 1024;
  run<64, 1>("SW128 MN-major A (+3 rows, LBO 16K, SBO 8 rows)", d, mnh4);
  Cfg mnn = {0, 16, 160, 180 * 16, 128, 128 * 16, 1, 1, 2 * 160, 256};
  run<64, 1>("NOSWZ MN-major A +16B LBO 160", d, mnn);
  run<128, 1>("NOSWZ MN-major A +16B LBO 160", d, mnn);
  // 2-CTA pairs
  run<64, 2>("SW128 K-major aligned", d, sw);
  run<128, 2>("SW128 K-major aligned", d, sw);
  run<256, 2>("SW128 K-major aligned", d, sw);
  run<64, 2>("NOSWZ K-major A +16B, SBO 160 (halo rows)", d, ns1);
  run<128, 2>("NOSWZ K-major A +16B, SBO 160 (halo rows)", d, ns1);
  run<64, 2>("SW128 MN-major aligned", d, mn);
  run<64, 2>("NOSWZ MN-major A +16B LBO 160", d, mnn);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
