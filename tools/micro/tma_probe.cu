// Micro-benchmark (B200): TMA box-load throughput for the stage-1 activation
// (8 x 23 x 28 x 23 x 64 bf16, L2-resident) with (a) SW128 boxes {64ch,10w,18h,1d}
// and (b) 16-B-inner boxes {8ch,10w,18h,1d,8 chunks} (no swizzle, chunk-major smem),
// (c) cp.async 16-B copies into the chunk-major layout by 2 warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2104_05035_b200/csrc tma_probe.cu -o tma_probe -lcuda
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "tc_ptx.cuh"
using namespace rn;

constexpr int N = 8, D = 23, H = 28, W = 23, C = 64;
constexpr int BW = 10, BH = 18;
constexpr int BOX = BW * BH * 128;  // 23040
constexpr int ST = 6;

__global__ void __launch_bounds__(128, 1) ktma(const __grid_constant__ CUtensorMap m, int mode, int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[ST];
  if (threadIdx.x == 0) { for (int i = 0; i < ST; ++i) tc::mbar_init(&full[i], 1); tc::fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  int it = 0;
  for (int i = 0; i < iters; ++i) {
    const int st = i % ST;
    if (i >= ST) tc::mbar_wait(&full[st], ((i / ST) - 1) & 1);
    tc::mbar_arrive_expect_tx(&full[st], BOX);
    const int b = blockIdx.x * 7 + i;
    const int w0 = (b % 3) * 8 - 1, h0 = ((b / 3) % 2) * 16 - 1, d = (b / 6) % D, n = (b / 138) % N;
    if (mode == 0) tc::tma_load_5d(s + st * BOX, &m, &full[st], 0, w0, h0, d, n);
    else tc::tma_load_5d(s + st * BOX, &m, &full[st], 0, w0, h0, n * D + d, 0);
    ++it;
  }
  for (int i = iters - ST; i < iters; ++i) tc::mbar_wait(&full[i % ST], (i / ST) & 1);
  out[blockIdx.x] = clock64() - t0;
}

// cp.async chunk-major copy: warps 0..NW-1 copy a (10 x 18) x 64ch box as [8 chunks][180 rows][16 B]
__global__ void __launch_bounds__(128, 1) kcpa(const __nv_bfloat16 *x, int iters, int nw, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[ST];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { for (int i = 0; i < ST; ++i) tc::mbar_init(&full[i], nw * 32); tc::fence_barrier_init(); }
  __syncthreads();
  if (warp >= nw) return;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int st = i % ST;
    if (i >= ST) tc::mbar_wait(&full[st], ((i / ST) - 1) & 1);
    const int b = blockIdx.x * 7 + i;
    const int w0 = (b % 3) * 8 - 1, h0 = ((b / 3) % 2) * 16 - 1, d = (b / 6) % D, n = (b / 138) % N;
    const uint32_t dst0 = tc::smem_u32(s + st * BOX);
    for (int e = warp * 32 + lane; e < BW * BH * 8; e += nw * 32) {
      const int ch = e & 7, r = e >> 3, ww = w0 + r % BW, hh = h0 + r / BW;
      const bool ok = ww >= 0 && ww < W && hh >= 0 && hh < H;
      const __nv_bfloat16 *src = x + ((((int64_t)n * D + d) * H + (ok ? hh : 0)) * W + (ok ? ww : 0)) * C + ch * 8;
      const uint32_t dst = dst0 + (ch * (BW * BH + 4) + r) * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[st])) : "memory");
  }
  for (int i = iters - ST; i < iters; ++i) tc::mbar_wait(&full[i % ST], (i / ST) & 1);
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  __nv_bfloat16 *x;
  const size_t n = (size_t)N * D * H * W * C;
  cudaMalloc(&x, n * 2);
  cudaMemset(x, 0, n * 2);
  long long *d;
  cudaMalloc(&d, 148 * 8);
  void *fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m0, m1;
  {
    cuuint64_t dims[5] = {C, W, H, D, N};
    cuuint64_t str[4] = {C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2, (cuuint64_t)D * H * W * C * 2};
    cuuint32_t box[5] = {64, BW, BH, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    printf("enc0 %d\n", (int)enc(&m0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {
    cuuint64_t dims[5] = {8, W, H, (cuuint64_t)D * N, 8};
    cuuint64_t str[4] = {C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2, 16};
    cuuint32_t box[5] = {8, BW, BH, 1, 8}, es[5] = {1, 1, 1, 1, 1};
    printf("enc1 %d\n", (int)enc(&m1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  const int smem = ST * BOX + 2048;
  cudaFuncSetAttribute(ktma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kcpa, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * (BOX + 8 * 64) + 2048);
  const int iters = 2000;
  long long h[148];
  for (int rep = 0; rep < 2; ++rep) {
    for (int mode = 0; mode < 2; ++mode) {
      ktma<<<148, 128, smem>>>(mode ? m1 : m0, mode, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("TMA %s: %.1f B/cyc/SM, %.0f B/cyc chip  %s\n", mode ? "16B-inner chunk-major" : "SW128 64ch rows",
             (double)BOX * iters / mx, 148.0 * BOX * iters / mx, cudaGetErrorString(e));
    }
    for (int nw : {1, 2, 4}) {
      kcpa<<<148, 128, ST * (BOX + 8 * 64) + 2048>>>(x, iters, nw, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("cp.async %d warps: %.1f B/cyc/SM, %.0f B/cyc chip  %s\n", nw, (double)BOX * iters / mx, 148.0 * BOX * iters / mx,
             cudaGetErrorString(e));
    }
  }
}
