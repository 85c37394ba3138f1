// k_conv1x1.cu — the attention module's 1x1x1 convolutions at the stage-1
// resolution (the soft-mask branch's channel mixing; 64 -> 64
// channels over 8 x 23 x 28 x 23 voxels at the bench batch), forward and data
// gradient: y[v][n] = sum_k x[v][k] w[n][k] (+ bias[n]).  K = N = 64: one
// output row is 128 B and the whole GEMM is 1 GFLOP against 30 MB of HBM
// traffic, so the kernel is a streaming kernel on the warp tensor cores
// (mma.sync m16n8k16, bf16 -> fp32) rather than a tcgen05 one: the weights stay
// in smem (ldmatrix per tile), x tiles (128 voxels) stream through a cp.async double buffer,
// the output leaves through a swizzled smem tile as full-line stores, and the
// BatchNorm statistics (bnstats.cuh modes 1, 2, 3) accumulate per thread in
// registers across tiles — one [2][64] partial per block, no per-row warp
// transposes (what made the persistent tcgen05 kernel epilogue-bound here:
// 20-40 us per launch for a 5 us roofline).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "bnstats.cuh"
#include "error.h"
#include "kernels.h"
#include "launch.h"
#include "tc_conv.h"
#include "util.cuh"

namespace rn {

namespace {

constexpr int C1_THREADS = 256;  // 8 warps x 16 voxels = 128-voxel tiles
constexpr int C1_TILE = 128;
constexpr int C1_SMEM = 8192 + 2 * 16384 + 2 * 16384 + 16384 + (8 * 2 * 64 + 4 * 64) * 4;  // W, x[2], h[2], out, stats, consts

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
// byte offset of 16-B chunk j of row r in a 128-B-row tile, XOR-swizzled (conflict-free ldmatrix / row stores)
__device__ __forceinline__ uint32_t swz(int r, int j) { return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4)); }

struct C1Args {
  const bf16 *x, *w;
  const float *bias;
  bf16 *y;
  int64_t V;
  EpiStats st;
};

// tile t of x (and of h for the statistics of mode 3) into buffer b
__device__ __forceinline__ void c1_stage(const C1Args &a, int64_t t, uint32_t xs, uint32_t hs, int MODE) {
  const int64_t r0 = t * C1_TILE;
  for (int e = threadIdx.x; e < C1_TILE * 8; e += C1_THREADS) {
    const int r = e >> 3, j = e & 7;
    const bool ok = r0 + r < a.V;
    const int64_t g = ok ? (r0 + r) * 64 + j * 8 : 0;
    cp16(xs + swz(r, j), a.x + g, ok);
    if (MODE >= 2) cp16(hs + swz(r, j), a.st.h + g, ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int MODE>  // 0 no statistics, 1 forward (sum y, sum y^2), 2 / 3 backward (mask tensor / recomputed)
__global__ void __launch_bounds__(C1_THREADS, 2) conv1x1_k(const C1Args a) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t *sW = sm, *sX = sm + 8192, *sH = sX + 2 * 16384, *sO = sH + 2 * 16384;
  float *sred = reinterpret_cast<float *>(sO + 16384);  // [8 warps][2][64]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  float *sb = sred + 8 * 2 * 64, *smu = sb + 64, *sms = smu + 64, *smh = sms + 64;  // per-channel epilogue constants
  const int64_t ntiles = (a.V + C1_TILE - 1) / C1_TILE;
  pdl_begin();
  // weights [n][k] -> smem (swizzled rows) -> B fragments in registers for the whole kernel
  for (int e = threadIdx.x; e < 64 * 8; e += C1_THREADS) {
    const int r = e >> 3, j = e & 7;
    *reinterpret_cast<uint4 *>(sW + swz(r, j)) = *reinterpret_cast<const uint4 *>(a.w + r * 64 + j * 8);
  }
  if (threadIdx.x < 64) {
    const int n = threadIdx.x;
    sb[n] = a.bias ? a.bias[n] : 0.f;
    smu[n] = MODE >= 2 ? a.st.mean[n] : 0.f;
    sms[n] = MODE == 3 ? a.st.mscale[n] : 0.f;
    smh[n] = MODE == 3 ? a.st.mshift[n] : 0.f;
  }
  const uint32_t sWa = (uint32_t)__cvta_generic_to_shared(sW), sXa = (uint32_t)__cvta_generic_to_shared(sX),
                 sHa = (uint32_t)__cvta_generic_to_shared(sH);
  if ((int64_t)blockIdx.x < ntiles) c1_stage(a, blockIdx.x, sXa, sHa, MODE);
  __syncthreads();
  float s1[16], s2[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) s1[i] = s2[i] = 0.f;
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) {
      c1_stage(a, tn, sXa + ((it + 1) & 1) * 16384, sHa + ((it + 1) & 1) * 16384, MODE);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint32_t xb = sXa + (it & 1) * 16384;
    const uint8_t *hb = sH + (it & 1) * 16384;
    const int wr = warp * 16;  // this warp's 16 rows of the tile
    float acc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t af[4];
      // A (16 x 16): matrices (rows 0-7 / 8-15) x (k 0-7 / 8-15) -> a0, a1, a2, a3
      const int r = wr + (lane & 15), j = kk * 2 + (lane >> 4);
      ldsm_x4(xb + swz(r, j), af[0], af[1], af[2], af[3]);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        // B (k16 x n8 of w[n][k] rows) for n-tiles 2np, 2np+1: matrices (tile, k chunk 2kk / 2kk+1)
        uint32_t b0, b1, b2, b3;
        const int rb = (2 * np + (lane >> 4)) * 8 + (lane & 7), jb = kk * 2 + ((lane >> 3) & 1);
        ldsm_x4(sWa + swz(rb, jb), b0, b1, b2, b3);
        mma16816(acc[2 * np], af, b0, b1);
        mma16816(acc[2 * np + 1], af, b2, b3);
      }
    }
    // epilogue: rows wr + g (e = 0, 1) and wr + g + 8 (e = 2, 3), columns 8nt + 2q + (e & 1)
    const int64_t row0 = t * C1_TILE;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int r = wr + g + 8 * hr;
      const bool valid = row0 + r < a.V;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int n = nt * 8 + 2 * q;
        const float2 bv = *reinterpret_cast<const float2 *>(sb + n);
        const float f0 = acc[nt][2 * hr] + bv.x, f1 = acc[nt][2 * hr + 1] + bv.y;
        const __nv_bfloat162 o = __floats2bfloat162_rn(f0, f1);
        const uint32_t off = swz(r, nt) + 4 * q;
        *reinterpret_cast<__nv_bfloat162 *>(sO + off) = o;
        if (MODE != 0 && valid) {
          const float2 of = __bfloat1622float2(o);  // statistics of the stored values
          if (MODE == 1) {
            s1[2 * nt] += of.x;
            s2[2 * nt] = fmaf(of.x, of.x, s2[2 * nt]);
            s1[2 * nt + 1] += of.y;
            s2[2 * nt + 1] = fmaf(of.y, of.y, s2[2 * nt + 1]);
          } else {
            const float2 hv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(hb + off));
            const float2 muv = *reinterpret_cast<const float2 *>(smu + n);
            float2 mv;
            if (MODE == 3) {  // the consumer's ReLU mask recomputed from h
              const float2 msv = *reinterpret_cast<const float2 *>(sms + n);
              const float2 mhv = *reinterpret_cast<const float2 *>(smh + n);
              mv = make_float2(fmaf(hv.x, msv.x, mhv.x), fmaf(hv.y, msv.y, mhv.y));
            } else {  // mode 2: the stored mask tensor (non-default path; read in place)
              mv = __bfloat1622float2(
                  __ldg(reinterpret_cast<const __nv_bfloat162 *>(a.st.mask + (row0 + r) * 64 + n)));
            }
            const float d0 = mv.x > 0.f ? of.x : 0.f;
            const float d1 = mv.y > 0.f ? of.y : 0.f;
            s1[2 * nt] += d0;
            s2[2 * nt] = fmaf(d0, hv.x - muv.x, s2[2 * nt]);
            s1[2 * nt + 1] += d1;
            s2[2 * nt + 1] = fmaf(d1, hv.y - muv.y, s2[2 * nt + 1]);
          }
        }
      }
    }
    __syncwarp();
    // the warp's 16 rows leave as full 128-B lines
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = i * 32 + lane, r = wr + (e >> 3), j = e & 7;
      if (row0 + r < a.V)
        *reinterpret_cast<uint4 *>(a.y + (row0 + r) * 64 + j * 8) = *reinterpret_cast<const uint4 *>(sO + swz(r, j));
    }
    __syncthreads();  // buffer (it & 1) is restaged by the next iteration
  }
  if constexpr (MODE != 0) {
  // statistics: lanes sharing q (the 8 row groups g) in a fixed xor order, warps in order
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int o = 4; o <= 16; o <<= 1) {
      s1[i] += __shfl_xor_sync(0xffffffffu, s1[i], o);
      s2[i] += __shfl_xor_sync(0xffffffffu, s2[i], o);
    }
  if (g == 0)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = nt * 8 + 2 * q + e;
        sred[(warp * 2 + 0) * 64 + n] = s1[2 * nt + e];
        sred[(warp * 2 + 1) * 64 + n] = s2[2 * nt + e];
      }
  __syncthreads();
  if (threadIdx.x < 128) {
    const int k = threadIdx.x >> 6, n = threadIdx.x & 63;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += sred[(w * 2 + k) * 64 + n];
    a.st.part[(int64_t)blockIdx.x * 128 + k * 64 + n] = s;
  }
  }
}

}  // namespace

bool conv1x1_supported(const ConvGeom &g) {
  return g.k == 1 && g.s == 1 && g.p == 0 && g.Ci == 64 && g.Co == 64 && g.Di == g.Do && g.Hi == g.Ho &&
         g.Wi == g.Wo && g.out_vox() >= 16384;
}

int conv1x1(const ConvGeom &g, const bf16 *x, const bf16 *w, const float *bias, bf16 *y, cudaStream_t st,
            const EpiStats *stats) {
  const int mode = stats ? stats->mode : 0;
  if (!conv1x1_supported(g) || mode < 0 || mode > 3)
    throw Error(RN_ERR_ARG, "conv1x1: unsupported geometry / statistics mode");
  C1Args a{x, w, bias, y, g.out_vox(), stats ? *stats : EpiStats()};
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (a.V + C1_TILE - 1) / C1_TILE;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, 2 * nsm);
  static uint64_t attr_devs = 0;  // kernel attributes are per device
  if (!once_on_device(attr_devs)) {
    CUDA_CHECK(cudaFuncSetAttribute(conv1x1_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, C1_SMEM));
    CUDA_CHECK(cudaFuncSetAttribute(conv1x1_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, C1_SMEM));
    CUDA_CHECK(cudaFuncSetAttribute(conv1x1_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, C1_SMEM));
    CUDA_CHECK(cudaFuncSetAttribute(conv1x1_k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, C1_SMEM));
  }
  if (mode == 0) launch_k(conv1x1_k<0>, grid, C1_THREADS, C1_SMEM, st, a);
  else if (mode == 1) launch_k(conv1x1_k<1>, grid, C1_THREADS, C1_SMEM, st, a);
  else if (mode == 2) launch_k(conv1x1_k<2>, grid, C1_THREADS, C1_SMEM, st, a);
  else launch_k(conv1x1_k<3>, grid, C1_THREADS, C1_SMEM, st, a);
  LAUNCH_CHECK();
  return mode ? (int)grid : 0;
}

}  // namespace rn
