// k_stem.cu — the stem Conv block's 3x3x3 convolution with one input channel
// ("Conv blocks use a 3D filter for computation of the low-level
// feature representations"; reading X4: conv 1 -> C0, stride 2, pad 1).
// K = 27 is far too small for a tensor-core tile and the layer is bound by
// writing its C0-channel output (fprop) / reading it (wgrad), so both are
// fp32 SIMT kernels (fp32 master weights, fp32 input, exactly the arithmetic
// the bf16-storage oracle specifies):
//   fprop: one thread per output voxel computes all C0 channels; the 27 input
//          taps come through L1, the 27 x C0 weights are smem broadcasts;
//          the warp writes 32 consecutive voxels = one contiguous NDHWC run.
//   wgrad: dW[co][tap] = sum_v dh[v][co] x[v + off(tap)]; each block stages 32
//          voxels of dh (16-B vectors) and their 27-tap input patches in smem,
//          216 threads own (8 channels x 1 tap) accumulators; per-block
//          partials are reduced in a fixed order (deterministic).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "error.h"
#include "launch.h"
#include "kernels.h"
#include "util.cuh"

namespace rn {

namespace {

// part (optional): fused BN statistics of the stored output, [gridDim.x][2][CO] = (sum y, sum y^2)
template <typename T, int CO>
__global__ void __launch_bounds__(128) stem_fprop_k(ConvGeom g, const float *__restrict__ x,
                                                   const float *__restrict__ w, T *__restrict__ y,
                                                   float *__restrict__ part) {
  pdl_begin();
  constexpr int HG = 128 / CO;  // thread groups summing one channel
  float s1 = 0.f, s2 = 0.f;
  __shared__ __align__(16) float ws[27 * CO];
  for (int i = threadIdx.x; i < 27 * CO; i += blockDim.x) {
    const int co = i % CO, tap = i / CO;
    ws[i] = w[co * 27 + tap];
  }
  // Each thread computes VPT voxels (rows t, t + 128, ...): every weight vector
  // read from smem (a warp-wide broadcast) feeds VPT x 8 FMAs (one voxel per
  // thread measured smem-wavefront-bound at 68-79%).
  constexpr int VPT = (int)(sizeof(T) * CO * 256 <= 32768 ? 2 : 1);
  constexpr int ROWS = 128 * VPT;
  // output staging: the block's ROWS voxels x CO channels, stored back with
  // consecutive threads on consecutive 16-B chunks (full L2 sectors).  Row v's
  // 16-B chunk q sits at chunk (q ^ (v & SWM)): the per-thread row writes (one
  // row per thread, 128-B apart) would otherwise all hit the same 4 banks
  __shared__ __align__(16) T so[ROWS * CO];
  constexpr int VE = 16 / sizeof(T);   // elements per 16-B chunk
  constexpr int NCH = CO / VE;         // chunks per row
  constexpr int SWM = (NCH < 8 ? NCH : 8) - 1;
  auto chunk_ptr = [&](int row, int q) { return so + (row * NCH + (q ^ (row & SWM))) * VE; };
  __syncthreads();
  const int64_t total = g.out_vox();
  for (int64_t vb = blockIdx.x * (int64_t)ROWS; vb < total; vb += (int64_t)gridDim.x * ROWS) {
    float xv[VPT][27];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int64_t vo = vb + threadIdx.x + 128 * u;
      int64_t r = vo < total ? vo : total - 1;
      const int ow = (int)(r % g.Wo); r /= g.Wo;
      const int oh = (int)(r % g.Ho); r /= g.Ho;
      const int od = (int)(r % g.Do); r /= g.Do;
      const int n = (int)r;
#pragma unroll
      for (int tap = 0; tap < 27; ++tap) {
        const int id = od * g.s + tap / 9 - g.p, ih = oh * g.s + (tap / 3) % 3 - g.p, iw = ow * g.s + tap % 3 - g.p;
        const bool ok = id >= 0 && id < g.Di && ih >= 0 && ih < g.Hi && iw >= 0 && iw < g.Wi;
        xv[u][tap] = ok ? __ldg(&x[(((int64_t)n * g.Di + id) * g.Hi + ih) * g.Wi + iw]) : 0.f;
      }
    }
#pragma unroll
    for (int c0 = 0; c0 < CO; c0 += 8) {
      float acc[VPT][8];
#pragma unroll
      for (int u = 0; u < VPT; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[u][j] = 0.f;
#pragma unroll
      for (int tap = 0; tap < 27; ++tap) {
        const float4 a = *reinterpret_cast<const float4 *>(&ws[tap * CO + c0]);
        const float4 b = *reinterpret_cast<const float4 *>(&ws[tap * CO + c0 + 4]);
#pragma unroll
        for (int u = 0; u < VPT; ++u) {
          const float xt = xv[u][tap];
          acc[u][0] = fmaf(xt, a.x, acc[u][0]);
          acc[u][1] = fmaf(xt, a.y, acc[u][1]);
          acc[u][2] = fmaf(xt, a.z, acc[u][2]);
          acc[u][3] = fmaf(xt, a.w, acc[u][3]);
          acc[u][4] = fmaf(xt, b.x, acc[u][4]);
          acc[u][5] = fmaf(xt, b.y, acc[u][5]);
          acc[u][6] = fmaf(xt, b.z, acc[u][6]);
          acc[u][7] = fmaf(xt, b.w, acc[u][7]);
        }
      }
#pragma unroll
      for (int u = 0; u < VPT; ++u)
#pragma unroll
        for (int h = 0; h < 8; h += VE) store_vec(chunk_ptr(threadIdx.x + 128 * u, (c0 + h) / VE), acc[u] + h);
    }
    __syncthreads();
    const int64_t nvox = min((int64_t)ROWS, total - vb);
    if (part) {  // statistics of the stored (rounded) values, channel t % CO
      const int c = threadIdx.x % CO;
      for (int v = threadIdx.x / CO; v < nvox; v += HG) {
        const float f = to_f(chunk_ptr(v, c / VE)[c % VE]);
        s1 += f;
        s2 = fmaf(f, f, s2);
      }
    }
    const int nchunk = (int)(nvox * CO / VE);
    for (int i = threadIdx.x; i < nchunk; i += blockDim.x)
      reinterpret_cast<uint4 *>(y + vb * CO)[i] = *reinterpret_cast<const uint4 *>(chunk_ptr(i / NCH, i % NCH));
    __syncthreads();
  }
  if (part) {
    __shared__ float r1[128], r2[128];
    r1[threadIdx.x] = s1;
    r2[threadIdx.x] = s2;
    __syncthreads();
    if (threadIdx.x < CO) {
      float a = 0.f, b = 0.f;
      for (int q = 0; q < HG; ++q) {
        a += r1[q * CO + threadIdx.x];
        b += r2[q * CO + threadIdx.x];
      }
      part[(int64_t)blockIdx.x * 2 * CO + threadIdx.x] = a;
      part[(int64_t)blockIdx.x * 2 * CO + CO + threadIdx.x] = b;
    }
  }
}

constexpr int WV = 32;  // voxels staged per iteration

template <typename T, int CO>
__global__ void __launch_bounds__(256) stem_wgrad_k(ConvGeom g, const float *__restrict__ x,
                                                   const T *__restrict__ dh, float *__restrict__ part,
                                                   int64_t vox_per_block) {
  pdl_begin();
  constexpr int G = CO / 8;
  __shared__ __align__(16) float sdh[WV][CO];
  __shared__ float sx[WV][28];
  const int t = threadIdx.x;
  const int cg = t / 27, tap = t % 27;
  const bool active = t < G * 27;
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  const int64_t total = g.out_vox();
  const int64_t v0 = (int64_t)blockIdx.x * vox_per_block;
  const int64_t v1 = min(total, v0 + vox_per_block);
  for (int64_t vb = v0; vb < v1; vb += WV) {
    __syncthreads();
    // stage dh: WV voxels x CO channels
    for (int i = t; i < WV * G; i += blockDim.x) {
      const int vv = i / G, c = (i % G) * 8;
      float f[8];
      if (vb + vv < v1) {
        if constexpr (sizeof(T) == 2) {
          load_vec(dh + (vb + vv) * CO + c, f);
        } else {
          load_vec(dh + (vb + vv) * CO + c, f);
          load_vec(dh + (vb + vv) * CO + c + 4, f + 4);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sdh[vv][c + j] = f[j];
    }
    // stage the 27-tap input patches
    for (int i = t; i < WV * 27; i += blockDim.x) {
      const int vv = i / 27, tp = i % 27;
      float xv = 0.f;
      const int64_t vo = vb + vv;
      if (vo < v1) {
        int64_t r = vo;
        const int ow = (int)(r % g.Wo); r /= g.Wo;
        const int oh = (int)(r % g.Ho); r /= g.Ho;
        const int od = (int)(r % g.Do); r /= g.Do;
        const int n = (int)r;
        const int id = od * g.s + tp / 9 - g.p, ih = oh * g.s + (tp / 3) % 3 - g.p, iw = ow * g.s + tp % 3 - g.p;
        if (id >= 0 && id < g.Di && ih >= 0 && ih < g.Hi && iw >= 0 && iw < g.Wi)
          xv = __ldg(&x[(((int64_t)n * g.Di + id) * g.Hi + ih) * g.Wi + iw]);
      }
      sx[vv][tp] = xv;
    }
    __syncthreads();
    if (active) {
#pragma unroll 8
      for (int vv = 0; vv < WV; ++vv) {
        const float xv = sx[vv][tap];
        const float4 a = *reinterpret_cast<const float4 *>(&sdh[vv][cg * 8]);
        const float4 b = *reinterpret_cast<const float4 *>(&sdh[vv][cg * 8 + 4]);
        acc[0] = fmaf(a.x, xv, acc[0]);
        acc[1] = fmaf(a.y, xv, acc[1]);
        acc[2] = fmaf(a.z, xv, acc[2]);
        acc[3] = fmaf(a.w, xv, acc[3]);
        acc[4] = fmaf(b.x, xv, acc[4]);
        acc[5] = fmaf(b.y, xv, acc[5]);
        acc[6] = fmaf(b.z, xv, acc[6]);
        acc[7] = fmaf(b.w, xv, acc[7]);
      }
    }
  }
  if (active) {
    float *P = part + (int64_t)blockIdx.x * CO * 27;
#pragma unroll
    for (int j = 0; j < 8; ++j) P[(cg * 8 + j) * 27 + tap] = acc[j];
  }
}

// wgrad, warp-per-voxel-run: lane t < 27 owns tap t and all CO accumulators;
// the dh row of a voxel is read once per warp (same address in every lane =
// L1 broadcast), the input value at the lane's tap is a gather.
template <typename T, int CO>
__global__ void __launch_bounds__(256) stem_wgrad_warp_k(ConvGeom g, const float *__restrict__ x,
                                                        const T *__restrict__ dh, float *__restrict__ part,
                                                        int64_t vox_per_warp) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int64_t total = g.out_vox();
  const int64_t v0 = wid * vox_per_warp, v1 = min(total, v0 + vox_per_warp);
  const int tap = lane < 27 ? lane : 26;
  const int kd = tap / 9 - g.p, kh = (tap / 3) % 3 - g.p, kw = tap % 3 - g.p;
  float acc[CO];
#pragma unroll
  for (int c = 0; c < CO; ++c) acc[c] = 0.f;
  if (v0 < v1) {
    int64_t r = v0;
    int ow = (int)(r % g.Wo); r /= g.Wo;
    int oh = (int)(r % g.Ho); r /= g.Ho;
    int od = (int)(r % g.Do); r /= g.Do;
    int n = (int)r;
    for (int64_t v = v0; v < v1; ++v) {
      const int id = od * g.s + kd, ih = oh * g.s + kh, iw = ow * g.s + kw;
      float xv = 0.f;
      if (id >= 0 && id < g.Di && ih >= 0 && ih < g.Hi && iw >= 0 && iw < g.Wi)
        xv = __ldg(&x[(((int64_t)n * g.Di + id) * g.Hi + ih) * g.Wi + iw]);
      const T *row = dh + v * CO;
#pragma unroll
      for (int c = 0; c < CO; c += Vec<T>::N) {
        float d[Vec<T>::N];
        load_vec(row + c, d);
#pragma unroll
        for (int j = 0; j < Vec<T>::N; ++j) acc[c + j] = fmaf(d[j], xv, acc[c + j]);
      }
      if (++ow == g.Wo) {
        ow = 0;
        if (++oh == g.Ho) {
          oh = 0;
          if (++od == g.Do) { od = 0; ++n; }
        }
      }
    }
  }
  // block reduction of the 8 warps (fixed order): warps 4-7 store, warps 0-3 add, then 4 slots summed
  __shared__ float red[4][27 * CO];
  const int w = threadIdx.x / 32;
  if (w >= 4 && lane < 27)
#pragma unroll
    for (int c = 0; c < CO; ++c) red[w - 4][lane * CO + c] = acc[c];
  __syncthreads();
  if (w < 4 && lane < 27)
#pragma unroll
    for (int c = 0; c < CO; ++c) red[w][lane * CO + c] += acc[c];
  __syncthreads();
  for (int i = threadIdx.x; i < 27 * CO; i += blockDim.x) {
    const int tp = i / CO, co = i % CO;
    part[(int64_t)blockIdx.x * 27 * CO + co * 27 + tp] = ((red[0][i] + red[1][i]) + red[2][i]) + red[3][i];
  }
}

// wgrad on the legacy warp tensor cores (mma.sync m16n8k16, bf16 -> fp32) for the
// bf16 path: dW[co][tap] = sum_v dh[v][co] * x[v + off(tap)] is a thin GEMM
// (M = 64 channels, N = 27 taps padded to 32, K = voxels).  dh is bf16 already;
// the fp32 input is split x = x_hi + x_lo (two bf16, |x - x_hi - x_lo| <= 2^-17 |x|)
// and both halves go through the MMA, so every product dh*x is formed exactly
// to ~2^-17 and accumulated in fp32 — the fp32-input reading of the stem.
// Block = 8 warps over chunks of 256 voxels: dh tile [256][64] (16-B chunks
// XOR-swizzled by row for conflict-free ldmatrix.trans) and the 27-tap input
// patches [256][36] fp32 in smem; warp w takes k-steps w and w+8 (16 voxels
// each): 4 m-tiles x 4 n-tiles x (hi, lo) = 32 MMAs.  Per-block partials are
// reduced in a fixed order (split_reduce_add).
constexpr int SW_CH = 256;     // voxels per chunk
constexpr int SW_PS = 36;      // patch row stride (floats): conflict-free fragment reads
constexpr int SW_SMEM = SW_CH * 128 + SW_CH * SW_PS * 4;

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo_k, float hi_k) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo_k, hi_k);  // .x (low half) = first k
  uint32_t u;
  memcpy(&u, &v, 4);
  return u;
}

// fprop on the legacy warp tensor cores (bf16 path, C0 = 64): per warp a tile of
// 16 consecutive output voxels is the GEMM  Y[16 x 64] = P[16 x 32] W[32 x 64]
// (P = the 27-tap input patches, padded to K = 32).  Both fp32 operands are split
// into bf16 pairs (v = v_hi + v_lo, |v - v_hi - v_lo| <= 2^-17 |v|) and the three
// significant products hi*hi + hi*lo + lo*hi go through mma.m16n8k16 with fp32
// accumulation: each output is the fp32-input convolution to ~2^-16 relative,
// far below the bf16 rounding of the stored output (the SIMT kernel it replaces
// issued one smem weight load per 8 FMAs and was smem-pipe-bound at 150 us).
// W fragments (hi and lo) stay in registers for the whole kernel.  The tile goes
// through a per-warp smem staging tile (16-B chunks XOR-swizzled by row) so the
// global stores are full 16-B vectors; BN statistics (sum, sum of squares of
// the stored bf16 values) accumulate in registers and are reduced once per block.
constexpr int SF_WARPS = 4;
__global__ void __launch_bounds__(SF_WARPS * 32) stem_fprop_mma_k(ConvGeom g, const float *__restrict__ x,
                                                               const float *__restrict__ w, bf16 *__restrict__ y,
                                                               float *__restrict__ part) {
  __shared__ __align__(16) uint32_t stile[SF_WARPS][16 * 32];  // [voxel][64 ch] bf16, swizzled 16-B chunks
  __shared__ float sred[SF_WARPS][2][64];
  pdl_begin();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  // B fragments: k = tap (rows), n = channel (cols); b0 = (k 2tq, 2tq+1), b1 = (k 2tq+8, 2tq+9) + 16 ks
  uint32_t bh[2][8][2], bl[2][8][2];
#pragma unroll
  for (int ks = 0; ks < 2; ++ks)
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int t0 = 16 * ks + 2 * tq + 8 * r, co = n * 8 + gq;
        const float w0 = t0 < 27 ? w[co * 27 + t0] : 0.f, w1 = t0 + 1 < 27 ? w[co * 27 + t0 + 1] : 0.f;
        const float h0 = __bfloat162float(__float2bfloat16_rn(w0)), h1 = __bfloat162float(__float2bfloat16_rn(w1));
        bh[ks][n][r] = pack_bf16x2(h0, h1);
        bl[ks][n][r] = pack_bf16x2(w0 - h0, w1 - h1);
      }
  float s1[16], s2[16];  // channels n*8 + 2tq + e  (index n*2 + e)
#pragma unroll
  for (int i = 0; i < 16; ++i) s1[i] = s2[i] = 0.f;
  const int64_t total = g.out_vox();
  const int64_t ntiles = (total + 15) / 16;
  uint32_t *st = stile[warp];
  // the next tile's patch values are loaded while the current tile computes
  // (software pipeline: one L1/L2 round trip per tile is hidden)
  float xv[2][2][4], xn_[2][2][4];  // [voxel half][ks][j]: tap = 16 ks + 2tq + (j & 1) + 8 (j >> 1)
  // this thread's 8 taps (fixed by tq): element offset and (kd, kh, kw) bits
  int toff[2][4], tbits[2][4];
#pragma unroll
  for (int ks = 0; ks < 2; ++ks)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int tap = 16 * ks + 2 * tq + (j & 1) + 8 * (j >> 1);
      const int kd = tap / 9, kh = (tap / 3) % 3, kw = tap % 3;
      toff[ks][j] = (kd * g.Hi + kh) * g.Wi + kw;
      tbits[ks][j] = tap < 27 ? (1 << kd) | (8 << kh) | (64 << kw) : 0;  // all-zero: padding tap
    }
  const int HWi = g.Hi * g.Wi;
  // voxel index < 2^31 (checked by the launcher): 32-bit coordinate decode
  auto load_patch = [&](int64_t tile, float (&dst)[2][2][4]) {
#pragma unroll
    for (int hv = 0; hv < 2; ++hv) {
      const int vo = (int)(tile * 16) + gq + 8 * hv;
      const bool live = tile < ntiles && vo < (int)total;
      int r = live ? vo : 0;
      const int ow = r % g.Wo; r /= g.Wo;
      const int oh = r % g.Ho; r /= g.Ho;
      const int od = r % g.Do;
      const int nn = r / g.Do;
      const int id0 = od * g.s - g.p, ih0 = oh * g.s - g.p, iw0 = ow * g.s - g.p;
      // valid-offset masks: bit kd (d), 3 + kh (h), 6 + kw (w)
      int vm = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        vm |= (id0 + k >= 0 && id0 + k < g.Di) ? (1 << k) : 0;
        vm |= (ih0 + k >= 0 && ih0 + k < g.Hi) ? (8 << k) : 0;
        vm |= (iw0 + k >= 0 && iw0 + k < g.Wi) ? (64 << k) : 0;
      }
      if (!live) vm = 0;
      const float *xb = x + (int64_t)nn * g.Di * HWi + ((int64_t)id0 * g.Hi + ih0) * g.Wi + iw0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int tb = tbits[ks][j];
          const bool ok = tb != 0 && (tb & vm) == tb;
          dst[hv][ks][j] = ok ? __ldg(xb + toff[ks][j]) : 0.f;
        }
    }
  };
  const int64_t tstride = (int64_t)gridDim.x * SF_WARPS;
  load_patch((int64_t)blockIdx.x * SF_WARPS + warp, xn_);
  for (int64_t tile = (int64_t)blockIdx.x * SF_WARPS + warp; tile < ntiles; tile += tstride) {
    const int64_t v0 = tile * 16;
#pragma unroll
    for (int hv = 0; hv < 2; ++hv)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int j = 0; j < 4; ++j) xv[hv][ks][j] = xn_[hv][ks][j];
    load_patch(tile + tstride, xn_);
    float acc[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[n][q] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t ah[4], al[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // a_q: q=0 (row gq, k 2tq..), 1 (row gq+8), 2 (row gq, k +8), 3 (row gq+8, k +8)
        const int hv = q & 1, jj = (q >> 1) * 2;
        const float p0 = xv[hv][ks][jj], p1 = xv[hv][ks][jj + 1];
        const float h0 = __bfloat162float(__float2bfloat16_rn(p0)), h1 = __bfloat162float(__float2bfloat16_rn(p1));
        ah[q] = pack_bf16x2(h0, h1);
        al[q] = pack_bf16x2(p0 - h0, p1 - h1);
      }
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        mma_bf16_16816(acc[n], al, bh[ks][n][0], bh[ks][n][1]);
        mma_bf16_16816(acc[n], ah, bl[ks][n][0], bl[ks][n][1]);
        mma_bf16_16816(acc[n], ah, bh[ks][n][0], bh[ks][n][1]);
      }
    }
    // round, statistics of the stored values, stage: row (voxel) v, 16-B chunk n at (n ^ (v & 7))
    __syncwarp();
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int hv = 0; hv < 2; ++hv) {
        const int v = gq + 8 * hv;
        const bool live = v0 + v < total;
        const __nv_bfloat162 b = __floats2bfloat162_rn(acc[n][2 * hv], acc[n][2 * hv + 1]);
        const float2 f = __bfloat1622float2(b);
        if (live) {
          s1[2 * n] += f.x;
          s2[2 * n] = fmaf(f.x, f.x, s2[2 * n]);
          s1[2 * n + 1] += f.y;
          s2[2 * n + 1] = fmaf(f.y, f.y, s2[2 * n + 1]);
        }
        uint32_t u;
        memcpy(&u, &b, 4);
        st[v * 32 + ((n ^ (v & 7)) << 2) + tq] = u;
      }
    __syncwarp();
    // 16 voxels x 128 B = 128 chunks of 16 B: lane takes chunks lane, lane+32, ...
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = lane + 32 * q, v = c >> 3, n = c & 7;
      if (v0 + v < total) {
        const uint4 val = *reinterpret_cast<const uint4 *>(st + v * 32 + ((n ^ (v & 7)) << 2));
        *reinterpret_cast<uint4 *>(y + (v0 + v) * 64 + n * 8) = val;
      }
    }
  }
  if (!part) return;
  // statistics: lanes with the same tq hold the same channels -> butterfly over gq (fixed order)
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      s1[i] += __shfl_xor_sync(0xffffffffu, s1[i], off);
      s2[i] += __shfl_xor_sync(0xffffffffu, s2[i], off);
    }
  if (gq == 0)
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        sred[warp][0][n * 8 + 2 * tq + e] = s1[2 * n + e];
        sred[warp][1][n * 8 + 2 * tq + e] = s2[2 * n + e];
      }
  __syncthreads();
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    const int k = i >> 6, c = i & 63;
    float a = 0.f;
#pragma unroll
    for (int q = 0; q < SF_WARPS; ++q) a += sred[q][k][c];
    part[(int64_t)blockIdx.x * 128 + k * 64 + c] = a;
  }
}


// hx/coef (optional): the BN-backward apply fused into the staging, dh = bf16(A d' + B h + Cc)
// with dh holding d' (bn_bwd_apply_k's arithmetic, coef = [A | B | Cc] per channel)
__global__ void __launch_bounds__(256, 2) stem_wgrad_mma_k(ConvGeom g, const float *__restrict__ x,
                                                       const bf16 *__restrict__ dh, float *__restrict__ part,
                                                       const bf16 *__restrict__ hx, const float *__restrict__ coef) {
  extern __shared__ __align__(16) uint8_t sm[];
  pdl_begin();
  uint8_t *sdh = sm;                                  // [256][128 B], chunk c of row v at ((c ^ (v & 7)) * 16)
  float *sp = reinterpret_cast<float *>(sm + SW_CH * 128);  // [256][36]
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gq = lane >> 2, tq = lane & 3;
  float acc[4][4][4];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[m][n][r] = 0.f;
  const int64_t total = g.out_vox();
  // fused apply: this thread's staging chunk is always channel group (t & 7)
  float cA[8], cB[8], cC[8];
  if (coef) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = (t & 7) * 8 + e;
      cA[e] = coef[c];
      cB[e] = coef[64 + c];
      cC[e] = coef[128 + c];
    }
  }
  for (int64_t v0 = (int64_t)blockIdx.x * SW_CH; v0 < total; v0 += (int64_t)gridDim.x * SW_CH) {
    __syncthreads();
    // dh tile: 256 rows x 8 chunks of 16 B
    if (coef) {
      uint4 dv[8], hv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = t + 256 * j, row = i >> 3, c = i & 7;
        dv[j] = hv[j] = make_uint4(0, 0, 0, 0);
        if (v0 + row < total) {
          dv[j] = __ldg(reinterpret_cast<const uint4 *>(dh + (v0 + row) * 64) + c);
          hv[j] = __ldg(reinterpret_cast<const uint4 *>(hx + (v0 + row) * 64) + c);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = t + 256 * j, row = i >> 3, c = i & 7;
        float d[8], hh[8], o[8];
        const __nv_bfloat162 *pd = reinterpret_cast<const __nv_bfloat162 *>(&dv[j]);
        const __nv_bfloat162 *ph = reinterpret_cast<const __nv_bfloat162 *>(&hv[j]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 a = __bfloat1622float2(pd[q]), b = __bfloat1622float2(ph[q]);
          d[2 * q] = a.x; d[2 * q + 1] = a.y;
          hh[2 * q] = b.x; hh[2 * q + 1] = b.y;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = v0 + row < total ? fmaf(cA[e], d[e], fmaf(cB[e], hh[e], cC[e])) : 0.f;
        uint4 v;
        __nv_bfloat162 *pv = reinterpret_cast<__nv_bfloat162 *>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) pv[q] = __floats2bfloat162_rn(o[2 * q], o[2 * q + 1]);
        *reinterpret_cast<uint4 *>(sdh + row * 128 + ((c ^ (row & 7)) << 4)) = v;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = t + 256 * j, row = i >> 3, c = i & 7;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (v0 + row < total) v = __ldg(reinterpret_cast<const uint4 *>(dh + (v0 + row) * 64) + c);
        *reinterpret_cast<uint4 *>(sdh + row * 128 + ((c ^ (row & 7)) << 4)) = v;
      }
    }
    // input patches: thread t = voxel v0 + t, its 27 taps (stride-2 stem geometry)
    {
      const int64_t vo = v0 + t;
      float *prow = sp + t * SW_PS;
      if (vo < total) {
        int r = (int)vo;  // < 2^31 (checked by the launcher): 32-bit decode
        const int ow = r % g.Wo; r /= g.Wo;
        const int oh = r % g.Ho; r /= g.Ho;
        const int od = r % g.Do;
        const int n = r / g.Do;
        const float *xn = x + (int64_t)n * g.Di * g.Hi * g.Wi;
#pragma unroll
        for (int tap = 0; tap < 27; ++tap) {
          const int id = od * g.s + tap / 9 - g.p, ih = oh * g.s + (tap / 3) % 3 - g.p, iw = ow * g.s + tap % 3 - g.p;
          const bool ok = id >= 0 && id < g.Di && ih >= 0 && ih < g.Hi && iw >= 0 && iw < g.Wi;
          prow[tap] = ok ? __ldg(xn + ((int64_t)id * g.Hi + ih) * g.Wi + iw) : 0.f;
        }
      } else {
#pragma unroll
        for (int tap = 0; tap < 27; ++tap) prow[tap] = 0.f;
      }
#pragma unroll
      for (int tap = 27; tap < 32; ++tap) prow[tap] = 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int vb = (warp + 8 * ks) * 16;  // this warp's 16-voxel k-step
      // A fragments (dh^T: rows co, cols v) via ldmatrix.trans from the [v][co] tile
      uint32_t a[4][4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int q = lane >> 3, row = vb + (lane & 7) + ((q >> 1) << 3), c = m * 2 + (q & 1);
        const uint32_t addr = (uint32_t)__cvta_generic_to_shared(sdh + row * 128 + ((c ^ (row & 7)) << 4));
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a[m][0]), "=r"(a[m][1]), "=r"(a[m][2]), "=r"(a[m][3])
                     : "r"(addr));
      }
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const int col = n * 8 + gq;
        const float p0 = sp[(vb + 2 * tq) * SW_PS + col], p1 = sp[(vb + 2 * tq + 1) * SW_PS + col];
        const float p8 = sp[(vb + 2 * tq + 8) * SW_PS + col], p9 = sp[(vb + 2 * tq + 9) * SW_PS + col];
        const float h0 = __bfloat162float(__float2bfloat16_rn(p0)), h1 = __bfloat162float(__float2bfloat16_rn(p1));
        const float h8 = __bfloat162float(__float2bfloat16_rn(p8)), h9 = __bfloat162float(__float2bfloat16_rn(p9));
        const uint32_t bh0 = pack_bf16x2(h0, h1), bh1 = pack_bf16x2(h8, h9);
        const uint32_t bl0 = pack_bf16x2(p0 - h0, p1 - h1), bl1 = pack_bf16x2(p8 - h8, p9 - h9);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          mma_bf16_16816(acc[m][n], a[m], bh0, bh1);
          mma_bf16_16816(acc[m][n], a[m], bl0, bl1);
        }
      }
    }
  }
  // fixed-order reduction of the 8 warps' 64 x 32 accumulators through smem
  __syncthreads();
  float *red = reinterpret_cast<float *>(sm);  // [8 warps][64][32]
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int co = m * 16 + gq + ((r >> 1) << 3), tap = n * 8 + 2 * tq + (r & 1);
        red[(warp * 64 + co) * 32 + tap] = acc[m][n][r];
      }
  __syncthreads();
  for (int i = t; i < 64 * 27; i += 256) {
    const int co = i / 27, tap = i % 27;
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += red[(w * 64 + co) * 32 + tap];
    part[(int64_t)blockIdx.x * 64 * 27 + co * 27 + tap] = sum;
  }
}

template <typename T, int CO>
int stem_fprop_launch(const ConvGeom &g, const float *x, const float *w, void *y, float *part, cudaStream_t st) {
  const int64_t total = g.out_vox();
  if (std::is_same<T, bf16>::value && CO == 64 && !getenv("RN_STEM_FPROP_SIMT") && total + 64 < (1LL << 31)) {
    // tensor-core path; the grid is the statistics-partial count (<= 4 per SM)
    static int per_sm = 0;
    if (!per_sm) {
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stem_fprop_mma_k, SF_WARPS * 32, 0));
      per_sm = std::max(1, std::min(per_sm, 4));
    }
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 63) / 64, per_sm * 148));
    launch_k(stem_fprop_mma_k, blocks, SF_WARPS * 32, 0, st, g, x, w, (bf16 *)y, part);
    return part ? (int)blocks : 0;
  }
  // with fused statistics the grid is the partial count: 4 blocks per SM
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 127) / 128, part ? 4 * 148 : 148 * 16);
  launch_k(stem_fprop_k<T, CO>, blocks, 128, 0, st, g, x, w, (T *)y, part);
  return part ? (int)blocks : 0;
}

int stem_wgrad_blocks(const ConvGeom &g) {
  const int64_t total = g.out_vox();
  return (int)std::max<int64_t>(1, std::min<int64_t>(4 * 148, (total + 255) / 256));
}

template <typename T, int CO>
void stem_wgrad_launch(const ConvGeom &g, const float *x, const void *dh, float *dw, float *ws, cudaStream_t st,
                       const void *hx = nullptr, const float *coef = nullptr) {
  if (std::is_same<T, bf16>::value && CO == 64 && !getenv("RN_STEM_SIMT") && g.out_vox() < (1LL << 31)) {
    // tensor-core path (bf16 dh): 3 blocks per SM, partials reduced by split_reduce_add
    static uint64_t attr_devs = 0;  // kernel attributes are per device
    if (!once_on_device(attr_devs)) {
      CUDA_CHECK(cudaFuncSetAttribute(stem_wgrad_mma_k, cudaFuncAttributeMaxDynamicSharedMemorySize, SW_SMEM));
          }
    const int nb = std::min(stem_wgrad_blocks(g), 2 * 148);
    launch_k(stem_wgrad_mma_k, nb, 256, SW_SMEM, st, g, x, (const bf16 *)dh, ws, (const bf16 *)hx, coef);
    LAUNCH_CHECK();
    split_reduce_add(ws, nb, CO * 27, dw, st);
    return;
  }
  if (coef) throw Error(RN_ERR_ARG, "stem_wgrad: the fused BN apply needs the bf16 64-channel tensor-core path");
  // (stem_wgrad_warp_k measured 466 us vs 331 us for the smem-staged kernel on
  // the r18 stem: latency-bound with 16 warps/SM; kept for reference)
  const int nb = stem_wgrad_blocks(g);
  const int64_t vpb = (g.out_vox() + nb - 1) / nb;
  launch_k(stem_wgrad_k<T, CO>, nb, 256, 0, st, g, x, (const T *)dh, ws, vpb);
  LAUNCH_CHECK();
  split_reduce_add(ws, nb, CO * 27, dw, st);
}

}  // namespace

bool stem_fast_supported(const ConvGeom &g) {
  return g.Ci == 1 && g.k == 3 && (g.Co == 8 || g.Co == 16 || g.Co == 32 || g.Co == 64);
}

size_t stem_wgrad_ws_floats(const ConvGeom &g) { return (size_t)stem_wgrad_blocks(g) * g.Co * 27; }

int stem_fprop_fast(DType dt, const ConvGeom &g, const float *x, const float *w, void *y, cudaStream_t st,
                    float *part) {
  int P = 0;
#define STEM_F(CO)                                                              \
  if (g.Co == CO) {                                                             \
    if (dt == DT_F32) P = stem_fprop_launch<float, CO>(g, x, w, y, part, st);   \
    else P = stem_fprop_launch<bf16, CO>(g, x, w, y, part, st);                 \
  }
  STEM_F(8) STEM_F(16) STEM_F(32) STEM_F(64)
#undef STEM_F
  LAUNCH_CHECK();
  return P;
}


void stem_wgrad_fast(DType dt, const ConvGeom &g, const float *x, const void *dh, float *dw, float *ws,
                     cudaStream_t st) {
#define STEM_W(CO)                                                          \
  if (g.Co == CO) {                                                         \
    if (dt == DT_F32) stem_wgrad_launch<float, CO>(g, x, dh, dw, ws, st);   \
    else stem_wgrad_launch<bf16, CO>(g, x, dh, dw, ws, st);                 \
  }
  STEM_W(8) STEM_W(16) STEM_W(32) STEM_W(64)
#undef STEM_W
  LAUNCH_CHECK();
}

}  // namespace rn
