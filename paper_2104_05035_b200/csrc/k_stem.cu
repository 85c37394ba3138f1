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
  // output staging: the block's 128 voxels x CO channels, stored back with
  // consecutive threads on consecutive 16-B chunks (full L2 sectors)
  __shared__ __align__(16) T so[128 * CO];
  __syncthreads();
  const int64_t total = g.out_vox();
  for (int64_t vb = blockIdx.x * (int64_t)blockDim.x; vb < total; vb += (int64_t)gridDim.x * blockDim.x) {
    const int64_t vo = vb + threadIdx.x;
    const bool live = vo < total;
    int64_t r = live ? vo : total - 1;
    const int ow = (int)(r % g.Wo); r /= g.Wo;
    const int oh = (int)(r % g.Ho); r /= g.Ho;
    const int od = (int)(r % g.Do); r /= g.Do;
    const int n = (int)r;
    float xv[27];
#pragma unroll
    for (int tap = 0; tap < 27; ++tap) {
      const int id = od * g.s + tap / 9 - g.p, ih = oh * g.s + (tap / 3) % 3 - g.p, iw = ow * g.s + tap % 3 - g.p;
      const bool ok = id >= 0 && id < g.Di && ih >= 0 && ih < g.Hi && iw >= 0 && iw < g.Wi;
      xv[tap] = ok ? __ldg(&x[(((int64_t)n * g.Di + id) * g.Hi + ih) * g.Wi + iw]) : 0.f;
    }
#pragma unroll
    for (int c0 = 0; c0 < CO; c0 += 8) {
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
      for (int tap = 0; tap < 27; ++tap) {
        const float4 a = *reinterpret_cast<const float4 *>(&ws[tap * CO + c0]);
        const float4 b = *reinterpret_cast<const float4 *>(&ws[tap * CO + c0 + 4]);
        acc[0] = fmaf(xv[tap], a.x, acc[0]);
        acc[1] = fmaf(xv[tap], a.y, acc[1]);
        acc[2] = fmaf(xv[tap], a.z, acc[2]);
        acc[3] = fmaf(xv[tap], a.w, acc[3]);
        acc[4] = fmaf(xv[tap], b.x, acc[4]);
        acc[5] = fmaf(xv[tap], b.y, acc[5]);
        acc[6] = fmaf(xv[tap], b.z, acc[6]);
        acc[7] = fmaf(xv[tap], b.w, acc[7]);
      }
      store8(so + threadIdx.x * CO + c0, acc);
    }
    __syncthreads();
    constexpr int VE = 16 / sizeof(T);  // elements per 16-B chunk
    const int64_t nvox = min((int64_t)blockDim.x, total - vb);
    if (part) {  // statistics of the stored (rounded) values, channel t % CO
      const int c = threadIdx.x % CO;
      for (int v = threadIdx.x / CO; v < nvox; v += HG) {
        const float f = to_f(so[v * CO + c]);
        s1 += f;
        s2 = fmaf(f, f, s2);
      }
    }
    const int nchunk = (int)(nvox * CO / VE);
    for (int i = threadIdx.x; i < nchunk; i += blockDim.x)
      reinterpret_cast<uint4 *>(y + vb * CO)[i] = reinterpret_cast<const uint4 *>(so)[i];
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

__global__ void stem_reduce_k(const float *__restrict__ part, int nblk, int n, float *__restrict__ dw) {
  pdl_begin();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * n + i];
    dw[i] += s;
  }
}

template <typename T, int CO>
int stem_fprop_launch(const ConvGeom &g, const float *x, const float *w, void *y, float *part, cudaStream_t st) {
  const int64_t total = g.out_vox();
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
void stem_wgrad_launch(const ConvGeom &g, const float *x, const void *dh, float *dw, float *ws, cudaStream_t st) {
  // (stem_wgrad_warp_k measured 466 us vs 331 us for the smem-staged kernel on
  // the r18 stem: latency-bound with 16 warps/SM; kept for reference)
  const int nb = stem_wgrad_blocks(g);
  const int64_t vpb = (g.out_vox() + nb - 1) / nb;
  launch_k(stem_wgrad_k<T, CO>, nb, 256, 0, st, g, x, (const T *)dh, ws, vpb);
  LAUNCH_CHECK();
  launch_k(stem_reduce_k, (CO * 27 + 255) / 256, 256, 0, st, ws, nb, CO * 27, dw);
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
