// k_conv_simt.cu — SIMT implicit-GEMM 3D convolution (fprop, dgrad, wgrad) with
// fp32 FFMA accumulation (no TF32: the RN_F32 parity path, reading X19), plus the
// Cin = 1 stem convolution.  The convolution is the Conv block's 3x3x3 layer of
// PAPER.md:364/366 (complexity O(Co*Ci*T*H*W*Kt*Kh*Kw)); the backward kernels
// are its chain-rule gradients.  In RN_BF16 these kernels serve shapes
// the tcgen05 kernels do not take (e.g. Cin = 8).
#include <cuda_bf16.h>

#include <algorithm>

#include "error.h"
#include "launch.h"
#include "kernels.h"
#include "util.cuh"

namespace rn {

namespace {

constexpr int BM = 64, BN = 64, BK = 8, NT = 256;

// MODE 0: fprop  (GEMM rows = output voxels, cols = Co, K = taps*Ci)
// MODE 1: dgrad  (GEMM rows = input voxels,  cols = Ci, K = taps*Co)
template <typename T, int MODE>
__global__ void __launch_bounds__(NT) conv_simt_kernel(ConvGeom g, const T *__restrict__ src,
                                                       const T *__restrict__ w, const float *__restrict__ bias,
                                                       T *__restrict__ out, int accumulate,
                                                       const T *__restrict__ res, const T *__restrict__ res_mask) {
  pdl_begin();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  // GEMM extents
  const int Rd = MODE == 0 ? g.Do : g.Di, Rh = MODE == 0 ? g.Ho : g.Hi, Rw = MODE == 0 ? g.Wo : g.Wi;
  const int Sd = MODE == 0 ? g.Di : g.Do, Sh = MODE == 0 ? g.Hi : g.Ho, Sw = MODE == 0 ? g.Wi : g.Wo;
  const int Kc = MODE == 0 ? g.Ci : g.Co;  // gemm-K channels (of src)
  const int Nc = MODE == 0 ? g.Co : g.Ci;  // gemm-N channels (of out)
  const int64_t M = (int64_t)g.N * Rd * Rh * Rw;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  // each thread loads A row ar, k pair ak
  const int ar = t / 4, ak = (t % 4) * 2;
  const int64_t am = m0 + ar;
  int an = 0, ad = 0, ah = 0, aw = 0;
  const bool arow_ok = am < M;
  if (arow_ok) {
    int64_t r = am;
    aw = (int)(r % Rw); r /= Rw;
    ah = (int)(r % Rh); r /= Rh;
    ad = (int)(r % Rd); r /= Rd;
    an = (int)r;
  }
  // B: col bc, k pair bk
  const int bc = t / 4, bk = (t % 4) * 2;
  const int bcol = n0 + bc;
  const int taps = g.k * g.k * g.k;

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int tap = 0; tap < taps; ++tap) {
    const int kd = tap / (g.k * g.k), kh = (tap / g.k) % g.k, kw = tap % g.k;
    // source voxel for this row and tap
    bool valid = arow_ok;
    int sd, sh, sw;
    if (MODE == 0) {
      sd = ad * g.s + kd - g.p; sh = ah * g.s + kh - g.p; sw = aw * g.s + kw - g.p;
    } else {
      int td = ad + g.p - kd, th = ah + g.p - kh, tw = aw + g.p - kw;
      valid = valid && td >= 0 && th >= 0 && tw >= 0 && (td % g.s) == 0 && (th % g.s) == 0 && (tw % g.s) == 0;
      sd = td / g.s; sh = th / g.s; sw = tw / g.s;
    }
    valid = valid && sd >= 0 && sd < Sd && sh >= 0 && sh < Sh && sw >= 0 && sw < Sw;
    const T *srow = valid ? src + ((((int64_t)an * Sd + sd) * Sh + sh) * Sw + sw) * Kc : nullptr;
    for (int c0 = 0; c0 < Kc; c0 += BK) {
      // A tile
      float a0 = 0.f, a1 = 0.f;
      if (valid) {
        a0 = to_f(srow[c0 + ak]);
        a1 = to_f(srow[c0 + ak + 1]);
      }
      // B tile: element (k, col) of the GEMM
      float b0 = 0.f, b1 = 0.f;
      if (bcol < Nc) {
        if (MODE == 0) {  // w[co=bcol][tap][ci=c0+k]
          const T *wr = w + ((int64_t)bcol * taps + tap) * g.Ci + c0 + bk;
          b0 = to_f(wr[0]);
          b1 = to_f(wr[1]);
        } else {  // w[co=c0+k][tap][ci=bcol]
          const T *wr = w + ((int64_t)(c0 + bk) * taps + tap) * g.Ci + bcol;
          b0 = to_f(wr[0]);
          b1 = to_f(wr[(int64_t)taps * g.Ci]);
        }
      }
      __syncthreads();
      As[ak][ar] = a0;
      As[ak + 1][ar] = a1;
      Bs[bk][bc] = b0;
      Bs[bk + 1][bc] = b1;
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float4 av = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
        float4 bv = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
        float a[4] = {av.x, av.y, av.z, av.w}, b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
    }
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + tx * 4 + j;
      if (col >= Nc) continue;
      float v = acc[i][j];
      if (bias) v += bias[col];
      const int64_t o = m * Nc + col;
      if (accumulate) v += to_f(out[o]);
      if (res) {
        float r = to_f(res[o]);
        if (res_mask && !(to_f(res_mask[o]) > 0.f)) r = 0.f;
        v += r;
      }
      out[o] = from_f<T>(v);
    }
  }
}

// wgrad: GEMM rows = Co, cols = taps*Ci, K = output voxels (split-K over blockIdx.z)
template <typename TX, typename TY>
__global__ void __launch_bounds__(NT) wgrad_simt_kernel(ConvGeom g, const TX *__restrict__ x,
                                                        const TY *__restrict__ dy, float *__restrict__ part,
                                                        int64_t chunks_per_split) {
  pdl_begin();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int t = threadIdx.x, tx = t % 16, ty = t / 16;
  const int taps = g.k * g.k * g.k;
  const int NC = taps * g.Ci;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int64_t Kv = g.out_vox();
  const int64_t nchunks = (Kv + BK - 1) / BK;
  const int64_t c_begin = (int64_t)blockIdx.z * chunks_per_split;
  const int64_t c_end = min(nchunks, c_begin + chunks_per_split);
  // A load: voxel av = t/32, co pair (t%32)*2 ; B load: voxel bv = t/32, col pair (t%32)*2
  const int lv = t / 32, lc = (t % 32) * 2;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // per-thread B column decode (fixed for the block)
  int bt[2], bci[2], bkd[2], bkh[2], bkw[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    int col = n0 + lc + e;
    bt[e] = col < NC ? col / g.Ci : -1;
    bci[e] = col < NC ? col % g.Ci : 0;
    int tp = bt[e] < 0 ? 0 : bt[e];
    bkd[e] = tp / (g.k * g.k); bkh[e] = (tp / g.k) % g.k; bkw[e] = tp % g.k;
  }
  for (int64_t ch = c_begin; ch < c_end; ++ch) {
    const int64_t v = ch * BK + lv;
    float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
    if (v < Kv) {
      if (m0 + lc < g.Co) a0 = to_f(dy[v * g.Co + m0 + lc]);
      if (m0 + lc + 1 < g.Co) a1 = to_f(dy[v * g.Co + m0 + lc + 1]);
      int64_t r = v;
      int ow = (int)(r % g.Wo); r /= g.Wo;
      int oh = (int)(r % g.Ho); r /= g.Ho;
      int od = (int)(r % g.Do); r /= g.Do;
      int n = (int)r;
      float bb[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        bb[e] = 0.f;
        if (bt[e] >= 0) {
          int id = od * g.s + bkd[e] - g.p, ih = oh * g.s + bkh[e] - g.p, iw = ow * g.s + bkw[e] - g.p;
          if (id >= 0 && id < g.Di && ih >= 0 && ih < g.Hi && iw >= 0 && iw < g.Wi)
            bb[e] = to_f(x[((((int64_t)n * g.Di + id) * g.Hi + ih) * g.Wi + iw) * g.Ci + bci[e]]);
        }
      }
      b0 = bb[0];
      b1 = bb[1];
    }
    __syncthreads();
    As[lv][lc] = a0;
    As[lv][lc + 1] = a1;
    Bs[lv][lc] = b0;
    Bs[lv][lc + 1] = b1;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float4 av = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
      float4 bv = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
      float a[4] = {av.x, av.y, av.z, av.w}, b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
  }
  float *P = part + (int64_t)blockIdx.z * g.Co * NC;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int row = m0 + ty * 4 + i;
    if (row >= g.Co) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int col = n0 + tx * 4 + j;
      if (col < NC) P[(int64_t)row * NC + col] = acc[i][j];
    }
  }
}

void wgrad_split(const ConvGeom &g, int &splits, int64_t &chunks_per_split) {
  const int taps = g.k * g.k * g.k;
  const int64_t tiles = (int64_t)((g.Co + BM - 1) / BM) * ((taps * g.Ci + BN - 1) / BN);
  const int64_t nchunks = (g.out_vox() + BK - 1) / BK;
  int64_t want = (2 * 148 + tiles - 1) / tiles;
  if (want < 1) want = 1;
  if (want > 256) want = 256;
  if (want > nchunks) want = nchunks;
  chunks_per_split = (nchunks + want - 1) / want;
  splits = (int)((nchunks + chunks_per_split - 1) / chunks_per_split);
}

// stem: thread per (output voxel, 8 channels)
template <typename T>
__global__ void stem_kernel(ConvGeom g, const float *__restrict__ x, const float *__restrict__ w,
                            T *__restrict__ y) {
  pdl_begin();
  extern __shared__ float ws[];  // [27][Co]
  for (int i = threadIdx.x; i < 27 * g.Co; i += blockDim.x) {
    int co = i % g.Co, tap = i / g.Co;
    ws[i] = w[co * 27 + tap];
  }
  __syncthreads();
  const int groups = g.Co / 8;
  const int64_t total = g.out_vox() * groups;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int grp = (int)(idx % groups);
    int64_t r = idx / groups;
    const int64_t vo = r;
    int ow = (int)(r % g.Wo); r /= g.Wo;
    int oh = (int)(r % g.Ho); r /= g.Ho;
    int od = (int)(r % g.Do); r /= g.Do;
    int n = (int)r;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int tap = 0; tap < 27; ++tap) {
      int kd = tap / 9, kh = (tap / 3) % 3, kw = tap % 3;
      int id = od * g.s + kd - g.p, ih = oh * g.s + kh - g.p, iw = ow * g.s + kw - g.p;
      if (id < 0 || id >= g.Di || ih < 0 || ih >= g.Hi || iw < 0 || iw >= g.Wi) continue;
      float xv = __ldg(&x[(((int64_t)n * g.Di + id) * g.Hi + ih) * g.Wi + iw]);
      const float *wr = ws + tap * g.Co + grp * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = fmaf(xv, wr[j], acc[j]);
    }
    store8(y + vo * g.Co + grp * 8, acc);
  }
}

}  // namespace

void conv_fprop_simt(DType dt, const ConvGeom &g, const void *x, const void *w, const float *bias, void *y,
                     cudaStream_t st) {
  dim3 grid((unsigned)((g.out_vox() + BM - 1) / BM), (g.Co + BN - 1) / BN);
  if (dt == DT_F32)
    launch_k(conv_simt_kernel<float, 0>, grid, NT, 0, st, g, (const float *)x, (const float *)w, bias, (float *)y, 0,
                                                     nullptr, nullptr);
  else
    launch_k(conv_simt_kernel<bf16, 0>, grid, NT, 0, st, g, (const bf16 *)x, (const bf16 *)w, bias, (bf16 *)y, 0,
                                                    nullptr, nullptr);
  LAUNCH_CHECK();
}

void conv_dgrad_simt(DType dt, const ConvGeom &g, const void *dy, const void *w, void *dx, bool accumulate,
                     const void *res, const void *res_mask, cudaStream_t st) {
  dim3 grid((unsigned)((g.in_vox() + BM - 1) / BM), (g.Ci + BN - 1) / BN);
  if (dt == DT_F32)
    launch_k(conv_simt_kernel<float, 1>, grid, NT, 0, st, g, (const float *)dy, (const float *)w, nullptr, (float *)dx,
                                                     accumulate, (const float *)res, (const float *)res_mask);
  else
    launch_k(conv_simt_kernel<bf16, 1>, grid, NT, 0, st, g, (const bf16 *)dy, (const bf16 *)w, nullptr, (bf16 *)dx,
                                                    accumulate, (const bf16 *)res, (const bf16 *)res_mask);
  LAUNCH_CHECK();
}

size_t conv_wgrad_ws_floats(const ConvGeom &g) {
  int splits;
  int64_t cps;
  wgrad_split(g, splits, cps);
  return (size_t)splits * g.Co * g.taps() * g.Ci;
}

void conv_wgrad_simt(DType dt, bool x_is_f32, const ConvGeom &g, const void *x, const void *dy, float *dw,
                     float *ws, cudaStream_t st) {
  int splits;
  int64_t cps;
  wgrad_split(g, splits, cps);
  dim3 grid((g.Co + BM - 1) / BM, (g.taps() * g.Ci + BN - 1) / BN, splits);
  if (dt == DT_F32)
    launch_k(wgrad_simt_kernel<float, float>, grid, NT, 0, st, g, (const float *)x, (const float *)dy, ws, cps);
  else if (x_is_f32)
    launch_k(wgrad_simt_kernel<float, bf16>, grid, NT, 0, st, g, (const float *)x, (const bf16 *)dy, ws, cps);
  else
    launch_k(wgrad_simt_kernel<bf16, bf16>, grid, NT, 0, st, g, (const bf16 *)x, (const bf16 *)dy, ws, cps);
  LAUNCH_CHECK();
  int64_t n = (int64_t)g.Co * g.taps() * g.Ci;
  split_reduce_add(ws, splits, n, dw, st);
}

void stem_conv_fprop(DType dt, const ConvGeom &g, const float *x, const float *w, void *y, cudaStream_t st) {
  int64_t total = g.out_vox() * (g.Co / 8);
  unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  size_t sm = 27 * g.Co * sizeof(float);
  if (dt == DT_F32)
    launch_k(stem_kernel<float>, blocks, 256, sm, st, g, x, w, (float *)y);
  else
    launch_k(stem_kernel<bf16>, blocks, 256, sm, st, g, x, w, (bf16 *)y);
  LAUNCH_CHECK();
}

}  // namespace rn
