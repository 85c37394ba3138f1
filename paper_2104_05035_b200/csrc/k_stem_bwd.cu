// k_stem_bwd.cu — backward of the pooled stem Conv block (the
// "Conv block" = 3x3x3 conv + BN + ReLU; reading X4: max-pool k3 s2 p1 after it)
// at the POOLED resolution, bf16 path (reading X23c in DESIGN.md).
//
// Forward: h = conv(x, W) (k3 s2 p1, Ci = 1), z = s*h + b (BN, s = gamma*invstd),
// a = ReLU(z), y = maxpool(a) with argmax am (window tap 0..26, first maximum).
// Backward, with dz = (pool adjoint of dy) * (z > 0), nonzero only at the argmax
// voxel of a pooled output whose y > 0:
//   dbeta = S1 = sum dz,   dgamma = S2 = sum dz * xhat = invstd * sum dz (h - mean)
//   dh = A dz + B h + Cc,  A = gamma*invstd, B = -A*invstd*m2, Cc = -A*m1 + A*invstd*mean*m2
//        (m1 = S1/V, m2 = S2/V: the BatchNorm backward, Eq. of bn_backward in oracle/net.py)
//   dW[c][t] = sum_v dh[v][c] X[v][t]           (X = im2col of x, 27 taps)
//            = A T[c][t] + B (W G)[c][t] + Cc g[t]
// with T[c][t] = sum over pooled outputs o of dz[o][c] X[argmax(o, c)][t] (sparse),
// G = sum_v X[v] X[v]^T (27 x 27) and g = sum_v X[v] over every conv voxel: the
// 119 MB conv-resolution tensors (h, the pool adjoint, dh) are never read or formed.
// Precision: T, S1, S2 from fp32 per-thread sums and fp64 across blocks; h at the
// argmax is recomputed in fp32 from x and W (the stored bf16 h is never read); G on mma.sync with fp32 operands split into bf16 pairs (three
// products, ~2^-16 relative) accumulated in fp32 per warp, fp64 across warps.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "error.h"
#include "kernels.h"
#include "launch.h"
#include "util.cuh"

namespace rn {

namespace {

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// (v0, v1) -> bf16x2 hi and lo parts, v = hi + lo + O(2^-17 |v|); v0 in the low half (first k)
__device__ __forceinline__ void split2(float v0, float v1, uint32_t &hi, uint32_t &lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(v0, v1);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
  memcpy(&hi, &h, 4);
  memcpy(&lo, &l, 4);
}

// 4-byte async copy global -> smem, zero-filled when !valid (src-size 0): the
// region loads of a tile are all in flight at once instead of one round trip
// per element (an LDG -> STS loop waits on every load)
__device__ __forceinline__ void cp_async4(float *sdst, const float *gsrc, bool valid) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gsrc), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Gram matrix of the im2col rows: per warp 16 conv voxels per step as the K
// dimension of m16n8k16 MMAs, M = N = 32 tap slots (27 taps, slot 27 = 1 so that
// G[t][27] = g[t], slots 28..31 = 0).  Thread (gq = lane/4, q = lane%4) holds
// X[v][t] for voxels {2q, 2q+1, 2q+8, 2q+9} and taps {gq, gq+8, gq+16, gq+24}:
// exactly the values of its A fragments (rows = taps) and B fragments (cols =
// taps).  Persistent blocks over slabs (sample n, conv plane od, GROWS conv rows):
// the slab's input region (3 planes x (2 GROWS + 1) rows x W, zero padded) is
// staged in smem with coalesced loads, so the MMA loop reads only smem.  Output:
// one fp32 partial [32][32] per block (warps summed in order).
constexpr int GRAM_THREADS = 256;
constexpr int GROWS = 14;
constexpr int GRAM_SMEM_FLOATS = 8192;  // >= 3 * (2 GROWS + 1) * Wi (Wi <= 94) and >= 8 warps x 1024

__global__ void __launch_bounds__(GRAM_THREADS) stem_gram_k(ConvGeom g, const float *__restrict__ x,
                                                            float *__restrict__ part) {
  __shared__ float xs[GRAM_SMEM_FLOATS];
  pdl_begin();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, q = lane & 3;
  const int SW = g.Wi + 2;             // staged row: input columns -1 .. Wi (zero borders)
  const int SR = 2 * GROWS + 1;        // staged rows per plane
  int tof[4];                          // smem offset of tap slot gq + 8j from the patch origin
  int tcode[4];                        // 0 zero, 1 tap, 2 ones column
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int t = gq + 8 * j;
    tcode[j] = t < 27 ? 1 : (t == 27 ? 2 : 0);
    const int tt = t < 27 ? t : 0;
    tof[j] = ((tt / 9) * SR + (tt / 3) % 3) * SW + tt % 3;
  }
  float acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.f;
  const int vs[4] = {2 * q, 2 * q + 1, 2 * q + 8, 2 * q + 9};
  const int nhs = (g.Ho + GROWS - 1) / GROWS;
  const int nslab = g.N * g.Do * nhs;
  const int chunks_per_row = (g.Wo + 15) / 16;
  for (int slab = blockIdx.x; slab < nslab; slab += gridDim.x) {
    const int hs = slab % nhs, od = (slab / nhs) % g.Do, n = slab / (nhs * g.Do);
    const int oh0 = hs * GROWS, rows = min(GROWS, g.Ho - oh0);
    const int id0 = 2 * od - 1, ih0 = 2 * oh0 - 1;
    __syncthreads();  // previous slab consumed
    const float *xn = x + (int64_t)n * g.Di * g.Hi * g.Wi;
    for (int e = threadIdx.x; e < 3 * SR * SW; e += GRAM_THREADS) {
      const int c = e % SW, r = (e / SW) % SR, pl = e / (SW * SR);
      const int id = id0 + pl, ih = ih0 + r, iw = c - 1;
      const bool ok = id >= 0 && id < g.Di && ih >= 0 && ih < g.Hi && iw >= 0 && iw < g.Wi;
      cp_async4(xs + e, ok ? xn + ((int64_t)id * g.Hi + ih) * g.Wi + iw : xn, ok);
    }
    cp_async_wait_all();
    __syncthreads();
    for (int ck = warp; ck < rows * chunks_per_row; ck += GRAM_THREADS / 32) {
      const int r = ck / chunks_per_row, ow0 = (ck % chunks_per_row) * 16;
      float X[4][4];  // [voxel slot][tap slot j]
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int ow = ow0 + vs[s];
        const bool vv = ow < g.Wo;
        const float *pb = xs + (2 * r) * SW + 2 * ow;  // patch origin: plane 0, row 2r, column 2ow (= input 2ow - 1)
#pragma unroll
        for (int j = 0; j < 4; ++j) X[s][j] = !vv ? 0.f : (tcode[j] == 1 ? pb[tof[j]] : (tcode[j] == 2 ? 1.f : 0.f));
      }
      uint32_t ah[2][4], al[2][4], bh[4][2], bl[4][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        split2(X[0][2 * i], X[1][2 * i], ah[i][0], al[i][0]);
        split2(X[0][2 * i + 1], X[1][2 * i + 1], ah[i][1], al[i][1]);
        split2(X[2][2 * i], X[3][2 * i], ah[i][2], al[i][2]);
        split2(X[2][2 * i + 1], X[3][2 * i + 1], ah[i][3], al[i][3]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        split2(X[0][j], X[1][j], bh[j][0], bl[j][0]);
        split2(X[2][j], X[3][j], bh[j][1], bl[j][1]);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          mma16816(acc[i][j], ah[i], bh[j][0], bh[j][1]);
          mma16816(acc[i][j], ah[i], bl[j][0], bl[j][1]);
          mma16816(acc[i][j], al[i], bh[j][0], bh[j][1]);
        }
    }
  }
  __syncthreads();
  float *red = xs;  // [8][32*32]
  // C fragment: acc[i][j][0..1] = G[16i + gq][8j + 2q + 0..1], acc[i][j][2..3] = G[16i + gq + 8][...]
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r0 = 16 * i + gq, c0 = 8 * j + 2 * q;
      red[warp * 1024 + r0 * 32 + c0] = acc[i][j][0];
      red[warp * 1024 + r0 * 32 + c0 + 1] = acc[i][j][1];
      red[warp * 1024 + (r0 + 8) * 32 + c0] = acc[i][j][2];
      red[warp * 1024 + (r0 + 8) * 32 + c0 + 1] = acc[i][j][3];
    }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * 32; e += GRAM_THREADS) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < GRAM_THREADS / 32; ++w) s += red[w * 1024 + e];
    part[(int64_t)blockIdx.x * 1024 + e] = s;
  }
}

// sparse part: per thread one channel c (C in {8, 16, 32, 64}), groups of threads
// over the pooled voxels of a tile (2 x 4 x 8 pooled voxels).  Per tile the input
// region (11 x 19 x 35 floats, zero padded) and the tile's pooled y / dy / argmax
// are staged in smem by cp.async, double buffered: tile i+1 streams in while tile
// i is computed.  Each lane walks its own list of active pooled outputs (y > 0,
// dy != 0), so the lanes of a warp stay converged on useful work.  Per block one
// partial [29][C]: S1, sum dz (h - mean), T[27].
constexpr int SP_THREADS = 512;
constexpr int TD = 2, TH = 4, TW = 8, PPT = TD * TH * TW;
constexpr int ID = 4 * TD + 3, IH = 4 * TH + 3, IW = 4 * TW + 3;
constexpr int REG_F = ID * IH * IW;                     // 7315 region floats
constexpr int POOL_W = PPT * 64 * 5 / 4;                // y, dy (bf16) + argmax (u8) of 64 channels, in words
constexpr int SP_BUF_W = (REG_F + POOL_W + 3) & ~3;     // one buffer, 4-byte words
constexpr int SP_SMEM = 2 * SP_BUF_W * 4;               // 98.6 KB
constexpr int KMAX = PPT / (SP_THREADS / 64);           // pooled voxels per thread (C = 64)

struct SparseArgs {
  ConvGeom g;  // the stem conv
  int D2, H2, W2;
  const float *x, *w, *mean;
  const bf16 *y, *dy;
  const uint8_t *am;
  float *part;
};

// stage tile `tile` into buffer b: region floats, then y [PPT][C] bf16, dy, am [PPT][C] u8
__device__ __forceinline__ void sp_stage(const SparseArgs &a, int tile, float *b) {
  const ConvGeom &g = a.g;
  const int C = g.Co;
  const int td = (a.D2 + TD - 1) / TD, th = (a.H2 + TH - 1) / TH, tw = (a.W2 + TW - 1) / TW;
  int r = tile;
  const int bw = r % tw; r /= tw;
  const int bh = r % th; r /= th;
  const int bd = r % td;
  const int n = r / td;
  const int od0 = bd * TD, oh0 = bh * TH, ow0 = bw * TW;
  const int id0 = 4 * od0 - 3, ih0 = 4 * oh0 - 3, iw0 = 4 * ow0 - 3;
  const float *xn = a.x + (int64_t)n * g.Di * g.Hi * g.Wi;
  for (int e = threadIdx.x; e < REG_F; e += SP_THREADS) {
    const int lw = e % IW, lh = (e / IW) % IH, ld = e / (IW * IH);
    const int iw = iw0 + lw, ih = ih0 + lh, id = id0 + ld;
    const bool ok = id >= 0 && id < g.Di && ih >= 0 && ih < g.Hi && iw >= 0 && iw < g.Wi;
    cp_async4(b + e, ok ? xn + ((int64_t)id * g.Hi + ih) * g.Wi + iw : xn, ok);
  }
  // pooled rows: C/2 words of y, C/2 of dy, C/4 of am per pooled voxel
  float *py = b + REG_F, *pdy = py + PPT * C / 2, *pam = pdy + PPT * C / 2;
  const int wpr = C / 2, apr = C / 4;
  for (int e = threadIdx.x; e < PPT * (2 * wpr + apr); e += SP_THREADS) {
    int pi, wd, kind;
    if (e < PPT * wpr) { pi = e / wpr; wd = e % wpr; kind = 0; }
    else if (e < 2 * PPT * wpr) { pi = (e - PPT * wpr) / wpr; wd = (e - PPT * wpr) % wpr; kind = 1; }
    else { pi = (e - 2 * PPT * wpr) / apr; wd = (e - 2 * PPT * wpr) % apr; kind = 2; }
    const int pw = pi % TW, ph = (pi / TW) % TH, pd = pi / (TW * TH);
    const int od = od0 + pd, oh = oh0 + ph, ow = ow0 + pw;
    const bool ok = od < a.D2 && oh < a.H2 && ow < a.W2;
    const int64_t o = ok ? (((int64_t)n * a.D2 + od) * a.H2 + oh) * a.W2 + ow : 0;
    if (kind == 0) cp_async4(py + pi * wpr + wd, reinterpret_cast<const float *>(a.y + o * C) + wd, ok);
    else if (kind == 1) cp_async4(pdy + pi * wpr + wd, reinterpret_cast<const float *>(a.dy + o * C) + wd, ok);
    else cp_async4(pam + pi * apr + wd, reinterpret_cast<const float *>(a.am + o * C) + wd, ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(SP_THREADS, 1) stem_bwd_sparse_k(const SparseArgs a) {
  extern __shared__ __align__(16) float sbuf[];
  pdl_begin();
  const ConvGeom &g = a.g;
  const int C = g.Co;
  const int c = threadIdx.x % C, grp = threadIdx.x / C, ngrp = SP_THREADS / C;
  float w[27];
#pragma unroll
  for (int t = 0; t < 27; ++t) w[t] = a.w[c * 27 + t];
  const float mu = a.mean[c];
  float s1 = 0.f, sc = 0.f, T[27];
#pragma unroll
  for (int t = 0; t < 27; ++t) T[t] = 0.f;
  const int td = (a.D2 + TD - 1) / TD, th = (a.H2 + TH - 1) / TH, tw = (a.W2 + TW - 1) / TW;
  const int ntiles = g.N * td * th * tw;
  int it = 0;
  if ((int)blockIdx.x < ntiles) sp_stage(a, blockIdx.x, sbuf);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int nxt = tile + gridDim.x;
    if (nxt < ntiles) {
      sp_stage(a, nxt, sbuf + ((it + 1) & 1) * SP_BUF_W);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float *xs = sbuf + (it & 1) * SP_BUF_W;
    const uint16_t *py = reinterpret_cast<const uint16_t *>(xs + REG_F);
    const uint16_t *pdy = py + PPT * C;
    const uint8_t *pam = reinterpret_cast<const uint8_t *>(pdy + PPT * C);
    uint32_t mask = 0u;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      const int pi = grp + k * ngrp;
      if (pi < PPT) {
        const uint32_t yb = py[pi * C + c], db = pdy[pi * C + c];
        // ReLU closed (y = 0, also the all-zero window) or dy = 0: no contribution
        if ((yb & 0x8000u) == 0u && (yb & 0x7fffu) != 0u && (db & 0x7fffu) != 0u) mask |= 1u << k;
      }
    }
    while (mask) {
      const int k = __ffs(mask) - 1;
      mask &= mask - 1;
      const int pi = grp + k * ngrp;
      const float dz = __bfloat162float(__ushort_as_bfloat16(pdy[pi * C + c]));
      const int am = pam[pi * C + c];
      const int pw = pi % TW, ph = (pi / TW) % TH, pd = pi / (TW * TH);
      const int kd = am / 9, kh = (am / 3) % 3, kw = am % 3;
      const float *p = xs + ((4 * pd + 2 * kd) * IH + (4 * ph + 2 * kh)) * IW + (4 * pw + 2 * kw);
      float h0 = 0.f, h1 = 0.f, h2 = 0.f;  // three chains: kd = 0, 1, 2
#pragma unroll
      for (int t = 0; t < 27; ++t) {
        const float X = p[((t / 9) * IH + (t / 3) % 3) * IW + t % 3];
        if (t < 9) h0 = fmaf(w[t], X, h0);
        else if (t < 18) h1 = fmaf(w[t], X, h1);
        else h2 = fmaf(w[t], X, h2);
        T[t] = fmaf(dz, X, T[t]);
      }
      const float h = (h0 + h1) + h2;
      s1 += dz;
      sc = fmaf(dz, h - mu, sc);  // fp32 h (reading X23c), not the stored bf16 copy
    }
    __syncthreads();  // buffer (it & 1) is restaged two tiles later
  }
  // fixed-order sum over the groups, in two halves of the smem buffer: groups
  // [0, ngrp/2) then [ngrp/2, ngrp)
  float *red = sbuf;  // [ngrp/2][29][C]
  const int half = ngrp / 2;
  float tot[29 * 64 / SP_THREADS + 1];
#pragma unroll
  for (int i = 0; i < 29 * 64 / SP_THREADS + 1; ++i) tot[i] = 0.f;
  for (int ph = 0; ph < 2; ++ph) {
    __syncthreads();
    if (grp / half == ph) {
      const int gq = grp - ph * half;
      red[(gq * 29 + 0) * C + c] = s1;
      red[(gq * 29 + 1) * C + c] = sc;
#pragma unroll
      for (int t = 0; t < 27; ++t) red[(gq * 29 + 2 + t) * C + c] = T[t];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 29 * 64 / SP_THREADS + 1; ++i) {
      const int e = threadIdx.x + i * SP_THREADS;
      if (e < 29 * C)
        for (int q = 0; q < half; ++q) tot[i] += red[q * 29 * C + e];
    }
  }
#pragma unroll
  for (int i = 0; i < 29 * 64 / SP_THREADS + 1; ++i) {
    const int e = threadIdx.x + i * SP_THREADS;
    if (e < 29 * C) a.part[(int64_t)blockIdx.x * 29 * C + e] = tot[i];
  }
}

// fp64 Gram matrix from the per-block partials (fixed order): Gd[32][32]; block =
// 32 entries, warp w sums partials w, w+8, ... and the 8 warp sums are added in order
__global__ void __launch_bounds__(256) stem_gram_fin_k(const float *__restrict__ part, int P, double *__restrict__ Gd) {
  __shared__ double red[8][32];
  pdl_begin();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double s = 0.0;
  for (int p = w; p < P; p += 8) s += (double)part[(int64_t)p * 1024 + e];
  red[w][lane] = s;
  __syncthreads();
  if (w == 0) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][lane];
    Gd[e] = t;
  }
}

// finalize, one block per channel c: fp64 sums of the sparse partials, the
// BN-backward coefficients, dgamma / dbeta and dW[c][t] = A T + B (W G) + Cc g
struct FinArgs {
  const double *G;     // [32][32], column 27 = g
  const float *spart;  // [Ps][29][C]
  int Ps, C;
  int64_t V;
  const float *w, *gamma, *mean, *invstd;
  float *dgamma, *dbeta, *dw;
};

__global__ void __launch_bounds__(256) stem_bwd_fin_k(const FinArgs a) {
  __shared__ double sred[8][29];
  __shared__ double sums[29];
  pdl_begin();
  const int c = blockIdx.x, tid = threadIdx.x;
  {
    const int k = tid & 31, sp = tid >> 5;
    double s = 0.0;
    if (k < 29)
      for (int p = sp; p < a.Ps; p += 8) s += (double)a.spart[((int64_t)p * 29 + k) * a.C + c];
    if (k < 29) sred[sp][k] = s;
  }
  __syncthreads();
  if (tid < 29) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += sred[q][tid];
    sums[tid] = t;
  }
  __syncthreads();
  const double is = a.invstd[c], mu = a.mean[c];
  const double S1 = sums[0], S2 = is * sums[1];
  const double m1 = S1 / (double)a.V, m2 = S2 / (double)a.V;
  const double A = (double)a.gamma[c] * is;
  const double B = -A * is * m2, Cc = -A * m1 + A * is * mu * m2;
  if (tid < 27) {
    double H = 0.0;
    for (int tp = 0; tp < 27; ++tp) H += (double)a.w[c * 27 + tp] * a.G[tp * 32 + tid];
    a.dw[c * 27 + tid] += (float)(A * sums[2 + tid] + B * H + Cc * a.G[tid * 32 + 27]);
  }
  if (tid == 0) {
    a.dgamma[c] += (float)S2;
    a.dbeta[c] += (float)S1;
  }
}

}  // namespace

constexpr int GRAM_BLOCKS = 2 * 148, SP_BLOCKS = 148;  // the sparse kernel: one 512-thread block per SM

size_t stem_gram_ws_floats() { return (size_t)GRAM_BLOCKS * 1024; }
size_t stem_bwd_sparse_ws_floats() { return (size_t)SP_BLOCKS * 29 * 64; }

bool stem_bwd_sparse_supported(const ConvGeom &g) {
  return g.Ci == 1 && g.k == 3 && g.s == 2 && g.p == 1 && (g.Co == 8 || g.Co == 16 || g.Co == 32 || g.Co == 64) &&
         3 * (2 * GROWS + 1) * (g.Wi + 2) <= GRAM_SMEM_FLOATS;
}

void stem_gram(const ConvGeom &g, const float *x, float *ws, double *Gd, cudaStream_t st) {
  if (!stem_bwd_sparse_supported(g)) throw Error(RN_ERR_ARG, "stem_gram: unsupported stem geometry");
  launch_k(stem_gram_k, GRAM_BLOCKS, GRAM_THREADS, 0, st, g, x, ws);
  LAUNCH_CHECK();
  launch_k(stem_gram_fin_k, 32, 256, 0, st, (const float *)ws, GRAM_BLOCKS, Gd);
  LAUNCH_CHECK();
}

void stem_bwd_sparse(const ConvGeom &g, int D2, int H2, int W2, const float *x, const float *w, const void *y,
                     const void *dy, const uint8_t *am, const float *gamma, const float *mean, const float *invstd,
                     const double *Gd, float *dgamma, float *dbeta, float *dw, float *ws, cudaStream_t st) {
  if (!stem_bwd_sparse_supported(g)) throw Error(RN_ERR_ARG, "stem_bwd_sparse: unsupported stem geometry");
  static uint64_t attr_devs = 0;  // kernel attributes are per device
  if (!once_on_device(attr_devs))
    CUDA_CHECK(cudaFuncSetAttribute(stem_bwd_sparse_k, cudaFuncAttributeMaxDynamicSharedMemorySize, SP_SMEM));
  SparseArgs sa{g, D2, H2, W2, x, w, mean, (const bf16 *)y, (const bf16 *)dy, am, ws};
  launch_k(stem_bwd_sparse_k, SP_BLOCKS, SP_THREADS, SP_SMEM, st, sa);
  LAUNCH_CHECK();
  FinArgs fa{Gd, ws, SP_BLOCKS, g.Co, (int64_t)g.N * g.Do * g.Ho * g.Wo, w, gamma, mean, invstd, dgamma, dbeta, dw};
  launch_k(stem_bwd_fin_k, g.Co, 256, 0, st, fa);
  LAUNCH_CHECK();
}

}  // namespace rn
