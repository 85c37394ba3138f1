// bnstats.cuh — BatchNorm statistics accumulated in a convolution epilogue
// (PAPER.md:366 Conv block = conv + BN + ReLU; readings X8/X9: train-mode BN
// over the layer output of the micro-batch).  Instead of a separate pass that
// re-reads the conv output, every CTA of the conv reduces the values it stores:
//   forward  (mode 1): S1 = sum y,   S2 = sum y^2           (y as stored, bf16)
//   backward (mode 2): S1 = sum dy', S2 = sum dy' * (h - mean),  dy' = y * (mask > 0)
//   (centred by the consumer BN's batch mean: no cancellation in the apply)
// and writes one fp32 partial [2][C] per CTA; the BN apply kernel reduces the
// partials in CTA order (deterministic) in fp64 and finalizes.
#pragma once
#include <cuda_bf16.h>

#include "util.cuh"

namespace rn {

struct EpiStats {
  float *part = nullptr;       // [gridDim.x][2][C]
  const bf16 *mask = nullptr;  // mode 2
  const bf16 *h = nullptr;     // modes 2, 3
  const float *mean = nullptr; // modes 2, 3: the consumer BN's batch mean per channel
  // mode 3: the consumer's ReLU mask recomputed from h, (h*mscale + mshift > 0) — the
  // forward apply's own fp32 pre-activation (scale/shift as it stored them), so one
  // tensor stream less than mode 2 (valid for a BN + ReLU without residual)
  const float *mscale = nullptr, *mshift = nullptr;
  int mode = 0;                // 0 off, 1 forward, 2 backward (mask tensor), 3 backward (recomputed mask)
};

// x[j] (channel j of this lane's row) summed over the 32 lanes; lane l returns
// the sum for channel l (butterfly transpose-reduce: 31 shuffles)
__device__ __forceinline__ float transpose_sum32(float (&x)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < off; ++j) {
      const float send = upper ? x[j] : x[j + off];
      const float keep = upper ? x[j + off] : x[j];
      x[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return x[0];
}

// mode-2 operands of one row x 32 channels (mask and h, bf16), loaded one chunk
// ahead of their use so the epilogue does not wait a memory round trip per chunk
struct StatsPf {
  uint4 m[4], h[4];
};
__device__ __forceinline__ void epi_stats_prefetch(const EpiStats &st, bool valid, int64_t eo, StatsPf &pf) {
  if (st.mode < 2 || !valid) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (st.mode == 2) pf.m[i] = __ldg(reinterpret_cast<const uint4 *>(st.mask + eo) + i);
    pf.h[i] = __ldg(reinterpret_cast<const uint4 *>(st.h + eo) + i);
  }
}

__device__ __forceinline__ void unpack_bf16x8(const uint4 &u, float *v) {
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

// Epilogue contribution of one row x 32 channels: f = final fp32 values, pf =
// the row's prefetched mask / h (mode 2), red = this warp's smem accumulators
// [2][BN] at channel c0.
__device__ __forceinline__ void epi_stats_add(const EpiStats &st, const float *f, bool valid, const StatsPf &pf,
                                              int c0, int lane, float *red0, float *red1) {
  float x1[32], x2[32];
  if (st.mode == 1) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float r = valid ? __bfloat162float(__float2bfloat16_rn(f[j])) : 0.f;
      x1[j] = r;
      x2[j] = r * r;
    }
  } else if (valid) {
    float m[32], h[32];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      unpack_bf16x8(pf.h[i], h + 8 * i);
      if (st.mode == 2) unpack_bf16x8(pf.m[i], m + 8 * i);
    }
    if (st.mode == 3)
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(st.mscale + c0 + j));
        const float4 b = __ldg(reinterpret_cast<const float4 *>(st.mshift + c0 + j));
        m[j] = fmaf(h[j], a.x, b.x);
        m[j + 1] = fmaf(h[j + 1], a.y, b.y);
        m[j + 2] = fmaf(h[j + 2], a.z, b.z);
        m[j + 3] = fmaf(h[j + 3], a.w, b.w);
      }
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 mu = __ldg(reinterpret_cast<const float4 *>(st.mean + c0 + j));
      h[j] -= mu.x;
      h[j + 1] -= mu.y;
      h[j + 2] -= mu.z;
      h[j + 3] -= mu.w;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float r = __bfloat162float(__float2bfloat16_rn(f[j]));
      const float d = m[j] > 0.f ? r : 0.f;
      x1[j] = d;
      x2[j] = d * h[j];
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) x1[j] = x2[j] = 0.f;
  }
  const float s1 = transpose_sum32(x1, lane);
  const float s2 = transpose_sum32(x2, lane);
  red0[lane] += s1;
  red1[lane] += s2;
}

// epilogue warps (128 threads, named barrier 1): sum the 4 warps' accumulators
// in fixed order and write this CTA's partial
__device__ __forceinline__ void epi_stats_flush(const EpiStats &st, const float *red, int BN, int C, int et) {
  asm volatile("bar.sync 1, 128;" ::: "memory");
  for (int c = et; c < BN; c += 128) {
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      a += red[(w * 2 + 0) * BN + c];
      b += red[(w * 2 + 1) * BN + c];
    }
    st.part[(int64_t)blockIdx.x * 2 * C + c] = a;
    st.part[(int64_t)blockIdx.x * 2 * C + C + c] = b;
  }
}

}  // namespace rn
