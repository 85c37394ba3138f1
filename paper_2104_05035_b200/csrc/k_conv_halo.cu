// k_conv_halo.cu — stage-1 3x3x3 convolutions (64 -> 64 channels, stride 1) on
// tcgen05 with a HALOED A operand (the Conv block's 3x3x3
// convolution; these 64-channel layers carry about half of the step's FLOPs).
//
// The per-tap implicit GEMM (k_conv_tc.cu) re-reads a 16 KB activation tile
// for each of the 27 taps (432 KB of L2->SM traffic per 128 output voxels),
// which bounds it by L2 bandwidth, not by the tensor cores.  Here one TMA box of
// (8+2) x (16+2) x (2+2) voxels x 64 channels (92 KB) per CTA work item holds
// every tap-shifted operand of two 8x16 output slices: the A descriptor of tap
// (kd,kh,kw) for slice s starts at row ((s+kd)*18 + kh)*10 + kw of the box, its
// 16 row-groups (the 16 output rows h) are 10 rows apart (SBO = 1280 B) — the
// hardware takes the swizzle phase from the address, so any row start works.
// Traffic per 128 output voxels: 46 KB of activations + 108 KB of weights.
//
// Roles: warp 0 TMA (A box double-buffered, B = one tap's 64x64 weights per
// ring stage), warp 1 single-thread tcgen05.mma (M=128, N=64, K=16; two slice
// accumulators per item, two items in flight in TMEM), warps 2-5 epilogue
// (tcgen05.ld -> bias / accumulate / masked residual -> bf16 stores).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "bnstats.cuh"
#include "error.h"
#include "launch.h"
#include "kernels.h"
#include "tc_conv.h"
#include "tc_ptx.cuh"
#include "util.cuh"

namespace rn {

void make_act_map(CUtensorMap *m, const void *base, int C, int W, int H, int D, int N, int64_t sw, int64_t sh,
                  int64_t sd, int64_t sn, int bw, int bh, int bd, int bn);
void make_w_map(CUtensorMap *m, const void *base, int rows, int64_t ktot, int bn);

namespace {

constexpr int HW = 10, HH = 18, HD = 4;              // haloed box (w, h, d)
constexpr int A_BYTES = HW * HH * HD * 128;          // 92160
constexpr int B_BYTES = 64 * 128;                    // one tap: 64 out channels x 64 in channels
constexpr int BSTAGES = 4;
constexpr int RED_BYTES = 4 * 2 * 64 * 4;  // [4 warps][2][64] BN-statistics accumulators
constexpr int SMEM = 2 * A_BYTES + BSTAGES * B_BYTES + RED_BYTES + 256 + 1024;
constexpr int THREADS = 192;

struct __align__(64) HaloParams {
  CUtensorMap a_map;
  CUtensorMap b_map;
  int kcoord[27];
  int OW, OH, OD, ON;
  int tw, th, td;
  int64_t n_items;
  bf16 *y;
  int64_t s_n, s_d, s_h, s_w;
  const float *bias;
  int accumulate;
  const bf16 *res, *res_mask;
  EpiStats st;
};

__global__ void __launch_bounds__(THREADS, 1) conv_halo_kernel(const __grid_constant__ HaloParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = smem;                       // 2 x A_BYTES
  uint8_t *sB = smem + 2 * A_BYTES;         // BSTAGES x B_BYTES
  float *red = (float *)(sB + BSTAGES * B_BYTES);
  uint64_t *bar = (uint64_t *)(sB + BSTAGES * B_BYTES + RED_BYTES);
  uint64_t *a_full = bar, *a_empty = bar + 2, *b_full = bar + 4, *b_empty = b_full + BSTAGES;
  uint64_t *t_full = b_empty + BSTAGES, *t_empty = t_full + 2;
  uint32_t *tmem_slot = (uint32_t *)(t_empty + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&a_full[i], 1);
      tc::mbar_init(&a_empty[i], 1);
      tc::mbar_init(&t_full[i], 1);
      tc::mbar_init(&t_empty[i], 4);
    }
    for (int i = 0; i < BSTAGES; ++i) {
      tc::mbar_init(&b_full[i], 1);
      tc::mbar_init(&b_empty[i], 1);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&p.a_map);
    tc::tma_prefetch(&p.b_map);
  }
  if (warp == 1) tc::tmem_alloc<256>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_begin();  // prologue above overlaps the predecessor's tail

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t bph = 0;
      int local = 0;
      for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x, ++local) {
        int64_t r = it;
        const int tw = (int)(r % p.tw); r /= p.tw;
        const int th = (int)(r % p.th); r /= p.th;
        const int td = (int)(r % p.td); r /= p.td;
        const int n = (int)r;
        const int ab = local & 1;
        tc::mbar_wait(&a_empty[ab], ((local >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&a_full[ab], A_BYTES);
        tc::tma_load_5d(sA + ab * A_BYTES, &p.a_map, &a_full[ab], 0, tw * 8 - 1, th * 16 - 1, td * 2 - 1, n);
        for (int t = 0; t < 27; ++t) {
          tc::mbar_wait(&b_empty[s], bph ^ 1);
          tc::mbar_arrive_expect_tx(&b_full[s], B_BYTES);
          tc::tma_load_2d(sB + s * B_BYTES, &p.b_map, &b_full[s], p.kcoord[t], 0);
          if (++s == BSTAGES) { s = 0; bph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDESC = tc::idesc_bf16(128, 64);
    int s = 0;
    uint32_t bph = 0;
    int local = 0;
    for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x, ++local) {
      const int ab = local & 1, acc = local & 1;
      const uint32_t ph = (local >> 1) & 1;
      tc::mbar_wait(&t_empty[acc], ph ^ 1);
      tc::mbar_wait(&a_full[ab], ph);
      tc::tc_fence_after();
      const uint32_t a0 = tc::smem_u32(sA + ab * A_BYTES);
      for (int t = 0; t < 27; ++t) {
        tc::mbar_wait(&b_full[s], bph);
        tc::tc_fence_after();
        {
          const int kd = t / 9, kh = (t / 3) % 3, kw = t % 3;
          const uint32_t b0 = tc::smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int sl = 0; sl < 2; ++sl) {
            const uint32_t arow = a0 + (uint32_t)((((sl + kd) * HH + kh) * HW + kw) * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = tc::smem_desc(arow + k * 32, 16, HW * 128, 2);
              const uint64_t bd = tc::smem_desc(b0 + k * 32, 16, 1024, 2);
              tc::mma_bf16_warp(tmem_base + acc * 128 + sl * 64, ad, bd, IDESC, (t | k) != 0);
            }
          }
          tc::mma_commit_warp(&b_empty[s]);
          if (t == 26) {
            tc::mma_commit_warp(&a_empty[ab]);
            tc::mma_commit_warp(&t_full[acc]);
          }
        }
        __syncwarp();
        if (++s == BSTAGES) { s = 0; bph ^= 1; }
      }
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;  // output row in a slice: w = row % 8, h = row / 8
    const int wx = row % 8, hy = row / 8;
    const int et = threadIdx.x - 64;
    if (p.st.mode) {
      for (int i = et; i < 8 * 64; i += 128) red[i] = 0.f;
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    int local = 0;
    for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x, ++local) {
      int64_t r = it;
      const int tw = (int)(r % p.tw); r /= p.tw;
      const int th = (int)(r % p.th); r /= p.th;
      const int td = (int)(r % p.td); r /= p.td;
      const int n = (int)r;
      const int acc = local & 1;
      const int ow = tw * 8 + wx, oh = th * 16 + hy;
      // chunk ch = (slice, 32-channel half); mask / h of the next chunk are prefetched
      auto chunk_valid = [&](int sl) { return ow < p.OW && oh < p.OH && td * 2 + sl < p.OD; };
      auto chunk_base = [&](int sl) { return n * p.s_n + (td * 2 + sl) * p.s_d + oh * p.s_h + ow * p.s_w; };
      StatsPf pf_cur, pf_nxt;
      epi_stats_prefetch(p.st, chunk_valid(0), chunk_base(0), pf_cur);
      tc::mbar_wait(&t_full[acc], (local >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int sl = 0; sl < 2; ++sl) {
        const bool valid = chunk_valid(sl);
        const int64_t obase = chunk_base(sl);
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
          if (c0 == 0) epi_stats_prefetch(p.st, valid, obase + 32, pf_nxt);
          else if (sl == 0) epi_stats_prefetch(p.st, chunk_valid(1), chunk_base(1), pf_nxt);
          uint32_t v[32];
          tc::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * 128 + sl * 64 + c0, v);
          tc::tmem_wait_ld();
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
          if (valid) {
            if (p.bias) {
#pragma unroll
              for (int j = 0; j < 32; ++j) f[j] += p.bias[c0 + j];
            }
            bf16 *dst = p.y + obase + c0;
            if (p.accumulate) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                float o[8];
                load_vec(dst + j, o);
#pragma unroll
                for (int e = 0; e < 8; ++e) f[j + e] += o[e];
              }
            }
            if (p.res) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                float rv[8], mv[8];
                load_vec(p.res + obase + c0 + j, rv);
                load_vec(p.res_mask + obase + c0 + j, mv);
#pragma unroll
                for (int e = 0; e < 8; ++e) f[j + e] += mv[e] > 0.f ? rv[e] : 0.f;
              }
            }
#pragma unroll
            for (int j = 0; j < 32; j += 8) store_vec(dst + j, f + j);
          }
          if (p.st.mode) {
            epi_stats_add(p.st, f, valid, pf_cur, c0, lane, red + (q * 2) * 64 + c0, red + (q * 2 + 1) * 64 + c0);
            pf_cur = pf_nxt;
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&t_empty[acc]);
    }
    if (p.st.mode) epi_stats_flush(p.st, red, 64, 64, et);
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<256>(tmem_base);
  }
}

}  // namespace

bool halo_conv_supported(const ConvGeom &g, bool dgrad) {
  const int kc = dgrad ? g.Co : g.Ci, nout = dgrad ? g.Ci : g.Co;
  return kc == 64 && nout == 64 && g.k == 3 && g.s == 1 && g.p == 1 && g.Wi >= 1;
}

// fprop (w = [Co][27][Ci]) or stride-1 dgrad (src = dy, w = flipped [Ci][27][Co]):
// out[v][n] (=|+=) sum_t src[v + off_t][:] . w[n][t][:]  (+ bias) (+ res*(mask>0))
int conv_halo(const ConvGeom &g, bool dgrad, const bf16 *src, const bf16 *w, const float *bias, bf16 *out,
              bool accumulate, const bf16 *res, const bf16 *res_mask, cudaStream_t st, const EpiStats *est) {
  HaloParams p;
  memset(&p, 0, sizeof p);
  // output grid == input grid (stride 1, pad 1)
  const int W = dgrad ? g.Wi : g.Wo, H = dgrad ? g.Hi : g.Ho, D = dgrad ? g.Di : g.Do;
  make_act_map(&p.a_map, src, 64, W, H, D, g.N, 1, W, (int64_t)W * H, (int64_t)W * H * D, HW, HH, HD, 1);
  make_w_map(&p.b_map, w, 64, 27 * 64, 64);
  for (int t = 0; t < 27; ++t) p.kcoord[t] = t * 64;
  p.OW = W; p.OH = H; p.OD = D; p.ON = g.N;
  p.tw = (W + 7) / 8;
  p.th = (H + 15) / 16;
  p.td = (D + 1) / 2;
  p.n_items = (int64_t)g.N * p.td * p.th * p.tw;
  p.y = out;
  p.s_w = 64;
  p.s_h = (int64_t)W * 64;
  p.s_d = (int64_t)H * W * 64;
  p.s_n = (int64_t)D * H * W * 64;
  p.bias = bias;
  p.accumulate = accumulate;
  p.res = res;
  p.res_mask = res_mask;
  if (est && est->mode) p.st = *est;
  static uint64_t attr_devs = 0;  // kernel attributes are per device
  if (!once_on_device(attr_devs)) {
    CUDA_CHECK(cudaFuncSetAttribute(conv_halo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(p.n_items, sms);
  launch_k(conv_halo_kernel, grid, THREADS, SMEM, st, p);
  LAUNCH_CHECK();
  return p.st.mode ? grid : 0;
}

}  // namespace rn
