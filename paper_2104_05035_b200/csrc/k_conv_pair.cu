// k_conv_pair.cu — the stage-1 3x3x3 convolutions (64 -> 64 channels, stride 1:
// PAPER.md:364/366, the Conv blocks of the first residual stage; about half of
// the step's FLOPs) on CTA PAIRS (tcgen05 cta_group::2) with RESIDENT weights.
//
// Why: with 64 output channels an M=128 x N=64 MMA reads 6 KB of operands from
// smem per 32 tensor cycles (measured 48 cycles: smem-bound, 66 % of peak) and
// the haloed single-CTA kernel streams every tap's weights from L2 again for
// each work item.  A pair MMA (M=256, N=64) reads 4 KB of A + 1 KB of B per SM
// (measured 43 cycles, 74 %), and each CTA holds only its 32 output channels of
// the weights: 27 taps x 32 x 64 bf16 = 108 KB, loaded once per launch.
//
// Work item = one 8 (w) x 16 (h) x 2 (d) output tile of one CTA; a pair runs two
// items in lockstep (same taps, one MMA covering both).  A operands come from 4
// haloed planes (10 x 18 voxels x 64 channels, one TMA box each) in a 4-slot
// ring: plane p of an item is first needed by the taps of slice 0 (p <= 2) or
// slice 1 (p = 3) and released after its last tap, so the next item's planes
// stream in while the current item's later taps run.  Tap (kd, kh, kw) of
// slice s reads plane s + kd starting at row kh*10 + kw (8-row groups 10 rows
// apart).  TMEM: 2 slices x 64 columns, double buffered across items.
//
// Roles per CTA: warp 0 TMA (both CTAs load their own halves; completion is
// counted on the LEADER's barriers), warp 1 MMA issuer (leader only), warps 2-5
// epilogue (each CTA reads its own 128 TMEM lanes: bias / accumulate / masked
// residual / fused BN statistics, as in k_conv_tc.cu).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "bnstats.cuh"
#include "error.h"
#include "kernels.h"
#include "launch.h"
#include "tc_conv.h"
#include "tc_ptx.cuh"
#include "util.cuh"

namespace rn {

void make_act_map(CUtensorMap *m, const void *base, int C, int W, int H, int D, int N, int64_t sw, int64_t sh,
                  int64_t sd, int64_t sn, int bw, int bh, int bd, int bn);
void make_w_map(CUtensorMap *m, const void *base, int rows, int64_t ktot, int bn);

namespace {

constexpr int PW = 10, PH = 18;              // haloed plane box (w, h)
constexpr int PLANE_BYTES = PW * PH * 128;   // 23040 loaded per plane
constexpr int PLANE_SLOT = 23 * 1024;        // 1024-B aligned slots (SW128 TMA destination)
constexpr int B_TAP = 32 * 128;              // this CTA's 32 output channels x 64 input channels
constexpr int B_BYTES = 27 * B_TAP;          // 110592, resident
constexpr int A_OFF = B_BYTES;
constexpr int RED_OFF = A_OFF + 4 * PLANE_SLOT;
constexpr int BAR_OFF = RED_OFF + 4 * 2 * 64 * 4;
constexpr int SMEM = BAR_OFF + 256 + 1024;
constexpr int THREADS = 192;

struct __align__(64) PairParams {
  CUtensorMap a_map;  // 5-D {64, W, H, D, N}, box {64, 10, 18, 1, 1}
  CUtensorMap b_map;  // 2-D {27*64, 64}, box {64, 32}
  int OW, OH, OD, ON;
  int tw, th, td;
  int n_items, n_pair_items;
  bf16 *y;
  int64_t s_n, s_d, s_h, s_w;
  const float *bias;
  int accumulate;
  const bf16 *res, *res_mask;
  EpiStats st;
  int res_pf;  // prefetch the residual operands (RN_PAIR_RES_PF=0 turns it off for A/B)
  unsigned long long *trace;  // debug (RN_PAIR_TRACE): [cta][32] %globaltimer stamps
};

// trace slots: 0 entry, 1 after setup + dependency wait, 2 weights resident (MMA
// warp), 4+2i / 5+2i first / last MMA issue of item i, 16+2i / 17+2i epilogue of
// item i (accumulator acquired / done), 31 exit
__device__ __forceinline__ void pair_stamp(const PairParams &p, int k) {
  if (p.trace && k < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * 32 + k] = t;
  }
}

struct Item {
  int n, td, th, tw;
  bool real;
};
__device__ __forceinline__ Item decode(const PairParams &p, int it) {
  Item r;
  r.real = it < p.n_items;
  if (!r.real) it = 0;
  r.tw = it % p.tw; it /= p.tw;
  r.th = it % p.th; it /= p.th;
  r.td = it % p.td; it /= p.td;
  r.n = it;
  return r;
}

__global__ void __launch_bounds__(THREADS, 1) conv_pair_kernel(const __grid_constant__ PairParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sB = smem, *sA = smem + A_OFF;
  float *red = (float *)(smem + RED_OFF);
  uint64_t *bar = (uint64_t *)(smem + BAR_OFF);
  uint64_t *a_full = bar;        // [4] leader: both CTAs' plane bytes
  uint64_t *a_empty = bar + 4;   // [4] each CTA: multicast MMA commit
  uint64_t *b_full = bar + 8;    // leader: both CTAs' weight bytes
  uint64_t *t_full = bar + 9;    // [2] each CTA: multicast MMA commit
  uint64_t *t_empty = bar + 11;  // [2] leader: 4 epilogue warps x 2 CTAs
  uint32_t *tmem_slot = (uint32_t *)(bar + 13);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = tc::cluster_ctarank();
  const int pair = blockIdx.x / 2, n_pairs = gridDim.x / 2;
  if (threadIdx.x == 0) pair_stamp(p, 0);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&a_full[i], 1);
      tc::mbar_init(&a_empty[i], 1);
    }
    tc::mbar_init(b_full, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&t_full[i], 1);
      tc::mbar_init(&t_empty[i], 8);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&p.a_map);
    tc::tma_prefetch(&p.b_map);
  }
  if (warp == 1) tc::tmem_alloc_pair<256>(tmem_slot);
  tc::tc_fence_before();
  tc::cluster_sync();  // both CTAs' barriers initialised and TMEM allocated
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_begin();
  if (threadIdx.x == 0) pair_stamp(p, 1);

  if (warp == 0) {
    if (lane == 0) {
      // resident weights: this CTA's 32 output channels of every tap
      const uint32_t bf = tc::mapa(tc::smem_u32(b_full), 0);
      if (rank == 0) tc::mbar_arrive_expect_tx(b_full, 2 * B_BYTES);
      for (int t = 0; t < 27; ++t) tc::tma_load_2d_pair(sB + t * B_TAP, &p.b_map, bf, t * 64, (int)rank * 32);
      int local = 0;
      for (int pk = pair; pk < p.n_pair_items; pk += n_pairs, ++local) {
        const Item q = decode(p, 2 * pk + (int)rank);
        const int d0 = q.real ? q.td * 2 - 1 : -64;  // a filler item loads out-of-range (zero) planes
        for (int pl = 0; pl < 4; ++pl) {
          tc::mbar_wait(&a_empty[pl], (local & 1) ^ 1);
          if (rank == 0) tc::mbar_arrive_expect_tx(&a_full[pl], 2 * PLANE_BYTES);
          tc::tma_load_5d_pair(sA + pl * PLANE_SLOT, &p.a_map, tc::mapa(tc::smem_u32(&a_full[pl]), 0), 0,
                               q.tw * 8 - 1, q.th * 16 - 1, d0 + pl, q.n);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t IDESC = tc::idesc_bf16(256, 64);
      // precomputed descriptors: A(plane, kh, kw, k) = dA0 + (pl*PLANE_SLOT + (kh*PW+kw)*128 + 32k) >> 4,
      // B(tap, k) = dB0 + (tap*B_TAP + 32k) >> 4
      const uint64_t dA0 = tc::smem_desc(tc::smem_u32(sA), 16, PW * 128, 2);
      const uint64_t dB0 = tc::smem_desc(tc::smem_u32(sB), 16, 1024, 2);
      tc::mbar_wait_cluster(b_full, 0);
      tc::tc_fence_after();
      if (lane == 0) pair_stamp(p, 2);
      int local = 0;
      for (int pk = pair; pk < p.n_pair_items; pk += n_pairs, ++local) {
        const int acc = local & 1;
        tc::mbar_wait_cluster(&t_empty[acc], ((local >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        bool first = true;
        for (int sl = 0; sl < 2; ++sl) {
          for (int kd = 0; kd < 3; ++kd) {
            const int pl = sl + kd;
            if (sl == 0 || pl == 3) {  // first use of plane pl in this item
              tc::mbar_wait_cluster(&a_full[pl], local & 1);
              tc::tc_fence_after();
            }
            if (first && lane == 0 && local < 6) pair_stamp(p, 4 + 2 * local);
            first = false;
            const uint64_t dAp = dA0 + (uint32_t)(pl * PLANE_SLOT >> 4);
            const uint32_t dtm = tmem_base + acc * 128 + sl * 64;
#pragma unroll
            for (int kh = 0; kh < 3; ++kh) {
#pragma unroll
              for (int kw = 0; kw < 3; ++kw) {
                const int tap = (kd * 3 + kh) * 3 + kw;
                const uint64_t ad = dAp + (uint32_t)((kh * PW + kw) * 8);
                const uint64_t bd = dB0 + (uint32_t)(tap * (B_TAP >> 4));
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  tc::mma_bf16_pair(dtm, ad + 2 * k, bd + 2 * k, IDESC, (kd | kh | kw | k) != 0);
              }
            }
            // last uses: plane 0 after (0,0); plane 1 after (1,0); plane 2 after (1,1); plane 3 after (1,2)
            if (sl == 0 && kd == 0) tc::mma_commit_pair(&a_empty[0], 3);
            if (sl == 1) tc::mma_commit_pair(&a_empty[kd + 1], 3);
          }
        }
        tc::mma_commit_pair(&t_full[acc], 3);
        if (lane == 0 && local < 6) pair_stamp(p, 5 + 2 * local);
        __syncwarp();
      }
    }
    // every MMA of the pair is issued: the dependent grid may start launching
    if (lane == 0) pdl_trigger();
  } else {
    // ---------------- epilogue (warps 2..5, both CTAs) ----------------
    const int q = warp & 3;
    const int row = q * 32 + lane;  // w = row % 8, h = row / 8
    const int wx = row % 8, hy = row / 8;
    const int et = threadIdx.x - 64;
    if (p.st.mode) {
      for (int i = et; i < 8 * 64; i += 128) red[i] = 0.f;
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    const uint32_t te0 = tc::mapa(tc::smem_u32(&t_empty[0]), 0), te1 = tc::mapa(tc::smem_u32(&t_empty[1]), 0);
    int local = 0;
    for (int pk = pair; pk < p.n_pair_items; pk += n_pairs, ++local) {
      const Item it = decode(p, 2 * pk + (int)rank);
      const int acc = local & 1;
      const int ow = it.tw * 8 + wx, oh = it.th * 16 + hy;
      auto chunk_valid = [&](int sl) { return it.real && ow < p.OW && oh < p.OH && it.td * 2 + sl < p.OD; };
      auto chunk_base = [&](int sl) {
        return it.n * p.s_n + (it.td * 2 + sl) * p.s_d + oh * p.s_h + ow * p.s_w;
      };
      StatsPf pf_cur, pf_nxt;
      // identity-skip residual (dgrad without fused statistics): its residual and mask
      // rows travel in the statistics prefetch registers, one 32-channel chunk ahead --
      // the first chunk's before the accumulator wait (latency behind the mainloop)
      const bool res_pf = p.res && p.st.mode < 2 && p.res_pf;
      // accumulate without residual / backward statistics: the existing output rows
      // travel in the same prefetch registers, one chunk ahead
      const bool acc_pf = p.accumulate && !p.res && p.st.mode < 2 && p.res_pf;
      auto prefetch = [&](bool valid, int64_t eo, StatsPf &pf) {
        if (res_pf) {
          if (!valid) return;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            pf.m[i] = __ldg(reinterpret_cast<const uint4 *>(p.res_mask + eo) + i);
            pf.h[i] = __ldg(reinterpret_cast<const uint4 *>(p.res + eo) + i);
          }
        } else if (acc_pf) {
          if (!valid) return;
#pragma unroll
          for (int i = 0; i < 4; ++i) pf.h[i] = *(reinterpret_cast<const uint4 *>(p.y + eo) + i);
        } else {
          epi_stats_prefetch(p.st, valid, eo, pf);
        }
      };
      prefetch(chunk_valid(0), chunk_base(0), pf_cur);
      tc::mbar_wait(&t_full[acc], (local >> 1) & 1);
      tc::tc_fence_after();
      if (et == 0 && local < 6) pair_stamp(p, 16 + 2 * local);
#pragma unroll 1
      for (int sl = 0; sl < 2; ++sl) {
        const bool valid = chunk_valid(sl);
        const int64_t obase = chunk_base(sl);
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
          if (c0 == 0) prefetch(valid, obase + 32, pf_nxt);
          else if (sl == 0) prefetch(chunk_valid(1), chunk_base(1), pf_nxt);
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
            if (acc_pf) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                float o[8];
                unpack_bf16x8(pf_cur.h[j], o);
#pragma unroll
                for (int e = 0; e < 8; ++e) f[8 * j + e] += o[e];
              }
            } else if (p.accumulate) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                float o[8];
                load_vec(dst + j, o);
#pragma unroll
                for (int e = 0; e < 8; ++e) f[j + e] += o[e];
              }
            }
            if (res_pf) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                float rv[8], mv[8];
                unpack_bf16x8(pf_cur.h[j], rv);
                unpack_bf16x8(pf_cur.m[j], mv);
#pragma unroll
                for (int e = 0; e < 8; ++e) f[8 * j + e] += mv[e] > 0.f ? rv[e] : 0.f;
              }
            } else if (p.res) {
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
          if (p.st.mode) epi_stats_add(p.st, f, valid, pf_cur, c0, lane, red + (q * 2) * 64 + c0,
                                       red + (q * 2 + 1) * 64 + c0);
          if (p.st.mode || res_pf || acc_pf) pf_cur = pf_nxt;
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(acc ? te1 : te0);  // the leader's accumulator-free barrier
      if (et == 0 && local < 6) pair_stamp(p, 17 + 2 * local);
    }
    if (p.st.mode) epi_stats_flush(p.st, red, 64, 64, et);
  }
  tc::tc_fence_before();
  tc::cluster_sync();  // no CTA leaves while its pair may still read its smem / TMEM
  if (threadIdx.x == 0) pair_stamp(p, 31);
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc_pair<256>(tmem_base);
  }
}

}  // namespace

unsigned long long *g_pair_trace = nullptr;
int g_pair_trace_n = 0;
int g_pair_meta[64][4];

bool pair_conv_supported(const ConvGeom &g, bool dgrad) { return halo_conv_supported(g, dgrad); }

// fprop (w = [Co][27][Ci]) or stride-1 dgrad (src = dy, w = flipped [Ci][27][Co]):
// out[v][n] (=|+=) sum_t src[v + off_t][:] . w[n][t][:]  (+ bias) (+ res*(mask>0))
int conv_pair(const ConvGeom &g, bool dgrad, const bf16 *src, const bf16 *w, const float *bias, bf16 *out,
              bool accumulate, const bf16 *res, const bf16 *res_mask, cudaStream_t st, const EpiStats *est) {
  PairParams p;
  memset(&p, 0, sizeof p);
  const int W = dgrad ? g.Wi : g.Wo, H = dgrad ? g.Hi : g.Ho, D = dgrad ? g.Di : g.Do;
  make_act_map(&p.a_map, src, 64, W, H, D, g.N, 1, W, (int64_t)W * H, (int64_t)W * H * D, PW, PH, 1, 1);
  make_w_map(&p.b_map, w, 64, 27 * 64, 32);
  p.OW = W; p.OH = H; p.OD = D; p.ON = g.N;
  p.tw = (W + 7) / 8;
  p.th = (H + 15) / 16;
  p.td = (D + 1) / 2;
  p.n_items = g.N * p.td * p.th * p.tw;
  p.n_pair_items = (p.n_items + 1) / 2;
  p.y = out;
  p.s_w = 64;
  p.s_h = (int64_t)W * 64;
  p.s_d = (int64_t)H * W * 64;
  p.s_n = (int64_t)D * H * W * 64;
  p.bias = bias;
  p.accumulate = accumulate;
  p.res = res;
  p.res_pf = !(getenv("RN_PAIR_RES_PF") && atoi(getenv("RN_PAIR_RES_PF")) == 0);
  p.res_mask = res_mask;
  if (est && est->mode) p.st = *est;
  if (getenv("RN_PAIR_TRACE") && g_pair_trace_n < 64) {
    if (!g_pair_trace) CUDA_CHECK(cudaMalloc(&g_pair_trace, sizeof(unsigned long long) * 64 * 148 * 32));
    CUDA_CHECK(cudaMemsetAsync(g_pair_trace + (size_t)g_pair_trace_n * 148 * 32, 0, sizeof(unsigned long long) * 148 * 32, st));
    p.trace = g_pair_trace + (size_t)g_pair_trace_n * 148 * 32;
    g_pair_meta[g_pair_trace_n][0] = dgrad;
    g_pair_meta[g_pair_trace_n][1] = res != nullptr;
    g_pair_meta[g_pair_trace_n][2] = p.st.mode;
    g_pair_meta[g_pair_trace_n][3] = p.n_pair_items;
    ++g_pair_trace_n;
  }
  static uint64_t attr_devs = 0;  // kernel attributes are per device
  if (!once_on_device(attr_devs)) {
    CUDA_CHECK(cudaFuncSetAttribute(conv_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int pairs = std::max(1, std::min(p.n_pair_items, sms / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, conv_pair_kernel, p));
  LAUNCH_CHECK();
  return p.st.mode ? 2 * pairs : 0;
}

}  // namespace rn

// debug: copy the RN_PAIR_TRACE stamps of the first launches (148 CTAs x 32 slots each)
extern "C" int rn_dbg_pair_trace(unsigned long long *host, int max_launches, int *meta) {
  using namespace rn;
  const int n = std::min(g_pair_trace_n, max_launches);
  if (n > 0 && g_pair_trace) {
    cudaDeviceSynchronize();
    cudaMemcpy(host, g_pair_trace, sizeof(unsigned long long) * (size_t)n * 148 * 32, cudaMemcpyDeviceToHost);
    memcpy(meta, g_pair_meta, sizeof(int) * 4 * n);
  }
  return n;
}
