// k_conv_tc.cu — 3D convolution as an implicit GEMM on the 5th-generation tensor
// cores (tcgen05, accumulators in TMEM), operands staged by TMA (PAPER.md:366:
// the Conv block's 3x3x3 convolution, complexity O(Co*Ci*T*H*W*Kt*Kh*Kw), is
// where the step's operations are).
//
// GEMM view of one launch ("implicit GEMM over taps"):
//   rows    M = output voxels, tiled by a 3-D/4-D box of 128 voxels (bw x bh x bd x bn)
//   columns N = output channels, tile BN in {64, 128, 256}
//   K       = sum over taps t of 64-channel blocks of the A tensor
//   A[m, (t,c)] = src[view_t](voxel(m) + offset_t)[c]   (TMA 5-D box, OOB -> 0)
//   B[n, (t,c)] = W[n][kcoord_t + c]                      (TMA 2-D box)
// fprop: src = x, W = W[co][tap][ci];  dgrad (stride 1): src = dy, W = flipped
// W^T[ci][tap'][co];  dgrad stride 2: ONE launch over the 8 output parity
// classes ("classes": each a strided output view with its own subset of taps,
// work items enumerated class after class, heaviest first), optionally with the
// stage-entry 1x1x1 stride-2 projection's dgrad appended to class (0,0,0) as a
// 28th tap from a second A/B tensor pair;  stride-2 fprop: the A views are the
// 8 parity sub-lattices of x.
//
// Kernel: persistent, one CTA per SM, warp-specialised: warp 0 TMA producer,
// warp 1 MMA issuer (one elected lane, tcgen05.mma M=128, N=BN, K=16), warps
// 2-5 epilogue (tcgen05.ld 32x32b -> fp32 registers -> bias / accumulate /
// masked residual -> bf16 stores).  STAGES-deep smem ring (mbarriers), 2 TMEM
// accumulators so the epilogue of tile i overlaps the main loop of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "bnstats.cuh"
#include "error.h"
#include "launch.h"
#include "kernels.h"
#include "tc_conv.h"
#include "tc_ptx.cuh"
#include "util.cuh"

namespace rn {

namespace {

constexpr int TC_THREADS = 192;
// one-CTA-per-SM variants (deep ring) run 8 warps: in the direct TMA epilogue of
// their single work item the producer and MMA warps join the four epilogue warps
// once their loops are done (two warps per TMEM lane quarter, columns split; the
// 4-warp epilogue was latency-bound, one warp per scheduler).  8 warps keep the
// 255-register budget (10 would cap it at 168: 3 warps on one 16 K-register SMSP)
template <int BN, int STAGES, bool PAIR = false>
constexpr int tc_threads() {
  return (!PAIR && STAGES * (128 * 128 + BN * 128) > 110 * 1024) ? 256 : TC_THREADS;
}
constexpr bool kPdlLate = true;  // explicit late PDL trigger (after the last MMA issue)

constexpr int MAX_TAPS = 28;  // 27 taps + the appended projection tap (stride-2 dgrad)

struct __align__(64) TcParams {
  CUtensorMap a_map[8];
  CUtensorMap b_map, b_map2;
  int n_taps;
  int kblocks_per_tap;  // A channels / 64
  int8_t tap_map[MAX_TAPS];   // A tensor map of the tap
  int8_t tap_bsel[MAX_TAPS];  // 0: b_map, 1: b_map2
  int8_t tap_od[MAX_TAPS], tap_oh[MAX_TAPS], tap_ow[MAX_TAPS];
  int tap_kcoord[MAX_TAPS];
  // classes of work items (1 for plain launches; the parity classes of a stride-2
  // dgrad): items [cls_item0[c], cls_item0[c+1]) = tiles x cls_ks[c] splits of
  // class c, whose taps are [cls_tap0[c], cls_tap0[c] + cls_ntaps[c])
  int n_cls;
  int64_t cls_item0[9];
  int cls_ks[8], cls_tap0[8], cls_ntaps[8];
  int cls_OW[8], cls_OH[8], cls_OD[8];  // valid extents of the class view
  int64_t cls_yoff[8];                  // element offset of the class view in y / res / mask / h
  int64_t cls_pbase[8];                 // split-K partial base (floats)
  // output tiling: view extents and box
  int OD, OH, OW, ON;
  int bw, bh, bd, bn;
  int tw, th, td, tn, t_nblk;  // tiles per dim, N-blocks of BN
  int64_t n_tiles;
  // output addressing (elements)
  bf16 *y;
  int64_t s_n, s_d, s_h, s_w;
  int ych;  // channels of y per voxel
  const float *bias;
  int accumulate;
  const bf16 *res;
  const bf16 *res_mask;
  // split-K over the K blocks (layers with fewer tiles than SMs): ksplit of a
  // one-class launch; use_part = the epilogue writes fp32 partials (finish kernel)
  int ksplit;
  int use_part;
  float *part;
  int64_t n_view_vox;
  EpiStats st;  // fused BN statistics of the stored output (needs !use_part, t_nblk == 1)
  unsigned long long *trace;  // debug (RN_TC_TRACE): per-CTA %globaltimer stamps [grid][8]
  // CTA pairs (cta_group::2, one-class launches): a cluster of 2 CTAs runs M-tiles
  // 2j and 2j+1 of the same (N-block, split) as ONE M=256 MMA; each CTA streams its
  // own A tile and HALF of the B tile (BN/2 output channels), so the per-SM smem
  // traffic per FLOP drops (operand reads + TMA fills: the stage-2/3 bound).
  // Work items count pairs; n_mt = M-tiles (an odd last pair has an empty half).
  int pair;
  int64_t n_mt;
  const bf16 *w_base;  // host: weights behind b_map (re-encoded with a BN/2 box for pairs)
  int w_rows;
  int64_t w_ktot;
  // TMA-store epilogue (launches whose CTAs own at most one work item): the tile is
  // staged in the (then idle) smem ring, SW128-swizzled, and written by
  // cp.async.bulk.tensor -- coalesced, instead of one 16-B store per row per thread.
  // tma_st 1: bf16 y through y_map (box {64, bw, bh, bd, bn}); 2: fp32 split-K
  // partials through part_map (box {32, ...}, 5th dim = split * ON + n)
  int tma_ok;  // host: the maps are valid for this launch (one class, aligned views)
  int tma_st;
  CUtensorMap y_map, part_map;
  // direct path inputs loaded by TMA into the ring at the epilogue: residual and its
  // mask (identity-skip dgrad), the consumer BN's h / ReLU mask (backward statistics)
  CUtensorMap res_map, resm_map, h_map, m_map;
};

// smem bytes of the TMA epilogue (direct path): output tile + every input tile
__host__ __device__ inline int tma_epi_bytes(int BN, bool res, int stmode) {
  const int t = 128 * BN * 2;
  return t * (1 + (res ? 2 : 0) + (stmode == 2 ? 2 : stmode == 3 ? 1 : 0));
}

__device__ __forceinline__ void tc_stamp(const TcParams &p, int k) {
  if (p.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * 8 + k] = t;
  }
}

template <int BN, int STAGES, bool PAIR = false>
struct Smem {
  static constexpr int A_BYTES = 128 * 128;                  // 128 rows x 64 bf16
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * 128;  // BN (pair: BN/2) rows x 64 bf16
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int RED_OFF = STAGES * STAGE;   // [4 warps][2][BN] fp32 BN-statistics accumulators
  static constexpr int BAR_OFF = RED_OFF + 4 * 2 * BN * 4;
  static constexpr int TAB_OFF = BAR_OFF + 256;       // per-tap TMA table (the producer's hot loop)
  static constexpr int TOTAL = TAB_OFF + MAX_TAPS * 16 + 1024;  // + alignment slack
};

struct Item {
  int c, split, nb, tw, th, td, tn, kb0, kb1;
};
// one tap's TMA coordinates, staged in smem (indexed kernel-parameter loads in
// the producer loop measured as a visible stall)
struct __align__(16) TapEnt {
  const CUtensorMap *amap, *bmap;
  int16_t od, oh, ow, pad;
  int kcoord;
};
__device__ __forceinline__ Item decode_item(const TcParams &p, int64_t item, int rank = 0) {
  Item it;
  int c = 0;
  while (c + 1 < p.n_cls && item >= p.cls_item0[c + 1]) ++c;
  it.c = c;
  int64_t r = item - p.cls_item0[c];
  const int ks = p.cls_ks[c];
  it.split = (int)(r % ks); r /= ks;
  it.nb = (int)(r % p.t_nblk); r /= p.t_nblk;
  if (p.pair) r = 2 * r + rank;  // this CTA's M-tile of the pair (>= n_mt: empty half, tn out of range)
  it.tw = (int)(r % p.tw); r /= p.tw;
  it.th = (int)(r % p.th); r /= p.th;
  it.td = (int)(r % p.td); r /= p.td;
  it.tn = (int)r;
  const int nk = p.cls_ntaps[c] * p.kblocks_per_tap;
  it.kb0 = it.split * nk / ks;
  it.kb1 = (it.split + 1) * nk / ks;
  return it;
}

// deep-ring variants (one CTA per SM by smem) get the whole register file: no spills
template <int BN, int STAGES, bool PAIR = false>
__global__ void __launch_bounds__(tc_threads<BN, STAGES, PAIR>(),
                                  (STAGES * Smem<BN, STAGES, PAIR>::STAGE > 110 * 1024) ? 1 : 2)
    conv_tc_kernel(const __grid_constant__ TcParams p) {
  using S = Smem<BN, STAGES, PAIR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + S::BAR_OFF);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = (uint32_t *)(tempty + 3);  // tempty[2] = the TMA epilogue's input barrier
  TapEnt *tab = (TapEnt *)(smem + S::TAB_OFF);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // pairs: rank in the cluster (0 = leader: issues the pair MMAs, owns the full /
  // tempty barriers both CTAs count on); the pair's item stream is blockIdx / 2
  const int rank = PAIR ? (int)tc::cluster_ctarank() : 0;
  const int64_t wid = PAIR ? blockIdx.x / 2 : blockIdx.x, wstride = PAIR ? gridDim.x / 2 : gridDim.x;
  if (threadIdx.x == 0) tc_stamp(p, 0);
  if (warp == 0 && lane < p.n_taps) {
    TapEnt e;
    e.amap = &p.a_map[p.tap_map[lane]];
    e.bmap = p.tap_bsel[lane] ? &p.b_map2 : &p.b_map;
    e.od = p.tap_od[lane]; e.oh = p.tap_oh[lane]; e.ow = p.tap_ow[lane]; e.pad = 0;
    e.kcoord = p.tap_kcoord[lane];
    tab[lane] = e;
  }
  constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                  : (2 * BN <= 256) ? 256 : 512;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], PAIR ? 8 : 4);  // epilogue warps (of both CTAs of a pair)
    }
    tc::mbar_init(&tempty[2], 1);
    tc::fence_barrier_init();
    for (int i = 0; i < p.n_taps; ++i)
      if (i == 0 || p.tap_map[i] != p.tap_map[i - 1]) tc::tma_prefetch(&p.a_map[p.tap_map[i]]);
    tc::tma_prefetch(&p.b_map);
    for (int i = 0; i < p.n_taps; ++i)
      if (p.tap_bsel[i]) { tc::tma_prefetch(&p.b_map2); break; }
  }
  if (warp == 1) {
    if constexpr (PAIR) tc::tmem_alloc_pair<TMEM_COLS>(tmem_slot);
    else tc::tmem_alloc<TMEM_COLS>(tmem_slot);
  }
  tc::tc_fence_before();
  if constexpr (PAIR) tc::cluster_sync();  // both CTAs' barriers initialised, TMEM allocated
  else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_begin();  // prologue above overlaps the predecessor's tail
  if (threadIdx.x == 0) tc_stamp(p, 1);

  const int64_t n_items = p.cls_item0[p.n_cls];

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t item = wid; item < n_items; item += wstride) {
        const Item it = decode_item(p, item, rank);
        const int w0 = it.tw * p.bw, h0 = it.th * p.bh, d0 = it.td * p.bd, n0 = it.tn * p.bn;
        const int nb = it.nb;
        const int tap0 = p.cls_tap0[it.c], kpt = p.kblocks_per_tap;
        int t = tap0 + it.kb0 / kpt, cb = it.kb0 % kpt;
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          const TapEnt e = tab[t];
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *sa = smem + stage * S::STAGE;
          uint8_t *sb = sa + S::A_BYTES;
          if (kb == it.kb0 && item == wid) tc_stamp(p, 2);
          if constexpr (PAIR) {
            // both CTAs' bytes land on the leader's full barrier
            const uint32_t fb = tc::mapa(tc::smem_u32(&full[stage]), 0);
            if (rank == 0) tc::mbar_arrive_expect_tx(&full[stage], 2 * S::STAGE);
            tc::tma_load_5d_pair(sa, e.amap, fb, cb * 64, w0 + e.ow, h0 + e.oh, d0 + e.od, n0);
            tc::tma_load_2d_pair(sb, e.bmap, fb, e.kcoord + cb * 64, nb * BN + rank * (BN / 2));
          } else {
            tc::mbar_arrive_expect_tx(&full[stage], S::STAGE);
            tc::tma_load_5d(sa, e.amap, &full[stage], cb * 64, w0 + e.ow, h0 + e.oh, d0 + e.od, n0);
            tc::tma_load_2d(sb, e.bmap, &full[stage], e.kcoord + cb * 64, nb * BN);
          }
          if (++cb == kpt) { cb = 0; ++t; }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // descriptors precomputed: stage s, k-step k = base + (s * STAGE + 32 k) >> 4
    // (the issue loop must sustain one MMA per 32-64 tensor cycles)
    constexpr uint32_t IDESC = tc::idesc_bf16(PAIR ? 256 : 128, BN);
    const uint64_t dA0 = tc::smem_desc(tc::smem_u32(smem), 16, 1024, 2);
    const uint64_t dB0 = tc::smem_desc(tc::smem_u32(smem) + S::A_BYTES, 16, 1024, 2);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    if (!PAIR || rank == 0)  // pairs: the leader issues for both CTAs
      for (int64_t item = wid; item < n_items; item += wstride, ++local) {
        const Item it = decode_item(p, item, rank);
        const int kb0 = it.kb0, kb1 = it.kb1;
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        if constexpr (PAIR) tc::mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        else tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        uint32_t accum = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
          if constexpr (PAIR) tc::mbar_wait_cluster(&full[stage], phase);
          else tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          if (local == 0 && kb == kb0 && lane == 0) tc_stamp(p, 3);
          const uint32_t soff = (uint32_t)(stage * S::STAGE) >> 4;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if constexpr (PAIR) tc::mma_bf16_pair(d_tmem, dA0 + soff + 2 * k, dB0 + soff + 2 * k, IDESC, accum);
            else tc::mma_bf16_warp(d_tmem, dA0 + soff + 2 * k, dB0 + soff + 2 * k, IDESC, accum);
            accum = 1;
          }
          if constexpr (PAIR) {
            tc::mma_commit_pair(&empty[stage], 3);  // both producers' stage is free
            if (kb == kb1 - 1) tc::mma_commit_pair(&tfull[acc], 3);
          } else {
            tc::mma_commit_warp(&empty[stage]);
            if (kb == kb1 - 1) tc::mma_commit_warp(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    // every MMA of this CTA is issued: the dependent grid may start launching
    // (persistent grid: no later wave of this kernel to be displaced)
    if (lane == 0) tc_stamp(p, 4);
    if (kPdlLate) pdl_trigger();
  }
  const bool direct = p.tma_st == 1 && wid < n_items;
  constexpr bool ALLW = tc_threads<BN, STAGES, PAIR>() == 256;
  if ((direct && ALLW) || (warp >= 2 && warp < 6)) {
    // ---------------- epilogue (warps 2..5; every warp in the 8-warp direct epilogue) ----------------
    __syncwarp();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    const int et = (direct && ALLW) ? (int)threadIdx.x : (int)threadIdx.x - 64;
    const int NEPI = (direct && ALLW) ? 256 : 128;  // epilogue threads
    float *red = (float *)(smem + S::RED_OFF);
    if (p.st.mode) {
      for (int i = et; i < 8 * BN; i += NEPI) red[i] = 0.f;
      asm volatile("bar.sync 1, %0;" ::"r"(NEPI) : "memory");
    }
    const int wx = row % p.bw, hy = (row / p.bw) % p.bh, dz = (row / (p.bw * p.bh)) % p.bd,
              nz = row / (p.bw * p.bh * p.bd);
    if (direct) {
      // ---- direct TMA epilogue: this CTA's single work item ----
      const int NH = NEPI / 128;                        // warps per TMEM lane quarter
      const int half = ALLW ? warp / 4 : 0;             // this warp's column slice
      const int cbeg = half * (BN / NH), cend = cbeg + BN / NH;
      const Item it = decode_item(p, wid, rank);
      const int nb = it.nb;
      const int w0 = it.tw * p.bw, h0 = it.th * p.bh, d0 = it.td * p.bd, n0 = it.tn * p.bn;
      constexpr int NCH = BN / 64, TB = 128 * BN * 2;
      uint8_t *s_out = smem;  // output (and the accumulate input)
      int off = TB;
      uint8_t *s_res = nullptr, *s_rm = nullptr, *s_h = nullptr, *s_m = nullptr;
      if (p.res) { s_res = smem + off; off += TB; s_rm = smem + off; off += TB; }
      if (p.st.mode >= 2) { s_h = smem + off; off += TB; }
      if (p.st.mode == 2) { s_m = smem + off; off += TB; }
      uint64_t *ebar = tempty + 2;  // epilogue input barrier (after tempty[2], before tmem_slot)
      tc::mbar_wait(&tfull[0], 0);
      tc::tc_fence_after();
      const bool need_in = p.accumulate || p.res || p.st.mode >= 2;
      if (need_in) {
        if (et == 0) {
          const uint32_t bytes = (uint32_t)(off - (p.accumulate ? 0 : TB));
          tc::mbar_arrive_expect_tx(ebar, bytes);
          for (int j = 0; j < NCH; ++j) {
            const int cc = nb * BN + j * 64;
            if (p.accumulate) tc::tma_load_5d(s_out + j * 16384, &p.y_map, ebar, cc, w0, h0, d0, n0);
            if (p.res) {
              tc::tma_load_5d(s_res + j * 16384, &p.res_map, ebar, cc, w0, h0, d0, n0);
              tc::tma_load_5d(s_rm + j * 16384, &p.resm_map, ebar, cc, w0, h0, d0, n0);
            }
            if (s_h) tc::tma_load_5d(s_h + j * 16384, &p.h_map, ebar, cc, w0, h0, d0, n0);
            if (s_m) tc::tma_load_5d(s_m + j * 16384, &p.m_map, ebar, cc, w0, h0, d0, n0);
          }
        }
        tc::mbar_wait(ebar, 0);
      }
      if (et == 0) tc_stamp(p, 5);
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        uint32_t v[32];
        tc::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + c0, v);
        tc::tmem_wait_ld();
        const int chk = (c0 / 64) * 16384 + row * 128, q0 = (c0 % 64) / 8;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int po = chk + (((q0 + j) ^ (row & 7)) << 4);
          float f[8], o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[8 * j + e]);
          if (p.bias)
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] += p.bias[nb * BN + c0 + 8 * j + e];
          if (p.accumulate) {
            unpack_bf16x8(*reinterpret_cast<const uint4 *>(s_out + po), o);
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] += o[e];
          }
          if (p.res) {
            float rv[8], mv[8];
            unpack_bf16x8(*reinterpret_cast<const uint4 *>(s_res + po), rv);
            unpack_bf16x8(*reinterpret_cast<const uint4 *>(s_rm + po), mv);
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] += mv[e] > 0.f ? rv[e] : 0.f;
          }
          uint4 u;
          __nv_bfloat162 *pv = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) pv[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
          *reinterpret_cast<uint4 *>(s_out + po) = u;
        }
      }
      tc::tc_fence_before();
      tc::fence_proxy_async();
      asm volatile("bar.sync 1, %0;" ::"r"(NEPI) : "memory");
      if (et == 0 && n0 < p.ON) {  // (the empty half of an odd last pair stores nothing)
        for (int j = 0; j < NCH; ++j) tc::tma_store_5d(&p.y_map, s_out + j * 16384, nb * BN + j * 64, w0, h0, d0, n0);
        tc::bulk_commit();
      }
      if (p.st.mode) {
        // BN statistics of the stored tile by columns from smem (no shuffles): the
        // bf16 values the store writes; out-of-volume rows are zero (TMA zero fill).
        // NEPI threads: column c = et % BN over row slice et / BN of NRS slices
        const int NRS = NEPI >= BN ? NEPI / BN : 1, RPS = 128 / NRS;
        const int rs = et / BN;
        for (int c = et % BN; c < BN && rs < NRS; c += NEPI) {
          const int cb = (c / 64) * 16384 + (c % 8) * 2, pq = (c % 64) / 8;
          const float mu = p.st.mode >= 2 ? p.st.mean[nb * BN + c] : 0.f;
          const float ms = p.st.mode == 3 ? p.st.mscale[nb * BN + c] : 0.f;
          const float mh = p.st.mode == 3 ? p.st.mshift[nb * BN + c] : 0.f;
          float s1 = 0.f, s2 = 0.f;
#pragma unroll 4
          for (int r = rs * RPS; r < (rs + 1) * RPS; ++r) {
            const int a = cb + r * 128 + ((pq ^ (r & 7)) << 4);
            const float o = __bfloat162float(*reinterpret_cast<const bf16 *>(s_out + a));
            if (p.st.mode == 1) {
              s1 += o;
              s2 = fmaf(o, o, s2);
            } else {
              const float h = __bfloat162float(*reinterpret_cast<const bf16 *>(s_h + a));
              const float m = p.st.mode == 2 ? __bfloat162float(*reinterpret_cast<const bf16 *>(s_m + a))
                                             : fmaf(h, ms, mh);
              const float d = m > 0.f ? o : 0.f;
              s1 += d;
              s2 = fmaf(d, h - mu, s2);
            }
          }
          red[(rs * 2) * BN + c] += s1;      // slice rs in the warp-rs accumulator slot
          red[(rs * 2 + 1) * BN + c] += s2;
        }
        // every slot written: sum the (<= 4) row slices in order and write the partial
        asm volatile("bar.sync 1, %0;" ::"r"(NEPI) : "memory");
        for (int c = et; c < BN; c += NEPI) {
          float a = 0.f, b2 = 0.f;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            a += red[(w * 2 + 0) * BN + c];
            b2 += red[(w * 2 + 1) * BN + c];
          }
          p.st.part[(int64_t)blockIdx.x * 2 * BN + c] = a;
          p.st.part[(int64_t)blockIdx.x * 2 * BN + BN + c] = b2;
        }
      }
      if (et == 0) tc::bulk_wait0();
    } else {
    int local = 0;
    for (int64_t item = wid; item < n_items; item += wstride, ++local) {
      const Item it = decode_item(p, item, rank);
      const int split = it.split, nb = it.nb, c = it.c;
      const int ow = it.tw * p.bw + wx, oh = it.th * p.bh + hy, od = it.td * p.bd + dz, on = it.tn * p.bn + nz;
      const bool valid = ow < p.cls_OW[c] && oh < p.cls_OH[c] && od < p.cls_OD[c] && on < p.ON;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int64_t obase =
          p.cls_yoff[c] + on * p.s_n + od * p.s_d + oh * p.s_h + ow * p.s_w + (int64_t)nb * BN;
      StatsPf pf_cur, pf_nxt;
      epi_stats_prefetch(p.st, valid, obase, pf_cur);  // before the accumulator wait
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::tc_fence_after();
      if (local == 0 && et == 0) tc_stamp(p, 5);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        if (c0 + 32 < BN) epi_stats_prefetch(p.st, valid, obase + c0 + 32, pf_nxt);
        uint32_t v[32];
        tc::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c0, v);
        tc::tmem_wait_ld();
        if (p.tma_st == 2) {  // fp32 partial row -> staging chunk c0/32 (16 KB), SW128
          uint8_t *ch = smem + (c0 / 32) * 16384 + row * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4 *>(ch + ((j ^ (row & 7)) << 4)) = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2],
                                                                                 v[4 * j + 3]);
          continue;
        }
        if (valid && p.use_part) {
          // split-K: raw fp32 partial [class][split][view voxel][Nout]; epilogue in the finish kernel
          const int64_t vidx = ((int64_t)(on * p.OD + od) * p.OH + oh) * p.OW + ow;
          float *dst = p.part + p.cls_pbase[c] + ((int64_t)split * p.n_view_vox + vidx) * p.ych + nb * BN + c0;
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4 *>(dst + j) = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                               __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
          continue;
        }
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        if (valid) {
          if (p.bias) {
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] += p.bias[nb * BN + c0 + j];
          }
        }
        if (p.tma_st == 1) {  // bf16 row segment -> staging chunk c0/64 (16 KB), SW128
          uint8_t *ch = smem + (c0 / 64) * 16384 + row * 128;
          const int q0 = (c0 % 64) / 8;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 u;
            __nv_bfloat162 *pv = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) pv[e] = __floats2bfloat162_rn(f[8 * j + 2 * e], f[8 * j + 2 * e + 1]);
            *reinterpret_cast<uint4 *>(ch + (((q0 + j) ^ (row & 7)) << 4)) = u;
          }
        } else if (valid) {
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
            const int64_t ro = obase + c0;
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              float rv[8], mv[8];
              load_vec(p.res + ro + j, rv);
              load_vec(p.res_mask + ro + j, mv);
#pragma unroll
              for (int e = 0; e < 8; ++e) f[j + e] += mv[e] > 0.f ? rv[e] : 0.f;
            }
          }
#pragma unroll
          for (int j = 0; j < 32; j += 8) store_vec(dst + j, f + j);
        }
        if (p.st.mode) {
          epi_stats_add(p.st, f, valid, pf_cur, c0, lane, red + (q * 2) * BN + c0, red + (q * 2 + 1) * BN + c0);
          pf_cur = pf_nxt;
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&tempty[acc]), 0));  // the leader's
        else tc::mbar_arrive(&tempty[acc]);
      }
      if (p.tma_st == 2) {
        // every row of the tile is staged: make the generic-proxy smem writes visible
        // to the async proxy, then one thread writes the tile with TMA
        tc::fence_proxy_async();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int n0 = it.tn * p.bn;
        if (et == 0 && n0 < p.ON) {  // (an empty pair half must not write into the next split's rows)
          const int w0 = it.tw * p.bw, h0 = it.th * p.bh, d0 = it.td * p.bd;
          for (int j = 0; j < BN / 32; ++j)
            tc::tma_store_5d(&p.part_map, smem + j * 16384, nb * BN + j * 32, w0, h0, d0, split * p.ON + n0);
          tc::bulk_commit();
          tc::bulk_wait0();  // complete before the grid does (the finish / BN kernels read it)
        }
      }
    }
      if (p.st.mode) epi_stats_flush(p.st, red, BN, BN, et);
    }  // generic epilogue (warps 2..5)
    if (et == 0) tc_stamp(p, 6);
  }
  tc::tc_fence_before();
  if constexpr (PAIR) tc::cluster_sync();  // no CTA leaves while the pair's MMAs may read its smem / TMEM
  else __syncthreads();
  if (threadIdx.x == 0) tc_stamp(p, 7);
  if (warp == 1) {
    tc::tc_fence_after();
    if constexpr (PAIR) tc::tmem_dealloc_pair<TMEM_COLS>(tmem_base);
    else tc::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

void load_encode() {
  if (g_encode) return;
  cudaDriverEntryPointQueryResult q;
  void *fn = nullptr;
  CUDA_CHECK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) throw Error(RN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

}  // namespace

// 5-D view of an NDHWC bf16 tensor: dims {C, W, H, D, N} with element strides
// (sw, sh, sd, sn) in voxels (a parity sub-lattice uses doubled strides).
static thread_local size_t *g_dry_need = nullptr;  // non-null: size the split-K workspace only

void make_act_map(CUtensorMap *m, const void *base, int C, int W, int H, int D, int N, int64_t sw, int64_t sh,
                  int64_t sd, int64_t sn, int bw, int bh, int bd, int bn) {
  if (g_dry_need) return;
  load_encode();
  cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)D, (cuuint64_t)N};
  cuuint64_t strides[4] = {(cuuint64_t)(sw * C * 2), (cuuint64_t)(sh * C * 2), (cuuint64_t)(sd * C * 2),
                           (cuuint64_t)(sn * C * 2)};
  cuuint32_t box[5] = {64, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bd, (cuuint32_t)bn};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(RN_ERR_CUDA, "cuTensorMapEncodeTiled (activation) failed: " + std::to_string(r));
}

// 5-D output view of a contiguous NDHWC tensor (bf16 or fp32) for TMA stores:
// dims {C, W, H, D, N}, box {128 B of channels, bw, bh, bd, bn}, SW128
static void make_out_map(CUtensorMap *m, const void *base, bool f32, int C, int W, int H, int D, int N, int bw, int bh,
                         int bd, int bn) {
  if (g_dry_need) return;
  load_encode();
  const int es = f32 ? 4 : 2;
  cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)D, (cuuint64_t)N};
  cuuint64_t strides[4] = {(cuuint64_t)C * es, (cuuint64_t)C * es * W, (cuuint64_t)C * es * W * H,
                           (cuuint64_t)C * es * W * H * D};
  cuuint32_t box[5] = {(cuuint32_t)(128 / es), (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bd, (cuuint32_t)bn};
  cuuint32_t ess[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                        const_cast<void *>(base), dims, strides, box, ess, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(RN_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed: " + std::to_string(r));
}

void make_w_map(CUtensorMap *m, const void *base, int rows, int64_t ktot, int bn) {
  if (g_dry_need) return;
  load_encode();
  cuuint64_t dims[2] = {(cuuint64_t)ktot, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ktot * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)bn};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(RN_ERR_CUDA, "cuTensorMapEncodeTiled (weights) failed: " + std::to_string(r));
}

namespace {

// choose a 128-voxel box (bw, bh, bd, bn) minimising the padded volume
void choose_box(int W, int H, int D, int N, int &bw, int &bh, int &bd, int &bn) {
  double best = 1e30;
  for (int a = 1; a <= 128; a *= 2)
    for (int b = 1; a * b <= 128; b *= 2)
      for (int c = 1; a * b * c <= 128; c *= 2) {
        int e = 128 / (a * b * c);
        if (a * b * c * e != 128) continue;
        double pad = (double)((W + a - 1) / a * a) * ((H + b - 1) / b * b) * ((D + c - 1) / c * c) *
                     ((N + e - 1) / e * e);
        // prefer wider w (contiguous rows) on ties
        double score = pad * (1.0 + 1e-6 * (8 - std::min(a, 8)));
        if (score < best) { best = score; bw = a; bh = b; bd = c; bn = e; }
      }
}

thread_local int g_pair_force = -1;  // rn_op_conv3d impl 2 / 5 (kernel tests)
int tc_pair_mode() {  // RN_TC_PAIR: 0 off, 1 every eligible launch, 2 (default) launches without split-K
  static const int m = getenv("RN_TC_PAIR") ? atoi(getenv("RN_TC_PAIR")) : 2;
  return g_pair_force >= 0 ? g_pair_force : m;
}

bool tma_store_off() {
  static const bool off = getenv("RN_TC_TMA_STORE") && atoi(getenv("RN_TC_TMA_STORE")) == 0;
  return off;
}

unsigned long long *g_trace = nullptr;
int g_trace_n = 0;
int g_trace_meta[256][8];

template <int BN, int STAGES>
int launch(const TcParams &p0, cudaStream_t st) {
  TcParams p = p0;
  p.trace = nullptr;
  using S = Smem<BN, STAGES>;
  static uint64_t attr_devs = 0;  // kernel attributes are per device
  if (!once_on_device(attr_devs)) {
    CUDA_CHECK(cudaFuncSetAttribute(conv_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    S::TOTAL));
    // the whole unified L1/smem as shared memory: the 96 KB-ring variants fit two
    // CTAs per SM only with the maximum carveout (the default gave 1 CTA per SM)
    CUDA_CHECK(cudaFuncSetAttribute(conv_tc_kernel<BN, STAGES>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared));
      }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // resident CTAs per SM: smem and TMEM (2*BN columns each, 512 per SM) permitting
  static int per_sm = 0;
  if (!per_sm) {
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_tc_kernel<BN, STAGES>,
                                                             tc_threads<BN, STAGES>(),
                                                             S::TOTAL));
    // the 96 KB-ring variants are compiled for 2 CTAs per SM (launch bounds) and two
    // fit in smem (2 x 101 KB of 228 KB); the occupancy query reports 1 for them
    // (measured), which left half of every SM idle in the epilogue-heavy launches
    const int by_smem = (int)(232448 / (S::TOTAL + 1024));
    const int by_bounds = (STAGES * S::STAGE > 110 * 1024) ? 1 : 2;
    per_sm = std::max(per_sm, std::min(by_smem, by_bounds));
    per_sm = std::max(1, std::min(per_sm, 512 / (2 * BN)));
  }
  const int grid = (int)std::min<int64_t>(p.cls_item0[p.n_cls], (int64_t)sms * per_sm);
  // TMA-store epilogue: every CTA owns at most one item (the ring is idle at its
  // epilogue and doubles as the staging buffer) and the tile fits the ring
  const int stg_bytes = p.use_part ? 128 * BN * 4 : tma_epi_bytes(BN, p.res != nullptr, p.st.mode);
  p.tma_st = (p.tma_ok && p.n_cls == 1 && p.cls_item0[p.n_cls] <= grid && stg_bytes <= STAGES * S::STAGE &&
              !tma_store_off())
                 ? (p.use_part ? 2 : 1)
                 : 0;
  if (getenv("RN_TC_TRACE") && g_trace_n < 256) {
    if (!g_trace) CUDA_CHECK(cudaMalloc(&g_trace, sizeof(unsigned long long) * 256 * 296 * 8));
    p.trace = g_trace + (size_t)g_trace_n * 296 * 8;
    int *m = g_trace_meta[g_trace_n++];
    m[0] = BN; m[1] = STAGES; m[2] = grid; m[3] = (int)p.cls_item0[p.n_cls]; m[4] = p.ksplit; m[5] = p.n_cls;
    m[6] = p.use_part; m[7] = p.n_taps * p.kblocks_per_tap;
  }
  if (getenv("RN_DEBUG_GRID"))
    fprintf(stderr, "conv_tc<%d,%d> items %lld per_sm %d grid %d smem %d\n", BN, STAGES,
            (long long)p.cls_item0[p.n_cls], per_sm, grid, S::TOTAL);
  launch_k(conv_tc_kernel<BN, STAGES>, grid, tc_threads<BN, STAGES>(), S::TOTAL, st, p);
  LAUNCH_CHECK();
  return grid;
}

// CTA-pair launch (cluster of 2, cta_group::2): one pair per 2 SMs, persistent over
// the pair items; a pair's two CTAs own M-tiles 2j, 2j+1 of the same (N-block, split)
template <int BN, int STAGES>
int launch_pair(const TcParams &p0, cudaStream_t st) {
  TcParams p = p0;
  p.trace = nullptr;
  using S = Smem<BN, STAGES, true>;
  static uint64_t attr_devs = 0;
  if (!once_on_device(attr_devs)) {
    CUDA_CHECK(cudaFuncSetAttribute(conv_tc_kernel<BN, STAGES, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    S::TOTAL));
    CUDA_CHECK(cudaFuncSetAttribute(conv_tc_kernel<BN, STAGES, true>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = p.cls_item0[1];
  const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(items, sms / 2));
  const int grid = 2 * pairs;
  const int stg_bytes = p.use_part ? 128 * BN * 4 : tma_epi_bytes(BN, p.res != nullptr, p.st.mode);
  p.tma_st = (p.tma_ok && items <= pairs && stg_bytes <= STAGES * S::STAGE && !tma_store_off())
                 ? (p.use_part ? 2 : 1)
                 : 0;
  if (getenv("RN_TC_TRACE") && g_trace_n < 256) {
    if (!g_trace) CUDA_CHECK(cudaMalloc(&g_trace, sizeof(unsigned long long) * 256 * 296 * 8));
    p.trace = g_trace + (size_t)g_trace_n * 296 * 8;
    int *m = g_trace_meta[g_trace_n++];
    m[0] = BN; m[1] = -STAGES; m[2] = grid; m[3] = (int)items; m[4] = p.ksplit; m[5] = p.n_cls;
    m[6] = p.use_part; m[7] = p.n_taps * p.kblocks_per_tap;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tc_threads<BN, STAGES, true>());
  cfg.dynamicSmemBytes = S::TOTAL;
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
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, conv_tc_kernel<BN, STAGES, true>, p));
  LAUNCH_CHECK();
  return grid;
}

// split-K finish: out = sum_s part[s] (+bias) (+existing) (+res*(mask>0)), bf16 store through the view
// split-K finish: out = sum_s part[s] (+bias) (+existing) (+res*(mask>0)), bf16 store
// through the view; the partials of 8 splits are loaded per batch (summed in split
// order).  With statistics (st.mode) each thread keeps a fixed 8-channel group (the
// grid stride is a multiple of ych/8) and the block writes one BN-statistics
// partial [2][ych] of the values it stored (fixed-order smem reduction).
__global__ void __launch_bounds__(512) splitk_finish_k(const float *__restrict__ part, int ks, int64_t nvv, int ych,
                                                       int OW, int OH, int OD, bf16 *__restrict__ y, int64_t s_n,
                                                       int64_t s_d, int64_t s_h, int64_t s_w,
                                                       const float *__restrict__ bias, int accumulate,
                                                       const bf16 *__restrict__ res,
                                                       const bf16 *__restrict__ res_mask, EpiStats st) {
  extern __shared__ float fred[];  // [2][blockDim][8] when st.mode
  pdl_begin();
  const int G = ych / 8;
  const int64_t n = nvv * G;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float a1[8], a2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a1[j] = a2[j] = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int c0 = (int)(i % G) * 8;
    const int64_t vidx = i / G;
    int64_t r = vidx;
    const int ow = (int)(r % OW); r /= OW;
    const int oh = (int)(r % OH); r /= OH;
    const int od = (int)(r % OD); r /= OD;
    const int on = (int)r;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = 0.f;
    for (int s0 = 0; s0 < ks; s0 += 8) {
      float4 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < ks) {
          const float *src = part + ((int64_t)(s0 + u) * nvv + vidx) * ych + c0;
          a[u] = *reinterpret_cast<const float4 *>(src);
          b[u] = *reinterpret_cast<const float4 *>(src + 4);
        }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < ks) {
          f[0] += a[u].x; f[1] += a[u].y; f[2] += a[u].z; f[3] += a[u].w;
          f[4] += b[u].x; f[5] += b[u].y; f[6] += b[u].z; f[7] += b[u].w;
        }
    }
    if (bias)
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += bias[c0 + j];
    const int64_t o = on * s_n + od * s_d + oh * s_h + ow * s_w + c0;
    if (accumulate) {
      float e[8];
      load_vec(y + o, e);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += e[j];
    }
    if (res) {
      float rv[8], mv[8];
      load_vec(res + o, rv);
      load_vec(res_mask + o, mv);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += mv[j] > 0.f ? rv[j] : 0.f;
    }
    store_vec(y + o, f);
    if (st.mode) {
      float m[8], h[8];
      if (st.mode >= 2) {
        load_vec(st.h + o, h);
        if (st.mode == 2) load_vec(st.mask + o, m);
        else
#pragma unroll
          for (int j = 0; j < 8; ++j) m[j] = fmaf(h[j], st.mscale[c0 + j], st.mshift[c0 + j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float q = __bfloat162float(__float2bfloat16_rn(f[j]));
        if (st.mode == 1) {
          a1[j] += q;
          a2[j] = fmaf(q, q, a2[j]);
        } else {
          const float d = m[j] > 0.f ? q : 0.f;
          a1[j] += d;
          a2[j] = fmaf(d, h[j] - st.mean[c0 + j], a2[j]);
        }
      }
    }
  }
  if (!st.mode) return;
  const int nt = blockDim.x;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    fred[threadIdx.x * 8 + j] = a1[j];
    fred[(nt + threadIdx.x) * 8 + j] = a2[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ych; c += nt) {  // threads t == c/8 (mod G) own channel c: fixed order
    float x1 = 0.f, x2 = 0.f;
    for (int tt = c >> 3; tt < nt; tt += G) {
      x1 += fred[tt * 8 + (c & 7)];
      x2 += fred[(nt + tt) * 8 + (c & 7)];
    }
    st.part[(int64_t)blockIdx.x * 2 * ych + c] = x1;
    st.part[(int64_t)blockIdx.x * 2 * ych + ych + c] = x2;
  }
}

// finish of a stride-2 dgrad launched as parity classes: every voxel v of dx
// (contiguous NDHWC) belongs to the class of its parity; its value is the sum of
// that class's split partials at the coarse voxel (v / 2) (zero for a parity no
// tap reaches), then accumulate / masked residual / statistics as splitk_finish_k
struct ClsFin {
  int slot[8];        // parity (pd*2+ph)*2+pw -> class index, -1: no tap reaches it
  int ks[8];          // splits of the class
  int64_t pbase[8];   // partial base of the class (floats)
};
__global__ void __launch_bounds__(512) splitk_finish_cls_k(const float *__restrict__ part, ClsFin cf, int64_t nvv,
                                                           int ych, int OW, int OH, int OD, int Wi, int Hi, int Di,
                                                           int64_t nvox, bf16 *__restrict__ y, int accumulate,
                                                           const bf16 *__restrict__ res,
                                                           const bf16 *__restrict__ res_mask, EpiStats st) {
  extern __shared__ float fred[];  // [2][blockDim][8] when st.mode
  pdl_begin();
  const int G = ych / 8;
  const int64_t n = nvox * G;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float a1[8], a2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a1[j] = a2[j] = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int c0 = (int)(i % G) * 8;
    const int64_t v = i / G;
    int64_t r = v;
    const int w = (int)(r % Wi); r /= Wi;
    const int h = (int)(r % Hi); r /= Hi;
    const int d = (int)(r % Di); r /= Di;
    const int nn = (int)r;
    const int slot = cf.slot[((d & 1) * 2 + (h & 1)) * 2 + (w & 1)];
    const int ks = slot < 0 ? 0 : cf.ks[slot];
    const float *src0 = part + (slot < 0 ? 0 : cf.pbase[slot]) +
                        ((((int64_t)nn * OD + (d >> 1)) * OH + (h >> 1)) * OW + (w >> 1)) * ych + c0;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = 0.f;
    for (int s0 = 0; s0 < ks; s0 += 8) {
      float4 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < ks) {
          const float *src = src0 + (int64_t)(s0 + u) * nvv * ych;
          a[u] = *reinterpret_cast<const float4 *>(src);
          b[u] = *reinterpret_cast<const float4 *>(src + 4);
        }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < ks) {
          f[0] += a[u].x; f[1] += a[u].y; f[2] += a[u].z; f[3] += a[u].w;
          f[4] += b[u].x; f[5] += b[u].y; f[6] += b[u].z; f[7] += b[u].w;
        }
    }
    const int64_t o = v * ych + c0;
    if (accumulate) {
      float e[8];
      load_vec(y + o, e);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += e[j];
    }
    if (res) {
      float rv[8], mv[8];
      load_vec(res + o, rv);
      load_vec(res_mask + o, mv);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += mv[j] > 0.f ? rv[j] : 0.f;
    }
    store_vec(y + o, f);
    if (st.mode) {
      float m[8], hh[8];
      if (st.mode >= 2) {
        load_vec(st.h + o, hh);
        if (st.mode == 2) load_vec(st.mask + o, m);
        else
#pragma unroll
          for (int j = 0; j < 8; ++j) m[j] = fmaf(hh[j], st.mscale[c0 + j], st.mshift[c0 + j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float q = __bfloat162float(__float2bfloat16_rn(f[j]));
        if (st.mode == 1) {
          a1[j] += q;
          a2[j] = fmaf(q, q, a2[j]);
        } else {
          const float dd = m[j] > 0.f ? q : 0.f;
          a1[j] += dd;
          a2[j] = fmaf(dd, hh[j] - st.mean[c0 + j], a2[j]);
        }
      }
    }
  }
  if (!st.mode) return;
  const int nt = blockDim.x;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    fred[threadIdx.x * 8 + j] = a1[j];
    fred[(nt + threadIdx.x) * 8 + j] = a2[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ych; c += nt) {  // threads t == c/8 (mod G) own channel c: fixed order
    float x1 = 0.f, x2 = 0.f;
    for (int tt = c >> 3; tt < nt; tt += G) {
      x1 += fred[tt * 8 + (c & 7)];
      x2 += fred[(nt + tt) * 8 + (c & 7)];
    }
    st.part[(int64_t)blockIdx.x * 2 * ych + c] = x1;
    st.part[(int64_t)blockIdx.x * 2 * ych + ych + c] = x2;
  }
}

// split-K factor for launches with fewer tiles than SMs: as many splits as fit
// in ONE wave of 148 CTAs (rounding up leaves a few CTAs with two items and
// doubles the launch time)
int choose_ksplit(int64_t n_tiles, int nk) {
  if (n_tiles >= 100) return 1;
  int ks = (int)(148 / std::max<int64_t>(n_tiles, 1));
  ks = std::min(ks, nk / 4);
  return std::max(ks, 1);
}

// one class covering the whole launch (every launch but the stride-2 dgrad)
void one_class(TcParams &p) {
  p.n_cls = 1;
  p.cls_item0[0] = 0;
  p.cls_item0[1] = p.n_tiles * p.ksplit;
  p.cls_ks[0] = p.ksplit;
  p.cls_tap0[0] = 0;
  p.cls_ntaps[0] = p.n_taps;
  p.cls_OW[0] = p.OW; p.cls_OH[0] = p.OH; p.cls_OD[0] = p.OD;
  p.cls_yoff[0] = 0;
  p.cls_pbase[0] = 0;
  p.use_part = p.ksplit > 1;
}

// The TMA ring must hold ~latency x bandwidth (measured ~1600 cycles x ~85 B/clk
// per SM from L2): launches with more work items than SMs run two CTAs per SM
// (two rings of 96 KB); launches with at most one item per SM run one CTA with
// a 192 KB ring (a 96 KB ring measured latency-bound: 29 us vs ~15 us)
int launch_ring(const TcParams &p, int BN, cudaStream_t st) {
  const bool one_wave = p.cls_item0[p.n_cls] <= 148;
  if (BN == 64) return one_wave ? launch<64, 8>(p, st) : launch<64, 4>(p, st);
  if (BN == 128) return one_wave ? launch<128, 6>(p, st) : launch<128, 3>(p, st);
  return launch<256, 4>(p, st);
}

// returns the number of BN-statistics partials written (0: statistics not fused)
int run(TcParams &p, int BN, float *ws, size_t ws_floats, const EpiStats *est, cudaStream_t st) {
  const int nk = p.n_taps * p.kblocks_per_tap;
  p.n_view_vox = (int64_t)p.ON * p.OD * p.OH * p.OW;
  p.ksplit = choose_ksplit(p.n_tiles, nk);
  if (g_dry_need) {
    if (p.ksplit > 1) *g_dry_need = std::max(*g_dry_need, (size_t)p.ksplit * p.n_view_vox * p.ych);
    return 0;
  }
  if (!ws || (size_t)p.ksplit * p.n_view_vox * p.ych > ws_floats) p.ksplit = 1;
  p.part = ws;
  one_class(p);
  // fused statistics: whole-K tiles covering every output channel in the conv
  // epilogue, or the split-K finish kernel (which sees whole rows)
  const bool stats = est && est->mode && p.ksplit == 1 && p.t_nblk == 1;
  const bool fin_stats = est && est->mode && p.ksplit > 1;
  if (stats) p.st = *est;
  // TMA-store epilogue maps (used when every CTA owns one item; decided at launch):
  // split-K partials always (the finish kernel applies bias / accumulate / residual),
  // direct bf16 output without accumulate / residual; aligned views only
  const bool aligned = ((uintptr_t)p.y % 16 == 0) && ((uintptr_t)ws % 16 == 0);
  if (aligned && p.ksplit > 1 && p.ON % p.bn == 0) {
    make_out_map(&p.part_map, ws, true, p.ych, p.OW, p.OH, p.OD, p.ON * p.ksplit, p.bw, p.bh, p.bd, p.bn);
    p.tma_ok = 1;
  } else if (aligned && p.ksplit == 1 && (!p.res || ((uintptr_t)p.res % 16 == 0 && (uintptr_t)p.res_mask % 16 == 0))) {
    make_out_map(&p.y_map, p.y, false, p.ych, p.OW, p.OH, p.OD, p.ON, p.bw, p.bh, p.bd, p.bn);
    if (p.res) {
      make_out_map(&p.res_map, p.res, false, p.ych, p.OW, p.OH, p.OD, p.ON, p.bw, p.bh, p.bd, p.bn);
      make_out_map(&p.resm_map, p.res_mask, false, p.ych, p.OW, p.OH, p.OD, p.ON, p.bw, p.bh, p.bd, p.bn);
    }
    if (p.st.mode >= 2) make_out_map(&p.h_map, p.st.h, false, p.ych, p.OW, p.OH, p.OD, p.ON, p.bw, p.bh, p.bd, p.bn);
    if (p.st.mode == 2)
      make_out_map(&p.m_map, p.st.mask, false, p.ych, p.OW, p.OH, p.OD, p.ON, p.bw, p.bh, p.bd, p.bn);
    p.tma_ok = 1;
  }
  int grid;
  // CTA pairs for the one-class launches with N tiles of 128 / 256 (stage 2-4 3x3x3
  // and stride-2 convs): M=256 MMAs, half of B per CTA (RN_TC_PAIR=0 turns them off)
  const int64_t n_mt = p.n_tiles / p.t_nblk;
  if (tc_pair_mode() && (tc_pair_mode() == 1 || p.ksplit == 1) && p.n_cls == 1 && (BN == 128 || BN == 256) &&
      n_mt >= 2 && p.w_base) {
    p.pair = 1;
    p.n_mt = n_mt;
    p.cls_item0[1] = (n_mt + 1) / 2 * p.t_nblk * p.ksplit;
    make_w_map(&p.b_map, p.w_base, p.w_rows, p.w_ktot, BN / 2);
    grid = BN == 256 ? launch_pair<256, 6>(p, st) : launch_pair<128, 8>(p, st);
  } else {
    grid = launch_ring(p, BN, st);
  }
  if (p.ksplit > 1) {
    const int64_t n = p.n_view_vox * (p.ych / 8);
    // with statistics: <= 148 blocks (the partial count), stride a multiple of ych/8
    const unsigned fg = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 511) / 512, fin_stats ? 148 : 148 * 8));
    EpiStats fst;
    if (fin_stats) fst = *est;
    launch_k(splitk_finish_k, fg, 512, fin_stats ? (size_t)2 * 512 * 8 * sizeof(float) : 0, st, ws, p.ksplit,
             p.n_view_vox, p.ych, p.OW, p.OH, p.OD, p.y, p.s_n, p.s_d, p.s_h, p.s_w, p.bias, p.accumulate, p.res,
             p.res_mask, fst);
    LAUNCH_CHECK();
    if (fin_stats) return (int)fg;
  }
  return stats ? grid : 0;
}

// Largest N tile dividing nout, halved while the launch has fewer tiles than
// SMs (small late-stage layers trade MMA width for parallelism before split-K).
int pick_bn(int nout, int OW, int OH, int OD, int ON, int mult = 1, int kblocks = 1 << 20) {
  int bw, bh, bd, bn;
  choose_box(OW, OH, OD, ON, bw, bh, bd, bn);
  const int64_t mt = (int64_t)((OW + bw - 1) / bw) * ((OH + bh - 1) / bh) * ((OD + bd - 1) / bd) * ((ON + bn - 1) / bn);
  int BN = nout % 256 == 0 ? 256 : nout % 128 == 0 ? 128 : 64;
  // halving BN for small layers measured slower overall (more A re-reads): only
  // when even split-K cannot fill the machine (fewer than 16 tiles) -- or when K
  // is too short to split (1x1x1 convs, <= 8 K-blocks): there the A re-read is
  // cheap and narrower tiles are the only source of parallelism
  const int64_t want = kblocks <= 8 ? 148 : 16;
  while (BN > 64 && mt * mult * (nout / BN) < want) BN /= 2;
  return BN;
}

void fill_tiles(TcParams &p, int OW, int OH, int OD, int ON, int nout, int BN) {
  p.OW = OW; p.OH = OH; p.OD = OD; p.ON = ON;
  choose_box(OW, OH, OD, ON, p.bw, p.bh, p.bd, p.bn);
  p.tw = (OW + p.bw - 1) / p.bw;
  p.th = (OH + p.bh - 1) / p.bh;
  p.td = (OD + p.bd - 1) / p.bd;
  p.tn = (ON + p.bn - 1) / p.bn;
  p.t_nblk = nout / BN;
  p.n_tiles = (int64_t)p.tn * p.td * p.th * p.tw * p.t_nblk;
}

}  // namespace

void tc_pair_force(int mode) { g_pair_force = mode; }

bool tc_conv_supported(const ConvGeom &g, bool dgrad) {
  const int kc = dgrad ? g.Co : g.Ci;     // A channels
  const int nout = dgrad ? g.Ci : g.Co;   // output channels
  if (kc % 64 != 0 || nout % 64 != 0) return false;
  if (g.k != 1 && g.k != 3) return false;
  if (g.s != 1 && g.s != 2) return false;
  if (g.k == 3 && g.p != 1) return false;
  if (g.k == 1 && g.p != 0) return false;
  if (g.s == 2) {  // output = ceil(in/2) lattice, every parity sub-lattice non-empty
    if (g.Do != (g.Di + 1) / 2 || g.Ho != (g.Hi + 1) / 2 || g.Wo != (g.Wi + 1) / 2) return false;
    if (g.Di < 2 || g.Hi < 2 || g.Wi < 2) return false;
  }
  return true;
}

// fprop: y[vo][co] = sum x[...] w[co][tap][ci] (+bias)
int conv_fprop_tc(const ConvGeom &g, const bf16 *x, const bf16 *w, const float *bias, bf16 *y, float *ws,
                  size_t ws_floats, cudaStream_t st, const EpiStats *est) {
  TcParams p;
  memset(&p, 0, sizeof p);
  const int BN = pick_bn(g.Co, g.Wo, g.Ho, g.Do, g.N, 1, g.taps() * g.Ci / 64);
  fill_tiles(p, g.Wo, g.Ho, g.Do, g.N, g.Co, BN);
  const int taps = g.taps();
  p.n_taps = taps;
  p.kblocks_per_tap = g.Ci / 64;
  if (g.s == 1) {
    make_act_map(&p.a_map[0], x, g.Ci, g.Wi, g.Hi, g.Di, g.N, 1, g.Wi, (int64_t)g.Wi * g.Hi,
                 (int64_t)g.Wi * g.Hi * g.Di, p.bw, p.bh, p.bd, p.bn);
  } else {
    // 8 parity sub-lattices: map index = (pd*2 + ph)*2 + pw ; base offset by the parity voxel
    for (int pd = 0; pd < 2; ++pd)
      for (int ph = 0; ph < 2; ++ph)
        for (int pw = 0; pw < 2; ++pw) {
          const int Wv = (g.Wi - pw + 1) / 2, Hv = (g.Hi - ph + 1) / 2, Dv = (g.Di - pd + 1) / 2;
          const bf16 *b = x + (((int64_t)pd * g.Hi + ph) * g.Wi + pw) * g.Ci;
          make_act_map(&p.a_map[(pd * 2 + ph) * 2 + pw], b, g.Ci, std::max(Wv, 1), std::max(Hv, 1), std::max(Dv, 1),
                       g.N, 2, 2LL * g.Wi, 2LL * g.Wi * g.Hi, (int64_t)g.Wi * g.Hi * g.Di, p.bw, p.bh, p.bd, p.bn);
        }
  }
  for (int t = 0; t < taps; ++t) {
    const int kd = t / (g.k * g.k), kh = (t / g.k) % g.k, kw = t % g.k;
    const int od = kd - g.p, oh = kh - g.p, ow = kw - g.p;  // input offset = s*o + (k - p)
    if (g.s == 1) {
      p.tap_map[t] = 0;
      p.tap_od[t] = od; p.tap_oh[t] = oh; p.tap_ow[t] = ow;
    } else {
      // i = 2o + off: off = 0 -> even lattice at o; off = 1 -> odd at o; off = -1 -> odd at o-1
      auto par = [](int off) { return off == 0 ? 0 : 1; };
      auto sh = [](int off) { return off < 0 ? -1 : 0; };
      p.tap_map[t] = (par(od) * 2 + par(oh)) * 2 + par(ow);
      p.tap_od[t] = sh(od); p.tap_oh[t] = sh(oh); p.tap_ow[t] = sh(ow);
    }
    p.tap_kcoord[t] = t * g.Ci;
  }
  make_w_map(&p.b_map, w, g.Co, (int64_t)taps * g.Ci, BN);
  p.w_base = w; p.w_rows = g.Co; p.w_ktot = (int64_t)taps * g.Ci;
  p.y = y;
  p.ych = g.Co;
  p.s_w = g.Co;
  p.s_h = (int64_t)g.Wo * g.Co;
  p.s_d = (int64_t)g.Ho * g.Wo * g.Co;
  p.s_n = (int64_t)g.Do * g.Ho * g.Wo * g.Co;
  p.bias = bias;
  return run(p, BN, ws, ws_floats, est, st);
}

// dgrad: dx[vi][ci] (=|+=) sum dy[vo][co] W[co][tap][ci]; wd = [ci][taps-1-tap][co]
int conv_dgrad_tc(const ConvGeom &g, const bf16 *dy, const bf16 *wd, bf16 *dx, bool accumulate, const bf16 *res,
                  const bf16 *res_mask, float *ws, size_t ws_floats, cudaStream_t st, const EpiStats *est,
                  const bf16 *dy2, const bf16 *wd2) {
  if (dy2 && !(g.s == 2 && g.k == 3)) throw Error(RN_ERR_ARG, "conv_dgrad_tc: projection merge needs a k3 s2 conv");
  const int taps = g.taps();
  if (g.s == 1) {
    const int BN = pick_bn(g.Ci, g.Wi, g.Hi, g.Di, g.N, 1, g.taps() * g.Co / 64);
    TcParams p;
    memset(&p, 0, sizeof p);
    fill_tiles(p, g.Wi, g.Hi, g.Di, g.N, g.Ci, BN);
    p.n_taps = taps;
    p.kblocks_per_tap = g.Co / 64;
    make_act_map(&p.a_map[0], dy, g.Co, g.Wo, g.Ho, g.Do, g.N, 1, g.Wo, (int64_t)g.Wo * g.Ho,
                 (int64_t)g.Wo * g.Ho * g.Do, p.bw, p.bh, p.bd, p.bn);
    for (int t = 0; t < taps; ++t) {
      // dx[i] = sum_t dy[i + p - k_t] W[t]  ==  sum_t' dy[i + k_t' - p] Wflip[t'] with t' = taps-1-t
      const int kd = t / (g.k * g.k), kh = (t / g.k) % g.k, kw = t % g.k;
      p.tap_map[t] = 0;
      p.tap_od[t] = kd - g.p; p.tap_oh[t] = kh - g.p; p.tap_ow[t] = kw - g.p;
      p.tap_kcoord[t] = t * g.Co;  // wd row layout [ci][t'][co] indexed by t' = t here
    }
    make_w_map(&p.b_map, wd, g.Ci, (int64_t)taps * g.Co, BN);
    p.w_base = wd; p.w_rows = g.Ci; p.w_ktot = (int64_t)taps * g.Co;
    p.y = dx;
    p.ych = g.Ci;
    p.s_w = g.Ci;
    p.s_h = (int64_t)g.Wi * g.Ci;
    p.s_d = (int64_t)g.Hi * g.Wi * g.Ci;
    p.s_n = (int64_t)g.Di * g.Hi * g.Wi * g.Ci;
    p.accumulate = accumulate;
    p.res = res;
    p.res_mask = res_mask;
    return run(p, BN, ws, ws_floats, est, st);
  }
  // stride 2: output parity classes (pd, ph, pw); input index i = 2a + par.
  // Contributions: i = 2o + k - p  =>  for k=3,p=1: par 0 <- (k=1, o=a); par 1 <- (k=2, o=a), (k=0, o=a+1)
  //                                    for k=1,p=0: par 0 <- (k=0, o=a); par 1 <- none
  // All classes run in ONE launch over a common coarse tiling (extents of parity
  // 0, the largest); with dy2/wd2 the 1x1x1 stride-2 projection's dgrad is an
  // extra tap of class (0,0,0) reading A from dy2 and B from wd2.
  struct Cls { int par, nt; int8_t map[MAX_TAPS], bsel[MAX_TAPS], od[MAX_TAPS], oh[MAX_TAPS], ow[MAX_TAPS];
               int kc[MAX_TAPS]; };
  std::vector<Cls> cls;
  bool empty_class = false;
  for (int par = 0; par < 8; ++par) {
    const int pd = par >> 2, ph = (par >> 1) & 1, pw = par & 1;
    Cls c;
    memset(&c, 0, sizeof c);
    c.par = par;
    auto add_taps = [&](int k, int pad, int ntaps_w, int amap) {
      for (int t = 0; t < ntaps_w; ++t) {
        const int kk[3] = {t / (k * k), (t / k) % k, t % k};
        const int pp[3] = {pd, ph, pw};
        int off[3];
        bool ok = true;
        for (int q = 0; q < 3; ++q) {
          // need 2o + k - p = 2a' + par  ->  o = a' + (par + p - k)/2, integer
          const int num = pp[q] + pad - kk[q];
          if (num % 2 != 0) { ok = false; break; }
          off[q] = num / 2;
        }
        if (!ok) continue;
        c.map[c.nt] = (int8_t)amap;
        c.bsel[c.nt] = (int8_t)amap;
        c.od[c.nt] = off[0]; c.oh[c.nt] = off[1]; c.ow[c.nt] = off[2];
        c.kc[c.nt] = (ntaps_w - 1 - t) * g.Co;  // wd[ci][taps-1-t][co] == W[co][ci][t]
        ++c.nt;
      }
    };
    add_taps(g.k, g.p, taps, 0);
    if (dy2) add_taps(1, 0, 1, 1);
    if (c.nt == 0) { empty_class = true; continue; }
    cls.push_back(c);
  }
  std::stable_sort(cls.begin(), cls.end(), [](const Cls &x, const Cls &y) { return x.nt > y.nt; });
  const int Wv0 = (g.Wi + 1) / 2, Hv0 = (g.Hi + 1) / 2, Dv0 = (g.Di + 1) / 2;
  const int BN = pick_bn(g.Ci, Wv0, Hv0, Dv0, g.N, (int)cls.size());
  TcParams p;
  memset(&p, 0, sizeof p);
  fill_tiles(p, Wv0, Hv0, Dv0, g.N, g.Ci, BN);
  p.kblocks_per_tap = g.Co / 64;
  p.n_view_vox = (int64_t)p.ON * p.OD * p.OH * p.OW;
  // split-K per class in proportion to its K (uniform item cost), one wave in total
  const int ncls = (int)cls.size();
  int64_t kwork = 0;
  for (const Cls &c : cls) kwork += p.n_tiles * c.nt * p.kblocks_per_tap;
  const bool split = p.n_tiles * ncls < 100;
  const int64_t chunk = std::max<int64_t>(4, (kwork + 147) / 148);
  p.n_cls = ncls;
  p.n_taps = 0;
  int64_t items = 0, pfl = 0;
  for (int ci = 0; ci < ncls; ++ci) {
    const Cls &c = cls[ci];
    const int nk = c.nt * p.kblocks_per_tap;
    const int ks = split ? (int)std::max<int64_t>(1, std::min<int64_t>(nk, nk / chunk)) : 1;
    const int pd = c.par >> 2, ph = (c.par >> 1) & 1, pw = c.par & 1;
    p.cls_item0[ci] = items;
    p.cls_ks[ci] = ks;
    p.cls_tap0[ci] = p.n_taps;
    p.cls_ntaps[ci] = c.nt;
    p.cls_OW[ci] = (g.Wi - pw + 1) / 2; p.cls_OH[ci] = (g.Hi - ph + 1) / 2; p.cls_OD[ci] = (g.Di - pd + 1) / 2;
    p.cls_yoff[ci] = (((int64_t)pd * g.Hi + ph) * g.Wi + pw) * g.Ci;
    p.cls_pbase[ci] = pfl;
    for (int t = 0; t < c.nt; ++t) {
      const int j = p.n_taps++;
      p.tap_map[j] = c.map[t]; p.tap_bsel[j] = c.bsel[t];
      p.tap_od[j] = c.od[t]; p.tap_oh[j] = c.oh[t]; p.tap_ow[j] = c.ow[t];
      p.tap_kcoord[j] = c.kc[t];
    }
    items += p.n_tiles * ks;
    pfl += (int64_t)ks * p.n_view_vox * g.Ci;
  }
  p.cls_item0[ncls] = items;
  // partial mode (finish kernel): split launches, and launches with a parity no
  // tap reaches (the finish writes every voxel of dx)
  p.use_part = split || empty_class;
  p.ych = g.Ci;
  if (g_dry_need) {
    if (p.use_part) *g_dry_need = std::max(*g_dry_need, (size_t)pfl);
    return 0;
  }
  if (p.use_part && (!ws || (size_t)pfl > ws_floats))
    throw Error(RN_ERR_STATE, "conv_dgrad_tc: stride-2 split-K workspace too small");
  if (!p.use_part && empty_class && !accumulate)
    throw Error(RN_ERR_STATE, "conv_dgrad_tc: empty parity class needs accumulate");
  p.ksplit = p.use_part ? 2 : 1;
  p.part = ws;
  make_act_map(&p.a_map[0], dy, g.Co, g.Wo, g.Ho, g.Do, g.N, 1, g.Wo, (int64_t)g.Wo * g.Ho,
               (int64_t)g.Wo * g.Ho * g.Do, p.bw, p.bh, p.bd, p.bn);
  make_w_map(&p.b_map, wd, g.Ci, (int64_t)taps * g.Co, BN);
  if (dy2) {
    make_act_map(&p.a_map[1], dy2, g.Co, g.Wo, g.Ho, g.Do, g.N, 1, g.Wo, (int64_t)g.Wo * g.Ho,
                 (int64_t)g.Wo * g.Ho * g.Do, p.bw, p.bh, p.bd, p.bn);
    make_w_map(&p.b_map2, wd2, g.Ci, (int64_t)g.Co, BN);
  }
  // strided output views: class voxel (a_d, a_h, a_w) -> (2a_d+pd, 2a_h+ph, 2a_w+pw)
  p.y = dx;
  p.s_w = 2LL * g.Ci;
  p.s_h = 2LL * g.Wi * g.Ci;
  p.s_d = 2LL * g.Hi * g.Wi * g.Ci;
  p.s_n = (int64_t)g.Di * g.Hi * g.Wi * g.Ci;
  p.accumulate = accumulate;
  p.res = res;
  p.res_mask = res_mask;
  const bool stats = est && est->mode && !p.use_part && p.t_nblk == 1;
  const bool fin_stats = est && est->mode && p.use_part;
  if (stats) p.st = *est;
  const int grid = launch_ring(p, BN, st);
  if (!p.use_part) return stats ? grid : 0;
  ClsFin cf;
  for (int q = 0; q < 8; ++q) cf.slot[q] = -1;
  for (int ci = 0; ci < ncls; ++ci) {
    cf.slot[cls[ci].par] = ci;
    cf.ks[ci] = p.cls_ks[ci];
    cf.pbase[ci] = p.cls_pbase[ci];
  }
  const int64_t nvox = (int64_t)g.N * g.Di * g.Hi * g.Wi;
  const int64_t n = nvox * (g.Ci / 8);
  const unsigned fg = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 511) / 512, fin_stats ? 148 : 148 * 8));
  EpiStats fst;
  if (fin_stats) fst = *est;
  launch_k(splitk_finish_cls_k, fg, 512, fin_stats ? (size_t)2 * 512 * 8 * sizeof(float) : 0, st, ws, cf,
           p.n_view_vox, g.Ci, p.OW, p.OH, p.OD, g.Wi, g.Hi, g.Di, nvox, dx, (int)accumulate, res, res_mask, fst);
  LAUNCH_CHECK();
  return fin_stats ? (int)fg : 0;
}

size_t tc_conv_ws_floats(const ConvGeom &g, bool dgrad) {
  size_t need = 0;
  g_dry_need = &need;
  try {
    if (!dgrad) conv_fprop_tc(g, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr);
    else {
      conv_dgrad_tc(g, nullptr, nullptr, nullptr, true, nullptr, nullptr, nullptr, 0, nullptr, nullptr);
      // the k3 stride-2 dgrad may run with the projection merged (a different split)
      static const bf16 dummy{};
      if (g.s == 2 && g.k == 3)
        conv_dgrad_tc(g, nullptr, nullptr, nullptr, true, nullptr, nullptr, nullptr, 0, nullptr, nullptr, &dummy,
                      &dummy);
    }
  } catch (...) {
    g_dry_need = nullptr;
    throw;
  }
  g_dry_need = nullptr;
  return need;
}

}  // namespace rn

// debug: the traced conv_tc launches (RN_TC_TRACE): host[l][cta][8] %globaltimer stamps,
// meta[l][8] = {BN, STAGES, grid, items, ksplit, n_cls, use_part, k-blocks}; returns the count
extern "C" int rn_dbg_tc_trace(unsigned long long *host, int max_launches, int *meta) {
  using namespace rn;
  const int n = std::min(g_trace_n, max_launches);
  if (n > 0 && g_trace) {
    cudaDeviceSynchronize();
    cudaMemcpy(host, g_trace, sizeof(unsigned long long) * (size_t)n * 296 * 8, cudaMemcpyDeviceToHost);
    memcpy(meta, g_trace_meta, sizeof(int) * 8 * n);
  }
  return n;
}
