// k_wgrad_tc.cu — convolution weight gradient on tcgen05 (the
// gradient of w_q by the chain rule; P:366 conv complexity).
//
//   dW[co][tap][ci] = sum_{voxels v} dy[v][co] * x[v + off(tap)][ci]
//
// GEMM per launch: D[(tap,ci) rows][co cols] = A^T B with K = output voxels:
//   A "atoms": 64-channel x-blocks shifted by a tap, [K voxels][64 ci] (MN-major, SW128)
//   B atoms  : dy 64-channel blocks, [K voxels][64 co] (MN-major, SW128)
// One M-tile = two A atoms (128 rows: two taps of a 64-channel input, or two
// 64-channel blocks of one tap).  Each CTA owns G M-tiles (G*BN <= 512 TMEM
// columns), one co block of BN, and a contiguous split of the voxel tiles;
// it writes fp32 partials [split][co][tap][ci] reduced in a fixed order
// (deterministic, reading X24).
//
// x staging: "haloed" mode (stride 1, k = 3, Ci = 64): one TMA box of
// (bw+2) x (bh+2) x (bd+2) voxels per voxel tile holds all 27 tap-shifted
// operands; each MMA's A descriptor points at the tap's 8-row groups inside it
// (uniform group stride = (bw+2)*128 B, base-offset field for the row phase).
// Otherwise ("per-tap" mode) every atom is its own TMA box (stride-2 convs use
// the parity sub-lattice tensor maps of k_conv_tc.cu).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "error.h"
#include "launch.h"
#include "kernels.h"
#include "tc_conv.h"
#include "tc_ptx.cuh"
#include "util.cuh"

namespace rn {

namespace {

constexpr int WG_THREADS = 192;
constexpr int MAX_ATOMS = 128;  // M-tiles per problem (2 atoms each)
constexpr int ATAB_MAX = 32;    // x atoms staged per CTA (per-tap mode: 2 G)

struct __align__(64) WgParams {
  CUtensorMap x_map[8];
  CUtensorMap dy_map;
  int haloed;
  int G;          // M-tiles per CTA (this launch's m-group size)
  int n_mgroups;  // CTA groups over M
  int n_cob;      // co blocks of BN
  int splits;
  int accum;  // splits == 1: part is dW itself and the epilogue accumulates
  int overwrite;  // with accum: store dW instead of adding (first contribution of a backward)
  // atoms of the whole problem: atom a = (tap, ci block); M-tile i = atoms 2i, 2i+1
  int n_mtiles;
  int8_t atom_map[2 * MAX_ATOMS];  // x map index (per-tap mode)
  int8_t atom_od[2 * MAX_ATOMS], atom_oh[2 * MAX_ATOMS], atom_ow[2 * MAX_ATOMS];
  int16_t atom_tap[2 * MAX_ATOMS];
  int8_t atom_cb[2 * MAX_ATOMS];
  int8_t atom_valid[2 * MAX_ATOMS];
  // voxel tiles of dy
  int bw, bh, bd, bn;
  int tw, th, td, tn;
  int64_t n_vtiles;
  int vt_per_split;
  // output partials
  float *part;  // [split][Co][taps][Ci]
  int Co, Ci, taps;
  int hw, hh, hd;  // haloed box extents
};

template <int BN>
struct WgSmem {
  static constexpr int DY_BYTES = (BN / 64) * 16384;
  static constexpr int X_MAX = 110 * 1024 - DY_BYTES;  // x bytes per stage (haloed region or atoms)
};

// one x atom's TMA coordinates, staged in smem for the producer (indexed
// kernel-parameter loads stall the single issuing thread)
struct __align__(16) AtomEnt {
  const CUtensorMap *map;
  int c;
  int8_t od, oh, ow, pad;
};

template <int BN, int STAGES, int XBYTES>
__global__ void __launch_bounds__(WG_THREADS, 1) wgrad_tc_kernel(const __grid_constant__ WgParams p) {
  constexpr int DYB = (BN / 64) * 16384;
  constexpr int STAGE = DYB + XBYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + STAGES * STAGE);
  uint64_t *empty = full + STAGES;
  uint64_t *done = empty + STAGES;
  uint32_t *tmem_slot = (uint32_t *)(done + 1);
  AtomEnt *atab = (AtomEnt *)(smem + STAGES * STAGE + 256);  // [2 * G]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  // CTA -> (m-group, co block, split)
  int b = blockIdx.x;
  const int mg = b % p.n_mgroups; b /= p.n_mgroups;
  const int cob = b % p.n_cob; b /= p.n_cob;
  const int split = b;
  const int mt0 = mg * p.G;
  const int G = min(p.G, p.n_mtiles - mt0);
  const int64_t vt0 = (int64_t)split * p.vt_per_split;
  const int64_t vt1 = min(p.n_vtiles, vt0 + p.vt_per_split);

  if (warp == 0 && !p.haloed)
    for (int a = lane; a < 2 * G; a += 32) {
      const int at = 2 * mt0 + a;
      AtomEnt e;
      e.map = &p.x_map[p.atom_map[at]];
      e.c = p.atom_cb[at] * 64;
      e.od = p.atom_od[at]; e.oh = p.atom_oh[at]; e.ow = p.atom_ow[at]; e.pad = 0;
      atab[a] = e;
    }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_begin();  // prologue above overlaps the predecessor's tail

  if (warp == 0) {
    if (lane == 0 && G > 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t vt = vt0; vt < vt1; ++vt) {
        int64_t r = vt;
        const int tw = (int)(r % p.tw); r /= p.tw;
        const int th = (int)(r % p.th); r /= p.th;
        const int td = (int)(r % p.td); r /= p.td;
        const int tn = (int)r;
        const int w0 = tw * p.bw, h0 = th * p.bh, d0 = td * p.bd, n0 = tn * p.bn;
        tc::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t *sdy = smem + stage * STAGE;
        uint8_t *sx = sdy + DYB;
        uint32_t bytes = DYB;
        if (p.haloed) bytes += p.hw * p.hh * p.hd * 128;
        else bytes += 2 * G * 16384;
        tc::mbar_arrive_expect_tx(&full[stage], bytes);
        for (int c = 0; c < BN / 64; ++c)
          tc::tma_load_5d(sdy + c * 16384, &p.dy_map, &full[stage], cob * BN + c * 64, w0, h0, d0, n0);
        if (p.haloed) {
          tc::tma_load_5d(sx, &p.x_map[0], &full[stage], 0, w0 - 1, h0 - 1, d0 - 1, n0);
        } else {
          for (int a = 0; a < 2 * G; ++a) {
            const AtomEnt e = atab[a];
            tc::tma_load_5d(sx + a * 16384, e.map, &full[stage], e.c, w0 + e.ow, h0 + e.oh, d0 + e.od, n0);
          }
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (G > 0 && p.haloed) {
      // Haloed x: every descriptor is precomputed — A of M-tile i at K-step j is
      // dA[i] (the two taps' rows at LBO distance) + goff[j] (the j-th pair of
      // 8-voxel row groups) + the stage offset; per MMA only an add remains
      // (the issue loop must sustain one MMA per ~48 cycles)
      constexpr uint32_t IDESC = tc::idesc_bf16(128, BN, 1, 1);
      const uint32_t sdy0 = tc::smem_u32(smem), sx0 = sdy0 + DYB;
      uint64_t dA[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        dA[i] = 0;
        if (i < G) {
          const int t0 = p.atom_tap[2 * (mt0 + i)], t1 = p.atom_tap[2 * (mt0 + i) + 1];
          const int r0 = ((t0 / 9) * p.hh + (t0 / 3) % 3) * p.hw + t0 % 3;
          const int r1 = ((t1 / 9) * p.hh + (t1 / 3) % 3) * p.hw + t1 % 3;
          dA[i] = tc::smem_desc(sx0 + r0 * 128, (r1 - r0) * 128, p.hw * 128, 2);
        }
      }
      uint32_t goff[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) goff[j] = (uint32_t)((((2 * j) / p.bh) * p.hh + (2 * j) % p.bh) * p.hw * 8);
      const uint64_t dB0 = tc::smem_desc(sdy0, 16384, 1024, 2);
      int stage = 0;
      uint32_t phase = 0;
      bool first = true;
      for (int64_t vt = vt0; vt < vt1; ++vt) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t sadd = (uint32_t)(stage * STAGE) >> 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < G) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              tc::mma_bf16_warp(tmem_base + i * BN, dA[i] + sadd + goff[j], dB0 + sadd + j * 128, IDESC,
                                (first && j == 0) ? 0u : 1u);
          }
        }
        tc::mma_commit_warp(&empty[stage]);
        __syncwarp();
        first = false;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      tc::mma_commit_warp(done);
      __syncwarp();
    } else if (G > 0) {
      constexpr uint32_t IDESC = tc::idesc_bf16(128, BN, 1, 1);
      int stage = 0;
      uint32_t phase = 0;
      bool first = true;
      for (int64_t vt = vt0; vt < vt1; ++vt) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        {
          const uint32_t sdy = tc::smem_u32(smem + stage * STAGE);
          const uint32_t sx = sdy + DYB;
          for (int i = 0; i < G; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // K = 16 voxels = 2 row groups per MMA
              const uint64_t ad = tc::smem_desc(sx + (2 * i) * 16384 + j * 2048, 16384, 1024, 2);
              const uint64_t bd = tc::smem_desc(sdy + j * 2048, 16384, 1024, 2);
              tc::mma_bf16_warp(tmem_base + i * BN, ad, bd, IDESC, (first && j == 0) ? 0u : 1u);
            }
          }
          tc::mma_commit_warp(&empty[stage]);
        }
        __syncwarp();
        first = false;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      tc::mma_commit_warp(done);
      __syncwarp();
    }
  } else {
    // epilogue: row = (atom half, ci), 32 co columns per tcgen05.ld
    if (G > 0) {
      const int q = warp & 3;
      const int row = q * 32 + lane;
      tc::mbar_wait(done, 0);
      tc::tc_fence_after();
      float *P = p.part + (int64_t)split * p.Co * p.taps * p.Ci;
      for (int i = 0; i < G; ++i) {
        const int at = 2 * (mt0 + i) + (row >= 64 ? 1 : 0);
        const bool ok = p.atom_valid[at] != 0;
        const int tap = p.atom_tap[at];
        const int ci = p.atom_cb[at] * 64 + (row & 63);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t v[32];
          tc::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + i * BN + c0, v);
          tc::tmem_wait_ld();
          if (ok) {
            float *dst = P + ((int64_t)(cob * BN + c0) * p.taps + tap) * p.Ci + ci;
            const int64_t cs = (int64_t)p.taps * p.Ci;  // stride between co
            if (p.accum && p.overwrite) {  // single split, first contribution: plain stores
#pragma unroll
              for (int j = 0; j < 32; ++j) dst[j * cs] = __uint_as_float(v[j]);
            } else if (p.accum) {  // single split: straight into dW (all 32 loads issued before the stores)
              float old[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) old[j] = dst[j * cs];
#pragma unroll
              for (int j = 0; j < 32; ++j) dst[j * cs] = old[j] + __uint_as_float(v[j]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) dst[j * cs] = __uint_as_float(v[j]);
            }
          }
        }
      }
      tc::tc_fence_before();
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

// out[i] += sum over z < splits of part[z * n + i] (split-K weight-gradient
// partials).  Deterministic and parallel over the splits: group g of a block
// sums z = g, g + G, ... in ascending order (four loads in flight), then the G
// group sums are added in g order.  The former one-thread-per-element loop was
// latency-bound for the 1x1x1 and stem weights (n = 4096 / 1728 elements,
// 138-444 splits: 16 / 7 blocks, ~18 us each).
template <int G>
__global__ void __launch_bounds__(256) split_reduce_add_k(const float *__restrict__ part, int splits, int64_t n,
                                                          float *__restrict__ out, int overwrite) {
  constexpr int E = 256 / G;
  __shared__ float red[G][E];
  pdl_begin();
  const int e = threadIdx.x % E, g = threadIdx.x / E;
  for (int64_t base = (int64_t)blockIdx.x * E; base < n; base += (int64_t)gridDim.x * E) {
    const int64_t i = base + e;
    float s = 0.f;
    if (i < n) {
      int z = g;
      for (; z + 3 * G < splits; z += 4 * G) {
        const float a = part[(int64_t)z * n + i], b = part[(int64_t)(z + G) * n + i];
        const float c = part[(int64_t)(z + 2 * G) * n + i], d = part[(int64_t)(z + 3 * G) * n + i];
        s += a;
        s += b;
        s += c;
        s += d;
      }
      for (; z < splits; z += G) s += part[(int64_t)z * n + i];
    }
    if (G > 1) {
      red[g][e] = s;
      __syncthreads();
      if (g == 0 && i < n) {
        float t = red[0][e];
#pragma unroll
        for (int q = 1; q < G; ++q) t += red[q][e];
        out[i] = overwrite ? t : out[i] + t;
      }
      __syncthreads();
    } else if (i < n) {
      out[i] = overwrite ? s : out[i] + s;
    }
  }
}

template <int BN, int STAGES, int XBYTES>
void wg_launch(const WgParams &p, int grid, cudaStream_t st) {
  constexpr int STAGE = (BN / 64) * 16384 + XBYTES;
  constexpr int SMEM = STAGES * STAGE + 256 + ATAB_MAX * 16 + 1024;
  static uint64_t attr_devs = 0;  // kernel attributes are per device
  if (!once_on_device(attr_devs)) {
    CUDA_CHECK(cudaFuncSetAttribute(wgrad_tc_kernel<BN, STAGES, XBYTES>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      }
  launch_k(wgrad_tc_kernel<BN, STAGES, XBYTES>, grid, WG_THREADS, SMEM, st, p);
  LAUNCH_CHECK();
}

// launch-shape decision shared by the workspace query and the launcher
struct WgShape {
  int BN, G, haloed, n_mtiles, n_mgroups, n_cob, splits, vt_per_split;
  int bw, bh, bd, bn, tw, th, td, tn;
  int64_t n_vtiles;
};

void choose_box_wg(int W, int H, int D, int N, int &bw, int &bh, int &bd, int &bn) {
  double best = 1e30;
  for (int a = 1; a <= 128; a *= 2)
    for (int b = 1; a * b <= 128; b *= 2)
      for (int c = 1; a * b * c <= 128; c *= 2) {
        int e = 128 / (a * b * c);
        if (a * b * c * e != 128) continue;
        double pad = (double)((W + a - 1) / a * a) * ((H + b - 1) / b * b) * ((D + c - 1) / c * c) *
                     ((N + e - 1) / e * e);
        if (pad < best) { best = pad; bw = a; bh = b; bd = c; bn = e; }
      }
}

WgShape wg_shape(const ConvGeom &g) {
  WgShape s;
  s.BN = g.Co % 256 == 0 ? 256 : g.Co % 128 == 0 ? 128 : 64;
  // haloed staging cuts L2 traffic 9x; its MMAs read operands from arbitrary
  // row offsets at full speed (tools/micro/tc_probe.cu) — it first measured
  // slower only because the issue loop recomputed the descriptors with integer
  // divisions per MMA (now precomputed).  RN_WG_NOHALO=1: per-tap staging.
  s.haloed = (g.s == 1 && g.k == 3 && g.Ci == 64 && !getenv("RN_WG_NOHALO")) ? 1 : 0;
  const int atoms = g.taps() * (g.Ci / 64);
  s.n_mtiles = (atoms + 1) / 2;
  if (s.haloed) {
    s.bw = 8; s.bh = 4; s.bd = 4; s.bn = 1;
    const int groups = (s.n_mtiles + 512 / s.BN - 1) / (512 / s.BN);  // balanced M-groups (14 tiles -> 7 + 7)
    s.G = (s.n_mtiles + groups - 1) / groups;
  } else {
    choose_box_wg(g.Wo, g.Ho, g.Do, g.N, s.bw, s.bh, s.bd, s.bn);
    const int dyb = (s.BN / 64) * 16;
    int G = (100 - dyb) / 32;  // KB per stage budget for x atoms
    G = std::max(1, std::min(G, 512 / s.BN));
    s.G = std::min(G, s.n_mtiles);
  }
  s.n_mgroups = (s.n_mtiles + s.G - 1) / s.G;
  s.n_cob = g.Co / s.BN;
  s.tw = (g.Wo + s.bw - 1) / s.bw;
  s.th = (g.Ho + s.bh - 1) / s.bh;
  s.td = (g.Do + s.bd - 1) / s.bd;
  s.tn = (g.N + s.bn - 1) / s.bn;
  s.n_vtiles = (int64_t)s.tw * s.th * s.td * s.tn;
  if (!s.haloed && s.n_vtiles <= 24) {
    // short K (late stages): no split (its fp32 partials would be as large as
    // dW itself); one M-tile per CTA and narrower N blocks supply the CTAs
    s.G = 1;
    while (s.BN > 64 && (int64_t)s.n_mtiles * (g.Co / s.BN) < 100) s.BN /= 2;
    s.n_mgroups = s.n_mtiles;
    s.n_cob = g.Co / s.BN;
    s.splits = 1;
    s.vt_per_split = (int)s.n_vtiles;
    return s;
  }
  const int ctas0 = s.n_mgroups * s.n_cob;
  int splits = std::max(1, 148 / ctas0);  // one wave: every CTA resident (a 2nd partial wave doubles the time)
  splits = (int)std::max<int64_t>(1, std::min<int64_t>(splits, s.n_vtiles));
  s.vt_per_split = (int)((s.n_vtiles + splits - 1) / splits);
  s.splits = (int)((s.n_vtiles + s.vt_per_split - 1) / s.vt_per_split);
  return s;
}

}  // namespace

void split_reduce_add(const float *part, int splits, int64_t n, float *out, cudaStream_t st, bool overwrite) {
  auto go = [&](auto kern, int G) {
    const int64_t per = 256 / G;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 8));
    launch_k(kern, grid, 256, 0, st, part, splits, n, out, overwrite ? 1 : 0);
  };
  // enough blocks to cover the SMs: the more splits per element, the more groups
  if (splits >= 64 && n <= 148 * 64) go(split_reduce_add_k<8>, 8);
  else if (splits >= 16 && n <= 148 * 256) go(split_reduce_add_k<4>, 4);
  else if (splits >= 4 && n <= 148 * 512) go(split_reduce_add_k<2>, 2);
  else go(split_reduce_add_k<1>, 1);
  LAUNCH_CHECK();
}

void make_act_map(CUtensorMap *m, const void *base, int C, int W, int H, int D, int N, int64_t sw, int64_t sh,
                  int64_t sd, int64_t sn, int bw, int bh, int bd, int bn);

bool tc_wgrad_supported(const ConvGeom &g) {
  if (g.Ci % 64 != 0 || g.Co % 64 != 0) return false;
  if (!tc_conv_supported(g, false)) return false;
  const int atoms = g.taps() * (g.Ci / 64);
  if (atoms > 2 * MAX_ATOMS) return false;
  return true;
}

size_t tc_wgrad_ws_floats(const ConvGeom &g) {
  if (!tc_wgrad_supported(g)) return 0;
  WgShape s = wg_shape(g);
  return s.splits > 1 ? (size_t)s.splits * g.Co * g.taps() * g.Ci : 0;
}

void conv_wgrad_tc(const ConvGeom &g, const bf16 *x, const bf16 *dy, float *dw, float *ws, cudaStream_t st,
                   bool overwrite) {
  WgShape s = wg_shape(g);
  WgParams p;
  memset(&p, 0, sizeof p);
  p.haloed = s.haloed;
  p.G = s.G;
  if (!s.haloed && 2 * s.G > ATAB_MAX) throw Error(RN_ERR_STATE, "conv_wgrad_tc: atom table overflow");
  p.n_mgroups = s.n_mgroups;
  p.n_cob = s.n_cob;
  p.splits = s.splits;
  p.n_mtiles = s.n_mtiles;
  p.bw = s.bw; p.bh = s.bh; p.bd = s.bd; p.bn = s.bn;
  p.tw = s.tw; p.th = s.th; p.td = s.td; p.tn = s.tn;
  p.n_vtiles = s.n_vtiles;
  p.vt_per_split = s.vt_per_split;
  p.accum = s.splits == 1;
  p.overwrite = overwrite ? 1 : 0;
  p.part = p.accum ? dw : ws;
  p.Co = g.Co; p.Ci = g.Ci; p.taps = g.taps();
  // dy map: NDHWC [N][Do][Ho][Wo][Co]
  make_act_map(&p.dy_map, dy, g.Co, g.Wo, g.Ho, g.Do, g.N, 1, g.Wo, (int64_t)g.Wo * g.Ho,
               (int64_t)g.Wo * g.Ho * g.Do, s.bw, s.bh, s.bd, s.bn);
  // atoms in (tap, ci block) order; paired atoms may start at any 128-B row of
  // the swizzled tile (the hardware derives the swizzle phase from the address)
  const int cbs = g.Ci / 64;
  int na = 0;
  auto add_atom = [&](int t, int cb, int valid) {
    const int kd = t / (g.k * g.k), kh = (t / g.k) % g.k, kw = t % g.k;
    const int od = kd - g.p, oh = kh - g.p, ow = kw - g.p;
    p.atom_tap[na] = (int16_t)t;
    p.atom_cb[na] = (int8_t)cb;
    p.atom_valid[na] = (int8_t)valid;
    if (g.s == 1) {
      p.atom_map[na] = 0;
      p.atom_od[na] = od; p.atom_oh[na] = oh; p.atom_ow[na] = ow;
    } else {
      auto par = [](int off) { return off == 0 ? 0 : 1; };
      auto sh = [](int off) { return off < 0 ? -1 : 0; };
      p.atom_map[na] = (par(od) * 2 + par(oh)) * 2 + par(ow);
      p.atom_od[na] = sh(od); p.atom_oh[na] = sh(oh); p.atom_ow[na] = sh(ow);
    }
    ++na;
  };
  {
    int lt = 0, lc = 0;
    for (int t = 0; t < g.taps(); ++t)
      for (int cb = 0; cb < cbs; ++cb) {
        add_atom(t, cb, 1);
        lt = t;
        lc = cb;
      }
    if (na % 2) add_atom(lt, lc, 0);
  }
  if (na / 2 != s.n_mtiles) throw Error(RN_ERR_STATE, "wgrad: atom count mismatch");
  if (s.haloed) {
    p.hw = getenv("RN_WG_HW16") ? 16 : s.bw + 2;
    p.hh = s.bh + 2;
    p.hd = s.bd + 2;
    make_act_map(&p.x_map[0], x, g.Ci, g.Wi, g.Hi, g.Di, g.N, 1, g.Wi, (int64_t)g.Wi * g.Hi,
                 (int64_t)g.Wi * g.Hi * g.Di, p.hw, p.hh, p.hd, 1);
  } else if (g.s == 1) {
    make_act_map(&p.x_map[0], x, g.Ci, g.Wi, g.Hi, g.Di, g.N, 1, g.Wi, (int64_t)g.Wi * g.Hi,
                 (int64_t)g.Wi * g.Hi * g.Di, s.bw, s.bh, s.bd, s.bn);
  } else {
    for (int pd = 0; pd < 2; ++pd)
      for (int ph = 0; ph < 2; ++ph)
        for (int pw = 0; pw < 2; ++pw) {
          const int Wv = (g.Wi - pw + 1) / 2, Hv = (g.Hi - ph + 1) / 2, Dv = (g.Di - pd + 1) / 2;
          const bf16 *b = x + (((int64_t)pd * g.Hi + ph) * g.Wi + pw) * g.Ci;
          make_act_map(&p.x_map[(pd * 2 + ph) * 2 + pw], b, g.Ci, Wv, Hv, Dv, g.N, 2, 2LL * g.Wi,
                       2LL * g.Wi * g.Hi, (int64_t)g.Wi * g.Hi * g.Di, s.bw, s.bh, s.bd, s.bn);
        }
  }
  const int grid = s.n_mgroups * s.n_cob * s.splits;
  // the haloed region: 10 x 6 x 6 voxels x 128 B = 46080 B
  if (s.haloed) {
    if (s.BN == 64 && p.hw == 16) wg_launch<64, 2, 73728>(p, grid, st);
    else if (s.BN == 64) wg_launch<64, 3, 46080>(p, grid, st);
    else if (s.BN == 128) wg_launch<128, 2, 46080>(p, grid, st);
    else wg_launch<256, 2, 46080>(p, grid, st);
  } else {
    if (s.BN == 64) wg_launch<64, 2, 2 * 32768>(p, grid, st);        // G <= 2 (G*32 KB + 16 KB)
    else if (s.BN == 128) wg_launch<128, 2, 2 * 32768>(p, grid, st);  // G <= 2
    else wg_launch<256, 2, 1 * 32768>(p, grid, st);                   // G <= 1
  }
  if (p.accum) return;
  const int64_t n = (int64_t)g.Co * g.taps() * g.Ci;
  split_reduce_add(ws, s.splits, n, dw, st, overwrite);
}

}  // namespace rn
