// k_elem.cu — HBM-bound kernels of the 3D-ResAttNet step: BatchNorm (train
// mode) statistics / apply / backward, ReLU, residual add, 3D max-pool (k3 s2 p1)
// forward + gather-form backward, trilinear upsampling (align_corners=False) and
// its adjoint, the soft-mask attention combine (1 + sigmoid(m)) * T and its
// backward, GAP + FC + softmax cross-entropy, SGD and weight repacking.
// PAPER.md:364-366 (Conv block = conv + 3D BN + ReLU; residual self-attention
// block), P:486 (cross-entropy, SGD), P:156 (chain rule / update); concrete
// readings X4-X12 in DESIGN.md.
//
// Layout: NDHWC, every thread owns one 16-byte channel vector (Vec<T>::N
// channels) of one voxel; per-channel reductions write per-block partials that
// a finalize kernel sums in a fixed order (deterministic, no float atomics).
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "error.h"
#include "kernels.h"
#include "util.cuh"

namespace rn {

namespace cg = cooperative_groups;

namespace {

constexpr int NT = 256;

inline unsigned grid_for(int64_t items, int per_block = NT, int64_t cap = 148 * 32) {
  int64_t b = (items + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// ---------------------------------------------------------------------------
// generic per-channel block reduction: each block reduces rows [r0, r0 + rpb)
// ---------------------------------------------------------------------------
template <typename T, typename Op>
__device__ __forceinline__ void chan_reduce_block(Op &op, int64_t V, int C, float *__restrict__ partial, int64_t rpb,
                                                  float *sm);

template <typename T, typename Op>
__global__ void __launch_bounds__(NT) chan_reduce_k(Op op, int64_t V, int C, float *__restrict__ partial,
                                                    int64_t rpb) {
  extern __shared__ float sm[];
  chan_reduce_block<T>(op, V, C, partial, rpb, sm);
}

template <typename T, typename Op>
__device__ __forceinline__ void chan_reduce_block(Op &op, int64_t V, int C, float *__restrict__ partial, int64_t rpb,
                                                  float *sm) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int RPI = NT / G;
  const int t = threadIdx.x, rr = t / G, cg = t % G;
  float a1[VEC], a2[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) a1[j] = a2[j] = 0.f;
  if (rr < RPI) {
    op.init(cg * VEC);
    const int64_t r0 = (int64_t)blockIdx.x * rpb;
    const int64_t r1 = min(V, r0 + rpb);
    int64_t r = r0 + rr;
    for (; r + 3 * RPI < r1; r += 4 * RPI) {  // 4 independent rows per iteration (memory-level parallelism)
      op.row(r, cg * VEC, a1, a2);
      op.row(r + RPI, cg * VEC, a1, a2);
      op.row(r + 2 * RPI, cg * VEC, a1, a2);
      op.row(r + 3 * RPI, cg * VEC, a1, a2);
    }
    for (; r < r1; r += RPI) op.row(r, cg * VEC, a1, a2);
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      sm[rr * C + cg * VEC + j] = a1[j];
      sm[RPI * C + rr * C + cg * VEC + j] = a2[j];
    }
  }
  __syncthreads();
  for (int c = t; c < C; c += NT) {
    float s1 = 0.f, s2 = 0.f;
    for (int r = 0; r < RPI; ++r) {
      s1 += sm[r * C + c];
      s2 += sm[RPI * C + r * C + c];
    }
    partial[(int64_t)blockIdx.x * 2 * C + c] = s1;
    partial[(int64_t)blockIdx.x * 2 * C + C + c] = s2;
  }
}

template <typename T>
void launch_chan_reduce_dims(int64_t V, int C, int nblk, int64_t &rpb, size_t &smem) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int RPI = NT / G;
  rpb = (V + nblk - 1) / nblk;
  smem = (size_t)2 * RPI * C * sizeof(float);
}

template <typename T>
struct StatsOp {
  const T *x;
  int C;
  float K[Vec<T>::N];
  __device__ void init(int c0) { load_vec(x + c0, K); }
  __device__ void row(int64_t r, int c0, float *a1, float *a2) {
    float v[Vec<T>::N];
    load_vec(x + r * C + c0, v);
#pragma unroll
    for (int j = 0; j < Vec<T>::N; ++j) {
      float d = v[j] - K[j];
      a1[j] += d;
      a2[j] = fmaf(d, d, a2[j]);
    }
  }
};

template <typename T>
__device__ __forceinline__ void masked_dy(const T *dy, const T *x, const T *mask_t, int mode, const float *scale,
                                          const float *shift, int64_t off, int c0, float *d, float *xv) {
  constexpr int VEC = Vec<T>::N;
  load_vec(dy + off, d);
  load_vec(x + off, xv);
  if (mode == MASK_TENSOR) {
    float m[VEC];
    load_vec(mask_t + off, m);
#pragma unroll
    for (int j = 0; j < VEC; ++j) d[j] = m[j] > 0.f ? d[j] : 0.f;
  } else if (mode == MASK_RECOMPUTE) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) d[j] = fmaf(xv[j], scale[c0 + j], shift[c0 + j]) > 0.f ? d[j] : 0.f;
  }
}

template <typename T>
struct BwdOp {
  const T *dy, *x, *mask_t;
  int mode, C;
  const float *scale, *shift, *mean, *invstd;
  __device__ void init(int) {}
  __device__ void row(int64_t r, int c0, float *a1, float *a2) {
    constexpr int VEC = Vec<T>::N;
    float d[VEC], xv[VEC];
    masked_dy(dy, x, mask_t, mode, scale, shift, r * C + c0, c0, d, xv);
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float xh = (xv[j] - mean[c0 + j]) * invstd[c0 + j];
      a1[j] += d[j];
      a2[j] = fmaf(d[j], xh, a2[j]);
    }
  }
};

template <typename T>
struct AttBwdOp {
  const T *dout, *m, *Tt;
  T *dT, *dm;
  int C;
  __device__ void init(int) {}
  __device__ void row(int64_t r, int c0, float *a1, float *a2) {
    constexpr int VEC = Vec<T>::N;
    float g[VEC], mv[VEC], tv[VEC], o1[VEC], o2[VEC];
    const int64_t off = r * C + c0;
    load_vec(dout + off, g);
    load_vec(m + off, mv);
    load_vec(Tt + off, tv);
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float s = 1.f / (1.f + __expf(-mv[j]));
      o1[j] = g[j] * (1.f + s);
      o2[j] = g[j] * tv[j] * s * (1.f - s);
    }
    store_vec(dT + off, o1);
    store_vec(dm + off, o2);
#pragma unroll
    for (int j = 0; j < VEC; ++j) a1[j] += o2[j];
  }
};

// Sum of per-block partials for channel c: one warp per channel, lanes stride
// over the blocks in double, fixed shuffle tree (deterministic).
__device__ __forceinline__ void warp_partial_sums(const float *partial, int nblk, int C, int c, double &S1,
                                                  double &S2) {
  const int lane = threadIdx.x & 31;
  double a = 0.0, b = 0.0;
  for (int k = lane; k < nblk; k += 32) {
    a += (double)partial[(int64_t)k * 2 * C + c];
    b += (double)partial[(int64_t)k * 2 * C + C + c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  S1 = a;
  S2 = b;
}

template <typename T>
__device__ __forceinline__ void bn_finalize_channel(int c, const T *x, const float *partial, int nblk, int64_t V,
                                                    int C, const float *gamma, const float *beta, float *mean,
                                                    float *invstd, float *scale, float *shift, float *run_mean,
                                                    float *run_var, float momentum, float eps) {
  double S, Q;
  warp_partial_sums(partial, nblk, C, c, S, Q);
  if ((threadIdx.x & 31) != 0) return;
  const double K = (double)to_f(x[c]);
  const double ms = S / (double)V;
  double var = Q / (double)V - ms * ms;
  if (var < 0) var = 0;
  const double mu = K + ms;
  const double is = 1.0 / sqrt(var + (double)eps);
  mean[c] = (float)mu;
  invstd[c] = (float)is;
  const double sc = (double)gamma[c] * is;
  scale[c] = (float)sc;
  shift[c] = (float)((double)beta[c] - mu * sc);
  if (run_mean) {
    const double unb = V > 1 ? var * (double)V / (double)(V - 1) : var;
    run_mean[c] = (float)((1.0 - momentum) * run_mean[c] + momentum * mu);
    run_var[c] = (float)((1.0 - momentum) * run_var[c] + momentum * unb);
  }
}

template <typename T>
__global__ void bn_finalize_k(const T *x, const float *partial, int nblk, int64_t V, int C, const float *gamma,
                              const float *beta, float *mean, float *invstd, float *scale, float *shift,
                              float *run_mean, float *run_var, float momentum, float eps) {
  const int c = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (c >= C) return;
  bn_finalize_channel<T>(c, x, partial, nblk, V, C, gamma, beta, mean, invstd, scale, shift, run_mean, run_var,
                         momentum, eps);
}

__device__ __forceinline__ void bn_bwd_finalize_channel(int c, const float *partial, int nblk, int64_t V, int C,
                                                        const float *gamma, const float *mean, const float *invstd,
                                                        float *dgamma, float *dbeta, float *coef) {
  double S1, S2;
  warp_partial_sums(partial, nblk, C, c, S1, S2);
  if ((threadIdx.x & 31) != 0) return;
  dgamma[c] += (float)S2;
  dbeta[c] += (float)S1;
  const double m1 = S1 / (double)V, m2 = S2 / (double)V;
  const double is = invstd[c];
  const double A = (double)gamma[c] * is;
  coef[c] = (float)A;
  coef[C + c] = (float)(-A * is * m2);
  coef[2 * C + c] = (float)(-A * m1 + A * is * (double)mean[c] * m2);
}

__global__ void bn_bwd_finalize_k(const float *partial, int nblk, int64_t V, int C, const float *gamma,
                                  const float *mean, const float *invstd, float *dgamma, float *dbeta,
                                  float *coef) {
  const int c = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (c >= C) return;
  bn_bwd_finalize_channel(c, partial, nblk, V, C, gamma, mean, invstd, dgamma, dbeta, coef);
}

// ---------------------------------------------------------------------------
// Fused BatchNorm passes (one cooperative launch per BN layer):
//   forward : per-block channel sums -> grid sync -> finalize (warp per channel)
//             -> grid sync -> y = act(x*scale + shift + R) on the block's rows
//   backward: per-block (sum dy', sum dy'*xhat) -> grid sync -> finalize
//             (dgamma, dbeta, coefficients) -> grid sync -> dx on the block's rows
// The apply pass re-reads rows this block just reduced (L2-resident), and the
// three launches of the unfused version become one.
// ---------------------------------------------------------------------------
template <typename T>
struct BnFwdArgs {
  const T *x;
  int64_t V, rpb;
  int C;
  float *partial;
  const float *gamma, *beta;
  float *mean, *invstd, *scale, *shift, *run_mean, *run_var;
  float momentum, eps;
  const T *res;
  const float *rscale, *rshift;
  int relu;
  T *y;
};

template <typename T>
__global__ void __launch_bounds__(NT) bn_fwd_fused_k(BnFwdArgs<T> a) {
  extern __shared__ float sm[];
  cg::grid_group grid = cg::this_grid();
  StatsOp<T> op{a.x, a.C, {}};
  chan_reduce_block<T>(op, a.V, a.C, a.partial, a.rpb, sm);
  grid.sync();
  const int warps = blockDim.x / 32;
  for (int c = blockIdx.x * warps + threadIdx.x / 32; c < a.C; c += gridDim.x * warps)
    bn_finalize_channel<T>(c, a.x, a.partial, gridDim.x, a.V, a.C, a.gamma, a.beta, a.mean, a.invstd, a.scale,
                           a.shift, a.run_mean, a.run_var, a.momentum, a.eps);
  if (!a.y) return;
  grid.sync();
  constexpr int VEC = Vec<T>::N;
  const int G = a.C / VEC;
  const int c0 = (threadIdx.x % G) * VEC;  // fixed per thread (blockDim % G == 0)
  float sc[VEC], sh[VEC], rs[VEC], rh[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    sc[j] = __ldcg(a.scale + c0 + j);
    sh[j] = __ldcg(a.shift + c0 + j);
    rs[j] = a.rscale ? __ldcg(a.rscale + c0 + j) : 1.f;
    rh[j] = a.rscale ? __ldcg(a.rshift + c0 + j) : 0.f;
  }
  const int64_t r0 = (int64_t)blockIdx.x * a.rpb, r1 = min(a.V, r0 + a.rpb);
  for (int64_t i = r0 * G + threadIdx.x; i < r1 * G; i += blockDim.x) {
    const int64_t off = (i / G) * a.C + c0;
    float v[VEC];
    load_vec(a.x + off, v);
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[j] = fmaf(v[j], sc[j], sh[j]);
    if (a.res) {
      float r[VEC];
      load_vec(a.res + off, r);
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] += fmaf(r[j], rs[j], rh[j]);
    }
    if (a.relu) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = fmaxf(v[j], 0.f);
    }
    store_vec(a.y + off, v);
  }
}

template <typename T>
struct BnBwdArgs {
  const T *dy, *x, *mask_t;
  int64_t V, rpb;
  int C, mode;
  float *partial;
  const float *scale, *shift, *mean, *invstd, *gamma;
  float *dgamma, *dbeta, *coef;
  T *dx;
};

template <typename T>
__global__ void __launch_bounds__(NT) bn_bwd_fused_k(BnBwdArgs<T> a) {
  extern __shared__ float sm[];
  cg::grid_group grid = cg::this_grid();
  BwdOp<T> op{a.dy, a.x, a.mask_t, a.mode, a.C, a.scale, a.shift, a.mean, a.invstd};
  chan_reduce_block<T>(op, a.V, a.C, a.partial, a.rpb, sm);
  grid.sync();
  const int warps = blockDim.x / 32;
  for (int c = blockIdx.x * warps + threadIdx.x / 32; c < a.C; c += gridDim.x * warps)
    bn_bwd_finalize_channel(c, a.partial, gridDim.x, a.V, a.C, a.gamma, a.mean, a.invstd, a.dgamma, a.dbeta, a.coef);
  grid.sync();
  constexpr int VEC = Vec<T>::N;
  const int G = a.C / VEC;
  const int c0 = (threadIdx.x % G) * VEC;
  float A[VEC], B[VEC], Cc[VEC], sc[VEC], sh[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    A[j] = __ldcg(a.coef + c0 + j);
    B[j] = __ldcg(a.coef + a.C + c0 + j);
    Cc[j] = __ldcg(a.coef + 2 * a.C + c0 + j);
    sc[j] = a.scale[c0 + j];
    sh[j] = a.shift[c0 + j];
  }
  const int64_t r0 = (int64_t)blockIdx.x * a.rpb, r1 = min(a.V, r0 + a.rpb);
  for (int64_t i = r0 * G + threadIdx.x; i < r1 * G; i += blockDim.x) {
    const int64_t off = (i / G) * a.C + c0;
    float d[VEC], xv[VEC], o[VEC];
    load_vec(a.dy + off, d);
    load_vec(a.x + off, xv);
    if (a.mode == MASK_TENSOR) {
      float m[VEC];
      load_vec(a.mask_t + off, m);
#pragma unroll
      for (int j = 0; j < VEC; ++j) d[j] = m[j] > 0.f ? d[j] : 0.f;
    } else if (a.mode == MASK_RECOMPUTE) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) d[j] = fmaf(xv[j], sc[j], sh[j]) > 0.f ? d[j] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) o[j] = fmaf(A[j], d[j], fmaf(B[j], xv[j], Cc[j]));
    store_vec(a.dx + off, o);
  }
}

template <typename K>
int coop_grid(K kernel, size_t smem, int64_t V, int C) {
  static int max_blocks = 0;
  if (!max_blocks) {
    int per_sm = 0, dev = 0, sms = 148;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, NT, smem));
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    max_blocks = std::max(1, std::min(per_sm, 3)) * sms;
  }
  const int want = chan_reduce_blocks(V, C);
  return std::max(1, std::min(want, max_blocks));
}

template <typename K, typename A>
void coop_launch(K kernel, int grid, size_t smem, const A &args, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, args));
}

__global__ void chan_sum_finalize_k(const float *partial, int nblk, int C, float *out) {
  const int c = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (c >= C) return;
  double S1, S2;
  warp_partial_sums(partial, nblk, C, c, S1, S2);
  if ((threadIdx.x & 31) == 0) out[c] += (float)S1;
}

template <typename T>
__global__ void bn_apply_k(const T *__restrict__ x, int64_t V, int C, const float *__restrict__ scale,
                           const float *__restrict__ shift, const T *__restrict__ res,
                           const float *__restrict__ rscale, const float *__restrict__ rshift, int relu,
                           T *__restrict__ y) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = V * G;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % G) * VEC;
    const int64_t off = (i / G) * C + c0;
    float v[VEC];
    load_vec(x + off, v);
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[j] = fmaf(v[j], scale[c0 + j], shift[c0 + j]);
    if (res) {
      float r[VEC];
      load_vec(res + off, r);
      if (rscale) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] += fmaf(r[j], rscale[c0 + j], rshift[c0 + j]);
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] += r[j];
      }
    }
    if (relu) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = fmaxf(v[j], 0.f);
    }
    store_vec(y + off, v);
  }
}

template <typename T>
__global__ void bn_bwd_apply_k(const T *__restrict__ dy, const T *__restrict__ x, int64_t V, int C, int mode,
                               const T *__restrict__ mask_t, const float *__restrict__ scale,
                               const float *__restrict__ shift, const float *__restrict__ coef,
                               T *__restrict__ dx) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = V * G;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % G) * VEC;
    const int64_t off = (i / G) * C + c0;
    float d[VEC], xv[VEC], o[VEC];
    masked_dy(dy, x, mask_t, mode, scale, shift, off, c0, d, xv);
#pragma unroll
    for (int j = 0; j < VEC; ++j)
      o[j] = fmaf(coef[c0 + j], d[j], fmaf(coef[C + c0 + j], xv[j], coef[2 * C + c0 + j]));
    store_vec(dx + off, o);
  }
}

// max-pool k3 s2 p1, -inf padding; first maximum in (kd,kh,kw) order (reading X10)
template <typename T>
__global__ void maxpool_fwd_k(const T *__restrict__ x, int N, int D, int H, int W, int C,
                              const float *__restrict__ scale, const float *__restrict__ shift, int relu,
                              T *__restrict__ y, uint8_t *__restrict__ am, int Do, int Ho, int Wo) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = (int64_t)N * Do * Ho * Wo * G;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % G) * VEC;
    int64_t r = i / G;
    const int64_t vo = r;
    const int ow = (int)(r % Wo); r /= Wo;
    const int oh = (int)(r % Ho); r /= Ho;
    const int od = (int)(r % Do); r /= Do;
    const int nn = (int)r;
    float best[VEC];
    uint8_t arg[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) { best[j] = -INFINITY; arg[j] = 0; }
    for (int tap = 0; tap < 27; ++tap) {
      const int id = 2 * od + tap / 9 - 1, ih = 2 * oh + (tap / 3) % 3 - 1, iw = 2 * ow + tap % 3 - 1;
      if (id < 0 || id >= D || ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
      float v[VEC];
      load_vec(x + ((((int64_t)nn * D + id) * H + ih) * W + iw) * C + c0, v);
      if (scale) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          v[j] = fmaf(v[j], scale[c0 + j], shift[c0 + j]);
          if (relu) v[j] = fmaxf(v[j], 0.f);
        }
      }
#pragma unroll
      for (int j = 0; j < VEC; ++j)
        if (v[j] > best[j]) { best[j] = v[j]; arg[j] = (uint8_t)tap; }
    }
    store_vec(y + vo * C + c0, best);
#pragma unroll
    for (int j = 0; j < VEC; ++j) am[vo * C + c0 + j] = arg[j];
  }
}

// gather-form adjoint: each input voxel sums dy of the (<= 8) windows whose argmax is it
template <typename T>
__global__ void maxpool_bwd_k(const T *__restrict__ dy, const uint8_t *__restrict__ am, int N, int D, int H,
                              int W, int C, int Do, int Ho, int Wo, T *__restrict__ dx, int accumulate) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = (int64_t)N * D * H * W * G;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % G) * VEC;
    int64_t r = i / G;
    const int64_t vi = r;
    const int iw = (int)(r % W); r /= W;
    const int ih = (int)(r % H); r /= H;
    const int id = (int)(r % D); r /= D;
    const int nn = (int)r;
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
    // windows o with 2o-1 <= i <= 2o+1  <=>  o in [ceil((i-1)/2), floor((i+1)/2)]
    const int d_lo = max(0, id / 2), d_hi = min(Do - 1, (id + 1) / 2);
    const int h_lo = max(0, ih / 2), h_hi = min(Ho - 1, (ih + 1) / 2);
    const int w_lo = max(0, iw / 2), w_hi = min(Wo - 1, (iw + 1) / 2);
    for (int od = d_lo; od <= d_hi; ++od)
      for (int oh = h_lo; oh <= h_hi; ++oh)
        for (int ow = w_lo; ow <= w_hi; ++ow) {
          const int tap = ((id - 2 * od + 1) * 3 + (ih - 2 * oh + 1)) * 3 + (iw - 2 * ow + 1);
          const int64_t o = ((((int64_t)nn * Do + od) * Ho + oh) * Wo + ow) * C + c0;
          float g[VEC];
          load_vec(dy + o, g);
#pragma unroll
          for (int j = 0; j < VEC; ++j)
            if (am[o + j] == tap) acc[j] += g[j];
        }
    if (accumulate) {
      float p[VEC];
      load_vec(dx + vi * C + c0, p);
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] += p[j];
    }
    store_vec(dx + vi * C + c0, acc);
  }
}

template <typename T>
__global__ void upsample_fwd_k(const T *__restrict__ x, int N, int Di, int Hi, int Wi, int C, T *__restrict__ y,
                               int Do, int Ho, int Wo, UpTables t) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = (int64_t)N * Do * Ho * Wo * G;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % G) * VEC;
    int64_t r = i / G;
    const int64_t vo = r;
    const int ow = (int)(r % Wo); r /= Wo;
    const int oh = (int)(r % Ho); r /= Ho;
    const int od = (int)(r % Do); r /= Do;
    const int nn = (int)r;
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
    for (int a = 0; a < 2; ++a) {
      const int id = t.fw_idx[0][2 * od + a];
      const float wa = t.fw_w[0][2 * od + a];
      for (int b = 0; b < 2; ++b) {
        const int ih = t.fw_idx[1][2 * oh + b];
        const float wb = wa * t.fw_w[1][2 * oh + b];
        for (int c = 0; c < 2; ++c) {
          const int iw = t.fw_idx[2][2 * ow + c];
          const float wc = wb * t.fw_w[2][2 * ow + c];
          float v[VEC];
          load_vec(x + ((((int64_t)nn * Di + id) * Hi + ih) * Wi + iw) * C + c0, v);
#pragma unroll
          for (int j = 0; j < VEC; ++j) acc[j] = fmaf(wc, v[j], acc[j]);
        }
      }
    }
    store_vec(y + vo * C + c0, acc);
  }
}

template <typename T>
__global__ void upsample_bwd_k(const T *__restrict__ dy, int N, int Di, int Hi, int Wi, int C, T *__restrict__ dx,
                               int Do, int Ho, int Wo, UpTables t) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = (int64_t)N * Di * Hi * Wi * G;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % G) * VEC;
    int64_t r = i / G;
    const int64_t vi = r;
    const int iw = (int)(r % Wi); r /= Wi;
    const int ih = (int)(r % Hi); r /= Hi;
    const int id = (int)(r % Di); r /= Di;
    const int nn = (int)r;
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
    for (int a = t.bw_start[0][id]; a < t.bw_start[0][id + 1]; ++a) {
      const int od = t.bw_o[0][a];
      const float wa = t.bw_w[0][a];
      for (int b = t.bw_start[1][ih]; b < t.bw_start[1][ih + 1]; ++b) {
        const int oh = t.bw_o[1][b];
        const float wb = wa * t.bw_w[1][b];
        for (int c = t.bw_start[2][iw]; c < t.bw_start[2][iw + 1]; ++c) {
          const int ow = t.bw_o[2][c];
          const float wc = wb * t.bw_w[2][c];
          float v[VEC];
          load_vec(dy + ((((int64_t)nn * Do + od) * Ho + oh) * Wo + ow) * C + c0, v);
#pragma unroll
          for (int j = 0; j < VEC; ++j) acc[j] = fmaf(wc, v[j], acc[j]);
        }
      }
    }
    store_vec(dx + vi * C + c0, acc);
  }
}

template <typename T>
__global__ void att_fwd_k(const T *__restrict__ m, const T *__restrict__ Tt, int64_t V, int C, T *__restrict__ out) {
  constexpr int VEC = Vec<T>::N;
  const int64_t n = V * (C / VEC);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t off = i * VEC;
    float mv[VEC], tv[VEC];
    load_vec(m + off, mv);
    load_vec(Tt + off, tv);
#pragma unroll
    for (int j = 0; j < VEC; ++j) tv[j] = (1.f + 1.f / (1.f + __expf(-mv[j]))) * tv[j];
    store_vec(out + off, tv);
  }
}

// GAP: g[n][c] = mean_v x[n][v][c]; block per (n, 256-channel chunk)
template <typename T>
__global__ void gap_k(const T *__restrict__ x, int V, int C, float *__restrict__ g) {
  const int nn = blockIdx.x;
  for (int c = blockIdx.y * blockDim.x + threadIdx.x; c < C; c += gridDim.y * blockDim.x) {
    float s = 0.f;
    for (int v = 0; v < V; ++v) s += to_f(x[((int64_t)nn * V + v) * C + c]);
    g[nn * C + c] = s / (float)V;
  }
}

// logits, softmax CE (mean over the micro-batch), dz = (p - onehot) * dz_scale; one block
__global__ void ce_k(const float *__restrict__ g, int N, int C, const float *__restrict__ W,
                     const float *__restrict__ b, const int32_t *__restrict__ y, float dz_scale, float loss_scale,
                     float *__restrict__ dz, float *__restrict__ loss_acc) {
  __shared__ float z[64][2];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int p = warp; p < N * 2; p += nw) {
    const int nn = p / 2, k = p % 2;
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s = fmaf(g[nn * C + c], W[k * C + c], s);
    s = warp_sum(s);
    if (lane == 0) z[nn][k] = s + b[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int nn = 0; nn < N; ++nn) {
      const float z0 = z[nn][0], z1 = z[nn][1];
      const float mx = fmaxf(z0, z1);
      const float e0 = expf(z0 - mx), e1 = expf(z1 - mx);
      const float se = e0 + e1;
      const int yy = y[nn];
      tot += -((yy == 0 ? z0 : z1) - mx - logf(se));
      dz[nn * 2 + 0] = (e0 / se - (yy == 0 ? 1.f : 0.f)) * dz_scale;
      dz[nn * 2 + 1] = (e1 / se - (yy == 1 ? 1.f : 0.f)) * dz_scale;
    }
    *loss_acc += tot / (float)N * loss_scale;
  }
}

__global__ void head_wgrad_k(const float *__restrict__ dz, const float *__restrict__ g, int N, int C,
                             float *__restrict__ dW, float *__restrict__ db) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * C; i += gridDim.x * blockDim.x) {
    const int k = i / C, c = i % C;
    float s = 0.f;
    for (int nn = 0; nn < N; ++nn) s = fmaf(dz[nn * 2 + k], g[nn * C + c], s);
    dW[i] += s;
  }
  if (blockIdx.x == 0 && threadIdx.x < 2) {
    float s = 0.f;
    for (int nn = 0; nn < N; ++nn) s += dz[nn * 2 + threadIdx.x];
    db[threadIdx.x] += s;
  }
}

template <typename T>
__global__ void head_dx_k(const float *__restrict__ dz, const float *__restrict__ W, int N, int V, int C,
                          T *__restrict__ dx) {
  const int64_t n = (int64_t)N * V * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int nn = (int)(i / ((int64_t)V * C));
    const float dg = dz[nn * 2] * W[c] + dz[nn * 2 + 1] * W[C + c];
    dx[i] = from_f<T>(dg / (float)V);
  }
}

__global__ void sgd_k(float *__restrict__ w, const float *__restrict__ g, int64_t n, float lr) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<float4 *>(w)[i];
    const float4 b = reinterpret_cast<const float4 *>(g)[i];
    a.x -= lr * b.x; a.y -= lr * b.y; a.z -= lr * b.z; a.w -= lr * b.w;
    reinterpret_cast<float4 *>(w)[i] = a;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] -= lr * g[i];
}

template <typename T>
__global__ void repack_k(const float *__restrict__ w, int Co, int taps, int Ci, T *__restrict__ wf,
                         T *__restrict__ wd) {
  // 32x32 tile of one tap: read/write wf along ci, write wd along co (smem transpose)
  __shared__ float tile[32][33];
  const int ci0 = blockIdx.x * 32, co0 = blockIdx.y * 32, tap = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += 8) {
    const int co = co0 + r, ci = ci0 + tx;
    float v = 0.f;
    if (co < Co && ci < Ci) {
      const int64_t i = ((int64_t)co * taps + tap) * Ci + ci;
      v = w[i];
      if (wf) wf[i] = from_f<T>(v);
    }
    tile[r][tx] = v;
  }
  if (!wd) return;
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int ci = ci0 + r, co = co0 + tx;
    if (co < Co && ci < Ci) wd[((int64_t)ci * taps + (taps - 1 - tap)) * Co + co] = from_f<T>(tile[tx][r]);
  }
}

__global__ void check_finite_k(const float *v, int n, int *flag) {
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!isfinite(v[i])) *flag = 1;
}

}  // namespace

int chan_reduce_blocks(int64_t V, int C) {
  // ~2048 elements per block at least; at most one full wave (3 resident blocks/SM)
  int64_t b = (V * C + 2047) / 2048;
  if (b > 3 * 148) b = 3 * 148;
  if (b < 1) b = 1;
  return (int)b;
}

#define DISPATCH(dt, ...)                      \
  do {                                         \
    if ((dt) == DT_F32) {                      \
      typedef float T;                         \
      __VA_ARGS__;                             \
    } else {                                   \
      typedef bf16 T;                          \
      __VA_ARGS__;                             \
    }                                          \
  } while (0)

void bn_stats(DType dt, const void *x, int64_t V, int C, float *partial, int nblk, cudaStream_t st) {
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    launch_chan_reduce_dims<T>(V, C, nblk, rpb, smem);
    StatsOp<T> op{(const T *)x, C, {}};
    chan_reduce_k<T, StatsOp<T>><<<nblk, NT, smem, st>>>(op, V, C, partial, rpb);
  });
  LAUNCH_CHECK();
}

void bn_finalize(DType dt, const void *x, const float *partial, int nblk, int64_t V, int C, const float *gamma,
                 const float *beta, float *mean, float *invstd, float *scale, float *shift, float *run_mean,
                 float *run_var, float momentum, float eps, cudaStream_t st) {
  DISPATCH(dt, bn_finalize_k<T><<<(C + 7) / 8, 256, 0, st>>>((const T *)x, partial, nblk, V, C, gamma, beta, mean,
                                                             invstd, scale, shift, run_mean, run_var, momentum, eps));
  LAUNCH_CHECK();
}

void bn_apply(DType dt, const void *x, int64_t V, int C, const float *scale, const float *shift, const void *res,
              const float *rscale, const float *rshift, bool relu, void *y, cudaStream_t st) {
  DISPATCH(dt, bn_apply_k<T><<<grid_for(V * C / Vec<T>::N), NT, 0, st>>>(
                   (const T *)x, V, C, scale, shift, (const T *)res, rscale, rshift, relu ? 1 : 0, (T *)y));
  LAUNCH_CHECK();
}

void bn_bwd_reduce(DType dt, const void *dy, const void *x, int64_t V, int C, int mask_mode, const void *mask_t,
                   const float *scale, const float *shift, const float *mean, const float *invstd, float *partial,
                   int nblk, cudaStream_t st) {
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    launch_chan_reduce_dims<T>(V, C, nblk, rpb, smem);
    BwdOp<T> op{(const T *)dy, (const T *)x, (const T *)mask_t, mask_mode, C, scale, shift, mean, invstd};
    chan_reduce_k<T, BwdOp<T>><<<nblk, NT, smem, st>>>(op, V, C, partial, rpb);
  });
  LAUNCH_CHECK();
}

void bn_bwd_finalize(const float *partial, int nblk, int64_t V, int C, const float *gamma, const float *mean,
                     const float *invstd, float *dgamma, float *dbeta, float *coef, cudaStream_t st) {
  bn_bwd_finalize_k<<<(C + 7) / 8, 256, 0, st>>>(partial, nblk, V, C, gamma, mean, invstd, dgamma, dbeta, coef);
  LAUNCH_CHECK();
}

void bn_forward_fused(DType dt, const void *x, int64_t V, int C, float *partial, const float *gamma,
                      const float *beta, float *mean, float *invstd, float *scale, float *shift, float *run_mean,
                      float *run_var, float momentum, float eps, const void *res, const float *rscale,
                      const float *rshift, bool relu, void *y, cudaStream_t st) {
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    const int grid = coop_grid(bn_fwd_fused_k<T>, (size_t)2 * NT * Vec<T>::N * sizeof(float), V, C);
    launch_chan_reduce_dims<T>(V, C, grid, rpb, smem);
    BnFwdArgs<T> a{(const T *)x, V, rpb, C, partial, gamma, beta, mean, invstd, scale, shift, run_mean, run_var,
                   momentum, eps, (const T *)res, rscale, rshift, relu ? 1 : 0, (T *)y};
    coop_launch(bn_fwd_fused_k<T>, grid, smem, a, st);
  });
  count_launch();
}

void bn_backward_fused(DType dt, const void *dy, const void *x, int64_t V, int C, int mask_mode, const void *mask_t,
                       const float *scale, const float *shift, const float *mean, const float *invstd,
                       const float *gamma, float *partial, float *dgamma, float *dbeta, float *coef, void *dx,
                       cudaStream_t st) {
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    const int grid = coop_grid(bn_bwd_fused_k<T>, (size_t)2 * NT * Vec<T>::N * sizeof(float), V, C);
    launch_chan_reduce_dims<T>(V, C, grid, rpb, smem);
    BnBwdArgs<T> a{(const T *)dy, (const T *)x, (const T *)mask_t, V, rpb, C, mask_mode, partial, scale, shift,
                   mean, invstd, gamma, dgamma, dbeta, coef, (T *)dx};
    coop_launch(bn_bwd_fused_k<T>, grid, smem, a, st);
  });
  count_launch();
}

void bn_bwd_apply(DType dt, const void *dy, const void *x, int64_t V, int C, int mask_mode, const void *mask_t,
                  const float *scale, const float *shift, const float *coef, void *dx, cudaStream_t st) {
  DISPATCH(dt, bn_bwd_apply_k<T><<<grid_for(V * C / Vec<T>::N), NT, 0, st>>>(
                   (const T *)dy, (const T *)x, V, C, mask_mode, (const T *)mask_t, scale, shift, coef, (T *)dx));
  LAUNCH_CHECK();
}

void maxpool_fwd(DType dt, const void *x, int N, int D, int H, int W, int C, const float *scale, const float *shift,
                 bool relu, void *y, uint8_t *argmax, int Do, int Ho, int Wo, cudaStream_t st) {
  DISPATCH(dt, maxpool_fwd_k<T><<<grid_for((int64_t)N * Do * Ho * Wo * C / Vec<T>::N), NT, 0, st>>>(
                   (const T *)x, N, D, H, W, C, scale, shift, relu ? 1 : 0, (T *)y, argmax, Do, Ho, Wo));
  LAUNCH_CHECK();
}

void maxpool_bwd(DType dt, const void *dy, const uint8_t *argmax, int N, int D, int H, int W, int C, int Do, int Ho,
                 int Wo, void *dx, bool accumulate, cudaStream_t st) {
  DISPATCH(dt, maxpool_bwd_k<T><<<grid_for((int64_t)N * D * H * W * C / Vec<T>::N), NT, 0, st>>>(
                   (const T *)dy, argmax, N, D, H, W, C, Do, Ho, Wo, (T *)dx, accumulate ? 1 : 0));
  LAUNCH_CHECK();
}

void upsample_fwd(DType dt, const void *x, int N, int Di, int Hi, int Wi, int C, void *y, int Do, int Ho, int Wo,
                  const UpTables &t, cudaStream_t st) {
  DISPATCH(dt, upsample_fwd_k<T><<<grid_for((int64_t)N * Do * Ho * Wo * C / Vec<T>::N), NT, 0, st>>>(
                   (const T *)x, N, Di, Hi, Wi, C, (T *)y, Do, Ho, Wo, t));
  LAUNCH_CHECK();
}

void upsample_bwd(DType dt, const void *dy, int N, int Di, int Hi, int Wi, int C, void *dx, int Do, int Ho, int Wo,
                  const UpTables &t, cudaStream_t st) {
  DISPATCH(dt, upsample_bwd_k<T><<<grid_for((int64_t)N * Di * Hi * Wi * C / Vec<T>::N), NT, 0, st>>>(
                   (const T *)dy, N, Di, Hi, Wi, C, (T *)dx, Do, Ho, Wo, t));
  LAUNCH_CHECK();
}

void att_fwd(DType dt, const void *m, const void *T_, int64_t V, int C, void *out, cudaStream_t st) {
  DISPATCH(dt, att_fwd_k<T><<<grid_for(V * C / Vec<T>::N), NT, 0, st>>>((const T *)m, (const T *)T_, V, C,
                                                                          (T *)out));
  LAUNCH_CHECK();
}

void att_bwd(DType dt, const void *dout, const void *m, const void *T_, int64_t V, int C, void *dT, void *dm,
             float *partial, int nblk, cudaStream_t st) {
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    launch_chan_reduce_dims<T>(V, C, nblk, rpb, smem);
    AttBwdOp<T> op{(const T *)dout, (const T *)m, (const T *)T_, (T *)dT, (T *)dm, C};
    chan_reduce_k<T, AttBwdOp<T>><<<nblk, NT, smem, st>>>(op, V, C, partial, rpb);
  });
  LAUNCH_CHECK();
}

void chan_sum_finalize(const float *partial, int nblk, int C, float *out, cudaStream_t st) {
  chan_sum_finalize_k<<<(C + 7) / 8, 256, 0, st>>>(partial, nblk, C, out);
  LAUNCH_CHECK();
}

void head_fwd(DType dt, const void *x, int N, int V, int C, const float *W, const float *b, const int32_t *y,
              float dz_scale, float loss_scale, float *g, float *dz, float *loss_acc, cudaStream_t st) {
  dim3 grid(N, (C + 255) / 256);
  DISPATCH(dt, gap_k<T><<<grid, 256, 0, st>>>((const T *)x, V, C, g));
  LAUNCH_CHECK();
  ce_k<<<1, 256, 0, st>>>(g, N, C, W, b, y, dz_scale, loss_scale, dz, loss_acc);
  LAUNCH_CHECK();
}

void head_bwd(DType dt, const float *dz, const float *g, const float *W, int N, int V, int C, float *dW, float *db,
              void *dx, cudaStream_t st) {
  head_wgrad_k<<<(2 * C + 255) / 256, 256, 0, st>>>(dz, g, N, C, dW, db);
  LAUNCH_CHECK();
  DISPATCH(dt, head_dx_k<T><<<grid_for((int64_t)N * V * C), 256, 0, st>>>(dz, W, N, V, C, (T *)dx));
  LAUNCH_CHECK();
}

void sgd_update(float *w, const float *g, int64_t n, float lr, cudaStream_t st) {
  sgd_k<<<grid_for((n + 3) / 4), NT, 0, st>>>(w, g, n, lr);
  LAUNCH_CHECK();
}

void repack_conv(DType dt, const float *w, int Co, int taps, int Ci, void *wf, void *wd, cudaStream_t st) {
  dim3 grid((Ci + 31) / 32, (Co + 31) / 32, taps);
  DISPATCH(dt, repack_k<T><<<grid, dim3(32, 8), 0, st>>>(w, Co, taps, Ci, (T *)wf, (T *)wd));
  LAUNCH_CHECK();
}

__global__ void __launch_bounds__(256) sgd_repack_all_k(const ConvPack *__restrict__ tab, int n, float *master,
                                                        const float *__restrict__ grad, float lr) {
  __shared__ float tile[32][33];
  __shared__ int ti;
  const int64_t b = blockIdx.x;
  if (threadIdx.x == 0 && threadIdx.y == 0) {  // tensor of this tile: binary search on tile0
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (tab[mid].tile0 <= b) lo = mid;
      else hi = mid - 1;
    }
    ti = lo;
  }
  __syncthreads();
  const ConvPack t = tab[ti];
  int64_t r = b - t.tile0;
  const int nci = (t.Ci + 31) / 32, nco = (t.Co + 31) / 32;
  const int cit = (int)(r % nci); r /= nci;
  const int cot = (int)(r % nco); r /= nco;
  const int tap = (int)r;
  const int ci0 = cit * 32, co0 = cot * 32, tx = threadIdx.x, ty = threadIdx.y;
  float *w = master + t.off;
  const float *g = grad ? grad + t.off : nullptr;
  bf16 *wf = (bf16 *)t.wf, *wd = (bf16 *)t.wd;
  for (int rr = ty; rr < 32; rr += 8) {
    const int co = co0 + rr, ci = ci0 + tx;
    float v = 0.f;
    if (co < t.Co && ci < t.Ci) {
      const int64_t i = ((int64_t)co * t.taps + tap) * t.Ci + ci;
      v = w[i];
      if (g) {
        v -= lr * g[i];
        w[i] = v;
      }
      wf[i] = __float2bfloat16_rn(v);
    }
    tile[rr][tx] = v;
  }
  __syncthreads();
  for (int rr = ty; rr < 32; rr += 8) {
    const int ci = ci0 + rr, co = co0 + tx;
    if (co < t.Co && ci < t.Ci)
      wd[((int64_t)ci * t.taps + (t.taps - 1 - tap)) * t.Co + co] = __float2bfloat16_rn(tile[tx][rr]);
  }
}

__global__ void sgd_ranges_k(const int64_t *__restrict__ rg, float *master, const float *__restrict__ grad, float lr) {
  const int64_t a = rg[2 * blockIdx.x], e = rg[2 * blockIdx.x + 1];
  for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x) master[i] -= lr * grad[i];
}

template <typename T>
__global__ void flip_k(const T *__restrict__ w, int Co, int taps, int Ci, T *__restrict__ wd) {
  const int64_t n = (int64_t)Co * taps * Ci;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int ci = (int)(i % Ci);
    const int tap = (int)((i / Ci) % taps);
    const int co = (int)(i / ((int64_t)Ci * taps));
    wd[((int64_t)ci * taps + (taps - 1 - tap)) * Co + co] = w[i];
  }
}

void sgd_repack_all(const ConvPack *table_dev, int n, int64_t total_tiles, float *master, const float *grad, float lr,
                    cudaStream_t st) {
  if (n <= 0 || total_tiles <= 0) return;
  sgd_repack_all_k<<<(unsigned)total_tiles, dim3(32, 8), 0, st>>>(table_dev, n, master, grad, lr);
  LAUNCH_CHECK();
}

void sgd_ranges(const int64_t *ranges_dev, int n, float *master, const float *grad, float lr, cudaStream_t st) {
  if (n <= 0) return;
  sgd_ranges_k<<<n, 256, 0, st>>>(ranges_dev, master, grad, lr);
  LAUNCH_CHECK();
}

void flip_weights(DType dt, const void *w, int Co, int taps, int Ci, void *wd, cudaStream_t st) {
  DISPATCH(dt, flip_k<T><<<grid_for((int64_t)Co * taps * Ci), NT, 0, st>>>((const T *)w, Co, taps, Ci, (T *)wd));
  LAUNCH_CHECK();
}

void check_finite(const float *v, int n, int *flag, cudaStream_t st) {
  check_finite_k<<<1, 256, 0, st>>>(v, n, flag);
  LAUNCH_CHECK();
}

}  // namespace rn
