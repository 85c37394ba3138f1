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
#include <cuda_bf16.h>

#include <algorithm>

#include "error.h"
#include "launch.h"
#include "kernels.h"
#include "util.cuh"

namespace rn {

namespace {

constexpr int NT = 256;

inline unsigned grid_for(int64_t items, int per_block = NT, int64_t cap = 148 * 32) {
  int64_t b = (items + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// ---------------------------------------------------------------------------
// Per-channel reductions over the rows (voxels) of an NDHWC tensor, with the
// finalize in the same launch.  Block b reduces rows [b*rpb, (b+1)*rpb): each
// thread owns one 16-byte channel vector and walks rows RPI apart, loading
// U rows before accumulating (all U loads in flight: memory-level parallelism),
// then a fixed-order smem tree gives the block's partial [2][C].  The last block
// to finish (atomic ticket, reset afterwards for the next launch / graph
// replay) sums all partials in block order — fixed order, so the result is
// deterministic (reading X24) — and applies `fin` per channel.  The partials
// are read with plain weak loads after the ticket's __threadfence (which also
// invalidates L1): strong ld.global.cg loads measured fully serialised on B200
// (~0.3 us each, 45 us for 148 partials).
// ---------------------------------------------------------------------------
constexpr int NTR = 512;  // threads of a reduction block
constexpr int RU = 8;     // rows in flight per thread

// 16-byte read-only load as a volatile asm: the compiler keeps a batch of these
// ahead of the arithmetic that consumes them (plain __ldg loads were sunk next
// to their uses, one L2/HBM round trip per row)
template <typename T>
__device__ __forceinline__ uint4 ld16(const T *p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void unpack16(const uint4 &u, float *v, const float *) {
  v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y); v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void unpack16(const uint4 &u, float *v, const bf16 *) {
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

template <typename T, typename Op>
__device__ __forceinline__ void chan_reduce_body(Op &op, int64_t V, int C, float *__restrict__ partial, int64_t rpb,
                                                 float *sm) {
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int RPI = NTR / G;
  const int t = threadIdx.x, rr = t / G, c0 = (t % G) * VEC;
  float a1[VEC], a2[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) a1[j] = a2[j] = 0.f;
  if (rr < RPI) {
    op.init(c0);
    const int64_t r0 = (int64_t)blockIdx.x * rpb;
    const int64_t r1 = min(V, r0 + rpb);
    int64_t r = r0 + rr;
    for (; r < r1; r += RU * RPI) {  // the last batch is predicated, not a serial remainder
      typename Op::Buf b[RU];
#pragma unroll
      for (int q = 0; q < RU; ++q)
        if (r + q * RPI < r1) op.load(r + q * RPI, c0, b[q]);
#pragma unroll
      for (int q = 0; q < RU; ++q)
        if (r + q * RPI < r1) op.acc(b[q], r + q * RPI, c0, a1, a2);
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      sm[rr * C + c0 + j] = a1[j];
      sm[RPI * C + rr * C + c0 + j] = a2[j];
    }
  }
  __syncthreads();
  for (int c = t; c < C; c += NTR) {
    float s1 = 0.f, s2 = 0.f;
    for (int q = 0; q < RPI; ++q) {
      s1 += sm[q * C + c];
      s2 += sm[RPI * C + q * C + c];
    }
    partial[(int64_t)blockIdx.x * 2 * C + c] = s1;
    partial[(int64_t)blockIdx.x * 2 * C + C + c] = s2;
  }
}

// per-block partials only (the BN apply kernels finalize them: bn_*_part_k)
template <typename T, typename Op>
__global__ void __launch_bounds__(NTR) chan_partials_k(Op op, int64_t V, int C, float *__restrict__ partial,
                                                       int64_t rpb) {
  extern __shared__ float sm[];
  pdl_begin();
  chan_reduce_body<T>(op, V, C, partial, rpb, sm);
}

template <typename T, typename Op, typename Fin>
__global__ void __launch_bounds__(NTR) chan_reduce_fin_k(Op op, Fin fin, int64_t V, int C, float *__restrict__ partial,
                                                         int64_t rpb, unsigned *counter) {
  extern __shared__ float sm[];
  pdl_begin();
  chan_reduce_body<T>(op, V, C, partial, rpb, sm);
  const int t = threadIdx.x;
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (t == 0) is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double *dsm = reinterpret_cast<double *>(sm);  // 2 * NTR doubles <= the reduce scratch
  const int Cb = C < NTR ? C : NTR, P = NTR / Cb;
  const int s = t / Cb, cc = t % Cb;
  const int nb = (int)gridDim.x;
  for (int cb = 0; cb < C; cb += Cb) {
    const int c = cb + cc;
    if (s < P && c < C) {
      // batches of 8 independent loads per operand: one L2 round trip per batch
      double a = 0.0, b = 0.0;
      for (int k0 = s; k0 < nb; k0 += 8 * P) {
        float va[8], vb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = k0 + j * P;
          va[j] = k < nb ? partial[(int64_t)k * 2 * C + c] : 0.f;
          vb[j] = k < nb ? partial[(int64_t)k * 2 * C + C + c] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          a += (double)va[j];
          b += (double)vb[j];
        }
      }
      dsm[s * Cb + cc] = a;
      dsm[NTR + s * Cb + cc] = b;
    }
    __syncthreads();
    if (s == 0 && c < C) {
      double A = 0.0, B = 0.0;
      for (int q = 0; q < P; ++q) {
        A += dsm[q * Cb + cc];
        B += dsm[NTR + q * Cb + cc];
      }
      fin(c, A, B);
    }
    __syncthreads();
  }
  if (t == 0) *counter = 0u;
}

template <typename T>
void chan_reduce_dims(int64_t V, int C, int nblk, int64_t &rpb, size_t &smem) {
  const int G = C / Vec<T>::N;
  const int RPI = NTR / G;
  rpb = (V + nblk - 1) / nblk;
  smem = std::max((size_t)2 * RPI * C * sizeof(float), (size_t)2 * NTR * sizeof(double));
}

// forward statistics of x, shifted by K = x[0][c] (cancellation-safe variance)
template <typename T>
struct StatsOp {
  const T *x;
  int C;
  float K[Vec<T>::N];
  struct Buf {
    uint4 v;
  };
  bool shifted = true;  // false: plain sums (the convention of the fused conv-epilogue partials)
  __device__ void init(int c0) {
    if (shifted) load_vec(x + c0, K);
    else
#pragma unroll
      for (int j = 0; j < Vec<T>::N; ++j) K[j] = 0.f;
  }
  __device__ void load(int64_t r, int c0, Buf &b) const { b.v = ld16(x + r * C + c0); }
  __device__ void acc(const Buf &b, int64_t, int, float *a1, float *a2) const {
    float v[Vec<T>::N];
    unpack16(b.v, v, x);
#pragma unroll
    for (int j = 0; j < Vec<T>::N; ++j) {
      const float d = v[j] - K[j];
      a1[j] += d;
      a2[j] = fmaf(d, d, a2[j]);
    }
  }
};

// BN backward sums over dy' = dy * mask: (sum dy', sum dy' * xhat)
template <typename T>
struct BwdOp {
  const T *dy, *x, *mask_t;
  int mode, C;
  const float *scale, *shift, *mean, *invstd;
  struct Buf {
    uint4 d, x, m;
  };
  __device__ void init(int) {}
  __device__ void load(int64_t r, int c0, Buf &b) const {
    const int64_t off = r * C + c0;
    b.d = ld16(dy + off);
    b.x = ld16(x + off);
    if (mode == MASK_TENSOR) b.m = ld16(mask_t + off);
  }
  __device__ void acc(const Buf &b, int64_t, int c0, float *a1, float *a2) const {
    constexpr int VEC = Vec<T>::N;
    float d[VEC], xv[VEC];
    unpack16(b.d, d, dy);
    unpack16(b.x, xv, x);
    if (mode == MASK_TENSOR) {
      float m[VEC];
      unpack16(b.m, m, x);
#pragma unroll
      for (int j = 0; j < VEC; ++j) d[j] = m[j] > 0.f ? d[j] : 0.f;
    } else if (mode == MASK_RECOMPUTE) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) d[j] = fmaf(xv[j], scale[c0 + j], shift[c0 + j]) > 0.f ? d[j] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const float xh = (xv[j] - mean[c0 + j]) * invstd[c0 + j];
      a1[j] += d[j];
      a2[j] = fmaf(d[j], xh, a2[j]);
    }
  }
};

// BN backward sums in the fused-partials convention: (sum dy', sum dy' (h - mean)), dy' = dy * (mask > 0)
template <typename T>
struct BwdHOp {
  const T *dy, *x, *mask_t;
  int C;
  const float *mean;
  float mu[Vec<T>::N];  // this thread's channels (fixed per thread)
  struct Buf {
    uint4 d, x, m;
  };
  __device__ void init(int c0) {
#pragma unroll
    for (int j = 0; j < Vec<T>::N; ++j) mu[j] = mean[c0 + j];
  }
  __device__ void load(int64_t r, int c0, Buf &b) const {
    const int64_t off = r * C + c0;
    b.d = ld16(dy + off);
    b.x = ld16(x + off);
    b.m = ld16(mask_t + off);
  }
  __device__ void acc(const Buf &b, int64_t, int c0, float *a1, float *a2) const {
    constexpr int VEC = Vec<T>::N;
    float d[VEC], xv[VEC], m[VEC];
    unpack16(b.d, d, dy);
    unpack16(b.x, xv, x);
    unpack16(b.m, m, x);
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const float dd = m[j] > 0.f ? d[j] : 0.f;
      a1[j] += dd;
      a2[j] = fmaf(dd, xv[j] - mu[j], a2[j]);
    }
  }
};

// attention backward: dT = dout (1 + s), dm = dout T s (1 - s), s = sigmoid(m); sums dm
template <typename T>
struct AttBwdOp {
  const T *dout, *m, *Tt;
  T *dT, *dm;
  int C;
  struct Buf {
    uint4 g, m, t;
  };
  __device__ void init(int) {}
  __device__ void load(int64_t r, int c0, Buf &b) const {
    const int64_t off = r * C + c0;
    b.g = ld16(dout + off);
    b.m = ld16(m + off);
    b.t = ld16(Tt + off);
  }
  __device__ void acc(const Buf &b, int64_t r, int c0, float *a1, float *) const {
    constexpr int VEC = Vec<T>::N;
    float g[VEC], mv[VEC], tv[VEC], o1[VEC], o2[VEC];
    unpack16(b.g, g, dout);
    unpack16(b.m, mv, m);
    unpack16(b.t, tv, Tt);
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const float s = 1.f / (1.f + __expf(-mv[j]));
      o1[j] = g[j] * (1.f + s);
      o2[j] = g[j] * tv[j] * s * (1.f - s);
    }
    const int64_t off = r * C + c0;
    store_vec(dT + off, o1);
    store_vec(dm + off, o2);
#pragma unroll
    for (int j = 0; j < VEC; ++j) a1[j] += o2[j];
  }
};

// forward statistics -> mean / invstd / scale / shift, running-stat momentum update
template <typename T>
struct StatsFin {
  const T *x;
  int64_t V;
  const float *gamma, *beta;
  float *mean, *invstd, *scale, *shift, *run_mean, *run_var;
  float momentum, eps;
  __device__ void operator()(int c, double S, double Q) const {
    const double K = (double)to_f(x[c]);  // the shift of StatsOp
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
};

// backward sums (S1 = sum dy', S2 = sum dy' xhat) -> dgamma, dbeta, dx coefficients
// dx = A dy' + B x + Cc with A = gamma invstd, B = -A invstd S2/V, Cc = -A S1/V + A invstd mean S2/V
struct BwdFin {
  int64_t V;
  int C;
  const float *gamma, *mean, *invstd;
  float *dgamma, *dbeta, *coef;
  __device__ void operator()(int c, double S1, double S2) const {
    dgamma[c] += (float)S2;
    dbeta[c] += (float)S1;
    const double m1 = S1 / (double)V, m2 = S2 / (double)V;
    const double is = invstd[c];
    const double A = (double)gamma[c] * is;
    coef[c] = (float)A;
    coef[C + c] = (float)(-A * is * m2);
    coef[2 * C + c] = (float)(-A * m1 + A * is * (double)mean[c] * m2);
  }
};

struct SumFin {
  float *out;
  __device__ void operator()(int c, double S1, double) const { out[c] += (float)S1; }
};

// Elementwise BN passes: each thread owns a fixed 16-byte channel vector
// (grid stride is a multiple of C/VEC, so its per-channel coefficients stay in
// registers) and loads EU vectors before computing (memory-level parallelism).
constexpr int EU = 4;

// blocks rounded to a multiple of G / gcd(G, threads): the grid stride must be a
// multiple of the G = C/VEC channel vectors of a voxel (C = 24 has G = 3)
inline int64_t stride_multiple(int64_t b, int threads, int G) {
  int a = G, c = threads;
  while (c) { const int t = a % c; a = c; c = t; }
  const int64_t m = G / a;
  return (b + m - 1) / m * m;
}

inline unsigned grid_elem(int64_t vecs, int G) {
  int64_t b = (vecs + (int64_t)NT * EU - 1) / ((int64_t)NT * EU);
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  return (unsigned)stride_multiple(b, NT, G);
}

// y = act(x*scale + shift + R), R = 0 | res | res*rscale + rshift
template <typename T>
__global__ void __launch_bounds__(NT) bn_apply_k(const T *__restrict__ x, int64_t V, int C,
                                                 const float *__restrict__ scale, const float *__restrict__ shift,
                                                 const T *__restrict__ res, const float *__restrict__ rscale,
                                                 const float *__restrict__ rshift, int relu, T *__restrict__ y) {
  pdl_begin();
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = V * G;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c0 = (int)(i0 % G) * VEC;
  float sc[VEC], sh[VEC], rs[VEC], rh[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    sc[j] = scale[c0 + j];
    sh[j] = shift[c0 + j];
    rs[j] = rscale ? rscale[c0 + j] : 1.f;
    rh[j] = rscale ? rshift[c0 + j] : 0.f;
  }
  for (int64_t i = i0; i < n; i += EU * stride) {
    uint4 xv[EU], rv[EU];
#pragma unroll
    for (int q = 0; q < EU; ++q) {
      const int64_t k = i + q * stride;
      if (k < n) {
        xv[q] = ld16(x + k * VEC);
        if (res) rv[q] = ld16(res + k * VEC);
      }
    }
#pragma unroll
    for (int q = 0; q < EU; ++q) {
      const int64_t k = i + q * stride;
      if (k >= n) break;
      float v[VEC];
      unpack16(xv[q], v, x);
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = fmaf(v[j], sc[j], sh[j]);
      if (res) {
        float r[VEC];
        unpack16(rv[q], r, x);
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] += fmaf(r[j], rs[j], rh[j]);
      }
      if (relu) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] = fmaxf(v[j], 0.f);
      }
      store_vec(y + k * VEC, v);
    }
  }
}

// dx = A dy' + B x + Cc, dy' = dy * mask (mask tensor > 0, or recomputed ReLU of BN(x))
template <typename T>
__global__ void __launch_bounds__(NT) bn_bwd_apply_k(const T *__restrict__ dy, const T *__restrict__ x, int64_t V,
                                                     int C, int mode, const T *__restrict__ mask_t,
                                                     const float *__restrict__ scale, const float *__restrict__ shift,
                                                     const float *__restrict__ coef, T *__restrict__ dx) {
  pdl_begin();
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = V * G;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c0 = (int)(i0 % G) * VEC;
  float A[VEC], B[VEC], Cc[VEC], sc[VEC], sh[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    A[j] = coef[c0 + j];
    B[j] = coef[C + c0 + j];
    Cc[j] = coef[2 * C + c0 + j];
    sc[j] = mode == MASK_RECOMPUTE ? scale[c0 + j] : 0.f;
    sh[j] = mode == MASK_RECOMPUTE ? shift[c0 + j] : 0.f;
  }
  for (int64_t i = i0; i < n; i += EU * stride) {
    uint4 dv[EU], xv[EU], mv[EU];
#pragma unroll
    for (int q = 0; q < EU; ++q) {
      const int64_t k = i + q * stride;
      if (k < n) {
        dv[q] = ld16(dy + k * VEC);
        xv[q] = ld16(x + k * VEC);
        if (mode == MASK_TENSOR) mv[q] = ld16(mask_t + k * VEC);
      }
    }
#pragma unroll
    for (int q = 0; q < EU; ++q) {
      const int64_t k = i + q * stride;
      if (k >= n) break;
      float d[VEC], xf[VEC], o[VEC];
      unpack16(dv[q], d, dy);
      unpack16(xv[q], xf, x);
      if (mode == MASK_TENSOR) {
        float m[VEC];
        unpack16(mv[q], m, x);
#pragma unroll
        for (int j = 0; j < VEC; ++j) d[j] = m[j] > 0.f ? d[j] : 0.f;
      } else if (mode == MASK_RECOMPUTE) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) d[j] = fmaf(xf[j], sc[j], sh[j]) > 0.f ? d[j] : 0.f;
      }
#pragma unroll
      for (int j = 0; j < VEC; ++j) o[j] = fmaf(A[j], d[j], fmaf(B[j], xf[j], Cc[j]));
      store_vec(dx + k * VEC, o);
    }
  }
}

// ---------------------------------------------------------------------------
// BN apply passes fed by per-CTA statistics partials of the producing
// convolution (bnstats.cuh).  Every block finalizes the statistics it needs in
// its prologue (all partials, CTA order, fp64: identical in every block, so
// deterministic) and block 0 publishes them (mean / invstd / scale / shift,
// running statistics; dgamma / dbeta in backward).  No separate statistics pass
// over the tensor and no serial finalize launch.
// ---------------------------------------------------------------------------
constexpr int NTA = 512;

// BN statistics finalized once per layer by a small kernel (RN_BN_FIN_SEPARATE=1)
// instead of in every apply block's prologue (default: measured equal within run
// noise, 2186-2227 vs 2194-2227 samples/s, and one launch fewer per BN)
static bool bn_fin_separate() {
  static const bool v = getenv("RN_BN_FIN_SEPARATE") && atoi(getenv("RN_BN_FIN_SEPARATE")) != 0;
  return v;
}

// per-channel sums over the P partials [P][2][C] -> dscr[0..C) / dscr[C..2C) (fp64)
__device__ __forceinline__ void reduce_partials(const float *part, int P, int C, double *out, double *scr) {
  const int t = threadIdx.x, nt = blockDim.x;
  const int Cb = C < nt ? C : nt, S = nt / Cb;
  for (int cb = 0; cb < C; cb += Cb) {
    const int c = cb + t % Cb, s = t / Cb;
    if (s < S && c < C) {
      // fp32 chain within a batch of 8 (short dependent-add latency), fp64 across batches
      double a = 0.0, b = 0.0;
      for (int k0 = s; k0 < P; k0 += 8 * S) {
        float va[8], vb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = k0 + j * S;
          va[j] = k < P ? part[(int64_t)k * 2 * C + c] : 0.f;
          vb[j] = k < P ? part[(int64_t)k * 2 * C + C + c] : 0.f;
        }
        float fa = 0.f, fb = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          fa += va[j];
          fb += vb[j];
        }
        a += (double)fa;
        b += (double)fb;
      }
      scr[s * Cb + t % Cb] = a;
      scr[nt + s * Cb + t % Cb] = b;
    }
    __syncthreads();
    if (s == 0 && c < C) {
      double A = 0.0, B = 0.0;
      for (int q = 0; q < S; ++q) {
        A += scr[q * Cb + t % Cb];
        B += scr[nt + q * Cb + t % Cb];
      }
      out[c] = A;
      out[C + c] = B;
    }
    __syncthreads();
  }
}

struct BnPart {
  const float *part;  // [P][2][C]: (sum y, sum y^2) of the stored conv output
  int P;
  int64_t V;
  const float *gamma, *beta;
  float *mean, *invstd, *scale, *shift, *run_mean, *run_var;
  float momentum, eps;
};

// sc/sh (smem) = scale/shift of the set; block 0 publishes the statistics
__device__ __forceinline__ void bn_part_finalize(const BnPart &b, int C, float *sc, float *sh, double *sums,
                                                 double *scr) {
  reduce_partials(b.part, b.P, C, sums, scr);
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const double mu = sums[c] / (double)b.V;
    double var = sums[C + c] / (double)b.V - mu * mu;
    if (var < 0) var = 0;
    const double is = 1.0 / sqrt(var + (double)b.eps);
    const double scd = (double)b.gamma[c] * is;
    const float s_ = (float)scd, h_ = (float)((double)b.beta[c] - mu * scd);
    sc[c] = s_;
    sh[c] = h_;
    if (blockIdx.x == 0) {
      b.mean[c] = (float)mu;
      b.invstd[c] = (float)is;
      b.scale[c] = s_;
      b.shift[c] = h_;
      if (b.run_mean) {
        const double unb = b.V > 1 ? var * (double)b.V / (double)(b.V - 1) : var;
        b.run_mean[c] = (float)((1.0 - b.momentum) * b.run_mean[c] + b.momentum * mu);
        b.run_var[c] = (float)((1.0 - b.momentum) * b.run_var[c] + b.momentum * unb);
      }
    }
  }
  __syncthreads();
}

// One finalize per BN layer (instead of every apply block reducing all P
// partials in its prologue): block = 32 channels, warp w sums partials
// k = w, w+8, ... in fp64 (fixed order), warp 0 combines the 8 warps in order and
// finalizes exactly as bn_part_finalize (mean / invstd / scale / shift, running
// statistics).  The apply kernels then read scale / shift (b.P < 0).
__global__ void __launch_bounds__(256) bn_fin_fwd_k(BnPart b, int C) {
  __shared__ double red[8][2][32];
  pdl_begin();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double s1 = 0.0, s2 = 0.0;
  if (c < C)
    for (int k = w; k < b.P; k += 8) {
      s1 += (double)b.part[(int64_t)k * 2 * C + c];
      s2 += (double)b.part[(int64_t)k * 2 * C + C + c];
    }
  red[w][0][lane] = s1;
  red[w][1][lane] = s2;
  __syncthreads();
  if (w == 0 && c < C) {
    double S1 = 0.0, S2 = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      S1 += red[q][0][lane];
      S2 += red[q][1][lane];
    }
    const double mu = S1 / (double)b.V;
    double var = S2 / (double)b.V - mu * mu;
    if (var < 0) var = 0;
    const double is = 1.0 / sqrt(var + (double)b.eps);
    const double scd = (double)b.gamma[c] * is;
    b.mean[c] = (float)mu;
    b.invstd[c] = (float)is;
    b.scale[c] = (float)scd;
    b.shift[c] = (float)((double)b.beta[c] - mu * scd);
    if (b.run_mean) {
      const double unb = b.V > 1 ? var * (double)b.V / (double)(b.V - 1) : var;
      b.run_mean[c] = (float)((1.0 - b.momentum) * b.run_mean[c] + b.momentum * mu);
      b.run_var[c] = (float)((1.0 - b.momentum) * b.run_var[c] + b.momentum * unb);
    }
  }
}

// sc/sh (smem) from statistics finalized by bn_fin_fwd_k (b.P < 0) or from the partials
__device__ __forceinline__ void bn_part_coefs(const BnPart &b, int C, float *sc, float *sh, double *sums,
                                              double *scr) {
  if (b.P >= 0) {
    bn_part_finalize(b, C, sc, sh, sums, scr);
    return;
  }
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    sc[c] = b.scale[c];
    sh[c] = b.shift[c];
  }
  __syncthreads();
}

// y = act(x*scale + shift + R), R = 0 | res | BN_r(res) (set r.part != null)
template <typename T>
__global__ void __launch_bounds__(NTA) bn_apply_part_k(const T *__restrict__ x, int64_t V, int C, BnPart b,
                                                       BnPart rb, const T *__restrict__ res, int relu,
                                                       T *__restrict__ y) {
  extern __shared__ double dsm[];
  constexpr int EUA = 8;  // rows in flight per thread (stage-1 tensors: one 512-thread block per SM)
  pdl_begin();
  double *sums = dsm, *scr = dsm + 2 * C;  // 2C + 2*NTA doubles
  float *fs = (float *)(scr + 2 * NTA);     // sc, sh, rsc, rsh: 4C floats
  float *sc = fs, *sh = fs + C, *rsc = fs + 2 * C, *rsh = fs + 3 * C;
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = V * G;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // multiple of G
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c0 = (int)(i0 % G) * VEC;
  // the first batch of the stream is in flight while the statistics are finalized
  uint4 xv[EUA], rv[EUA];
#pragma unroll
  for (int q = 0; q < EUA; ++q) {
    const int64_t k = i0 + q * stride;
    if (k < n) {
      xv[q] = ld16(x + k * VEC);
      if (res) rv[q] = ld16(res + k * VEC);
    }
  }
  bn_part_coefs(b, C, sc, sh, sums, scr);
  const bool rbn = rb.part != nullptr;
  if (rbn) bn_part_coefs(rb, C, rsc, rsh, sums, scr);
  float a[VEC], bb[VEC], ra[VEC], rbv[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    a[j] = sc[c0 + j];
    bb[j] = sh[c0 + j];
    ra[j] = rbn ? rsc[c0 + j] : 1.f;
    rbv[j] = rbn ? rsh[c0 + j] : 0.f;
  }
  for (int64_t i = i0; i < n; i += EUA * stride) {
    if (i != i0) {
#pragma unroll
      for (int q = 0; q < EUA; ++q) {
        const int64_t k = i + q * stride;
        if (k < n) {
          xv[q] = ld16(x + k * VEC);
          if (res) rv[q] = ld16(res + k * VEC);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < EUA; ++q) {
      const int64_t k = i + q * stride;
      if (k >= n) break;
      float v[VEC];
      unpack16(xv[q], v, x);
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = fmaf(v[j], a[j], bb[j]);
      if (res) {
        float r[VEC];
        unpack16(rv[q], r, x);
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] += fmaf(r[j], ra[j], rbv[j]);
      }
      if (relu) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] = fmaxf(v[j], 0.f);
      }
      store_vec(y + k * VEC, v);
    }
  }
}

struct BnBwdPart {
  const float *part;  // [P][2][C]: (sum dy', sum dy' (h - mean)), dy' = dy * (mask > 0)
  int P;              // < 0: coefficients precomputed by bn_fin_bwd_k into coef
  int64_t V;
  const float *gamma, *mean, *invstd;
  float *dgamma, *dbeta;
  float *coef;        // [3][C] (A, B, Cc) when P < 0
};

// backward finalize (one per BN layer, as bn_fin_fwd_k): dx = A dy' + B h + Cc,
// A = gamma*invstd, B = -A*invstd*m2, Cc = -A*m1 + A*invstd*mean*m2 with
// m1 = mean(dy'), m2 = mean(dy' * xhat); dgamma += S2, dbeta += S1
__global__ void __launch_bounds__(256) bn_fin_bwd_k(BnBwdPart b, int C) {
  __shared__ double red[8][2][32];
  pdl_begin();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double s1 = 0.0, s2 = 0.0;
  if (c < C)
    for (int k = w; k < b.P; k += 8) {
      s1 += (double)b.part[(int64_t)k * 2 * C + c];
      s2 += (double)b.part[(int64_t)k * 2 * C + C + c];
    }
  red[w][0][lane] = s1;
  red[w][1][lane] = s2;
  __syncthreads();
  if (w == 0 && c < C) {
    double S1 = 0.0, S2r = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      S1 += red[q][0][lane];
      S2r += red[q][1][lane];
    }
    const double is = b.invstd[c], mu = b.mean[c];
    const double S2 = is * S2r;  // sum dy' * xhat
    const double m1 = S1 / (double)b.V, m2 = S2 / (double)b.V;
    const double A = (double)b.gamma[c] * is;
    b.coef[c] = (float)A;
    b.coef[C + c] = (float)(-A * is * m2);
    b.coef[2 * C + c] = (float)(-A * m1 + A * is * mu * m2);
    b.dgamma[c] += (float)S2;
    b.dbeta[c] += (float)S1;
  }
}

// dx = A dy' + B h + Cc with the coefficients finalized from the partials
template <typename T>
__global__ void __launch_bounds__(NTA) bn_bwd_apply_part_k(const T *__restrict__ dy, const T *__restrict__ h,
                                                           const T *__restrict__ mask_t, int64_t V, int C,
                                                           BnBwdPart b, T *__restrict__ dx, T *__restrict__ dp) {
  extern __shared__ double dsm[];
  pdl_begin();
  double *sums = dsm, *scr = dsm + 2 * C;
  float *fs = (float *)(scr + 2 * NTA);
  float *cA = fs, *cB = fs + C, *cC = fs + 2 * C;
  constexpr int VEC = Vec<T>::N;
  const int G = C / VEC;
  const int64_t n = V * G;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c0 = (int)(i0 % G) * VEC;
  // the first batch of the stream is in flight while the coefficients are finalized
  uint4 dv[EU], xv[EU], mv[EU];
#pragma unroll
  for (int q = 0; q < EU; ++q) {
    const int64_t k = i0 + q * stride;
    if (k < n) {
      dv[q] = ld16(dy + k * VEC);
      xv[q] = ld16(h + k * VEC);
      mv[q] = ld16(mask_t + k * VEC);
    }
  }
  if (b.P < 0) {
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      cA[c] = b.coef[c];
      cB[c] = b.coef[C + c];
      cC[c] = b.coef[2 * C + c];
    }
  } else {
  reduce_partials(b.part, b.P, C, sums, scr);
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const double S1 = sums[c], is = b.invstd[c], mu = b.mean[c];
    const double S2 = is * sums[C + c];  // sum dy' * xhat
    const double m1 = S1 / (double)b.V, m2 = S2 / (double)b.V;
    const double A = (double)b.gamma[c] * is;
    cA[c] = (float)A;
    cB[c] = (float)(-A * is * m2);
    cC[c] = (float)(-A * m1 + A * is * mu * m2);
    if (blockIdx.x == 0) {
      b.dgamma[c] += (float)S2;
      b.dbeta[c] += (float)S1;
    }
  }
  }
  __syncthreads();
  float A[VEC], B[VEC], Cc[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    A[j] = cA[c0 + j];
    B[j] = cB[c0 + j];
    Cc[j] = cC[c0 + j];
  }
  for (int64_t i = i0; i < n; i += EU * stride) {
    if (i != i0) {
#pragma unroll
      for (int q = 0; q < EU; ++q) {
        const int64_t k = i + q * stride;
        if (k < n) {
          dv[q] = ld16(dy + k * VEC);
          xv[q] = ld16(h + k * VEC);
          mv[q] = ld16(mask_t + k * VEC);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < EU; ++q) {
      const int64_t k = i + q * stride;
      if (k >= n) break;
      float d[VEC], xf[VEC], m[VEC], o[VEC];
      unpack16(dv[q], d, dy);
      unpack16(xv[q], xf, h);
      unpack16(mv[q], m, h);
      float dd[VEC];
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        dd[j] = m[j] > 0.f ? d[j] : 0.f;
        o[j] = fmaf(A[j], dd[j], fmaf(B[j], xf[j], Cc[j]));
      }
      store_vec(dx + k * VEC, o);
      if (dp) store_vec(dp + k * VEC, dd);  // dy' (exact: dy or 0) for a later accumulate
    }
  }
}

// ---------------------------------------------------------------------------
// Channel-sliced BN apply (default; RN_BN_APPLY_CS=0 falls back to the kernels
// above).  Block = (slice of CS = 16 channels, chunk of voxel rows): it finalizes
// only its 16 channels — 16 splits x 16 channels of threads, partials
// k = s, s+16, ... of channel j summed in batches of 8 in fp32, fp64 across
// batches and splits in fixed order (so every block of a slice computes the same
// coefficients) — instead of every block reducing all P x 2C partials (the
// prologue that dominated the apply: 4-8 us per launch, most of a stage-3/4
// apply).  Rows are read 32 B (bf16) / 64 B (fp32) per slice: full sectors.
// The chunk-0 block of a slice publishes its statistics / dgamma, dbeta.
// ---------------------------------------------------------------------------
constexpr int CS = 16, NTS = 256, CS_SPLIT = NTS / CS;

// fp64 per-channel sums (a, b) of the slice's 16 channels over P partials [P][2][C]
__device__ __forceinline__ void cs_sums(const float *part, int P, int C, int c0, double (*red)[NTS], double *sa,
                                        double *sb) {
  const int j = threadIdx.x % CS, sp = threadIdx.x / CS;
  const int c = c0 + j;
  double a = 0.0, b = 0.0;
  for (int k0 = sp; k0 < P; k0 += 8 * CS_SPLIT) {
    float va[8], vb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int k = k0 + i * CS_SPLIT;
      va[i] = k < P ? __ldcg(part + (int64_t)k * 2 * C + c) : 0.f;
      vb[i] = k < P ? __ldcg(part + (int64_t)k * 2 * C + C + c) : 0.f;
    }
    float fa = 0.f, fb = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      fa += va[i];
      fb += vb[i];
    }
    a += (double)fa;
    b += (double)fb;
  }
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x < CS) {
    double A = 0.0, B = 0.0;
#pragma unroll
    for (int q = 0; q < CS_SPLIT; ++q) {
      A += red[0][q * CS + threadIdx.x];
      B += red[1][q * CS + threadIdx.x];
    }
    sa[threadIdx.x] = A;
    sb[threadIdx.x] = B;
  }
}

// scale / shift of the slice's channels (smem), published by the chunk-0 block
__device__ __forceinline__ void cs_coefs_fwd(const BnPart &q, int C, int c0, bool publish, double (*red)[NTS],
                                             double *sa, double *sb, float *sc, float *sh) {
  if (q.P >= 0) {
    cs_sums(q.part, q.P, C, c0, red, sa, sb);
    if (threadIdx.x < CS) {
      const int c = c0 + threadIdx.x;
      const double mu = sa[threadIdx.x] / (double)q.V;
      double var = sb[threadIdx.x] / (double)q.V - mu * mu;
      if (var < 0) var = 0;
      const double is = 1.0 / sqrt(var + (double)q.eps);
      const double scd = (double)q.gamma[c] * is;
      const float s_ = (float)scd, h_ = (float)((double)q.beta[c] - mu * scd);
      sc[threadIdx.x] = s_;
      sh[threadIdx.x] = h_;
      if (publish) {
        q.mean[c] = (float)mu;
        q.invstd[c] = (float)is;
        q.scale[c] = s_;
        q.shift[c] = h_;
        if (q.run_mean) {
          const double unb = q.V > 1 ? var * (double)q.V / (double)(q.V - 1) : var;
          q.run_mean[c] = (float)((1.0 - q.momentum) * q.run_mean[c] + q.momentum * mu);
          q.run_var[c] = (float)((1.0 - q.momentum) * q.run_var[c] + q.momentum * unb);
        }
      }
    }
  } else if (threadIdx.x < CS) {
    sc[threadIdx.x] = q.scale[c0 + threadIdx.x];
    sh[threadIdx.x] = q.shift[c0 + threadIdx.x];
  }
  __syncthreads();
}

// y = act(x*scale + shift + R) over the slice's channels, R = 0 | res | BN_r(res)
template <typename T>
__global__ void __launch_bounds__(NTS) bn_apply_cs_k(const T *__restrict__ x, int64_t V, int C, BnPart b, BnPart rb,
                                                     const T *__restrict__ res, int relu, T *__restrict__ y,
                                                     int nslice, int64_t rows_per_chunk) {
  __shared__ double red[2][NTS];
  __shared__ double sa[CS], sb[CS];
  __shared__ float sc[CS], sh[CS], rsc[CS], rsh[CS];
  constexpr int VEC = Vec<T>::N, VPR = CS / VEC, RPI = NTS / VPR;
  const int slice = blockIdx.x % nslice, chunk = blockIdx.x / nslice;
  const int c0 = slice * CS;
  const int64_t r0 = (int64_t)chunk * rows_per_chunk, r1 = min(V, r0 + rows_per_chunk);
  const int vi = threadIdx.x % VPR, rr = threadIdx.x / VPR;
  const int cv = c0 + vi * VEC;
  pdl_begin();
  // the first batch of rows is in flight while the coefficients are finalized
  uint4 xv[EU], rv[EU];
#pragma unroll
  for (int q = 0; q < EU; ++q) {
    const int64_t r = r0 + rr + (int64_t)q * RPI;
    if (r < r1) {
      xv[q] = ld16(x + r * C + cv);
      if (res) rv[q] = ld16(res + r * C + cv);
    }
  }
  cs_coefs_fwd(b, C, c0, chunk == 0, red, sa, sb, sc, sh);
  const bool rbn = rb.part != nullptr;
  if (rbn) cs_coefs_fwd(rb, C, c0, chunk == 0, red, sa, sb, rsc, rsh);
  float a[VEC], bb[VEC], ra[VEC], rbv[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    a[e] = sc[vi * VEC + e];
    bb[e] = sh[vi * VEC + e];
    ra[e] = rbn ? rsc[vi * VEC + e] : 1.f;
    rbv[e] = rbn ? rsh[vi * VEC + e] : 0.f;
  }
  for (int64_t rb0 = r0 + rr; rb0 < r1; rb0 += (int64_t)EU * RPI) {
    if (rb0 != r0 + rr) {
#pragma unroll
      for (int q = 0; q < EU; ++q) {
        const int64_t r = rb0 + (int64_t)q * RPI;
        if (r < r1) {
          xv[q] = ld16(x + r * C + cv);
          if (res) rv[q] = ld16(res + r * C + cv);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < EU; ++q) {
      const int64_t r = rb0 + (int64_t)q * RPI;
      if (r >= r1) break;
      float v[VEC];
      unpack16(xv[q], v, x);
#pragma unroll
      for (int e = 0; e < VEC; ++e) v[e] = fmaf(v[e], a[e], bb[e]);
      if (res) {
        float rf[VEC];
        unpack16(rv[q], rf, x);
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[e] += fmaf(rf[e], ra[e], rbv[e]);
      }
      if (relu) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[e] = fmaxf(v[e], 0.f);
      }
      store_vec(y + r * C + cv, v);
    }
  }
}

// dx = A dy' + B h + Cc over the slice's channels, dy' = dy * (mask > 0)
template <typename T>
__global__ void __launch_bounds__(NTS) bn_bwd_apply_cs_k(const T *__restrict__ dy, const T *__restrict__ h,
                                                         const T *__restrict__ mask_t, int64_t V, int C, BnBwdPart b,
                                                         T *__restrict__ dx, int nslice, int64_t rows_per_chunk,
                                                         T *__restrict__ dp) {
  __shared__ double red[2][NTS];
  __shared__ double sa[CS], sb[CS];
  __shared__ float cA[CS], cB[CS], cC[CS];
  constexpr int VEC = Vec<T>::N, VPR = CS / VEC, RPI = NTS / VPR;
  const int slice = blockIdx.x % nslice, chunk = blockIdx.x / nslice;
  const int c0 = slice * CS;
  const int64_t r0 = (int64_t)chunk * rows_per_chunk, r1 = min(V, r0 + rows_per_chunk);
  const int vi = threadIdx.x % VPR, rr = threadIdx.x / VPR;
  const int cv = c0 + vi * VEC;
  pdl_begin();
  uint4 dv[EU], xv[EU], mv[EU];
#pragma unroll
  for (int q = 0; q < EU; ++q) {
    const int64_t r = r0 + rr + (int64_t)q * RPI;
    if (r < r1) {
      dv[q] = ld16(dy + r * C + cv);
      xv[q] = ld16(h + r * C + cv);
      mv[q] = ld16(mask_t + r * C + cv);
    }
  }
  if (b.P >= 0) {
    cs_sums(b.part, b.P, C, c0, red, sa, sb);
    if (threadIdx.x < CS) {
      const int c = c0 + threadIdx.x;
      const double S1 = sa[threadIdx.x], is = b.invstd[c], mu = b.mean[c];
      const double S2 = is * sb[threadIdx.x];  // sum dy' * xhat
      const double m1 = S1 / (double)b.V, m2 = S2 / (double)b.V;
      const double A = (double)b.gamma[c] * is;
      cA[threadIdx.x] = (float)A;
      cB[threadIdx.x] = (float)(-A * is * m2);
      cC[threadIdx.x] = (float)(-A * m1 + A * is * mu * m2);
      if (chunk == 0) {
        b.dgamma[c] += (float)S2;
        b.dbeta[c] += (float)S1;
      }
    }
  } else if (threadIdx.x < CS) {
    cA[threadIdx.x] = b.coef[c0 + threadIdx.x];
    cB[threadIdx.x] = b.coef[C + c0 + threadIdx.x];
    cC[threadIdx.x] = b.coef[2 * C + c0 + threadIdx.x];
  }
  __syncthreads();
  float A[VEC], B[VEC], Cc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    A[e] = cA[vi * VEC + e];
    B[e] = cB[vi * VEC + e];
    Cc[e] = cC[vi * VEC + e];
  }
  for (int64_t rb0 = r0 + rr; rb0 < r1; rb0 += (int64_t)EU * RPI) {
    if (rb0 != r0 + rr) {
#pragma unroll
      for (int q = 0; q < EU; ++q) {
        const int64_t r = rb0 + (int64_t)q * RPI;
        if (r < r1) {
          dv[q] = ld16(dy + r * C + cv);
          xv[q] = ld16(h + r * C + cv);
          mv[q] = ld16(mask_t + r * C + cv);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < EU; ++q) {
      const int64_t r = rb0 + (int64_t)q * RPI;
      if (r >= r1) break;
      float d[VEC], xf[VEC], m[VEC], o[VEC];
      unpack16(dv[q], d, dy);
      unpack16(xv[q], xf, h);
      unpack16(mv[q], m, h);
      float dd[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        dd[e] = m[e] > 0.f ? d[e] : 0.f;
        o[e] = fmaf(A[e], dd[e], fmaf(B[e], xf[e], Cc[e]));
      }
      store_vec(dx + r * C + cv, o);
      if (dp) store_vec(dp + r * C + cv, dd);  // dy' (exact: dy or 0) for a later accumulate
    }
  }
}

// ---------------------------------------------------------------------------
// Stem Conv block tail (reading X4: BN + ReLU + max-pool k3 s2 p1), bf16.
// Forward: the stem conv wrote its BN statistics partials; every block
// finalizes them, and the pool compares RAW h values: max and first argmax of
// ReLU(s*h + b) over a window are those of s*h (s = gamma*invstd) — h itself
// for s > 0, -h for s < 0 (sign flip of the bf16 bit pattern) — except when the
// window maximum is not positive (ReLU makes every tap 0: the first valid tap
// wins) or s == 0.  Packed bf16x2 compares: 4 instructions per 2 channels and
// tap.  The backward runs at the pooled resolution (k_stem_bwd.cu).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t sel32(uint32_t m, uint32_t a, uint32_t b) { return (a & m) | (b & ~m); }

template <int DUMMY>
__global__ void __launch_bounds__(NTA) stem_pool_fwd_k(const bf16 *__restrict__ h, int N, int D, int H, int W, int C,
                                                       BnPart b, bf16 *__restrict__ y, uint8_t *__restrict__ am,
                                                       int Do, int Ho, int Wo) {
  extern __shared__ double dsm[];
  pdl_begin();
  double *sums = dsm, *scr = dsm + 2 * C;
  float *fs = (float *)(scr + 2 * NTA);
  float *sc = fs, *sh = fs + C;
  bn_part_coefs(b, C, sc, sh, sums, scr);
  const int G = C / 8;
  const int ipr = Wo * G;  // items per output row
  const int total = N * Do * Ho * ipr;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int row = idx / ipr, it = idx - row * ipr;
    const int ow = it / G, c0 = (it - ow * G) * 8;
    const int oh = row % Ho, od = (row / Ho) % Do, nn = row / (Ho * Do);
    float s_[8], b_[8];
    uint32_t fm[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s_[j] = sc[c0 + j];
      b_[j] = sh[c0 + j];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) fm[q] = (s_[2 * q] < 0.f ? 0x8000u : 0u) | (s_[2 * q + 1] < 0.f ? 0x80000000u : 0u);
    uint32_t best[4] = {0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u}, arg[4] = {0u, 0u, 0u, 0u};
    // the 9 taps of plane kd + 1 are requested before plane kd is compared: about
    // one memory round trip per output instead of three
    uint4 vb[2][9];
    bool okb[2][9];
    auto load_plane = [&](int kd, uint4 (&v)[9], bool (&ok)[9]) {
      const int id = 2 * od + kd - 1;
#pragma unroll
      for (int tp = 0; tp < 9; ++tp) {
        const int ih = 2 * oh + tp / 3 - 1, iw = 2 * ow + tp % 3 - 1;
        ok[tp] = id >= 0 && id < D && ih >= 0 && ih < H && iw >= 0 && iw < W;
        v[tp] = ok[tp] ? ld16(h + ((int64_t)((nn * D + id) * H + ih) * W + iw) * C + c0) : make_uint4(0, 0, 0, 0);
      }
    };
    load_plane(0, vb[0], okb[0]);
#pragma unroll
    for (int kd = 0; kd < 3; ++kd) {
      if (kd < 2) load_plane(kd + 1, vb[(kd + 1) & 1], okb[(kd + 1) & 1]);
      const uint4 (&v)[9] = vb[kd & 1];
      const bool (&ok)[9] = okb[kd & 1];
#pragma unroll
      for (int tp = 0; tp < 9; ++tp) {
        if (!ok[tp]) continue;
        const uint32_t code = (uint32_t)(kd * 9 + tp) * 0x00010001u;
        const uint32_t w4[4] = {v[tp].x, v[tp].y, v[tp].z, v[tp].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t u = w4[q] ^ fm[q];
          __nv_bfloat162 ub, bb;
          memcpy(&ub, &u, 4);
          memcpy(&bb, &best[q], 4);
          const uint32_t m = __hgt2_mask(ub, bb);
          best[q] = sel32(m, u, best[q]);
          arg[q] = sel32(m, code, arg[q]);
        }
      }
    }
    // first valid tap of the window (the winner when every ReLU value is 0)
    const int t0 = (od == 0 ? 9 : 0) + (oh == 0 ? 3 : 0) + (ow == 0 ? 1 : 0);
    float out[8];
    uint8_t codes[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t raw = best[q] ^ fm[q];
      __nv_bfloat162 hb;
      memcpy(&hb, &raw, 4);
      const float2 hv = __bfloat1622float2(hb);
      const float hv2[2] = {hv.x, hv.y};
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 2 * q + e;
        const float yv = fmaf(hv2[e], s_[j], b_[j]);
        const bool zero = !(yv > 0.f) || s_[j] == 0.f;
        out[j] = yv > 0.f ? yv : 0.f;
        codes[j] = zero ? (uint8_t)t0 : (uint8_t)((arg[q] >> (16 * e)) & 0xFF);
      }
    }
    const int64_t vo = (int64_t)row * Wo + ow;
    store_vec(y + vo * C + c0, out);
    uint2 pk;
    memcpy(&pk, codes, 8);
    *reinterpret_cast<uint2 *>(am + vo * C + c0) = pk;
  }
}

inline int bn_grid_mult() {
  static const int m = getenv("RN_BN_GRID_MULT") ? std::max(1, atoi(getenv("RN_BN_GRID_MULT"))) : 1;
  return m;
}

inline unsigned grid_part(int64_t vecs, int G) {
  int64_t b = (vecs + (int64_t)NTA * EU - 1) / ((int64_t)NTA * EU);
  if (b > 148 * bn_grid_mult()) b = 148 * bn_grid_mult();
  if (b < 1) b = 1;
  return (unsigned)stride_multiple(b, NTA, G);
}

// max-pool k3 s2 p1, -inf padding; first maximum in (kd,kh,kw) order (reading X10).
// One thread per (output voxel, 16-byte channel vector); the 9 taps of each kd
// plane are loaded as one predicated batch before comparing (memory-level
// parallelism); argmax codes of the vector go out as one 8-/4-byte store.
template <int VEC>
struct ArgVec;
template <>
struct ArgVec<8> {
  typedef uint2 type;
};
template <>
struct ArgVec<4> {
  typedef uint32_t type;
};

template <typename T>
__global__ void __launch_bounds__(NT) maxpool_fwd_k(const T *__restrict__ x, int N, int D, int H, int W, int C,
                                                    const float *__restrict__ scale, const float *__restrict__ shift,
                                                    int relu, T *__restrict__ y, uint8_t *__restrict__ am, int Do,
                                                    int Ho, int Wo) {
  pdl_begin();
  constexpr int VEC = Vec<T>::N;
  typedef typename ArgVec<VEC>::type AT;
  // flattened over (n, od, oh, ow, channel group): every thread busy (one block per
  // output row left most of a block idle on the 12-14 voxel rows of the mask
  // branch); 32-bit index math, any G = C/VEC (C = 24 has G = 3)
  const unsigned G = (unsigned)(C / VEC);
  const unsigned total = (unsigned)(N * Do * Ho * Wo) * G;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const unsigned vox = t / G;
    const int c0 = (int)(t - vox * G) * VEC;
    const int ow = (int)(vox % (unsigned)Wo);
    const unsigned row = vox / (unsigned)Wo;
    const int oh = (int)(row % (unsigned)Ho), od = (int)((row / (unsigned)Ho) % (unsigned)Do);
    const int nn = (int)(row / ((unsigned)Ho * Do));
    const int64_t vo = (int64_t)vox;
    float sc[VEC], sh[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      sc[j] = scale ? scale[c0 + j] : 1.f;
      sh[j] = scale ? shift[c0 + j] : 0.f;
    }
    float best[VEC];
    uint8_t arg[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      best[j] = -INFINITY;
      arg[j] = 0;
    }
#pragma unroll
    for (int kd = 0; kd < 3; ++kd) {
      const int id = 2 * od + kd - 1;
      uint4 v[9];
      bool ok[9];
#pragma unroll
      for (int tp = 0; tp < 9; ++tp) {
        const int ih = 2 * oh + tp / 3 - 1, iw = 2 * ow + tp % 3 - 1;
        ok[tp] = id >= 0 && id < D && ih >= 0 && ih < H && iw >= 0 && iw < W;
        if (ok[tp]) v[tp] = ld16(x + ((int64_t)((nn * D + id) * H + ih) * W + iw) * C + c0);
      }
#pragma unroll
      for (int tp = 0; tp < 9; ++tp) {
        if (!ok[tp]) continue;
        float f[VEC];
        unpack16(v[tp], f, x);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          float e = fmaf(f[j], sc[j], sh[j]);
          if (relu) e = fmaxf(e, 0.f);
          if (e > best[j]) {
            best[j] = e;
            arg[j] = (uint8_t)(kd * 9 + tp);
          }
        }
      }
    }
    store_vec(y + vo * C + c0, best);
    AT packed;
    memcpy(&packed, arg, sizeof(AT));
    *reinterpret_cast<AT *>(am + vo * C + c0) = packed;
  }
}

// gather-form adjoint: each input voxel sums dy of the (<= 8) windows whose
// argmax is it.  Per dimension the covering windows are o = floor(i/2) and
// o = floor((i+1)/2) (one window when i is even); all candidates are loaded as
// one predicated batch.
template <typename T>
__global__ void __launch_bounds__(NT) maxpool_bwd_k(const T *__restrict__ dy, const uint8_t *__restrict__ am, int N,
                                                    int D, int H, int W, int C, int Do, int Ho, int Wo,
                                                    T *__restrict__ dx, int accumulate) {
  pdl_begin();
  constexpr int VEC = Vec<T>::N;
  typedef typename ArgVec<VEC>::type AT;
  // one block per input row (n, id, ih); 32-bit index math, any G = C/VEC
  const int G = C / VEC;
  const int ih = (int)(blockIdx.x % (unsigned)H), id = (int)((blockIdx.x / (unsigned)H) % (unsigned)D);
  const int nn = (int)(blockIdx.x / ((unsigned)H * D));
  const int items = W * G;
  for (int t = threadIdx.x; t < items; t += blockDim.x) {
    const int iw = t / G, c0 = (t - iw * G) * VEC;
    const int64_t vi = (int64_t)blockIdx.x * W + iw;
    uint4 g[8];
    AT a[8];
    bool ok[8];
    int tap[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int od = (id + (q >> 2 & 1)) >> 1, oh = (ih + (q >> 1 & 1)) >> 1, ow = (iw + (q & 1)) >> 1;
      // the second candidate of a dimension exists only for odd i (else it repeats the first)
      ok[q] = od < Do && oh < Ho && ow < Wo && (!(q & 4) || (id & 1)) && (!(q & 2) || (ih & 1)) &&
              (!(q & 1) || (iw & 1));
      tap[q] = ((id - 2 * od + 1) * 3 + (ih - 2 * oh + 1)) * 3 + (iw - 2 * ow + 1);
      if (ok[q]) {
        const int64_t o = ((int64_t)((nn * Do + od) * Ho + oh) * Wo + ow) * C + c0;
        g[q] = ld16(dy + o);
        a[q] = *reinterpret_cast<const AT *>(am + o);
      }
    }
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (!ok[q]) continue;
      float f[VEC];
      unpack16(g[q], f, dy);
      uint8_t code[VEC];
      memcpy(code, &a[q], sizeof(AT));
#pragma unroll
      for (int j = 0; j < VEC; ++j)
        if (code[j] == tap[q]) acc[j] += f[j];
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

// bf16 gather-form adjoint with the pooled rows staged in smem: a block owns the
// input rows ih = 2j, 2j+1 of one (n, id) plane; both need only pooled rows
// oh = j, j+1 of od = id/2 (and (id+1)/2 for odd id), so <= 4 pooled rows of dy
// and argmax codes are loaded once (coalesced 16-B vectors) and every candidate
// window is then read from smem.  Same candidate order / arithmetic as maxpool_bwd_k.
__global__ void __launch_bounds__(256) maxpool_bwd_stage_k(const bf16 *__restrict__ dy,
                                                           const uint8_t *__restrict__ am, int N, int D, int H,
                                                           int W, int C, int Do, int Ho, int Wo,
                                                           bf16 *__restrict__ dx, int accumulate) {
  extern __shared__ __align__(16) uint8_t smp[];
  pdl_begin();
  const int rowel = Wo * C;                  // elements of one pooled row
  bf16 *sdy = reinterpret_cast<bf16 *>(smp);  // [4][Wo][C]
  uint8_t *sam = smp + 4 * rowel * 2;         // [4][Wo][C]
  const int Hj = (H + 1) / 2;
  const int j = blockIdx.x % Hj, id = (blockIdx.x / Hj) % D, nn = blockIdx.x / (Hj * D);
  const int od0 = id >> 1, od1 = (id & 1) && ((id + 1) >> 1) < Do ? (id + 1) >> 1 : -1;
  // stage pooled rows slot = sd*2 + sh (od0/od1 x oh j/j+1)
  const int vecs = rowel / 8;
  for (int i = threadIdx.x; i < 4 * vecs; i += blockDim.x) {
    const int slot = i / vecs, e = (i - slot * vecs) * 8;
    const int od = (slot >> 1) ? od1 : od0, oh = j + (slot & 1);
    uint4 v = make_uint4(0, 0, 0, 0);
    uint2 a = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);  // no code matches 255
    if (od >= 0 && oh < Ho) {
      const int64_t o = ((int64_t)(nn * Do + od) * Ho + oh) * rowel + e;
      v = ld16(dy + o);
      a = *reinterpret_cast<const uint2 *>(am + o);
    }
    *reinterpret_cast<uint4 *>(sdy + slot * rowel + e) = v;
    *reinterpret_cast<uint2 *>(sam + slot * rowel + e) = a;
  }
  __syncthreads();
  const int G = C / 8;
  const int items = 2 * W * G;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int r = it / (W * G), rem = it - r * W * G, iw = rem / G, c0 = (rem - iw * G) * 8;
    const int ih = 2 * j + r;
    if (ih >= H) continue;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int od = (q & 4) ? od1 : od0;
      const int oh = (ih + (q >> 1 & 1)) >> 1, ow = (iw + (q & 1)) >> 1;
      const bool ok = od >= 0 && oh < Ho && ow < Wo && (!(q & 4) || (id & 1)) && (!(q & 2) || (ih & 1)) &&
                      (!(q & 1) || (iw & 1));
      if (!ok) continue;
      const int slot = ((q & 4) ? 2 : 0) + (oh - j);
      const int tap = ((id - 2 * od + 1) * 3 + (ih - 2 * oh + 1)) * 3 + (iw - 2 * ow + 1);
      const int e0 = slot * rowel + ow * C + c0;
      float f[8];
      load_vec(sdy + e0, f);
      uint8_t code[8];
      const uint2 a = *reinterpret_cast<const uint2 *>(sam + e0);
      memcpy(code, &a, 8);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (code[e] == tap) acc[e] += f[e];
    }
    const int64_t o = (((int64_t)(nn * D + id) * H + ih) * W + iw) * C + c0;
    if (accumulate) {
      float pv[8];
      load_vec(dx + o, pv);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += pv[e];
    }
    store_vec(dx + o, acc);
  }
}

template <typename T>
__global__ void upsample_fwd_k(const T *__restrict__ x, int N, int Di, int Hi, int Wi, int C, T *__restrict__ y,
                               int Do, int Ho, int Wo, UpTables t) {
  pdl_begin();
  constexpr int VEC = Vec<T>::N;
  // 32-bit index math (the 64-bit div/mod chain made this kernel instruction-bound);
  // G = C/VEC a power of two; the 6 table entries and the 8 taps are loaded before
  // the FMAs (same accumulation order as before: a, b, c nested); any G = C/VEC
  const unsigned G = (unsigned)(C / VEC);
  const unsigned total = (unsigned)(N * Do * Ho * Wo) * G;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned vo = i / G;
    const int c0 = (int)(i - vo * G) * VEC;
    const int ow = (int)(vo % (unsigned)Wo);
    unsigned r = vo / (unsigned)Wo;
    const int oh = (int)(r % (unsigned)Ho); r /= (unsigned)Ho;
    const int od = (int)(r % (unsigned)Do);
    const int nn = (int)(r / (unsigned)Do);
    const int2 di = *reinterpret_cast<const int2 *>(t.fw_idx[0] + 2 * od);
    const int2 hi = *reinterpret_cast<const int2 *>(t.fw_idx[1] + 2 * oh);
    const int2 wi = *reinterpret_cast<const int2 *>(t.fw_idx[2] + 2 * ow);
    const float2 dw = *reinterpret_cast<const float2 *>(t.fw_w[0] + 2 * od);
    const float2 hw = *reinterpret_cast<const float2 *>(t.fw_w[1] + 2 * oh);
    const float2 ww = *reinterpret_cast<const float2 *>(t.fw_w[2] + 2 * ow);
    const int ids[2] = {di.x, di.y}, ihs[2] = {hi.x, hi.y}, iws[2] = {wi.x, wi.y};
    const float wds[2] = {dw.x, dw.y}, whs[2] = {hw.x, hw.y}, wws[2] = {ww.x, ww.y};
    float v[8][VEC];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const unsigned src = (((unsigned)nn * Di + ids[q >> 2]) * Hi + ihs[(q >> 1) & 1]) * Wi + iws[q & 1];
      load_vec(x + (int64_t)src * C + c0, v[q]);
    }
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float wc = (wds[q >> 2] * whs[(q >> 1) & 1]) * wws[q & 1];
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] = fmaf(wc, v[q][j], acc[j]);
    }
    store_vec(y + (int64_t)vo * C + c0, acc);
  }
}

template <typename T>
__global__ void upsample_bwd_k(const T *__restrict__ dy, int N, int Di, int Hi, int Wi, int C, T *__restrict__ dx,
                               int Do, int Ho, int Wo, UpTables t) {
  pdl_begin();
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
  pdl_begin();
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
  pdl_begin();
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
  pdl_begin();
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
  pdl_begin();
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
  pdl_begin();
  const int64_t n = (int64_t)N * V * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int nn = (int)(i / ((int64_t)V * C));
    const float dg = dz[nn * 2] * W[c] + dz[nn * 2 + 1] * W[C + c];
    dx[i] = from_f<T>(dg / (float)V);
  }
}

__global__ void sgd_k(float *__restrict__ w, const float *__restrict__ g, int64_t n, float lr) {
  pdl_begin();
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
  pdl_begin();
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
  pdl_begin();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!isfinite(v[i])) *flag = 1;
}

}  // namespace

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

int chan_fin_blocks(int64_t V, int C) {
  // one block per ~32K elements, at most one per SM: whoever finalizes reads
  // every partial (a small tensor needs few)
  int64_t b = (V * C + 32767) / 32768;
  if (b > 148) b = 148;
  if (b < 1) b = 1;
  return (int)b;
}

// partials-only passes (their consumer, a BN apply, reduces the partials of the
// channels it needs: the channel-sliced applies 16 at a time): one block per ~8K
// elements, at most one per SM — small stage-3/4 tensors get 4x the blocks of the
// last-block-finalize passes above (a 16-block pass was a 10 us latency chain)
int chan_part_blocks(int64_t V, int C) {
  int64_t b = (V * C + 8191) / 8192;
  if (b > 148) b = 148;
  if (b < 1) b = 1;
  return (int)b;
}

void bn_stats_finalize(DType dt, const void *x, int64_t V, int C, float *partial, unsigned *counter,
                       const float *gamma, const float *beta, float *mean, float *invstd, float *scale, float *shift,
                       float *run_mean, float *run_var, float momentum, float eps, cudaStream_t st) {
  const int nblk = chan_fin_blocks(V, C);
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    chan_reduce_dims<T>(V, C, nblk, rpb, smem);
    StatsOp<T> op{(const T *)x, C, {}, true};
    StatsFin<T> fin{(const T *)x, V, gamma, beta, mean, invstd, scale, shift, run_mean, run_var, momentum, eps};
    launch_k(chan_reduce_fin_k<T, StatsOp<T>, StatsFin<T>>, nblk, NTR, smem, st, op, fin, V, C, partial, rpb, counter);
  });
  LAUNCH_CHECK();
}

void bn_bwd_reduce_finalize(DType dt, const void *dy, const void *x, int64_t V, int C, int mask_mode,
                            const void *mask_t, const float *scale, const float *shift, const float *mean,
                            const float *invstd, const float *gamma, float *partial, unsigned *counter, float *dgamma,
                            float *dbeta, float *coef, cudaStream_t st) {
  const int nblk = chan_fin_blocks(V, C);
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    chan_reduce_dims<T>(V, C, nblk, rpb, smem);
    BwdOp<T> op{(const T *)dy, (const T *)x, (const T *)mask_t, mask_mode, C, scale, shift, mean, invstd};
    BwdFin fin{V, C, gamma, mean, invstd, dgamma, dbeta, coef};
    launch_k(chan_reduce_fin_k<T, BwdOp<T>, BwdFin>, nblk, NTR, smem, st, op, fin, V, C, partial, rpb, counter);
  });
  LAUNCH_CHECK();
}

void att_bwd_finalize(DType dt, const void *dout, const void *m, const void *T_, int64_t V, int C, void *dT, void *dm,
                      float *partial, unsigned *counter, float *dbias, cudaStream_t st) {
  const int nblk = chan_fin_blocks(V, C);
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    chan_reduce_dims<T>(V, C, nblk, rpb, smem);
    AttBwdOp<T> op{(const T *)dout, (const T *)m, (const T *)T_, (T *)dT, (T *)dm, C};
    SumFin fin{dbias};
    launch_k(chan_reduce_fin_k<T, AttBwdOp<T>, SumFin>, nblk, NTR, smem, st, op, fin, V, C, partial, rpb, counter);
  });
  LAUNCH_CHECK();
}

void bn_apply(DType dt, const void *x, int64_t V, int C, const float *scale, const float *shift, const void *res,
              const float *rscale, const float *rshift, bool relu, void *y, cudaStream_t st) {
  DISPATCH(dt, launch_k(bn_apply_k<T>, grid_elem(V * C / Vec<T>::N, C / Vec<T>::N), NT, 0, st, 
                   (const T *)x, V, C, scale, shift, (const T *)res, rscale, rshift, relu ? 1 : 0, (T *)y));
  LAUNCH_CHECK();
}

void bn_bwd_apply(DType dt, const void *dy, const void *x, int64_t V, int C, int mask_mode, const void *mask_t,
                  const float *scale, const float *shift, const float *coef, void *dx, cudaStream_t st) {
  DISPATCH(dt, launch_k(bn_bwd_apply_k<T>, grid_elem(V * C / Vec<T>::N, C / Vec<T>::N), NT, 0, st, 
                   (const T *)dy, (const T *)x, V, C, mask_mode, (const T *)mask_t, scale, shift, coef, (T *)dx));
  LAUNCH_CHECK();
}

int bn_stats_partials(DType dt, const void *x, int64_t V, int C, float *part, cudaStream_t st) {
  const int nblk = chan_part_blocks(V, C);
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    chan_reduce_dims<T>(V, C, nblk, rpb, smem);
    StatsOp<T> op{(const T *)x, C, {}, false};
    launch_k(chan_partials_k<T, StatsOp<T>>, nblk, NTR, smem, st, op, V, C, part, rpb);
  });
  LAUNCH_CHECK();
  return nblk;
}

int bn_bwd_partials(DType dt, const void *dy, const void *h, const void *mask_t, const float *mean, int64_t V, int C,
                    float *part, cudaStream_t st) {
  const int nblk = chan_part_blocks(V, C);
  DISPATCH(dt, {
    int64_t rpb;
    size_t smem;
    chan_reduce_dims<T>(V, C, nblk, rpb, smem);
    BwdHOp<T> op{(const T *)dy, (const T *)h, (const T *)mask_t, C, mean, {}};
    launch_k(chan_partials_k<T, BwdHOp<T>>, nblk, NTR, smem, st, op, V, C, part, rpb);
  });
  LAUNCH_CHECK();
  return nblk;
}

// channel-sliced for the small tensors of stages 2-4, where the partials reduce
// dominated; the full-row kernels stay faster for stage 1 (7.6 M elements:
// 11-15 us sliced vs 10-12 us per launch measured)
static bool bn_apply_cs(int64_t V, int C) {
  static const bool v = !getenv("RN_BN_APPLY_CS") || atoi(getenv("RN_BN_APPLY_CS")) != 0;
  return v && C % CS == 0 && V * C <= ((int64_t)4 << 20);
}
// slices x chunks of whole rows
static void cs_grid(int64_t V, int C, int &nslice, int &nchunk, int64_t &rpc) {
  // about one 256-thread block per SM (A/B, RN_CS_BLOCKS: 148 -> 3.0930 ms, 296 -> 3.0984,
  // 592 -> 3.1334, 100 -> 3.0995, 74 -> 3.1252), chunks of >= 64 rows
  static const int target = getenv("RN_CS_BLOCKS") ? std::max(1, atoi(getenv("RN_CS_BLOCKS"))) : 148;
  nslice = C / CS;
  nchunk = (int)std::max<int64_t>(1, std::min<int64_t>((target + nslice - 1) / nslice, (V + 63) / 64));
  rpc = (V + nchunk - 1) / nchunk;
  nchunk = (int)((V + rpc - 1) / rpc);
}

void bn_apply_fused(DType dt, const void *x, int64_t V, int C, const BnFinal &f, const BnFinal *rf, const void *res,
                    bool relu, void *y, cudaStream_t st) {
  auto mk = [&](const BnFinal &q) {
    return BnPart{q.part, q.P, V, q.gamma, q.beta, q.mean, q.invstd, q.scale, q.shift, q.run_mean, q.run_var,
                  q.momentum, q.eps};
  };
  BnPart b = mk(f);
  BnPart r{};
  if (rf) r = mk(*rf);
  if (bn_fin_separate()) {
    launch_k(bn_fin_fwd_k, (unsigned)((C + 31) / 32), 256, 0, st, b, C);
    LAUNCH_CHECK();
    b.P = -1;
    if (rf) {
      launch_k(bn_fin_fwd_k, (unsigned)((C + 31) / 32), 256, 0, st, r, C);
      LAUNCH_CHECK();
      r.P = -1;
    }
  }
  if (bn_apply_cs(V, C)) {
    int nslice, nchunk;
    int64_t rpc;
    cs_grid(V, C, nslice, nchunk, rpc);
    DISPATCH(dt, launch_k(bn_apply_cs_k<T>, (unsigned)(nslice * nchunk), NTS, 0, st, (const T *)x, V, C, b, r,
                          (const T *)res, relu ? 1 : 0, (T *)y, nslice, rpc));
    LAUNCH_CHECK();
    return;
  }
  const size_t smem = (2 * (size_t)C + 2 * NTA) * sizeof(double) + 4 * (size_t)C * sizeof(float);
  DISPATCH(dt, launch_k(bn_apply_part_k<T>, grid_part(V * C / Vec<T>::N, C / Vec<T>::N), NTA, smem, st, (const T *)x, V, C, b, r,
                        (const T *)res, relu ? 1 : 0, (T *)y));
  LAUNCH_CHECK();
}

void bn_bwd_apply_fused(DType dt, const void *dy, const void *h, const void *mask_t, int64_t V, int C,
                        const float *part, int P, const float *gamma, const float *mean, const float *invstd,
                        float *dgamma, float *dbeta, void *dx, cudaStream_t st, float *coef, void *dprime) {
  BnBwdPart b{part, P, V, gamma, mean, invstd, dgamma, dbeta, coef};
  if (bn_fin_separate() && coef) {
    launch_k(bn_fin_bwd_k, (unsigned)((C + 31) / 32), 256, 0, st, b, C);
    LAUNCH_CHECK();
    b.P = -1;
  }
  if (bn_apply_cs(V, C)) {
    int nslice, nchunk;
    int64_t rpc;
    cs_grid(V, C, nslice, nchunk, rpc);
    DISPATCH(dt, launch_k(bn_bwd_apply_cs_k<T>, (unsigned)(nslice * nchunk), NTS, 0, st, (const T *)dy,
                          (const T *)h, (const T *)mask_t, V, C, b, (T *)dx, nslice, rpc, (T *)dprime));
    LAUNCH_CHECK();
    return;
  }
  const size_t smem = (2 * (size_t)C + 2 * NTA) * sizeof(double) + 3 * (size_t)C * sizeof(float);
  DISPATCH(dt, launch_k(bn_bwd_apply_part_k<T>, grid_part(V * C / Vec<T>::N, C / Vec<T>::N), NTA, smem, st, (const T *)dy,
                        (const T *)h, (const T *)mask_t, V, C, b, (T *)dx, (T *)dprime));
  LAUNCH_CHECK();
}

void stem_pool_fwd(const void *h, int N, int D, int H, int W, int C, const BnFinal &f, int64_t V, void *y,
                   uint8_t *am, int Do, int Ho, int Wo, cudaStream_t st) {
  BnPart b{f.part, f.P, V, f.gamma, f.beta, f.mean, f.invstd, f.scale, f.shift, f.run_mean, f.run_var,
           f.momentum, f.eps};
  if (bn_fin_separate()) {
    launch_k(bn_fin_fwd_k, (unsigned)((C + 31) / 32), 256, 0, st, b, C);
    LAUNCH_CHECK();
    b.P = -1;
  }
  const size_t smem = (2 * (size_t)C + 2 * NTA) * sizeof(double) + 2 * (size_t)C * sizeof(float);
  launch_k(stem_pool_fwd_k<0>, 148, NTA, smem, st, (const bf16 *)h, N, D, H, W, C, b, (bf16 *)y, am, Do, Ho, Wo);
  LAUNCH_CHECK();
}

void maxpool_fwd(DType dt, const void *x, int N, int D, int H, int W, int C, const float *scale, const float *shift,
                 bool relu, void *y, uint8_t *argmax, int Do, int Ho, int Wo, cudaStream_t st) {
  DISPATCH(dt, launch_k(maxpool_fwd_k<T>, grid_for((int64_t)N * Do * Ho * Wo * C / Vec<T>::N, NT, 148 * 8), NT, 0, st,
                   (const T *)x, N, D, H, W, C, scale, shift, relu ? 1 : 0, (T *)y, argmax, Do, Ho, Wo));
  LAUNCH_CHECK();
}

void maxpool_bwd(DType dt, const void *dy, const uint8_t *argmax, int N, int D, int H, int W, int C, int Do, int Ho,
                 int Wo, void *dx, bool accumulate, cudaStream_t st) {
  const size_t smem = (size_t)4 * Wo * C * 3;
  if (dt == DT_BF16 && C % 8 == 0 && smem <= 48 * 1024) {
    launch_k(maxpool_bwd_stage_k, (unsigned)(N * D * ((H + 1) / 2)), 256, smem, st, (const bf16 *)dy, argmax, N, D, H,
             W, C, Do, Ho, Wo, (bf16 *)dx, accumulate ? 1 : 0);
    LAUNCH_CHECK();
    return;
  }
  DISPATCH(dt, launch_k(maxpool_bwd_k<T>, (unsigned)(N * D * H), NT, 0, st, 
                   (const T *)dy, argmax, N, D, H, W, C, Do, Ho, Wo, (T *)dx, accumulate ? 1 : 0));
  LAUNCH_CHECK();
}


// Grad-CAM at the last conv layer (oracle gradcam_last):
// alpha_k = W[c, k] / V (the GAP + FC head's gradient, averaged over voxels),
// coarse[v] = ReLU(sum_k alpha_k A[v][k]) — one warp per voxel, fixed-order
// lane sums + butterfly; then a 1-channel fp32 trilinear upsample to the input grid.
template <typename T>
__global__ void cam_k(const T *__restrict__ A, const float *__restrict__ wrow, float invV, int C, int64_t nvox,
                      float *__restrict__ coarse) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nvox; v += nw) {
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s = fmaf(to_f(A[v * C + c]), wrow[c] * invV, s);
    s = warp_sum(s);
    if (lane == 0) coarse[v] = s > 0.f ? s : 0.f;
  }
}
__global__ void up1_k(const float *__restrict__ in, int N, int d, int h, int w, float *__restrict__ out, int D,
                      int H, int W, UpTables t) {
  pdl_begin();
  const int n = N * D * H * W;  // < 2^31 (checked by the launcher): 32-bit index math
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int r = i;
    const int ow = r % W; r /= W;
    const int oh = r % H; r /= H;
    const int od = r % D;
    const int nn = r / D;
    const float *src = in + nn * d * h * w;
    float acc = 0.f;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int id = t.fw_idx[0][2 * od + a];
      const float wd = t.fw_w[0][2 * od + a];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int ih = t.fw_idx[1][2 * oh + b];
        const float wh = wd * t.fw_w[1][2 * oh + b];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int iw = t.fw_idx[2][2 * ow + c];
          acc = fmaf(wh * t.fw_w[2][2 * ow + c], src[(id * h + ih) * w + iw], acc);
        }
      }
    }
    out[i] = acc;
  }
}

void gradcam_last(DType dt, const void *A, const float *wrow, int N, int d, int h, int w, int C, float *coarse,
                  float *map, int D, int H, int W, const UpTables &t, cudaStream_t st) {
  const int64_t nvox = (int64_t)N * d * h * w;
  const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nvox * 32 + 255) / 256, 148 * 8));
  DISPATCH(dt, launch_k(cam_k<T>, gb, 256, 0, st, (const T *)A, wrow, 1.0f / (float)(d * h * w), C, nvox, coarse));
  LAUNCH_CHECK();
  const int64_t nout = (int64_t)N * D * H * W;
  if (nout >= (1LL << 31)) throw Error(RN_ERR_SIZE, "gradcam_last: map too large");
  launch_k(up1_k, (unsigned)std::max<int64_t>(1, std::min<int64_t>((nout + 255) / 256, 148 * 16)), 256, 0, st,
           (const float *)coarse, N, d, h, w, map, D, H, W, t);
  LAUNCH_CHECK();
}

void upsample_fwd(DType dt, const void *x, int N, int Di, int Hi, int Wi, int C, void *y, int Do, int Ho, int Wo,
                  const UpTables &t, cudaStream_t st) {
  DISPATCH(dt, launch_k(upsample_fwd_k<T>, grid_for((int64_t)N * Do * Ho * Wo * C / Vec<T>::N), NT, 0, st, 
                   (const T *)x, N, Di, Hi, Wi, C, (T *)y, Do, Ho, Wo, t));
  LAUNCH_CHECK();
}

// One separable pass of the trilinear adjoint (reading X11: the upsampling is
// U_d (x) U_h (x) U_w, so its adjoint is applied one dimension at a time):
//   out[a][j][b] = sum_{k in CSR row j} w_k * in[a][o_k][b]
// with the dimension's coarse-index CSR (bw_start / bw_o / bw_w).  Four
// consecutive b per thread (coalesced rows); fp32 intermediates, one final
// rounding.  (The fused gather it replaces read ~55 fine voxels per coarse
// voxel through L1/L2: 25-38 us on stage 1.)
__device__ __forceinline__ void ld4f(const float *p, float *v) {
  const float4 a = *reinterpret_cast<const float4 *>(p);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void ld4f(const bf16 *p, float *v) {
  const uint2 u = *reinterpret_cast<const uint2 *>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.y));
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void st4f(float *p, const float *v) {
  *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void st4f(bf16 *p, const float *v) {
  uint2 u;
  *reinterpret_cast<__nv_bfloat162 *>(&u.x) = __floats2bfloat162_rn(v[0], v[1]);
  *reinterpret_cast<__nv_bfloat162 *>(&u.y) = __floats2bfloat162_rn(v[2], v[3]);
  *reinterpret_cast<uint2 *>(p) = u;
}
template <typename Ti, typename To>
__global__ void up_adj_pass_k(const Ti *__restrict__ in, int64_t A, int Lin, int Lout, int64_t B,
                              const int *__restrict__ start, const int *__restrict__ oidx,
                              const float *__restrict__ w, To *__restrict__ out) {
  pdl_begin();
  // 32-bit index math (the launcher checks the sizes fit)
  const unsigned B4 = (unsigned)(B / 4);
  const unsigned n = (unsigned)A * Lout * B4;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned b = (i % B4) * 4;
    const unsigned r = i / B4;
    const int j = (int)(r % (unsigned)Lout);
    const unsigned a = r / (unsigned)Lout;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int k1 = start[j + 1];
    for (int k = start[j]; k < k1; ++k) {
      float v[4];
      ld4f(in + ((int64_t)a * Lin + oidx[k]) * B + b, v);
      const float wk = w[k];
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] = fmaf(wk, v[e], acc[e]);
    }
    st4f(out + ((int64_t)a * Lout + j) * B + b, acc);
  }
}

size_t upsample_bwd_ws_floats(int N, int Di, int Hi, int Wi, int C, int Do, int Ho, int Wo) {
  (void)Di; (void)Wo;
  return (size_t)N * C * ((size_t)Do * Ho * Wi + (size_t)Do * Hi * Wi);
}

// separable adjoint (bf16 path): w, then h, then d; ws >= upsample_bwd_ws_floats
void upsample_bwd_sep(const void *dy, int N, int Di, int Hi, int Wi, int C, void *dx, int Do, int Ho, int Wo,
                      const UpTables &t, float *ws, cudaStream_t st) {
  if (C % 4 != 0) throw Error(RN_ERR_ARG, "upsample_bwd_sep: C % 4");
  if ((int64_t)N * Di * Hi * Wi * C >= (1LL << 31)) throw Error(RN_ERR_ARG, "upsample_bwd_sep: tensor too large");
  float *t1 = ws, *t2 = ws + (size_t)N * Do * Ho * Wi * C;
  auto grid = [](int64_t vec) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((vec + 255) / 256, 148 * 16)); };
  // w: [N*Do*Ho][Wo][C] -> [N*Do*Ho][Wi][C]
  launch_k(up_adj_pass_k<bf16, float>, grid((int64_t)N * Do * Ho * Wi * C / 4), 256, 0, st, (const bf16 *)dy,
           (int64_t)N * Do * Ho, Wo, Wi, (int64_t)C, t.bw_start[2], t.bw_o[2], t.bw_w[2], t1);
  LAUNCH_CHECK();
  // h: [N*Do][Ho][Wi*C] -> [N*Do][Hi][Wi*C]
  launch_k(up_adj_pass_k<float, float>, grid((int64_t)N * Do * Hi * Wi * C / 4), 256, 0, st, (const float *)t1,
           (int64_t)N * Do, Ho, Hi, (int64_t)Wi * C, t.bw_start[1], t.bw_o[1], t.bw_w[1], t2);
  LAUNCH_CHECK();
  // d: [N][Do][Hi*Wi*C] -> [N][Di][Hi*Wi*C]
  launch_k(up_adj_pass_k<float, bf16>, grid((int64_t)N * Di * Hi * Wi * C / 4), 256, 0, st, (const float *)t2,
           (int64_t)N, Do, Di, (int64_t)Hi * Wi * C, t.bw_start[0], t.bw_o[0], t.bw_w[0], (bf16 *)dx);
  LAUNCH_CHECK();
}

void upsample_bwd(DType dt, const void *dy, int N, int Di, int Hi, int Wi, int C, void *dx, int Do, int Ho, int Wo,
                  const UpTables &t, cudaStream_t st) {
  DISPATCH(dt, launch_k(upsample_bwd_k<T>, grid_for((int64_t)N * Di * Hi * Wi * C / Vec<T>::N), NT, 0, st, 
                   (const T *)dy, N, Di, Hi, Wi, C, (T *)dx, Do, Ho, Wo, t));
  LAUNCH_CHECK();
}

void att_fwd(DType dt, const void *m, const void *T_, int64_t V, int C, void *out, cudaStream_t st) {
  DISPATCH(dt, launch_k(att_fwd_k<T>, grid_for(V * C / Vec<T>::N), NT, 0, st, (const T *)m, (const T *)T_, V, C,
                                                                          (T *)out));
  LAUNCH_CHECK();
}

void head_fwd(DType dt, const void *x, int N, int V, int C, const float *W, const float *b, const int32_t *y,
              float dz_scale, float loss_scale, float *g, float *dz, float *loss_acc, cudaStream_t st) {
  dim3 grid(N, (C + 255) / 256);
  DISPATCH(dt, launch_k(gap_k<T>, grid, 256, 0, st, (const T *)x, V, C, g));
  LAUNCH_CHECK();
  launch_k(ce_k, 1, 256, 0, st, g, N, C, W, b, y, dz_scale, loss_scale, dz, loss_acc);
  LAUNCH_CHECK();
}

void head_bwd(DType dt, const float *dz, const float *g, const float *W, int N, int V, int C, float *dW, float *db,
              void *dx, cudaStream_t st) {
  launch_k(head_wgrad_k, (2 * C + 255) / 256, 256, 0, st, dz, g, N, C, dW, db);
  LAUNCH_CHECK();
  DISPATCH(dt, launch_k(head_dx_k<T>, grid_for((int64_t)N * V * C), 256, 0, st, dz, W, N, V, C, (T *)dx));
  LAUNCH_CHECK();
}

void sgd_update(float *w, const float *g, int64_t n, float lr, cudaStream_t st) {
  launch_k(sgd_k, grid_for((n + 3) / 4), NT, 0, st, w, g, n, lr);
  LAUNCH_CHECK();
}

void repack_conv(DType dt, const float *w, int Co, int taps, int Ci, void *wf, void *wd, cudaStream_t st) {
  dim3 grid((Ci + 31) / 32, (Co + 31) / 32, taps);
  DISPATCH(dt, launch_k(repack_k<T>, grid, dim3(32, 8), 0, st, w, Co, taps, Ci, (T *)wf, (T *)wd));
  LAUNCH_CHECK();
}

constexpr int SGD_MAX_TENSORS = 512;

__global__ void __launch_bounds__(256) sgd_repack_all_k(const ConvPack *__restrict__ tab, int n, int64_t tile_begin,
                                                        int64_t total_tiles, float *master,
                                                        const float *__restrict__ grad, float lr) {
  pdl_begin();
  __shared__ float tile[64][65];
  __shared__ int64_t t0s[SGD_MAX_TENSORS];  // tile0 of every tensor, searched in smem (not L2)
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int i = ty * 32 + tx; i < n; i += 256) t0s[i] = tab[i].tile0;
  __syncthreads();
  // persistent: blocks stride over the 64x64 (co, ci) tiles of every tap of every conv tensor;
  // a thread owns two consecutive ci of 8 rows: 128-B rows for the fp32 loads and
  // for both bf16 copies (the transposed one through smem)
  for (int64_t b = tile_begin + blockIdx.x; b < total_tiles; b += gridDim.x) {
    int lo = 0, hi = n - 1;  // tensor of this tile: binary search on tile0 (uniform across the block)
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (t0s[mid] <= b) lo = mid;
      else hi = mid - 1;
    }
    const ConvPack t = tab[lo];
    int64_t r = b - t.tile0;
    const int nci = (t.Ci + 63) / 64, nco = (t.Co + 63) / 64;
    const int cit = (int)(r % nci); r /= nci;
    const int cot = (int)(r % nco); r /= nco;
    const int tap = (int)r;
    const int ci0 = cit * 64, co0 = cot * 64;
    float *w = master + t.off;
    const float *g = grad ? grad + t.off : nullptr;
    bf16 *wf = (bf16 *)t.wf, *wd = (bf16 *)t.wd;
    const int ci = ci0 + 2 * tx;
    const bool pair = ci + 1 < t.Ci && ((t.Ci & 1) == 0);  // float2 path (every r18 conv but the 1-channel stem)
    float v[8][2], gv[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // all loads first
      const int co = co0 + ty + 8 * q;
      const int64_t i0 = ((int64_t)co * t.taps + tap) * t.Ci + ci;
      v[q][0] = v[q][1] = gv[q][0] = gv[q][1] = 0.f;
      if (co < t.Co && pair) {
        const float2 a = *reinterpret_cast<const float2 *>(w + i0);
        v[q][0] = a.x;
        v[q][1] = a.y;
        if (g) {
          const float2 c = *reinterpret_cast<const float2 *>(g + i0);
          gv[q][0] = c.x;
          gv[q][1] = c.y;
        }
      } else if (co < t.Co) {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (ci + e < t.Ci) {
            v[q][e] = w[i0 + e];
            if (g) gv[q][e] = g[i0 + e];
          }
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int co = co0 + ty + 8 * q;
      const int64_t i0 = ((int64_t)co * t.taps + tap) * t.Ci + ci;
      if (g) {
        v[q][0] -= lr * gv[q][0];
        v[q][1] -= lr * gv[q][1];
      }
      if (co < t.Co && pair) {
        if (g) *reinterpret_cast<float2 *>(w + i0) = make_float2(v[q][0], v[q][1]);
        *reinterpret_cast<__nv_bfloat162 *>(wf + i0) = __floats2bfloat162_rn(v[q][0], v[q][1]);
      } else if (co < t.Co) {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (ci + e < t.Ci) {
            if (g) w[i0 + e] = v[q][e];
            wf[i0 + e] = __float2bfloat16_rn(v[q][e]);
          }
      }
      tile[ty + 8 * q][2 * tx] = v[q][0];
      tile[ty + 8 * q][2 * tx + 1] = v[q][1];
    }
    __syncthreads();
    const int co = co0 + 2 * tx;
    const bool cpair = co + 1 < t.Co && ((t.Co & 1) == 0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int cil = ty + 8 * q, cir = ci0 + cil;
      if (cir >= t.Ci) continue;
      bf16 *dst = wd + ((int64_t)cir * t.taps + (t.taps - 1 - tap)) * t.Co + co;
      if (cpair) {
        *reinterpret_cast<__nv_bfloat162 *>(dst) = __floats2bfloat162_rn(tile[2 * tx][cil], tile[2 * tx + 1][cil]);
      } else {
        if (co < t.Co) dst[0] = __float2bfloat16_rn(tile[2 * tx][cil]);
        if (co + 1 < t.Co) dst[1] = __float2bfloat16_rn(tile[2 * tx + 1][cil]);
      }
    }
    __syncthreads();
  }
}

// w <- w - lr g over the ranges: blockIdx.y = range, blockIdx.x strides within it
// (one range can hold every parameter of the fp32 path: spread it over the SMs)
__global__ void sgd_ranges_k(const int64_t *__restrict__ rg, float *master, const float *__restrict__ grad, float lr) {
  pdl_begin();
  const int64_t a = rg[2 * blockIdx.y], e = rg[2 * blockIdx.y + 1];
  for (int64_t i = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
    master[i] -= lr * grad[i];
}

template <typename T>
__global__ void flip_k(const T *__restrict__ w, int Co, int taps, int Ci, T *__restrict__ wd) {
  pdl_begin();
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
  if (n > SGD_MAX_TENSORS) throw Error(RN_ERR_STATE, "sgd_repack_all: too many conv tensors");
  const unsigned grid = (unsigned)std::min<int64_t>(total_tiles, 148 * 8);
  launch_k(sgd_repack_all_k, grid, dim3(32, 8), 0, st, table_dev, n, (int64_t)0, total_tiles, master, grad, lr);
  LAUNCH_CHECK();
}

void sgd_repack_range(const ConvPack *table_dev, int n, int64_t tile_begin, int64_t tile_end, float *master,
                      const float *grad, float lr, cudaStream_t st) {
  if (n <= 0 || tile_end <= tile_begin) return;
  if (n > SGD_MAX_TENSORS) throw Error(RN_ERR_STATE, "sgd_repack_range: too many conv tensors");
  const unsigned grid = (unsigned)std::min<int64_t>(tile_end - tile_begin, 148 * 8);
  launch_k(sgd_repack_all_k, grid, dim3(32, 8), 0, st, table_dev, n, tile_begin, tile_end, master, grad, lr);
  LAUNCH_CHECK();
}

__global__ void zero_ranges_k(const int64_t *__restrict__ rg, float *g) {
  pdl_begin();
  const int64_t a = rg[2 * blockIdx.y], e = rg[2 * blockIdx.y + 1];
  for (int64_t i = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
    g[i] = 0.f;
}

void zero_ranges(const int64_t *ranges_dev, int n, float *g, cudaStream_t st) {
  if (n <= 0) return;
  launch_k(zero_ranges_k, dim3((unsigned)std::max(1, 148 * 4 / n), (unsigned)n), 256, 0, st, ranges_dev, g);
  LAUNCH_CHECK();
}

void sgd_ranges(const int64_t *ranges_dev, int n, float *master, const float *grad, float lr, cudaStream_t st) {
  if (n <= 0) return;
  launch_k(sgd_ranges_k, dim3((unsigned)std::max(1, 148 * 4 / n), (unsigned)n), 256, 0, st, ranges_dev, master, grad,
           lr);
  LAUNCH_CHECK();
}

void flip_weights(DType dt, const void *w, int Co, int taps, int Ci, void *wd, cudaStream_t st) {
  DISPATCH(dt, launch_k(flip_k<T>, grid_for((int64_t)Co * taps * Ci), NT, 0, st, (const T *)w, Co, taps, Ci, (T *)wd));
  LAUNCH_CHECK();
}

void check_finite(const float *v, int n, int *flag, cudaStream_t st) {
  launch_k(check_finite_k, 1, 256, 0, st, v, n, flag);
  LAUNCH_CHECK();
}

}  // namespace rn
