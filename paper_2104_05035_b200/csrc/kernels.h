// kernels.h — host launchers for the sm_100a kernels of the 3D-ResAttNet step.
// Plain pointers; layouts: activations NDHWC (channels fastest) of element type
// T = float (RN_F32) or __nv_bfloat16 (RN_BF16); conv weights [Cout][tap][Cin]
// (tap = (kd*k + kh)*k + kw); BN statistics / gradients fp32.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace rn {

enum DType { DT_F32 = 0, DT_BF16 = 1 };
inline size_t dt_size(DType t) { return t == DT_F32 ? 4 : 2; }

struct ConvGeom {
  int N;
  int Di, Hi, Wi, Ci;
  int Do, Ho, Wo, Co;
  int k, s, p;
  __host__ __device__ int64_t in_vox() const { return (int64_t)N * Di * Hi * Wi; }
  __host__ __device__ int64_t out_vox() const { return (int64_t)N * Do * Ho * Wo; }
  __host__ __device__ int taps() const { return k * k * k; }
};

// ---------------- convolution (SIMT implicit GEMM, fp32 accumulate) ----------------
// y[vo][co] = sum_{tap,ci} x[vi(vo,tap)][ci] * w[co][tap][ci] (+ bias[co])
void conv_fprop_simt(DType dt, const ConvGeom &g, const void *x, const void *w, const float *bias, void *y,
                     cudaStream_t st);
// dx[vi][ci] (=|+=) sum_{tap,co} dy[vo(vi,tap)][co] * w[co][tap][ci]  (+ res[vi][ci]*(mask[vi][ci]>0))
void conv_dgrad_simt(DType dt, const ConvGeom &g, const void *dy, const void *w, void *dx, bool accumulate,
                     const void *res, const void *res_mask, cudaStream_t st);
// dw[co][tap][ci] += sum_vo dy[vo][co] * x[vi(vo,tap)][ci]; x_is_f32: input is fp32 (stem)
size_t conv_wgrad_ws_floats(const ConvGeom &g);
void conv_wgrad_simt(DType dt, bool x_is_f32, const ConvGeom &g, const void *x, const void *dy, float *dw,
                     float *ws, cudaStream_t st);
// out[i] += sum_z part[z*n + i] over z < splits, fixed order (split-K weight-gradient partials)
void split_reduce_add(const float *part, int splits, int64_t n, float *out, cudaStream_t st, bool overwrite = false);
// g[a, e) = 0 over n ranges [2][n] (device table)
void zero_ranges(const int64_t *ranges_dev, int n, float *g, cudaStream_t st);
// stem: Ci = 1, x fp32 [N][D][H][W], w fp32 [Co][27]
void stem_conv_fprop(DType dt, const ConvGeom &g, const float *x, const float *w, void *y, cudaStream_t st);
// k_stem.cu: Co in {8,16,32,64}
bool stem_fast_supported(const ConvGeom &g);
size_t stem_wgrad_ws_floats(const ConvGeom &g);
// part (optional): fused BN statistics partials [P][2][Co] of the stored output; returns P
int stem_fprop_fast(DType dt, const ConvGeom &g, const float *x, const float *w, void *y, cudaStream_t st,
                    float *part = nullptr);
// pooled stem backward (bf16, k3 s2 p1 conv, Ci = 1, Co in {8,16,32,64}; reading X23c):
// dgamma / dbeta / dW (+=) from the pooled output y, its argmax am and gradient dy,
// the input x and the stem weights, without any conv-resolution tensor
// Gd [32][32] fp64: G = sum_v X_v X_v^T of the im2col rows, column 27 = sum_v X_v
// (depends only on x: may run on another stream ahead of the backward)
bool stem_bwd_sparse_supported(const ConvGeom &g);
size_t stem_gram_ws_floats();
size_t stem_bwd_sparse_ws_floats();
void stem_gram(const ConvGeom &g, const float *x, float *ws, double *Gd, cudaStream_t st);
void stem_bwd_sparse(const ConvGeom &g, int D2, int H2, int W2, const float *x, const float *w, const void *y,
                     const void *dy, const uint8_t *am, const float *gamma, const float *mean, const float *invstd,
                     const double *Gd, float *dgamma, float *dbeta, float *dw, float *ws, cudaStream_t st);
void stem_wgrad_fast(DType dt, const ConvGeom &g, const float *x, const void *dh, float *dw, float *ws,
                     cudaStream_t st);

// ---------------- BatchNorm (train mode), ReLU, residual ----------------
// y = act(x*scale + shift + R), R = 0 | res | res*rscale + rshift ; act = relu if relu
void bn_apply(DType dt, const void *x, int64_t V, int C, const float *scale, const float *shift, const void *res,
              const float *rscale, const float *rshift, bool relu, void *y, cudaStream_t st);
enum MaskMode { MASK_NONE = 0, MASK_TENSOR = 1, MASK_RECOMPUTE = 2 };
// dx = A dy' + B x + Cc with the coefficients of bn_bwd_reduce_finalize, dy' = dy * mask
void bn_bwd_apply(DType dt, const void *dy, const void *x, int64_t V, int C, int mask_mode, const void *mask_t,
                  const float *scale, const float *shift, const float *coef, void *dx, cudaStream_t st);
// Reduction + finalize in one launch (last-block finalize, deterministic order);
// counter: a zero-initialised uint32 in device memory, left at zero afterwards.
// bn_stats_finalize: statistics of x (shifted by x[0][c]) -> mean / invstd /
//   scale = gamma*invstd / shift = beta - mean*scale, running stats (momentum,
//   unbiased variance).
// bn_bwd_reduce_finalize: S1 = sum dy', S2 = sum dy'*xhat -> dgamma += S2,
//   dbeta += S1, coef[0..C) = A, [C..2C) = B, [2C..3C) = Cc.
int chan_fin_blocks(int64_t V, int C);
void bn_stats_finalize(DType dt, const void *x, int64_t V, int C, float *partial, unsigned *counter,
                       const float *gamma, const float *beta, float *mean, float *invstd, float *scale, float *shift,
                       float *run_mean, float *run_var, float momentum, float eps, cudaStream_t st);
void bn_bwd_reduce_finalize(DType dt, const void *dy, const void *x, int64_t V, int C, int mask_mode,
                            const void *mask_t, const float *scale, const float *shift, const float *mean,
                            const float *invstd, const float *gamma, float *partial, unsigned *counter, float *dgamma,
                            float *dbeta, float *coef, cudaStream_t st);
// BN apply fed by per-CTA statistics partials of the producing convolution
// (bnstats.cuh): part [P][2][C] = (sum y, sum y^2); the kernel finalizes them
// in every block and block 0 publishes mean / invstd / scale / shift and the
// running statistics.  rf (optional): a second BN applied to `res` (projection).
struct BnFinal {
  const float *part;
  int P;
  const float *gamma, *beta;
  float *mean, *invstd, *scale, *shift, *run_mean, *run_var;
  float momentum, eps;
};
void bn_apply_fused(DType dt, const void *x, int64_t V, int C, const BnFinal &f, const BnFinal *rf, const void *res,
                    bool relu, void *y, cudaStream_t st);
// the same partials from a standalone pass over the tensor (layers whose conv
// could not fuse them: split-K, SIMT); returns P
int bn_stats_partials(DType dt, const void *x, int64_t V, int C, float *part, cudaStream_t st);
int bn_bwd_partials(DType dt, const void *dy, const void *h, const void *mask_t, const float *mean, int64_t V, int C,
                    float *part, cudaStream_t st);
// BN backward apply fed by partials (sum dy', sum dy' (h - mean)), dy' = dy * (mask > 0):
// dgamma += sum dy' xhat, dbeta += sum dy', dx = BN-backward(dy')
void bn_bwd_apply_fused(DType dt, const void *dy, const void *h, const void *mask_t, int64_t V, int C,
                        const float *part, int P, const float *gamma, const float *mean, const float *invstd,
                        float *dgamma, float *dbeta, void *dx, cudaStream_t st, float *coef = nullptr,
                        void *dprime = nullptr);  // dprime (optional): dy' = dy * (mask > 0) as well
// stem tail, bf16 (reading X4): y = maxpool(ReLU(BN(h))) with the BN statistics
// finalized from the stem conv's partials (f.part, f.P) and published; argmax uint8
void stem_pool_fwd(const void *h, int N, int D, int H, int W, int C, const BnFinal &f, int64_t V, void *y,
                   uint8_t *am, int Do, int Ho, int Wo, cudaStream_t st);
// attention backward + dbias (sum of dm) in one launch
void att_bwd_finalize(DType dt, const void *dout, const void *m, const void *T_, int64_t V, int C, void *dT, void *dm,
                      float *partial, unsigned *counter, float *dbias, cudaStream_t st);
// ---------------- pooling / upsampling / attention ----------------
// y = maxpool3(act(x*scale+shift)) (scale == nullptr: identity, no act); argmax uint8 (0..26)
void maxpool_fwd(DType dt, const void *x, int N, int D, int H, int W, int C, const float *scale, const float *shift,
                 bool relu, void *y, uint8_t *argmax, int Do, int Ho, int Wo, cudaStream_t st);
void maxpool_bwd(DType dt, const void *dy, const uint8_t *argmax, int N, int D, int H, int W, int C, int Do, int Ho,
                 int Wo, void *dx, bool accumulate, cudaStream_t st);
struct UpTables {  // device pointers
  const int *fw_idx[3];    // [out][2] (i0, i1)
  const float *fw_w[3];    // [out][2] (1-lambda, lambda)
  const int *bw_start[3];  // [in+1]
  const int *bw_o[3];      // [nnz]
  const float *bw_w[3];    // [nnz]
};
// Grad-CAM at the last conv layer: map[n][D][H][W] = trilinear(ReLU(sum_k W[c,k]/V A[n][v][k]))
void gradcam_last(DType dt, const void *A, const float *wrow, int N, int d, int h, int w, int C, float *coarse,
                  float *map, int D, int H, int W, const UpTables &t, cudaStream_t st);
void upsample_fwd(DType dt, const void *x, int N, int Di, int Hi, int Wi, int C, void *y, int Do, int Ho, int Wo,
                  const UpTables &t, cudaStream_t st);
// separable trilinear adjoint (bf16): three passes w, h, d with fp32 intermediates in ws
size_t upsample_bwd_ws_floats(int N, int Di, int Hi, int Wi, int C, int Do, int Ho, int Wo);
void upsample_bwd_sep(const void *dy, int N, int Di, int Hi, int Wi, int C, void *dx, int Do, int Ho, int Wo,
                      const UpTables &t, float *ws, cudaStream_t st);
void upsample_bwd(DType dt, const void *dy, int N, int Di, int Hi, int Wi, int C, void *dx, int Do, int Ho, int Wo,
                  const UpTables &t, cudaStream_t st);
// out = (1 + sigmoid(m)) * T
void att_fwd(DType dt, const void *m, const void *T, int64_t V, int C, void *out, cudaStream_t st);
// dT = dout*(1+s), dm = dout*T*s*(1-s); partial[blk][2][C] = (sum dm, 0)
// out[c] += sum_blk partial[blk][0][c]

// ---------------- head: GAP + FC + softmax cross-entropy ----------------
void head_fwd(DType dt, const void *x, int N, int V, int C, const float *W, const float *b, const int32_t *y,
              float dz_scale, float loss_scale, float *g, float *dz, float *loss_acc, cudaStream_t st);
void head_bwd(DType dt, const float *dz, const float *g, const float *W, int N, int V, int C, float *dW, float *db,
              void *dx, cudaStream_t st);

// ---------------- optimizer ----------------
void sgd_update(float *w, const float *g, int64_t n, float lr, cudaStream_t st);
// wf[co][tap][ci] = w, wd[ci][taps-1-tap][co] = w  (either may be null)
void repack_conv(DType dt, const float *w, int Co, int taps, int Ci, void *wf, void *wd, cudaStream_t st);
// One launch for every conv tensor of the plan: w -= lr * g (g may be null: repack only),
// then the bf16 forward copy wf and the flipped transposed dgrad copy wd (64x64 tiles per tap).
struct ConvPack {
  int64_t off;    // offset of the tensor in the master / gradient arrays
  int64_t tile0;  // first tile index of this tensor in the launch
  int Co, taps, Ci, pad;
  void *wf, *wd;
};
void sgd_repack_all(const ConvPack *table_dev, int n, int64_t total_tiles, float *master, const float *grad, float lr,
                    cudaStream_t st);
// the same over a slice of the table: tiles [tile_begin, tile_end) (absolute tile0
// numbering) of the n tensors at table_dev
void sgd_repack_range(const ConvPack *table_dev, int n, int64_t tile_begin, int64_t tile_end, float *master,
                      const float *grad, float lr, cudaStream_t st);
// SGD over a device list of (offset, count) ranges, one block per range
void sgd_ranges(const int64_t *ranges_dev, int n, float *master, const float *grad, float lr, cudaStream_t st);
void check_finite(const float *v, int n, int *flag, cudaStream_t st);
// wd[ci][taps-1-tap][co] = w[co][tap][ci] (element type dt)
void flip_weights(DType dt, const void *w, int Co, int taps, int Ci, void *wd, cudaStream_t st);

}  // namespace rn
