// tc_conv.h — tcgen05 implicit-GEMM convolution launchers (k_conv_tc.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "bnstats.cuh"
#include "kernels.h"

namespace rn {

// true if the tcgen05 kernels take this convolution (bf16, channels % 64 == 0,
// k in {1, 3}, stride in {1, 2} with the 'same' ceil(in/2) lattice)
bool tc_conv_supported(const ConvGeom &g, bool dgrad);
// CTA-pair dispatch of the persistent tcgen05 kernel for the calling thread:
// -1 = default (RN_TC_PAIR), 0 = never, 1 = every launch it takes (kernel tests)
void tc_pair_force(int mode);
// ws: fp32 split-K workspace of >= tc_conv_ws_floats(g, dgrad) floats (layers with few tiles)
size_t tc_conv_ws_floats(const ConvGeom &g, bool dgrad);
// est (optional): fused BN statistics of the stored output (bnstats.cuh); the
// return value is the number of per-CTA partials written, 0 when not fused
// (split-K or multi-N-block launches, stride-2 dgrad)
int conv_fprop_tc(const ConvGeom &g, const __nv_bfloat16 *x, const __nv_bfloat16 *w, const float *bias,
                  __nv_bfloat16 *y, float *ws, size_t ws_floats, cudaStream_t st, const EpiStats *est = nullptr);
// wd: [Ci][taps][Co] with the tap order flipped (repack_conv's wd).  Stride 2 runs
// the 8 output parity classes in one launch; dy2/wd2 (k3 stride-2 convs only) add
// the stage-entry 1x1x1 stride-2 projection's dgrad (same Ci, Co, geometry) to it
int conv_dgrad_tc(const ConvGeom &g, const __nv_bfloat16 *dy, const __nv_bfloat16 *wd, __nv_bfloat16 *dx,
                  bool accumulate, const __nv_bfloat16 *res, const __nv_bfloat16 *res_mask, float *ws,
                  size_t ws_floats, cudaStream_t st, const EpiStats *est = nullptr,
                  const __nv_bfloat16 *dy2 = nullptr, const __nv_bfloat16 *wd2 = nullptr);

// haloed-A kernel for the 64 -> 64 channel stride-1 3x3x3 convs (k_conv_halo.cu)
bool halo_conv_supported(const ConvGeom &g, bool dgrad);
int conv_halo(const ConvGeom &g, bool dgrad, const __nv_bfloat16 *src, const __nv_bfloat16 *w, const float *bias,
              __nv_bfloat16 *out, bool accumulate, const __nv_bfloat16 *res, const __nv_bfloat16 *res_mask,
              cudaStream_t st, const EpiStats *est = nullptr);

// CTA-pair kernel (cta_group::2, resident weights) for the same 64 -> 64 stride-1
// 3x3x3 convs (k_conv_pair.cu); returns the BN-statistics partial count (0: none)
bool pair_conv_supported(const ConvGeom &g, bool dgrad);
int conv_pair(const ConvGeom &g, bool dgrad, const __nv_bfloat16 *src, const __nv_bfloat16 *w, const float *bias,
              __nv_bfloat16 *out, bool accumulate, const __nv_bfloat16 *res, const __nv_bfloat16 *res_mask,
              cudaStream_t st, const EpiStats *est = nullptr);

// 64 -> 64 channel 1x1x1 stride-1 convs over >= 16 K voxels (k_conv1x1.cu, warp tensor
// cores, streaming): y = x w^T (+ bias) with w [n][k] (forward copy, or the dgrad copy for
// the data gradient); est modes 0-3; returns the BN-statistics partial count
bool conv1x1_supported(const ConvGeom &g);
int conv1x1(const ConvGeom &g, const __nv_bfloat16 *x, const __nv_bfloat16 *w, const float *bias, __nv_bfloat16 *y,
            cudaStream_t st, const EpiStats *est = nullptr);

// weight gradient dw[co][tap][ci] += sum dy x (fp32 partials in ws, fixed-order reduce)
bool tc_wgrad_supported(const ConvGeom &g);
size_t tc_wgrad_ws_floats(const ConvGeom &g);
// overwrite: dW = (not +=) the gradient — the first contribution of a backward pass
void conv_wgrad_tc(const ConvGeom &g, const __nv_bfloat16 *x, const __nv_bfloat16 *dy, float *dw, float *ws,
                   cudaStream_t st, bool overwrite = false);

}  // namespace rn
