// util.cuh — small device helpers shared by the kernels (type conversion,
// 16-byte vector loads/stores of NDHWC channel vectors).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace rn {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(bf16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// number of elements in a 16-byte vector
template <typename T>
struct Vec {
  static constexpr int N = 16 / sizeof(T);
};

// load / store N = Vec<T>::N consecutive elements (16-byte aligned)
__device__ __forceinline__ void load_vec(const float *p, float *v) {
  float4 a = *reinterpret_cast<const float4 *>(p);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void load_vec(const bf16 *p, float *v) {
  uint4 a = *reinterpret_cast<const uint4 *>(p);
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void store_vec(float *p, const float *v) {
  *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void store_vec(bf16 *p, const float *v) {
  uint4 a;
  __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4 *>(p) = a;
}

// store 8 consecutive elements
__device__ __forceinline__ void store8(float *p, const float *v) {
  store_vec(p, v);
  store_vec(p + 4, v + 4);
}
__device__ __forceinline__ void store8(bf16 *p, const float *v) { store_vec(p, v); }

// Programmatic Dependent Launch (see launch.h): wait for the predecessor grid
// (no-op when launched without PDL), then allow the successor to launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// (no early trigger: the dependent grid may launch when this one's blocks exit,
// so its launch latency / prologue overlap this grid's teardown; an early
// trigger measured slower — dependents squat on SMs the remaining waves need)
__device__ __forceinline__ void pdl_begin() { pdl_wait(); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}


// pull one line into L2 ahead of use (no register, no completion tracking)
__device__ __forceinline__ void prefetch_l2(const void *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
}  // namespace rn
