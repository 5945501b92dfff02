// FlashButterfly-B200: element I/O helpers shared by the kernels.
// I/O types: float, __nv_bfloat16, __half (fb_dtype); arithmetic is fp32.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fb {

__device__ __forceinline__ float tof(float v) { return v; }
__device__ __forceinline__ float tof(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float tof(__half v) { return __half2float(v); }

template <typename T>
__device__ __forceinline__ float ld(const T* p) {
  return tof(__ldg(p));
}

template <typename T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ float cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ __half cvt<__half>(float v) { return __float2half_rn(v); }

template <typename T>
__device__ __forceinline__ void st(T* p, float v) { *p = cvt<T>(v); }

// Interleaved complex (re, im) element of type T at p (p 2*sizeof(T)-aligned).
template <typename T>
__device__ __forceinline__ float2 ldc(const T* p);
template <>
__device__ __forceinline__ float2 ldc<float>(const float* p) {
  return __ldg(reinterpret_cast<const float2*>(p));
}
template <>
__device__ __forceinline__ float2 ldc<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat1622float2(__ldg(reinterpret_cast<const __nv_bfloat162*>(p)));
}
template <>
__device__ __forceinline__ float2 ldc<__half>(const __half* p) {
  return __half22float2(__ldg(reinterpret_cast<const __half2*>(p)));
}

// Same from shared (or any generic) memory: a plain load (__ldg is global-only).
template <typename T>
__device__ __forceinline__ float2 ldc_any(const T* p);
template <>
__device__ __forceinline__ float2 ldc_any<float>(const float* p) {
  return *reinterpret_cast<const float2*>(p);
}
template <>
__device__ __forceinline__ float2 ldc_any<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}
template <>
__device__ __forceinline__ float2 ldc_any<__half>(const __half* p) {
  return __half22float2(*reinterpret_cast<const __half2*>(p));
}

template <typename T>
__device__ __forceinline__ void stc(T* p, float2 v);
template <>
__device__ __forceinline__ void stc<float>(float* p, float2 v) {
  *reinterpret_cast<float2*>(p) = v;
}
template <>
__device__ __forceinline__ void stc<__nv_bfloat16>(__nv_bfloat16* p, float2 v) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __float22bfloat162_rn(v);
}
template <>
__device__ __forceinline__ void stc<__half>(__half* p, float2 v) {
  *reinterpret_cast<__half2*>(p) = __float22half2_rn(v);
}

}  // namespace fb
