// FlashButterfly-B200 K1 regularizer math per element (fp64, the
// reference's summation order), shared by the stand-alone regularizer
// kernels (fb_prep.cu) and the fused spectrum / finalize kernels
// (fb_single.cu).  Reference: smooth regularize.cpp:22-34, smooth_frequency
// :36-53, squash :12-20, kernel_dropout :55-64.
#pragma once
#include "fb_common.cuh"

namespace fb {

__device__ __forceinline__ double dropped(const float* __restrict__ K, const uint8_t* keep,
                                          double keep_scale, size_t idx) {
  const double v = (double)__ldg(K + idx);
  if (!keep) return v;
  return keep[idx] ? v * keep_scale : 0.0;
}

// Dirichlet window of smooth_frequency (see header comment).
__device__ __forceinline__ double freq_window(int64_t t, int64_t N, int64_t p) {
  double acc = 1.0;
  const double step = 2.0 * 3.14159265358979323846 / (double)N;
  for (int64_t d = 1; d <= p; ++d) acc += 2.0 * cos(step * (double)((d * t) % N));
  return acc / (double)(2 * p + 1);
}

// squash(smooth(dropout(K)))[t] for row `base` (regularize.cpp:93-107)
__device__ __forceinline__ float reg_value(const float* __restrict__ K, const uint8_t* keep,
                                           double keep_scale, size_t base, int64_t t, int64_t N,
                                           int64_t p, double lambda, int freq) {
  double s;
  if (freq) {
    s = dropped(K, keep, keep_scale, base + t) * freq_window(t, N, p);
  } else {
    const double inv_w = 1.0 / (double)(2 * p + 1);
    const int64_t lo = t >= p ? t - p : 0;
    const int64_t hi = (t + p < N - 1) ? t + p : N - 1;
    double acc = 0.0;
    for (int64_t j = lo; j <= hi; ++j) acc += dropped(K, keep, keep_scale, base + j);
    s = acc * inv_w;
  }
  const double mag = fabs(s) - lambda;
  return mag > 0.0 ? (float)copysign(mag, s) : 0.0f;
}

// chain rule of reg_value at t: dropout'(t) * smooth^T(1[kbar != 0] dkbar)[t]
// (kbar_row / dkbar_row: this head's rows, global or shared memory)
__device__ __forceinline__ float reg_grad(const float* kbar_row, const float* dkbar_row,
                                          const uint8_t* keep_row, int64_t t, int64_t N,
                                          int64_t p, double keep_scale, int freq) {
  double g;
  if (freq) {
    g = (kbar_row[t] != 0.f ? (double)dkbar_row[t] : 0.0) * freq_window(t, N, p);
  } else {
    const int64_t lo = t >= p ? t - p : 0;
    const int64_t hi = (t + p < N - 1) ? t + p : N - 1;
    double acc = 0.0;
    for (int64_t j = lo; j <= hi; ++j)
      if (kbar_row[j] != 0.f) acc += (double)dkbar_row[j];
    g = acc / (double)(2 * p + 1);
  }
  if (keep_row) g = keep_row[t] ? g * keep_scale : 0.0;
  return (float)g;
}

}  // namespace fb
