// FlashButterfly-B200 K1 regularizers: dropout -> Smooth -> Squash
// (Algorithm 1 lines 1-3) and their chain rule.
//
// Reference: regularize_bank (proj/src/regularize.cpp:93-107) with
//   kernel_dropout (:55-64), smooth (:22-34), smooth_frequency (:36-53),
//   squash (:12-20).
// The regularizer math runs in fp64 with the reference's summation order so
// the squash support (and therefore the dK mask) matches the fp64 oracle
// exactly; only the final Kbar is rounded to fp32.
//
// smooth_frequency is evaluated without the O(N^2) DFT of the reference: a
// circular (2p+1)-window average of the spectrum is, by the shift theorem,
// the pointwise product of the signal with the Dirichlet window
//   w[t] = (2p+1)^-1 sum_{d=-p..p} exp(-2 pi i d t / N)
//        = (2p+1)^-1 (1 + 2 sum_{d=1..p} cos(2 pi d t / N)),
// which is real, so smooth_frequency(k) = k * w (and is self-adjoint).
#include "fb_common.cuh"
#include "fb_internal.h"
#include "fb_reg.cuh"

namespace fb {

// SeededRng (rng.cpp:12-55): splitmix64-seeded xoshiro256++.
struct DevRng {
  uint64_t s[4];
  __device__ static uint64_t splitmix(uint64_t& x) {
    x += 0x9E3779B97F4A7C15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  __device__ void seed_with(uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) s[i] = splitmix(x);
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 1;
  }
  // SeededRng(seed).child(stream)  (rng.cpp:35-39)
  __device__ void child_of(uint64_t seed, uint64_t stream) {
    uint64_t base = seed;
    uint64_t v = splitmix(base) + stream;
    seed_with(splitmix(v));
  }
  __device__ uint64_t next() {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  __device__ double uniform01() { return (double)(next() >> 11) * 0x1.0p-53; }
};

// keep[h][i] = !(uniform01() < rate), drawn in order from child stream h.
// The stream is sequential by construction, so one thread walks one head.
__global__ void dropout_keep_kernel(uint8_t* __restrict__ keep, int H, int64_t N, double rate,
                                    uint64_t seed, int64_t head0) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= H) return;
  DevRng r;
  r.child_of(seed, (uint64_t)(head0 + h));
  uint8_t* k = keep + (size_t)h * N;
  for (int64_t i = 0; i < N; ++i) k[i] = (r.uniform01() < rate) ? 0 : 1;
}

// kbar[h][t] = squash(smooth(dropout(K))[t], lambda)
__global__ void regularize_kernel(const float* __restrict__ K, const uint8_t* __restrict__ keep,
                                  float* __restrict__ kbar, int64_t N, int64_t p, double lambda,
                                  double keep_scale, int freq) {
  const int64_t t = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (t >= N) return;
  const size_t base = (size_t)blockIdx.x * N;
  kbar[base + t] = reg_value(K, keep, keep_scale, base, t, N, p, lambda, freq);
}

// dK[h][t] = dropout'(t) * smooth^T(1[kbar != 0] * dkbar)[t]
__global__ void regularizer_backward_kernel(const float* __restrict__ kbar,
                                            const float* __restrict__ dkbar,
                                            const uint8_t* __restrict__ keep,
                                            float* __restrict__ dK, int64_t N, int64_t p,
                                            double keep_scale, int freq) {
  const int64_t t = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (t >= N) return;
  const size_t base = (size_t)blockIdx.x * N;
  dK[base + t] = reg_grad(kbar + base, dkbar + base, keep ? keep + base : nullptr, t, N, p,
                          keep_scale, freq);
}

// Time-domain fast path (smooth width p <= kRegHalo): a CTA stages a tile of
// the row (plus the +-p halo) in smem once and every output reads its window
// from there, with 32-bit indexing; same fp64 arithmetic and summation order
// as reg_value / reg_grad.
constexpr int kRegTile = 2048, kRegHalo = 32, kRegThreads = 256;

__global__ void __launch_bounds__(kRegThreads)
    regularize_tile_kernel(const float* __restrict__ K, const uint8_t* __restrict__ keep,
                           float* __restrict__ kbar, int N, int p, double lambda, double keep_scale) {
  __shared__ double sk[kRegTile + 2 * kRegHalo];
  const size_t base = (size_t)blockIdx.y * N;
  const int t0 = blockIdx.x * kRegTile;
  for (int i = threadIdx.x; i < kRegTile + 2 * p; i += kRegThreads) {
    const int t = t0 - p + i;
    sk[i] = (t >= 0 && t < N) ? dropped(K, keep, keep_scale, base + t) : 0.0;
  }
  __syncthreads();
  const double inv_w = 1.0 / (double)(2 * p + 1);
  for (int i = threadIdx.x; i < kRegTile; i += kRegThreads) {
    const int t = t0 + i;
    if (t >= N) break;
    const int lo = t >= p ? -p : -t;
    const int hi = (t + p < N - 1) ? p : N - 1 - t;
    double acc = 0.0;
    for (int d = lo; d <= hi; ++d) acc += sk[i + p + d];
    const double sv = acc * inv_w;
    const double mag = fabs(sv) - lambda;
    kbar[base + t] = mag > 0.0 ? (float)copysign(mag, sv) : 0.0f;
  }
}

__global__ void __launch_bounds__(kRegThreads)
    regularizer_backward_tile_kernel(const float* __restrict__ kbar, const float* __restrict__ dkbar,
                                     const uint8_t* __restrict__ keep, float* __restrict__ dK, int N,
                                     int p, double keep_scale) {
  __shared__ double sg[kRegTile + 2 * kRegHalo];  // 1[kbar != 0] dkbar
  const size_t base = (size_t)blockIdx.y * N;
  const int t0 = blockIdx.x * kRegTile;
  for (int i = threadIdx.x; i < kRegTile + 2 * p; i += kRegThreads) {
    const int t = t0 - p + i;
    double g = 0.0;
    if (t >= 0 && t < N && __ldg(kbar + base + t) != 0.f) g = (double)__ldg(dkbar + base + t);
    sg[i] = g;
  }
  __syncthreads();
  const double w = (double)(2 * p + 1);
  for (int i = threadIdx.x; i < kRegTile; i += kRegThreads) {
    const int t = t0 + i;
    if (t >= N) break;
    const int lo = t >= p ? -p : -t;
    const int hi = (t + p < N - 1) ? p : N - 1 - t;
    double acc = 0.0;
    for (int d = lo; d <= hi; ++d) acc += sg[i + p + d];
    double g = acc / w;
    if (keep) g = keep[base + t] ? g * keep_scale : 0.0;
    dK[base + t] = (float)g;
  }
}

int dropout_keep_dev(fb_plan* p, double rate, uint64_t seed, cudaStream_t s) {
  dropout_keep_kernel<<<(unsigned)((p->H + 127) / 128), 128, 0, s>>>(p->keep, (int)p->H, p->N,
                                                                       rate, seed, p->head0);
  return cuda_status(cudaGetLastError(), "dropout_keep");
}

int regularize_bank_dev(fb_plan* p, const float* K, cudaStream_t s) {
  if (p->smooth_domain != FB_SMOOTH_FREQUENCY && p->p <= kRegHalo && p->N < (int64_t(1) << 30)) {
    const dim3 g((unsigned)((p->N + kRegTile - 1) / kRegTile), (unsigned)p->H);
    regularize_tile_kernel<<<g, kRegThreads, 0, s>>>(K, p->use_keep ? p->keep : nullptr, p->kbar,
                                                     (int)p->N, (int)p->p, p->lambda, p->keep_scale);
    return cuda_status(cudaGetLastError(), "regularize_bank");
  }
  const dim3 g((unsigned)p->H, (unsigned)((p->N + 255) / 256));
  regularize_kernel<<<g, 256, 0, s>>>(K, p->use_keep ? p->keep : nullptr, p->kbar, p->N, p->p,
                                      p->lambda, p->keep_scale,
                                      p->smooth_domain == FB_SMOOTH_FREQUENCY);
  return cuda_status(cudaGetLastError(), "regularize_bank");
}

int regularizer_backward_dev(fb_plan* p, const float* dkbar, float* dK, cudaStream_t s) {
  if (p->smooth_domain != FB_SMOOTH_FREQUENCY && p->p <= kRegHalo && p->N < (int64_t(1) << 30)) {
    const dim3 g((unsigned)((p->N + kRegTile - 1) / kRegTile), (unsigned)p->H);
    regularizer_backward_tile_kernel<<<g, kRegThreads, 0, s>>>(
        p->kbar, dkbar, p->use_keep ? p->keep : nullptr, dK, (int)p->N, (int)p->p, p->keep_scale);
    return cuda_status(cudaGetLastError(), "regularizer_backward");
  }
  const dim3 g((unsigned)p->H, (unsigned)((p->N + 255) / 256));
  regularizer_backward_kernel<<<g, 256, 0, s>>>(p->kbar, dkbar, p->use_keep ? p->keep : nullptr,
                                                dK, p->N, p->p, p->keep_scale,
                                                p->smooth_domain == FB_SMOOTH_FREQUENCY);
  return cuda_status(cudaGetLastError(), "regularizer_backward");
}

}  // namespace fb
