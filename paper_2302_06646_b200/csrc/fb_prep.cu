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
#include <mutex>
#include <vector>

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

// Jump-ahead: the xoshiro256 state update is linear over GF(2)^256, so s_k =
// M^k s_0.  jump_mats() holds P_j = M^(2^j), j < 32, as 256 rows x 4 words
// (row i: the state bits that feed output bit i); a thread reaches draw k of a
// stream with popcount(k) matrix-vector products, then walks its chunk
// sequentially — every head's stream splits over many threads with results
// bit-identical to the sequential reference walk.
constexpr int kJumpBits = 32;
__device__ __forceinline__ void rng_jump(uint64_t s[4], uint64_t steps, const uint64_t* __restrict__ P) {
  for (int j = 0; steps; ++j, steps >>= 1) {
    if (!(steps & 1)) continue;
    const uint64_t* rows = P + (size_t)j * 256 * 4;
    uint64_t o[4] = {0, 0, 0, 0};
    for (int i = 0; i < 256; ++i) {
      const uint64_t* r = rows + 4 * i;
      const uint64_t v = (__ldg(r) & s[0]) ^ (__ldg(r + 1) & s[1]) ^ (__ldg(r + 2) & s[2]) ^ (__ldg(r + 3) & s[3]);
      o[i >> 6] |= (uint64_t)(__popcll(v) & 1) << (i & 63);
    }
    for (int w = 0; w < 4; ++w) s[w] = o[w];
  }
}
constexpr int64_t kRngChunk = 512;  // draws per thread

// keep[h][i] = !(uniform01() < rate), draw i of child stream h; thread (h, c)
// jumps to draw c kRngChunk and walks its chunk.
__global__ void dropout_keep_kernel(uint8_t* __restrict__ keep, int H, int64_t N, double rate,
                                    uint64_t seed, int64_t head0, const uint64_t* __restrict__ P) {
  const int64_t chunks = (N + kRngChunk - 1) / kRngChunk;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= H * chunks) return;
  const int h = (int)(g / chunks);
  const int64_t i0 = (g % chunks) * kRngChunk, i1 = min(N, i0 + kRngChunk);
  DevRng r;
  r.child_of(seed, (uint64_t)(head0 + h));
  rng_jump(r.s, (uint64_t)i0, P);
  uint8_t* k = keep + (size_t)h * N;
  for (int64_t i = i0; i < i1; ++i) k[i] = (r.uniform01() < rate) ? 0 : 1;
}

// init_kernels (regularize.cpp:66-91): K[h][i] = normal draw i of child
// stream h (Box-Muller pairs, rng.cpp:57-69: cos then the cached sin), times
// the geometric envelope exp(-(i / N) (H / 2)^(h / H)) for kind 1; D[h] = draw
// h of child stream H.  fp64 like the reference, stored f32 and/or f64.
__global__ void init_kernels_kernel(int kind, int H, int64_t N, uint64_t seed, float* __restrict__ K,
                                    double* __restrict__ K64, const uint64_t* __restrict__ P) {
  const int64_t chunks = (N + kRngChunk - 1) / kRngChunk;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= H * chunks) return;
  const int h = (int)(g / chunks);
  const int64_t i0 = (g % chunks) * kRngChunk, i1 = min(N, i0 + kRngChunk);
  DevRng r;
  r.child_of(seed, (uint64_t)h);
  rng_jump(r.s, (uint64_t)i0, P);  // kRngChunk is even: chunks start on a pair
  const double decay = pow((double)H / 2.0, (double)h / (double)H);
  for (int64_t i = i0; i < i1; i += 2) {
    const double u1 = 1.0 - r.uniform01(), u2 = r.uniform01();
    const double rad = sqrt(-2.0 * log(u1)), ang = 2.0 * M_PI * u2;
    double v[2] = {rad * cos(ang), rad * sin(ang)};
    for (int e = 0; e < 2 && i + e < i1; ++e) {
      double x = v[e];
      if (kind) x *= exp(-((double)(i + e) / (double)N) * decay);
      if (K) K[(size_t)h * N + i + e] = (float)x;
      if (K64) K64[(size_t)h * N + i + e] = x;
    }
  }
}
__global__ void init_skip_kernel(int H, uint64_t seed, float* __restrict__ D, double* __restrict__ D64) {
  DevRng r;
  r.child_of(seed, (uint64_t)H);
  for (int h = 0; h < H; h += 2) {
    const double u1 = 1.0 - r.uniform01(), u2 = r.uniform01();
    const double rad = sqrt(-2.0 * log(u1)), ang = 2.0 * M_PI * u2;
    const double v[2] = {rad * cos(ang), rad * sin(ang)};
    for (int e = 0; e < 2 && h + e < H; ++e) {
      if (D) D[h + e] = (float)v[e];
      if (D64) D64[h + e] = v[e];
    }
  }
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
  if (!keep && (N & 3) == 0 && t0 + kRegTile <= N) {
    // whole tile: both 16-byte loads per thread in flight at once, halo apart
    const float4* src = reinterpret_cast<const float4*>(K + base + t0);
    float4 v[kRegTile / (4 * kRegThreads)];
#pragma unroll
    for (int j = 0; j < kRegTile / (4 * kRegThreads); ++j) v[j] = __ldg(src + threadIdx.x + j * kRegThreads);
#pragma unroll
    for (int j = 0; j < kRegTile / (4 * kRegThreads); ++j) {
      double* d = sk + p + 4 * (threadIdx.x + j * kRegThreads);
      d[0] = v[j].x;
      d[1] = v[j].y;
      d[2] = v[j].z;
      d[3] = v[j].w;
    }
    if ((int)threadIdx.x < 2 * p) {
      const int i = threadIdx.x < (unsigned)p ? (int)threadIdx.x : kRegTile + (int)threadIdx.x;
      const int t = t0 - p + i;
      sk[i] = (t >= 0 && t < N) ? (double)__ldg(K + base + t) : 0.0;
    }
  } else {
    for (int i = threadIdx.x; i < kRegTile + 2 * p; i += kRegThreads) {
      const int t = t0 - p + i;
      sk[i] = (t >= 0 && t < N) ? dropped(K, keep, keep_scale, base + t) : 0.0;
    }
  }
  __syncthreads();
  const double inv_w = 1.0 / (double)(2 * p + 1);
#pragma unroll 4
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
  if ((N & 3) == 0 && t0 + kRegTile <= N) {
    constexpr int V = kRegTile / (4 * kRegThreads);
    const float4* kb = reinterpret_cast<const float4*>(kbar + base + t0);
    const float4* dk = reinterpret_cast<const float4*>(dkbar + base + t0);
    float4 a[V], g[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      a[j] = __ldg(kb + threadIdx.x + j * kRegThreads);
      g[j] = __ldg(dk + threadIdx.x + j * kRegThreads);
    }
#pragma unroll
    for (int j = 0; j < V; ++j) {
      double* d = sg + p + 4 * (threadIdx.x + j * kRegThreads);
      d[0] = a[j].x != 0.f ? (double)g[j].x : 0.0;
      d[1] = a[j].y != 0.f ? (double)g[j].y : 0.0;
      d[2] = a[j].z != 0.f ? (double)g[j].z : 0.0;
      d[3] = a[j].w != 0.f ? (double)g[j].w : 0.0;
    }
    if ((int)threadIdx.x < 2 * p) {
      const int i = threadIdx.x < (unsigned)p ? (int)threadIdx.x : kRegTile + (int)threadIdx.x;
      const int t = t0 - p + i;
      double gv = 0.0;
      if (t >= 0 && t < N && __ldg(kbar + base + t) != 0.f) gv = (double)__ldg(dkbar + base + t);
      sg[i] = gv;
    }
  } else {
    for (int i = threadIdx.x; i < kRegTile + 2 * p; i += kRegThreads) {
      const int t = t0 - p + i;
      double gv = 0.0;
      if (t >= 0 && t < N && __ldg(kbar + base + t) != 0.f) gv = (double)__ldg(dkbar + base + t);
      sg[i] = gv;
    }
  }
  __syncthreads();
  const double inv_w = 1.0 / (double)(2 * p + 1);
#pragma unroll 4
  for (int i = threadIdx.x; i < kRegTile; i += kRegThreads) {
    const int t = t0 + i;
    if (t >= N) break;
    const int lo = t >= p ? -p : -t;
    const int hi = (t + p < N - 1) ? p : N - 1 - t;
    double acc = 0.0;
    for (int d = lo; d <= hi; ++d) acc += sg[i + p + d];
    double g = acc * inv_w;
    if (keep) g = keep[base + t] ? g * keep_scale : 0.0;
    dK[base + t] = (float)g;
  }
}

namespace {
// P_j = M^(2^j) of the xoshiro256 state update, built once per device
void xo_step(uint64_t s[4]) {
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}
const uint64_t* jump_mats(int device, int& rc) {
  static const uint64_t* dev[64] = {nullptr};
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  rc = FB_OK;
  if (device < 0 || device >= 64) {
    rc = FB_ERR_ARG;
    return nullptr;
  }
  if (dev[device]) return dev[device];
  std::vector<uint64_t> P((size_t)kJumpBits * 256 * 4, 0);
  for (int j = 0; j < 256; ++j) {  // M: column j = one step of the unit state e_j
    uint64_t e[4] = {0, 0, 0, 0};
    e[j >> 6] = uint64_t(1) << (j & 63);
    xo_step(e);
    for (int i = 0; i < 256; ++i)
      if ((e[i >> 6] >> (i & 63)) & 1) P[(size_t)4 * i + (j >> 6)] |= uint64_t(1) << (j & 63);
  }
  for (int k = 1; k < kJumpBits; ++k) {  // P_k = P_{k-1}^2 (rows: XOR of the rows they select)
    const uint64_t* A = &P[(size_t)(k - 1) * 1024];
    uint64_t* R = &P[(size_t)k * 1024];
    for (int i = 0; i < 256; ++i)
      for (int j = 0; j < 256; ++j)
        if ((A[4 * i + (j >> 6)] >> (j & 63)) & 1)
          for (int w = 0; w < 4; ++w) R[4 * i + w] ^= A[4 * j + w];
  }
  uint64_t* d = nullptr;
  rc = cuda_status(cudaMalloc(&d, P.size() * 8), "cudaMalloc(rng jump)");
  if (!rc) rc = cuda_status(cudaMemcpy(d, P.data(), P.size() * 8, cudaMemcpyHostToDevice), "copy rng jump");
  if (rc) return nullptr;
  dev[device] = d;
  return d;
}
unsigned rng_blocks(int64_t H, int64_t N) {
  return (unsigned)((H * ((N + kRngChunk - 1) / kRngChunk) + 127) / 128);
}
}  // namespace

int dropout_keep_dev(fb_plan* p, double rate, uint64_t seed, cudaStream_t s) {
  int rc = FB_OK;
  const uint64_t* P = jump_mats(p->device, rc);
  if (rc) return rc;
  dropout_keep_kernel<<<rng_blocks(p->H, p->N), 128, 0, s>>>(p->keep, (int)p->H, p->N, rate, seed,
                                                             p->head0, P);
  return cuda_status(cudaGetLastError(), "dropout_keep");
}

int init_kernels_dev(int kind, int64_t H, int64_t N, uint64_t seed, float* K, float* D, double* K64,
                     double* D64, int device, cudaStream_t s) {
  int rc = FB_OK;
  const uint64_t* P = jump_mats(device, rc);
  if (rc) return rc;
  if (K || K64)
    init_kernels_kernel<<<rng_blocks(H, N), 128, 0, s>>>(kind, (int)H, N, seed, K, K64, P);
  if (D || D64) init_skip_kernel<<<1, 1, 0, s>>>((int)H, seed, D, D64);
  return cuda_status(cudaGetLastError(), "init_kernels");
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
