// FlashButterfly-B200: complex row transforms and convolutions through the
// butterfly plan — the device side of the reference's single-row entry points
//   build_plan / apply_plan   (butterfly.hpp:74-79, butterfly.cpp:72-185)
//   conv_butterfly            (butterfly.hpp:82-83, butterfly.cpp:187-210)
//   conv_three_pass           (three_pass.hpp:119-120: a circular convolution
//                              with a precomputed kernel spectrum)
// for rows of complex f32 (interleaved re, im).  The transform is the
// plan's own stage chain with the exact DFT blocks (the learned-butterfly
// kernels of fb_learned.cu initialised like LearnedButterfly::from_plan,
// butterfly.cpp:221-227), so any n build_plan(n, r) accepts runs, not only
// powers of two.  Lengths whose stage walk does not fit one CTA's shared
// memory (n > kDirectMax) run as a four-step composition n = n1 n2 of two
// such row transforms with a twiddle and three transposes in between.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "fb_common.cuh"
#include "fb_internal.h"

struct fb_dft_plan {
  int64_t n = 0, r = 0;
  int device = 0;
  // direct: one stage chain of length n; four-step: n = n1 * n2
  int64_t n1 = 0, n2 = 0;
  fb_learned_plan* lp[2] = {nullptr, nullptr};
  float* blocks[2] = {nullptr, nullptr};  // exact DFT blocks per stage chain
  std::vector<int64_t> factors;           // build_plan(n, r) greedy chain
};

namespace fb {
namespace {

constexpr int64_t kDirectMax = 8192;

__global__ void conj_scale_kernel(float2* __restrict__ y, const float2* __restrict__ x, int64_t count,
                                  float scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = x[i];
    y[i] = make_float2(v.x * scale, -v.y * scale);
  }
}

// out[r][t] = t < N ? in[r][t] : 0   (rows of n)
__global__ void pad_kernel(float2* __restrict__ out, const float2* __restrict__ in, int64_t N, int64_t n,
                           int64_t rows) {
  const int64_t count = rows * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, t = i % n;
    out[i] = t < N ? in[r * N + t] : make_float2(0.f, 0.f);
  }
}

// a[r][t] = conj(a[r][t] * b[r % brows][t])  (conj: the inverse runs as conj . F . conj)
__global__ void mul_conj_kernel(float2* __restrict__ a, const float2* __restrict__ b, int64_t n,
                                int64_t rows, int64_t brows) {
  const int64_t count = rows * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, t = i % n;
    const float2 x = a[i], y = b[(r % brows) * n + t];
    a[i] = make_float2(x.x * y.x - x.y * y.y, -(x.x * y.y + x.y * y.x));
  }
}

// out[r][t] = conj(in[r][t]) * scale, t < N  (rows of n in, rows of N out)
__global__ void crop_conj_kernel(float2* __restrict__ out, const float2* __restrict__ in, int64_t N,
                                 int64_t n, int64_t rows, float scale) {
  const int64_t count = rows * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, t = i % N;
    const float2 v = in[r * n + t];
    out[i] = make_float2(v.x * scale, -v.y * scale);
  }
}

// [R][a][b] -> [R][b][a], 32 x 32 tiles through shared memory
__global__ void transpose_kernel(float2* __restrict__ out, const float2* __restrict__ in, int64_t A,
                                 int64_t Bd) {
  __shared__ float2 tile[32][33];
  const int64_t r = blockIdx.z;
  const int64_t a0 = (int64_t)blockIdx.y * 32, b0 = (int64_t)blockIdx.x * 32;
  const float2* src = in + r * A * Bd;
  float2* dst = out + r * A * Bd;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t a = a0 + i, b = b0 + threadIdx.x;
    if (a < A && b < Bd) tile[i][threadIdx.x] = src[a * Bd + b];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t b = b0 + i, a = a0 + threadIdx.x;
    if (a < A && b < Bd) dst[b * A + a] = tile[threadIdx.x][i];
  }
}

// x[r][t2][k1] *= exp(-2 pi i t2 k1 / n)   (the four-step twiddle, fp64 angle)
__global__ void twiddle_kernel(float2* __restrict__ x, int64_t n1, int64_t n2, int64_t rows) {
  const int64_t n = n1 * n2, count = rows * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t loc = i % n, t2 = loc / n1, k1 = loc % n1;
    const int64_t e = (t2 * k1) % n;
    double s, c;
    sincospi(-2.0 * (double)e / (double)n, &s, &c);
    const float2 v = x[i];
    const float cr = (float)c, ci = (float)s;
    x[i] = make_float2(v.x * cr - v.y * ci, v.x * ci + v.y * cr);
  }
}

unsigned grid_for(int64_t count) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148 * 16));
}

int dft_blocks(fb_learned_plan* lp, float** out) {
  int64_t f[32], cnt = 0, pc = 0;
  int rc = fb_learned_plan_factors(lp, f, &cnt, &pc);
  if (rc) return rc;
  std::vector<float2> h((size_t)pc);
  size_t o = 0;
  for (int64_t s = 0; s < cnt; ++s)  // dense_dft_block (butterfly.cpp:13-20): exp(-2 pi i pq / f)
    for (int64_t p = 0; p < f[s]; ++p)
      for (int64_t q = 0; q < f[s]; ++q) {
        const double a = -2.0 * M_PI * (double)((p * q) % f[s]) / (double)f[s];
        h[o++] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
  rc = cuda_status(cudaMalloc(out, sizeof(float2) * std::max<int64_t>(pc, 1)), "cudaMalloc(dft blocks)");
  if (!rc && pc)
    rc = cuda_status(cudaMemcpy(*out, h.data(), sizeof(float2) * pc, cudaMemcpyHostToDevice),
                     "copy dft blocks");
  return rc;
}

// forward transform of `rows` rows (x -> y, distinct buffers); tmp: rows * n
int forward(fb_dft_plan* p, const float2* x, float2* y, int64_t rows, float2* tmp, cudaStream_t s) {
  if (p->n == 1) return cuda_status(cudaMemcpyAsync(y, x, sizeof(float2) * rows, cudaMemcpyDeviceToDevice, s),
                                    "dft copy");
  if (!p->n2)
    return fb_learned_fwd(p->lp[0], p->blocks[0], x, y, rows, nullptr, s);
  const int64_t n1 = p->n1, n2 = p->n2, count = rows * p->n;
  const dim3 tb(32, 8);
  // x [R][t1 n1][t2 n2] -> tmp [R][t2][t1]
  transpose_kernel<<<dim3((unsigned)((n2 + 31) / 32), (unsigned)((n1 + 31) / 32), (unsigned)rows), tb, 0,
                     s>>>(tmp, x, n1, n2);
  int rc = fb_learned_fwd(p->lp[0], p->blocks[0], tmp, y, rows * n2, nullptr, s);  // DFT_n1 over t1
  if (rc) return rc;
  twiddle_kernel<<<grid_for(count), 256, 0, s>>>(y, n1, n2, rows);
  // y [R][t2][k1] -> tmp [R][k1][t2]
  transpose_kernel<<<dim3((unsigned)((n1 + 31) / 32), (unsigned)((n2 + 31) / 32), (unsigned)rows), tb, 0,
                     s>>>(tmp, y, n2, n1);
  rc = fb_learned_fwd(p->lp[1], p->blocks[1], tmp, y, rows * n1, nullptr, s);  // DFT_n2 over t2
  if (rc) return rc;
  // y [R][k1][k2] -> tmp [R][k2][k1] = natural order k1 + n1 k2
  transpose_kernel<<<dim3((unsigned)((n2 + 31) / 32), (unsigned)((n1 + 31) / 32), (unsigned)rows), tb, 0,
                     s>>>(tmp, y, n1, n2);
  return cuda_status(cudaMemcpyAsync(y, tmp, sizeof(float2) * count, cudaMemcpyDeviceToDevice, s),
                     "dft copy");
}

}  // namespace
}  // namespace fb

using namespace fb;

extern "C" {

int fb_dft_plan_create(fb_dft_plan** out, int64_t n, int64_t r, int device) {
  if (!out) {
    set_error("fb_dft_plan_create: null output");
    return FB_ERR_ARG;
  }
  *out = nullptr;
  if (n < 1) {
    set_error("build_plan: n must be >= 1");
    return FB_ERR_PLAN;
  }
  if (r < 2) {
    set_error("build_plan: block size r must be >= 2");
    return FB_ERR_PLAN;
  }
  if (n > (int64_t)UINT32_MAX) {
    set_error("build_plan: n too large");
    return FB_ERR_PLAN;
  }
  // greedy factor chain (butterfly.cpp:83-100): validates n like the reference
  auto* p = new fb_dft_plan();
  p->n = n;
  p->r = r;
  p->device = device;
  for (int64_t seg = n; seg > 1;) {
    int64_t f = 0;
    if (seg <= r) f = seg;
    else
      for (int64_t d = std::min(seg, r); d >= 2; --d)
        if (seg % d == 0) {
          f = d;
          break;
        }
    if (!f) {
      delete p;
      set_error("build_plan: remainder " + std::to_string(seg) + " has no factor <= " +
                std::to_string(r) + "; pad the input to a power of two");
      return FB_ERR_PLAN;
    }
    p->factors.push_back(f);
    seg /= f;
  }
  if (n == 1) {
    *out = p;
    return FB_OK;
  }
  DevGuard dg_(device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (!rc) {
    if (n <= kDirectMax) {
      rc = fb_learned_plan_create(&p->lp[0], n, r, 1, FB_F32, device);
      if (!rc) rc = dft_blocks(p->lp[0], &p->blocks[0]);
    } else {
      // n = n1 n2, both <= kDirectMax: n1 = the shortest prefix product of the
      // plan's factor chain that leaves a remainder <= kDirectMax
      int64_t n1 = 1, best = 0;
      for (int64_t f : p->factors) {
        n1 *= f;
        if (n1 > kDirectMax) break;
        if (n / n1 <= kDirectMax) {
          best = n1;
          break;
        }
      }
      n1 = best;
      if (n1 <= 1) {
        set_error("apply_plan: n = " + std::to_string(n) +
                  " does not split into two device transforms of length <= 8192");
        rc = FB_ERR_UNSUPPORTED;
      } else {
        p->n1 = n1;
        p->n2 = n / n1;
        rc = fb_learned_plan_create(&p->lp[0], p->n1, r, 1, FB_F32, device);
        if (!rc) rc = fb_learned_plan_create(&p->lp[1], p->n2, r, 1, FB_F32, device);
        if (!rc) rc = dft_blocks(p->lp[0], &p->blocks[0]);
        if (!rc) rc = dft_blocks(p->lp[1], &p->blocks[1]);
      }
    }
  }
  if (rc) {
    fb_dft_plan_destroy(p);
    return rc;
  }
  *out = p;
  return FB_OK;
}

int fb_dft_plan_destroy(fb_dft_plan* p) {
  if (!p) return FB_OK;
  for (int i = 0; i < 2; ++i) {
    fb_learned_plan_destroy(p->lp[i]);
    cudaFree(p->blocks[i]);
  }
  delete p;
  return FB_OK;
}

int fb_dft_plan_factors(const fb_dft_plan* p, int64_t* factors, int64_t* count) {
  if (!p) {
    set_error("fb_dft_plan_factors: null plan");
    return FB_ERR_ARG;
  }
  if (count) *count = (int64_t)p->factors.size();
  if (factors)
    for (size_t i = 0; i < p->factors.size(); ++i) factors[i] = p->factors[i];
  return FB_OK;
}

// row buffers of the transform length: dft (k_rows = 0): the conjugated
// input and the four-step scratch; conv: the spectrum of u, the padded input,
// the kernel spectrum (k_rows rows) and the four-step scratch
size_t fb_dft_workspace_size(const fb_dft_plan* p, int64_t rows, int64_t k_rows) {
  if (!p || rows < 1) return 0;
  const int64_t kr = std::max<int64_t>(k_rows, 0);
  const int64_t nrows = kr ? 2 * rows + kr + std::max(rows, kr) : 2 * rows;
  return sizeof(float2) * (size_t)p->n * (size_t)nrows + 256;
}

int fb_dft(fb_dft_plan* p, const float* x, float* y, int64_t rows, int inverse, void* ws, void* stream) {
  if (!p || !x || !y || !ws) {
    set_error("fb_dft: null argument");
    return FB_ERR_ARG;
  }
  if (rows < 1) {
    set_error("apply_plan: rows must be >= 1");
    return FB_ERR_DIM;
  }
  DevGuard dg_(p->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t count = rows * p->n;
  float2* a = (float2*)ws;
  float2* tmp = a + count;
  if (!inverse) {
    rc = forward(p, (const float2*)x, (float2*)y, rows, tmp, s);
  } else {  // inverse = conj(F conj(x)) / n  (butterfly.cpp:178-184)
    conj_scale_kernel<<<grid_for(count), 256, 0, s>>>(a, (const float2*)x, count, 1.f);
    rc = forward(p, a, (float2*)y, rows, tmp, s);
    if (!rc)
      conj_scale_kernel<<<grid_for(count), 256, 0, s>>>((float2*)y, (const float2*)y, count,
                                                         (float)(1.0 / (double)p->n));
  }
  if (rc) return rc;
  return cuda_status(cudaGetLastError(), "fb_dft");
}

// y = conv(u, k) per row: circular (plan n == N) or causal (plan n == 2N, the
// first N of the zero-padded circular result).  k: k_rows rows (1: shared by
// every row, else rows); kspec (if k is null): the kernel's forward spectrum,
// k_rows rows of length n (conv_three_pass's precomputed K_hat).
static int conv_impl(fb_dft_plan* p, const float* u, const float* k, const float* kspec, float* y,
                     int64_t N, int64_t rows, int64_t k_rows, int mode, void* ws, void* stream) {
  if (!p || !u || (!k && !kspec) || !y || !ws) {
    set_error("fb_conv_rows: null argument");
    return FB_ERR_ARG;
  }
  if (rows < 1 || N < 1 || (k_rows != 1 && k_rows != rows)) {
    set_error("conv_butterfly: u and k length mismatch");
    return FB_ERR_DIM;
  }
  if (mode == FB_MODE_CIRCULAR ? p->n != N : p->n != 2 * N) {
    set_error(mode == FB_MODE_CIRCULAR ? "conv_butterfly: circular mode needs plan.n == N"
                                       : "conv_butterfly: causal mode needs plan.n == 2N");
    return FB_ERR_DIM;
  }
  DevGuard dg_(p->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = p->n;
  float2* U = (float2*)ws;              // rows x n: spectrum of u
  float2* T = U + rows * n;             // rows x n: padded rows
  float2* KS = T + rows * n;            // k_rows x n: kernel spectrum
  float2* SCR = KS + k_rows * n;        // max(rows, k_rows) x n: four-step scratch
  pad_kernel<<<grid_for(rows * n), 256, 0, s>>>(T, (const float2*)u, N, n, rows);
  rc = forward(p, T, U, rows, SCR, s);
  if (rc) return rc;
  const float2* kf = (const float2*)kspec;
  if (!kspec) {
    pad_kernel<<<grid_for(k_rows * n), 256, 0, s>>>(T, (const float2*)k, N, n, k_rows);
    rc = forward(p, T, KS, k_rows, SCR, s);
    if (rc) return rc;
    kf = KS;
  }
  mul_conj_kernel<<<grid_for(rows * n), 256, 0, s>>>(U, kf, n, rows, k_rows);
  rc = forward(p, U, T, rows, SCR, s);
  if (rc) return rc;
  crop_conj_kernel<<<grid_for(rows * N), 256, 0, s>>>((float2*)y, T, N, n, rows,
                                                       (float)(1.0 / (double)n));
  return cuda_status(cudaGetLastError(), "fb_conv_rows");
}

int fb_conv_rows(fb_dft_plan* p, const float* u, const float* k, float* y, int64_t N, int64_t rows,
                 int64_t k_rows, int mode, void* ws, void* stream) {
  return conv_impl(p, u, k, nullptr, y, N, rows, k_rows, mode, ws, stream);
}

int fb_conv_rows_spectrum(fb_dft_plan* p, const float* u, const float* kspec, float* y, int64_t N,
                          int64_t rows, int64_t k_rows, int mode, void* ws, void* stream) {
  return conv_impl(p, u, nullptr, kspec, y, N, rows, k_rows, mode, ws, stream);
}

}  // extern "C"
