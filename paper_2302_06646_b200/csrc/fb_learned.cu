// FlashButterfly-B200 learned butterfly (K5): the DFT blocks of the plan
// become trainable per-head f x f complex matrices (§3.2.1).
//
// Reference: LearnedButterfly / learned_forward / learned_gradients
// (proj/src/butterfly.cpp:221-307) over the stage walk apply_stages
// (:124-163).  Writing the reference's gather / dense block / scatter +
// twiddle of stage s (factor f, segment L, rest = L/f) in matrix form, each
// length-L segment viewed as an f x rest matrix M[p][q] = cur[p*rest + q]
// is updated in place as
//     M'[a][q] = exp(-2 pi i a q / L) * sum_p W_s[a][p] M[p][q]
// (the gather/scatter permutations cancel), and the final output is
// y[i] = cur[output_map[i]] (:161).  The adjoint (:248-307) is
//     w[a][q]  = conj(tw(a,q)) g[a*rest + q]
//     G_s[a][p] += sum_{seg,q} w[a][q] conj(M_s[p][q])        (block grad)
//     g'[p*rest + q] = sum_a conj(W_s[a][p]) w[a][q]          (input grad)
// starting from g[output_map[i]] = upstream[i].
//
// One CTA per head owns the head's blocks in shared memory; the backward CTA
// walks all B rows of its head in order, so dblocks (summed over b) are
// deterministic without atomics.
#include <algorithm>
#include <cmath>
#include <vector>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"

namespace fb {

constexpr int kLbThreads = 256;
constexpr int kLbMaxStages = 32;

struct LbStages {
  int nstages;
  int f[kLbMaxStages];
  int L[kLbMaxStages];
  int off[kLbMaxStages];  // complex offset of stage block in the per-head params
};

// stage s in place: dst = T .* (W_s x M) per segment (src -> dst buffers)
__device__ __forceinline__ void lb_stage(const float2* __restrict__ src, float2* __restrict__ dst,
                                         const float2* __restrict__ W, int f, int L, uint32_t n,
                                         const float2* __restrict__ tw) {
  const int rest = L / f;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t seg = i / L, loc = i % L, a = loc / rest, q = loc % rest;
    const float2* col = src + seg * L + q;
    const float2* wr = W + a * f;
    float2 acc = make_float2(0.f, 0.f);
    for (int p = 0; p < f; ++p) {
      const float2 w = wr[p], x = col[p * rest];
      acc.x = fmaf(w.x, x.x, fmaf(-w.y, x.y, acc.x));
      acc.y = fmaf(w.x, x.y, fmaf(w.y, x.x, acc.y));
    }
    // exp(-2 pi i a q / L) = tw_n[a q (n / L)]
    dst[i] = cmul(acc, __ldg(tw + (size_t)a * q * (n / L)));
  }
}

template <typename IO>
__global__ void __launch_bounds__(kLbThreads)
    lb_fwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x, IO* __restrict__ y,
                  const uint32_t* __restrict__ omap, const float2* __restrict__ tw, LbStages st,
                  int B, int H, uint32_t n, int P, int rows_per_cta) {
  extern __shared__ __align__(16) float2 lsm[];
  float2* W = lsm;          // [P]
  float2* b0 = W + P;       // [n]
  float2* b1 = b0 + n;      // [n]
  const int h = blockIdx.x;
  const float2* wg = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) W[i] = wg[i];
  const int r0 = blockIdx.y * rows_per_cta, r1 = min(B, r0 + rows_per_cta);
  for (int b = r0; b < r1; ++b) {
    const IO* xr = x + ((size_t)b * H + h) * 2 * n;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) b0[i] = ldc<IO>(xr + 2 * i);
    __syncthreads();
    float2 *s = b0, *d = b1;
    for (int k = 0; k < st.nstages; ++k) {
      lb_stage(s, d, W + st.off[k], st.f[k], st.L[k], n, tw);
      __syncthreads();
      float2* t = s;
      s = d;
      d = t;
    }
    IO* yr = y + ((size_t)b * H + h) * 2 * n;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) stc<IO>(yr + 2 * i, s[__ldg(omap + i)]);
  }
}

// CTA (h, split): rows b in [split * rows, ...) of head h, in order; the
// block gradient partial of the split goes to gpart[split][h] and
// lb_reduce_kernel sums the splits in a fixed order (deterministic).
template <typename IO>
__global__ void __launch_bounds__(kLbThreads)
    lb_bwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x,
                  const IO* __restrict__ g, IO* __restrict__ dx, float2* __restrict__ gpart,
                  const uint32_t* __restrict__ omap, const float2* __restrict__ tw, LbStages st,
                  int B, int H, uint32_t n, int P, int rows) {
  extern __shared__ __align__(16) float2 lsm[];
  float2* W = lsm;                          // [P]
  float2* G = W + P;                        // [P] gradient accumulator
  float2* red = G + P;                      // [kLbThreads] column-split partials
  float2* saved = red + kLbThreads;         // [S][n] stage inputs
  float2* ga = saved + (size_t)st.nstages * n;  // [n]
  float2* gb = ga + n;                      // [n]
  const int h = blockIdx.x;
  const int b_begin = blockIdx.y * rows, b_end = min(B, b_begin + rows);
  const float2* wg = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    W[i] = wg[i];
    G[i] = make_float2(0.f, 0.f);
  }
  for (int b = b_begin; b < b_end; ++b) {
    const IO* xr = x + ((size_t)b * H + h) * 2 * n;
    const IO* gr = g + ((size_t)b * H + h) * 2 * n;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) saved[i] = ldc<IO>(xr + 2 * i);
    __syncthreads();
    // forward, keeping each stage's input
    for (int k = 0; k + 1 < st.nstages; ++k) {
      lb_stage(saved + (size_t)k * n, saved + (size_t)(k + 1) * n, W + st.off[k], st.f[k], st.L[k],
               n, tw);
      __syncthreads();
    }
    // adjoint of the output permutation
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) ga[__ldg(omap + i)] = ldc<IO>(gr + 2 * i);
    __syncthreads();
    for (int k = st.nstages - 1; k >= 0; --k) {
      const int f = st.f[k], L = st.L[k], rest = L / f;
      const float2* v = saved + (size_t)k * n;
      const float2* Wk = W + st.off[k];
      // w = conj(tw) * g, in place in ga
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t loc = i % L, a = loc / rest, q = loc % rest;
        ga[i] = cmulc(ga[i], __ldg(tw + (size_t)a * q * (n / L)));
      }
      __syncthreads();
      // G[a][p] += sum_{seg, q} w[a][q] conj(v[p][q]): entry e = (a, p) by
      // ns threads, each over every ns-th column, then a fixed-order sum
      {
        const int ff = f * f;
        const int ns = ff >= (int)blockDim.x ? 1 : (int)blockDim.x / ff;
        const uint32_t cols = n / f;  // (segment, q) pairs
        for (int t = threadIdx.x; t < ff * ns; t += blockDim.x) {
          const int e = t % ff, grp = t / ff, a = e / f, p = e % f;
          float2 acc = make_float2(0.f, 0.f);
          for (uint32_t cidx = grp; cidx < cols; cidx += ns) {
            const uint32_t off = (cidx / rest) * L + (cidx % rest);
            const float2 wv = ga[off + a * rest], vv = v[off + p * rest];
            acc.x = fmaf(wv.x, vv.x, fmaf(wv.y, vv.y, acc.x));
            acc.y = fmaf(wv.y, vv.x, fmaf(-wv.x, vv.y, acc.y));
          }
          if (ns == 1) G[st.off[k] + e] = cadd(G[st.off[k] + e], acc);
          else red[t] = acc;
        }
        if (ns > 1) {
          __syncthreads();
          for (int e = threadIdx.x; e < ff; e += blockDim.x) {
            float2 acc = G[st.off[k] + e];
            for (int grp = 0; grp < ns; ++grp) acc = cadd(acc, red[grp * ff + e]);
            G[st.off[k] + e] = acc;
          }
        }
      }
      // g' = W^H w
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t seg = i / L, loc = i % L, p = loc / rest, q = loc % rest;
        float2 acc = make_float2(0.f, 0.f);
        for (int a = 0; a < f; ++a) {
          const float2 w = Wk[a * f + p], x2 = ga[seg * L + a * rest + q];
          acc.x = fmaf(w.x, x2.x, fmaf(w.y, x2.y, acc.x));
          acc.y = fmaf(w.x, x2.y, fmaf(-w.y, x2.x, acc.y));
        }
        gb[i] = acc;
      }
      __syncthreads();
      float2* t = ga;
      ga = gb;
      gb = t;
    }
    IO* dr = dx + ((size_t)b * H + h) * 2 * n;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) stc<IO>(dr + 2 * i, ga[i]);
  }
  __syncthreads();
  float2* dg = gpart + ((size_t)blockIdx.y * H + h) * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) dg[i] = G[i];
}

__global__ void lb_reduce_kernel(const float2* __restrict__ gpart, float2* __restrict__ dblocks,
                                 int splits, size_t HP) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= HP) return;
  float2 acc = make_float2(0.f, 0.f);
  for (int sp = 0; sp < splits; ++sp) acc = cadd(acc, gpart[(size_t)sp * HP + i]);
  dblocks[i] = acc;
}

struct LbDevice {
  uint32_t* omap = nullptr;
  float2* tw = nullptr;
  LbStages st{};
};

}  // namespace fb

// The C-ABI plan carries the device tables through an opaque extension.
struct fb_learned_ext {
  fb::LbDevice dev;
};

namespace {

using namespace fb;

// Greedy factor chain of build_plan (butterfly.cpp:83-100).
int greedy_factors(int64_t n, int64_t r, std::vector<int64_t>& out) {
  int64_t seg = n;
  while (seg > 1) {
    int64_t f = 0;
    if (seg <= r) {
      f = seg;
    } else {
      for (int64_t d = std::min(seg, r); d >= 2; --d)
        if (seg % d == 0) {
          f = d;
          break;
        }
    }
    if (f == 0) return FB_ERR_PLAN;
    out.push_back(f);
    seg /= f;
  }
  return FB_OK;
}

// Composed output map (butterfly.cpp:103-116).
std::vector<uint32_t> output_map(int64_t n, const std::vector<int64_t>& f) {
  std::vector<uint32_t> m((size_t)n);
  for (int64_t i = 0; i < n; ++i) m[(size_t)i] = (uint32_t)i;
  int64_t L = n;
  for (size_t d = 0; d + 1 < f.size(); ++d) {
    const int64_t rest = L / f[d];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t off = (m[(size_t)i] / L) * L, local = m[(size_t)i] % L;
      const int64_t j2 = local / f[d], j1 = local % f[d];
      m[(size_t)i] = (uint32_t)(off + j1 * rest + j2);
    }
    L = rest;
  }
  return m;
}

fb_learned_ext* ext_of(const fb_learned_plan* p) {
  return static_cast<fb_learned_ext*>(p->ext);
}

}  // namespace

extern "C" {

int fb_learned_plan_create(fb_learned_plan** out, int64_t n, int64_t r, int64_t H, int dtype,
                           int device) {
  if (!out) {
    set_error("fb_learned_plan_create: null output");
    return FB_ERR_ARG;
  }
  *out = nullptr;
  if (n < 1 || H < 1) {
    set_error("learned: n and H must be >= 1");
    return FB_ERR_DIM;
  }
  if (r < 2) {
    set_error("build_plan: block size r must be >= 2");
    return FB_ERR_PLAN;
  }
  if (dtype < FB_F32 || dtype > FB_F16) {
    set_error("learned: bad dtype");
    return FB_ERR_ARG;
  }
  std::vector<int64_t> f;
  if (greedy_factors(n, r, f) != FB_OK) {
    set_error("build_plan: remainder has no factor <= r; pad the input to a power of two");
    return FB_ERR_PLAN;
  }
  if ((int)f.size() > kLbMaxStages - 1) {
    set_error("learned: too many stages");
    return FB_ERR_PLAN;
  }
  int rc = cuda_status(cudaSetDevice(device), "cudaSetDevice");
  if (rc) return rc;
  auto* p = new fb_learned_plan();
  p->n = n;
  p->r = r;
  p->H = H;
  p->dtype = dtype;
  p->device = device;
  p->nstages = (int)f.size();
  auto* ext = new fb_learned_ext();
  LbStages& st = ext->dev.st;
  st.nstages = (int)f.size();
  int64_t L = n, off = 0;
  for (size_t i = 0; i < f.size(); ++i) {
    p->factors[i] = f[i];
    st.f[i] = (int)f[i];
    st.L[i] = (int)L;
    st.off[i] = (int)off;
    off += f[i] * f[i];
    L /= f[i];
  }
  p->param_count = off;
  std::vector<uint32_t> om = output_map(n, f);
  std::vector<float2> tw((size_t)n);
  for (int64_t t = 0; t < n; ++t) {
    const double a = -2.0 * M_PI * (double)t / (double)n;
    tw[(size_t)t] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  rc = cuda_status(cudaMalloc(&ext->dev.omap, sizeof(uint32_t) * n), "cudaMalloc(omap)");
  if (!rc) rc = cuda_status(cudaMalloc(&ext->dev.tw, sizeof(float2) * n), "cudaMalloc(tw)");
  if (!rc)
    rc = cuda_status(cudaMemcpy(ext->dev.omap, om.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice),
                     "copy omap");
  if (!rc)
    rc = cuda_status(cudaMemcpy(ext->dev.tw, tw.data(), sizeof(float2) * n, cudaMemcpyHostToDevice),
                     "copy tw");
  p->ext = ext;
  if (rc) {
    fb_learned_plan_destroy(p);
    return rc;
  }
  *out = p;
  return FB_OK;
}

int fb_learned_plan_destroy(fb_learned_plan* p) {
  if (!p) return FB_OK;
  fb_learned_ext* ext = ext_of(p);
  if (ext) {
    cudaFree(ext->dev.omap);
    cudaFree(ext->dev.tw);
    delete ext;
  }
  delete p;
  return FB_OK;
}

int fb_learned_plan_factors(const fb_learned_plan* p, int64_t* factors, int64_t* count,
                            int64_t* param_count) {
  if (!p) {
    set_error("fb_learned_plan_factors: null plan");
    return FB_ERR_ARG;
  }
  if (count) *count = p->nstages;
  if (param_count) *param_count = p->param_count;
  if (factors)
    for (int i = 0; i < p->nstages; ++i) factors[i] = p->factors[i];
  return FB_OK;
}

// Row splits per head for the backward: enough CTAs to fill the SMs twice.
static int lb_splits(const fb_learned_plan* p, int64_t B) {
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, p->device);
  int64_t s = (2 * dev_sms + p->H - 1) / p->H;
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, B));
}

size_t fb_learned_workspace_size(const fb_learned_plan* p, int64_t B) {
  if (!p || B < 1) return 0;
  return (size_t)lb_splits(p, B) * p->H * p->param_count * sizeof(float2);
}

int fb_learned_fwd(fb_learned_plan* p, const float* blocks, const void* x, void* y, int64_t B,
                   void*, void* stream) {
  if (!p || !blocks || !x || !y) {
    set_error("fb_learned_fwd: null argument");
    return FB_ERR_ARG;
  }
  if (B < 1) {
    set_error("learned_forward: batch must be >= 1");
    return FB_ERR_DIM;
  }
  int rc = cuda_status(cudaSetDevice(p->device), "cudaSetDevice");
  if (rc) return rc;
  fb_learned_ext* ext = ext_of(p);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sm = (p->param_count + 2 * p->n) * sizeof(float2);
  const int rows = 4;
  const dim3 g((unsigned)p->H, (unsigned)((B + rows - 1) / rows));
  auto go = [&](auto io) {
    using IO = decltype(io);
    auto k = lb_fwd_kernel<IO>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<g, kLbThreads, sm, s>>>(blocks, (const IO*)x, (IO*)y, ext->dev.omap, ext->dev.tw,
                                ext->dev.st, (int)B, (int)p->H, (uint32_t)p->n,
                                (int)p->param_count, rows);
  };
  if (p->dtype == FB_F32) go(float{});
  else if (p->dtype == FB_BF16) go(__nv_bfloat16{});
  else go(__half{});
  return cuda_status(cudaGetLastError(), "fb_learned_fwd");
}

int fb_learned_bwd(fb_learned_plan* p, const float* blocks, const void* x, const void* g, void* dx,
                   float* dblocks, int64_t B, void* ws, void* stream) {
  if (!p || !blocks || !x || !g || !dx || !dblocks) {
    set_error("fb_learned_bwd: null argument");
    return FB_ERR_ARG;
  }
  if (B < 1) {
    set_error("learned_gradients: batch must be >= 1");
    return FB_ERR_DIM;
  }
  int rc = cuda_status(cudaSetDevice(p->device), "cudaSetDevice");
  if (rc) return rc;
  fb_learned_ext* ext = ext_of(p);
  cudaStream_t s = (cudaStream_t)stream;
  if (!ws) {
    set_error("fb_learned_bwd: workspace required (fb_learned_workspace_size)");
    return FB_ERR_ARG;
  }
  const int splits = lb_splits(p, B);
  const int rows = (int)((B + splits - 1) / splits);
  const size_t sm = (2 * p->param_count + kLbThreads + (p->nstages + 2) * p->n) * sizeof(float2);
  if (sm > 227 * 1024) {
    set_error("learned_gradients: row too long for the on-chip backward");
    return FB_ERR_UNSUPPORTED;
  }
  auto go = [&](auto io) {
    using IO = decltype(io);
    auto k = lb_bwd_kernel<IO>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<dim3((unsigned)p->H, (unsigned)splits), kLbThreads, sm, s>>>(
        blocks, (const IO*)x, (const IO*)g, (IO*)dx, (float2*)ws, ext->dev.omap, ext->dev.tw,
        ext->dev.st, (int)B, (int)p->H, (uint32_t)p->n, (int)p->param_count, rows);
  };
  if (p->dtype == FB_F32) go(float{});
  else if (p->dtype == FB_BF16) go(__nv_bfloat16{});
  else go(__half{});
  const size_t HP = (size_t)p->H * p->param_count;
  lb_reduce_kernel<<<(unsigned)((HP + 255) / 256), 256, 0, s>>>((const float2*)ws, (float2*)dblocks,
                                                               splits, HP);
  return cuda_status(cudaGetLastError(), "fb_learned_bwd");
}

}  // extern "C"
