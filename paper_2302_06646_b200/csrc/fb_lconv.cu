// FlashButterfly-B200: the learned-butterfly long convolution — the paper's
// extension (sCIFAR / WikiText usage :1210-1225) in which
// the Butterfly matrices of the FlashButterfly transform are learned instead
// of fixed to the FFT.  Per head h, with L(W, x) the reference's learned
// butterfly (learned_forward, butterfly.cpp:235-246: the build_plan(n, r)
// scaffolding with trainable per-stage blocks W) and IL(W, z) =
// conj(L(W, conj z)) / n its inverse counterpart:
//     y[b,h] = Re IL(W_i[h], L(W_f[h], pad u[b,h]) * L(W_f[h], pad Kbar[h]))[:N]
//              + D[h] u[b,h]
// n = 2N zero-padded (causal) or n = N (circular).  At W_f = W_i = the DFT
// blocks (LearnedButterfly::from_plan) this is exactly regularized_long_conv.
// The backward gives du, dKbar, dD and the block gradients dW_f, dW_i (exact
// adjoints through learned_gradients, butterfly.cpp:248-307).  Each real
// channel is its own complex row: the learned operator is complex-linear but
// not conjugate-symmetric, so two channels cannot share a transform.
//
// Composition of the K5 learned-butterfly kernels (fb_learned.cu) with fused
// elementwise kernels here; deterministic (fixed-order reductions).
#include <cuda_runtime.h>

#include <algorithm>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"

struct fb_lconv_plan {
  int64_t N = 0, H = 0, n = 0, r = 0;
  int mode = FB_MODE_CAUSAL, device = 0;
  fb_learned_plan* lp = nullptr;  // L(W, .) over rows of length n, per-head blocks, f32
  int64_t P = 0;                  // complex block parameters per head
};

namespace fb {
namespace {

unsigned nblk(int64_t count) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148 * 32));
}

// X[row][t] = scale * (t < N ? src[row][t] : 0) as complex (imag 0)
__global__ void lc_pad_kernel(const float* __restrict__ src, float2* __restrict__ X, int64_t rows, int64_t N,
                              int64_t n, float scale) {
  const int64_t count = rows * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, t = i % n;
    X[i] = make_float2(t < N ? scale * src[r * N + t] : 0.f, 0.f);
  }
}

// Zc[b,h] = conj(U[b,h] * Kf[h])  (the input of IL's forward learned pass)
__global__ void lc_mul_conj_kernel(const float2* __restrict__ U, const float2* __restrict__ Kf,
                                   float2* __restrict__ Zc, int64_t B, int64_t H, int64_t n) {
  const int64_t count = B * H * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i % n, h = (i / n) % H;
    const float2 z = cmul(U[i], Kf[h * n + t]);
    Zc[i] = make_float2(z.x, -z.y);
  }
}

// y[b][h][t] = Re V[b,h][t] / n + D[h] u[b][h][t]   (Re conj(V) = Re V)
__global__ void lc_out_kernel(const float2* __restrict__ V, const float* __restrict__ u,
                              const float* __restrict__ D, float* __restrict__ y, int64_t B, int64_t H,
                              int64_t N, int64_t n) {
  const int64_t count = B * H * N;
  const float inv_n = 1.0f / (float)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i % N, bh = i / N, h = bh % H;
    y[i] = V[bh * n + t].x * inv_n + __ldg(D + h) * u[i];
  }
}

// From gV = dx of IL's learned pass (the gradient w.r.t. conj Z):
//   gZ = conj(gV); gU = gZ conj(Kf) (in place over gV)
__global__ void lc_gu_kernel(float2* __restrict__ gV, const float2* __restrict__ Kf, int64_t B, int64_t H,
                             int64_t n) {
  const int64_t count = B * H * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i % n, h = (i / n) % H;
    const float2 g = gV[i], k = Kf[h * n + t];
    const float2 gz = make_float2(g.x, -g.y);
    gV[i] = cmulc(gz, k);
  }
}

// gKf[h][t] = sum_b gZ[b,h][t] conj(U[b,h][t])  (b in order: deterministic), gZ = conj(gV)
__global__ void lc_gk_kernel(const float2* __restrict__ gV, const float2* __restrict__ U,
                             float2* __restrict__ gKf, int64_t B, int64_t H, int64_t n) {
  const int64_t count = H * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float2 acc = make_float2(0.f, 0.f);
    for (int64_t b = 0; b < B; ++b) {
      const float2 g = gV[b * count + i];
      acc = cadd(acc, cmulc(make_float2(g.x, -g.y), U[b * count + i]));
    }
    gKf[i] = acc;
  }
}

// du[b][h][t] = Re dX[b,h][t] + D[h] dy ; dKbar[h][t] = Re dXk[h][t]; dD[h] = sum dy u
__global__ void lc_du_kernel(const float2* __restrict__ dX, const float* __restrict__ dy,
                             const float* __restrict__ D, float* __restrict__ du, int64_t B, int64_t H,
                             int64_t N, int64_t n) {
  const int64_t count = B * H * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i % N, bh = i / N, h = bh % H;
    du[i] = dX[bh * n + t].x + __ldg(D + h) * dy[i];
  }
}
__global__ void lc_dk_kernel(const float2* __restrict__ dXk, float* __restrict__ dk, int64_t H, int64_t N,
                             int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < H * N;
       i += (int64_t)gridDim.x * blockDim.x)
    dk[i] = dXk[(i / N) * n + i % N].x;
}
// dD[h] = sum_{b,t} dy u, one CTA per head, fixed-order tree
__global__ void lc_dd_kernel(const float* __restrict__ dy, const float* __restrict__ u, float* __restrict__ dD,
                             int64_t B, int64_t H, int64_t N) {
  __shared__ float red[256];
  const int64_t h = blockIdx.x;
  float acc = 0.f;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t t = threadIdx.x; t < N; t += blockDim.x) {
      const int64_t i = (b * H + h) * N + t;
      acc = fmaf(dy[i], u[i], acc);
    }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) dD[h] = red[0];
}
__global__ void lc_add_kernel(float* __restrict__ a, const float* __restrict__ b, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] += b[i];
}

// workspace carve-up: row buffers of n complex
struct LcWs {
  float2 *X, *U, *Kp, *Kf, *Zc, *V, *G, *lw;
  float* dWtmp;
};
size_t lc_ws_bytes(const fb_lconv_plan* p, int64_t B, LcWs* w, void* base) {
  const int64_t R = B * p->H, n = p->n;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t oX = take(sizeof(float2) * R * n), oU = take(sizeof(float2) * R * n),
               oKp = take(sizeof(float2) * p->H * n), oKf = take(sizeof(float2) * p->H * n),
               oZ = take(sizeof(float2) * R * n), oV = take(sizeof(float2) * R * n),
               oG = take(sizeof(float2) * R * n), oW = take(sizeof(float2) * p->H * p->P),
               oL = take(std::max(fb_learned_workspace_size(p->lp, B), fb_learned_workspace_size(p->lp, 1)));
  if (w) {
    char* c = (char*)base;
    w->X = (float2*)(c + oX);
    w->U = (float2*)(c + oU);
    w->Kp = (float2*)(c + oKp);
    w->Kf = (float2*)(c + oKf);
    w->Zc = (float2*)(c + oZ);
    w->V = (float2*)(c + oV);
    w->G = (float2*)(c + oG);
    w->dWtmp = (float*)(c + oW);
    w->lw = (float2*)(c + oL);
  }
  return off;
}

// the forward's shared front: X = pad u, U = L(W_f, X), Kp = pad Kbar,
// Kf = L(W_f, Kp), Zc = conj(U Kf)
int lc_front(fb_lconv_plan* p, const float* u, const float* kbar, const float* Wf, int64_t B, LcWs& w,
             cudaStream_t s) {
  const int64_t R = B * p->H, n = p->n;
  lc_pad_kernel<<<nblk(R * n), 256, 0, s>>>(u, w.X, R, p->N, n, 1.f);
  int rc = fb_learned_fwd(p->lp, Wf, w.X, w.U, B, nullptr, s);
  if (rc) return rc;
  lc_pad_kernel<<<nblk(p->H * n), 256, 0, s>>>(kbar, w.Kp, p->H, p->N, n, 1.f);
  rc = fb_learned_fwd(p->lp, Wf, w.Kp, w.Kf, 1, nullptr, s);
  if (rc) return rc;
  lc_mul_conj_kernel<<<nblk(R * n), 256, 0, s>>>(w.U, w.Kf, w.Zc, B, p->H, n);
  return cuda_status(cudaGetLastError(), "learned conv front");
}

}  // namespace
}  // namespace fb

using namespace fb;

extern "C" {

int fb_lconv_plan_create(fb_lconv_plan** out, int64_t N, int64_t H, int64_t r, int mode, int device) {
  if (!out) {
    set_error("fb_lconv_plan_create: null output");
    return FB_ERR_ARG;
  }
  *out = nullptr;
  if (N < 1 || H < 1) {
    set_error("learned conv: N and H must be >= 1");
    return FB_ERR_DIM;
  }
  if (mode != FB_MODE_CAUSAL && mode != FB_MODE_CIRCULAR) {
    set_error("learned conv: bad mode");
    return FB_ERR_ARG;
  }
  auto* p = new fb_lconv_plan();
  p->N = N;
  p->H = H;
  p->r = r;
  p->mode = mode;
  p->device = device;
  p->n = mode == FB_MODE_CAUSAL ? 2 * N : N;
  int rc = fb_learned_plan_create(&p->lp, p->n, r, H, FB_F32, device);
  if (!rc) rc = fb_learned_plan_factors(p->lp, nullptr, nullptr, &p->P);
  if (rc) {
    fb_lconv_plan_destroy(p);
    return rc;
  }
  *out = p;
  return FB_OK;
}

int fb_lconv_plan_destroy(fb_lconv_plan* p) {
  if (!p) return FB_OK;
  fb_learned_plan_destroy(p->lp);
  delete p;
  return FB_OK;
}

int fb_lconv_plan_dims(const fb_lconv_plan* p, int64_t* n, int64_t* param_count) {
  if (!p) {
    set_error("fb_lconv_plan_dims: null plan");
    return FB_ERR_ARG;
  }
  if (n) *n = p->n;
  if (param_count) *param_count = p->P;
  return FB_OK;
}

size_t fb_lconv_workspace_size(const fb_lconv_plan* p, int64_t B) {
  if (!p || B < 1) return 0;
  return lc_ws_bytes(p, B, nullptr, nullptr) + 256;
}

int fb_lconv_fwd(fb_lconv_plan* p, const float* u, const float* kbar, const float* D, const float* Wf,
                 const float* Wi, float* y, int64_t B, void* ws, void* stream) {
  if (!p || !u || !kbar || !D || !Wf || !Wi || !y || !ws) {
    set_error("fb_lconv_fwd: null argument");
    return FB_ERR_ARG;
  }
  if (B < 1) {
    set_error("learned conv: batch must be >= 1");
    return FB_ERR_DIM;
  }
  DevGuard dg_(p->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  LcWs w;
  lc_ws_bytes(p, B, &w, ws);
  if ((rc = lc_front(p, u, kbar, Wf, B, w, s))) return rc;
  if ((rc = fb_learned_fwd(p->lp, Wi, w.Zc, w.V, B, nullptr, s))) return rc;
  lc_out_kernel<<<nblk(B * p->H * p->N), 256, 0, s>>>(w.V, u, D, y, B, p->H, p->N, p->n);
  return cuda_status(cudaGetLastError(), "fb_lconv_fwd");
}

int fb_lconv_bwd(fb_lconv_plan* p, const float* dy, const float* u, const float* kbar, const float* D,
                 const float* Wf, const float* Wi, float* du, float* dkbar, float* dD, float* dWf, float* dWi,
                 int64_t B, void* ws, void* stream) {
  if (!p || !dy || !u || !kbar || !D || !Wf || !Wi || !du || !dkbar || !dD || !dWf || !dWi || !ws) {
    set_error("fb_lconv_bwd: null argument");
    return FB_ERR_ARG;
  }
  if (B < 1) {
    set_error("learned conv: batch must be >= 1");
    return FB_ERR_DIM;
  }
  DevGuard dg_(p->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t R = B * p->H, n = p->n;
  LcWs w;
  lc_ws_bytes(p, B, &w, ws);
  if ((rc = lc_front(p, u, kbar, Wf, B, w, s))) return rc;  // recompute U, Kf, Zc
  // J = sum dy Re(conj(V)/n)[:N]  =>  upstream of V (w.r.t. Re<., V>) = pad(dy) / n
  lc_pad_kernel<<<nblk(R * n), 256, 0, s>>>(dy, w.X, R, p->N, n, 1.0f / (float)n);
  if ((rc = fb_learned_bwd(p->lp, Wi, w.Zc, w.X, w.G, dWi, B, w.lw, s))) return rc;  // G = d/d conj(Z)
  lc_gk_kernel<<<nblk(p->H * n), 256, 0, s>>>(w.G, w.U, w.Kp, B, p->H, n);          // Kp <- gKf
  lc_gu_kernel<<<nblk(R * n), 256, 0, s>>>(w.G, w.Kf, B, p->H, n);                  // G <- gU
  // X <- pad u again (the learned backward's input), V <- dX
  lc_pad_kernel<<<nblk(R * n), 256, 0, s>>>(u, w.X, R, p->N, n, 1.f);
  if ((rc = fb_learned_bwd(p->lp, Wf, w.X, w.G, w.V, dWf, B, w.lw, s))) return rc;
  // Kf <- pad Kbar, Zc <- dXk (the Kf branch of W_f's gradient)
  lc_pad_kernel<<<nblk(p->H * n), 256, 0, s>>>(kbar, w.Kf, p->H, p->N, n, 1.f);
  if ((rc = fb_learned_bwd(p->lp, Wf, w.Kf, w.Kp, w.Zc, w.dWtmp, 1, w.lw, s))) return rc;
  lc_add_kernel<<<nblk(2 * p->H * p->P), 256, 0, s>>>(dWf, w.dWtmp, 2 * p->H * p->P);
  lc_du_kernel<<<nblk(R * p->N), 256, 0, s>>>(w.V, dy, D, du, B, p->H, p->N, n);
  lc_dk_kernel<<<nblk(p->H * p->N), 256, 0, s>>>(w.Zc, dkbar, p->H, p->N, n);
  lc_dd_kernel<<<(unsigned)p->H, 256, 0, s>>>(dy, u, dD, B, p->H, p->N);
  return cuda_status(cudaGetLastError(), "fb_lconv_bwd");
}

}  // extern "C"
