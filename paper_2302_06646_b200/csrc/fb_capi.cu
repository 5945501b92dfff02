// FlashButterfly-B200 C ABI (include/flashbutterfly.h): plan lifetime, engine
// resolution, argument checking and dispatch.  No CPU compute path exists:
// every entry point either launches sm_100a kernels or returns an error.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fb_internal.h"

namespace fb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FB_OK;
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return FB_ERR_CUDA;
}

static int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

static bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
static int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Host-side twiddle table exp(-2 pi i t / n), computed in fp64 then rounded.
static int upload_twiddles(float2** dst, int64_t n) {
  std::vector<float2> h((size_t)n);
  for (int64_t t = 0; t < n; ++t) {
    const double a = -2.0 * M_PI * (double)t / (double)n;
    h[(size_t)t] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  int rc = cuda_status(cudaMalloc(dst, sizeof(float2) * n), "cudaMalloc(twiddles)");
  if (rc) return rc;
  return cuda_status(cudaMemcpy(*dst, h.data(), sizeof(float2) * n, cudaMemcpyHostToDevice),
                     "cudaMemcpy(twiddles)");
}

// Two-level table [w^i (i < 64) | w^(64 i) (i < n/64)], w = exp(-2 pi i / n).
static int upload_twiddles2(float2** dst, int64_t n) {
  const int64_t lo = 64, hi = n / 64 > 0 ? n / 64 : 1;
  std::vector<float2> h((size_t)(lo + hi));
  for (int64_t t = 0; t < lo; ++t) {
    const double a = -2.0 * M_PI * (double)t / (double)n;
    h[(size_t)t] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  for (int64_t i = 0; i < hi; ++i) {
    const double a = -2.0 * M_PI * (double)(64 * i) / (double)n;
    h[(size_t)(lo + i)] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  int rc = cuda_status(cudaMalloc(dst, sizeof(float2) * h.size()), "cudaMalloc(twiddles2)");
  if (rc) return rc;
  return cuda_status(cudaMemcpy(*dst, h.data(), sizeof(float2) * h.size(), cudaMemcpyHostToDevice),
                     "cudaMemcpy(twiddles2)");
}

// [w^t (t < 4096) | w^(4096 i) (i < n/4096)], w = exp(-2 pi i / n)
static int upload_twiddles_big(float2** dst, int64_t n) {
  const int64_t hi = std::max<int64_t>(1, n / 4096);
  std::vector<float2> h((size_t)(4096 + hi));
  for (int64_t t = 0; t < 4096; ++t) {
    const double a = -2.0 * M_PI * (double)t / (double)n;
    h[(size_t)t] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  for (int64_t i = 0; i < hi; ++i) {
    const double a = -2.0 * M_PI * (double)(4096 * i) / (double)n;
    h[(size_t)(4096 + i)] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  int rc = cuda_status(cudaMalloc(dst, sizeof(float2) * h.size()), "cudaMalloc(twiddles big)");
  if (rc) return rc;
  return cuda_status(cudaMemcpy(*dst, h.data(), sizeof(float2) * h.size(), cudaMemcpyHostToDevice),
                     "cudaMemcpy(twiddles big)");
}

// kind 0: full table, 1: two-level (64), 2: two-level (4096) — shared with
// the sequence-sharded plan in fb_three.cu
int upload_table(float2** dst, int64_t n, int kind) {
  return kind == 0 ? upload_twiddles(dst, n) : kind == 1 ? upload_twiddles2(dst, n)
                                                         : upload_twiddles_big(dst, n);
}

constexpr int64_t kSinglePassMax = 8192;   // fp32 complex transform in smem
constexpr int64_t kThreePassRow = 8192;    // l: row length of pass 2
constexpr int64_t kMinTransform = 256;

}  // namespace fb

using namespace fb;

namespace fb {
// ---- zero-padded staging for causal three-pass plans with N % l != 0 ----
// rows of `w` bytes with pitch `sp` -> rows of pitch `dp`, the tail of each
// destination row (dp - w bytes) zeroed
// 16-byte row copy: dst[r][j] = j < w16 ? src[r][j] : 0 for j < dw16 (one
// streaming pass at HBM rate; the 2-D copy engine path ran at a fraction)
__global__ void row_copy_kernel(uint4* __restrict__ dst, size_t dp16, const uint4* __restrict__ src,
                                size_t sp16, size_t w16, size_t dw16) {
  const size_t r = blockIdx.y;
  const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < dw16) dst[r * dp16 + j] = j < w16 ? __ldg(src + r * sp16 + j) : make_uint4(0, 0, 0, 0);
}
static bool row_copy(void* dst, size_t dp, const void* src, size_t sp, size_t w, size_t dw,
                     size_t rows, cudaStream_t s) {
  const bool ok = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | dp | sp | w |
                    dw) & 15) == 0 && rows > 0 && rows <= 65535;
  if (!ok) return false;
  const dim3 g((unsigned)((dw / 16 + 255) / 256), (unsigned)rows);
  row_copy_kernel<<<g, 256, 0, s>>>((uint4*)dst, dp / 16, (const uint4*)src, sp / 16, w / 16, dw / 16);
  return true;
}
static int pad_rows(void* dst, size_t dp, const void* src, size_t sp, size_t w, size_t rows,
                    cudaStream_t s) {
  if (row_copy(dst, dp, src, sp, w, dp, rows, s)) return cuda_status(cudaGetLastError(), "pad copy");
  int rc = cuda_status(cudaMemcpy2DAsync(dst, dp, src, sp, w, rows, cudaMemcpyDeviceToDevice, s),
                       "pad copy");
  if (!rc && dp > w) rc = cuda_status(cudaMemset2DAsync((char*)dst + w, dp, 0, dp - w, rows, s),
                                      "pad zero");
  return rc;
}
static int crop_rows(void* dst, size_t dp, const void* src, size_t sp, size_t w, size_t rows,
                     cudaStream_t s) {
  if (row_copy(dst, dp, src, sp, w, w, rows, s)) return cuda_status(cudaGetLastError(), "crop copy");
  return cuda_status(cudaMemcpy2DAsync(dst, dp, src, sp, w, rows, cudaMemcpyDeviceToDevice, s),
                     "crop copy");
}
static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
static size_t es_of(int dtype) { return dtype == FB_F32 ? 4 : 2; }

// workspace of a padded plan: [inner workspace | u' | v' | w' | dK' | dKbar']
struct PadWs {
  char *inner, *a, *b, *c;
  float *dk, *dkbar;
};
static size_t pad_ws_bytes(const fb_plan* p, int64_t B, PadWs* w, void* base) {
  const fb_plan* q = p->inner;
  const size_t sig = al256((size_t)B * q->H * q->N * es_of(q->dtype));
  const size_t bank = al256((size_t)q->H * q->N * sizeof(float));
  const size_t inner = al256(tp_workspace(q, B));
  if (w) {
    char* c = (char*)base;
    w->inner = c;
    w->a = c + inner;
    w->b = w->a + sig;
    w->c = w->b + sig;
    w->dk = (float*)(w->c + sig);
    w->dkbar = (float*)((char*)w->dk + bank);
  }
  return inner + 3 * sig + 2 * bank + 256;
}
}  // namespace fb

extern "C" {

const char* fb_last_error(void) { return g_last_error.c_str(); }
int fb_version(void) { return FB_VERSION; }

int fb_plan_create(fb_plan** out, int64_t N, int64_t H, int mode, int dtype, int engine,
                   int device) {
  if (!out) return fail(FB_ERR_ARG, "fb_plan_create: null output pointer");
  *out = nullptr;
  if (N < 1 || H < 1) return fail(FB_ERR_DIM, "fb_plan_create: N and H must be >= 1");
  if (mode != FB_MODE_CAUSAL && mode != FB_MODE_CIRCULAR)
    return fail(FB_ERR_ARG, "fb_plan_create: bad mode");
  if (dtype < FB_F32 || dtype > FB_F16) return fail(FB_ERR_ARG, "fb_plan_create: bad dtype");
  if (engine < FB_ENGINE_AUTO || engine > FB_ENGINE_SINGLE_SIMT)
    return fail(FB_ERR_ARG, "fb_plan_create: bad engine");
  if (mode == FB_MODE_CIRCULAR && !is_pow2(N))
    return fail(FB_ERR_PLAN, "fb_plan_create: circular mode needs a power-of-two N "
                             "(causal mode accepts any N; pad the input)");
  DevGuard dg(device);
  int rc = cuda_status(dg.err, "cudaSetDevice");
  if (rc) return rc;
  fb_plan* p = new fb_plan();
  p->N = N;
  p->H = H;
  p->mode = mode;
  p->dtype = dtype;
  p->device = device;
  int64_t n = mode == FB_MODE_CAUSAL ? next_pow2(2 * N) : N;
  if (n < kMinTransform) n = kMinTransform;
  // the tensor-core single pass also serves N = 2048 on its n = 8192 transform
  const bool tc_pad = mode == FB_MODE_CAUSAL && N == 2048 && dtype != FB_F32 &&
                      (engine == FB_ENGINE_AUTO || engine == FB_ENGINE_SINGLE) && tc_length_ok(N) &&
                      !(std::getenv("FB_TC2") && std::getenv("FB_TC2")[0] == '1');
  if (tc_pad) n = 8192;
  p->n = n;
  p->periodic = (mode == FB_MODE_CIRCULAR) && n > N;
  const bool simt = engine == FB_ENGINE_SINGLE_SIMT;
  if (simt) engine = FB_ENGINE_SINGLE;
  if (engine == FB_ENGINE_AUTO) engine = n <= kSinglePassMax ? FB_ENGINE_SINGLE : FB_ENGINE_THREE;
  if (engine == FB_ENGINE_SINGLE && n > kSinglePassMax) {
    delete p;
    return fail(FB_ERR_PLAN, "fb_plan_create: single-pass engine supports transforms up to " +
                                 std::to_string(kSinglePassMax) + " points; use three-pass");
  }
  if (engine == FB_ENGINE_THREE && (n < 2 * kThreePassRow || n > 1024 * kThreePassRow)) {
    delete p;
    return fail(FB_ERR_PLAN, "fb_plan_create: three-pass engine needs a transform of " +
                                 std::to_string(2 * kThreePassRow) + ".." +
                                 std::to_string(1024 * kThreePassRow) + " points (l = " +
                                 std::to_string(kThreePassRow) + ", m = 2..1024)");
  }
  p->engine = engine;
  if (engine == FB_ENGINE_THREE) {
    p->l = kThreePassRow;
    p->m = n / p->l;
  } else {
    p->l = n;
    p->m = 1;
  }
  if (engine == FB_ENGINE_THREE && mode == FB_MODE_CAUSAL && N % kThreePassRow) {
    // the column passes tile the data rows c < N / l; pad N to whole rows
    // (same transform length: N' <= n / 2) and crop the outputs
    const int64_t Np = (N + kThreePassRow - 1) / kThreePassRow * kThreePassRow;
    rc = fb_plan_create(&p->inner, Np, H, mode, dtype, FB_ENGINE_THREE, device);
    if (!rc) rc = cuda_status(cudaMalloc(&p->kraw, sizeof(float) * H * Np), "cudaMalloc(K pad)");
    if (rc) {
      fb_plan_destroy(p);
      return rc;
    }
    *out = p;
    return FB_OK;
  }
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);
  p->use_tc = engine == FB_ENGINE_SINGLE && !simt && tc_eligible(p);
  {  // experiment switch: FB_TC2=1 selects the 128 x 64 TMEM-resident design
     // (fb_tc2.cu; measured slower end to end than the 64 x 128 default)
    const char* e = std::getenv("FB_TC2");
    p->tc_ver = (e && e[0] == '1') ? 2 : 1;
  }
  rc = upload_twiddles2(&p->tw2, n);
  if (!rc && engine == FB_ENGINE_THREE && p->m <= 16) rc = upload_twiddles(&p->tw_n, n);
  if (!rc && engine == FB_ENGINE_THREE) rc = upload_twiddles2(&p->tw_l, p->l);
  if (!rc && engine == FB_ENGINE_THREE && p->m > 16) rc = upload_twiddles(&p->tw_m, p->m);
  if (!rc && engine == FB_ENGINE_THREE && p->m > 16) rc = upload_twiddles_big(&p->tw_big, n);
  if (!rc) rc = cuda_status(cudaMalloc(&p->kf, sizeof(float2) * H * n), "cudaMalloc(kf)");
  if (!rc) rc = cuda_status(cudaMalloc(&p->kbar, sizeof(float) * H * N), "cudaMalloc(kbar)");
  if (!rc) rc = cuda_status(cudaMalloc(&p->d, sizeof(float) * H), "cudaMalloc(D)");
  if (!rc && p->use_tc) rc = tc_init(p);
  if (!rc && engine == FB_ENGINE_SINGLE && !simt && !p->use_tc && sc_config(p, &p->sc_stc, &p->sc_lgfl)) {
    p->use_sc = true;
    rc = sc_init(p);
  }
  if (!rc && p->engine == FB_ENGINE_THREE) {
    rc = cuda_status(cudaMalloc(&p->kraw, sizeof(float) * H * N), "cudaMalloc(K copy)");
    if (!rc) rc = cuda_status(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking), "aux stream");
    for (cudaEvent_t* e : {&p->ev_fork, &p->ev_prep, &p->ev_join})
      if (!rc) rc = cuda_status(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
  }
  if (rc) {
    fb_plan_destroy(p);
    return rc;
  }
  *out = p;
  return FB_OK;
}

int fb_plan_destroy(fb_plan* p) {
  if (!p) return FB_OK;
  DevGuard dg(p->device);
  if (p->inner) fb_plan_destroy(p->inner);
  cudaFree(p->tw_n);
  cudaFree(p->tw2);
  cudaFree(p->tw_l);
  cudaFree(p->tw_m);
  cudaFree(p->tw_big);
  cudaFree(p->kf);
  cudaFree(p->kbar);
  cudaFree(p->keep);
  cudaFree(p->d);
  cudaFree(p->kraw);
  cudaFree(p->tc_mats);
  cudaFree(p->kf_tc);
  cudaFree(p->tcr_mats);
  cudaFree(p->kf_scale);
  cudaFree(p->sc_blocks);
  cudaFree(p->sc_tw);
  if (p->aux) cudaStreamSynchronize(p->aux);
  for (cudaEvent_t e : {p->ev_fork, p->ev_prep, p->ev_join})
    if (e) cudaEventDestroy(e);
  if (p->aux) cudaStreamDestroy(p->aux);
  delete p;
  return FB_OK;
}

int fb_plan_get_info(const fb_plan* p, fb_plan_info* info) {
  if (!p || !info) return fail(FB_ERR_ARG, "fb_plan_get_info: null argument");
  const fb_plan* q = p->inner ? p->inner : p;
  info->N = p->N;
  info->H = p->H;
  info->n = q->n;
  info->l = q->l;
  info->m = q->m;
  info->engine = q->engine;
  info->dtype = q->dtype;
  info->mode = q->mode;
  info->tensor_cores = (q->use_tc || q->use_sc) ? 1 : 0;
  return FB_OK;
}

int fb_plan_copy_kbar(const fb_plan* p, float* dst, void* stream) {
  if (!p || !dst) return fail(FB_ERR_ARG, "fb_plan_copy_kbar: null argument");
  DevGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (p->inner) {
    int rc = prep_wait(p->inner, s);
    if (rc) return rc;
    return crop_rows(dst, p->N * sizeof(float), p->inner->kbar, p->inner->N * sizeof(float),
                     p->N * sizeof(float), p->H, s);
  }
  int rc = prep_wait(p, s);
  if (rc) return rc;
  return cuda_status(cudaMemcpyAsync(dst, p->kbar, sizeof(float) * p->H * p->N,
                                     cudaMemcpyDeviceToDevice, s),
                     "fb_plan_copy_kbar");
}

int fb_init_kernels(int kind, int64_t H, int64_t N, uint64_t seed, float* K, float* D, double* K64,
                    double* D64, int device, void* stream) {
  if (H < 1 || N < 1) return fail(FB_ERR_DIM, "init_kernels: heads and len must be >= 1");
  if (kind != FB_INIT_RANDOM && kind != FB_INIT_GEOMETRIC) return fail(FB_ERR_ARG, "init_kernels: bad kind");
  DevGuard dg(device);
  int rc = cuda_status(dg.err, "cudaSetDevice");
  if (rc) return rc;
  return init_kernels_dev(kind, H, N, seed, K, D, K64, D64, device, (cudaStream_t)stream);
}

int fb_kernel_prep(fb_plan* p, const float* K, const float* D, const fb_reg_config* cfg,
                   int training, void* stream) {
  if (!p || !K || !D || !cfg) return fail(FB_ERR_ARG, "fb_kernel_prep: null argument");
  if (cfg->lambda < 0.0) return fail(FB_ERR_DIM, "squash: lambda must be >= 0");
  if (cfg->dropout_rate < 0.0 || cfg->dropout_rate >= 1.0)
    return fail(FB_ERR_DIM, "kernel_dropout: rate must be in [0, 1)");
  if (cfg->smooth_width < 0) return fail(FB_ERR_DIM, "smooth: width must be >= 0");
  if (cfg->smooth_domain != FB_SMOOTH_TIME && cfg->smooth_domain != FB_SMOOTH_FREQUENCY)
    return fail(FB_ERR_ARG, "fb_kernel_prep: bad smooth domain");
  cudaStream_t s = (cudaStream_t)stream;
  DevGuard dg(p->device);
  int rc = cuda_status(dg.err, "cudaSetDevice");
  if (rc) return rc;
  if (p->inner) {
    // zero-padded kernels: smooth's zero padding beyond N and causal taps >= N
    // never reach outputs t < N, so y, du, dK[:N] equal the unpadded ones
    // (the frequency-domain smooth transforms the whole length: not padded)
    if (cfg->smooth_domain == FB_SMOOTH_FREQUENCY)
      return fail(FB_ERR_UNSUPPORTED, "fb_kernel_prep: smooth_frequency needs N divisible by " +
                                          std::to_string(kThreePassRow) + " on three-pass");
    fb_plan* q = p->inner;
    q->head0 = p->head0;
    if ((rc = prep_wait(q, s))) return rc;  // the previous prep still reads kraw
    rc = pad_rows(p->kraw, q->N * sizeof(float), K, p->N * sizeof(float), p->N * sizeof(float),
                  p->H, s);
    if (!rc) rc = fb_kernel_prep(q, p->kraw, D, cfg, training, stream);
    if (!rc) p->prepared = true;
    return rc;
  }
  // three-pass: the prep chain runs on the plan's auxiliary stream (after
  // everything already queued on s), so the next forward's pass 1 overlaps it;
  // consumers of the plan state wait on ev_prep.  Not while s is capturing.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const bool async = p->aux && cap == cudaStreamCaptureStatusNone;
  if (p->prep_async) {  // the previous prep must be done before its state is rewritten
    if ((rc = prep_wait(p, s))) return rc;
    p->prep_async = false;
  }
  // K and D are copied on the caller's stream, so the caller may overwrite
  // them as soon as this call returns (stream order), even when the rest of
  // the prep runs on the auxiliary stream
  rc = cuda_status(cudaMemcpyAsync(p->d, D, sizeof(float) * p->H, cudaMemcpyDeviceToDevice, s),
                   "copy D");
  if (rc) return rc;
  const float* Kin = K;
  if (p->kraw && K != p->kraw) {
    rc = cuda_status(cudaMemcpyAsync(p->kraw, K, sizeof(float) * p->H * p->N,
                                     cudaMemcpyDeviceToDevice, s), "copy K");
    if (rc) return rc;
    Kin = p->kraw;
  }
  cudaStream_t ps = s;
  if (async) {
    rc = cuda_status(cudaEventRecord(p->ev_fork, s), "fork");
    if (!rc) rc = cuda_status(cudaStreamWaitEvent(p->aux, p->ev_fork, 0), "fork wait");
    if (rc) return rc;
    ps = p->aux;
  }
  p->lambda = cfg->lambda;
  p->p = cfg->smooth_width;
  p->smooth_domain = cfg->smooth_domain;
  p->use_keep = training && cfg->dropout_rate > 0.0;
  p->keep_scale = 1.0 / (1.0 - cfg->dropout_rate);
  if (p->use_keep) {
    if (!p->keep) {
      rc = cuda_status(cudaMalloc(&p->keep, (size_t)p->H * p->N), "cudaMalloc(keep)");
      if (rc) return rc;
    }
    rc = dropout_keep_dev(p, cfg->dropout_rate, cfg->seed, ps);
    if (rc) return rc;
  }
  rc = p->engine == FB_ENGINE_SINGLE ? sp_prep(p, Kin, ps) : tp_prep(p, Kin, ps);
  if (rc) return rc;
  if (async) {
    rc = cuda_status(cudaEventRecord(p->ev_prep, p->aux), "prep event");
    if (rc) return rc;
    p->prep_async = true;
  }
  p->prepared = true;
  return FB_OK;
}

size_t fb_workspace_size(const fb_plan* p, int64_t B) {
  if (!p || B < 1) return 0;
  if (p->inner) return pad_ws_bytes(p, B, nullptr, nullptr);
  return p->engine == FB_ENGINE_SINGLE ? sp_workspace(p, B) : tp_workspace(p, B);
}

static int check_run(const fb_plan* p, int64_t B, const char* who) {
  if (!p) return fail(FB_ERR_ARG, std::string(who) + ": null plan");
  if (!p->prepared) return fail(FB_ERR_ARG, std::string(who) + ": call fb_kernel_prep first");
  if (B < 1) return fail(FB_ERR_DIM, std::string(who) + ": batch must be >= 1");
  if (B > 65535 * 2) return fail(FB_ERR_DIM, std::string(who) + ": batch too large");
  return FB_OK;
}

int fb_plan_profile_events(fb_plan* p, int which, void* begin, void* end) {
  if (!p) return fail(FB_ERR_ARG, "fb_plan_profile_events: null plan");
  if (which != 0 && which != 1) return fail(FB_ERR_ARG, "fb_plan_profile_events: which must be 0 or 1");
  if (p->inner) return fb_plan_profile_events(p->inner, which, begin, end);
  p->prof[which][0] = (cudaEvent_t)begin;
  p->prof[which][1] = (cudaEvent_t)end;
  return FB_OK;
}

size_t fb_saved_size(const fb_plan* p, int64_t B) {
  if (!p || B < 1) return 0;
  if (p->inner) return fb_saved_size(p->inner, B);
  if (p->use_tc) return tc_saved_size(p, B);
  // three-pass: the saved row spectra are kept in the intermediate precision,
  // which for fp16 on the CUDA-core rows cannot hold FFT_l of a long
  // non-zero-mean row (|U[0]| = l |mean| overflows 65504): those plans
  // recompute U in the backward; fp16 on the tcgen05 rows keeps bf16 rows
  if (p->engine == FB_ENGINE_THREE && !p->periodic && (p->dtype != FB_F16 || tp_uses_tc_rows(p)))
    return tp_saved_size(p, B);
  return 0;
}

// forward of a padded plan: u -> u' (zero-padded rows), inner forward, y' -> y
static int pad_fwd(fb_plan* p, const void* u, void* y, void* saved, int64_t B, void* ws,
                   cudaStream_t s) {
  fb_plan* q = p->inner;
  PadWs w;
  pad_ws_bytes(p, B, &w, ws);
  const size_t es = es_of(p->dtype), rows = (size_t)B * p->H;
  int rc = pad_rows(w.a, q->N * es, u, p->N * es, p->N * es, rows, s);
  if (!rc) rc = saved ? fb_fwd_save(q, w.a, w.b, saved, B, w.inner, s)
                      : fb_fwd(q, w.a, w.b, B, w.inner, s);
  if (!rc) rc = crop_rows(y, p->N * es, w.b, q->N * es, p->N * es, rows, s);
  return rc;
}

static int pad_bwd(fb_plan* p, const void* dy, const void* u, const void* saved, void* du,
                   float* dK, float* dKbar, float* dD, int64_t B, void* ws, cudaStream_t s) {
  fb_plan* q = p->inner;
  PadWs w;
  pad_ws_bytes(p, B, &w, ws);
  const size_t es = es_of(p->dtype), rows = (size_t)B * p->H;
  int rc = pad_rows(w.a, q->N * es, dy, p->N * es, p->N * es, rows, s);
  if (!rc && u) rc = pad_rows(w.b, q->N * es, u, p->N * es, p->N * es, rows, s);
  if (!rc) rc = saved ? fb_bwd_saved(q, w.a, u ? w.b : nullptr, saved, w.c, w.dk,
                                     dKbar ? w.dkbar : nullptr, dD, B, w.inner, s)
                      : fb_bwd(q, w.a, w.b, w.c, w.dk, dKbar ? w.dkbar : nullptr, dD, B, w.inner, s);
  if (!rc) rc = crop_rows(du, p->N * es, w.c, q->N * es, p->N * es, rows, s);
  const size_t f = sizeof(float);
  if (!rc) rc = crop_rows(dK, p->N * f, w.dk, q->N * f, p->N * f, p->H, s);
  if (!rc && dKbar) rc = crop_rows(dKbar, p->N * f, w.dkbar, q->N * f, p->N * f, p->H, s);
  return rc;
}

int fb_fwd(fb_plan* p, const void* u, void* y, int64_t B, void* ws, void* stream) {
  int rc = check_run(p, B, "fb_fwd");
  if (rc) return rc;
  if (!u || !y) return fail(FB_ERR_ARG, "fb_fwd: null tensor");
  if (p->engine == FB_ENGINE_THREE && !ws) return fail(FB_ERR_ARG, "fb_fwd: workspace required");
  DevGuard dg(p->device);
  if ((rc = cuda_status(dg.err, "cudaSetDevice"))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->inner) return pad_fwd(p, u, y, nullptr, B, ws, s);
  // tp_fwd waits for the prep after its pass 1
  if (p->engine == FB_ENGINE_SINGLE && (rc = prep_wait(p, s))) return rc;
  return p->engine == FB_ENGINE_SINGLE ? sp_fwd(p, u, y, B, s) : tp_fwd(p, u, y, B, ws, s);
}

int fb_fwd_save(fb_plan* p, const void* u, void* y, void* saved, int64_t B, void* ws,
                void* stream) {
  if (!saved || !p || !fb_saved_size(p, B)) return fb_fwd(p, u, y, B, ws, stream);
  int rc = check_run(p, B, "fb_fwd_save");
  if (rc) return rc;
  if (!u || !y) return fail(FB_ERR_ARG, "fb_fwd_save: null tensor");
  DevGuard dg(p->device);
  if ((rc = cuda_status(dg.err, "cudaSetDevice"))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->use_tc) {
    if ((rc = prep_wait(p, s))) return rc;
    return tc_fwd(p, u, y, B, s, saved);
  }
  if (!ws) return fail(FB_ERR_ARG, "fb_fwd_save: workspace required");
  if (p->inner) return pad_fwd(p, u, y, saved, B, ws, s);
  return tp_fwd(p, u, y, B, ws, s, saved);
}

int fb_bwd_saved(fb_plan* p, const void* dy, const void* u, const void* saved, void* du,
                 float* dK, float* dKbar, float* dD, int64_t B, void* ws, void* stream) {
  if (!saved || !p || !fb_saved_size(p, B))
    return fb_bwd(p, dy, u, du, dK, dKbar, dD, B, ws, stream);
  int rc = check_run(p, B, "fb_bwd_saved");
  if (rc) return rc;
  if (!dy || !du || !dK || !dD || !ws) return fail(FB_ERR_ARG, "fb_bwd_saved: null argument");
  DevGuard dg(p->device);
  if ((rc = cuda_status(dg.err, "cudaSetDevice"))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->inner) return pad_bwd(p, dy, u, saved, du, dK, dKbar, dD, B, ws, s);
  if ((rc = prep_wait(p, s))) return rc;
  if (p->use_tc) return tc_bwd(p, dy, u, du, dK, dKbar, dD, B, ws, s, saved);
  return tp_bwd(p, dy, u, du, dK, dKbar, dD, B, ws, s, saved);
}

int fb_bwd(fb_plan* p, const void* dy, const void* u, void* du, float* dK, float* dKbar,
           float* dD, int64_t B, void* ws, void* stream) {
  int rc = check_run(p, B, "fb_bwd");
  if (rc) return rc;
  if (!dy || !u || !du || !dK || !dD || !ws) return fail(FB_ERR_ARG, "fb_bwd: null argument");
  DevGuard dg(p->device);
  if ((rc = cuda_status(dg.err, "cudaSetDevice"))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->inner) return pad_bwd(p, dy, u, nullptr, du, dK, dKbar, dD, B, ws, s);
  if ((rc = prep_wait(p, s))) return rc;
  return p->engine == FB_ENGINE_SINGLE ? sp_bwd(p, dy, u, du, dK, dKbar, dD, B, ws, s)
                                       : tp_bwd(p, dy, u, du, dK, dKbar, dD, B, ws, s);
}

}  // extern "C"

// ---------------------------------------------------------------- host runner
constexpr int kRunnerBufs = 3;  // device buffer sets: copies of chunks c-1, c, c+1 in flight
struct fb_host_runner {
  fb_plan* plan = nullptr;  // Hc heads, reused chunk after chunk on the compute stream
  // Hc / 2 and Hc / 4 heads: the first and last chunks are smaller, so the
  // pipeline fills and drains in a fraction of a full chunk's copy time
  fb_plan* small[2] = {nullptr, nullptr};
  int64_t N = 0, H = 0, Hc = 0, B = 0;
  size_t es = 2;
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaEvent_t start = nullptr;
  struct Buf {
    void *u = nullptr, *dy = nullptr, *y = nullptr, *du = nullptr, *ws = nullptr;
    void* saved = nullptr;  // the forward's transform of u (tensor-core plans)
    float *K = nullptr, *D = nullptr, *dK = nullptr, *dD = nullptr;
    cudaEvent_t in_ready = nullptr, comp_done = nullptr, out_done = nullptr;
    bool used = false;
  } buf[kRunnerBufs];
};

extern "C" {

int fb_host_runner_destroy(fb_host_runner* r) {
  if (!r) return FB_OK;
  DevGuard dg(r->plan ? r->plan->device : 0);
  for (auto& b : r->buf) {
    cudaFree(b.u);
    cudaFree(b.dy);
    cudaFree(b.y);
    cudaFree(b.du);
    cudaFree(b.ws);
    cudaFree(b.saved);
    cudaFree(b.K);
    cudaFree(b.D);
    cudaFree(b.dK);
    cudaFree(b.dD);
    if (b.in_ready) cudaEventDestroy(b.in_ready);
    if (b.comp_done) cudaEventDestroy(b.comp_done);
    if (b.out_done) cudaEventDestroy(b.out_done);
  }
  if (r->start) cudaEventDestroy(r->start);
  if (r->s_in) cudaStreamDestroy(r->s_in);
  if (r->s_comp) cudaStreamDestroy(r->s_comp);
  if (r->s_out) cudaStreamDestroy(r->s_out);
  fb_plan_destroy(r->plan);
  fb_plan_destroy(r->small[0]);
  fb_plan_destroy(r->small[1]);
  delete r;
  return FB_OK;
}

int fb_host_runner_create(fb_host_runner** out, int64_t N, int64_t H, int mode, int dtype,
                          int engine, int device, int64_t B, int64_t heads_per_chunk) {
  if (!out) return fail(FB_ERR_ARG, "fb_host_runner_create: null output");
  *out = nullptr;
  if (H < 1 || B < 1 || heads_per_chunk < 1)
    return fail(FB_ERR_DIM, "fb_host_runner_create: H, B and heads_per_chunk must be >= 1");
  int64_t hc = std::min(H, heads_per_chunk);
  while (H % hc) --hc;
  auto* r = new fb_host_runner();
  r->N = N;
  r->H = H;
  r->Hc = hc;
  r->B = B;
  r->es = dtype == FB_F32 ? 4 : 2;
  int rc = fb_plan_create(&r->plan, N, hc, mode, dtype, engine, device);
  if (rc) {
    delete r;
    return rc;
  }
  if (H / hc >= 4 && hc % 4 == 0) {
    rc = fb_plan_create(&r->small[0], N, hc / 2, mode, dtype, engine, device);
    if (!rc) rc = fb_plan_create(&r->small[1], N, hc / 4, mode, dtype, engine, device);
    if (rc) {
      fb_host_runner_destroy(r);
      return rc;
    }
  }
  const size_t sig = (size_t)B * hc * N * r->es, bank = (size_t)hc * N * sizeof(float);
  const size_t wsb = fb_workspace_size(r->plan, B);
  auto mk = [&](void** p2, size_t bytes) {
    return rc ? rc : (rc = cuda_status(cudaMalloc(p2, bytes), "fb_host_runner: cudaMalloc"));
  };
  for (auto& b : r->buf) {
    mk(&b.u, sig);
    mk(&b.dy, sig);
    mk(&b.y, sig);
    mk(&b.du, sig);
    mk(&b.ws, wsb);
    if (const size_t sv = fb_saved_size(r->plan, B)) mk(&b.saved, sv);
    mk((void**)&b.K, bank);
    mk((void**)&b.D, hc * sizeof(float));
    mk((void**)&b.dK, bank);
    mk((void**)&b.dD, hc * sizeof(float));
    if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&b.in_ready, cudaEventDisableTiming), "event");
    if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&b.comp_done, cudaEventDisableTiming), "event");
    if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&b.out_done, cudaEventDisableTiming), "event");
  }
  if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&r->start, cudaEventDisableTiming), "event");
  if (!rc) rc = cuda_status(cudaStreamCreateWithFlags(&r->s_in, cudaStreamNonBlocking), "stream");
  if (!rc) rc = cuda_status(cudaStreamCreateWithFlags(&r->s_comp, cudaStreamNonBlocking), "stream");
  if (!rc) rc = cuda_status(cudaStreamCreateWithFlags(&r->s_out, cudaStreamNonBlocking), "stream");
  if (rc) {
    fb_host_runner_destroy(r);
    return rc;
  }
  *out = r;
  return FB_OK;
}

int64_t fb_host_runner_chunk_heads(const fb_host_runner* r) { return r ? r->Hc : 0; }

int fb_host_runner_run(fb_host_runner* r, const fb_reg_config* cfg, int training, const void* u,
                       const void* dy, const float* K, const float* D, void* y, void* du,
                       float* dK, float* dD, void* stream) {
  if (!r || !cfg || !u || !dy || !K || !D || !y || !du || !dK || !dD)
    return fail(FB_ERR_ARG, "fb_host_runner_run: null argument");
  fb_plan* p = r->plan;
  DevGuard dg(p->device);
  int rc = cuda_status(dg.err, "cudaSetDevice");
  if (rc) return rc;
  cudaStream_t caller = (cudaStream_t)stream;
  const int64_t N = r->N, H = r->H, Hc = r->Hc, B = r->B;
  const size_t es = r->es;
  const size_t pitch = (size_t)H * N * es;  // host row pitch (one batch row of all heads)
  rc = cuda_status(cudaEventRecord(r->start, caller), "event record");
  for (cudaStream_t s : {r->s_in, r->s_comp, r->s_out})
    if (!rc) rc = cuda_status(cudaStreamWaitEvent(s, r->start, 0), "stream wait");
  // chunk schedule: Hc heads each, or (small plans present) Hc/4, Hc/4, Hc/2,
  // Hc ..., Hc/2, Hc/4, Hc/4
  std::vector<fb_plan*> sched;
  if (r->small[0]) {
    sched = {r->small[1], r->small[1], r->small[0]};
    for (int64_t i = 0; i < H / Hc - 2; ++i) sched.push_back(p);
    for (fb_plan* q : {r->small[0], r->small[1], r->small[1]}) sched.push_back(q);
  } else {
    sched.assign((size_t)(H / Hc), p);
  }
  int64_t h0 = 0;
  for (size_t c = 0; c < sched.size() && !rc; ++c) {
    auto& b = r->buf[c % kRunnerBufs];
    fb_plan* q = sched[c];
    const int64_t Hk = q->H;
    const size_t row = (size_t)Hk * N * es;
    const char* hu = (const char*)u + h0 * N * es;
    const char* hdy = (const char*)dy + h0 * N * es;
    // inputs: the previous user of this buffer must be done reading u / dy
    if (b.used) rc = cuda_status(cudaStreamWaitEvent(r->s_in, b.comp_done, 0), "wait");
    if (!rc) rc = cuda_status(cudaMemcpy2DAsync(b.u, row, hu, pitch, row, B, cudaMemcpyHostToDevice, r->s_in), "h2d u");
    if (!rc) rc = cuda_status(cudaMemcpy2DAsync(b.dy, row, hdy, pitch, row, B, cudaMemcpyHostToDevice, r->s_in), "h2d dy");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(b.K, K + h0 * N, Hk * N * sizeof(float), cudaMemcpyHostToDevice, r->s_in), "h2d K");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(b.D, D + h0, Hk * sizeof(float), cudaMemcpyHostToDevice, r->s_in), "h2d D");
    if (!rc) rc = cuda_status(cudaEventRecord(b.in_ready, r->s_in), "event record");
    // compute: inputs landed, and the previous results of this buffer copied out
    if (!rc) rc = cuda_status(cudaStreamWaitEvent(r->s_comp, b.in_ready, 0), "wait");
    if (!rc && b.used) rc = cuda_status(cudaStreamWaitEvent(r->s_comp, b.out_done, 0), "wait");
    q->head0 = h0;
    if (!rc) rc = fb_kernel_prep(q, b.K, b.D, cfg, training, r->s_comp);
    if (!rc) rc = fb_fwd_save(q, b.u, b.y, b.saved, B, b.ws, r->s_comp);
    if (!rc) rc = fb_bwd_saved(q, b.dy, b.u, b.saved, b.du, b.dK, nullptr, b.dD, B, b.ws, r->s_comp);
    if (!rc) rc = cuda_status(cudaEventRecord(b.comp_done, r->s_comp), "event record");
    // outputs
    if (!rc) rc = cuda_status(cudaStreamWaitEvent(r->s_out, b.comp_done, 0), "wait");
    if (!rc) rc = cuda_status(cudaMemcpy2DAsync((char*)y + h0 * N * es, pitch, b.y, row, row, B, cudaMemcpyDeviceToHost, r->s_out), "d2h y");
    if (!rc) rc = cuda_status(cudaMemcpy2DAsync((char*)du + h0 * N * es, pitch, b.du, row, row, B, cudaMemcpyDeviceToHost, r->s_out), "d2h du");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(dK + h0 * N, b.dK, Hk * N * sizeof(float), cudaMemcpyDeviceToHost, r->s_out), "d2h dK");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(dD + h0, b.dD, Hk * sizeof(float), cudaMemcpyDeviceToHost, r->s_out), "d2h dD");
    if (!rc) rc = cuda_status(cudaEventRecord(b.out_done, r->s_out), "event record");
    b.used = true;
    q->head0 = 0;
    h0 += Hk;
  }
  // the caller's stream resumes after everything
  for (auto& b : r->buf)
    if (!rc && b.used) rc = cuda_status(cudaStreamWaitEvent(caller, b.out_done, 0), "wait");
  return rc;
}

}  // extern "C"

