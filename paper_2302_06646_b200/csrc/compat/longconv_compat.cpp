// C++ drop-in for the reference longconv layer API (include/longconv_b200.hpp)
// on top of the C ABI (include/flashbutterfly.h).  Host fp64 containers in,
// device compute, host fp64 containers out — the reference's ownership model
// (inputs by const reference, outputs returned by value, regularize.hpp:67-70).
#include "longconv_b200.hpp"

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <memory>

#include "flashbutterfly.h"

namespace longconv {

namespace {

thread_local Precision g_prec = Precision::kFp32;
thread_local int g_device = 0;

[[noreturn]] void raise(int rc, const std::string& where) {
  const std::string msg = where + ": " + fb_last_error();
  switch (rc) {
    case FB_ERR_DIM: throw DimensionError(msg);
    case FB_ERR_PLAN:
    case FB_ERR_UNSUPPORTED: throw PlanError(msg);
    default: throw DeviceError(msg);
  }
}
void check(int rc, const char* where) {
  if (rc != FB_OK) raise(rc, where);
}
void cuda(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw DeviceError(std::string(where) + ": " + cudaGetErrorString(e));
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

struct Plan {
  fb_plan* p = nullptr;
  ~Plan() { fb_plan_destroy(p); }
};

int io_dtype() {
  return g_prec == Precision::kFp32 ? FB_F32 : g_prec == Precision::kBf16 ? FB_BF16 : FB_F16;
}
size_t io_size() { return g_prec == Precision::kFp32 ? 4 : 2; }

// fp64 host -> device I/O precision
std::unique_ptr<DevBuf> upload_io(const std::vector<double>& v) {
  auto b = std::make_unique<DevBuf>(v.size() * io_size());
  if (g_prec == Precision::kFp32) {
    std::vector<float> h(v.begin(), v.end());
    cuda(cudaMemcpy(b->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "upload");
  } else if (g_prec == Precision::kBf16) {
    std::vector<__nv_bfloat16> h(v.size());
    for (size_t i = 0; i < v.size(); ++i) h[i] = __float2bfloat16((float)v[i]);
    cuda(cudaMemcpy(b->p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "upload");
  } else {
    std::vector<__half> h(v.size());
    for (size_t i = 0; i < v.size(); ++i) h[i] = __float2half((float)v[i]);
    cuda(cudaMemcpy(b->p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "upload");
  }
  return b;
}
void download_io(const DevBuf& b, std::vector<double>& v) {
  if (g_prec == Precision::kFp32) {
    std::vector<float> h(v.size());
    cuda(cudaMemcpy(h.data(), b.p, h.size() * 4, cudaMemcpyDeviceToHost), "download");
    for (size_t i = 0; i < v.size(); ++i) v[i] = h[i];
  } else if (g_prec == Precision::kBf16) {
    std::vector<__nv_bfloat16> h(v.size());
    cuda(cudaMemcpy(h.data(), b.p, h.size() * 2, cudaMemcpyDeviceToHost), "download");
    for (size_t i = 0; i < v.size(); ++i) v[i] = __bfloat162float(h[i]);
  } else {
    std::vector<__half> h(v.size());
    cuda(cudaMemcpy(h.data(), b.p, h.size() * 2, cudaMemcpyDeviceToHost), "download");
    for (size_t i = 0; i < v.size(); ++i) v[i] = __half2float(h[i]);
  }
}
std::unique_ptr<DevBuf> upload_f32(const std::vector<double>& v) {
  auto b = std::make_unique<DevBuf>(v.size() * 4);
  std::vector<float> h(v.begin(), v.end());
  cuda(cudaMemcpy(b->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "upload");
  return b;
}
std::vector<double> download_f32(const DevBuf& b, size_t n) {
  std::vector<float> h(n);
  cuda(cudaMemcpy(h.data(), b.p, n * 4, cudaMemcpyDeviceToHost), "download");
  return std::vector<double>(h.begin(), h.end());
}

fb_reg_config to_c(const RegularizationConfig& c) {
  fb_reg_config r{};
  r.lambda = c.lambda;
  r.smooth_width = (int64_t)c.smooth_width;
  r.dropout_rate = c.dropout_rate;
  r.smooth_domain = c.smooth_domain == SmoothDomain::kTime ? FB_SMOOTH_TIME : FB_SMOOTH_FREQUENCY;
  r.seed = c.seed;
  return r;
}

// The reference's engines agree to tolerance (regularize.hpp:66); kButterfly
// maps to the best device path for the length, kThreePass to the three-pass
// kernels when the length admits them.
int engine_of(Engine e, size_t N, ConvMode mode) {
  if (e == Engine::kNaive)
    throw PlanError("Engine::kNaive is the O(N^2) CPU oracle; not offered on the device");
  if (e == Engine::kThreePass) {
    const size_t n = mode == ConvMode::kCausal ? 2 * N : N;
    if (n >= 16384) return FB_ENGINE_THREE;
  }
  return FB_ENGINE_AUTO;
}

void make_plan(Plan& pl, size_t N, size_t H, ConvMode mode, Engine e) {
  check(fb_plan_create(&pl.p, (int64_t)N, (int64_t)H, mode == ConvMode::kCausal ? FB_MODE_CAUSAL : FB_MODE_CIRCULAR,
                       io_dtype(), engine_of(e, N, mode), g_device),
        "fb_plan_create");
}

void check_bank(const SignalBatch& u, const KernelBank& bank, const char* who) {
  if (bank.heads != u.heads || bank.len != u.len)
    throw DimensionError(std::string(who) + ": bank dimensions must match the batch");
  if (u.data.size() != u.size()) throw DimensionError(std::string(who) + ": malformed batch");
  if (bank.kernels.size() != bank.heads * bank.len || bank.skip_gain.size() != bank.heads)
    throw DimensionError(std::string(who) + ": malformed bank");
}

}  // namespace

void set_device_precision(Precision p) { g_prec = p; }
Precision device_precision() { return g_prec; }
void set_device(int device) { g_device = device; }

KernelBank regularize_bank(const KernelBank& bank, const RegularizationConfig& cfg, bool training) {
  if (bank.heads == 0 || bank.len == 0) return bank;
  Plan pl;
  const Precision saved = g_prec;
  g_prec = Precision::kFp32;
  make_plan(pl, bank.len, bank.heads, ConvMode::kCausal, Engine::kButterfly);
  g_prec = saved;
  auto K = upload_f32(bank.kernels);
  auto D = upload_f32(bank.skip_gain);
  const fb_reg_config c = to_c(cfg);
  check(fb_kernel_prep(pl.p, (const float*)K->p, (const float*)D->p, &c, training ? 1 : 0, nullptr),
        "fb_kernel_prep");
  DevBuf out(bank.kernels.size() * 4);
  check(fb_plan_copy_kbar(pl.p, (float*)out.p, nullptr), "fb_plan_copy_kbar");
  cuda(cudaDeviceSynchronize(), "sync");
  KernelBank r = bank;
  r.kernels = download_f32(out, bank.kernels.size());
  return r;
}

SignalBatch regularized_long_conv(const SignalBatch& u, const KernelBank& bank,
                                  const RegularizationConfig& cfg, Engine engine, ConvMode mode,
                                  bool training, int /*threads*/) {
  check_bank(u, bank, "regularized_long_conv");
  if (u.size() == 0) return u;
  cuda(cudaSetDevice(g_device), "cudaSetDevice");
  Plan pl;
  make_plan(pl, u.len, u.heads, mode, engine);
  auto K = upload_f32(bank.kernels);
  auto D = upload_f32(bank.skip_gain);
  const fb_reg_config c = to_c(cfg);
  check(fb_kernel_prep(pl.p, (const float*)K->p, (const float*)D->p, &c, training ? 1 : 0, nullptr),
        "fb_kernel_prep");
  auto du = upload_io(u.data);
  DevBuf dy(u.size() * io_size());
  DevBuf ws(fb_workspace_size(pl.p, (int64_t)u.batch));
  check(fb_fwd(pl.p, du->p, dy.p, (int64_t)u.batch, ws.p, nullptr), "fb_fwd");
  cuda(cudaDeviceSynchronize(), "sync");
  SignalBatch y(u.batch, u.heads, u.len);
  download_io(dy, y.data);
  return y;
}

LongConvGradients regularized_long_conv_backward(const SignalBatch& dy, const SignalBatch& u,
                                                 const KernelBank& bank,
                                                 const RegularizationConfig& cfg, Engine engine,
                                                 ConvMode mode, bool training) {
  check_bank(u, bank, "regularized_long_conv_backward");
  if (dy.batch != u.batch || dy.heads != u.heads || dy.len != u.len || dy.data.size() != dy.size())
    throw DimensionError("regularized_long_conv_backward: dy and u shapes differ");
  cuda(cudaSetDevice(g_device), "cudaSetDevice");
  Plan pl;
  make_plan(pl, u.len, u.heads, mode, engine);
  auto K = upload_f32(bank.kernels);
  auto D = upload_f32(bank.skip_gain);
  const fb_reg_config c = to_c(cfg);
  check(fb_kernel_prep(pl.p, (const float*)K->p, (const float*)D->p, &c, training ? 1 : 0, nullptr),
        "fb_kernel_prep");
  auto g = upload_io(dy.data);
  auto x = upload_io(u.data);
  DevBuf dx(u.size() * io_size());
  DevBuf dK(bank.kernels.size() * 4), dD(bank.heads * 4);
  DevBuf ws(fb_workspace_size(pl.p, (int64_t)u.batch));
  check(fb_bwd(pl.p, g->p, x->p, dx.p, (float*)dK.p, nullptr, (float*)dD.p, (int64_t)u.batch, ws.p,
               nullptr),
        "fb_bwd");
  cuda(cudaDeviceSynchronize(), "sync");
  LongConvGradients r;
  r.du = SignalBatch(u.batch, u.heads, u.len);
  download_io(dx, r.du.data);
  r.dkernels = download_f32(dK, bank.kernels.size());
  r.dskip_gain = download_f32(dD, bank.heads);
  return r;
}

std::vector<double> learned_forward_batched(std::size_t n, std::size_t r, std::size_t B,
                                            std::size_t H, const std::vector<double>& blocks,
                                            const std::vector<double>& x) {
  fb_learned_plan* p = nullptr;
  check(fb_learned_plan_create(&p, (int64_t)n, (int64_t)r, (int64_t)H, io_dtype(), g_device),
        "fb_learned_plan_create");
  std::unique_ptr<fb_learned_plan, int (*)(fb_learned_plan*)> guard(p, fb_learned_plan_destroy);
  int64_t nst = 0, pc = 0;
  check(fb_learned_plan_factors(p, nullptr, &nst, &pc), "fb_learned_plan_factors");
  if (blocks.size() != H * 2 * (size_t)pc) throw DimensionError("learned_forward: block count != stage count");
  if (x.size() != B * H * 2 * n) throw DimensionError("learned_forward: input length != plan.n");
  auto bl = upload_f32(blocks);
  auto xd = upload_io(x);
  DevBuf yd(x.size() * io_size());
  check(fb_learned_fwd(p, (const float*)bl->p, xd->p, yd.p, (int64_t)B, nullptr, nullptr),
        "fb_learned_fwd");
  cuda(cudaDeviceSynchronize(), "sync");
  std::vector<double> y(x.size());
  download_io(yd, y);
  return y;
}

LearnedBatchGradients learned_gradients_batched(std::size_t n, std::size_t r, std::size_t B,
                                                std::size_t H, const std::vector<double>& blocks,
                                                const std::vector<double>& x,
                                                const std::vector<double>& upstream) {
  fb_learned_plan* p = nullptr;
  check(fb_learned_plan_create(&p, (int64_t)n, (int64_t)r, (int64_t)H, io_dtype(), g_device),
        "fb_learned_plan_create");
  std::unique_ptr<fb_learned_plan, int (*)(fb_learned_plan*)> guard(p, fb_learned_plan_destroy);
  int64_t nst = 0, pc = 0;
  check(fb_learned_plan_factors(p, nullptr, &nst, &pc), "fb_learned_plan_factors");
  if (blocks.size() != H * 2 * (size_t)pc) throw DimensionError("learned_gradients: shape mismatch");
  if (x.size() != B * H * 2 * n || upstream.size() != x.size())
    throw DimensionError("learned_gradients: shape mismatch");
  auto bl = upload_f32(blocks);
  auto xd = upload_io(x);
  auto gd = upload_io(upstream);
  DevBuf dxd(x.size() * io_size()), dbd(blocks.size() * 4);
  DevBuf wsd(fb_learned_workspace_size(p, (int64_t)B));
  check(fb_learned_bwd(p, (const float*)bl->p, xd->p, gd->p, dxd.p, (float*)dbd.p, (int64_t)B, wsd.p,
                       nullptr),
        "fb_learned_bwd");
  cuda(cudaDeviceSynchronize(), "sync");
  LearnedBatchGradients g;
  g.input_grad.resize(x.size());
  download_io(dxd, g.input_grad);
  g.block_grads = download_f32(dbd, blocks.size());
  return g;
}

}  // namespace longconv
