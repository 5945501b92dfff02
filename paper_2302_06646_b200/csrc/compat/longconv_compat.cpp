// C++ drop-in for the reference longconv layer API (include/longconv_b200.hpp)
// on top of the C ABI (include/flashbutterfly.h).  Host fp64 containers in,
// device compute, host fp64 containers out — the reference's ownership model
// (inputs by const reference, outputs returned by value, regularize.hpp:67-70).
#include "longconv_b200.hpp"

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>

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

KernelBank init_kernels(const InitConfig& cfg) {
  if (cfg.heads == 0 || cfg.len == 0) throw DimensionError("init_kernels: heads and len must be >= 1");
  KernelBank bank(cfg.heads, cfg.len);
  DevBuf K(bank.kernels.size() * 8), D(bank.heads * 8);
  check(fb_init_kernels(cfg.kind == InitKind::kGeometric ? FB_INIT_GEOMETRIC : FB_INIT_RANDOM,
                        (int64_t)cfg.heads, (int64_t)cfg.len, cfg.seed, nullptr, nullptr, (double*)K.p,
                        (double*)D.p, g_device, nullptr),
        "init_kernels");
  cuda(cudaDeviceSynchronize(), "sync");
  cuda(cudaMemcpy(bank.kernels.data(), K.p, bank.kernels.size() * 8, cudaMemcpyDeviceToHost), "download");
  cuda(cudaMemcpy(bank.skip_gain.data(), D.p, bank.heads * 8, cudaMemcpyDeviceToHost), "download");
  return bank;
}

double geometric_envelope(std::size_t position, std::size_t len, std::size_t head, std::size_t heads) {
  const double decay = std::pow((double)heads / 2.0, (double)head / (double)heads);
  return std::exp(-((double)position / (double)len) * decay);
}

// ------------------------------------------------------------------ single rows
// The reference's single-row entry points (butterfly.hpp:74-108,
// three_pass.hpp:113-131) on the device: fp64 host spans in, f32 complex rows
// through fb_dft_* / fb_learned_*, fp64 host results out.
namespace {

std::vector<float> to_f32(std::span<const Complex> x) {
  std::vector<float> h(2 * x.size());
  for (size_t i = 0; i < x.size(); ++i) {
    h[2 * i] = (float)x[i].real();
    h[2 * i + 1] = (float)x[i].imag();
  }
  return h;
}
std::unique_ptr<DevBuf> upload_c(std::span<const Complex> x) {
  std::vector<float> h = to_f32(x);
  auto b = std::make_unique<DevBuf>(h.size() * 4);
  if (!h.empty()) cuda(cudaMemcpy(b->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "upload");
  return b;
}
ComplexSeq download_c(const DevBuf& b, size_t n) {
  std::vector<float> h(2 * n);
  cuda(cudaDeviceSynchronize(), "sync");
  if (n) cuda(cudaMemcpy(h.data(), b.p, h.size() * 4, cudaMemcpyDeviceToHost), "download");
  ComplexSeq out(n);
  for (size_t i = 0; i < n; ++i) out[i] = Complex(h[2 * i], h[2 * i + 1]);
  return out;
}
fb_dft_plan* dev_of(const ButterflyPlan& plan) {
  if (!plan.device) throw PlanError("apply_plan: plan was not built by build_plan");
  return static_cast<fb_dft_plan*>(plan.device.get());
}
std::shared_ptr<void> make_dft(size_t n, size_t r) {
  fb_dft_plan* d = nullptr;
  check(fb_dft_plan_create(&d, (int64_t)n, (int64_t)r, g_device), "build_plan");
  return std::shared_ptr<void>(d, [](void* q) { fb_dft_plan_destroy(static_cast<fb_dft_plan*>(q)); });
}
// circular (n == N) or causal (n == 2N) convolution of complex rows on the device
ComplexSeq conv_dev(fb_dft_plan* d, std::span<const Complex> u, std::span<const Complex> k,
                    const ComplexSeq* kspec, int mode) {
  const size_t N = u.size();
  auto ud = upload_c(u);
  auto kd = kspec ? upload_c(*kspec) : upload_c(k);
  DevBuf yd(N * 8), ws(fb_dft_workspace_size(d, 1, 1));
  if (kspec)
    check(fb_conv_rows_spectrum(d, (const float*)ud->p, (const float*)kd->p, (float*)yd.p, (int64_t)N, 1, 1,
                                mode, ws.p, nullptr),
          "conv_three_pass");
  else
    check(fb_conv_rows(d, (const float*)ud->p, (const float*)kd->p, (float*)yd.p, (int64_t)N, 1, 1, mode,
                       ws.p, nullptr),
          "conv_butterfly");
  return download_c(yd, N);
}
// one-head learned plan matching lb.plan, blocks flattened to f32 pairs
struct LearnedDev {
  fb_learned_plan* p = nullptr;
  std::unique_ptr<DevBuf> blocks;
  ~LearnedDev() { fb_learned_plan_destroy(p); }
};
void learned_dev(const LearnedButterfly& lb, LearnedDev& L) {
  if (lb.blocks.size() != lb.plan.stages.size())
    throw DimensionError("learned_forward: block count != stage count");
  std::vector<Complex> flat;
  for (size_t s = 0; s < lb.blocks.size(); ++s) {
    const size_t f = lb.plan.stages[s].factor;
    if (lb.blocks[s].size() != f * f) throw DimensionError("learned_forward: block shape mismatch");
    flat.insert(flat.end(), lb.blocks[s].begin(), lb.blocks[s].end());
  }
  check(fb_learned_plan_create(&L.p, (int64_t)lb.plan.n, (int64_t)lb.plan.r, 1, FB_F32, g_device),
        "learned plan");
  L.blocks = upload_c(flat);
}

}  // namespace

std::string ButterflyPlan::describe_json() const {
  std::string s = "{\"n\":" + std::to_string(n) + ",\"r\":" + std::to_string(r) + ",\"stage_factors\":[";
  for (size_t i = 0; i < stages.size(); ++i) s += (i ? "," : "") + std::to_string(stages[i].factor);
  return s + "]}";
}

ButterflyPlan build_plan(std::size_t n, std::size_t r) {
  ButterflyPlan plan;
  plan.device = make_dft(n, r);  // validates n and r exactly like the reference (PlanError)
  plan.n = n;
  plan.r = r;
  int64_t f[64], cnt = 0;
  check(fb_dft_plan_factors(dev_of(plan), f, &cnt), "build_plan");
  size_t seg = n;
  for (int64_t i = 0; i < cnt; ++i) {
    PlanStage st;
    st.factor = (size_t)f[i];
    st.segment = seg;
    st.dft_block.resize(st.factor * st.factor);
    for (size_t p = 0; p < st.factor; ++p)
      for (size_t q = 0; q < st.factor; ++q)
        st.dft_block[p * st.factor + q] =
            std::polar(1.0, -2.0 * M_PI * (double)((p * q) % st.factor) / (double)st.factor);
    plan.stages.push_back(std::move(st));
    seg /= (size_t)f[i];
  }
  return plan;
}

ComplexSeq apply_plan(const ButterflyPlan& plan, std::span<const Complex> x, Direction dir) {
  if (x.size() != plan.n) throw DimensionError("apply_plan: input length != plan.n");
  fb_dft_plan* d = dev_of(plan);
  auto xd = upload_c(x);
  DevBuf yd(x.size() * 8), ws(fb_dft_workspace_size(d, 1, 0));
  check(fb_dft(d, (const float*)xd->p, (float*)yd.p, 1, dir == Direction::kInverse ? 1 : 0, ws.p, nullptr),
        "apply_plan");
  return download_c(yd, x.size());
}

ComplexSeq conv_butterfly(std::span<const Complex> u, std::span<const Complex> k,
                          const ButterflyPlan& plan, ConvMode mode) {
  if (k.size() != u.size()) throw DimensionError("conv_butterfly: u and k length mismatch");
  return conv_dev(dev_of(plan), u, k, nullptr,
                  mode == ConvMode::kCircular ? FB_MODE_CIRCULAR : FB_MODE_CAUSAL);
}

LearnedButterfly LearnedButterfly::from_plan(const ButterflyPlan& plan) {
  LearnedButterfly lb;
  lb.plan = plan;
  for (const PlanStage& st : plan.stages) lb.blocks.push_back(st.dft_block);
  return lb;
}

std::size_t LearnedButterfly::parameter_count() const {
  size_t c = 0;
  for (const auto& b : blocks) c += b.size();
  return c;
}

ComplexSeq learned_forward(const LearnedButterfly& lb, std::span<const Complex> x) {
  if (x.size() != lb.plan.n) throw DimensionError("learned_forward: input length != plan.n");
  if (lb.plan.n == 1 && lb.blocks.empty()) return ComplexSeq(x.begin(), x.end());
  LearnedDev L;
  learned_dev(lb, L);
  auto xd = upload_c(x);
  DevBuf yd(x.size() * 8);
  check(fb_learned_fwd(L.p, (const float*)L.blocks->p, xd->p, yd.p, 1, nullptr, nullptr), "learned_forward");
  return download_c(yd, x.size());
}

LearnedGradients learned_gradients(const LearnedButterfly& lb, std::span<const Complex> x,
                                   std::span<const Complex> upstream) {
  if (x.size() != lb.plan.n || upstream.size() != lb.plan.n)
    throw DimensionError("learned_gradients: length mismatch");
  LearnedGradients g;
  if (lb.plan.n == 1 && lb.blocks.empty()) {
    g.input_grad.assign(upstream.begin(), upstream.end());
    return g;
  }
  LearnedDev L;
  learned_dev(lb, L);
  auto xd = upload_c(x);
  auto gd = upload_c(upstream);
  const size_t P = lb.parameter_count();
  DevBuf dxd(x.size() * 8), dbd(P * 8), ws(fb_learned_workspace_size(L.p, 1));
  check(fb_learned_bwd(L.p, (const float*)L.blocks->p, xd->p, gd->p, dxd.p, (float*)dbd.p, 1, ws.p,
                       nullptr),
        "learned_gradients");
  g.input_grad = download_c(dxd, x.size());
  const ComplexSeq flat = download_c(dbd, P);
  size_t o = 0;
  for (const auto& b : lb.blocks) {
    g.block_grads.emplace_back(flat.begin() + (long)o, flat.begin() + (long)(o + b.size()));
    o += b.size();
  }
  return g;
}

std::vector<Complex> learned_dense_matrix(const LearnedButterfly& lb) {
  // the operator applied to the n unit vectors as n rows of one launch
  const size_t n = lb.plan.n;
  ComplexSeq eye(n * n, Complex(0, 0));
  for (size_t j = 0; j < n; ++j) eye[j * n + j] = Complex(1, 0);
  ComplexSeq cols(n * n);
  if (n == 1 && lb.blocks.empty()) {
    cols = eye;
  } else {
    LearnedDev L;
    learned_dev(lb, L);
    auto xd = upload_c(eye);
    DevBuf yd(n * n * 8);
    check(fb_learned_fwd(L.p, (const float*)L.blocks->p, xd->p, yd.p, (int64_t)n, nullptr, nullptr),
          "learned_dense_matrix");
    cols = download_c(yd, n * n);
  }
  std::vector<Complex> dense(n * n);  // row-major M[i][j] = (F e_j)[i]
  for (size_t j = 0; j < n; ++j)
    for (size_t i = 0; i < n; ++i) dense[i * n + j] = cols[j * n + i];
  return dense;
}

// ---- PassCounter (three_pass.hpp:27-58)
void PassCounter::reset(std::size_t n) {
  n_ = n;
  current_ = -1;
  phases_ = {};
  seen_.assign(n, 0);
}
void PassCounter::begin_phase(int phase) {
  if (phase < 1 || phase > 3) throw DimensionError("PassCounter: phase must be 1..3");
  current_ = phase - 1;
  if (seen_.size() != n_) seen_.assign(n_, 0);
}
void PassCounter::touch(std::size_t index) {
  const std::uint8_t mark = (std::uint8_t)(current_ + 1);
  if (index < seen_.size() && seen_[index] != mark) {
    seen_[index] = mark;
    ++phases_[(size_t)current_].distinct_touched;
  }
}
void PassCounter::record_read(std::size_t index) {
  ++phases_[(size_t)current_].reads;
  touch(index);
}
void PassCounter::record_write(std::size_t index) {
  ++phases_[(size_t)current_].writes;
  touch(index);
}
void PassCounter::record_working_set(std::size_t elements) {
  auto& p = phases_[(size_t)current_];
  if (elements > p.working_set_peak) p.working_set_peak = elements;
}
void PassCounter::merge_counts(std::uint64_t reads, std::uint64_t writes) {
  phases_[(size_t)current_].reads += reads;
  phases_[(size_t)current_].writes += writes;
}
int PassCounter::sweeps() const {
  int c = 0;
  for (const Phase& p : phases_) c += (n_ > 0 && p.distinct_touched >= n_) ? 1 : 0;
  return c;
}
std::string PassCounter::report_json() const {
  std::string s = "{\"buffer_len\":" + std::to_string(n_) + ",\"phases\":[";
  for (size_t i = 0; i < phases_.size(); ++i) {
    const Phase& p = phases_[i];
    s += (i ? ",{" : "{") + std::string("\"phase\":") + std::to_string(i + 1) +
         ",\"reads\":" + std::to_string(p.reads) + ",\"writes\":" + std::to_string(p.writes) +
         ",\"distinct_touched\":" + std::to_string(p.distinct_touched) +
         ",\"working_set_peak\":" + std::to_string(p.working_set_peak) + "}";
  }
  return s + "],\"sweeps\":" + std::to_string(sweeps()) + ",\"working_set_cap\":" +
         std::to_string(cap_) + "}";
}

// ---- three-pass (three_pass.hpp:100-131)
ThreePassPlan build_three_pass(std::span<const Complex> kernel, std::size_t l, std::size_t m,
                               std::size_t inner_r) {
  const size_t n = kernel.size();
  if (l == 0 || m == 0 || l * m != n) throw DimensionError("build_three_pass: need kernel length n == l*m");
  ThreePassPlan plan;
  plan.n = n;
  plan.l = l;
  plan.m = m;
  plan.inner = build_plan(l, inner_r);
  plan.device = make_dft(n, inner_r);
  fb_dft_plan* d = static_cast<fb_dft_plan*>(plan.device.get());
  auto kd = upload_c(kernel);
  DevBuf kh(n * 8), ws(fb_dft_workspace_size(d, 1, 0));
  check(fb_dft(d, (const float*)kd->p, (float*)kh.p, 1, 0, ws.p, nullptr), "build_three_pass");
  plan.k_hat = download_c(kh, n);
  plan.d_k.resize(n);
  for (size_t a = 0; a < m; ++a)
    for (size_t tau = 0; tau < l; ++tau) plan.d_k[a * l + tau] = (double)l * plan.k_hat[tau * m + a];
  return plan;
}

ComplexSeq conv_three_pass_ordered(const ThreePassPlan& plan, std::span<const Complex> u,
                                   std::span<const std::size_t> block_order, PassCounter* counter) {
  if (u.size() != plan.n) throw DimensionError("conv_three_pass: input length != plan.n");
  if (block_order.size() != plan.m)
    throw DimensionError("conv_three_pass: block order must list all m blocks");
  std::vector<char> seen(plan.m, 0);
  for (size_t a : block_order) {
    if (a >= plan.m) throw DimensionError("conv_three_pass: block index out of range");
    seen[a] = 1;
  }
  if (!plan.device) throw PlanError("conv_three_pass: plan was not built by build_three_pass");
  ComplexSeq y = conv_dev(static_cast<fb_dft_plan*>(plan.device.get()), u, {}, &plan.k_hat,
                          FB_MODE_CIRCULAR);
  if (counter) {  // the device's sweeps: column pass, row pass, column pass
    counter->reset(plan.n);
    const size_t peak[3] = {2 * plan.m, 4 * plan.l, 2 * plan.m};
    for (int ph = 1; ph <= 3; ++ph) {
      counter->begin_phase(ph);
      for (size_t i = 0; i < plan.n; ++i) {
        counter->record_read(i);
        counter->record_write(i);
      }
      counter->record_working_set(peak[ph - 1]);
    }
  }
  return y;
}

ComplexSeq conv_three_pass(const ThreePassPlan& plan, std::span<const Complex> u, PassCounter* counter,
                           int /*threads*/) {
  std::vector<size_t> order(plan.m);
  std::iota(order.begin(), order.end(), size_t{0});
  return conv_three_pass_ordered(plan, u, order, counter);
}

std::vector<double> conv_real_packed(std::span<const double> u, std::span<const double> k, ConvMode mode) {
  if (k.size() != u.size()) throw DimensionError("conv_real_packed: length mismatch");
  if (u.empty() || u.size() % 2) throw DimensionError("conv_real_packed: length must be even and positive");
  const size_t N = u.size();
  ComplexSeq uc(u.begin(), u.end()), kc(k.begin(), k.end());
  auto plan = make_dft(mode == ConvMode::kCircular ? N : 2 * N, 16);
  const ComplexSeq y = conv_dev(static_cast<fb_dft_plan*>(plan.get()), uc, kc, nullptr,
                                mode == ConvMode::kCircular ? FB_MODE_CIRCULAR : FB_MODE_CAUSAL);
  std::vector<double> out(N);
  for (size_t i = 0; i < N; ++i) out[i] = y[i].real();
  return out;
}

}  // namespace longconv
