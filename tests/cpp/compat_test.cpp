// Drop-in check of the C++ reference-shaped API (include/longconv_b200.hpp):
// code written against the reference `longconv` layer compiles unchanged and
// agrees with the fp64 oracle (oracle/lc_oracle.c, test infrastructure only).
#include <cmath>
#include <cstdio>
#include <vector>

#include "longconv_b200.hpp"
#include "../../oracle/lc_oracle.h"

using namespace longconv;

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

static int fails = 0;
static void expect(bool ok, const char* what, double v = 0) {
  std::printf("%-48s %s %g\n", what, ok ? "ok" : "FAIL", v);
  if (!ok) ++fails;
}

int main() {
  // causal u=[1,2,3,4], k=[1,1,0,0] -> [1,3,5,7] (through the layer, D = 0)
  {
    SignalBatch u(1, 1, 4);
    u.data = {1, 2, 3, 4};
    KernelBank bank(1, 4);
    bank.kernels = {1, 1, 0, 0};
    SignalBatch y = regularized_long_conv(u, bank, RegularizationConfig{}, Engine::kButterfly,
                                          ConvMode::kCausal);
    const std::vector<double> want = {1, 3, 5, 7};
    expect(rel_l2(y.data, want) < 1e-6, "SPEC causal [1,3,5,7]", rel_l2(y.data, want));
    SignalBatch yc = regularized_long_conv(u, bank, RegularizationConfig{}, Engine::kButterfly,
                                           ConvMode::kCircular);
    const std::vector<double> wantc = {5, 3, 5, 7};
    expect(rel_l2(yc.data, wantc) < 1e-6, "SPEC circular [5,3,5,7]", rel_l2(yc.data, wantc));
  }
  // random layer vs the oracle, fwd + bwd, fp32 validation mode (1e-5)
  {
    const size_t B = 3, H = 4, N = 2048;
    SignalBatch u(B, H, N), dy(B, H, N);
    lco_signal_batch(1, B, H, N, u.data.data());
    lco_signal_batch(2, B, H, N, dy.data.data());
    KernelBank bank(H, N);
    lco_init_kernels(1, H, N, 3, bank.kernels.data(), bank.skip_gain.data());
    // round inputs to the device precision so both sides see the same values
    for (auto* v : {&u.data, &dy.data, &bank.kernels, &bank.skip_gain})
      for (double& x : *v) x = (double)(float)x;
    RegularizationConfig cfg;
    cfg.lambda = 0.003;
    cfg.smooth_width = 1;
    SignalBatch y = regularized_long_conv(u, bank, cfg, Engine::kButterfly, ConvMode::kCausal, false, 8);
    std::vector<double> yr(B * H * N), kbar(H * N);
    lco_regularized_long_conv(u.data.data(), B, H, N, bank.kernels.data(), bank.skip_gain.data(), 0.003,
                              1, 0.0, 0, 0, 1, 0, yr.data());
    expect(rel_l2(y.data, yr) < 1e-5, "regularized_long_conv vs oracle", rel_l2(y.data, yr));
    KernelBank rb = regularize_bank(bank, cfg, false);
    lco_regularize_bank(bank.kernels.data(), H, N, 0.003, 1, 0.0, 0, 0, 0, kbar.data());
    expect(rel_l2(rb.kernels, kbar) < 1e-6, "regularize_bank vs oracle", rel_l2(rb.kernels, kbar));
    LongConvGradients g =
        regularized_long_conv_backward(dy, u, bank, cfg, Engine::kButterfly, ConvMode::kCausal);
    std::vector<double> du(B * H * N), dkb(H * N), dD(H), dK(H * N);
    lco_long_conv_backward(u.data.data(), dy.data.data(), B, H, N, kbar.data(), bank.skip_gain.data(), 1,
                           du.data(), dkb.data(), dD.data());
    lco_regularizer_backward(bank.kernels.data(), H, N, 0.003, 1, 0.0, 0, 0, dkb.data(), dK.data());
    expect(rel_l2(g.du.data, du) < 1e-5, "backward du vs oracle", rel_l2(g.du.data, du));
    expect(rel_l2(g.dkernels, dK) < 1e-5, "backward dK vs oracle", rel_l2(g.dkernels, dK));
    expect(rel_l2(g.dskip_gain, dD) < 1e-5, "backward dD vs oracle", rel_l2(g.dskip_gain, dD));
    // three-pass engine on a long sequence
    const size_t N2 = 16384;
    SignalBatch u2(2, 1, N2);
    lco_signal_batch(5, 2, 1, N2, u2.data.data());
    for (double& x : u2.data) x = (double)(float)x;
    KernelBank b2(1, N2);
    lco_init_kernels(1, 1, N2, 6, b2.kernels.data(), b2.skip_gain.data());
    for (double& x : b2.kernels) x = (double)(float)x;
    for (double& x : b2.skip_gain) x = (double)(float)x;
    SignalBatch y2 = regularized_long_conv(u2, b2, cfg, Engine::kThreePass, ConvMode::kCausal);
    std::vector<double> y2r(2 * N2);
    lco_regularized_long_conv(u2.data.data(), 2, 1, N2, b2.kernels.data(), b2.skip_gain.data(), 0.003, 1,
                              0.0, 0, 0, 1, 0, y2r.data());
    expect(rel_l2(y2.data, y2r) < 1e-5, "three-pass engine vs oracle", rel_l2(y2.data, y2r));
  }
  // error behaviour mirrors the reference
  {
    SignalBatch u(1, 2, 8);
    KernelBank bank(3, 8);
    bool threw = false;
    try {
      regularized_long_conv(u, bank, RegularizationConfig{}, Engine::kButterfly, ConvMode::kCausal);
    } catch (const DimensionError&) {
      threw = true;
    }
    expect(threw, "DimensionError on bank/batch mismatch");
    threw = false;
    try {
      KernelBank b2(2, 8);
      regularized_long_conv(u, b2, RegularizationConfig{}, Engine::kNaive, ConvMode::kCausal);
    } catch (const PlanError&) {
      threw = true;
    }
    expect(threw, "PlanError for the CPU-only naive engine");
  }
  // learned butterfly, DFT init == FFT
  {
    const size_t n = 64, r = 4, B = 2, H = 2;
    size_t pc = 0;
    lco_learned_param_count(n, r, &pc);
    std::vector<double> one(2 * pc), blocks;
    lco_learned_init(n, r, one.data());
    for (size_t h = 0; h < H; ++h) blocks.insert(blocks.end(), one.begin(), one.end());
    std::vector<double> x(B * H * 2 * n);
    lco_signal_batch(9, 1, 1, x.size(), x.data());
    for (double& v : x) v = (double)(float)v;
    std::vector<double> y = learned_forward_batched(n, r, B, H, blocks, x), want(x.size());
    for (size_t row = 0; row < B * H; ++row)
      lco_apply_plan(n, r, x.data() + row * 2 * n, 0, want.data() + row * 2 * n);
    expect(rel_l2(y, want) < 1e-5, "learned_forward (DFT init) == apply_plan", rel_l2(y, want));
  }
  std::printf(fails ? "COMPAT FAIL\n" : "COMPAT OK\n");
  return fails ? 1 : 0;
}
