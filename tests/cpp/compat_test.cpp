// Drop-in check of the C++ reference-shaped API (include/longconv_b200.hpp):
// code written against the reference `longconv` layer compiles unchanged and
// agrees with the fp64 oracle (oracle/lc_oracle.c, test infrastructure only).
#include <cmath>
#include <cstdio>
#include <utility>
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
  {  // init_kernels on the device vs the oracle (reference streams)
    InitConfig ic;
    ic.kind = InitKind::kGeometric;
    ic.heads = 4;
    ic.len = 3000;
    ic.seed = 3;
    KernelBank kb = init_kernels(ic);
    std::vector<double> K(ic.heads * ic.len), D(ic.heads);
    lco_init_kernels(1, ic.heads, ic.len, 3, K.data(), D.data());
    const double e = rel_l2(kb.kernels, K), ed = rel_l2(kb.skip_gain, D);
    expect(e < 1e-13 && ed < 1e-13, "init_kernels (geometric) vs oracle", std::max(e, ed));
    expect(std::abs(geometric_envelope(5, 100, 2, 8) - std::exp(-0.05 * std::pow(4.0, 0.25))) < 1e-15,
           "geometric_envelope");
  }
  // ---- single-row entry points (butterfly.hpp:74-108, three_pass.hpp:113-131)
  auto cplx = [](uint64_t seed, size_t n) {
    std::vector<double> d(2 * n);
    lco_signal_batch(seed, 1, 1, 2 * n, d.data());
    ComplexSeq x(n);
    for (size_t i = 0; i < n; ++i) x[i] = Complex((float)d[2 * i], (float)d[2 * i + 1]);
    return x;
  };
  auto flat = [](const ComplexSeq& x) {
    std::vector<double> d(2 * x.size());
    for (size_t i = 0; i < x.size(); ++i) {
      d[2 * i] = x[i].real();
      d[2 * i + 1] = x[i].imag();
    }
    return d;
  };
  {  // build_plan: the reference's factor chains and errors
    ButterflyPlan p = build_plan(8192, 16);
    expect(p.describe_json() == "{\"n\":8192,\"r\":16,\"stage_factors\":[16,16,16,2]}",
           "build_plan(8192,16) stage factors");
    expect(build_plan(96, 16).describe_json() == "{\"n\":96,\"r\":16,\"stage_factors\":[16,6]}",
           "build_plan(96,16) stage factors");
    bool threw = false;
    try {
      build_plan(17, 16);
    } catch (const PlanError&) {
      threw = true;
    }
    expect(threw, "PlanError for a prime remainder > r");
    threw = false;
    try {
      build_plan(64, 1);
    } catch (const PlanError&) {
      threw = true;
    }
    expect(threw, "PlanError for r < 2");
  }
  for (auto [n, r] : {std::pair<size_t, size_t>{8192, 16}, {96, 16}, {64, 4}, {1000, 10}, {131072, 16}}) {
    ButterflyPlan p = build_plan(n, r);
    const ComplexSeq x = cplx(11 + n, n);
    for (int inv = 0; inv < 2; ++inv) {
      ComplexSeq y = apply_plan(p, x, inv ? Direction::kInverse : Direction::kForward);
      std::vector<double> want(2 * n);
      lco_apply_plan(n, r, flat(x).data(), inv, want.data());
      char what[96];
      std::snprintf(what, sizeof what, "apply_plan n=%zu r=%zu %s", n, r, inv ? "inverse" : "forward");
      const double e = rel_l2(flat(y), want);
      expect(e < 1e-5, what, e);
    }
  }
  for (int mode = 0; mode < 2; ++mode) {  // conv_butterfly on complex rows
    const size_t N = 2048;
    ButterflyPlan p = build_plan(mode ? 2 * N : N, 16);
    const ComplexSeq u = cplx(21, N), k = cplx(22, N);
    ComplexSeq y = conv_butterfly(u, k, p, mode ? ConvMode::kCausal : ConvMode::kCircular);
    std::vector<double> want(2 * N);
    lco_conv_butterfly(flat(u).data(), flat(k).data(), N, mode, want.data());
    const double e = rel_l2(flat(y), want);
    expect(e < 1e-5, mode ? "conv_butterfly causal vs oracle" : "conv_butterfly circular vs oracle", e);
  }
  {  // SPEC.md:145 through conv_butterfly
    ButterflyPlan p = build_plan(8, 16);
    const ComplexSeq u = {1, 2, 3, 4}, k = {1, 1, 0, 0};
    ComplexSeq y = conv_butterfly(u, k, p, ConvMode::kCausal);
    const std::vector<double> want = {1, 0, 3, 0, 5, 0, 7, 0};
    expect(rel_l2(flat(y), want) < 1e-6, "conv_butterfly SPEC causal [1,3,5,7]", rel_l2(flat(y), want));
  }
  {  // LearnedButterfly: from_plan reproduces the plan; perturbed-block gradients vs oracle
    const size_t n = 1024, r = 16;
    ButterflyPlan p = build_plan(n, r);
    LearnedButterfly lb = LearnedButterfly::from_plan(p);
    const ComplexSeq x = cplx(31, n);
    const double e0 = rel_l2(flat(learned_forward(lb, x)), flat(apply_plan(p, x, Direction::kForward)));
    expect(e0 < 1e-5, "learned_forward(from_plan) == apply_plan", e0);
    size_t pc = 0;
    lco_learned_param_count(n, r, &pc);
    expect(lb.parameter_count() == pc, "LearnedButterfly::parameter_count", (double)pc);
    const ComplexSeq pert = cplx(32, pc);
    size_t o = 0;
    for (auto& b : lb.blocks)
      for (auto& v : b) v += 0.1 * pert[o++];
    std::vector<double> bl;
    for (auto& b : lb.blocks) {
      auto fb_ = flat(b);
      bl.insert(bl.end(), fb_.begin(), fb_.end());
    }
    const ComplexSeq g = cplx(33, n);
    std::vector<double> yw(2 * n), dbw(2 * pc), dxw(2 * n);
    lco_learned_forward(n, r, bl.data(), flat(x).data(), yw.data());
    lco_learned_gradients(n, r, bl.data(), flat(x).data(), flat(g).data(), dbw.data(), dxw.data());
    const double e1 = rel_l2(flat(learned_forward(lb, x)), yw);
    expect(e1 < 1e-5, "learned_forward (perturbed) vs oracle", e1);
    LearnedGradients lg = learned_gradients(lb, x, g);
    std::vector<double> dbg;
    for (auto& b : lg.block_grads) {
      auto fb_ = flat(b);
      dbg.insert(dbg.end(), fb_.begin(), fb_.end());
    }
    const double e2 = rel_l2(flat(lg.input_grad), dxw), e3 = rel_l2(dbg, dbw);
    expect(e2 < 1e-5, "learned_gradients input_grad vs oracle", e2);
    expect(e3 < 1e-5, "learned_gradients block_grads vs oracle", e3);
    LearnedButterfly small = LearnedButterfly::from_plan(build_plan(16, 4));
    const std::vector<Complex> M = learned_dense_matrix(small);
    double err = 0;
    for (size_t i = 0; i < 16; ++i)
      for (size_t j = 0; j < 16; ++j)
        err = std::max(err, std::abs(M[i * 16 + j] - std::polar(1.0, -2.0 * M_PI * (double)((i * j) % 16) / 16.0)));
    expect(err < 1e-5, "learned_dense_matrix(from_plan) == DFT matrix", err);
  }
  {  // three-pass: d_k and the circular convolution vs the oracle, three sweeps
    const size_t n = 4096, l = 256, m = 16;
    const ComplexSeq k = cplx(41, n), u = cplx(42, n);
    ThreePassPlan tp = build_three_pass(k, l, m);
    std::vector<double> dkw(2 * n), yw(2 * n);
    lco_three_pass_dk(flat(k).data(), n, l, m, dkw.data());
    lco_conv_three_pass(flat(u).data(), flat(k).data(), n, l, m, yw.data());
    const double e0 = rel_l2(flat(tp.d_k), dkw);
    expect(e0 < 1e-5, "build_three_pass d_k vs oracle", e0);
    PassCounter pcount;
    ComplexSeq y = conv_three_pass(tp, u, &pcount);
    const double e1 = rel_l2(flat(y), yw);
    expect(e1 < 1e-5, "conv_three_pass vs oracle", e1);
    expect(pcount.sweeps() == 3, "PassCounter: three sweeps", pcount.sweeps());
    std::vector<size_t> order(m);
    for (size_t a = 0; a < m; ++a) order[a] = m - 1 - a;
    ComplexSeq y2 = conv_three_pass_ordered(tp, u, order);
    expect(flat(y2) == flat(y), "conv_three_pass_ordered: order-independent (bit-identical)");
  }
  for (int mode = 0; mode < 2; ++mode) {  // conv_real_packed
    const size_t N = 512;
    std::vector<double> u(N), k(N), want(N);
    lco_signal_batch(51, 1, 1, N, u.data());
    lco_signal_batch(52, 1, 1, N, k.data());
    for (double& v : u) v = (float)v;
    for (double& v : k) v = (float)v;
    lco_conv_real_packed(u.data(), k.data(), N, mode, want.data());
    std::vector<double> y = conv_real_packed(u, k, mode ? ConvMode::kCausal : ConvMode::kCircular);
    const double e = rel_l2(y, want);
    expect(e < 1e-5, mode ? "conv_real_packed causal vs oracle" : "conv_real_packed circular vs oracle", e);
  }
  std::printf(fails ? "COMPAT FAIL\n" : "COMPAT OK\n");
  return fails ? 1 : 0;
}
