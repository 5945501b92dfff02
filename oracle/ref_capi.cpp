// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference
// library (/root/reference/proj, compiled in place by oracle/Makefile into
// oracle/_ref/liblongconv_ref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it.  No reference
// source is copied here: this file only calls the reference's public API.
//
// Every entry returns 0 on success, 1 on DimensionError, 2 on PlanError,
// 3 on any other exception (message via ref_last_error()).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "longconv/butterfly.hpp"
#include "longconv/dft_reference.hpp"
#include "longconv/parallel.hpp"
#include "longconv/regularize.hpp"
#include "longconv/rng.hpp"
#include "longconv/three_pass.hpp"

using namespace longconv;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 1;
  } catch (const PlanError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

ComplexSeq load_c(const double* p, std::size_t n) {
  ComplexSeq v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = Complex(p[2 * i], p[2 * i + 1]);
  return v;
}
void store_c(const ComplexSeq& v, double* p) {
  for (std::size_t i = 0; i < v.size(); ++i) {
    p[2 * i] = v[i].real();
    p[2 * i + 1] = v[i].imag();
  }
}
RegularizationConfig make_cfg(double lambda, std::size_t p, double rate, int domain,
                              std::uint64_t seed) {
  RegularizationConfig c;
  c.lambda = lambda;
  c.smooth_width = p;
  c.dropout_rate = rate;
  c.smooth_domain = domain ? SmoothDomain::kFrequency : SmoothDomain::kTime;
  c.seed = seed;
  return c;
}
KernelBank make_bank(const double* K, const double* D, std::size_t H, std::size_t N) {
  KernelBank bank(H, N);
  std::memcpy(bank.kernels.data(), K, sizeof(double) * H * N);
  std::memcpy(bank.skip_gain.data(), D, sizeof(double) * H);
  return bank;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// SeededRng(seed).child(stream) -> count standard normals (rng.cpp:35-69).
int ref_normal_draws(std::uint64_t seed, std::uint64_t stream, std::size_t count,
                     double* out) {
  return guard([&] {
    SeededRng r = SeededRng(seed).child(stream);
    auto v = standard_normal_draws(r, count);
    std::memcpy(out, v.data(), sizeof(double) * count);
  });
}

int ref_uniform_draws(std::uint64_t seed, std::uint64_t stream, std::size_t count,
                      double* out) {
  return guard([&] {
    SeededRng r = SeededRng(seed).child(stream);
    for (std::size_t i = 0; i < count; ++i) out[i] = r.uniform01();
  });
}

// init_kernels (regularize.cpp:73-91). kind 0 random, 1 geometric.
int ref_init_kernels(int kind, std::size_t H, std::size_t N, std::uint64_t seed, double* K,
                     double* D) {
  return guard([&] {
    InitConfig c;
    c.kind = kind ? InitKind::kGeometric : InitKind::kRandom;
    c.heads = H;
    c.len = N;
    c.seed = seed;
    KernelBank b = init_kernels(c);
    std::memcpy(K, b.kernels.data(), sizeof(double) * H * N);
    std::memcpy(D, b.skip_gain.data(), sizeof(double) * H);
  });
}

int ref_squash(const double* k, std::size_t n, double lambda, double* out) {
  return guard([&] {
    auto v = squash({k, n}, lambda);
    std::memcpy(out, v.data(), sizeof(double) * n);
  });
}
int ref_smooth(const double* k, std::size_t n, std::size_t p, double* out) {
  return guard([&] {
    auto v = smooth({k, n}, p);
    std::memcpy(out, v.data(), sizeof(double) * n);
  });
}
int ref_smooth_frequency(const double* k, std::size_t n, std::size_t p, double* out) {
  return guard([&] {
    auto v = smooth_frequency({k, n}, p);
    std::memcpy(out, v.data(), sizeof(double) * n);
  });
}

// regularize_bank (regularize.cpp:93-107).
int ref_regularize_bank(const double* K, const double* D, std::size_t H, std::size_t N,
                        double lambda, std::size_t p, double rate, int domain,
                        std::uint64_t seed, int training, double* Kout) {
  return guard([&] {
    KernelBank b = make_bank(K, D, H, N);
    KernelBank r = regularize_bank(b, make_cfg(lambda, p, rate, domain, seed), training != 0);
    std::memcpy(Kout, r.kernels.data(), sizeof(double) * H * N);
  });
}

// regularized_long_conv (regularize.cpp:149-190). engine 0 naive, 1 butterfly,
// 2 three-pass; mode 0 circular, 1 causal.
int ref_regularized_long_conv(const double* u, std::size_t B, std::size_t H, std::size_t N,
                              const double* K, const double* D, double lambda,
                              std::size_t p, double rate, int domain, std::uint64_t seed,
                              int engine, int mode, int training, int threads, double* y) {
  return guard([&] {
    SignalBatch sb(B, H, N);
    std::memcpy(sb.data.data(), u, sizeof(double) * B * H * N);
    KernelBank bank = make_bank(K, D, H, N);
    const Engine e = engine == 0 ? Engine::kNaive
                     : engine == 1 ? Engine::kButterfly
                                   : Engine::kThreePass;
    SignalBatch out =
        regularized_long_conv(sb, bank, make_cfg(lambda, p, rate, domain, seed), e,
                              mode ? ConvMode::kCausal : ConvMode::kCircular,
                              training != 0, threads);
    std::memcpy(y, out.data.data(), sizeof(double) * B * H * N);
  });
}

// Backward of the layer, COMPOSED from reference forward primitives (the
// reference has no backward):
//   du[b,h] = R(conv(R(dy[b,h]), Kbar[h])) + D[h] dy[b,h]
//   dKbar[h] = sum_b R(conv(R(dy[b,h]), u[b,h]))
//   dD[h] = sum dy*u
// R = time reversal; conv = conv_butterfly causal (butterfly.cpp:187-210).
// Kbar is the regularized bank (regularize_bank).  dK returned here is
// dKbar (w.r.t. the REGULARIZED kernel); the chain through squash/smooth is
// applied by ref_regularizer_backward.  Causal mode only.
int ref_long_conv_backward(const double* u, const double* dy, std::size_t B, std::size_t H,
                           std::size_t N, const double* Kbar, const double* D, int threads,
                           double* du, double* dKbar, double* dD) {
  return guard([&] {
    const ButterflyPlan plan = build_plan(2 * N, 16);
    parallel_for(B * H, threads, [&](std::size_t task) {
      const std::size_t b = task / H, h = task % H;
      const double* dyc = dy + (b * H + h) * N;
      ComplexSeq rdy(N), kk(N);
      for (std::size_t i = 0; i < N; ++i) {
        rdy[i] = Complex(dyc[N - 1 - i], 0.0);
        kk[i] = Complex(Kbar[h * N + i], 0.0);
      }
      ComplexSeq c = conv_butterfly(rdy, kk, plan, ConvMode::kCausal);
      double* duc = du + (b * H + h) * N;
      for (std::size_t i = 0; i < N; ++i) duc[i] = c[N - 1 - i].real() + D[h] * dyc[i];
    });
    parallel_for(H, threads, [&](std::size_t h) {
      std::vector<double> acc(N, 0.0);
      double dd = 0.0;
      for (std::size_t b = 0; b < B; ++b) {
        const double* dyc = dy + (b * H + h) * N;
        const double* uc = u + (b * H + h) * N;
        ComplexSeq rdy(N), uu(N);
        for (std::size_t i = 0; i < N; ++i) {
          rdy[i] = Complex(dyc[N - 1 - i], 0.0);
          uu[i] = Complex(uc[i], 0.0);
          dd += dyc[i] * uc[i];
        }
        ComplexSeq c = conv_butterfly(rdy, uu, plan, ConvMode::kCausal);
        for (std::size_t i = 0; i < N; ++i) acc[i] += c[N - 1 - i].real();
      }
      std::memcpy(dKbar + h * N, acc.data(), sizeof(double) * N);
      dD[h] = dd;
    });
  });
}

// Chain rule through regularize_bank (time-domain smooth, eval or training):
// dK = dropmask/(1-rate) * smooth(1[|smooth(drop K)| > lambda] * dKbar, p).
// smooth() is a symmetric zero-padded band, so it is self-adjoint.
int ref_regularizer_backward(const double* K, std::size_t H, std::size_t N, double lambda,
                             std::size_t p, double rate, std::uint64_t seed, int training,
                             const double* dKbar, double* dK) {
  return guard([&] {
    const SeededRng base(seed);
    for (std::size_t h = 0; h < H; ++h) {
      SeededRng stream = base.child(h);
      std::vector<double> ones(N, 1.0);
      // dropout mask from the same stream regularize_bank uses.
      std::vector<double> mask = kernel_dropout(ones, rate, stream, training != 0);
      std::vector<double> dk(K + h * N, K + (h + 1) * N);
      for (std::size_t i = 0; i < N; ++i) dk[i] *= mask[i];
      std::vector<double> s = smooth(dk, p);
      std::vector<double> g(N);
      for (std::size_t i = 0; i < N; ++i)
        g[i] = (std::abs(s[i]) > lambda) ? dKbar[h * N + i] : 0.0;
      std::vector<double> sg = smooth(g, p);
      for (std::size_t i = 0; i < N; ++i) dK[h * N + i] = sg[i] * mask[i];
    }
  });
}

// build_plan stage factors (butterfly.cpp:72-118).
int ref_plan_factors(std::size_t n, std::size_t r, std::size_t* factors, std::size_t* count) {
  return guard([&] {
    ButterflyPlan p = build_plan(n, r);
    *count = p.stages.size();
    for (std::size_t i = 0; i < p.stages.size(); ++i) factors[i] = p.stages[i].factor;
  });
}

// apply_plan (butterfly.cpp:173-185). dir 0 forward, 1 inverse. Interleaved complex.
int ref_apply_plan(std::size_t n, std::size_t r, const double* x, int dir, double* y) {
  return guard([&] {
    ButterflyPlan p = build_plan(n, r);
    store_c(apply_plan(p, load_c(x, n), dir ? Direction::kInverse : Direction::kForward), y);
  });
}

int ref_dft_naive(const double* x, std::size_t n, int inverse, double* y) {
  return guard([&] {
    ComplexSeq v = load_c(x, n);
    store_c(inverse ? idft_naive(v) : dft_naive(v), y);
  });
}

// conv_butterfly (butterfly.cpp:187-210), complex interleaved, length-N inputs.
int ref_conv_butterfly(const double* u, const double* k, std::size_t N, int mode, double* y) {
  return guard([&] {
    const ConvMode m = mode ? ConvMode::kCausal : ConvMode::kCircular;
    ButterflyPlan p = build_plan(mode ? 2 * N : N, 16);
    store_c(conv_butterfly(load_c(u, N), load_c(k, N), p, m), y);
  });
}

int ref_conv_naive_real(const double* u, const double* k, std::size_t N, int mode,
                        double* y) {
  return guard([&] {
    auto v = mode ? conv_causal_naive_real({u, N}, {k, N})
                  : conv_circular_naive_real({u, N}, {k, N});
    std::memcpy(y, v.data(), sizeof(double) * N);
  });
}

// build_three_pass + conv_three_pass (three_pass.cpp:183-288): circular conv
// of length n = l*m; also returns the pass-counter sweeps.
int ref_conv_three_pass(const double* u, const double* k, std::size_t n, std::size_t l,
                        std::size_t m, double* y, int* sweeps) {
  return guard([&] {
    ThreePassPlan plan = build_three_pass(load_c(k, n), l, m);
    PassCounter pc(n);
    store_c(conv_three_pass(plan, load_c(u, n), &pc), y);
    if (sweeps) *sweeps = pc.sweeps();
  });
}

// d_k layout of build_three_pass (three_pass.cpp:197-203).
int ref_three_pass_dk(const double* k, std::size_t n, std::size_t l, std::size_t m,
                      double* dk) {
  return guard([&] {
    ThreePassPlan plan = build_three_pass(load_c(k, n), l, m);
    store_c(plan.d_k, dk);
  });
}

// conv_real_packed (three_pass.cpp:356-371).
int ref_conv_real_packed(const double* u, const double* k, std::size_t N, int mode,
                         double* y) {
  return guard([&] {
    auto v = conv_real_packed({u, N}, {k, N}, mode ? ConvMode::kCausal : ConvMode::kCircular);
    std::memcpy(y, v.data(), sizeof(double) * N);
  });
}

// Learned butterfly (butterfly.cpp:221-307). blocks: concatenated per-stage
// factor x factor complex matrices (interleaved), stages of build_plan(n, r).
static LearnedButterfly make_lb(std::size_t n, std::size_t r, const double* blocks) {
  LearnedButterfly lb = LearnedButterfly::from_plan(build_plan(n, r));
  std::size_t off = 0;
  for (auto& blk : lb.blocks) {
    for (std::size_t i = 0; i < blk.size(); ++i)
      blk[i] = Complex(blocks[2 * (off + i)], blocks[2 * (off + i) + 1]);
    off += blk.size();
  }
  return lb;
}

int ref_learned_param_count(std::size_t n, std::size_t r, std::size_t* count) {
  return guard([&] {
    *count = LearnedButterfly::from_plan(build_plan(n, r)).parameter_count();
  });
}

// Writes the DFT-initialized blocks (from_plan).
int ref_learned_init(std::size_t n, std::size_t r, double* blocks) {
  return guard([&] {
    LearnedButterfly lb = LearnedButterfly::from_plan(build_plan(n, r));
    std::size_t off = 0;
    for (auto& blk : lb.blocks) {
      for (std::size_t i = 0; i < blk.size(); ++i) {
        blocks[2 * (off + i)] = blk[i].real();
        blocks[2 * (off + i) + 1] = blk[i].imag();
      }
      off += blk.size();
    }
  });
}

int ref_learned_forward(std::size_t n, std::size_t r, const double* blocks, const double* x,
                        double* y) {
  return guard([&] {
    LearnedButterfly lb = make_lb(n, r, blocks);
    store_c(learned_forward(lb, load_c(x, n)), y);
  });
}

int ref_learned_gradients(std::size_t n, std::size_t r, const double* blocks, const double* x,
                          const double* g, double* dblocks, double* dx) {
  return guard([&] {
    LearnedButterfly lb = make_lb(n, r, blocks);
    LearnedGradients lg = learned_gradients(lb, load_c(x, n), load_c(g, n));
    std::size_t off = 0;
    for (auto& blk : lg.block_grads) {
      for (std::size_t i = 0; i < blk.size(); ++i) {
        dblocks[2 * (off + i)] = blk[i].real();
        dblocks[2 * (off + i) + 1] = blk[i].imag();
      }
      off += blk.size();
    }
    store_c(lg.input_grad, dx);
  });
}

int ref_hardware_threads(void) { return hardware_threads(); }

}  // extern "C"
