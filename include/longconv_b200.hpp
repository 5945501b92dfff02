// longconv_b200.hpp — C++ drop-in for the reference `longconv` API
// (/root/reference/proj/include/longconv/{types,errors,regularize,butterfly,
// three_pass}.hpp), implemented on the B200 C ABI (flashbutterfly.h).
//
// A caller of the reference switches by including this header instead of
// "longconv/regularize.hpp" and linking liblongconv_b200.so: the namespace,
// type names, field names, enum values, argument order and exception types
// are the reference's.  Differences (documented, not silent):
//   * arithmetic runs on the GPU in the precision selected by
//     set_device_precision() (default Precision::kFp32, the 1e-5 validation
//     mode; kBf16 / kFp16 use the tensor-core path) instead of fp64;
//   * `threads` is accepted and ignored (the grid is the parallelism);
//   * Engine::kNaive (the O(N^2) oracle) is not offered on the device and
//     throws PlanError;
//   * regularized_long_conv_backward is new: the reference has no backward;
//   * the single-row entry points (apply_plan, conv_butterfly, learned_*,
//     conv_three_pass, conv_real_packed) compute in fp32 on the device; plans
//     keep the reference's descriptive fields (n, r, stage factors / segments /
//     DFT blocks; l, m, inner, d_k) but not its host-side gather / scatter /
//     twiddle tables or the BlockDiagonalButterfly mixers (the device builds
//     its own); PassCounter is filled with the three sweeps the device makes.
#pragma once

#include <array>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace longconv {

// errors.hpp:9-26
struct DimensionError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct PlanError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ConditioningError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// device failure (no reference counterpart: the reference cannot fail here)
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// types.hpp:37-57
struct SignalBatch {
  std::size_t batch = 0;
  std::size_t heads = 0;
  std::size_t len = 0;
  std::vector<double> data;

  SignalBatch() = default;
  SignalBatch(std::size_t b, std::size_t h, std::size_t n)
      : batch(b), heads(h), len(n), data(b * h * n, 0.0) {}
  std::size_t size() const { return batch * heads * len; }
  double* channel(std::size_t b, std::size_t h) { return data.data() + (b * heads + h) * len; }
  const double* channel(std::size_t b, std::size_t h) const {
    return data.data() + (b * heads + h) * len;
  }
};

// types.hpp:60-75
struct KernelBank {
  std::size_t heads = 0;
  std::size_t len = 0;
  std::vector<double> kernels;    // [h][n]
  std::vector<double> skip_gain;  // [h]

  KernelBank() = default;
  KernelBank(std::size_t h, std::size_t n) : heads(h), len(n), kernels(h * n, 0.0), skip_gain(h, 0.0) {}
  double* kernel(std::size_t h) { return kernels.data() + h * len; }
  const double* kernel(std::size_t h) const { return kernels.data() + h * len; }
};

// butterfly.hpp:68-69, regularize.hpp:16-25
enum class ConvMode { kCircular, kCausal };
enum class SmoothDomain { kTime, kFrequency };
enum class Engine { kNaive, kButterfly, kThreePass };

struct RegularizationConfig {
  double lambda = 0.0;
  std::size_t smooth_width = 0;
  double dropout_rate = 0.0;
  SmoothDomain smooth_domain = SmoothDomain::kTime;
  std::uint64_t seed = 0;
};

// regularize.hpp:27-34, 55-59 (init_kernels draws on the device, the
// reference's streams exactly)
enum class InitKind { kRandom, kGeometric };
struct InitConfig {
  InitKind kind = InitKind::kRandom;
  std::size_t heads = 1;
  std::size_t len = 1;
  std::uint64_t seed = 0;
};
KernelBank init_kernels(const InitConfig& cfg);
double geometric_envelope(std::size_t position, std::size_t len, std::size_t head, std::size_t heads);

enum class Precision { kFp32, kBf16, kFp16 };
void set_device_precision(Precision p);
Precision device_precision();
void set_device(int device);

// regularize.hpp:62-63 (computed on the device, returned on the host)
KernelBank regularize_bank(const KernelBank& bank, const RegularizationConfig& cfg, bool training);

// regularize.hpp:67-70
SignalBatch regularized_long_conv(const SignalBatch& u, const KernelBank& bank,
                                  const RegularizationConfig& cfg, Engine engine, ConvMode mode,
                                  bool training = false, int threads = 1);

// Backward of the layer (no reference counterpart).
struct LongConvGradients {
  SignalBatch du;                  // dJ/du
  std::vector<double> dkernels;    // dJ/dK (raw bank), [h][n]
  std::vector<double> dskip_gain;  // dJ/dD, [h]
};
LongConvGradients regularized_long_conv_backward(const SignalBatch& dy, const SignalBatch& u,
                                                 const KernelBank& bank,
                                                 const RegularizationConfig& cfg, Engine engine,
                                                 ConvMode mode, bool training = false);

// ---------------------------------------------------------------- single rows
// types.hpp:12-13
using Complex = std::complex<double>;
using ComplexSeq = std::vector<Complex>;

// butterfly.hpp:52-66 (descriptive fields; the device plan is built once per
// ButterflyPlan and shared by its copies)
struct PlanStage {
  std::size_t factor = 0;
  std::size_t segment = 0;
  std::vector<Complex> dft_block;  // factor x factor, row-major: exp(-2 pi i pq / f)
};
struct ButterflyPlan {
  std::size_t n = 0;
  std::size_t r = 0;
  std::vector<PlanStage> stages;
  std::shared_ptr<void> device;  // fb_dft_plan

  std::size_t stage_count() const { return stages.size(); }
  std::string describe_json() const;  // {"n":..,"r":..,"stage_factors":[..]}
};

enum class Direction { kForward, kInverse };  // butterfly.hpp:68

// butterfly.hpp:74-83
ButterflyPlan build_plan(std::size_t n, std::size_t r);
ComplexSeq apply_plan(const ButterflyPlan& plan, std::span<const Complex> x, Direction dir);
ComplexSeq conv_butterfly(std::span<const Complex> u, std::span<const Complex> k,
                          const ButterflyPlan& plan, ConvMode mode);

// butterfly.hpp:88-108
struct LearnedButterfly {
  ButterflyPlan plan;
  std::vector<std::vector<Complex>> blocks;  // [stage][factor*factor]

  static LearnedButterfly from_plan(const ButterflyPlan& plan);
  std::size_t parameter_count() const;
};
ComplexSeq learned_forward(const LearnedButterfly& lb, std::span<const Complex> x);
struct LearnedGradients {
  std::vector<std::vector<Complex>> block_grads;
  ComplexSeq input_grad;
};
LearnedGradients learned_gradients(const LearnedButterfly& lb, std::span<const Complex> x,
                                   std::span<const Complex> upstream);
std::vector<Complex> learned_dense_matrix(const LearnedButterfly& lb);

// three_pass.hpp:23-58
inline constexpr std::size_t kDefaultWorkingSet = 8192;
class PassCounter {
 public:
  struct Phase {
    std::uint64_t reads = 0;
    std::uint64_t writes = 0;
    std::uint64_t distinct_touched = 0;
    std::size_t working_set_peak = 0;
  };
  explicit PassCounter(std::size_t n = 0, std::size_t working_set_cap = kDefaultWorkingSet)
      : n_(n), cap_(working_set_cap) {}
  void reset(std::size_t n);
  void begin_phase(int phase);  // 1..3
  void record_read(std::size_t index);
  void record_write(std::size_t index);
  void record_working_set(std::size_t elements);
  void merge_counts(std::uint64_t reads, std::uint64_t writes);
  std::size_t buffer_len() const { return n_; }
  std::size_t working_set_cap() const { return cap_; }
  const std::array<Phase, 3>& phases() const { return phases_; }
  int sweeps() const;
  std::string report_json() const;

 private:
  void touch(std::size_t index);
  std::size_t n_ = 0;
  std::size_t cap_ = 0;
  int current_ = -1;
  std::array<Phase, 3> phases_{};
  std::vector<std::uint8_t> seen_;  // phase (1..3) that last touched each element
};

// three_pass.hpp:100-120 (the mixers are not materialised on the host)
struct ThreePassPlan {
  std::size_t n = 0;
  std::size_t l = 0;
  std::size_t m = 0;
  ButterflyPlan inner;  // length-l plan of the middle pass
  ComplexSeq d_k;       // d_k[a l + tau] = l K_hat[tau m + a]
  ComplexSeq k_hat;     // K_hat = F_n k (natural order; the device multiplies by it)
  std::shared_ptr<void> device;  // fb_dft_plan of length n
};
ThreePassPlan build_three_pass(std::span<const Complex> kernel, std::size_t l, std::size_t m,
                               std::size_t inner_r = 16);
ComplexSeq conv_three_pass(const ThreePassPlan& plan, std::span<const Complex> u,
                           PassCounter* counter = nullptr, int threads = 1);
ComplexSeq conv_three_pass_ordered(const ThreePassPlan& plan, std::span<const Complex> u,
                                   std::span<const std::size_t> block_order,
                                   PassCounter* counter = nullptr);
// three_pass.hpp:128-131
std::vector<double> conv_real_packed(std::span<const double> u, std::span<const double> k,
                                     ConvMode mode);

// Learned butterfly, batched per head (butterfly.hpp:88-108).  blocks: per
// head the concatenated stage blocks of build_plan(n, r) (interleaved re/im
// doubles, [H][2P]); x, g: [B][H][n] interleaved complex.
struct LearnedBatchGradients {
  std::vector<double> block_grads;  // [H][2P], summed over the batch
  std::vector<double> input_grad;   // [B][H][2n]
};
std::vector<double> learned_forward_batched(std::size_t n, std::size_t r, std::size_t B,
                                            std::size_t H, const std::vector<double>& blocks,
                                            const std::vector<double>& x);
LearnedBatchGradients learned_gradients_batched(std::size_t n, std::size_t r, std::size_t B,
                                                std::size_t H, const std::vector<double>& blocks,
                                                const std::vector<double>& x,
                                                const std::vector<double>& upstream);

}  // namespace longconv
