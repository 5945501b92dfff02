// longconv_b200.hpp — C++ drop-in for the reference `longconv` layer API
// (/root/reference/proj/include/longconv/{types,errors,regularize,butterfly}.hpp),
// implemented on the B200 C ABI (flashbutterfly.h).
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
//   * regularized_long_conv_backward is new: the reference has no backward.
#pragma once

#include <cstddef>
#include <cstdint>
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
