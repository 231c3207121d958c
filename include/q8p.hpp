// q8p C++ host API: the reference `latq` inference-path types and functions
// (namespace latq, core/include/latq/{pipeline,bitpack,hadamard,errors}.hpp)
// restated without Eigen, backed by the sm_100a kernels behind the C ABI in
// q8p.h.  Same field layout, same QSHP v1 bytes, same error taxonomy.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "q8p.h"

namespace q8p {

// Error taxonomy of core/include/latq/errors.hpp:9-53 plus device failures.
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class SizeError : public Error {
 public:
  using Error::Error;
};
class ValidationError : public Error {
 public:
  using Error::Error;
};
class FormatError : public Error {
 public:
  using Error::Error;
};
class BadMagicError : public FormatError {
 public:
  using FormatError::FormatError;
};
class UnsupportedVersionError : public FormatError {
 public:
  using FormatError::FormatError;
};
class TruncatedArtifactError : public FormatError {
 public:
  using FormatError::FormatError;
};
class UnsupportedError : public Error {  // valid artifact, not on this path (e.g. > 2 RVQ stages)
 public:
  using Error::Error;
};
class DeviceError : public Error {  // CUDA / NCCL failures
 public:
  using Error::Error;
};
class NcclError : public DeviceError {  // NCCL failures (Q8P_ERR_NCCL)
 public:
  using DeviceError::DeviceError;
};

// Throws the typed exception for a non-OK status (message: q8p_last_error()).
void throw_status(q8p_status s);
inline void check(q8p_status s) {
  if (s != Q8P_OK) throw_status(s);
}

inline constexpr std::uint16_t kFormatVersion = 1;  // version.hpp:10

enum class TransformKind : std::uint8_t { rht = 0, rfft = 1 };  // transforms.hpp:14-17

// +-1 diagonal, 1 bit per entry, LSB-first, bit set = -1 (bitpack.hpp:11-41).
class SignVector {
 public:
  SignVector() = default;
  explicit SignVector(std::size_t length) : length_(length), bytes_((length + 7) / 8, 0) {}
  static SignVector from_bytes(std::size_t length, std::span<const std::uint8_t> bytes);

  std::size_t size() const { return length_; }
  std::size_t byte_size() const { return (length_ + 7) / 8; }
  int get(std::size_t i) const { return (bytes_[i >> 3] >> (i & 7)) & 1 ? -1 : 1; }
  void set(std::size_t i, int sign);
  const std::vector<std::uint8_t>& bytes() const { return bytes_; }
  void apply(std::span<double> x) const;
  bool operator==(const SignVector&) const = default;

 private:
  std::size_t length_ = 0;
  std::vector<std::uint8_t> bytes_;
};

struct StageInfo {  // pipeline.hpp:27-32
  std::string codebook;
  float scale = 1.0f;
  bool operator==(const StageInfo&) const = default;
};

// pipeline.hpp:38-49.  Phases (rfft) are carried as their f32 storage form.
struct QuantizedLinear {
  std::uint16_t version = kFormatVersion;
  std::uint32_t m = 0;
  std::uint32_t n = 0;
  TransformKind transform = TransformKind::rht;
  std::vector<StageInfo> stages;
  SignVector left_signs, right_signs;
  std::vector<float> left_phases, right_phases;
  std::vector<std::vector<std::uint16_t>> codes;  // [stage][row * nb + blk]
  bool operator==(const QuantizedLinear&) const = default;
};

struct HadamardSpec {  // hadamard.hpp:18-22
  std::size_t n = 0, p = 1, q = 1;
};
HadamardSpec plan_hadamard(std::size_t n);

// Codebook ids on this path: "e8p-2bit" (16-bit words) and "e8-1bit" (8-bit).
int codebook_code_bytes(const std::string& id);  // throws ValidationError for others

std::vector<std::uint8_t> serialize(const QuantizedLinear& a);
QuantizedLinear deserialize(std::span<const std::uint8_t> bytes);
std::size_t serialized_size(const QuantizedLinear& a);
double bits_per_weight(const QuantizedLinear& a);
int artifact_block_dim(const QuantizedLinear& a);

// A QuantizedLinear resident on one B200 (or a row shard of one).
class DeviceLayer {
 public:
  DeviceLayer(const QuantizedLinear& a, int device = 0);
  DeviceLayer(std::span<const std::uint8_t> qshp, int device = 0);
  DeviceLayer(std::span<const std::uint8_t> qshp, std::uint32_t row_begin, std::uint32_t row_end,
              int device = 0);
  q8p_layer* get() const { return layer_.get(); }
  q8p_layer_info info() const;
  std::size_t workspace_bytes(int batch) const { return q8p_workspace_bytes(get(), batch); }
  // Device fp32 buffers, stream-ordered (see q8p_forward).
  void forward(const float* x, float* y, int batch, void* workspace, std::size_t ws_bytes,
               void* stream = nullptr) const {
    check(q8p_forward(get(), x, y, batch, workspace, ws_bytes, stream));
  }
  // Host f64, synchronous: the latq::infer calling convention.
  std::vector<double> infer(std::span<const double> x) const;

 private:
  struct Deleter {
    void operator()(q8p_layer* l) const { q8p_layer_destroy(l); }
  };
  std::unique_ptr<q8p_layer, Deleter> layer_;
};

// latq::infer drop-in (pipeline.hpp:73-74): uploads `a`, runs one forward.
// For repeated calls keep a DeviceLayer instead.
std::vector<double> infer(const QuantizedLinear& a, std::span<const double> x);

}  // namespace q8p
