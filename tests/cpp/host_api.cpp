// Host C++ API (include/q8p.hpp) exercised the way a latq caller would use it:
// deserialize / serialize (pipeline.cpp:269-413), typed errors (errors.hpp),
// plan_hadamard, and -- in "gpu" mode -- DeviceLayer::infer / q8p::infer
// against the reference's golden output.  Built and run by
// tests/test_cpp_host_api.py.
//   host_api cpu QSHP
//   host_api gpu QSHP X.f64 Y.f64 COUNT
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "q8p.hpp"

namespace {
int failures = 0;
void expect(bool ok, const char* what) {
  if (!ok) {
    std::fprintf(stderr, "FAIL: %s\n", what);
    ++failures;
  }
}
std::vector<std::uint8_t> read_file(const char* path) {
  std::ifstream f(path, std::ios::binary);
  return std::vector<std::uint8_t>(std::istreambuf_iterator<char>(f), {});
}
template <typename E, typename F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const std::string mode = argv[1];
  const std::vector<std::uint8_t> bytes = read_file(argv[2]);
  const q8p::QuantizedLinear a = q8p::deserialize(bytes);
  expect(q8p::serialize(a) == bytes, "serialize(deserialize(b)) == b");
  expect(q8p::serialized_size(a) == bytes.size(), "serialized_size");
  expect(q8p::artifact_block_dim(a) == 8, "artifact_block_dim");
  expect(std::fabs(q8p::bits_per_weight(a) - 8.0 * double(bytes.size()) / (double(a.m) * a.n)) < 1e-9,
         "bits_per_weight");
  {
    std::vector<std::uint8_t> bad = bytes;
    bad[0] = 'X';
    expect(throws<q8p::BadMagicError>([&] { q8p::deserialize(bad); }), "BadMagicError");
    bad = bytes;
    bad[4] = 2;
    expect(throws<q8p::UnsupportedVersionError>([&] { q8p::deserialize(bad); }), "UnsupportedVersionError");
    expect(throws<q8p::TruncatedArtifactError>(
               [&] { q8p::deserialize(std::span(bytes.data(), bytes.size() - 1)); }),
           "TruncatedArtifactError");
    expect(throws<q8p::FormatError>([&] { q8p::deserialize(std::span(bytes.data(), 3)); }), "FormatError family");
  }
  {
    const q8p::HadamardSpec s = q8p::plan_hadamard(11008);
    expect(s.p == 64 && s.q == 172, "plan_hadamard(11008) = 64 x 172");
    expect(throws<q8p::SizeError>([] { q8p::plan_hadamard(36); }), "plan_hadamard(36) throws SizeError");
  }
  if (mode == "gpu") {
    if (argc < 6) return 2;
    const std::vector<std::uint8_t> xb = read_file(argv[3]), yb = read_file(argv[4]);
    const int count = std::atoi(argv[5]);
    const double* x = reinterpret_cast<const double*>(xb.data());
    const double* y = reinterpret_cast<const double*>(yb.data());
    q8p::DeviceLayer layer(bytes, 0);
    for (int i = 0; i < count; ++i) {
      const std::vector<double> got = layer.infer(std::span(x + std::size_t(i) * a.n, a.n));
      const std::vector<double> got2 = q8p::infer(a, std::span(x + std::size_t(i) * a.n, a.n));
      double num = 0, den = 0;
      for (std::uint32_t r = 0; r < a.m; ++r) {
        const double d = got[r] - y[std::size_t(i) * a.m + r];
        num += d * d;
        den += y[std::size_t(i) * a.m + r] * y[std::size_t(i) * a.m + r];
      }
      expect(std::sqrt(num / den) < 1e-5, "DeviceLayer::infer vs reference golden (rel L2 < 1e-5)");
      expect(got == got2, "q8p::infer == DeviceLayer::infer");
    }
    expect(throws<q8p::SizeError>([&] { layer.infer(std::vector<double>(a.n + 1)); }), "infer size check");
  }
  std::printf("%s: %s\n", mode.c_str(), failures ? "FAILED" : "ok");
  return failures ? 1 : 0;
}
