// C-ABI glue around the UNMODIFIED reference `latq` library, compiled in
// place from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libref_latq.so.  TEST INFRASTRUCTURE ONLY: loaded by tests/
// (to pin the C restatement and generate golden fixtures), by
// __graft_entry__.smoke() as a checker, and by bench.py's cpu_baseline /
// `--impl reference` leg as the timed CPU reference.  Never by the product.
//
// Everything here forwards to reference functions; the only restated piece
// is `gen_weights` ("gaussian" branch, proj/core/src/harness.cpp:136-146),
// because harness.cpp needs nlohmann/json + Eigen::rankUpdate which are not
// in this image.  rfft.cpp is compiled unmodified against oracle/shim/fftw3.h
// (FFTW3 is absent: the shim computes the same unnormalized DFT directly).
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "latq/codebook.hpp"
#include "latq/e8p.hpp"
#include "latq/errors.hpp"
#include "latq/hadamard.hpp"
#include "latq/ldlq.hpp"
#include "latq/pipeline.hpp"
#include "latq/rfft.hpp"
#include "latq/rng.hpp"
#include "latq/rvq.hpp"
#include "latq/transforms.hpp"

namespace {

thread_local std::string g_err;

// Error codes mirror the product's q8p_status (include/q8p.h).
int map_exception() {
  try {
    throw;
  } catch (const latq::SizeError& e) {
    g_err = e.what();
    return 1;
  } catch (const latq::ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const latq::BadMagicError& e) {
    g_err = e.what();
    return 4;
  } catch (const latq::UnsupportedVersionError& e) {
    g_err = e.what();
    return 5;
  } catch (const latq::TruncatedArtifactError& e) {
    g_err = e.what();
    return 6;
  } catch (const latq::FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

// harness.cpp:136-146 ("gaussian"): column-major fill, one Box-Muller draw per entry.
Eigen::MatrixXd gen_gaussian(std::size_t m, std::size_t n, std::uint64_t seed) {
  latq::Rng rng(seed);
  Eigen::MatrixXd w(static_cast<Eigen::Index>(m), static_cast<Eigen::Index>(n));
  for (Eigen::Index j = 0; j < w.cols(); ++j)
    for (Eigen::Index i = 0; i < w.rows(); ++i) w(i, j) = rng.gaussian();
  return w;
}

std::vector<std::uint8_t> to_vec(const std::uint8_t* p, std::size_t n) {
  return std::vector<std::uint8_t>(p, p + n);
}

int emit(const std::vector<std::uint8_t>& bytes, std::uint8_t** out, std::size_t* len) {
  *len = bytes.size();
  *out = static_cast<std::uint8_t*>(std::malloc(bytes.size()));
  std::memcpy(*out, bytes.data(), bytes.size());
  return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

std::uint64_t ref_substream_seed(std::uint64_t seed, std::uint64_t stream) {
  return latq::Rng(seed).substream(stream).seed();
}

// gen_weights(m, n, "gaussian", 0, seed) into a ROW-MAJOR m x n buffer.
int ref_gen_weights(std::size_t m, std::size_t n, std::uint64_t seed, double* out) {
  try {
    const Eigen::MatrixXd w = gen_gaussian(m, n, seed);
    for (std::size_t i = 0; i < m; ++i)
      for (std::size_t j = 0; j < n; ++j)
        out[i * n + j] = w(static_cast<Eigen::Index>(i), static_cast<Eigen::Index>(j));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// The full reference producer: quantize_layer(W, H, cfg) (pipeline.cpp:47-107).
// w: row-major m x n; h: row-major n x n (nullptr = identity).
int ref_quantize_layer(const double* w, const double* h, std::uint32_t m, std::uint32_t n,
                       int bits, int transform, std::uint64_t seed, int threads,
                       std::uint8_t** out, std::size_t* len) {
  try {
    Eigen::MatrixXd W(m, n), H(n, n);
    for (std::uint32_t i = 0; i < m; ++i)
      for (std::uint32_t j = 0; j < n; ++j) W(i, j) = w[std::size_t(i) * n + j];
    for (std::uint32_t i = 0; i < n; ++i)
      for (std::uint32_t j = 0; j < n; ++j)
        H(i, j) = h ? h[std::size_t(i) * n + j] : (i == j ? 1.0 : 0.0);
    latq::QuantConfig cfg;
    cfg.bits = bits;
    cfg.transform = static_cast<latq::TransformKind>(transform);
    cfg.seed = seed;
    cfg.threads = threads;
    return emit(latq::serialize(latq::quantize_layer(W, H, cfg).artifact), out, len);
  } catch (...) {
    return map_exception();
  }
}

// The H = I producer route for shapes where quantize_layer's O(n^3) steps
// are infeasible: the same reference calls quantize_layer makes for W
// (transforms.cpp:137-148 W half; pipeline.cpp:71-83 scales;
// ldlq.cpp nearest_round == block_ldlq under an exactly-identity H,
// harness.cpp:416-429).  W = gen_weights(m, n, gaussian, substream(10) of
// `seed`) exactly as `latq quantize` does (latq_cli.cpp:145-148).
int ref_quantize_hi(std::uint32_t m, std::uint32_t n, int bits, int transform, std::uint64_t seed,
                    int threads, std::uint8_t** out, std::size_t* len) {
  try {
    latq::Rng root(seed);
    Eigen::MatrixXd w = gen_gaussian(m, n, root.substream(10).seed());
    const latq::RvqScheme scheme = latq::default_scheme(bits);
    const int g = latq::make_codebook(scheme.front().codebook)->dim();
    if (n % static_cast<std::uint32_t>(g) != 0) throw latq::SizeError("n % 8 != 0");
    latq::Rng sides(seed);
    const bool rht = transform == 0;  // conjugate_layer's make_side (transforms.cpp:137-144)
    const latq::SideTransform left =
        rht ? latq::make_rht_side(m, sides.substream(0)) : latq::make_rfft_side(m, sides.substream(0));
    const latq::SideTransform right =
        rht ? latq::make_rht_side(n, sides.substream(1)) : latq::make_rfft_side(n, sides.substream(1));
    latq::transform_cols(left, w);
    latq::transform_rows(right, w);
    const double r1 = w.norm() / std::sqrt(static_cast<double>(m) * n);
    std::vector<double> scales = latq::stage_scales(scheme, r1);
    std::vector<latq::StageInfo> stages;
    for (std::size_t i = 0; i < scheme.size(); ++i) {
      const float s32 = static_cast<float>(scales[i]);
      stages.push_back({scheme[i].codebook, s32});
      scales[i] = static_cast<double>(s32);
    }
    const latq::RvqQuantizer q(scheme, scales);
    latq::LdlqResult rounded = latq::nearest_round(w, q, g, nullptr, threads);
    latq::QuantizedLinear a;
    a.m = m;
    a.n = n;
    a.transform = rht ? latq::TransformKind::rht : latq::TransformKind::rfft;
    a.stages = std::move(stages);
    if (rht) {
      a.left_signs = left.signs;
      a.right_signs = right.signs;
    } else {
      a.left_phases = left.phases;
      a.right_phases = right.phases;
    }
    a.codes = std::move(rounded.codes);
    return emit(latq::serialize(a), out, len);
  } catch (...) {
    return map_exception();
  }
}

int ref_roundtrip(const std::uint8_t* bytes, std::size_t len, std::uint8_t** out,
                  std::size_t* out_len) {
  try {
    return emit(latq::serialize(latq::deserialize(std::span(bytes, len))), out, out_len);
  } catch (...) {
    return map_exception();
  }
}

int ref_artifact_info(const std::uint8_t* bytes, std::size_t len, std::uint32_t* m,
                      std::uint32_t* n, int* stages) {
  try {
    const latq::QuantizedLinear a = latq::deserialize(std::span(bytes, len));
    *m = a.m;
    *n = a.n;
    *stages = static_cast<int>(a.stages.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// latq::infer on `count` vectors (row-major count x n) -> y (count x m).
// threads > 1: std::threads over vectors on the shared const artifact
// (re-entrant per SPEC.md:489), as BASELINE.md §3 plans.
int ref_infer(const std::uint8_t* bytes, std::size_t len, const double* x, int count,
              double* y, int threads) {
  try {
    const latq::QuantizedLinear a = latq::deserialize(std::span(bytes, len));
    auto run = [&](int begin, int end) {
      for (int i = begin; i < end; ++i) {
        Eigen::VectorXd xv(a.n);
        std::memcpy(xv.data(), x + std::size_t(i) * a.n, sizeof(double) * a.n);
        const Eigen::VectorXd yv = latq::infer(a, xv);
        std::memcpy(y + std::size_t(i) * a.m, yv.data(), sizeof(double) * a.m);
      }
    };
    if (threads <= 1 || count <= 1) {
      run(0, count);
    } else {
      std::vector<std::thread> pool;
      std::exception_ptr err;
      std::mutex mu;
      const int t = std::min(threads, count);
      for (int k = 0; k < t; ++k)
        pool.emplace_back([&, k] {
          try {
            run(count * k / t, count * (k + 1) / t);
          } catch (...) {
            std::scoped_lock l(mu);
            err = std::current_exception();
          }
        });
      for (auto& th : pool) th.join();
      if (err) std::rethrow_exception(err);
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// dequantize_layer -> row-major m x n.
int ref_dequantize(const std::uint8_t* bytes, std::size_t len, double* w) {
  try {
    const latq::QuantizedLinear a = latq::deserialize(std::span(bytes, len));
    const Eigen::MatrixXd d = latq::dequantize_layer(a);
    for (std::uint32_t i = 0; i < a.m; ++i)
      for (std::uint32_t j = 0; j < a.n; ++j) w[std::size_t(i) * a.n + j] = d(i, j);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Unscaled incoherent-domain decode of one stage -> row-major m x n
// (codebook decode of codes[stage][r*nb+k], pipeline.cpp:128-135 without scale).
int ref_decode_stage(const std::uint8_t* bytes, std::size_t len, int stage, double* w) {
  try {
    const latq::QuantizedLinear a = latq::deserialize(std::span(bytes, len));
    const auto cb = latq::make_codebook(a.stages.at(stage).codebook);
    const std::size_t nb = a.n / 8;
    std::vector<double> p(8);
    for (std::size_t r = 0; r < a.m; ++r)
      for (std::size_t k = 0; k < nb; ++k) {
        cb->decode(a.codes[stage][r * nb + k], p);
        for (int c = 0; c < 8; ++c) w[r * a.n + k * 8 + c] = p[c];
      }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_e8p_decode(std::uint16_t word, double* out8) {
  try {
    latq::e8p_decode(latq::e8p_tables(), word, std::span<double>(out8, 8));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_e8p_encode(const double* v8, std::uint16_t* word) {
  try {
    *word = latq::e8p_encode(latq::e8p_tables(), std::span<const double>(v8, 8));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_e8p_tables(std::int8_t* doubled /*256*8*/, std::uint8_t* odd_parity /*256*/) {
  const latq::E8PTables& t = latq::e8p_tables();
  for (int i = 0; i < 256; ++i) {
    for (int c = 0; c < 8; ++c) doubled[i * 8 + c] = t.doubled[i][c];
    odd_parity[i] = t.odd_parity[i];
  }
  return 0;
}

int ref_codebook_decode(const char* id, std::uint32_t code, double* out, int* dim) {
  try {
    const auto cb = latq::make_codebook(id);
    *dim = cb->dim();
    cb->decode(code, std::span<double>(out, static_cast<std::size_t>(cb->dim())));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_plan_hadamard(std::size_t n, std::size_t* p, std::size_t* q) {
  try {
    const latq::HadamardSpec s = latq::plan_hadamard(n);
    *p = s.p;
    *q = s.q;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_hadamard_base(std::size_t q, std::int8_t* out) {
  try {
    const latq::HadamardBase& b = latq::hadamard_base(q);
    std::memcpy(out, b.entries.data(), q * q);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_had_apply(std::size_t n, double* x, int transpose) {
  try {
    latq::had_apply(latq::plan_hadamard(n), std::span<double>(x, n), transpose != 0);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// SideTransform apply / apply_transpose for an rht side built from raw sign bytes.
int ref_side_apply(std::size_t n, const std::uint8_t* sign_bytes, double* x, int transpose) {
  try {
    latq::SideTransform side;
    side.kind = latq::TransformKind::rht;
    side.n = n;
    side.spec = latq::plan_hadamard(n);
    side.signs = latq::SignVector::from_bytes(n, std::span(sign_bytes, (n + 7) / 8));
    if (transpose)
      side.apply_transpose(std::span<double>(x, n));
    else
      side.apply(std::span<double>(x, n));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// RvqQuantizer(default_scheme(bits), scales).quantize on `count` 8-vectors
// (rvq.cpp:59-79) -> codes [stage][count].
int ref_rvq_quantize(int bits, const double* scales, const double* v, std::size_t count, std::uint16_t* codes) {
  try {
    const latq::RvqScheme scheme = latq::default_scheme(bits);
    const latq::RvqQuantizer q(scheme, std::vector<double>(scales, scales + scheme.size()));
    std::vector<double> out(8);
    std::vector<std::uint16_t> w(scheme.size());
    for (std::size_t i = 0; i < count; ++i) {
      q.quantize(std::span<const double>(v + 8 * i, 8), out, w.data(), i);
      for (std::size_t s = 0; s < scheme.size(); ++s) codes[s * count + i] = w[s];
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// rfft_apply (rfft.cpp:39-71) on one vector with the given n/2 phases.
int ref_rfft_apply(std::size_t n, const double* phases, double* x, int transpose) {
  try {
    latq::PhaseVector p;
    p.length = n;
    p.phases.assign(phases, phases + n / 2);
    latq::rfft_apply(p, std::span<double>(x, n), transpose != 0);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Random PhaseVector(length) drawn from Rng(seed) (bitpack.cpp:42-53).
int ref_random_phases(std::size_t n, std::uint64_t seed, double* out) {
  try {
    latq::Rng rng(seed);
    const latq::PhaseVector p = latq::PhaseVector::random(n, rng);
    std::memcpy(out, p.phases.data(), sizeof(double) * p.phases.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Random SignVector(length) drawn from Rng(seed) (bitpack.cpp:11-15).
int ref_random_signs(std::size_t n, std::uint64_t seed, std::uint8_t* out) {
  latq::Rng rng(seed);
  const latq::SignVector s = latq::SignVector::random(n, rng);
  std::memcpy(out, s.bytes().data(), s.byte_size());
  return 0;
}

}  // extern "C"
