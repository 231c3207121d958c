// Host side of the drop-in: QuantizedLinear, SignVector and the QSHP v1
// artifact reader/writer, byte-compatible with the reference
// (core/src/pipeline.cpp:200-413, core/src/bitpack.cpp:16-40), plus the
// DeviceLayer / infer wrappers over the C ABI.
#include <bit>
#include <cstring>

#include "internal.hpp"

namespace q8p {

// ---- SignVector (bitpack.cpp) --------------------------------------------
SignVector SignVector::from_bytes(std::size_t length, std::span<const std::uint8_t> bytes) {
  SignVector s(length);
  if (bytes.size() != s.byte_size()) throw SizeError("SignVector::from_bytes: byte count mismatch");
  std::copy(bytes.begin(), bytes.end(), s.bytes_.begin());
  if (length % 8 != 0) s.bytes_.back() &= static_cast<std::uint8_t>((1u << (length % 8)) - 1);
  return s;
}

void SignVector::set(std::size_t i, int sign) {
  const auto mask = static_cast<std::uint8_t>(1u << (i & 7));
  if (sign < 0)
    bytes_[i >> 3] |= mask;
  else
    bytes_[i >> 3] &= static_cast<std::uint8_t>(~mask);
}

void SignVector::apply(std::span<double> x) const {
  if (x.size() != length_) throw SizeError("SignVector::apply: length mismatch");
  for (std::size_t i = 0; i < length_; ++i)
    if ((bytes_[i >> 3] >> (i & 7)) & 1) x[i] = -x[i];
}

// ---- QSHP v1 -------------------------------------------------------------
int codebook_code_bytes(const std::string& id) {
  if (id == "e8p-2bit") return 2;
  if (id == "e8-1bit") return 1;
  throw ValidationError("unknown codebook id '" + id + "'");
}

int artifact_block_dim(const QuantizedLinear& a) {
  if (a.stages.empty()) throw ValidationError("artifact has no quantization stages");
  codebook_code_bytes(a.stages.front().codebook);  // validates the id
  return 8;  // both codebooks on this path are 8-dimensional
}

namespace {

constexpr char kMagic[4] = {'Q', 'S', 'H', 'P'};

struct Writer {
  std::vector<std::uint8_t>& out;
  void u8(std::uint8_t v) { out.push_back(v); }
  void u16(std::uint16_t v) {
    u8(static_cast<std::uint8_t>(v));
    u8(static_cast<std::uint8_t>(v >> 8));
  }
  void u32(std::uint32_t v) {
    for (int i = 0; i < 4; ++i) u8(static_cast<std::uint8_t>(v >> (8 * i)));
  }
  void f32(float v) { u32(std::bit_cast<std::uint32_t>(v)); }
  void bytes(std::span<const std::uint8_t> b) { out.insert(out.end(), b.begin(), b.end()); }
};

struct Reader {
  std::span<const std::uint8_t> in;
  std::size_t pos = 0;
  std::span<const std::uint8_t> take(std::size_t n) {
    if (pos + n > in.size())
      throw TruncatedArtifactError("artifact ends after " + std::to_string(in.size()) + " bytes");
    auto s = in.subspan(pos, n);
    pos += n;
    return s;
  }
  std::uint8_t u8() { return take(1)[0]; }
  std::uint16_t u16() {
    auto b = take(2);
    return static_cast<std::uint16_t>(b[0] | (b[1] << 8));
  }
  std::uint32_t u32() {
    auto b = take(4);
    return std::uint32_t(b[0]) | (std::uint32_t(b[1]) << 8) | (std::uint32_t(b[2]) << 16) |
           (std::uint32_t(b[3]) << 24);
  }
  float f32() { return std::bit_cast<float>(u32()); }
};

}  // namespace

std::size_t serialized_size(const QuantizedLinear& a) {
  std::size_t total = 16;
  for (const StageInfo& st : a.stages) total += 1 + st.codebook.size() + 4;
  if (a.transform == TransformKind::rht)
    total += (a.m + 7) / 8 + (a.n + 7) / 8;
  else
    total += 4 * (std::size_t(a.m) / 2 + std::size_t(a.n) / 2);
  artifact_block_dim(a);
  const std::size_t words = std::size_t(a.m) * (a.n / 8);
  for (const StageInfo& st : a.stages) total += words * codebook_code_bytes(st.codebook);
  return total;
}

double bits_per_weight(const QuantizedLinear& a) {
  if (a.m == 0 || a.n == 0) throw SizeError("bits_per_weight: empty artifact");
  return 8.0 * double(serialized_size(a)) / (double(a.m) * double(a.n));
}

std::vector<std::uint8_t> serialize(const QuantizedLinear& a) {
  std::vector<std::uint8_t> out;
  out.reserve(serialized_size(a));
  Writer w{out};
  w.bytes(std::span(reinterpret_cast<const std::uint8_t*>(kMagic), 4));
  w.u16(a.version);
  w.u32(a.m);
  w.u32(a.n);
  w.u8(static_cast<std::uint8_t>(a.transform));
  if (a.stages.size() > 255) throw ValidationError("serialize: too many stages");
  w.u8(static_cast<std::uint8_t>(a.stages.size()));
  for (const StageInfo& st : a.stages) {
    if (st.codebook.size() > 255) throw ValidationError("serialize: codebook id too long");
    w.u8(static_cast<std::uint8_t>(st.codebook.size()));
    w.bytes(std::span(reinterpret_cast<const std::uint8_t*>(st.codebook.data()), st.codebook.size()));
    w.f32(st.scale);
  }
  if (a.transform == TransformKind::rht) {
    if (a.left_signs.size() != a.m || a.right_signs.size() != a.n)
      throw SizeError("serialize: sign vector lengths disagree with m, n");
    w.bytes(a.left_signs.bytes());
    w.bytes(a.right_signs.bytes());
  } else {
    if (a.left_phases.size() != a.m / 2 || a.right_phases.size() != a.n / 2)
      throw SizeError("serialize: phase lengths disagree with m, n");
    for (float p : a.left_phases) w.f32(p);
    for (float p : a.right_phases) w.f32(p);
  }
  artifact_block_dim(a);
  const std::size_t words = std::size_t(a.m) * (a.n / 8);
  for (std::size_t s = 0; s < a.stages.size(); ++s) {
    if (a.codes[s].size() != words) throw SizeError("serialize: codeword count mismatch");
    const int bytes = codebook_code_bytes(a.stages[s].codebook);
    for (std::uint16_t word : a.codes[s]) {
      w.u8(static_cast<std::uint8_t>(word));
      if (bytes == 2) w.u8(static_cast<std::uint8_t>(word >> 8));
    }
  }
  return out;
}

QuantizedLinear deserialize(std::span<const std::uint8_t> bytes) {
  Reader r{bytes};
  if (std::memcmp(r.take(4).data(), kMagic, 4) != 0) throw BadMagicError("artifact does not start with QSHP");
  QuantizedLinear a;
  a.version = r.u16();
  if (a.version != kFormatVersion)
    throw UnsupportedVersionError("artifact format version " + std::to_string(a.version) +
                                  " (supported: " + std::to_string(kFormatVersion) + ")");
  a.m = r.u32();
  a.n = r.u32();
  const std::uint8_t kind = r.u8();
  if (kind > 1) throw FormatError("artifact: unknown transform kind");
  a.transform = static_cast<TransformKind>(kind);
  const std::uint8_t n_stages = r.u8();
  if (n_stages == 0) throw FormatError("artifact: zero stages");
  for (std::size_t s = 0; s < n_stages; ++s) {
    StageInfo st;
    const auto id = r.take(r.u8());
    st.codebook.assign(reinterpret_cast<const char*>(id.data()), id.size());
    st.scale = r.f32();
    a.stages.push_back(std::move(st));
  }
  if (a.transform == TransformKind::rht) {
    a.left_signs = SignVector::from_bytes(a.m, r.take((a.m + 7) / 8));
    a.right_signs = SignVector::from_bytes(a.n, r.take((a.n + 7) / 8));
  } else {
    if (a.m % 2 != 0 || a.n % 2 != 0) throw FormatError("artifact: phase transform needs even m and n");
    a.left_phases.resize(a.m / 2);
    a.right_phases.resize(a.n / 2);
    for (float& p : a.left_phases) p = r.f32();
    for (float& p : a.right_phases) p = r.f32();
  }
  artifact_block_dim(a);  // validates the first codebook id
  if (a.n % 8 != 0) throw FormatError("artifact: n not divisible by codeword dimension");
  const std::size_t words = std::size_t(a.m) * (a.n / 8);
  for (std::size_t s = 0; s < n_stages; ++s) {
    const int nbytes = codebook_code_bytes(a.stages[s].codebook);
    const auto raw = r.take(words * nbytes);
    std::vector<std::uint16_t> codes(words);
    if (nbytes == 2)
      for (std::size_t i = 0; i < words; ++i) codes[i] = std::uint16_t(raw[2 * i] | (raw[2 * i + 1] << 8));
    else
      for (std::size_t i = 0; i < words; ++i) codes[i] = raw[i];
    a.codes.push_back(std::move(codes));
  }
  if (r.pos != bytes.size()) throw FormatError("artifact: trailing bytes after payload");
  return a;
}

// ---- exceptions <-> status ------------------------------------------------
void throw_status(q8p_status s) {
  const std::string msg = q8p_last_error();
  switch (s) {
    case Q8P_OK:
      return;
    case Q8P_ERR_SIZE:
      throw SizeError(msg);
    case Q8P_ERR_VALIDATION:
      throw ValidationError(msg);
    case Q8P_ERR_FORMAT:
      throw FormatError(msg);
    case Q8P_ERR_BAD_MAGIC:
      throw BadMagicError(msg);
    case Q8P_ERR_UNSUPPORTED_VERSION:
      throw UnsupportedVersionError(msg);
    case Q8P_ERR_TRUNCATED:
      throw TruncatedArtifactError(msg);
    case Q8P_ERR_UNSUPPORTED:
      throw UnsupportedError(msg);
    case Q8P_ERR_NCCL:
      throw NcclError(msg);
    case Q8P_ERR_CUDA:
      throw DeviceError(msg);
    default:
      throw Error(msg);
  }
}

// ---- DeviceLayer -----------------------------------------------------------
namespace {
q8p_layer* make_from(const QuantizedLinear& a, int device) {
  // the checks decode_incoherent / serialize make (pipeline.cpp:116-117, 126-127)
  if (a.codes.size() != a.stages.size()) throw FormatError("artifact: stage/code count mismatch");
  if (a.n % 8 != 0) throw FormatError("artifact: n not divisible by codeword dimension");
  for (const auto& c : a.codes)
    if (c.size() != std::size_t(a.m) * (a.n / 8)) throw FormatError("artifact: codeword count mismatch");
  std::vector<q8p_stage_desc> st(a.stages.size());
  for (std::size_t s = 0; s < st.size(); ++s) {
    st[s].codebook = a.stages[s].codebook == "e8p-2bit" ? Q8P_CB_E8P_2BIT : Q8P_CB_E8_1BIT;
    codebook_code_bytes(a.stages[s].codebook);
    st[s].scale = a.stages[s].scale;
    st[s].codes = a.codes.at(s).data();
    st[s].code_bytes = 2;
  }
  q8p_layer_desc d{};
  d.m = a.m;
  d.n = a.n;
  d.transform = a.transform == TransformKind::rht ? 0 : 1;
  d.num_stages = static_cast<int>(st.size());
  d.stages = st.data();
  if (a.transform == TransformKind::rht) {
    d.signs_u = a.left_signs.bytes().data();
    d.signs_v = a.right_signs.bytes().data();
    if (a.left_signs.size() != a.m || a.right_signs.size() != a.n)
      throw SizeError("sign vector lengths disagree with m, n");
  } else {
    d.phases_u = a.left_phases.data();
    d.phases_v = a.right_phases.data();
    if (a.left_phases.size() != a.m / 2 || a.right_phases.size() != a.n / 2)
      throw SizeError("phase vector lengths disagree with m, n");
  }
  q8p_layer* l = nullptr;
  check(q8p_layer_create(&d, device, &l));
  return l;
}
}  // namespace

DeviceLayer::DeviceLayer(const QuantizedLinear& a, int device) : layer_(make_from(a, device)) {}

DeviceLayer::DeviceLayer(std::span<const std::uint8_t> qshp, int device) {
  q8p_layer* l = nullptr;
  check(q8p_layer_from_qshp(qshp.data(), qshp.size(), device, &l));
  layer_.reset(l);
}

DeviceLayer::DeviceLayer(std::span<const std::uint8_t> qshp, std::uint32_t row_begin,
                         std::uint32_t row_end, int device) {
  q8p_layer* l = nullptr;
  check(q8p_layer_from_qshp_rows(qshp.data(), qshp.size(), row_begin, row_end, device, &l));
  layer_.reset(l);
}

q8p_layer_info DeviceLayer::info() const {
  q8p_layer_info i{};
  check(q8p_layer_get_info(get(), &i));
  return i;
}

std::vector<double> DeviceLayer::infer(std::span<const double> x) const {
  const q8p_layer_info i = info();
  if (x.size() != i.n) throw SizeError("infer: input length != n");
  std::vector<double> y(i.m);
  check(q8p_infer_host(get(), x.data(), y.data(), 1));
  return y;
}

std::vector<double> infer(const QuantizedLinear& a, std::span<const double> x) {
  if (x.size() != a.n) throw SizeError("infer: input length != n");
  return DeviceLayer(a).infer(x);
}

}  // namespace q8p
