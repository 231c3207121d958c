// The C ABI (include/q8p.h): layer upload, forward orchestration
// (K1 -> K2 -> [all-gather] -> K3), host-buffer infer, and status mapping.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <future>
#include <string>

#include "device.hpp"

namespace q8p::detail {

std::atomic<std::uint64_t> g_launches{0};
namespace {
thread_local std::string t_last_error;
}

void set_last_error(const std::string& msg) { t_last_error = msg; }

int current_device() {
  int d = 0;
  cuda_check(cudaGetDevice(&d), "cudaGetDevice");
  return d;
}

void kernel_attrs(const void* fn, int max_dyn_smem, bool cluster) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  const int dev = current_device();
  std::scoped_lock lock(mu);
  for (const auto& e : done)
    if (e.first == fn && e.second == dev) return;
  cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem), "smem attr");
#ifndef Q8P_DBG_NO_CARVEOUT
  cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout attr");
#else
  if (max_dyn_smem > 150 * 1024)
    cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout attr");
#endif
  if (cluster) cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1), "cluster attr");
  done.emplace_back(fn, dev);
}

void throw_cuda(cudaError_t e, const char* what) {
  throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

q8p_status status_of_current_exception() {
  try {
    throw;
  } catch (const SizeError& e) {
    set_last_error(e.what());
    return Q8P_ERR_SIZE;
  } catch (const ValidationError& e) {
    set_last_error(e.what());
    return Q8P_ERR_VALIDATION;
  } catch (const BadMagicError& e) {
    set_last_error(e.what());
    return Q8P_ERR_BAD_MAGIC;
  } catch (const UnsupportedVersionError& e) {
    set_last_error(e.what());
    return Q8P_ERR_UNSUPPORTED_VERSION;
  } catch (const TruncatedArtifactError& e) {
    set_last_error(e.what());
    return Q8P_ERR_TRUNCATED;
  } catch (const FormatError& e) {
    set_last_error(e.what());
    return Q8P_ERR_FORMAT;
  } catch (const UnsupportedError& e) {
    set_last_error(e.what());
    return Q8P_ERR_UNSUPPORTED;
  } catch (const NcclError& e) {
    set_last_error(e.what());
    return Q8P_ERR_NCCL;
  } catch (const DeviceError& e) {
    set_last_error(e.what());
    return Q8P_ERR_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return Q8P_ERR_INTERNAL;
  } catch (...) {
    set_last_error("unknown exception");
    return Q8P_ERR_INTERNAL;
  }
}

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

void require_sm100(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    throw DeviceError("no CUDA device available (q8p requires an sm_100 B200)");
  if (device < 0 || device >= count) throw ValidationError("device index out of range");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    throw DeviceError("q8p kernels are built for sm_100a only; device is sm_" +
                      std::to_string(prop.major) + std::to_string(prop.minor));
}

void* dev_alloc(q8p_layer* L, std::size_t bytes) {
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc");
  L->allocations.push_back(p);
  L->device_bytes += bytes;
  return p;
}

void dev_free(q8p_layer* L, void* p, std::size_t bytes) {
  auto it = std::find(L->allocations.begin(), L->allocations.end(), p);
  if (it != L->allocations.end()) L->allocations.erase(it);
  L->device_bytes -= bytes;
  cuda_check(cudaFree(p), "cudaFree");
}

// Layer uploads run on the building thread's private non-blocking stream (no
// legacy-stream or device-wide synchronisation: concurrent forwards and other
// streams' captures are unaffected); build_layer synchronises it once at the end.
// (cudaMemcpyAsync from pageable memory returns once the source is staged.)
thread_local cudaStream_t t_build_stream = nullptr;

void* upload(q8p_layer* L, const void* host, std::size_t bytes) {
  void* d = dev_alloc(L, bytes);
  cuda_check(cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, t_build_stream), "upload");
  return d;
}

void setup_side(q8p_layer* L, DevSide& side, std::uint32_t n, const std::uint8_t* signs) {
  const HadamardSpec spec = plan_hadamard(n);
  side.n = n;
  side.p = static_cast<std::uint32_t>(spec.p);
  side.q = static_cast<std::uint32_t>(spec.q);
  std::vector<std::uint8_t> sb(signs, signs + (n + 7) / 8);
  if (n % 8) sb.back() &= static_cast<std::uint8_t>((1u << (n % 8)) - 1);  // from_bytes masks pad bits
  side.signs = static_cast<const std::uint8_t*>(upload(L, sb.data(), sb.size()));
  std::vector<float> colsum(spec.q, 1.f);
  if (spec.q > 1) {
    const std::vector<std::int8_t>& b = hadamard_base(spec.q);
    side.base = static_cast<const std::int8_t*>(upload(L, b.data(), b.size()));
    for (std::size_t j = 0; j < spec.q; ++j) {
      long c = 0;
      for (std::size_t i = 0; i < spec.q; ++i) c += b[i * spec.q + j];
      colsum[j] = float(c);
    }
  }
  side.colsum = static_cast<const float*>(upload(L, colsum.data(), colsum.size() * 4));
}

// rfft side (rfft.cpp): DFT factorization + rotor / twiddle tables.
void setup_side_rfft(q8p_layer* L, DevSide& side, std::uint32_t n, const float* phases, bool codewords) {
  side.kind = 1;
  side.n = n;
  if (!rfft_factor(n, codewords, side.M1, side.M2))
    throw UnsupportedError("rfft: DFT length " + std::to_string(n / 2) + " has no factorization the kernels fit");
  std::vector<float> rot, tw;
  rfft_tables(n, phases, rot, tw);
  side.rot = static_cast<const float2*>(upload(L, rot.data(), rot.size() * 4));
  side.tw = static_cast<const float2*>(upload(L, tw.data(), tw.size() * 4));
}

// Builds a device layer from host fields for rows [r0, r1).
q8p_layer* build_layer(const q8p_layer_desc& d, std::uint32_t r0, std::uint32_t r1, int device) {
  if (!d.stages || d.num_stages < 1) throw ValidationError("artifact has no quantization stages");
  if (d.num_stages > 2) throw UnsupportedError("more than two RVQ stages are not on this path");
  if (d.transform != 0 && d.transform != 1) throw ValidationError("unknown transform kind");
  const bool rfft = d.transform == 1;
  if (d.m == 0 || d.n == 0) throw SizeError("empty layer");
  if (d.n % 8 != 0) throw FormatError("artifact: n not divisible by codeword dimension");
  if (!(r0 < r1 && r1 <= d.m)) throw ValidationError("row range out of bounds");
  if (rfft) {
    if (!d.phases_u || !d.phases_v) throw ValidationError("phase vectors required");
    if (d.m % 2 != 0) throw SizeError("rfft_apply: length must be even and positive");  // rfft.cpp:41-42
    std::uint32_t a, b;
    if (!rfft_factor(d.n, true, a, b) || !rfft_factor(d.m, false, a, b))
      throw UnsupportedError("rfft: DFT length has no factorization the kernels fit");
  } else {
    if (!d.signs_u || !d.signs_v) throw ValidationError("sign vectors required");
    plan_hadamard(d.n);  // SizeError before any allocation
    plan_hadamard(d.m);
  }
  require_sm100(device);
  DeviceGuard g(device);
  struct BuildStream {  // this thread's upload / transcode stream for the duration of the build
    BuildStream() { cuda_check(cudaStreamCreateWithFlags(&t_build_stream, cudaStreamNonBlocking), "build stream"); }
    ~BuildStream() {
      cudaStreamDestroy(t_build_stream);
      t_build_stream = nullptr;
    }
  } build_stream;
  auto L = std::make_unique<q8p_layer>();
  L->device = device;
  L->m = d.m;
  L->n = d.n;
  L->row_begin = r0;
  L->row_end = r1;
  L->num_stages = d.num_stages;
  try {
    if (rfft) {
      setup_side_rfft(L.get(), L->side_u, d.m, d.phases_u, false);
      setup_side_rfft(L.get(), L->side_v, d.n, d.phases_v, true);
    } else {
      setup_side(L.get(), L->side_u, d.m, d.signs_u);
      setup_side(L.get(), L->side_v, d.n, d.signs_v);
    }
    {
      const std::vector<std::uint8_t> img = tc_lut_image();
      L->lut_img = static_cast<const std::uint8_t*>(upload(L.get(), img.data(), img.size()));
      const std::vector<std::uint32_t> tw = decode_table_words();
      L->dec_tables = static_cast<const std::uint32_t*>(upload(L.get(), tw.data(), tw.size() * 4));
    }
    const std::size_t nb = d.n / 8, words = std::size_t(r1 - r0) * nb;
    const std::uint8_t* odd_dev = nullptr;  // E8P odd-parity table for the device transcode
    for (int s = 0; s < d.num_stages; ++s) {
      const q8p_stage_desc& st = d.stages[s];
      if (st.codebook != Q8P_CB_E8P_2BIT && st.codebook != Q8P_CB_E8_1BIT)
        throw ValidationError("unknown codebook");
      if (!st.codes) throw ValidationError("stage codes missing");
      if (!(st.scale > 0.f) || !std::isfinite(st.scale)) throw ValidationError("stage scale must be positive");
      if (st.code_bytes != 1 && st.code_bytes != 2) throw ValidationError("code_bytes must be 1 or 2");
      if (st.codebook == Q8P_CB_E8P_2BIT && st.code_bytes != 2)
        throw ValidationError("e8p-2bit codes are 16-bit");
      L->cb[s] = st.codebook;
      L->scale[s] = st.scale;
      const auto* src = static_cast<const std::uint8_t*>(st.codes) + std::size_t(r0) * nb * st.code_bytes;
      if (st.codebook == Q8P_CB_E8P_2BIT) {
        L->codes[s] = upload(L.get(), src, words * 2);
        L->code_bytes += words * 2;
      } else {
        // e8-1bit codewords are < 256 (codebook.cpp:66): narrow to u8 losslessly.
        std::vector<std::uint8_t> narrow(words);
        for (std::size_t i = 0; i < words; ++i) {
          const std::uint32_t v = st.code_bytes == 2 ? reinterpret_cast<const std::uint16_t*>(src)[i] : src[i];
          if (v >= 256) throw ValidationError("decode: codeword out of range");
          narrow[i] = static_cast<std::uint8_t>(v);
        }
        L->codes[s] = upload(L.get(), narrow.data(), words);
        L->code_bytes += words;
      }
      // Tensor-core slab format (lossless re-layout, gemv_tc.cu), built on the device
      // from the plain codes just uploaded.
      {
        const int kind = st.codebook == Q8P_CB_E8P_2BIT ? 0 : 1;
        if (!odd_dev) {
          const E8PTable& t = e8p_table();
          odd_dev = static_cast<const std::uint8_t*>(upload(L.get(), t.odd_parity.data(), 256));
        }
        void* slabs = dev_alloc(L.get(), tc_code_bytes(r1 - r0, d.n, kind));
        tc_transcode_device(L->codes[s], r1 - r0, d.n, kind, static_cast<std::uint8_t*>(slabs), odd_dev,
                            t_build_stream);
        L->tc[s].codes = slabs;
      }
    }
    cuda_check(cudaStreamSynchronize(t_build_stream), "layer upload");
    cuda_check(cudaGetLastError(), "layer upload");
    // The slabs carry every code bit: the plain copy stays only where the portable
    // GEMV needs it (first stage not E8P), halving the code bytes held in HBM.
    if (L->cb[0] == Q8P_CB_E8P_2BIT) {
      for (int s = 0; s < d.num_stages; ++s) {
        if (!L->codes[s]) continue;
        const std::size_t bytes = words * (L->cb[s] == Q8P_CB_E8P_2BIT ? 2 : 1);
        dev_free(L.get(), L->codes[s], bytes);
        L->codes[s] = nullptr;
      }
    }
  } catch (...) {
    for (void* p : L->allocations) cudaFree(p);
    throw;
  }
  return L.release();
}

q8p_layer* layer_from_bytes(const std::uint8_t* bytes, std::size_t len, std::uint32_t r0,
                            std::uint32_t r1, bool full, int device) {
  const QuantizedLinear a = deserialize(std::span(bytes, len));
  std::vector<q8p_stage_desc> st(a.stages.size());
  for (std::size_t s = 0; s < st.size(); ++s) {
    codebook_code_bytes(a.stages[s].codebook);
    st[s].codebook = a.stages[s].codebook == "e8p-2bit" ? Q8P_CB_E8P_2BIT : Q8P_CB_E8_1BIT;
    st[s].scale = a.stages[s].scale;
    st[s].codes = a.codes[s].data();
    st[s].code_bytes = 2;
  }
  q8p_layer_desc d{};
  d.m = a.m;
  d.n = a.n;
  d.transform = a.transform == TransformKind::rht ? 0 : 1;
  d.num_stages = static_cast<int>(st.size());
  d.stages = st.data();
  d.signs_u = a.left_signs.bytes().data();
  d.signs_v = a.right_signs.bytes().data();
  d.phases_u = a.left_phases.data();
  d.phases_v = a.right_phases.data();
  if (full) {
    r0 = 0;
    r1 = a.m;
  }
  return build_layer(d, r0, r1, device);
}

std::size_t round_up(std::size_t v, std::size_t a) { return (v + a - 1) / a * a; }

// Records a caller event on `s`; under stream capture it must become an
// external event node to be timeable after graph replay.
void record_event(void* ev, cudaStream_t s) {
  if (!ev) return;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(s, &st), "capture status");
  if (st == cudaStreamCaptureStatusActive)
    cuda_check(cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev), s, cudaEventRecordExternal), "event record");
  else
    cuda_check(cudaEventRecord(static_cast<cudaEvent_t>(ev), s), "event record");
}

// Per-forward scratch, caller-provided (q8p_workspace_bytes).  Tensor-core path:
// RHT scratch, per-chunk sums of squares, alpha / TL per vector, the B images of
// the integer activations and the int32 accumulators.  Portable path: t, z.
struct Workspace {
  float* u;              // [batch][max(m, n)] RHT intermediate
  float* t;              // [batch][n] (portable path)
  float* z;              // [batch][m] (portable path)
  float* ssq;            // [batch][n / 4]
  float* alpha;          // [batch]
  long long* tl;         // [batch]
  std::uint8_t* bimg;    // tc_bimg_bytes(n, batch)
  std::int32_t* zacc;    // [stages][N][rows_pad]
  float* pt;             // prefill: t [batch][n] fp32
  std::uint8_t* pbt;     // prefill: bf16 B tiles
  float* pz;             // prefill: z [batch][m_local]
  float* z_loc;          // row-sharded: [batch][m_local] this rank's z rows
  float* z_full;         // row-sharded: [batch][m] all-gathered z
  float* pz_full;        // row-sharded prefill: [batch][m] all-gathered K3 pass-1 rows (row shards only)
  std::uint32_t rows_pad, zcols;
};
std::uint32_t rows_pad_of(const q8p_layer* L) { return tc_row_blocks(L->m_local()) * 128; }
// Batches above the tensor-core path's 32 vectors run as 32-vector chunks through
// it (weights streamed once per chunk).
int tc_chunk(const q8p_layer* L, int batch) {
  if (tc_supported(*L, batch)) return batch;
  if (batch > kTcMaxBatch && tc_supported(*L, kTcMaxBatch)) return kTcMaxBatch;
  return 0;  // portable path
}

// Batches of several whole chunks run K1 once for all vectors (B images per chunk),
// then K2 + K3 per chunk with K3 clearing the accumulators it read (multi-chunk K1).
bool multi_chunk_k1(const q8p_layer* L, int batch) {
  const int chunk = tc_chunk(L, batch);
  return chunk > 0 && batch > chunk && batch % chunk == 0 && L->side_v.kind == 0 && L->side_u.kind == 0 &&
         (L->n / 8) % 32 == 0;
}

// Prefill batches run the K4 decode-GEMM (gemm_prefill.cu) unless Q8P_PREFILL=0
// (A/B knob: the 32-vector chunks through K2 instead).
// K4 for this layer (or row shard) at this batch (Q8P_PREFILL=0: the 32-vector
// chunked GEMV instead, an A/B and debugging switch).
bool use_prefill_rows(const q8p_layer* L, int batch) {
  static const bool off = [] {
    const char* e = std::getenv("Q8P_PREFILL");
    return e && std::string(e) == "0";
  }();
  return !off && prefill_supported(*L, batch);
}
bool use_prefill(const q8p_layer* L, int batch) {  // the unsharded forward
  return L->row_begin == 0 && L->row_end == L->m && use_prefill_rows(L, batch);
}

std::size_t workspace_parts(const q8p_layer* L, int batch, Workspace* w, void* base) {
  auto* p0 = static_cast<std::uint8_t*>(base);
  std::size_t off = 0;
  auto take = [&](std::size_t bytes) {
    std::uint8_t* r = p0 ? p0 + off : nullptr;
    off += round_up(bytes ? bytes : 1, 256);
    return r;
  };
  const int batch_all = batch;
  const int chunk = tc_chunk(L, batch);
  const bool tc = chunk > 0;
  const bool multi = multi_chunk_k1(L, batch);
  const std::size_t BK = std::size_t(multi ? batch : chunk);  // vectors of one K1 launch
  if (tc) batch = chunk;  // otherwise the workspace holds one chunk
  const std::size_t B = std::size_t(batch), mx = std::max(L->n, L->m);
  Workspace v{};
  v.rows_pad = rows_pad_of(L);
  v.zcols = std::uint32_t(tc_ncols_pad(4 * batch));
  v.u = reinterpret_cast<float*>(take((tc ? BK : B) * mx * 4));  // transform scratch of one K1 launch
  if (tc) {
    v.ssq = reinterpret_cast<float*>(take(BK * std::max<std::size_t>(64, L->n / 4) * 4));
    v.alpha = reinterpret_cast<float*>(take(BK * 4));
    v.tl = reinterpret_cast<long long*>(take(BK * 8));
    v.bimg = take(tc_bimg_bytes(L->n, batch) * (BK / B));
    v.zacc = reinterpret_cast<std::int32_t*>(take(std::size_t(L->num_stages) * v.zcols * v.rows_pad * 4));
    v.z_full = reinterpret_cast<float*>(take(B * L->m * 4));      // q8p_forward_sharded: gathered rows
    v.z_loc = reinterpret_cast<float*>(take(B * L->m_local() * 4));  // this rank's rows (send buffer)
  } else {
    v.t = reinterpret_cast<float*>(take(B * L->n * 4));
    v.z = reinterpret_cast<float*>(take(B * L->m * 4));
  }
  if (use_prefill_rows(L, batch_all)) {  // K4 path; the chunked path stays sized for rows_z
    const std::size_t Ball = std::size_t(batch_all);
    v.pt = reinterpret_cast<float*>(take(Ball * L->n * 4));
    v.pbt = take(prefill_btile_bytes(*L, batch_all));
    v.pz = reinterpret_cast<float*>(take(std::size_t(prefill_parts(*L, batch_all)) * Ball * L->m_local() * 4));
    v.u = reinterpret_cast<float*>(take(Ball * mx * 4));  // also the sharded pass 1's send buffer
    if (L->m_local() != L->m) v.pz_full = reinterpret_cast<float*>(take(Ball * L->m * 4));
  }
  if (w) *w = v;
  return off;
}
std::size_t workspace_size(const q8p_layer* L, int batch) { return workspace_parts(L, batch, nullptr, nullptr); }

// K1 -> K2 on the layer's local rows: leaves int32 accumulators in w.zacc (tensor-core
// path) or fp32 z rows in w.z (portable path).
void forward_local(const q8p_layer* L, const float* x, int batch, const Workspace& w, cudaStream_t s,
                   const q8p_forward_opts* opts) {
  if (tc_supported(*L, batch)) {  // (callers chunk batches above kTcMaxBatch)
    // N from this call's batch (a chunk may be smaller than the workspace's 16)
    const std::uint32_t N = std::uint32_t(tc_ncols_pad(4 * batch)), KSL = tc_k_slabs(L->n), bb = 9u * N * 32u;
    const bool ragged = (L->n / 8) % 32 != 0;
#ifndef Q8P_EXP_SKIP_K1
    launch_rht_in_limbs(L->side_v, x, w.u, w.ssq, w.alpha, w.tl, w.bimg, bb, N,
                        ragged ? w.bimg + std::size_t(KSL - 1) * bb : nullptr, ragged ? bb : 0, w.zacc,
                        std::size_t(L->num_stages) * N * w.rows_pad, batch, s);
#endif
    if (opts) record_event(opts->gemv_start_event, s);
    launch_gemv_tc(*L, w.bimg, w.zacc, w.rows_pad, batch, s);
    if (opts) record_event(opts->gemv_end_event, s);
  } else if (L->side_v.kind == 1) {  // rfft (kernels_rfft.cu): t = T_v x through the scratch
    launch_rht_in(L->side_v, x, w.t, w.u, nullptr, nullptr, nullptr, 0, batch, s);
    if (opts) record_event(opts->gemv_start_event, s);
    launch_gemv_simple(*L, w.t, w.z, batch, static_cast<int>(L->m), s);
    if (opts) record_event(opts->gemv_end_event, s);
  } else {
    launch_rht(L->side_v, x, w.t, batch, /*transpose=*/false, s);  // t = T_v x
    if (opts) record_event(opts->gemv_start_event, s);
    launch_gemv_simple(*L, w.t, w.z, batch, static_cast<int>(L->m), s);
    if (opts) record_event(opts->gemv_end_event, s);
  }
}

[[noreturn]] void throw_nccl(ncclResult_t r, const char* what) {
  throw q8p::NcclError(std::string(what) + ": " + ncclGetErrorString(r));
}
inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw_nccl(r, what);
}

// Row-sharded forward.  Per chunk of vectors:
//   K1 (replicated) -> K2 on this rank's rows -> K3 pass 1 on this rank's rows,
//   straight from its accumulators into the send buffer [nb][m_local] (the rows of
//   a rank are whole pass-1 chunks) -> ONE ncclAllGather of nb * m_local floats
//   (rank-major [world][nb][m_local]) over NVLink -> K3 pass 2 on the gathered rows.
// Pass 1 acts on contiguous chunks independently, so each rank computes exactly
// the values the unsharded pass 1 computes for its chunks, and pass 2 is
// unchanged: sharded y equals unsharded y bit for bit.  When the rank's rows are
// not whole chunks (or transform = rfft): combine -> the same single all-gather ->
// both K3 passes on the gathered z (rank-major reads; rfft: one call per vector).
// No host synchronisation: the whole forward is stream-ordered and capturable
// in a CUDA graph (NCCL collectives capture as graph nodes).
void forward_sharded_impl(const q8p_layer* L, const float* x, float* y, int batch, void* ws, std::size_t ws_bytes,
                          ncclComm_t comm, cudaStream_t s) {
  if (!L) throw ValidationError("null layer");
  if (batch < 0) throw ValidationError("negative batch");
  if (batch == 0) return;
  if (!x || !y) throw ValidationError("null x / y");
  if (!comm) throw ValidationError("null communicator");
  const int chunk = tc_chunk(L, batch);  // batches above kTcMaxBatch go through in chunks
  if (chunk == 0) throw UnsupportedError("row-sharded forward needs the tensor-core path");
  int world = 0, rank = 0;
  nccl_check(ncclCommCount(comm, &world), "ncclCommCount");
  nccl_check(ncclCommUserRank(comm, &rank), "ncclCommUserRank");
  const std::uint32_t ml = L->m_local();
  if (std::size_t(ml) * std::size_t(world) != L->m || L->row_begin != std::uint32_t(rank) * ml)
    throw ValidationError("row shards must be equal-sized and ordered by rank");
  if (ml % 4 != 0) throw UnsupportedError("row shards must be multiples of 4 rows");
  if (!ws || ws_bytes < workspace_size(L, batch)) throw SizeError("workspace too small");
  DeviceGuard g(L->device);
  Workspace w;
  workspace_parts(L, batch, &w, ws);
  float zscale[2] = {L->scale[0], L->scale[1]};
  int ze8p[2] = {L->cb[0] == Q8P_CB_E8P_2BIT, L->cb[1] == Q8P_CB_E8P_2BIT};
  const bool local_p1 = rht_sharded_k3_ok(L->side_u, L->row_begin, ml);
  if (local_p1 && use_prefill_rows(L, batch)) {
    // prefill: K1 (replicated) -> K4 on this rank's rows -> K3 pass 1 on them (summing
    // the K-split partials) -> one all-gather -> K3 pass 2
    launch_rht_in(L->side_v, x, w.pt, w.u, prefill_amax(*L, batch, w.pbt), nullptr, nullptr, 0, batch, s);
    launch_prefill(*L, w.pt, w.pbt, w.pz, batch, s);
    const K4Sched ks = prefill_sched(*L, batch);
    launch_rht_out_local_f32(L->side_u, w.pz, int(ks.slices), L->row_begin, ml, w.u, nullptr, batch, s, &ks);
    if (world == 1) {
      launch_rht_out_pass2_gathered(L->side_u, w.u, ml, y, batch, s);
      return;
    }
    nccl_check(ncclAllGather(w.u, w.pz_full, std::size_t(batch) * ml, ncclFloat32, comm, s), "ncclAllGather");
    launch_rht_out_pass2_gathered(L->side_u, w.pz_full, ml, y, batch, s);
    return;
  }
  for (int b0 = 0; b0 < batch; b0 += chunk) {
    const int nb = std::min(chunk, batch - b0);
    float* yb = y + std::size_t(b0) * L->m;
    forward_local(L, x + std::size_t(b0) * L->n, nb, w, s, nullptr);
    if (local_p1) {
      launch_rht_out_acc_local(L->side_u, w.zacc, L->num_stages, w.rows_pad, std::uint32_t(tc_ncols_pad(4 * nb)),
                               zscale, ze8p, w.alpha, w.tl, L->row_begin, ml, w.z_loc, nb, s);
      if (world == 1) {  // a one-rank all-gather is the identity: pass 2 reads the send buffer
        launch_rht_out_pass2_gathered(L->side_u, w.z_loc, ml, yb, nb, s);
        continue;
      }
      nccl_check(ncclAllGather(w.z_loc, w.z_full, std::size_t(nb) * ml, ncclFloat32, comm, s), "ncclAllGather");
      launch_rht_out_pass2_gathered(L->side_u, w.z_full, ml, yb, nb, s);
      continue;
    }
    launch_combine_acc(w.zacc, L->num_stages, w.rows_pad, std::uint32_t(tc_ncols_pad(4 * nb)), zscale, ze8p, w.alpha,
                       w.tl, w.z_loc, ml, nb, s);
    if (L->side_u.kind == 0) {
      nccl_check(ncclAllGather(w.z_loc, w.z_full, std::size_t(nb) * ml, ncclFloat32, comm, s), "ncclAllGather");
      launch_rht_out_gathered(L->side_u, w.z_full, ml, w.u, yb, nb, s);
    } else {  // rfft K3 reads natural-layout z: one gather per vector
      nccl_check(ncclGroupStart(), "ncclGroupStart");
      for (int b = 0; b < nb; ++b)
        nccl_check(ncclAllGather(w.z_loc + std::size_t(b) * ml, w.z_full + std::size_t(b) * L->m, ml, ncclFloat32,
                                 comm, s),
                   "ncclAllGather");
      nccl_check(ncclGroupEnd(), "ncclGroupEnd");
      launch_rht_out(L->side_u, w.z_full, w.u, yb, nb, s);
    }
  }
}

// K3 pass 1 of one rank for the push all-gather (q8p_forward_sharded_push): the
// rank's rows straight into every rank's window.
void k3_push(const q8p_layer* L, const Workspace& w, const PushArgs& pa, int nb, cudaStream_t s) {
  float zscale[2] = {L->scale[0], L->scale[1]};
  int ze8p[2] = {L->cb[0] == Q8P_CB_E8P_2BIT, L->cb[1] == Q8P_CB_E8P_2BIT};
  launch_rht_out_acc_push(L->side_u, w.zacc, L->num_stages, w.rows_pad, std::uint32_t(tc_ncols_pad(4 * nb)), zscale,
                          ze8p, w.alpha, w.tl, L->row_begin, L->m_local(), pa, nb, s);
}

}  // namespace
}  // namespace q8p::detail

// Peer group of the push all-gather (device.hpp PeerCtl / PushArgs).
struct q8p_peers {
  int device = 0, world = 1, rank = 0;
  std::size_t slice_floats = 0;          // per-rank slice capacity of one parity (values)
  void* base = nullptr;                  // local allocation [PeerCtl][2][world][slice] words
  std::vector<void*> opened;             // peers' bases mapped by CUDA IPC (closed at destroy)
  unsigned long long** d_wins = nullptr; // device table [world] of the ranks' windows
  bool connected = false;
  q8p::detail::PushArgs args() const {
    q8p::detail::PushArgs a{};
    a.wins = d_wins;
    a.self_win = reinterpret_cast<unsigned long long*>(static_cast<std::uint8_t*>(base) + q8p::detail::kPeerCtlBytes);
    a.ctl = static_cast<q8p::detail::PeerCtl*>(base);
    a.rank = rank;
    a.world = world;
    a.win_words = std::size_t(world) * slice_floats;
    return a;
  }
};

namespace q8p::detail {
namespace {

std::size_t peer_bytes(int world, std::size_t slice_floats) {
  return kPeerCtlBytes + 2 * std::size_t(world) * slice_floats * 8;  // tagged 8-byte words
}

void peers_set_bases(q8p_peers* p, const std::vector<void*>& bases) {
  std::vector<unsigned long long*> w(p->world);
  for (int r = 0; r < p->world; ++r)
    w[r] = reinterpret_cast<unsigned long long*>(static_cast<std::uint8_t*>(bases[r]) + kPeerCtlBytes);
  cuda_check(cudaMemcpy(p->d_wins, w.data(), sizeof(void*) * p->world, cudaMemcpyHostToDevice), "peer table");
  p->connected = true;
}

void check_push_layer(const q8p_layer* L, const q8p_peers* p, int batch) {
  if (!L || !p) throw ValidationError("null layer / peers");
  if (!p->connected) throw ValidationError("peers not connected");
  if (L->device != p->device) throw ValidationError("layer and peers on different devices");
  const std::uint32_t ml = L->m_local();
  if (std::size_t(ml) * std::size_t(p->world) != L->m || L->row_begin != std::uint32_t(p->rank) * ml)
    throw ValidationError("row shards must be equal-sized and ordered by rank");
  if (tc_chunk(L, batch) == 0) throw UnsupportedError("push all-gather needs the tensor-core path");
  if (!rht_sharded_k3_ok(L->side_u, L->row_begin, ml))
    throw UnsupportedError("push all-gather: a rank's rows must be whole K3 pass-1 chunks (rht layers)");
  const std::size_t per_call = use_prefill_rows(L, batch) ? std::size_t(batch) : std::size_t(std::min(tc_chunk(L, batch), batch));
  if (per_call * ml > p->slice_floats)
    throw SizeError("push all-gather: window slice too small for this layer / batch");
}

void forward_push_impl(const q8p_layer* L, q8p_peers* p, const float* x, float* y, int batch, void* ws,
                       std::size_t ws_bytes, cudaStream_t s) {
  if (batch < 0) throw ValidationError("negative batch");
  if (batch == 0) return;
  if (!x || !y) throw ValidationError("null x / y");
  check_push_layer(L, p, batch);
  if (!ws || ws_bytes < workspace_size(L, batch)) throw SizeError("workspace too small");
  DeviceGuard g(L->device);
  Workspace w;
  workspace_parts(L, batch, &w, ws);
  const PushArgs pa = p->args();
  if (use_prefill_rows(L, batch)) {  // prefill: K1 -> K4 on this rank's rows -> pushing K3 pass 1 -> pass 2
    launch_rht_in(L->side_v, x, w.pt, w.u, prefill_amax(*L, batch, w.pbt), nullptr, nullptr, 0, batch, s);
    launch_prefill(*L, w.pt, w.pbt, w.pz, batch, s);
    const K4Sched ks = prefill_sched(*L, batch);
    launch_rht_out_local_f32(L->side_u, w.pz, int(ks.slices), L->row_begin, L->m_local(), nullptr, &pa, batch, s,
                             &ks);
    launch_rht_out_pass2_push(L->side_u, L->m_local(), pa, y, batch, s);
    return;
  }
  const int chunk = tc_chunk(L, batch);
  for (int b0 = 0; b0 < batch; b0 += chunk) {  // one push epoch per chunk
    const int nb = std::min(chunk, batch - b0);
    forward_local(L, x + std::size_t(b0) * L->n, nb, w, s, nullptr);
    k3_push(L, w, pa, nb, s);
    launch_rht_out_pass2_push(L->side_u, L->m_local(), pa, y + std::size_t(b0) * L->m, nb, s);
  }
}

// Prefill chunk: the whole batch, or the most 256-vector N tiles whose B tiles fit
// kPrefillBTileL2 (the chunks' K1 -> K4 -> K3 chains run back to back).
constexpr std::size_t kPrefillBTileL2 = std::size_t(64) << 20;
int prefill_chunk(const q8p_layer& L, int batch) {
  const std::size_t per_tile = std::size_t(L.n) * L.num_stages * 512;  // B bytes per 256-vector N tile
  const std::size_t tiles = std::max<std::size_t>(1, kPrefillBTileL2 / per_tile);
  const std::size_t chunk = tiles * 256;
  return chunk >= std::size_t(batch) ? batch : int(chunk);
}

void forward_impl(const q8p_layer* L, const float* x, float* y, int batch, void* ws, std::size_t ws_bytes,
                  cudaStream_t s, const q8p_forward_opts* opts = nullptr) {
  if (!L) throw ValidationError("null layer");
  if (batch < 0) throw ValidationError("negative batch");
  if (batch == 0) return;
  if (!x || !y) throw ValidationError("null x / y");
  if (L->row_begin != 0 || L->row_end != L->m)
    throw ValidationError("row-sharded layer: use q8p_forward_sharded");
  if (!ws || ws_bytes < workspace_size(L, batch)) throw SizeError("workspace too small");
  DeviceGuard g(L->device);
  Workspace w;
  workspace_parts(L, batch, &w, ws);
  if (use_prefill(L, batch)) {  // K1 (fp32 t) -> K4 (pack + decode-GEMM) -> K3
    // Large batches on long-K layers run in chunks whose B tiles (ceil(B / 256) x
    // n x stages x 512 bytes) stay L2-resident: 8192x28672 at batch 2048 would
    // stream 117 MB of B tiles through the 126 MB L2 next to the codes.
    const int chunk = prefill_chunk(*L, batch);
    if (chunk < batch) {
      if (opts) record_event(opts->gemv_start_event, s);  // (brackets the chunks' whole chains)
      for (int b0 = 0; b0 < batch; b0 += chunk)
        forward_impl(L, x + std::size_t(b0) * L->n, y + std::size_t(b0) * L->m, std::min(chunk, batch - b0), ws,
                     ws_bytes, s);
      if (opts) record_event(opts->gemv_end_event, s);
      return;
    }
    launch_rht_in(L->side_v, x, w.pt, w.u, prefill_amax(*L, batch, w.pbt), nullptr, nullptr, 0, batch, s);
    if (opts) record_event(opts->gemv_start_event, s);  // the events bracket pack + K4
    launch_prefill(*L, w.pt, w.pbt, w.pz, batch, s);
    if (opts) record_event(opts->gemv_end_event, s);
    // K3 sums the K splits' partial z in fixed order while loading them
    const K4Sched ks = prefill_sched(*L, batch);
    launch_rht_out(L->side_u, w.pz, w.u, y, batch, s, int(ks.slices), &ks);
    return;
  }
  if (const int chunk = tc_chunk(L, batch)) {
    float zscale[2] = {L->scale[0], L->scale[1]};
    int ze8p[2] = {L->cb[0] == Q8P_CB_E8P_2BIT, L->cb[1] == Q8P_CB_E8P_2BIT};
    if (multi_chunk_k1(L, batch)) {
      const std::uint32_t N = std::uint32_t(tc_ncols_pad(4 * chunk)), bb = 9u * N * 32u;
      const std::size_t cb = std::size_t(tc_k_slabs(L->n)) * bb;  // one chunk's B images
      launch_rht_in_limbs(L->side_v, x, w.u, w.ssq, w.alpha, w.tl, w.bimg, bb, N, nullptr, 0, w.zacc,
                          std::size_t(L->num_stages) * N * w.rows_pad, batch, s, std::uint32_t(chunk), cb);
      for (int b0 = 0, c = 0; b0 < batch; b0 += chunk, ++c) {
        if (opts && c == 0) record_event(opts->gemv_start_event, s);
        launch_gemv_tc(*L, w.bimg + std::size_t(c) * cb, w.zacc, w.rows_pad, chunk, s);
        if (opts && c == 0) record_event(opts->gemv_end_event, s);
        launch_rht_out_acc(L->side_u, w.zacc, L->num_stages, w.rows_pad, N, zscale, ze8p, w.alpha + b0, w.tl + b0,
                           w.u, y + std::size_t(b0) * L->m, chunk, s, /*zero_after=*/b0 + chunk < batch);
      }
      return;
    }
    for (int b0 = 0; b0 < batch; b0 += chunk) {  // one pass for batch <= kTcMaxBatch
      const int nb = std::min(chunk, batch - b0);
      forward_local(L, x + std::size_t(b0) * L->n, nb, w, s, b0 == 0 ? opts : nullptr);
#ifndef Q8P_EXP_SKIP_K3
      launch_rht_out_acc(L->side_u, w.zacc, L->num_stages, w.rows_pad, std::uint32_t(tc_ncols_pad(4 * nb)), zscale,
                         ze8p, w.alpha, w.tl, w.u, y + std::size_t(b0) * L->m, nb, s);
#endif
    }
  } else {
    forward_local(L, x, batch, w, s, opts);
    if (L->side_u.kind == 1)
      launch_rht_out(L->side_u, w.z, w.u, y, batch, s);  // rfft
    else
      launch_rht(L->side_u, w.z, y, batch, /*transpose=*/true, s);  // y = T_u^T z
  }
}

// q8p_forward fast path: the forward's 5-kernel chain is captured once per
// (x, y, batch, workspace) into a CUDA graph and replayed with a single
// cudaGraphLaunch -- one host launch instead of five, same kernels, same
// stream order.  Opt-in (Q8P_GRAPH_CACHE=1): it cuts the host cost per call
// from ~20 to ~4 us, but a graph boundary drops the programmatic-dependent-launch
// overlap between consecutive layers, so GPU-bound callers (bench.py e2e: 7.9 k
// vs 7.7 k tokens/s) are better served by plain launches.  Skipped while the
// caller's stream is itself capturing (the kernels then go into its graph).
void forward_cached(q8p_layer* L, const float* x, float* y, int batch, void* ws, std::size_t ws_bytes,
                    cudaStream_t s) {
  static const bool off = std::getenv("Q8P_GRAPH_CACHE") == nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (off || !L || batch <= 0 || cudaStreamIsCapturing(s, &cap) != cudaSuccess ||
      cap != cudaStreamCaptureStatusNone) {
    forward_impl(L, x, y, batch, ws, ws_bytes, s);
    return;
  }
  cudaGraphExec_t exec = nullptr;
  {
    std::scoped_lock lock(L->graph_mu);
    for (const auto& e : L->graphs)
      if (e.x == x && e.y == y && e.batch == batch && e.ws == ws && e.ws_bytes == ws_bytes) exec = e.exec;
    if (!exec) {
      DeviceGuard g(L->device);
      if (!L->capture_stream)
        cuda_check(cudaStreamCreateWithFlags(&L->capture_stream, cudaStreamNonBlocking), "capture stream");
      cudaGraph_t graph = nullptr;
      const std::uint64_t k0 = g_launches.load();
      cuda_check(cudaStreamBeginCapture(L->capture_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        forward_impl(L, x, y, batch, ws, ws_bytes, L->capture_stream);  // validates arguments
      } catch (...) {
        cudaStreamEndCapture(L->capture_stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      cuda_check(cudaStreamEndCapture(L->capture_stream, &graph), "end capture");
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      cuda_check(ie, "graph instantiate");
      if (L->graphs.size() >= 8) {  // bounded: evict the oldest
        cudaGraphExecDestroy(L->graphs.front().exec);
        L->graphs.erase(L->graphs.begin());
      }
      L->graphs.push_back({x, y, batch, ws, ws_bytes, exec, std::uint32_t(g_launches.load() - k0)});
      g_launches.fetch_sub(L->graphs.back().kernels);  // counted per replay below
    }
    for (const auto& e : L->graphs)
      if (e.exec == exec) g_launches.fetch_add(e.kernels, std::memory_order_relaxed);
  }
  cuda_check(cudaGraphLaunch(exec, s), "graph launch");
}

// ---- layer sets (q8p_forward_set / q8p_forward_set_host) ------------------
// Several independent layer forwards per call (one decode step through a
// model's linear layers).  The host variant stages the concatenated inputs /
// outputs through the tail of the workspace and, when the host buffers are
// pinned, replays the whole step (H2D, every layer's kernel chain with its PDL
// edges, D2H) as ONE cached CUDA graph: one host launch per step.
struct SetGraph {
  std::vector<const q8p_layer*> layers;
  const float* xh;
  float* yh;
  int batch;
  void* ws;
  std::size_t ws_bytes;
  int device;
  unsigned flags;
  cudaGraphExec_t exec;
  std::uint64_t kernels;
};
std::mutex g_set_mu;
std::vector<SetGraph> g_set_graphs;
cudaStream_t g_set_capture[64] = {};

// Workspace of a layer set: sequential -> one shared layer workspace (the largest);
// Q8P_SET_CONCURRENT -> one slice per layer (offset of layer i = layer_ws_offset);
// then the host variant's staging.
std::size_t layer_ws_offset(const q8p_layer* const* layers, int i, int batch, unsigned flags) {
  if (!(flags & Q8P_SET_CONCURRENT)) return 0;
  std::size_t off = 0;
  for (int j = 0; j < i; ++j) off += round_up(workspace_size(layers[j], batch), 256);
  return off;
}
std::size_t set_stage_offset(const q8p_layer* const* layers, int count, int batch, unsigned flags) {
  if (flags & Q8P_SET_CONCURRENT) return layer_ws_offset(layers, count, batch, flags);
  std::size_t ws = 0;
  for (int i = 0; i < count; ++i) ws = std::max(ws, workspace_size(layers[i], batch));
  return round_up(ws, 256);
}
std::size_t set_workspace_size(const q8p_layer* const* layers, int count, int batch, unsigned flags) {
  std::size_t io = 0;
  for (int i = 0; i < count; ++i) io += std::size_t(batch) * (layers[i]->n + layers[i]->m) * 4;
  return set_stage_offset(layers, count, batch, flags) + round_up(io, 256);
}

void check_set(const q8p_layer* const* layers, int count, int batch) {
  if (count < 0 || batch < 0) throw ValidationError("negative layer count / batch");
  if (count > 0 && !layers) throw ValidationError("null layer list");
  for (int i = 0; i < count; ++i) {
    if (!layers[i]) throw ValidationError("null layer");
    if (layers[i]->device != layers[0]->device) throw ValidationError("layers on different devices");
  }
}

// Per-device side streams + events for a layer set's copies / concurrent layers.
struct SetAux {
  cudaStream_t side = nullptr;   // a layer set's host -> device copies
  cudaStream_t side2 = nullptr;  // its device -> host copies (the other copy engine: full duplex)
  std::vector<cudaStream_t> lanes;
  std::vector<cudaEvent_t> ev;
};
SetAux g_set_aux[64];
std::mutex g_set_aux_mu;
constexpr int kSetLanes = 4;

// `lanes` streams and `events` events of device `dev` (created on first use).
SetAux& set_aux(int dev, int lanes, int events) {
  SetAux& aux = g_set_aux[dev];
  if (!aux.side) cuda_check(cudaStreamCreateWithFlags(&aux.side, cudaStreamNonBlocking), "side stream");
  if (!aux.side2) cuda_check(cudaStreamCreateWithFlags(&aux.side2, cudaStreamNonBlocking), "side stream");
  while (int(aux.lanes.size()) < lanes) {
    cudaStream_t st;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "lane stream");
    aux.lanes.push_back(st);
  }
  while (int(aux.ev.size()) < events) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    aux.ev.push_back(e);
  }
  return aux;
}

// Q8P_SET_CONCURRENT: layer i runs on lane i % kSetLanes with its own workspace
// slice; `body(i, lane)` enqueues layer i's work.  Forked from / joined back
// into `s` with events (also under stream capture: the graph gets parallel branches).
template <typename F>
void run_lanes(const q8p_layer* const* layers, int count, cudaStream_t s, F&& body) {
  const int dev = layers[0]->device, nl = std::min(count, kSetLanes);
  std::scoped_lock lock(g_set_aux_mu);
  SetAux& aux = set_aux(dev, nl, 2 + nl);
  cuda_check(cudaEventRecord(aux.ev[0], s), "fork");
  for (int k = 0; k < nl; ++k) cuda_check(cudaStreamWaitEvent(aux.lanes[k], aux.ev[0], 0), "fork wait");
  for (int i = 0; i < count; ++i) body(i, aux.lanes[i % nl]);
  for (int k = 0; k < nl; ++k) {
    cuda_check(cudaEventRecord(aux.ev[2 + k], aux.lanes[k]), "join");
    cuda_check(cudaStreamWaitEvent(s, aux.ev[2 + k], 0), "join wait");
  }
}

void forward_set_impl(const q8p_layer* const* layers, int count, const float* const* x, float* const* y, int batch,
                      void* ws, std::size_t ws_bytes, cudaStream_t s, unsigned flags) {
  if (count == 0 || batch == 0) return;
  if (!(flags & Q8P_SET_CONCURRENT)) {
    for (int i = 0; i < count; ++i) forward_impl(layers[i], x[i], y[i], batch, ws, ws_bytes, s);
    return;
  }
  if (!ws || ws_bytes < set_stage_offset(layers, count, batch, flags)) throw SizeError("workspace too small");
  DeviceGuard g(layers[0]->device);
  run_lanes(layers, count, s, [&](int i, cudaStream_t lane) {
    const std::size_t off = layer_ws_offset(layers, i, batch, flags);
    forward_impl(layers[i], x[i], y[i], batch, static_cast<std::uint8_t*>(ws) + off, ws_bytes - off, lane);
  });
}

// H2D of every input, the forwards, D2H of every output (stream-ordered on `s`
// when it returns, no sync).  The copies run on side streams; for large steps the
// inputs and outputs go on separate ones so the two directions overlap (PCIe is
// full duplex; on one stream a prefill step's copies serialised: 70B set, batch
// 512, e2e 149 k -> 200 k tokens/s):
// layer i waits only for its own input, and y_i goes back while later layers
// compute, so only the first input and the last output are exposed.
// x0_mapped / ylast_mapped (device addresses of pinned host memory, or nullptr):
// the first layer's K1 reads its x straight from the host buffer and the last
// layer's K3 writes its y straight into it, so neither end of the step waits for
// a copy-engine round trip; the other layers' copies overlap the kernels.
void forward_set_host_enqueue(const q8p_layer* const* layers, int count, const float* xh, float* yh, int batch,
                              void* ws, std::size_t ws_bytes, cudaStream_t s, unsigned flags,
                              const float* x0_mapped = nullptr, float* ylast_mapped = nullptr) {
  auto* stage = static_cast<std::uint8_t*>(ws) + set_stage_offset(layers, count, batch, flags);
  std::size_t nsum = 0;
  for (int i = 0; i < count; ++i) nsum += layers[i]->n;
  float* dx = reinterpret_cast<float*>(stage);
  float* dy = dx + std::size_t(batch) * nsum;
  if (flags & Q8P_SET_CONCURRENT) {  // each layer's H2D, forward and D2H on its own lane
    std::vector<std::size_t> xo(count + 1, 0), yo(count + 1, 0);
    for (int i = 0; i < count; ++i) {
      xo[i + 1] = xo[i] + std::size_t(batch) * layers[i]->n;
      yo[i + 1] = yo[i] + std::size_t(batch) * layers[i]->m;
    }
    run_lanes(layers, count, s, [&](int i, cudaStream_t lane) {
      const std::size_t off = layer_ws_offset(layers, i, batch, flags);
      cuda_check(cudaMemcpyAsync(dx + xo[i], xh + xo[i], (xo[i + 1] - xo[i]) * 4, cudaMemcpyHostToDevice, lane),
                 "set H2D");
      forward_impl(layers[i], dx + xo[i], dy + yo[i], batch, static_cast<std::uint8_t*>(ws) + off, ws_bytes - off,
                   lane);
      cuda_check(cudaMemcpyAsync(yh + yo[i], dy + yo[i], (yo[i + 1] - yo[i]) * 4, cudaMemcpyDeviceToHost, lane),
                 "set D2H");
    });
    return;
  }
  const int dev = layers[0]->device;
  std::scoped_lock lock(g_set_aux_mu);
  SetAux& aux = set_aux(dev, 0, 2 * count + 3);
  // Outputs on their own stream only when the copies are large.  70B set, e2e A/Bs
  // on one box: batch 1 (0.36 MB of I/O) 102.4 vs 100.4 us per step and batch 16
  // (5.8 MB) 42.6 k vs 45-60 k tokens/s favour one stream, batch 64 (23 MB) ties,
  // batch 128 (46 MB) 164 k vs 134 k and batch 512 200 k vs 149 k favour two.
  std::size_t io_bytes = 0;
  for (int i = 0; i < count; ++i) io_bytes += std::size_t(batch) * (layers[i]->n + layers[i]->m) * 4;
  const bool duplex = io_bytes > (std::size_t(32) << 20);
  cudaEvent_t fork = aux.ev[0], join = aux.ev[1], join2 = aux.ev[2 * count + 2];
  cuda_check(cudaEventRecord(fork, s), "fork");
  cuda_check(cudaStreamWaitEvent(aux.side, fork, 0), "fork wait");
  if (duplex) cuda_check(cudaStreamWaitEvent(aux.side2, fork, 0), "fork wait");
  std::size_t xo = 0;
  for (int i = 0; i < count; ++i) {
    const std::size_t nb = std::size_t(batch) * layers[i]->n;
    if (!(i == 0 && x0_mapped)) {
      cuda_check(cudaMemcpyAsync(dx + xo, xh + xo, nb * 4, cudaMemcpyHostToDevice, aux.side), "set H2D");
      cuda_check(cudaEventRecord(aux.ev[2 + i], aux.side), "H2D event");
    }
    xo += nb;
  }
  xo = 0;
  std::size_t yo = 0;
  for (int i = 0; i < count; ++i) {
    const std::size_t nb = std::size_t(batch) * layers[i]->n, mb = std::size_t(batch) * layers[i]->m;
    const bool xin = i == 0 && x0_mapped, yout = i == count - 1 && ylast_mapped;
    if (!xin) cuda_check(cudaStreamWaitEvent(s, aux.ev[2 + i], 0), "H2D wait");
    forward_impl(layers[i], xin ? x0_mapped : dx + xo, yout ? ylast_mapped + yo : dy + yo, batch, ws, ws_bytes, s);
    if (!yout) {
      cuda_check(cudaEventRecord(aux.ev[2 + count + i], s), "layer event");
      cudaStream_t ds = duplex ? aux.side2 : aux.side;
      cuda_check(cudaStreamWaitEvent(ds, aux.ev[2 + count + i], 0), "layer wait");
      cuda_check(cudaMemcpyAsync(yh + yo, dy + yo, mb * 4, cudaMemcpyDeviceToHost, ds), "set D2H");
    }
    xo += nb;
    yo += mb;
  }
  cuda_check(cudaEventRecord(join, aux.side), "join");
  cuda_check(cudaStreamWaitEvent(s, join, 0), "join wait");
  if (duplex) {
    cuda_check(cudaEventRecord(join2, aux.side2), "join");
    cuda_check(cudaStreamWaitEvent(s, join2, 0), "join wait");
  }
}

// Device-side address of pinned (page-locked, mapped) host memory, or nullptr.
void* mapped_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

void forward_set_host_impl(const q8p_layer* const* layers, int count, const float* xh, float* yh, int batch, void* ws,
                           std::size_t ws_bytes, cudaStream_t s, unsigned flags) {
  check_set(layers, count, batch);
  if (count == 0 || batch == 0) return;
  if (!xh || !yh) throw ValidationError("null host x / y");
  if (!ws || ws_bytes < set_workspace_size(layers, count, batch, flags)) throw SizeError("workspace too small");
  const int dev = layers[0]->device;
  DeviceGuard g(dev);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(s, &cap), "capture status");
  const auto* dxh = static_cast<const float*>(mapped_ptr(xh));
  auto* dyh = static_cast<float*>(mapped_ptr(yh));
  const bool ends = dxh && dyh && !(flags & Q8P_SET_CONCURRENT);
  auto enqueue = [&](cudaStream_t st) {
    forward_set_host_enqueue(layers, count, xh, yh, batch, ws, ws_bytes, st, flags, ends ? dxh : nullptr,
                             ends ? dyh : nullptr);
  };
  if (cap != cudaStreamCaptureStatusNone || !dxh || !dyh || dev < 0 || dev >= 64) {
    enqueue(s);
    cuda_check(cudaStreamSynchronize(s), "set sync");
    return;
  }
  cudaGraphExec_t exec = nullptr;
  {
    std::scoped_lock lock(g_set_mu);
    for (const auto& e : g_set_graphs)
      if (e.xh == xh && e.yh == yh && e.batch == batch && e.ws == ws && e.ws_bytes == ws_bytes && e.device == dev &&
          e.flags == flags &&
          e.layers.size() == std::size_t(count) && std::equal(e.layers.begin(), e.layers.end(), layers))
        exec = e.exec;
    if (!exec) {
      if (!g_set_capture[dev])
        cuda_check(cudaStreamCreateWithFlags(&g_set_capture[dev], cudaStreamNonBlocking), "capture stream");
      cudaStream_t cs = g_set_capture[dev];
      cudaGraph_t graph = nullptr;
      const std::uint64_t k0 = g_launches.load();
      cuda_check(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        enqueue(cs);
      } catch (...) {
        cudaStreamEndCapture(cs, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      cuda_check(cudaStreamEndCapture(cs, &graph), "end capture");
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      cuda_check(ie, "graph instantiate");
      if (g_set_graphs.size() >= 256) {  // bounded (a model's layer sets x rotating copies): evict the oldest
        cudaGraphExecDestroy(g_set_graphs.front().exec);
        g_set_graphs.erase(g_set_graphs.begin());
      }
      const std::uint64_t k = g_launches.load() - k0;
      g_launches.fetch_sub(k);  // counted per replay below
      g_set_graphs.push_back({std::vector<const q8p_layer*>(layers, layers + count), xh, yh, batch, ws, ws_bytes, dev,
                              flags, exec, k});
    }
    for (const auto& e : g_set_graphs)
      if (e.exec == exec) g_launches.fetch_add(e.kernels, std::memory_order_relaxed);
  }
  cuda_check(cudaGraphLaunch(exec, s), "graph launch");
  cuda_check(cudaStreamSynchronize(s), "set sync");
}

// Drops cached layer-set graphs that reference `L` (q8p_layer_destroy).
void forget_set_graphs(const q8p_layer* L) {
  std::scoped_lock lock(g_set_mu);
  for (auto it = g_set_graphs.begin(); it != g_set_graphs.end();) {
    if (std::find(it->layers.begin(), it->layers.end(), L) != it->layers.end()) {
      cudaGraphExecDestroy(it->exec);
      it = g_set_graphs.erase(it);
    } else {
      ++it;
    }
  }
}

}  // namespace
}  // namespace q8p::detail

using namespace q8p::detail;

extern "C" {

const char* q8p_version(void) { return "q8p 0.1.0 (sm_100a)"; }

const char* q8p_status_string(q8p_status s) {
  switch (s) {
    case Q8P_OK: return "ok";
    case Q8P_ERR_SIZE: return "size error";
    case Q8P_ERR_VALIDATION: return "validation error";
    case Q8P_ERR_FORMAT: return "format error";
    case Q8P_ERR_BAD_MAGIC: return "bad magic";
    case Q8P_ERR_UNSUPPORTED_VERSION: return "unsupported version";
    case Q8P_ERR_TRUNCATED: return "truncated artifact";
    case Q8P_ERR_UNSUPPORTED: return "unsupported on this path";
    case Q8P_ERR_CUDA: return "CUDA error";
    case Q8P_ERR_NCCL: return "NCCL error";
    default: return "internal error";
  }
}

const char* q8p_last_error(void) { return q8p::detail::t_last_error.c_str(); }

uint64_t q8p_kernel_launches(void) { return g_launches.load(); }

q8p_status q8p_plan_hadamard(size_t n, size_t* p, size_t* q) {
  try {
    const q8p::HadamardSpec s = q8p::plan_hadamard(n);
    if (p) *p = s.p;
    if (q) *q = s.q;
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_layer_create(const q8p_layer_desc* desc, int device, q8p_layer** out) {
  try {
    if (!desc || !out) throw q8p::ValidationError("null argument");
    *out = build_layer(*desc, 0, desc->m, device);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_layer_from_qshp(const uint8_t* bytes, size_t len, int device, q8p_layer** out) {
  try {
    if (!bytes || !out) throw q8p::ValidationError("null argument");
    *out = layer_from_bytes(bytes, len, 0, 0, true, device);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_layers_from_qshp(const uint8_t* const* bytes, const size_t* lens, int count, int device,
                                q8p_layer** out) {
  std::vector<q8p_layer*> made;
  try {
    if (count < 0) throw q8p::ValidationError("negative layer count");
    if (count > 0 && (!bytes || !lens || !out)) throw q8p::ValidationError("null argument");
    for (int i = 0; i < count; ++i) {
      if (!bytes[i]) throw q8p::ValidationError("null artifact");
      out[i] = nullptr;
    }
    // Every artifact is parsed and uploaded on its own worker thread (its own
    // private upload stream): one layer's host-side deserialize overlaps another's
    // H2D copies and device transcode.  At most kLoadWorkers in flight.
    constexpr int kLoadWorkers = 4;
    std::vector<std::future<q8p_layer*>> jobs;
    std::string first_error;
    q8p_status first_status = Q8P_OK;
    auto collect = [&](std::future<q8p_layer*>& f) {
      try {
        made.push_back(f.get());
      } catch (...) {
        const q8p_status st = status_of_current_exception();
        if (first_status == Q8P_OK) first_status = st, first_error = q8p_last_error();
        made.push_back(nullptr);
      }
    };
    for (int i = 0; i < count; ++i) {
      if (int(jobs.size()) - int(made.size()) >= kLoadWorkers) collect(jobs[made.size()]);
      jobs.push_back(std::async(std::launch::async, [=] { return layer_from_bytes(bytes[i], lens[i], 0, 0, true, device); }));
    }
    while (made.size() < jobs.size()) collect(jobs[made.size()]);
    if (first_status != Q8P_OK) {
      for (q8p_layer* L : made) q8p_layer_destroy(L);
      set_last_error(first_error);
      return first_status;
    }
    for (int i = 0; i < count; ++i) out[i] = made[i];
    return Q8P_OK;
  } catch (...) {
    for (q8p_layer* L : made) q8p_layer_destroy(L);
    return status_of_current_exception();
  }
}

q8p_status q8p_layer_from_qshp_rows(const uint8_t* bytes, size_t len, uint32_t row_begin,
                                    uint32_t row_end, int device, q8p_layer** out) {
  try {
    if (!bytes || !out) throw q8p::ValidationError("null argument");
    *out = layer_from_bytes(bytes, len, row_begin, row_end, false, device);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

void q8p_layer_destroy(q8p_layer* L) {
  if (!L) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(L->device);
  for (auto& e : L->graphs) cudaGraphExecDestroy(e.exec);
  L->graphs.clear();
  forget_set_graphs(L);
  if (L->capture_stream) cudaStreamDestroy(L->capture_stream);
  for (void* p : L->allocations) cudaFree(p);
  for (q8p_layer::Stage* st : L->stage_all) {
    if (st->dev) cudaFree(st->dev);
    if (st->host) cudaFreeHost(st->host);
    if (st->stream) cudaStreamDestroy(st->stream);
    delete st;
  }
  cudaSetDevice(prev);
  delete L;
}

q8p_status q8p_layer_get_info(const q8p_layer* L, q8p_layer_info* info) {
  if (!L || !info) {
    set_last_error("null argument");
    return Q8P_ERR_VALIDATION;
  }
  info->m = L->m;
  info->n = L->n;
  info->row_begin = L->row_begin;
  info->row_end = L->row_end;
  info->num_stages = L->num_stages;
  info->device = L->device;
  info->device_bytes = L->device_bytes;
  info->code_bytes = L->code_bytes;
  return Q8P_OK;
}

size_t q8p_workspace_bytes(const q8p_layer* L, int batch) {
  if (!L || batch <= 0) return 0;
  return workspace_size(L, batch);
}

q8p_status q8p_forward(const q8p_layer* L, const float* x, float* y, int batch, void* ws,
                       size_t ws_bytes, void* stream) {
  try {
    forward_cached(const_cast<q8p_layer*>(L), x, y, batch, ws, ws_bytes, static_cast<cudaStream_t>(stream));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_forward_ex(const q8p_layer* L, const float* x, float* y, int batch, void* ws,
                          size_t ws_bytes, void* stream, const q8p_forward_opts* opts) {
  try {
    forward_impl(L, x, y, batch, ws, ws_bytes, static_cast<cudaStream_t>(stream), opts);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

size_t q8p_forward_set_workspace_bytes_ex(const q8p_layer* const* layers, int count, int batch, unsigned flags) {
  try {
    check_set(layers, count, batch);
    return count > 0 && batch > 0 ? set_workspace_size(layers, count, batch, flags) : 0;
  } catch (...) {
    status_of_current_exception();
    return 0;
  }
}
size_t q8p_forward_set_workspace_bytes(const q8p_layer* const* layers, int count, int batch) {
  return q8p_forward_set_workspace_bytes_ex(layers, count, batch, 0);
}

q8p_status q8p_forward_set_ex(const q8p_layer* const* layers, int count, const float* const* x, float* const* y,
                              int batch, void* ws, size_t ws_bytes, void* stream, unsigned flags) {
  try {
    check_set(layers, count, batch);
    if (count > 0 && (!x || !y)) throw q8p::ValidationError("null x / y lists");
    forward_set_impl(layers, count, x, y, batch, ws, ws_bytes, static_cast<cudaStream_t>(stream), flags);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}
q8p_status q8p_forward_set(const q8p_layer* const* layers, int count, const float* const* x, float* const* y,
                           int batch, void* ws, size_t ws_bytes, void* stream) {
  return q8p_forward_set_ex(layers, count, x, y, batch, ws, ws_bytes, stream, 0);
}

q8p_status q8p_forward_set_host_ex(const q8p_layer* const* layers, int count, const float* x_host, float* y_host,
                                   int batch, void* ws, size_t ws_bytes, void* stream, unsigned flags) {
  try {
    forward_set_host_impl(layers, count, x_host, y_host, batch, ws, ws_bytes, static_cast<cudaStream_t>(stream),
                          flags);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}
q8p_status q8p_forward_set_host(const q8p_layer* const* layers, int count, const float* x_host, float* y_host,
                                int batch, void* ws, size_t ws_bytes, void* stream) {
  return q8p_forward_set_host_ex(layers, count, x_host, y_host, batch, ws, ws_bytes, stream, 0);
}

q8p_status q8p_e8p_encode(const double* v, uint16_t* words, size_t nblocks, int device, void* stream) {
  try {
    if (nblocks == 0) return Q8P_OK;
    if (!v || !words) throw q8p::ValidationError("null v / words");
    require_sm100(device);
    DeviceGuard g(device);
    launch_e8p_encode(v, words, nblocks, static_cast<cudaStream_t>(stream));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_rht_cols_f64(double* w, double* scratch, size_t rows, size_t cols, const uint8_t* signs, int device,
                            void* stream) {
  try {
    if (rows == 0 || cols == 0) return Q8P_OK;
    if (!w || !scratch || !signs) throw q8p::ValidationError("null argument");
    q8p::plan_hadamard(rows);
    require_sm100(device);
    DeviceGuard g(device);
    launch_rht_cols_f64(w, scratch, std::uint32_t(rows), std::uint32_t(cols), signs, static_cast<cudaStream_t>(stream));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_rvq_quantize(const double* v, uint16_t* codes, size_t nblocks, int num_stages,
                            const q8p_codebook* codebooks, const double* scales, int device, void* stream) {
  try {
    if (nblocks == 0) return Q8P_OK;
    if (!v || !codes || !codebooks || !scales) throw q8p::ValidationError("null argument");
    if (num_stages < 1 || num_stages > 2) throw q8p::ValidationError("1 or 2 RVQ stages on this path");
    int kinds[2] = {0, 0};
    for (int i = 0; i < num_stages; ++i) kinds[i] = codebooks[i] == Q8P_CB_E8P_2BIT ? 0 : 1;
    require_sm100(device);
    DeviceGuard g(device);
    launch_rvq_quantize(v, codes, nblocks, num_stages, kinds, scales, static_cast<cudaStream_t>(stream));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_infer_host(q8p_layer* L, const double* x, double* y, int batch) {
  try {
    if (!L || !x || !y) throw q8p::ValidationError("null argument");
    if (batch <= 0) return Q8P_OK;
    DeviceGuard g(L->device);
    q8p_layer::Stage* st = nullptr;
    {
      std::scoped_lock lock(L->stage_mu);
      if (!L->stage_free.empty()) {
        st = L->stage_free.back();
        L->stage_free.pop_back();
      } else {
        st = new q8p_layer::Stage();
        L->stage_all.push_back(st);
      }
    }
    struct Release {  // the context goes back to the pool on every exit path
      q8p_layer* L;
      q8p_layer::Stage* st;
      ~Release() {
        std::scoped_lock lock(L->stage_mu);
        L->stage_free.push_back(st);
      }
    } release{L, st};
    if (!st->stream) cuda_check(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking), "stream");
    const std::size_t xin = std::size_t(batch) * L->n, yout = std::size_t(batch) * L->m;
    const std::size_t host_need = (xin + yout) * sizeof(float);
    if (st->host_bytes < host_need) {
      if (st->host) cudaFreeHost(st->host);
      st->host = nullptr;
      st->host_bytes = 0;
      cuda_check(cudaMallocHost(&st->host, host_need), "cudaMallocHost");
      st->host_bytes = host_need;
    }
    const std::size_t ws = workspace_size(L, batch);
    const std::size_t dev_need = round_up(xin * 4, 256) + round_up(yout * 4, 256) + ws;
    if (st->dev_bytes < dev_need) {
      if (st->dev) cudaFree(st->dev);
      st->dev = nullptr;
      st->dev_bytes = 0;
      cuda_check(cudaMalloc(&st->dev, dev_need), "cudaMalloc stage");
      st->dev_bytes = dev_need;
    }
    float* hx = static_cast<float*>(st->host);
    float* hy = hx + xin;
    for (std::size_t i = 0; i < xin; ++i) hx[i] = static_cast<float>(x[i]);
    auto* dbase = static_cast<std::uint8_t*>(st->dev);
    float* dx = reinterpret_cast<float*>(dbase);
    float* dy = reinterpret_cast<float*>(dbase + round_up(xin * 4, 256));
    void* dws = dbase + round_up(xin * 4, 256) + round_up(yout * 4, 256);
    cuda_check(cudaMemcpyAsync(dx, hx, xin * 4, cudaMemcpyHostToDevice, st->stream), "H2D");
    forward_impl(L, dx, dy, batch, dws, ws, st->stream);
    cuda_check(cudaMemcpyAsync(hy, dy, yout * 4, cudaMemcpyDeviceToHost, st->stream), "D2H");
    cuda_check(cudaStreamSynchronize(st->stream), "sync");
    for (std::size_t i = 0; i < yout; ++i) y[i] = static_cast<double>(hy[i]);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_decode_stage(const q8p_layer* L, int stage, float* w_hat, void* stream) {
  try {
    if (!L || !w_hat) throw q8p::ValidationError("null argument");
    if (stage < 0 || stage >= L->num_stages) throw q8p::ValidationError("stage out of range");
    DeviceGuard g(L->device);
    // K2's own decoder over the slabs (q8p_k2_decode_stage), then the points as fp32
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const std::size_t total = std::size_t(L->m_local()) * L->n;
    void* tmp = nullptr;
    cuda_check(cudaMallocAsync(&tmp, total + total / 8 + 16, s), "decode scratch");
    auto* a = static_cast<std::int8_t*>(tmp);
    auto* b = reinterpret_cast<std::uint8_t*>(a + total);
    const int kind = L->cb[stage] == Q8P_CB_E8P_2BIT ? 0 : 1;
    launch_k2_decode(*L, stage, a, b, s);
    launch_points_f32(a, b, kind, total, w_hat, s);
    cuda_check(cudaFreeAsync(tmp, s), "decode scratch free");
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_bench_gemv(const q8p_layer* L, int batch, void* ws, size_t ws_bytes, int reps, void* stream) {
  try {
    if (!L || !ws) throw q8p::ValidationError("null argument");
    if (reps <= 0) return Q8P_OK;
    if (!tc_supported(*L, batch)) throw q8p::UnsupportedError("bench_gemv needs the tensor-core path (batch <= 32)");
    if (ws_bytes < workspace_size(L, batch)) throw q8p::SizeError("workspace too small");
    DeviceGuard g(L->device);
    Workspace w;
    workspace_parts(L, batch, &w, ws);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int r = 0; r < reps; ++r) launch_gemv_tc(*L, w.bimg, w.zacc, w.rows_pad, batch, s);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_bench_stream(const void* src, size_t bytes, int reps, void* stream) {
  try {
    if (!src) throw q8p::ValidationError("null argument");
    for (int r = 0; r < reps; ++r) launch_stream(src, bytes, nullptr, static_cast<cudaStream_t>(stream));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_layer_code_region(const q8p_layer* L, int stage, const void** codes, size_t* bytes) {
  try {
    if (!L || !codes || !bytes) throw q8p::ValidationError("null argument");
    if (stage < 0 || stage >= L->num_stages) throw q8p::ValidationError("stage out of range");
    *codes = L->tc[stage].codes;
    *bytes = tc_code_bytes(L->m_local(), L->n, L->cb[stage] == Q8P_CB_E8P_2BIT ? 0 : 1);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_dequantize(const q8p_layer* L, double* w_tilde, double* scratch, void* stream) {
  try {
    if (!L || !w_tilde || !scratch) throw q8p::ValidationError("null argument");
    if (L->row_begin != 0 || L->row_end != L->m) throw q8p::ValidationError("dequantize needs the full (unsharded) layer");
    if (L->side_u.kind != 0 || L->side_v.kind != 0)
      throw q8p::UnsupportedError("dequantize: rfft transforms are not on the f64 device path");
    DeviceGuard g(L->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const std::size_t total = std::size_t(L->m) * L->n, codes = total / 8;
    // decode_incoherent (pipeline.cpp:112-138): K2's decoder output per stage in the
    // scratch (2 x (m n + m n / 8) bytes <= 8 m n), combined in f64
    auto* base = reinterpret_cast<std::uint8_t*>(scratch);
    std::int8_t* a[2] = {reinterpret_cast<std::int8_t*>(base), reinterpret_cast<std::int8_t*>(base + total)};
    std::uint8_t* b[2] = {base + 2 * total, base + 2 * total + codes};
    for (int st = 0; st < L->num_stages; ++st) launch_k2_decode(*L, st, a[st], b[st], s);
    const int k0 = L->cb[0] == Q8P_CB_E8P_2BIT ? 0 : 1, k1 = L->cb[1] == Q8P_CB_E8P_2BIT ? 0 : 1;
    launch_dequant_combine(a[0], b[0], a[1], b[1], L->num_stages, k0, k1, double(L->scale[0]), double(L->scale[1]),
                           total, w_tilde, s);
    // dequantize_layer (pipeline.cpp:142-149): transform_cols(left, transpose), then
    // transform_rows(right, transpose) through an f64 transpose
    launch_rht_cols_f64(w_tilde, scratch, L->m, L->n, L->side_u.signs, s, true);
    launch_transpose_f64(w_tilde, scratch, L->m, L->n, s);
    launch_rht_cols_f64(scratch, w_tilde, L->n, L->m, L->side_v.signs, s, true);
    launch_transpose_f64(scratch, w_tilde, L->n, L->m, s);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_k2_decode_stage(const q8p_layer* L, int stage, int8_t* a_bytes, uint8_t* shift_bits, void* stream) {
  try {
    if (!L || !a_bytes) throw q8p::ValidationError("null argument");
    if (stage < 0 || stage >= L->num_stages) throw q8p::ValidationError("stage out of range");
    if (L->cb[stage] == Q8P_CB_E8P_2BIT && !shift_bits) throw q8p::ValidationError("E8P stage needs shift_bits");
    DeviceGuard g(L->device);
    launch_k2_decode(*L, stage, a_bytes, shift_bits, static_cast<cudaStream_t>(stream));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_rht(size_t n, const uint8_t* signs, const float* x, float* y, int batch, int transpose,
                   void* stream) {
  try {
    if (!signs || !x || !y) throw q8p::ValidationError("null argument");
    if (batch < 0) throw q8p::ValidationError("negative batch");
    if (batch == 0) return Q8P_OK;
    const q8p::HadamardSpec spec = q8p::plan_hadamard(n);
    DevSide side;
    side.n = static_cast<std::uint32_t>(n);
    side.p = static_cast<std::uint32_t>(spec.p);
    side.q = static_cast<std::uint32_t>(spec.q);
    side.signs = signs;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    // Per-(device, order) copies of the base, cached per process.
    static std::mutex mu;
    struct BaseCopy {
      int device;
      std::size_t q;
      void* ptr;
    };
    static std::vector<BaseCopy> bases;
    if (spec.q > 1) {
      const int dev = current_device();
      std::scoped_lock lock(mu);
      for (const BaseCopy& e : bases)
        if (e.device == dev && e.q == spec.q) side.base = static_cast<const std::int8_t*>(e.ptr);
      if (!side.base) {
        const auto& b = q8p::detail::hadamard_base(spec.q);
        void* d = nullptr;
        cuda_check(cudaMalloc(&d, b.size()), "cudaMalloc base");
        cuda_check(cudaMemcpy(d, b.data(), b.size(), cudaMemcpyHostToDevice), "base upload");
        bases.push_back({dev, spec.q, d});
        side.base = static_cast<const std::int8_t*>(d);
      }
    }
    if (n % 4 != 0) {  // tiny dims (n = 1, 2): single-CTA transform
      launch_rht(side, x, y, batch, transpose != 0, s);
      return Q8P_OK;
    }
    // Scratch for the two-pass transforms (and the amax the forward pass reports):
    // stream-ordered (cudaMallocAsync / cudaFreeAsync on `s`), so calls on other
    // streams or devices never share it and it is capturable in a graph.
    const std::size_t need = std::size_t(batch) * n * 4 + 256;
    void* scratch = nullptr;
    cuda_check(cudaMallocAsync(&scratch, need, s), "cudaMallocAsync rht scratch");
    float* u = static_cast<float*>(scratch);
    float* amax = reinterpret_cast<float*>(static_cast<std::uint8_t*>(scratch) + std::size_t(batch) * n * 4);
    try {
      if (!transpose) {
        launch_rht_in(side, x, y, u, amax, nullptr, nullptr, 0, batch, s);
      } else {
        launch_rht_out(side, x, u, y, batch, s);
      }
    } catch (...) {
      cudaFreeAsync(scratch, s);
      throw;
    }
    cuda_check(cudaFreeAsync(scratch, s), "cudaFreeAsync rht scratch");
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_qshp_inspect(const uint8_t* bytes, size_t len, q8p_artifact_info* info) {
  try {
    if (!bytes || !info) throw q8p::ValidationError("null argument");
    const q8p::QuantizedLinear a = q8p::deserialize(std::span(bytes, len));
    *info = q8p_artifact_info{};
    info->m = a.m;
    info->n = a.n;
    info->transform = static_cast<int>(a.transform);
    info->num_stages = static_cast<int>(a.stages.size());
    for (std::size_t s = 0; s < a.stages.size() && s < 8; ++s) {
      info->codebook[s] = a.stages[s].codebook == "e8p-2bit" ? Q8P_CB_E8P_2BIT : Q8P_CB_E8_1BIT;
      info->scale[s] = a.stages[s].scale;
    }
    info->serialized_size = q8p::serialized_size(a);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_qshp_reserialize(const uint8_t* bytes, size_t len, uint8_t* out, size_t cap,
                                size_t* out_len) {
  try {
    if (!bytes || !out_len) throw q8p::ValidationError("null argument");
    const std::vector<std::uint8_t> b = q8p::serialize(q8p::deserialize(std::span(bytes, len)));
    *out_len = b.size();
    if (!out || cap < b.size()) throw q8p::SizeError("output buffer too small");
    std::memcpy(out, b.data(), b.size());
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_e8p_decode_host(uint16_t word, float out[8]) {
  try {
    if (!out) throw q8p::ValidationError("null argument");
    q8p::detail::e8p_decode_host(word, out);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_codebook_table(q8p_codebook cb, int8_t* doubled, uint8_t* parity_out) {
  try {
    if (!doubled) throw q8p::ValidationError("null argument");
    if (cb == Q8P_CB_E8P_2BIT) {
      const auto& t = q8p::detail::e8p_table();
      for (int i = 0; i < 256; ++i) {
        for (int c = 0; c < 8; ++c) doubled[i * 8 + c] = t.doubled[i][c];
        if (parity_out) parity_out[i] = t.odd_parity[i];
      }
    } else if (cb == Q8P_CB_E8_1BIT) {
      const auto& t = q8p::detail::e8_1bit_doubled();
      for (int i = 0; i < 256; ++i)
        for (int c = 0; c < 8; ++c) doubled[i * 8 + c] = t[i][c];
    } else {
      throw q8p::ValidationError("unknown codebook");
    }
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_hadamard_base(size_t q, int8_t* out) {
  try {
    if (!out) throw q8p::ValidationError("null argument");
    const auto& b = q8p::detail::hadamard_base(q);
    std::memcpy(out, b.data(), b.size());
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_forward_rows_z(const q8p_layer* L, const float* x, float* z, int batch, void* ws, size_t ws_bytes,
                              void* stream) {
  try {
    if (!L || !x || !z) throw q8p::ValidationError("null argument");
    if (batch <= 0) return Q8P_OK;
    if (!tc_supported(*L, batch)) throw q8p::UnsupportedError("rows_z needs the tensor-core path (batch <= 32)");
    if (!ws || ws_bytes < workspace_size(L, batch)) throw q8p::SizeError("workspace too small");
    DeviceGuard g(L->device);
    Workspace w;
    workspace_parts(L, batch, &w, ws);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    forward_local(L, x, batch, w, s, nullptr);
    float zscale[2] = {L->scale[0], L->scale[1]};
    int ze8p[2] = {L->cb[0] == Q8P_CB_E8P_2BIT, L->cb[1] == Q8P_CB_E8P_2BIT};
    launch_combine_acc(w.zacc, L->num_stages, w.rows_pad, w.zcols, zscale, ze8p, w.alpha, w.tl, z, L->m_local(), batch,
                       s);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_forward_sharded(const q8p_layer* L, const float* x, float* y, int batch, void* ws, size_t ws_bytes,
                               void* nccl_comm, void* stream) {
  try {
    forward_sharded_impl(L, x, y, batch, ws, ws_bytes, static_cast<ncclComm_t>(nccl_comm),
                         static_cast<cudaStream_t>(stream));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}
q8p_status q8p_forward_sharded_sim(const q8p_layer* const* shards, int world, const float* x, float* y, int batch,
                                   void* ws, size_t ws_bytes, void* stream) {
  try {
    if (!shards || world < 1 || !x || !y || !ws) throw q8p::ValidationError("null argument");
    if (batch <= 0) return Q8P_OK;
    const q8p_layer* L0 = shards[0];
    if (!L0) throw q8p::ValidationError("null layer");
    const std::uint32_t ml = L0->m_local();
    for (int r = 0; r < world; ++r) {
      const q8p_layer* L = shards[r];
      if (!L || L->m != L0->m || L->n != L0->n || L->m_local() != ml || L->row_begin != std::uint32_t(r) * ml ||
          L->device != L0->device)
        throw q8p::ValidationError("shards must be the equal, rank-ordered row ranges of one layer");
    }
    if (std::size_t(ml) * world != L0->m) throw q8p::ValidationError("shards do not cover the layer");
    if (!tc_supported(*L0, batch)) throw q8p::UnsupportedError("sharded simulation: batch <= 32 on the tensor-core path");
    if (!rht_sharded_k3_ok(L0->side_u, 0, ml)) throw q8p::UnsupportedError("sharded simulation: rows not whole chunks");
    if (ws_bytes < workspace_size(L0, batch)) throw q8p::SizeError("workspace too small");
    DeviceGuard g(L0->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    float zscale[2] = {L0->scale[0], L0->scale[1]};
    int ze8p[2] = {L0->cb[0] == Q8P_CB_E8P_2BIT, L0->cb[1] == Q8P_CB_E8P_2BIT};
    Workspace w;
    for (int r = 0; r < world; ++r) {  // each rank's part of q8p_forward_sharded, in turn
      const q8p_layer* L = shards[r];
      workspace_parts(L, batch, &w, ws);
      forward_local(L, x, batch, w, s, nullptr);
      launch_rht_out_acc_local(L->side_u, w.zacc, L->num_stages, w.rows_pad, std::uint32_t(tc_ncols_pad(4 * batch)),
                               zscale, ze8p, w.alpha, w.tl, L->row_begin, ml, w.z_loc, batch, s);
      // the all-gather's data movement: rank r's slice -> [r][batch][m_local]
      cuda_check(cudaMemcpyAsync(w.z_full + std::size_t(r) * batch * ml, w.z_loc, std::size_t(batch) * ml * 4,
                                 cudaMemcpyDeviceToDevice, s),
                 "gather copy");
    }
    launch_rht_out_pass2_gathered(L0->side_u, w.z_full, ml, y, batch, s);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_peers_create(int device, int world, int rank, size_t slice_floats, q8p_peers** out,
                            uint8_t handle[Q8P_PEER_HANDLE_BYTES]) {
  q8p_peers* p = nullptr;
  try {
    if (!out || !handle) throw q8p::ValidationError("null argument");
    *out = nullptr;
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world) throw q8p::ValidationError("bad world / rank");
    if (slice_floats == 0 || slice_floats % 4 != 0) throw q8p::ValidationError("slice_floats must be a positive multiple of 4");
    DeviceGuard g(device);
    p = new q8p_peers;
    p->device = device;
    p->world = world;
    p->rank = rank;
    p->slice_floats = slice_floats;
    const std::size_t bytes = peer_bytes(world, slice_floats);
    cuda_check(cudaMalloc(&p->base, bytes), "cudaMalloc peer window");
    {  // tag 0 is never a call's tag; private stream: no legacy-stream / device-wide sync
      cudaStream_t st = nullptr;
      cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "peer init stream");
      const cudaError_t e1 = cudaMemsetAsync(p->base, 0, bytes, st);
      const cudaError_t e2 = cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
      cuda_check(e1, "peer window init");
      cuda_check(e2, "peer window init");
    }
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&p->d_wins), sizeof(void*) * world), "cudaMalloc peer table");
    static_assert(sizeof(cudaIpcMemHandle_t) <= Q8P_PEER_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, p->base), "cudaIpcGetMemHandle");
    std::memset(handle, 0, Q8P_PEER_HANDLE_BYTES);
    std::memcpy(handle, &h, sizeof(h));
    *out = p;
    return Q8P_OK;
  } catch (...) {
    if (p) q8p_peers_destroy(p);
    return status_of_current_exception();
  }
}

q8p_status q8p_peers_connect(q8p_peers* p, const uint8_t* handles) {
  try {
    if (!p || !handles) throw q8p::ValidationError("null argument");
    if (p->connected) throw q8p::ValidationError("peers already connected");
    DeviceGuard g(p->device);
    std::vector<void*> bases(p->world);
    for (int r = 0; r < p->world; ++r) {
      if (r == p->rank) {
        bases[r] = p->base;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + std::size_t(r) * Q8P_PEER_HANDLE_BYTES, sizeof(h));
      void* ptr = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      p->opened.push_back(ptr);
      bases[r] = ptr;
    }
    peers_set_bases(p, bases);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_peers_connect_local(q8p_peers* const* group, int world) {
  try {
    if (!group || world < 1) throw q8p::ValidationError("null argument");
    std::vector<void*> bases(world);
    for (int r = 0; r < world; ++r) {
      if (!group[r] || group[r]->world != world || group[r]->rank != r || group[r]->device != group[0]->device ||
          group[r]->slice_floats != group[0]->slice_floats || group[r]->connected)
        throw q8p::ValidationError("peers must be the unconnected, rank-ordered members of one group on one device");
      bases[r] = group[r]->base;
    }
    DeviceGuard g(group[0]->device);
    for (int r = 0; r < world; ++r) peers_set_bases(group[r], bases);
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_peers_state(const q8p_peers* p, uint64_t* epoch) {
  try {
    if (!p || !epoch) throw q8p::ValidationError("null argument");
    DeviceGuard g(p->device);
    PeerCtl c;
    cuda_check(cudaMemcpy(&c, p->base, sizeof(c), cudaMemcpyDeviceToHost), "peer state read");
    *epoch = c.epoch;
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_peers_destroy(q8p_peers* p) {
  if (!p) return Q8P_OK;
  try {
    DeviceGuard g(p->device);
    cudaDeviceSynchronize();
    for (void* ptr : p->opened) cudaIpcCloseMemHandle(ptr);
    if (p->d_wins) cudaFree(p->d_wins);
    if (p->base) cudaFree(p->base);
    delete p;
    return Q8P_OK;
  } catch (...) {
    delete p;
    return status_of_current_exception();
  }
}

q8p_status q8p_forward_sharded_push(const q8p_layer* L, q8p_peers* peers, const float* x, float* y, int batch,
                                    void* ws, size_t ws_bytes, void* stream) {
  try {
    forward_push_impl(L, peers, x, y, batch, ws, ws_bytes, static_cast<cudaStream_t>(stream));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_forward_sharded_push_sim(const q8p_layer* const* shards, q8p_peers* const* peers, int world,
                                        const float* x, float* y, int batch, void* ws, size_t ws_bytes,
                                        void* stream) {
  try {
    if (!shards || !peers || world < 1 || !x || !y || !ws) throw q8p::ValidationError("null argument");
    if (batch <= 0) return Q8P_OK;
    for (int r = 0; r < world; ++r) {
      if (!peers[r] || peers[r]->world != world || peers[r]->rank != r) throw q8p::ValidationError("peers out of order");
      check_push_layer(shards[r], peers[r], batch);
      if (shards[r]->m != shards[0]->m || shards[r]->n != shards[0]->n)
        throw q8p::ValidationError("shards of different layers");
      if (ws_bytes < workspace_size(shards[r], batch)) throw q8p::SizeError("workspace too small");
    }
    const q8p_layer* L0 = shards[0];
    DeviceGuard g(L0->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Workspace w;
    if (use_prefill_rows(L0, batch)) {  // prefill: every rank's K1, K4, pushing pass 1; then every pass 2
      for (int r = 0; r < world; ++r) {
        const q8p_layer* L = shards[r];
        workspace_parts(L, batch, &w, ws);
        const PushArgs pa = peers[r]->args();
        launch_rht_in(L->side_v, x, w.pt, w.u, prefill_amax(*L, batch, w.pbt), nullptr, nullptr, 0, batch, s);
        launch_prefill(*L, w.pt, w.pbt, w.pz, batch, s);
        const K4Sched ks = prefill_sched(*L, batch);
        launch_rht_out_local_f32(L->side_u, w.pz, int(ks.slices), L->row_begin, L->m_local(), nullptr, &pa, batch,
                                 s, &ks);
      }
      for (int r = 0; r < world; ++r)
        launch_rht_out_pass2_push(L0->side_u, L0->m_local(), peers[r]->args(), y + std::size_t(r) * batch * L0->m,
                                  batch, s);
      return Q8P_OK;
    }
    const int chunk = tc_chunk(L0, batch);
    for (int b0 = 0; b0 < batch; b0 += chunk) {
      const int nb = std::min(chunk, batch - b0);
      // every rank's K1, K2 and pushing pass 1 in turn, then every rank's pass 2
      // (each waits for all ranks' arrivals, already complete in stream order)
      for (int r = 0; r < world; ++r) {
        workspace_parts(shards[r], batch, &w, ws);
        forward_local(shards[r], x + std::size_t(b0) * L0->n, nb, w, s, nullptr);
        k3_push(shards[r], w, peers[r]->args(), nb, s);
      }
      for (int r = 0; r < world; ++r)
        launch_rht_out_pass2_push(L0->side_u, L0->m_local(), peers[r]->args(),
                                  y + (std::size_t(r) * batch + b0) * L0->m, nb, s);
    }
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

q8p_status q8p_nccl_unique_id(uint8_t out[128]) {
  try {
    if (!out) throw q8p::ValidationError("null argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}
q8p_status q8p_nccl_comm_init(const uint8_t id[128], int world, int rank, int device, void** comm) {
  try {
    if (!id || !comm) throw q8p::ValidationError("null argument");
    if (world <= 0 || rank < 0 || rank >= world) throw q8p::ValidationError("bad world / rank");
    DeviceGuard g(device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    nccl_check(ncclCommInitRank(&c, world, uid, rank), "ncclCommInitRank");
    *comm = c;
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}
q8p_status q8p_nccl_comm_destroy(void* comm) {
  try {
    if (comm) nccl_check(ncclCommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
    return Q8P_OK;
  } catch (...) {
    return status_of_current_exception();
  }
}

}  // extern "C"
