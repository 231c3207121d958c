/* q8p -- B200-native (sm_100a) QuIP# quantized-linear inference.
 *
 * C ABI: the drop-in boundary for the reference `latq` library's inference
 * path.  Plain pointers and sizes only; no exceptions cross this boundary
 * (every entry point returns a q8p_status; q8p_last_error() holds the
 * message of the calling thread's last failure).
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/proj):
 *   q8p_layer_from_qshp   latq::deserialize  core/include/latq/pipeline.hpp:84
 *                         (core/src/pipeline.cpp:323-383) + device upload
 *   q8p_layer_create      latq::QuantizedLinear  pipeline.hpp:38-49 (fields
 *                         given directly instead of as a parsed artifact)
 *   q8p_forward           latq::infer  pipeline.hpp:73-74
 *                         (pipeline.cpp:151-197), batched, device buffers, fp32
 *   q8p_infer_host        latq::infer with host f64 vectors (the exact
 *                         reference calling convention; CLI `latq infer`,
 *                         tools/latq_cli.cpp:192-215, loops it per row)
 *   q8p_decode_stage      Codebook::decode / e8p_decode  core/include/latq/
 *                         codebook.hpp:31, e8p.hpp:35 over a whole stage
 *   q8p_k2_decode_stage   the same decode as the GEMV kernel performs it
 *                         (parity probe of the hot-path decoder)
 *   q8p_dequantize        latq::dequantize_layer  pipeline.hpp:68
 *                         (pipeline.cpp:142-149), dense W~ on the device
 *   q8p_rht               SideTransform::apply / apply_transpose
 *                         core/include/latq/transforms.hpp:30-33 (rht kind)
 *   q8p_plan_hadamard     latq::plan_hadamard  core/include/latq/hadamard.hpp:42
 *                         (registry extended with order 172)
 *   q8p_forward_sharded   (new) row-sharded forward with an NCCL all-gather
 *   q8p_forward_sharded_push  (new) the same with the all-gather fused into K3 pass 1
 * Error mapping: SizeError -> Q8P_ERR_SIZE, ValidationError ->
 * Q8P_ERR_VALIDATION, FormatError -> Q8P_ERR_FORMAT, BadMagicError ->
 * Q8P_ERR_BAD_MAGIC, UnsupportedVersionError -> Q8P_ERR_UNSUPPORTED_VERSION,
 * TruncatedArtifactError -> Q8P_ERR_TRUNCATED (core/include/latq/errors.hpp).
 */
#ifndef Q8P_H_
#define Q8P_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  Q8P_OK = 0,
  Q8P_ERR_SIZE = 1,                /* latq::SizeError (length mismatch, unplannable dim) */
  Q8P_ERR_VALIDATION = 2,          /* latq::ValidationError (unknown codebook id, bad args) */
  Q8P_ERR_FORMAT = 3,              /* latq::FormatError */
  Q8P_ERR_BAD_MAGIC = 4,           /* latq::BadMagicError */
  Q8P_ERR_UNSUPPORTED_VERSION = 5, /* latq::UnsupportedVersionError */
  Q8P_ERR_TRUNCATED = 6,           /* latq::TruncatedArtifactError */
  Q8P_ERR_UNSUPPORTED = 7,         /* valid artifact, not on this path (e.g. > 2 RVQ stages) */
  Q8P_ERR_CUDA = 8,                /* CUDA runtime failure / no sm_100 device */
  Q8P_ERR_NCCL = 9,
  Q8P_ERR_INTERNAL = 10
} q8p_status;

typedef enum {
  Q8P_CB_E8P_2BIT = 0, /* "e8p-2bit": 16-bit E8P codewords (core/src/e8p.cpp) */
  Q8P_CB_E8_1BIT = 1   /* "e8-1bit": 256-entry E8 ball table (core/src/codebook.cpp:188-243) */
} q8p_codebook;

typedef struct {
  q8p_codebook codebook;
  float scale;        /* StageInfo::scale, f32-frozen (pipeline.hpp:27-32) */
  const void* codes;  /* host, m * (n / 8) codewords, row-major [r * (n/8) + k] */
  int code_bytes;     /* bytes per codeword in `codes`: 2 (uint16) or 1 (uint8, e8-1bit only) */
} q8p_stage_desc;

typedef struct {
  uint32_t m, n;                 /* W is m x n; x has n entries, y has m */
  int transform;                 /* TransformKind: 0 = rht, 1 = rfft (transforms.hpp) */
  int num_stages;                /* 1 (2-bit) or 2 (3-/4-bit RVQ) */
  const q8p_stage_desc* stages;
  const uint8_t* signs_u;        /* rht: left_signs, ceil(m/8) bytes, LSB-first, bit set = -1 */
  const uint8_t* signs_v;        /* rht: right_signs, ceil(n/8) bytes */
  const float* phases_u;         /* rfft: left_phases, m/2 angles (PhaseVector, f32 as serialized) */
  const float* phases_v;         /* rfft: right_phases, n/2 angles */
} q8p_layer_desc;

typedef struct {
  uint32_t m, n;          /* full layer shape */
  uint32_t row_begin;     /* this handle's rows [row_begin, row_end) (sharded layers) */
  uint32_t row_end;
  int num_stages;
  int device;
  size_t device_bytes;    /* HBM held by the layer */
  size_t code_bytes;      /* algorithmic code bytes (m_local * n / 8 * sum code bytes) */
} q8p_layer_info;

typedef struct q8p_layer q8p_layer;

/* Library / device queries. */
const char* q8p_version(void);
const char* q8p_status_string(q8p_status s);
const char* q8p_last_error(void);
/* Number of this library's kernels launched since load (process-wide counter). */
uint64_t q8p_kernel_launches(void);

/* Hadamard planning (registry {1, 4, 12, 20, 28, 172}). */
q8p_status q8p_plan_hadamard(size_t n, size_t* p, size_t* q);

/* Layer lifetime.  create/from_qshp copy host buffers to `device` memory;
 * the caller keeps ownership of its buffers.  The layer is immutable after
 * creation and may be used concurrently from different streams provided
 * each call gets its own workspace. */
q8p_status q8p_layer_create(const q8p_layer_desc* desc, int device, q8p_layer** out);
q8p_status q8p_layer_from_qshp(const uint8_t* bytes, size_t len, int device, q8p_layer** out);
/* Multi-layer loading (a model's artifacts, latq::deserialize
 * pipeline.cpp:323-383 per artifact): every artifact is parsed and uploaded on its
 * own worker thread and private stream (at most 4 in flight), so one layer's
 * host-side deserialize overlaps another's H2D copies and device transcode.
 * out[i] = the layer of bytes[i]; on any failure no layer is kept and the first
 * error is returned. */
q8p_status q8p_layers_from_qshp(const uint8_t* const* bytes, const size_t* lens, int count, int device,
                                q8p_layer** out);
/* Row shard [row_begin, row_end) of a full artifact for row-sharded
 * tensor parallelism; S_U / S_V stay full. */
q8p_status q8p_layer_from_qshp_rows(const uint8_t* bytes, size_t len, uint32_t row_begin,
                                    uint32_t row_end, int device, q8p_layer** out);
void q8p_layer_destroy(q8p_layer* layer);
q8p_status q8p_layer_get_info(const q8p_layer* layer, q8p_layer_info* info);

/* Device workspace needed by q8p_forward for `batch` vectors (bytes). */
size_t q8p_workspace_bytes(const q8p_layer* layer, int batch);

/* y = W_tilde x for `batch` vectors: x device fp32 [batch][n], y device fp32
 * [batch][m] (m = full m).  Stream-ordered on `stream` (a cudaStream_t, or
 * NULL for the legacy default stream); never allocates. */
q8p_status q8p_forward(const q8p_layer* layer, const float* x, float* y, int batch,
                       void* workspace, size_t workspace_bytes, void* stream);

/* q8p_forward with instrumentation: when non-NULL, `gemv_start_event` /
 * `gemv_end_event` (cudaEvent_t) are recorded on `stream` immediately
 * before / after the decode-GEMV kernel (K2), so callers can time the
 * dominant kernel live, including under CUDA-graph capture. */
typedef struct {
  void* gemv_start_event;
  void* gemv_end_event;
} q8p_forward_opts;
q8p_status q8p_forward_ex(const q8p_layer* layer, const float* x, float* y, int batch,
                          void* workspace, size_t workspace_bytes, void* stream,
                          const q8p_forward_opts* opts);

/* Row-sharded forward: `layer` holds rows [row_begin, row_end) of the full
 * layer on this rank.  Each rank computes its z slice, the slices are
 * all-gathered over `nccl_comm` (an ncclComm_t), then every rank applies
 * the output transform to the full z.  Shards must be equal-sized and
 * ordered by rank. */
/* This handle's rows of the incoherent-domain product, z = W_hat (T_v x) for
 * rows [row_begin, row_end): z [batch][row_end - row_begin] fp32 (the slice
 * q8p_forward_sharded all-gathers; y = T_u^T z over the concatenated slices).
 * Stream-ordered, uses the same workspace as the forward. */
q8p_status q8p_forward_rows_z(const q8p_layer* layer, const float* x, float* z, int batch,
                              void* workspace, size_t workspace_bytes, void* stream);

q8p_status q8p_forward_sharded(const q8p_layer* layer, const float* x, float* y, int batch,
                               void* workspace, size_t workspace_bytes, void* nccl_comm,
                               void* stream);

/* Layer sets: `count` independent forwards y_i = W_i x_i in one call (one
 * decode step through a model's linear layers), stream-ordered, sharing one
 * workspace of q8p_forward_set_workspace_bytes(...) bytes (the largest layer's
 * q8p_workspace_bytes plus staging for the host variant).  No reference
 * counterpart: the reference loops `infer` per layer (latq_cli.cpp:211-212). */
size_t q8p_forward_set_workspace_bytes(const q8p_layer* const* layers, int count, int batch);
/* Device buffers: x[i] fp32 [batch][n_i], y[i] fp32 [batch][m_i]. */
q8p_status q8p_forward_set(const q8p_layer* const* layers, int count, const float* const* x,
                           float* const* y, int batch, void* workspace, size_t workspace_bytes,
                           void* stream);
/* Host buffers: x_host = the inputs concatenated [i][batch][n_i], y_host = the
 * outputs concatenated [i][batch][m_i].  Copies in, runs every layer, copies
 * out and synchronizes `stream`.  With pinned host buffers the whole step is
 * captured once per (layers, x_host, y_host, batch, workspace) into a CUDA
 * graph and replayed (one host launch per step). */
q8p_status q8p_forward_set_host(const q8p_layer* const* layers, int count, const float* x_host,
                                float* y_host, int batch, void* workspace, size_t workspace_bytes,
                                void* stream);
/* Flags for the _ex variants.  Q8P_SET_CONCURRENT: the layers are independent
 * (each reads only its own input, e.g. q/k/v or gate/up projections), so they
 * run on parallel streams with one workspace slice each (size it with
 * q8p_forward_set_workspace_bytes_ex): one layer's latency-bound transforms
 * overlap another's bandwidth-bound GEMV.  Results are bit-identical to the
 * sequential call. */
#define Q8P_SET_CONCURRENT 1u
size_t q8p_forward_set_workspace_bytes_ex(const q8p_layer* const* layers, int count, int batch,
                                          unsigned flags);
q8p_status q8p_forward_set_ex(const q8p_layer* const* layers, int count, const float* const* x,
                              float* const* y, int batch, void* workspace, size_t workspace_bytes,
                              void* stream, unsigned flags);
q8p_status q8p_forward_set_host_ex(const q8p_layer* const* layers, int count, const float* x_host,
                                   float* y_host, int batch, void* workspace, size_t workspace_bytes,
                                   void* stream, unsigned flags);

/* e8p_encode (core/src/e8p.cpp:114-156) on `device`, bit-identical to the
 * reference: v = device f64 [nblocks][8] -> words = device uint16 [nblocks],
 * the nearest E8P codeword of each 8-vector (ties to the smaller word).  The
 * inner search of the offline producer (RvqQuantizer::quantize, rvq.cpp). */
q8p_status q8p_e8p_encode(const double* v, uint16_t* words, size_t nblocks, int device, void* stream);
/* RvqQuantizer::quantize (rvq.cpp:59-79) for every 8-vector, bit-identical:
 * per stage scaled = residual / scale_s, code = the codebook's nearest word,
 * residual -= scale_s * decode(code).  v = device f64 [nblocks][8], codes =
 * device uint16 [num_stages][nblocks].  With the H = I nearest rounding
 * (ldlq.cpp:128-226, u = nullptr) this is the producer's whole code search. */
q8p_status q8p_rvq_quantize(const double* v, uint16_t* codes, size_t nblocks, int num_stages,
                            const q8p_codebook* codebooks, const double* scales, int device, void* stream);
/* SideTransform::apply (rht: x <- H (S o x), transforms.cpp:28-36) on every
 * column of a row-major rows x cols device f64 matrix, in place, bit-identical
 * to the reference's transform_cols (transforms.cpp:66-79); signs: device,
 * ceil(rows/8) bytes; scratch: rows * cols doubles.  With a transpose it is
 * transform_rows; the producer's incoherence step W~ = T_u W T_v^T. */
q8p_status q8p_rht_cols_f64(double* w, double* scratch, size_t rows, size_t cols, const uint8_t* signs,
                            int device, void* stream);

/* latq::infer drop-in: host f64 x [batch][n] -> host f64 y [batch][m].
 * Synchronous; stages through an internal pinned buffer and workspace. */
q8p_status q8p_infer_host(q8p_layer* layer, const double* x, double* y, int batch);

/* Unscaled incoherent-domain decode of one stage into device fp32
 * w_hat[m_local][n] (decoded values are exact quarter-integers). */
q8p_status q8p_decode_stage(const q8p_layer* layer, int stage, float* w_hat, void* stream);

/* latq::dequantize_layer (core/src/pipeline.cpp:142-149) on the device, rht layers:
 * w_tilde[m][n] (f64, device) = T_u^T W_hat T_v with W_hat = sum_s scale_s *
 * decode_s accumulated in f64 in stage order (decode_incoherent, :112-138) and
 * the transforms applied column-wise then row-wise with the reference's
 * butterfly / base-sum order (transform_cols / transform_rows, transforms.cpp:
 * 66-94): bit-identical to the reference.  scratch: m * n doubles (device).
 * Full (unsharded) layers only; rfft layers -> Q8P_ERR_UNSUPPORTED. */
q8p_status q8p_dequantize(const q8p_layer* layer, double* w_tilde, double* scratch, void* stream);

/* Parity probe of the GEMV's own decoder (e8p_decode, core/src/e8p.cpp:81-100;
 * TableCodebook::decode, codebook.cpp:65-72): runs the tensor-core K2's operand
 * decode over the layer's transcoded slabs and writes the int8 A bytes it feeds
 * the tensor cores, a_bytes[m_local][n] (E8P: sigma_c * doubled_c; e8-1bit: the
 * doubled table row), and for E8P stages the shift bits shift_bits[m_local][n/8],
 * so that the decoded value is (2 a + 2 b - 1) / 4 (E8P) or a / 2 (e8-1bit).
 * Device pointers; stream-ordered. */
q8p_status q8p_k2_decode_stage(const q8p_layer* layer, int stage, int8_t* a_bytes, uint8_t* shift_bits,
                               void* stream);

/* Benchmark support (the reference's bm_infer, bench/bench.cpp:103-120):
 *  q8p_bench_gemv    `reps` back-to-back launches of the layer's decode-GEMV (K2)
 *                    on the B images already in `ws` (run a forward with the same
 *                    workspace and batch first); stream-ordered, chained with
 *                    programmatic dependent launch as inside a forward.
 *  q8p_bench_stream  `reps` launches of a plain HBM read of [src, src + bytes)
 *                    in K2's access pattern (bulk copies into shared memory): the
 *                    stream ceiling of the same bytes.
 *  q8p_layer_code_region  device address / size of a stage's code slabs. */
q8p_status q8p_bench_gemv(const q8p_layer* layer, int batch, void* workspace, size_t workspace_bytes, int reps,
                          void* stream);
q8p_status q8p_bench_stream(const void* src, size_t bytes, int reps, void* stream);
q8p_status q8p_layer_code_region(const q8p_layer* layer, int stage, const void** codes, size_t* bytes);

/* Randomized Hadamard transform on device fp32 vectors:
 *   transpose == 0:  y = H (S o x)          (SideTransform::apply)
 *   transpose != 0:  y = S o (H^T x)        (SideTransform::apply_transpose)
 * signs: device pointer to ceil(n/8) sign bytes. x and y may alias. */
q8p_status q8p_rht(size_t n, const uint8_t* signs, const float* x, float* y, int batch,
                   int transpose, void* stream);

/* Host-side helpers (no GPU needed): artifact inspection and round trip
 * (latq::deserialize / serialize, pipeline.cpp:269-383), codebook tables
 * (e8p.hpp:22-35, codebook.cpp:188-243) and Hadamard bases (hadamard.hpp:35). */
typedef struct {
  uint32_t m, n;
  int transform;          /* 0 = rht, 1 = rfft */
  int num_stages;
  q8p_codebook codebook[8];
  float scale[8];
  size_t serialized_size; /* == len for a valid artifact */
} q8p_artifact_info;
q8p_status q8p_qshp_inspect(const uint8_t* bytes, size_t len, q8p_artifact_info* info);
/* deserialize(bytes) then serialize into out[cap]; *out_len = bytes written. */
q8p_status q8p_qshp_reserialize(const uint8_t* bytes, size_t len, uint8_t* out, size_t cap,
                                size_t* out_len);
q8p_status q8p_e8p_decode_host(uint16_t word, float out[8]);
/* doubled coordinates [256][8] of a codebook table (E8P: magnitudes 1/3/5
 * with odd_parity[256] in parity_out; e8-1bit: signed, parity_out unused). */
q8p_status q8p_codebook_table(q8p_codebook cb, int8_t* doubled, uint8_t* parity_out);
q8p_status q8p_hadamard_base(size_t q, int8_t* out);

/* Test support for the row-sharded path on one GPU: runs every rank's part of
 * q8p_forward_sharded in turn (K1, K2 on the shard's rows, K3 pass 1 into the
 * send buffer) with the all-gather replaced by device copies into the gathered
 * buffer, then K3 pass 2 -> y [batch][m].  shards[r] = rows shard_rows(m, world, r)
 * of one layer, all on one device; batch <= 32; ws sized for shards[0]. */
q8p_status q8p_forward_sharded_sim(const q8p_layer* const* shards, int world, const float* x, float* y, int batch,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* Push all-gather (replaces the all-gather between
 * q8p_forward_sharded's K3 passes).  The reference's rows are independent
 * (core/src/pipeline.cpp:176-191), so each rank computes its rows' K3 pass 1
 * and stores them straight into every rank's window over NVLink (CUDA IPC
 * mappings) as 8-byte {value, call tag} words; K3 pass 2 reads its own window
 * as the tagged words arrive -- no collective launch, no fences, the transfer
 * overlaps pass 1 tile by tile.  Setup: every rank calls q8p_peers_create (one
 * device allocation of 256 B + 16 * world * slice_floats bytes; `handle`
 * receives its Q8P_PEER_HANDLE_BYTES IPC handle), the handles are exchanged out
 * of band (e.g. torch.distributed all_gather_object) and concatenated in rank
 * order, then every rank calls q8p_peers_connect.  world <= 16;
 * slice_floats >= min(batch, 32) * m_local for every layer / batch used
 * (batch * m_local for prefill batches, >= 64, which run K4 + one push).
 * Requirements as q8p_forward_sharded's fast path: equal rank-ordered row
 * shards that are whole K3 pass-1 chunks (rht layers), batches on the
 * tensor-core path; else Q8P_ERR_UNSUPPORTED.  All ranks must issue the same
 * sequence of push forwards (a rank whose peer never writes traps after ~20 s). */
#define Q8P_PEER_HANDLE_BYTES 64
typedef struct q8p_peers q8p_peers;
q8p_status q8p_peers_create(int device, int world, int rank, size_t slice_floats, q8p_peers** out,
                            uint8_t handle[Q8P_PEER_HANDLE_BYTES]);
q8p_status q8p_peers_connect(q8p_peers* peers, const uint8_t* handles /* world * Q8P_PEER_HANDLE_BYTES */);
q8p_status q8p_peers_destroy(q8p_peers* peers);
/* Diagnostics (synchronous): the number of push calls (K3 chunks) completed on this rank. */
q8p_status q8p_peers_state(const q8p_peers* peers, uint64_t* epoch);
q8p_status q8p_forward_sharded_push(const q8p_layer* layer, q8p_peers* peers, const float* x, float* y, int batch,
                                    void* workspace, size_t workspace_bytes, void* stream);
/* Test support: the `world` members of one group created in ONE process on one
 * device, wired to each other directly (no IPC); q8p_forward_sharded_push_sim
 * runs every rank's K1, K2 and pushing pass 1, then every rank's pass 2, in
 * stream order; y = [world][batch][m] (each rank's full output). */
q8p_status q8p_peers_connect_local(q8p_peers* const* group, int world);
q8p_status q8p_forward_sharded_push_sim(const q8p_layer* const* shards, q8p_peers* const* peers, int world,
                                        const float* x, float* y, int batch, void* workspace,
                                        size_t workspace_bytes, void* stream);

/* NCCL plumbing for q8p_forward_sharded (wraps ncclGetUniqueId /
 * ncclCommInitRank so callers need no NCCL headers). */
q8p_status q8p_nccl_unique_id(uint8_t out[128]);
q8p_status q8p_nccl_comm_init(const uint8_t id[128], int world, int rank, int device, void** comm);
q8p_status q8p_nccl_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif

#endif /* Q8P_H_ */
