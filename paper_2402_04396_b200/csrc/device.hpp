// Device-side layer representation and kernel launchers (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <utility>
#include <vector>

#include "internal.hpp"

namespace q8p::detail {

extern std::atomic<std::uint64_t> g_launches;  // kernels launched by this library

[[noreturn]] void throw_cuda(cudaError_t e, const char* what);
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw_cuda(e, what);
}

// Programmatic dependent launch (PDL): every q8p kernel is launched with
// programmatic stream serialization, waits (griddepcontrol.wait) before it
// touches its predecessor's output and then lets its own dependents start
// (griddepcontrol.launch_dependents), so launch latency and prologues (LUT
// build, weight prefetch) overlap the previous kernel's tail -- also inside
// CUDA graphs.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
#ifdef Q8P_EXP_NO_PDL
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "kernel launch");
}

// One-time (per device) kernel attributes: dynamic shared-memory limit, the
// maximum shared-memory carveout for every q8p kernel (so consecutive kernels of
// a forward never force an L1 / shared-memory reconfiguration of the SMs), and
// optionally non-portable cluster sizes.  Thread-safe; keyed by (kernel, device).
void kernel_attrs(const void* fn, int max_dyn_smem, bool cluster = false);
// Device of the calling thread (cudaGetDevice), for per-device one-time state.
int current_device();

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" :::); }
#endif

// One side transform on device: randomized Hadamard (kind 0) or rfft (kind 1).
struct DevSide {
  int kind = 0;                         // TransformKind: 0 = rht, 1 = rfft
  std::uint32_t n = 0, p = 1, q = 1;
  const std::uint8_t* signs = nullptr;  // ceil(n/8) bytes
  const std::int8_t* base = nullptr;    // q x q (+-1), nullptr when q == 1
  const float* colsum = nullptr;        // q column sums of the base (sum_i t_i in closed form)
  // rfft (kernels_rfft.cu): DFT length M = n / 2 = M1 * M2
  std::uint32_t M1 = 1, M2 = 1;
  const float2* rot = nullptr;          // [M] e^{i theta_k}
  const float2* tw = nullptr;           // [M] e^{-2 pi i e / M}
};

// Tensor-core GEMV slab records (gemv_tc.cu): [row block][k slab][slab bytes].
struct SlabCodes {
  void* codes = nullptr;
};

}  // namespace q8p::detail

struct q8p_layer {
  int device = 0;
  std::uint32_t m = 0, n = 0, row_begin = 0, row_end = 0;
  int num_stages = 0;
  int cb[2] = {0, 0};
  float scale[2] = {1.f, 1.f};
  q8p::detail::DevSide side_u, side_v;  // left (m) / right (n)
  // plain [m_local][n/8] codes, u16 (E8P) / u8 (e8-1bit): kept on the device only for
  // layers the tensor-core path cannot run (first stage not E8P; portable GEMV)
  void* codes[2] = {nullptr, nullptr};
  q8p::detail::SlabCodes tc[2];
  const std::uint8_t* lut_img = nullptr;   // device 64 KiB lane-replicated decode LUT (gemv_tc.cu)
  const std::uint32_t* dec_tables = nullptr;  // device [256] E8P nibble words + [256][2] e8-1bit rows (K4)
  std::size_t device_bytes = 0;
  std::size_t code_bytes = 0;
  std::vector<void*> allocations;
  // q8p_infer_host staging: a pool of per-call contexts (stream, pinned host and
  // device buffers); concurrent callers each take one, so infer is re-entrant as
  // the reference's and calls on one layer run in parallel.
  struct Stage {
    cudaStream_t stream = nullptr;
    void* host = nullptr;
    std::size_t host_bytes = 0;
    void* dev = nullptr;
    std::size_t dev_bytes = 0;
  };
  std::mutex stage_mu;
  std::vector<Stage*> stage_free;  // idle contexts
  std::vector<Stage*> stage_all;   // every context (freed by q8p_layer_destroy)
  // q8p_forward graph cache (capi.cpp): the forward's kernel chain captured once per
  // (x, y, batch, workspace) and replayed with one cudaGraphLaunch.
  struct GraphEntry {
    const float* x;
    float* y;
    int batch;
    void* ws;
    std::size_t ws_bytes;
    cudaGraphExec_t exec;
    std::uint32_t kernels;  // q8p kernels per replay (kernel_launches accounting)
  };
  std::mutex graph_mu;
  std::vector<GraphEntry> graphs;  // small, most recent last
  cudaStream_t capture_stream = nullptr;

  std::uint32_t m_local() const { return row_end - row_begin; }
};

namespace q8p::detail {

// Kernel launchers (kernels_*.cu).  All stream-ordered, no allocation.
void launch_rht(const DevSide& side, const float* x, float* y, int batch, bool transpose,
                cudaStream_t s);
void launch_gemv_simple(const q8p_layer& L, const float* t, float* z, int batch, int z_stride,
                        cudaStream_t s);
// e8p_encode (core/src/e8p.cpp:114-156) on device, bit-identical: v [nblocks][8] f64 -> words.
void launch_e8p_encode(const double* v, std::uint16_t* words, std::size_t nblocks, cudaStream_t s);
// RvqQuantizer::quantize (rvq.cpp:59-79) per 8-vector, bit-identical: codes [stage][nblocks].
void launch_rvq_quantize(const double* v, std::uint16_t* codes, std::size_t nblocks, int stages, const int* kinds,
                         const double* scales, cudaStream_t s);
// SideTransform::apply (rht) on every column of a row-major L x ncols f64 matrix, in place
// (scratch: L * ncols doubles), bit-identical to transform_cols (transforms.cpp:66-79).
// (transpose: SideTransform::apply_transpose per column, as transform_cols(..., true)).
void launch_rht_cols_f64(double* w, double* scratch, std::uint32_t L, std::uint32_t ncols, const std::uint8_t* signs,
                         cudaStream_t s, bool transpose = false);
// dequantize_layer pieces (kernels_encode.cu): stage points from K2's decoder output
// combined in f64 as decode_incoherent does, and an f64 transpose.
void launch_dequant_combine(const std::int8_t* a0, const std::uint8_t* b0, const std::int8_t* a1,
                            const std::uint8_t* b1, int nst, int kind0, int kind1, double s0, double s1,
                            std::size_t total, double* w, cudaStream_t s);
void launch_transpose_f64(const double* in, double* out, std::uint32_t rows, std::uint32_t cols, cudaStream_t s);
void launch_points_f32(const std::int8_t* a, const std::uint8_t* b, int kind, std::size_t total, float* w,
                       cudaStream_t s);

// Tensor-core path (gemv_tc.cu, kernels_rht.cu).
std::vector<std::uint8_t> tc_lut_image();  // the 64 KiB smem LUT window, bulk-copied per CTA
std::uint32_t tc_slab_bytes(int kind);
std::uint32_t tc_row_blocks(std::uint32_t m_local);
std::uint32_t tc_k_slabs(std::uint32_t n);
std::size_t tc_code_bytes(std::uint32_t m_local, std::uint32_t n, int kind);
// tc_transcode on the device from the uploaded plain codes (u16 E8P / u8 e8-1bit).
void tc_transcode_device(const void* codes, std::uint32_t m_local, std::uint32_t n, int kind, std::uint8_t* out,
                         const std::uint8_t* odd_parity_dev, cudaStream_t s);
constexpr int kTcMaxBatch = 32;  // tensor-core path: batch <= 32 per launch (MMA N <= 128)
bool tc_supported(const q8p_layer& L, int batch);
int tc_ncols_pad(int ncols);                              // MMA N for `ncols` B rows
std::uint32_t tc_bimg_bytes(std::uint32_t n, int batch);  // B images for all k slabs
// K4 prefill decode-GEMM (gemm_prefill.cu): batches >= kPrefillMinBatch.
constexpr int kPrefillMinBatch = 64;
bool prefill_supported(const q8p_layer& L, int batch);
std::size_t prefill_btile_bytes(const q8p_layer& L, int batch);
// Per-vector max |t| slot in the B-tile region: K1 (prefill) writes it, pack_b turns it into alpha.
float* prefill_amax(const q8p_layer& L, int batch, std::uint8_t* btiles);
// K4's stream-K schedule.  Tiles (N tile of `nt` vectors x M pair of `mrows` rows,
// tile = nt_index * MP + mp) each have KS8 k-slab steps; the `grid` CTAs own equal
// contiguous ranges of the tiles x KS8 steps in that order, so a tile is split
// into pieces at CTA boundaries.  Piece k of a tile writes z slice k; K3 sums a
// tile's pieces in piece order (k4_pieces, rht_device.cuh).  `slices` = the most
// pieces any tile has (the z allocation).
struct K4Sched {
  std::uint32_t KS8 = 0, MP = 0, NTL = 0, grid = 0, slices = 1;
  std::uint32_t nt = 256, mrows = 256;
};
#ifdef __CUDACC__
#define Q8P_HD __host__ __device__
#else
#define Q8P_HD
#endif
// (32-bit arithmetic: prefill_sched guarantees total * grid < 2^32.)
Q8P_HD inline std::uint32_t k4_total(const K4Sched& s) { return s.MP * s.NTL * s.KS8; }
Q8P_HD inline std::uint32_t k4_bound(const K4Sched& s, std::uint32_t c) {  // first step of CTA c
  return c * k4_total(s) / s.grid;
}
Q8P_HD inline std::uint32_t k4_cta_of(const K4Sched& s, std::uint32_t step) {  // the CTA owning `step`
  std::uint32_t c = step * s.grid / k4_total(s);
  while (c + 1 < s.grid && k4_bound(s, c + 1) <= step) ++c;
  while (c > 0 && k4_bound(s, c) > step) --c;
  return c;
}
Q8P_HD inline std::uint32_t k4_pieces(const K4Sched& s, std::uint32_t tile) {  // pieces of a tile
  const std::uint32_t t0 = tile * s.KS8;
  return k4_cta_of(s, t0 + s.KS8 - 1) - k4_cta_of(s, t0) + 1;
}
K4Sched prefill_sched(const q8p_layer& L, int batch);
std::uint32_t prefill_parts(const q8p_layer& L, int batch);  // = prefill_sched().slices: z is [P][batch][m_local]
void launch_prefill(const q8p_layer& L, const float* t, std::uint8_t* btiles, float* z, int batch, cudaStream_t s);
// Benchmark support (bench_kernels.cu): bulk-copy stream of `bytes` at src (the
// HBM read ceiling in K2's access pattern).
void launch_stream(const void* src, std::size_t bytes, unsigned* sink, cudaStream_t s);
// Parity probe: K2's own operand decode over the slabs of `stage` -> a[m_local][n] (s8,
// sigma*d for E8P, doubled row for e8-1bit) and side[m_local][n/8] (E8P shift bits).
void launch_k2_decode(const q8p_layer& L, int stage, std::int8_t* a_out, std::uint8_t* side, cudaStream_t s);
void launch_gemv_tc(const q8p_layer& L, const std::uint8_t* bimg, std::int32_t* zacc, std::uint32_t rows_pad,
                    int batch, cudaStream_t s);
std::vector<std::uint32_t> decode_table_words();  // host image of q8p_layer::dec_tables
// K1 (fp32 flavour, q8p_rht): t = T_v x (+ amax, tsum when non-null).
void launch_rht_in(const DevSide& side, const float* x, float* t, float* u_scratch, float* amax, float* tsum,
                   std::int32_t* zero_ptr, std::size_t zero_words, int batch, cudaStream_t s);
// K1 (limb flavour): x -> B images of the integer activations (gemv_tc.cu), alpha, TL;
// zeroes the GEMV accumulators and the B-image tail.
void launch_rht_in_limbs(const DevSide& side, const float* x, float* u_scratch, float* ssq, float* alpha,
                         long long* tl, std::uint8_t* bimg, std::uint32_t b_bytes, std::uint32_t bcols,
                         std::uint8_t* bimg_tail, std::size_t tail_bytes, std::int32_t* zero_ptr,
                         std::size_t zero_words, int batch, cudaStream_t s, std::uint32_t chunk_vec = 0,
                         std::size_t chunk_bytes = 0);
// Row-sharded K3 (q8p_forward_sharded): pass 1 on this rank's rows straight from
// its accumulators into the all-gather send buffer [batch][m_local] (when the rank's
// rows are whole pass-1 chunks: rht_sharded_k3_ok), pass 2 over the gathered
// rank-major [world][batch][m_local] buffer; launch_rht_out_gathered = both passes
// from gathered fp32 z (the fallback after combine).
bool rht_sharded_k3_ok(const DevSide& side, std::uint32_t row0, std::uint32_t m_local);
void launch_rht_out_acc_local(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                              std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                              const long long* tl, std::uint32_t row0, std::uint32_t m_local, float* z_send, int batch,
                              cudaStream_t s);
void launch_rht_out_pass2_gathered(const DevSide& side, const float* mid_gathered, std::uint32_t m_local, float* y,
                                   int batch, cudaStream_t s);
void launch_rht_out_gathered(const DevSide& side, const float* z_gathered, std::uint32_t m_local, float* u_scratch,
                             float* y, int batch, cudaStream_t s);
// Push all-gather (q8p_forward_sharded_push).  Each rank owns
// one device allocation [PeerCtl][2 parities][world][slice] of 8-byte words
// {float bits, call tag} whose base the other ranks map (CUDA IPC over NVLink /
// NVSwitch).  K3 pass 1 stores every value of its rows, tagged with the call
// number, straight into every rank's window of the call's parity; an aligned
// 8-byte store is single-copy atomic, so a reader that sees the tag sees the value
// (the LL protocol: no fences, no counters).  K3 pass 2 polls its own window until
// every word it needs carries this call's tag; its last CTA advances the rank's
// call counter (epoch).  Two parities: a rank runs at most one call ahead of a
// peer (its pass 2 needs the peer's pass 1 of the same call), so a parity is never
// overwritten while it is read.
constexpr int kMaxPeers = 16;
struct PeerCtl {
  unsigned long long epoch;  // calls completed on this rank (parity = epoch & 1, tag = epoch + 1)
  unsigned long long done;   // pass-2 CTAs finished in the current call
};
constexpr std::size_t kPeerCtlBytes = 256;
static_assert(sizeof(PeerCtl) <= kPeerCtlBytes, "peer control block");
struct PushArgs {
  unsigned long long* const* wins;     // device table [world]: every rank's window (parity 0) as mapped here
  unsigned long long* self_win;        // this rank's window (parity 0)
  PeerCtl* ctl;                        // this rank's control block
  int rank, world;
  std::size_t win_words;               // words per parity (world * slice)
};
void launch_rht_out_acc_push(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                             std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                             const long long* tl, std::uint32_t row0, std::uint32_t m_local, const PushArgs& push,
                             int batch, cudaStream_t s);
// Row-sharded prefill K3 pass 1: this rank's rows from K4's K-split partials
// [parts][batch][m_local] (summed in split order) into the send buffer
// [batch][m_local], or pushed into every rank's window when `push` is set.
void launch_rht_out_local_f32(const DevSide& side, const float* zparts, int parts, std::uint32_t row0,
                              std::uint32_t m_local, float* z_send, const PushArgs* push, int batch,
                              cudaStream_t s, const K4Sched* sched = nullptr);
void launch_rht_out_pass2_push(const DevSide& side, std::uint32_t m_local, const PushArgs& push, float* y, int batch,
                               cudaStream_t s);
// Row-sharded forward: this rank's fp32 z rows [batch][m_local] from the limb accumulators.
void launch_combine_acc(const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows, std::uint32_t zacc_cols,
                        const float zscale[2], const int ze8p[2], const float* alpha, const long long* tl, float* z,
                        std::uint32_t m_local, int batch, cudaStream_t s);
// rfft side transform (kernels_rfft.cu): factorization M = n / 2 = M1 * M2
// (`codewords`: M2 % 4 == 0 so K1 can emit whole codewords; false if no
// factorization fits the kernels), host tables (rot = e^{i theta}, tw =
// e^{-2 pi i e / M}, interleaved float pairs), fp32 apply / apply_transpose
// through `u_scratch` ([batch][n] floats), and K1's limb flavour.
bool rfft_factor(std::uint32_t n, bool codewords, std::uint32_t& M1, std::uint32_t& M2);
void rfft_tables(std::uint32_t n, const float* phases, std::vector<float>& rot, std::vector<float>& tw);
void launch_rfft_f32(const DevSide& side, const float* x, float* u_scratch, float* y, int batch, bool transpose,
                     cudaStream_t s);
void launch_rfft_out_acc(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                         std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                         const long long* tl, float* u_scratch, float* y, int batch, cudaStream_t s);
void launch_rfft_in_limbs(const DevSide& side, const float* x, float* u_scratch, float* ssq, float* alpha,
                          long long* tl, std::uint8_t* bimg, std::uint32_t b_bytes, std::uint32_t bcols,
                          std::uint8_t* bimg_tail, std::size_t tail_bytes, std::int32_t* zero_ptr,
                          std::size_t zero_words, int batch, cudaStream_t s);
// K3 (fp32 input): y = T_u^T z.
void launch_rht_out(const DevSide& side, const float* zin, float* u_scratch, float* y, int batch, cudaStream_t s,
                    int in_parts = 1, const K4Sched* sched = nullptr);
// K3 (accumulator input): z = sum_s zscale_s alpha (2 Z_s - [E8P] TL) / 4 from the int32
// limb accumulators [stage][zacc_cols][zacc_rows], then y = T_u^T z.
void launch_rht_out_acc(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                        std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                        const long long* tl, float* u_scratch, float* y, int batch, cudaStream_t s,
                        bool zero_after = false);

}  // namespace q8p::detail
