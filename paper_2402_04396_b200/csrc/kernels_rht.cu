// K1 / K3: randomized Hadamard transforms around the tensor-core GEMV.
//
// SideTransform (core/src/transforms.cpp:28-47) with had_apply
// (core/src/hadamard.cpp:170-210):  H = (H_p (x) B_q) / sqrt(n), flat index
// i = a * q + b.  The two Kronecker factors act on different index digits
// and commute, so each side is split into two embarrassingly parallel
// passes over HBM/L2-resident fp32 vectors:
//   base pass  (I (x) B_q):   rows a split across CTAs, q x q +-1 products
//   fwht pass  (H_p (x) I):   columns b split across CTAs, in-smem FWHT
// K1 (input side):   x --signs--> [base] --> fwht --> t, amax(|t|) per vector
// K3 (output side):  z_acc(int32 limbs) --> fwht --> [base^T] --signs--> y
// For q == 1 there is no base pass.  K1 also zeroes the GEMV's int32
// accumulators (extra CTAs), K3 consumes them.
#include <cuda_runtime.h>

#include "device.hpp"

namespace q8p::detail {
namespace {

constexpr int kThreads = 1024;

__device__ __forceinline__ bool sign_bit(const std::uint8_t* s, std::uint32_t i) {
  return (s[i >> 3] >> (i & 7)) & 1;
}

__device__ __forceinline__ void atomic_max_pos(float* addr, float v) {
  // |t| >= 0: IEEE ordering of non-negative floats equals their int ordering.
  atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
}

__device__ __forceinline__ float block_reduce_max(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < int(blockDim.x >> 5) ? red[l] : 0.f;
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;  // valid in thread 0
}

// In-smem unnormalized FWHT over `p` rows of `cw` contiguous floats each
// (row stride cw): butterflies between rows k and k + len.
__device__ void smem_fwht(float* s, std::uint32_t p, std::uint32_t cw) {
  const std::uint32_t half = (p >> 1) * cw;
  for (std::uint32_t len = 1; len < p; len <<= 1) {
    for (std::uint32_t t = threadIdx.x; t < half; t += blockDim.x) {
      const std::uint32_t pair = t / cw, j = t - pair * cw;
      const std::uint32_t blk = pair / len, off = pair - blk * len;
      const std::uint32_t k = blk * 2 * len + off;
      const float u = s[k * cw + j], v = s[(k + len) * cw + j];
      s[k * cw + j] = u + v;
      s[(k + len) * cw + j] = u - v;
    }
    __syncthreads();
  }
}

struct FwhtArgs {
  std::uint32_t n, p, q;
  std::uint32_t cols_per_cta;        // columns b handled by one CTA
  const std::uint8_t* signs;         // applied on input (fwd, q == 1) or output (trans, q == 1)
  const float* in;                   // fp32 input [batch][n] (fwd) / u (trans, q > 1 second pass input unused)
  const std::int32_t* zacc;          // trans: int32 limb accumulators [stages][batch*2][rows_pad]
  int zacc_stages;
  std::uint32_t zacc_rows;           // rows_pad
  const float* amax;                 // trans: per-vector amax of t (limb scale source)
  float zscale[2];                   // trans: per-stage 0.5 * stage_scale / 16256
  float* out;                        // [batch][n]
  float* amax_out;                   // fwd: per-vector amax (atomicMax; zeroed by caller pass)
  std::int32_t* zero_ptr;            // fwd: buffer to zero with spare CTAs
  std::size_t zero_words;
  float out_scale;                   // 1/sqrt(n) applied on output
  int fwd;                           // 1 = K1 (input side), 0 = K3
};

// FWHT pass.  grid = (ceil(q / cols_per_cta) [+ zero CTAs], batch).
__global__ void __launch_bounds__(kThreads) fwht_kernel(FwhtArgs a) {
  extern __shared__ float s[];
  __shared__ float red[32];
  const std::uint32_t ncta_cols = (a.q + a.cols_per_cta - 1) / a.cols_per_cta;
  const int b = blockIdx.y;
  if (blockIdx.x >= ncta_cols) {
    // Spare CTAs: zero the GEMV accumulators (only with the first vector's grid row).
    if (b == 0 && a.zero_ptr) {
      const std::size_t nz = gridDim.x - ncta_cols;
      for (std::size_t i = (blockIdx.x - ncta_cols) * std::size_t(blockDim.x) + threadIdx.x; i < a.zero_words;
           i += nz * blockDim.x)
        a.zero_ptr[i] = 0;
    }
    return;
  }
  const std::uint32_t c0 = blockIdx.x * a.cols_per_cta;
  const std::uint32_t cw = min(a.cols_per_cta, a.q - c0);
  const std::uint32_t n = a.n, q = a.q;
  // Load [p][cw] sub-block.
  for (std::uint32_t e = threadIdx.x; e < a.p * cw; e += blockDim.x) {
    const std::uint32_t r = e / cw, j = e - r * cw;
    const std::uint32_t i = r * q + c0 + j;
    float v;
    if (a.fwd) {
      v = a.in[std::size_t(b) * n + i];
      if (q == 1 && sign_bit(a.signs, i)) v = -v;
    } else if (a.zacc) {
      // z = sum_s zscale_s * amax * (128 * hi + lo)   (limb recombination)
      const float am = a.amax[b];
      double acc = 0.0;
      for (int st = 0; st < a.zacc_stages; ++st) {
        const std::int32_t* z = a.zacc + (std::size_t(st) * 8 + 2 * b) * a.zacc_rows;
        acc += double(a.zscale[st]) * (128.0 * double(z[i]) + double(z[a.zacc_rows + i]));
      }
      v = float(acc * double(am));
    } else {
      v = a.in[std::size_t(b) * n + i];
    }
    s[r * cw + j] = v;
  }
  __syncthreads();
  smem_fwht(s, a.p, cw);
  float mx = 0.f;
  for (std::uint32_t e = threadIdx.x; e < a.p * cw; e += blockDim.x) {
    const std::uint32_t r = e / cw, j = e - r * cw;
    const std::uint32_t i = r * q + c0 + j;
    float v = s[r * cw + j] * a.out_scale;
    if (!a.fwd && q == 1 && sign_bit(a.signs, i)) v = -v;
    a.out[std::size_t(b) * n + i] = v;
    mx = fmaxf(mx, fabsf(v));
  }
  if (a.fwd && a.amax_out) {
    mx = block_reduce_max(mx, red);
    if (threadIdx.x == 0) atomic_max_pos(a.amax_out + b, mx);
  }
}

struct BaseArgs {
  std::uint32_t n, p, q;
  std::uint32_t rows_per_cta;
  const std::int8_t* base;   // q x q
  const std::uint8_t* signs;
  const float* in;
  float* out;
  float out_scale;           // 1/sqrt(n) (trans) or 1 (fwd)
  float* amax_zero;          // fwd: zero the per-vector amax (CTA 0)
  int batch;
  int fwd;                   // 1: y = B (S o x) per row ; 0: y = S o (B^T x) * scale
};

// Base pass: rows a in [a0, a0 + rows_per_cta) of one vector per grid row.
// The +-1 base is staged in smem as float (q <= 28) or int8 (q = 172).
template <typename BT>
__global__ void __launch_bounds__(256) base_kernel(BaseArgs a) {
  extern __shared__ float sm[];
  const std::uint32_t q = a.q, n = a.n;
  BT* B = reinterpret_cast<BT*>(sm);
  float* seg = sm + (q * q * sizeof(BT) + 15) / 16 * 4;
  const int b = blockIdx.y;
  if (a.fwd && a.amax_zero && blockIdx.x == 0 && threadIdx.x < a.batch && b == 0) a.amax_zero[threadIdx.x] = 0.f;
  for (std::uint32_t i = threadIdx.x; i < q * q; i += blockDim.x) B[i] = BT(a.base[i]);
  const std::uint32_t r0 = blockIdx.x * a.rows_per_cta;
  const std::uint32_t nr = min(a.rows_per_cta, a.p - r0);
  for (std::uint32_t e = threadIdx.x; e < nr * q; e += blockDim.x) {
    const std::uint32_t i = r0 * q + e;
    float v = a.in[std::size_t(b) * n + i];
    if (a.fwd && sign_bit(a.signs, i)) v = -v;
    seg[e] = v;
  }
  __syncthreads();
  for (std::uint32_t e = threadIdx.x; e < nr * q; e += blockDim.x) {
    const std::uint32_t r = e / q, c = e - r * q;
    const float* x = seg + r * q;
    float acc = 0.f;
    if (a.fwd)
      for (std::uint32_t k = 0; k < q; ++k) acc += float(B[c * q + k]) * x[k];
    else
      for (std::uint32_t k = 0; k < q; ++k) acc += float(B[k * q + c]) * x[k];
    acc *= a.out_scale;
    const std::uint32_t i = (r0 + r) * q + c;
    if (!a.fwd && sign_bit(a.signs, i)) acc = -acc;
    a.out[std::size_t(b) * n + i] = acc;
  }
}

void set_smem(const void* fn, std::size_t bytes) {
  cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)), "smem attr");
}

std::uint32_t fwht_cols_per_cta(const DevSide& side) {
  if (side.q == 1) {
    if (side.p * 4 > 200 * 1024) throw SizeError("rht: power-of-two factor too large for one CTA");
    return 1;
  }
  return side.q % 4 == 0 ? 4 : 1;  // 16-byte row segments per CTA
}

void launch_base(const DevSide& side, BaseArgs a, int batch, cudaStream_t s) {
  a.rows_per_cta = std::max<std::uint32_t>(1, 256 / side.q);
  const bool fl = side.q <= 28;
  const std::size_t bsz = fl ? side.q * side.q * 4 : side.q * side.q;
  const std::size_t smem = (bsz + 15) / 16 * 16 + std::size_t(a.rows_per_cta) * side.q * 4;
  static std::once_flag once;
  std::call_once(once, [] {
    set_smem(reinterpret_cast<const void*>(base_kernel<float>), 200 * 1024);
    set_smem(reinterpret_cast<const void*>(base_kernel<std::int8_t>), 200 * 1024);
  });
  dim3 grid((side.p + a.rows_per_cta - 1) / a.rows_per_cta, batch);
  if (fl)
    base_kernel<float><<<grid, 256, smem, s>>>(a);
  else
    base_kernel<std::int8_t><<<grid, 256, smem, s>>>(a);
  cuda_check(cudaGetLastError(), "base launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}


}  // namespace

void launch_rht_in(const DevSide& side, const float* x, float* t, float* u_scratch, float* amax,
                   std::int32_t* zero_ptr, std::size_t zero_words, int batch, cudaStream_t s) {
  if (batch <= 0) return;
  const float scale = rsqrtf(float(side.n));
  const float* fw_in = x;
  if (side.q > 1) {
    BaseArgs a{};
    a.n = side.n;
    a.p = side.p;
    a.q = side.q;
    a.base = side.base;
    a.signs = side.signs;
    a.in = x;
    a.out = u_scratch;
    a.out_scale = 1.f;
    a.amax_zero = amax;
    a.batch = batch;
    a.fwd = 1;
    launch_base(side, a, batch, s);
    fw_in = u_scratch;
  } else {
    cuda_check(cudaMemsetAsync(amax, 0, sizeof(float) * batch, s), "amax zero");
  }
  FwhtArgs a{};
  a.n = side.n;
  a.p = side.p;
  a.q = side.q;
  a.cols_per_cta = fwht_cols_per_cta(side);
  a.signs = side.signs;
  a.in = fw_in;
  a.out = t;
  a.amax_out = amax;
  a.zero_ptr = zero_ptr;
  a.zero_words = zero_words;
  a.out_scale = scale;
  a.fwd = 1;
  const std::uint32_t ncols = (side.q + a.cols_per_cta - 1) / a.cols_per_cta;
  const std::uint32_t zero_ctas = zero_ptr && zero_words ? 16 : 0;
  const std::size_t smem = std::size_t(side.p) * std::min(a.cols_per_cta, side.q) * 4;
  static std::once_flag once;
  std::call_once(once, [] { set_smem(reinterpret_cast<const void*>(fwht_kernel), 200 * 1024); });
  fwht_kernel<<<dim3(ncols + zero_ctas, batch), kThreads, smem, s>>>(a);
  cuda_check(cudaGetLastError(), "fwht launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_rht_out(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                    const float zscale[2], const float* amax, float* u_scratch, float* y, int batch,
                    cudaStream_t s) {
  if (batch <= 0) return;
  const float scale = rsqrtf(float(side.n));
  FwhtArgs a{};
  a.n = side.n;
  a.p = side.p;
  a.q = side.q;
  a.cols_per_cta = fwht_cols_per_cta(side);
  a.signs = side.signs;
  a.zacc = zacc;
  a.zacc_stages = zacc_stages;
  a.zacc_rows = zacc_rows;
  a.amax = amax;
  a.zscale[0] = zscale[0];
  a.zscale[1] = zscale[1];
  a.out = side.q > 1 ? u_scratch : y;
  a.out_scale = side.q > 1 ? 1.f : scale;
  a.fwd = 0;
  const std::uint32_t ncols = (side.q + a.cols_per_cta - 1) / a.cols_per_cta;
  const std::size_t smem = std::size_t(side.p) * std::min(a.cols_per_cta, side.q) * 4;
  static std::once_flag once;
  std::call_once(once, [] { set_smem(reinterpret_cast<const void*>(fwht_kernel), 200 * 1024); });
  fwht_kernel<<<dim3(ncols, batch), kThreads, smem, s>>>(a);
  cuda_check(cudaGetLastError(), "fwht launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (side.q > 1) {
    BaseArgs bb{};
    bb.n = side.n;
    bb.p = side.p;
    bb.q = side.q;
    bb.base = side.base;
    bb.signs = side.signs;
    bb.in = u_scratch;
    bb.out = y;
    bb.out_scale = scale;
    bb.batch = batch;
    bb.fwd = 0;
    launch_base(side, bb, batch, s);
  }
}

}  // namespace q8p::detail
