// K0 (decode), K1/K3 (randomized Hadamard transform) and the portable K2
// GEMV used for batches the tensor-core GEMV does not cover.
//
// Reference semantics:
//   e8p_decode            core/src/e8p.cpp:81-100
//   TableCodebook decode  core/src/codebook.cpp:65-72 (e8-1bit table)
//   had_apply             core/src/hadamard.cpp:170-210
//   SideTransform         core/src/transforms.cpp:28-47
//   infer hot loop        core/src/pipeline.cpp:172-191
#include <cuda_runtime.h>

#include "device.hpp"

namespace q8p::detail {
namespace {

// E8P table in constant memory: per row 8 doubled magnitudes packed as
// nibbles + odd parity (bit 32 of the packed row word).
struct ConstTables {
  std::uint32_t e8p_abs[256];   // nibble c = doubled[c] (1, 3 or 5)
  std::uint8_t e8p_odd[256];
  std::int8_t e81[256][8];      // e8-1bit, doubled coordinates
};
__constant__ ConstTables c_tab;
// __constant__ memory is per device: one upload per device.
std::once_flag g_tab_once[64];

void upload_tables() {
  const int dev = current_device();
  if (dev < 0 || dev >= 64) throw DeviceError("device index beyond the table cache");
  std::call_once(g_tab_once[dev], [] {
    ConstTables h{};
    const E8PTable& t = e8p_table();
    for (int i = 0; i < 256; ++i) {
      std::uint32_t w = 0;
      for (int c = 0; c < 8; ++c) w |= std::uint32_t(t.doubled[i][c]) << (4 * c);
      h.e8p_abs[i] = w;
      h.e8p_odd[i] = t.odd_parity[i];
      for (int c = 0; c < 8; ++c) h.e81[i][c] = e8_1bit_doubled()[i][c];
    }
    cuda_check(cudaMemcpyToSymbol(c_tab, &h, sizeof h), "upload tables");
  });
}

// Decoded (unscaled) codeword, fp32 quarter-integers.  `words` is the raw
// code, `cb` 0 = E8P, 1 = e8-1bit; smem copies of the tables.
struct SmemTables {
  std::uint32_t abs[256];
  std::uint8_t odd[256];
  std::int8_t e81[256][8];
};

__device__ __forceinline__ void decode_word(const SmemTables& T, int cb, std::uint32_t w, float v[8]) {
  if (cb == 0) {
    const std::uint32_t idx = w >> 8, sb = (w >> 1) & 0x7Fu;
    const float sh = (w & 1u) ? 0.25f : -0.25f;
    const std::uint32_t a = T.abs[idx];
    const std::uint32_t neg0 = (__popc(sb) & 1u) ^ T.odd[idx];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float mag = 0.5f * float((a >> (4 * c)) & 0xFu);
      const std::uint32_t neg = c == 0 ? neg0 : ((sb >> (7 - c)) & 1u);
      v[c] = (neg ? -mag : mag) + sh;
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = 0.5f * float(T.e81[w & 0xFFu][c]);
  }
}

__device__ __forceinline__ void load_tables(SmemTables& T) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    T.abs[i] = c_tab.e8p_abs[i];
    T.odd[i] = c_tab.e8p_odd[i];
#pragma unroll
    for (int c = 0; c < 8; ++c) T.e81[i][c] = c_tab.e81[i][c];
  }
  __syncthreads();
}

__device__ __forceinline__ std::uint32_t load_code(const void* codes, int cb, std::size_t i) {
  return cb == 0 ? std::uint32_t(static_cast<const std::uint16_t*>(codes)[i])
                 : std::uint32_t(static_cast<const std::uint8_t*>(codes)[i]);
}

// ---- K1 / K3: randomized Hadamard transform ------------------------------
// One CTA per vector.  y = H (S o x) (forward) or y = S o (H^T x)
// (transpose), H = (H_p (x) B_q) / sqrt(n), flat index i = a * q + b.
__global__ void rht_kernel(std::uint32_t n, std::uint32_t p, std::uint32_t q,
                           const std::uint8_t* __restrict__ signs, const std::int8_t* __restrict__ base,
                           const float* __restrict__ x, float* __restrict__ y, int transpose) {
  extern __shared__ float sm[];
  float* s = sm;
  std::int8_t* B = reinterpret_cast<std::int8_t*>(sm + n);
  const float* xv = x + std::size_t(blockIdx.x) * n;
  float* yv = y + std::size_t(blockIdx.x) * n;
  for (std::uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    float v = xv[i];
    if (!transpose && ((signs[i >> 3] >> (i & 7)) & 1)) v = -v;
    s[i] = v;
  }
  if (q > 1)
    for (std::uint32_t i = threadIdx.x; i < q * q; i += blockDim.x) B[i] = base[i];
  __syncthreads();
  // Unnormalized butterflies along the power-of-two axis (stride q).
  const std::uint32_t half = (p >> 1) * q;
  for (std::uint32_t len = 1; len < p; len <<= 1) {
    for (std::uint32_t t = threadIdx.x; t < half; t += blockDim.x) {
      const std::uint32_t pair = t / q, j = t - pair * q;
      const std::uint32_t blk = pair / len, off = pair - blk * len;
      const std::uint32_t k = blk * 2 * len + off;
      const float u = s[k * q + j], v = s[(k + len) * q + j];
      s[k * q + j] = u + v;
      s[(k + len) * q + j] = u - v;
    }
    __syncthreads();
  }
  const float scale = rsqrtf(float(n));
  for (std::uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    float v;
    if (q == 1) {
      v = s[i];
    } else {
      const std::uint32_t r = i / q, a = i - r * q;
      const float* seg = s + r * q;
      float acc = 0.f;
      if (transpose)
        for (std::uint32_t b = 0; b < q; ++b) acc += float(B[b * q + a]) * seg[b];
      else
        for (std::uint32_t b = 0; b < q; ++b) acc += float(B[a * q + b]) * seg[b];
      v = acc;
    }
    v *= scale;
    if (transpose && ((signs[i >> 3] >> (i & 7)) & 1)) v = -v;
    yv[i] = v;
  }
}

// ---- K2 (portable): one warp per row, fp32 ---------------------------------
// z[b][r] = sum_s scale_s * sum_k <decode_s(code[s][r][k]), t[b][8k:8k+8]>
template <int BT>
__global__ void gemv_simple_kernel(const void* __restrict__ c0, const void* __restrict__ c1, int cb0,
                                   int cb1, float s0, float s1, int stages,
                                   const float* __restrict__ t, float* __restrict__ z,
                                   std::uint32_t rows, std::uint32_t n, int batch, int z_stride) {
  __shared__ SmemTables T;
  load_tables(T);
  const std::uint32_t nb = n / 8;
  const int lane = threadIdx.x & 31;
  const std::uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const std::uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int b0 = 0; b0 < batch; b0 += BT) {
    const int bn = min(BT, batch - b0);
    for (std::uint32_t r = warp; r < rows; r += nwarps) {
      float acc[BT];
#pragma unroll
      for (int b = 0; b < BT; ++b) acc[b] = 0.f;
      for (std::uint32_t k = lane; k < nb; k += 32) {
        float blk[8], v[8];
        decode_word(T, cb0, load_code(c0, cb0, std::size_t(r) * nb + k), v);
#pragma unroll
        for (int c = 0; c < 8; ++c) blk[c] = s0 * v[c];
        if (stages > 1) {
          decode_word(T, cb1, load_code(c1, cb1, std::size_t(r) * nb + k), v);
#pragma unroll
          for (int c = 0; c < 8; ++c) blk[c] += s1 * v[c];
        }
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          if (b < bn) {
            const float4* tv = reinterpret_cast<const float4*>(t + std::size_t(b0 + b) * n + 8 * k);
            const float4 lo = tv[0], hi = tv[1];
            acc[b] += blk[0] * lo.x + blk[1] * lo.y + blk[2] * lo.z + blk[3] * lo.w + blk[4] * hi.x +
                      blk[5] * hi.y + blk[6] * hi.z + blk[7] * hi.w;
          }
        }
      }
#pragma unroll
      for (int b = 0; b < BT; ++b) {
        float v = acc[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && b < bn) z[std::size_t(b0 + b) * z_stride + r] = v;
      }
    }
  }
}

int num_sms() {
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

}  // namespace

void launch_rht(const DevSide& side, const float* x, float* y, int batch, bool transpose,
                cudaStream_t s) {
  if (batch <= 0) return;
  const std::size_t smem = side.n * sizeof(float) + (side.q > 1 ? side.q * side.q : 0);
  kernel_attrs(reinterpret_cast<const void*>(rht_kernel), 227 * 1024);
  if (smem > 227 * 1024) throw SizeError("rht: n too large for the single-CTA transform");
  rht_kernel<<<batch, 1024, smem, s>>>(side.n, side.p, side.q, side.signs, side.base, x, y,
                                       transpose ? 1 : 0);
  cuda_check(cudaGetLastError(), "rht launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_gemv_simple(const q8p_layer& L, const float* t, float* z, int batch, int z_stride,
                        cudaStream_t s) {
  upload_tables();
  const int blocks = num_sms() * 4;
  gemv_simple_kernel<4><<<blocks, 256, 0, s>>>(L.codes[0], L.codes[1], L.cb[0], L.cb[1], L.scale[0],
                                               L.scale[1], L.num_stages, t, z, L.m_local(), L.n,
                                               batch, z_stride);
  cuda_check(cudaGetLastError(), "gemv launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}


}  // namespace q8p::detail
