// GPU producer piece: the exact E8P encoder
// e8p_encode (core/src/e8p.cpp:114-156) -- for every 8-vector the nearest of
// the 2^16 E8P codewords, found as the reference does: for each of the 256
// rows and both shift signs, the coordinatewise-optimal signs (ties keep +),
// parity repaired by flipping the coordinate with the smallest
// |v - shift| * d / 2, then the squared distance to the decoded point, the
// smallest distance winning with ties to the smaller word.
//
// Bit-identical to the reference: the arithmetic is IEEE double in the
// reference's order with explicit _rn intrinsics (no FMA contraction), and the
// decoded point sigma_c d_c / 2 + shift is exact (quarter-integers) whichever
// way it is formed.  One thread per 8-vector; the 256-row table lives in
// shared memory.  Used to quantize at 70B shapes without the CPU producer's
// minutes (the north star keeps the producer on the reference's CPU code; this
// is the optional accelerator of its inner search).
#include <cuda_runtime.h>

#include "device.hpp"

namespace q8p::detail {
namespace {

__global__ void __launch_bounds__(256) e8p_encode_kernel(const double* __restrict__ v, std::uint16_t* __restrict__ out,
                                                        std::size_t nblocks, const std::int8_t* __restrict__ doubled,
                                                        const std::uint8_t* __restrict__ odd) {
  __shared__ double half_d[256][8];  // doubled / 2 (exact)
  __shared__ std::uint8_t par[256];
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) half_d[i >> 3][i & 7] = 0.5 * double(doubled[i]);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) par[i] = odd[i];
  __syncthreads();
  for (std::size_t blk = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; blk < nblocks;
       blk += std::size_t(gridDim.x) * blockDim.x) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = v[blk * 8 + c];
    double best = __longlong_as_double(0x7FF0000000000000LL);  // +inf
    std::uint32_t best_word = 0;
    for (std::uint32_t idx = 0; idx < 256; ++idx) {
#pragma unroll
      for (std::uint32_t shift_bit = 0; shift_bit < 2; ++shift_bit) {
        const double shift = shift_bit ? 0.25 : -0.25;
        std::uint32_t negmask = 0, flips = 0, min_c = 0;
        double min_pen = __longlong_as_double(0x7FF0000000000000LL);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double y = __dsub_rn(x[c], shift);
          const bool neg = y < 0.0;
          negmask |= std::uint32_t(neg) << c;
          flips += neg;
          const double pen = __dmul_rn(fabs(y), half_d[idx][c]);
          if (pen < min_pen) {
            min_pen = pen;
            min_c = std::uint32_t(c);
          }
        }
        if ((flips & 1u) != par[idx]) negmask ^= 1u << min_c;
        // word: idx << 8 | sign bits of coordinates 7..1 (bit j-1 = coordinate 8-j) << 1 | shift bit
        std::uint32_t sb = 0;
#pragma unroll
        for (int j = 1; j <= 7; ++j) sb |= ((negmask >> (8 - j)) & 1u) << (j - 1);
        const std::uint32_t word = (idx << 8) | (sb << 1) | shift_bit;
        double dist = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double p = __dadd_rn(((negmask >> c) & 1u) ? -half_d[idx][c] : half_d[idx][c], shift);
          const double d = __dsub_rn(x[c], p);
          dist = __dadd_rn(dist, __dmul_rn(d, d));
        }
        if (dist < best || (dist == best && word < best_word)) {
          best = dist;
          best_word = word;
        }
      }
    }
    out[blk] = std::uint16_t(best_word);
  }
}

struct EncodeTables {
  std::int8_t* doubled = nullptr;
  std::uint8_t* odd = nullptr;
};

}  // namespace

void launch_e8p_encode(const double* v, std::uint16_t* words, std::size_t nblocks, cudaStream_t s) {
  if (nblocks == 0) return;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "get device");
  static std::mutex mu;
  static EncodeTables tabs[64];
  {
    std::scoped_lock lock(mu);
    if (dev < 0 || dev >= 64) throw DeviceError("device index out of range");
    if (!tabs[dev].doubled) {
      const E8PTable& t = e8p_table();
      cuda_check(cudaMalloc(&tabs[dev].doubled, 256 * 8), "encode tables");
      cuda_check(cudaMalloc(&tabs[dev].odd, 256), "encode tables");
      cuda_check(cudaMemcpy(tabs[dev].doubled, t.doubled.data(), 256 * 8, cudaMemcpyHostToDevice), "encode tables");
      cuda_check(cudaMemcpy(tabs[dev].odd, t.odd_parity.data(), 256, cudaMemcpyHostToDevice), "encode tables");
    }
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const std::size_t want = (nblocks + 255) / 256;
  const unsigned grid = unsigned(std::min<std::size_t>(want, std::size_t(sms) * 8));
  e8p_encode_kernel<<<grid, 256, 0, s>>>(v, words, nblocks, tabs[dev].doubled, tabs[dev].odd);
  cuda_check(cudaGetLastError(), "e8p encode launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
