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

#include <cmath>
#include <mutex>
#include <vector>

#include "device.hpp"

namespace q8p::detail {
namespace {

// e8p_encode of one 8-vector against the shared-memory tables.
__device__ std::uint32_t e8p_search(const double (&x)[8], const double (*half_d)[8], const std::uint8_t* par) {
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
    return best_word;
}

// E8P point of `word` (e8p.cpp:81-100): exact quarter-integers.
__device__ void e8p_point(std::uint32_t word, const double (*half_d)[8], const std::uint8_t* par, double (&p)[8]) {
  const std::uint32_t idx = word >> 8, sb = (word >> 1) & 0x7Fu;
  const double sh = (word & 1u) ? 0.25 : -0.25;
  const std::uint32_t neg0 = (__popc(sb) & 1u) ^ par[idx];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const std::uint32_t neg = c == 0 ? neg0 : ((sb >> (7 - c)) & 1u);
    p[c] = __dadd_rn(neg ? -half_d[idx][c] : half_d[idx][c], sh);
  }
}

// TableCodebook::encode (codebook.cpp:45-62) over the e8-1bit table: strict <, ties keep the smaller index.
__device__ std::uint32_t table_search(const double (&x)[8], const double (*tab)[8]) {
  double best = __longlong_as_double(0x7FF0000000000000LL);
  std::uint32_t best_i = 0;
  for (std::uint32_t i = 0; i < 256; ++i) {
    double dist = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double d = __dsub_rn(x[c], tab[i][c]);
      dist = __dadd_rn(dist, __dmul_rn(d, d));
    }
    if (dist < best) {
      best = dist;
      best_i = i;
    }
  }
  return best_i;
}

struct SharedTables {
  double half_d[256][8];  // E8P doubled / 2 (exact)
  double e81[256][8];     // e8-1bit entries (doubled / 2, exact)
  std::uint8_t par[256];
};

__device__ void load_tables(SharedTables& T, const std::int8_t* doubled, const std::uint8_t* odd,
                            const std::int8_t* e81_doubled) {
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) {
    T.half_d[i >> 3][i & 7] = 0.5 * double(doubled[i]);
    T.e81[i >> 3][i & 7] = 0.5 * double(e81_doubled[i]);
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) T.par[i] = odd[i];
  __syncthreads();
}

__global__ void __launch_bounds__(256) e8p_encode_kernel(const double* __restrict__ v, std::uint16_t* __restrict__ out,
                                                        std::size_t nblocks, const std::int8_t* __restrict__ doubled,
                                                        const std::uint8_t* __restrict__ odd,
                                                        const std::int8_t* __restrict__ e81) {
  __shared__ SharedTables T;
  load_tables(T, doubled, odd, e81);
  for (std::size_t blk = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; blk < nblocks;
       blk += std::size_t(gridDim.x) * blockDim.x) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = v[blk * 8 + c];
    out[blk] = std::uint16_t(e8p_search(x, T.half_d, T.par));
  }
}

// RvqQuantizer::quantize (rvq.cpp:59-79) per 8-vector: per stage scaled = residual / s,
// word = encode(scaled), residual -= s * decode(word).  kinds[i]: 0 = e8p-2bit, 1 = e8-1bit.
struct RvqStages {
  int n;
  int kind[2];
  double scale[2];
};
__global__ void __launch_bounds__(256) rvq_quantize_kernel(const double* __restrict__ v, std::uint16_t* __restrict__ codes,
                                                          std::size_t nblocks, RvqStages st,
                                                          const std::int8_t* __restrict__ doubled,
                                                          const std::uint8_t* __restrict__ odd,
                                                          const std::int8_t* __restrict__ e81) {
  __shared__ SharedTables T;
  load_tables(T, doubled, odd, e81);
  for (std::size_t blk = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; blk < nblocks;
       blk += std::size_t(gridDim.x) * blockDim.x) {
    double res[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) res[c] = v[blk * 8 + c];
    for (int i = 0; i < st.n; ++i) {
      const double s = st.scale[i];
      double sc[8], p[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) sc[c] = __ddiv_rn(res[c], s);
      std::uint32_t word;
      if (st.kind[i] == 0) {
        word = e8p_search(sc, T.half_d, T.par);
        e8p_point(word, T.half_d, T.par, p);
      } else {
        word = table_search(sc, T.e81);
#pragma unroll
        for (int c = 0; c < 8; ++c) p[c] = T.e81[word][c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) res[c] = __dsub_rn(res[c], __dmul_rn(s, p[c]));
      codes[std::size_t(i) * nblocks + blk] = std::uint16_t(word);
    }
  }
}

// SideTransform::apply (transforms.cpp:28-36) = had_apply(S o x) (hadamard.cpp:170-210)
// on every column of a row-major L x ncols f64 matrix, bit-identical to the
// reference's transform_cols (transforms.cpp:66-79): the same butterfly
// network (stride q, len ascending) and the same sequential base sums, in IEEE
// double without contraction.  CTA = 32 adjacent columns (lane = column, rows
// coalesced); butterflies in place in `w`, the base / 1/sqrt(n) step writes `out`.
__global__ void __launch_bounds__(256) rht_cols_f64_kernel(double* __restrict__ w, double* __restrict__ out,
                                                          std::uint32_t L, std::uint32_t ncols, std::uint32_t p,
                                                          std::uint32_t q, const std::uint8_t* __restrict__ signs,
                                                          const std::int8_t* __restrict__ base, double scale,
                                                          int transpose) {
  const std::uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const std::uint32_t col = blockIdx.x * 32 + lane;
  const bool on = col < ncols;
  // apply: signs, then H; apply_transpose: H^T (base transposed), then signs
  // (SideTransform::apply / apply_transpose, transforms.cpp:28-47)
  if (!transpose)
    for (std::uint32_t i = wid; i < L; i += nw)
      if (on && ((signs[i >> 3] >> (i & 7)) & 1u)) w[std::size_t(i) * ncols + col] = -w[std::size_t(i) * ncols + col];
  __syncthreads();
  for (std::uint32_t len = 1; len < p; len <<= 1) {
    for (std::uint32_t t = wid; t < (p / 2) * q; t += nw) {
      const std::uint32_t pi = t / q, j = t - pi * q;
      const std::uint32_t k = (pi / len) * 2 * len + pi % len;
      const std::size_t a = (std::size_t(k) * q + j) * ncols + col, b = (std::size_t(k + len) * q + j) * ncols + col;
      if (on) {
        const double u = w[a], v = w[b];
        w[a] = __dadd_rn(u, v);
        w[b] = __dsub_rn(u, v);
      }
    }
    __syncthreads();
  }
  for (std::uint32_t e = wid; e < L; e += nw) {
    if (!on) continue;
    double v;
    if (q == 1) {
      v = __dmul_rn(w[std::size_t(e) * ncols + col], scale);
    } else {
      const std::uint32_t r = e / q, a = e - r * q;
      double acc = 0.0;
      for (std::uint32_t b = 0; b < q; ++b)
        acc = __dadd_rn(acc, __dmul_rn(double(base[transpose ? b * q + a : a * q + b]),
                                       w[(std::size_t(r) * q + b) * ncols + col]));
      v = __dmul_rn(acc, scale);
    }
    if (transpose && ((signs[e >> 3] >> (e & 7)) & 1u)) v = -v;
    out[std::size_t(e) * ncols + col] = v;
  }
}

struct EncodeTables {
  std::int8_t* doubled = nullptr;
  std::uint8_t* odd = nullptr;
  std::int8_t* e81 = nullptr;
};

const EncodeTables& device_tables(int& dev) {
  cuda_check(cudaGetDevice(&dev), "get device");
  static std::mutex mu;
  static EncodeTables tabs[64];
  std::scoped_lock lock(mu);
  if (dev < 0 || dev >= 64) throw DeviceError("device index out of range");
  if (!tabs[dev].doubled) {
    const E8PTable& t = e8p_table();
    std::vector<std::int8_t> e81(256 * 8);
    for (int i = 0; i < 256; ++i)
      for (int c = 0; c < 8; ++c) e81[i * 8 + c] = e8_1bit_doubled()[i][c];
    cuda_check(cudaMalloc(&tabs[dev].doubled, 256 * 8), "encode tables");
    cuda_check(cudaMalloc(&tabs[dev].odd, 256), "encode tables");
    cuda_check(cudaMalloc(&tabs[dev].e81, 256 * 8), "encode tables");
    cuda_check(cudaMemcpy(tabs[dev].doubled, t.doubled.data(), 256 * 8, cudaMemcpyHostToDevice), "encode tables");
    cuda_check(cudaMemcpy(tabs[dev].odd, t.odd_parity.data(), 256, cudaMemcpyHostToDevice), "encode tables");
    cuda_check(cudaMemcpy(tabs[dev].e81, e81.data(), 256 * 8, cudaMemcpyHostToDevice), "encode tables");
  }
  return tabs[dev];
}

unsigned grid_for(std::size_t nblocks, int dev) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return unsigned(std::min<std::size_t>((nblocks + 255) / 256, std::size_t(sms) * 8));
}

// Dequantize (dequantize_layer, pipeline.cpp:112-149): w[r][8k+c] =
// sum_s scale_s * point_s[c], accumulated from 0.0 in stage order in f64 as
// decode_incoherent does; points from K2's decoder output (a, b): E8P
// (2a + 2b - 1) / 4, e8-1bit a / 2 (exact).
__global__ void __launch_bounds__(256) dequant_combine_kernel(const std::int8_t* __restrict__ a0,
                                                              const std::uint8_t* __restrict__ b0,
                                                              const std::int8_t* __restrict__ a1,
                                                              const std::uint8_t* __restrict__ b1, int nst, int kind0,
                                                              int kind1, double s0, double s1, std::size_t total,
                                                              double* __restrict__ w) {
  for (std::size_t i = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += std::size_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < nst; ++s) {
      const std::int8_t* a = s ? a1 : a0;
      const std::uint8_t* b = s ? b1 : b0;
      const int kind = s ? kind1 : kind0;
      const double pt = kind == 0 ? (2.0 * a[i] + 2.0 * b[i >> 3] - 1.0) * 0.25 : a[i] * 0.5;
      acc = __dadd_rn(acc, __dmul_rn(s ? s1 : s0, pt));
    }
    w[i] = acc;
  }
}
// Unscaled points of one stage (Codebook::decode) as fp32 from K2's decoder output.
__global__ void __launch_bounds__(256) points_f32_kernel(const std::int8_t* __restrict__ a,
                                                         const std::uint8_t* __restrict__ b, int kind,
                                                         std::size_t total, float* __restrict__ w) {
  for (std::size_t i = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += std::size_t(gridDim.x) * blockDim.x)
    w[i] = kind == 0 ? (2.f * a[i] + 2.f * b[i >> 3] - 1.f) * 0.25f : a[i] * 0.5f;
}
__global__ void __launch_bounds__(256) transpose_f64_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                            std::uint32_t rows, std::uint32_t cols) {
  __shared__ double t[32][33];
  const std::uint32_t bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (std::uint32_t j = threadIdx.y; j < 32; j += 8)
    if (by + j < rows && bx + threadIdx.x < cols) t[j][threadIdx.x] = in[std::size_t(by + j) * cols + bx + threadIdx.x];
  __syncthreads();
  for (std::uint32_t j = threadIdx.y; j < 32; j += 8)
    if (bx + j < cols && by + threadIdx.x < rows) out[std::size_t(bx + j) * rows + by + threadIdx.x] = t[threadIdx.x][j];
}

}  // namespace

void launch_dequant_combine(const std::int8_t* a0, const std::uint8_t* b0, const std::int8_t* a1,
                            const std::uint8_t* b1, int nst, int kind0, int kind1, double s0, double s1,
                            std::size_t total, double* w, cudaStream_t s) {
  dequant_combine_kernel<<<unsigned(std::min<std::size_t>((total + 255) / 256, 148 * 16)), 256, 0, s>>>(
      a0, b0, a1, b1, nst, kind0, kind1, s0, s1, total, w);
  cuda_check(cudaGetLastError(), "dequant combine launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_points_f32(const std::int8_t* a, const std::uint8_t* b, int kind, std::size_t total, float* w,
                       cudaStream_t s) {
  points_f32_kernel<<<unsigned(std::min<std::size_t>((total + 255) / 256, 148 * 16)), 256, 0, s>>>(a, b, kind, total, w);
  cuda_check(cudaGetLastError(), "points launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_transpose_f64(const double* in, double* out, std::uint32_t rows, std::uint32_t cols, cudaStream_t s) {
  transpose_f64_kernel<<<dim3((cols + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, s>>>(in, out, rows, cols);
  cuda_check(cudaGetLastError(), "transpose launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_e8p_encode(const double* v, std::uint16_t* words, std::size_t nblocks, cudaStream_t s) {
  if (nblocks == 0) return;
  int dev = 0;  // set by device_tables (the calling thread's device)
  const EncodeTables& t = device_tables(dev);
  e8p_encode_kernel<<<grid_for(nblocks, dev), 256, 0, s>>>(v, words, nblocks, t.doubled, t.odd, t.e81);
  cuda_check(cudaGetLastError(), "e8p encode launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_rht_cols_f64(double* w, double* scratch, std::uint32_t L, std::uint32_t ncols, const std::uint8_t* signs,
                         cudaStream_t s, bool transpose) {
  if (L == 0 || ncols == 0) return;
  const HadamardSpec spec = plan_hadamard(L);
  const int dev = current_device();
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, std::size_t>, std::int8_t*>> bases;  // (device, q) -> base
  const std::int8_t* base = nullptr;
  if (spec.q > 1) {
    std::scoped_lock lock(mu);
    for (auto& e : bases)
      if (e.first == std::make_pair(dev, spec.q)) base = e.second;
    if (!base) {
      const std::vector<std::int8_t>& hb = hadamard_base(spec.q);
      std::int8_t* d = nullptr;
      cuda_check(cudaMalloc(&d, hb.size()), "base alloc");
      cuda_check(cudaMemcpy(d, hb.data(), hb.size(), cudaMemcpyHostToDevice), "base upload");
      bases.push_back({{dev, spec.q}, d});
      base = d;
    }
  }
  const double scale = 1.0 / std::sqrt(double(L));  // had_apply's 1/sqrt(n) (hadamard.cpp:188)
  rht_cols_f64_kernel<<<(ncols + 31) / 32, 256, 0, s>>>(w, scratch, L, ncols, std::uint32_t(spec.p),
                                                        std::uint32_t(spec.q), signs, base, scale,
                                                        transpose ? 1 : 0);
  cuda_check(cudaGetLastError(), "rht f64 launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cuda_check(cudaMemcpyAsync(w, scratch, std::size_t(L) * ncols * 8, cudaMemcpyDeviceToDevice, s), "rht f64 copy");
}

void launch_rvq_quantize(const double* v, std::uint16_t* codes, std::size_t nblocks, int stages, const int* kinds,
                         const double* scales, cudaStream_t s) {
  if (nblocks == 0) return;
  if (stages < 1 || stages > 2) throw ValidationError("rvq: 1 or 2 stages on this path");
  RvqStages st{};
  st.n = stages;
  for (int i = 0; i < stages; ++i) {
    if (kinds[i] != 0 && kinds[i] != 1) throw ValidationError("rvq: unknown codebook");
    if (!(scales[i] > 0.0) || !std::isfinite(scales[i])) throw ValidationError("RvqQuantizer: scales must be positive");
    st.kind[i] = kinds[i];
    st.scale[i] = scales[i];
  }
  int dev = 0;  // set by device_tables (the calling thread's device)
  const EncodeTables& t = device_tables(dev);
  rvq_quantize_kernel<<<grid_for(nblocks, dev), 256, 0, s>>>(v, codes, nblocks, st, t.doubled, t.odd, t.e81);
  cuda_check(cudaGetLastError(), "rvq quantize launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
