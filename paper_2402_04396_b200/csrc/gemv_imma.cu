// K2: E8P / RVQ decode fused into a batch-1..4 GEMV on the tensor cores.
//
// Semantics: z[r] = sum_s scale_s * sum_k <decode_s(codes[s][r][k]), t[8k:8k+8]>
// (core/src/pipeline.cpp:172-191) with decode = e8p_decode
// (core/src/e8p.cpp:81-100) or the e8-1bit table (core/src/codebook.cpp:65-72).
//
// Why tensor cores for a GEMV: at 2 bits/weight B200 HBM delivers ~11.6
// codewords per SM-clock; the issue budget is ~11 thread-instructions per
// 8-weight codeword and the ALU pipe only half of that.  The decode is
// therefore reshaped so the tensor core does all multiply-adds and the ALU
// only builds int8 operand bytes:
//
//   v_c = sigma_c d_c / 2 + s / 4      (d in {1,3,5}, s = +-1 shift)
//   z   = 1/2 sum_c (sigma_c d_c) t_c  +  1/4 sum_k s_k T_k      (T_k = block sum)
//
// A operand (s8): sigma_c d_c, produced per 4 coordinates by ONE byte-permute
// from a constant 8-entry table {1,3,5,_,-1,-3,-5,_}; the selector nibbles
// (magnitude index from a smem LUT, negate flag from the sign bits) cost one
// LOP3.  The +-1/4 shift is a second "side" MMA with A = 4 s_k (one byte per
// codeword) against B = block sums / 8.  Activations are exact-ish int8:
// t = alpha (128 hi + lo) (2 limbs, |err| <= alpha/2, alpha = max|t|/16256),
// carried as separate MMA columns, so int32 accumulation is exact and the
// result is independent of summation order (split-K partials are combined
// with integer atomics -> deterministic).
//
// Device code layout ("tile format", built once at upload from the QSHP
// codes -- a lossless, documented re-layout):
//   tile (row tile rt = 16 rows, k-step ks = 32 codewords = 256 columns),
//   1 KiB = [half h][lane = 4 g + t][16 B]: the 8 codewords of row
//   16 rt + g + 8 h at blocks 32 ks + 4 j + t, j = 0..7:
//     bytes 0..7 : idx_j = word_j >> 8
//     bytes 8..15: two bit-sliced sign registers R0 (j = 0..3), R1 (j = 4..7):
//                  bit 4 c + j' = (c == 0) ? shift bit : word bit (8 - c)
//   The coordinate-0 sign (parity-inferred, e8p.cpp:97-98) is rebuilt with a
//   3-step XOR fold per register; odd_parity[idx] is folded into the LUT.
// e8-1bit tiles: [half][lane][8 B] = the 8 code bytes; A = LUT row directly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "device.hpp"

namespace q8p::detail {
namespace {

constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kChunk = 8;        // k-steps per B chunk
constexpr int kMaxChunks = 2;    // B chunks resident per CTA
constexpr int kBWords = 20;      // u32 per (k-step, lane) in the B smem image (18 used)
constexpr std::size_t kLutBytes = 256 * 256;
constexpr std::size_t kBBytes = std::size_t(kMaxChunks) * kChunk * 32 * kBWords * 4;
constexpr float kLimbMax = 16256.f;  // 127 * 128

struct ImmaArgs {
  const uint4* tiles0;   // stage 0 (always e8p-2bit)
  const void* tiles1;    // stage 1: e8p-2bit (uint4 lanes) or e8-1bit (uint2 lanes)
  int stages;
  int kind1;             // stage 1 codebook: 0 = e8p, 1 = e8-1bit
  std::uint32_t RT, KS, NKC, KL;  // row tiles, k-steps, chunks, k-steps in last chunk
  std::uint32_t nb, n;
  std::uint32_t units;
  const float* t;        // [batch][n]
  const float* amax;     // [batch]
  int batch;             // 1..4
  std::int32_t* zacc;    // [stage][8][rows_pad]
  std::uint32_t rows_pad;
  const std::uint32_t* lut_e8p;   // [256]: nibble c = delta_c | (c == 0 ? odd << 2 : 0)
  const std::uint32_t* lut_e81;   // [256][2]: doubled coordinates as s8
};

__device__ __forceinline__ void mma_s8(int (&d)[4], std::uint32_t a0, std::uint32_t a1, std::uint32_t a2,
                                       std::uint32_t a3, std::uint32_t b0, std::uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_stream2(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];\n" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// Unit u -> (row tile, k-step).  Units are ordered chunk-major (8 k-steps per
// chunk), then row tile, then k-step, so a warp's contiguous unit range walks
// the k-steps of one row tile before moving on.
__device__ __forceinline__ void unit_coords(const ImmaArgs& a, std::uint32_t u, std::uint32_t& rt,
                                            std::uint32_t& ks, std::uint32_t& kc) {
  const std::uint32_t full = kChunk * a.RT;
  kc = u / full;
  if (kc >= a.NKC) kc = a.NKC - 1;
  const std::uint32_t up = u - kc * full;
  const std::uint32_t size = (kc == a.NKC - 1) ? a.KL : kChunk;
  rt = up / size;
  ks = kc * kChunk + (up - rt * size);
}

// Parity fix of one sign register: slot (c=0, j') <- XOR of its 8 slots
// (= shift ^ parity(explicit signs)) XOR shift = parity.
__device__ __forceinline__ std::uint32_t parity_fix(std::uint32_t r) {
  const std::uint32_t f1 = r ^ (r * 16u) ^ (r * 256u);
  const std::uint32_t f2 = f1 ^ (f1 * 4096u) ^ (f1 * 16777216u);
  return r ^ __umulhi(f2, 16u);  // f2 >> 28
}

// Side-MMA operand: byte j' = shift ? +4 : -4 from slot (0, j').
__device__ __forceinline__ std::uint32_t side_bytes(std::uint32_t r) {
  const std::uint32_t spread = ((r & 0xFu) * 0x01020408u) & 0x08080808u;  // 8 * b_j'
  return (spread * 31u) ^ 0xFCFCFCFCu;                                     // 8b*31 ^ 0xFC = b ? 4 : -4
}

constexpr std::uint32_t kCtLo = 0x00050301u;  // {+1,+3,+5,0}
constexpr std::uint32_t kCtHi = 0x00FBFDFFu;  // {-1,-3,-5,0}

// Decodes codeword jj (0..3) of an E8P half-register pair into A bytes.
__device__ __forceinline__ void e8p_operands(const char* lut, std::uint32_t idxreg, std::uint32_t rfix,
                                             std::uint32_t lanebase, int jj, std::uint32_t& alo,
                                             std::uint32_t& ahi) {
  const std::uint32_t addr = __byte_perm(idxreg, lanebase, 0x5504u | (std::uint32_t(jj) << 4));
  const std::uint32_t nib = *reinterpret_cast<const std::uint32_t*>(lut + addr);
  std::uint32_t rs;
  if (jj == 0)
    rs = rfix * 4u;
  else if (jj == 1)
    rs = rfix * 2u;
  else if (jj == 2)
    rs = rfix;
  else
    rs = __umulhi(rfix, 0x80000000u);  // >> 1
  const std::uint32_t sel = nib ^ (rs & 0x44444444u);
  alo = __byte_perm(kCtLo, kCtHi, sel);
  ahi = __byte_perm(kCtLo, kCtHi, __umulhi(sel, 65536u));
}

__device__ __forceinline__ void e81_operands(const char* lut, std::uint32_t codereg, std::uint32_t lanebase8,
                                             int jj, std::uint32_t& alo, std::uint32_t& ahi) {
  const std::uint32_t addr = __byte_perm(codereg, lanebase8, 0x5504u | (std::uint32_t(jj) << 4));
  const uint2 v = *reinterpret_cast<const uint2*>(lut + addr);
  alo = v.x;
  ahi = v.y;
}

template <int STAGES, int KIND1>
__global__ void __launch_bounds__(kThreads, 1) gemv_imma_kernel(ImmaArgs a) {
  constexpr int kPrefetch = STAGES == 1 ? 4 : 2;  // code units in flight per warp
  extern __shared__ __align__(16) char smem[];
  char* lut = smem;                                              // 64 KiB
  std::uint32_t* bsm = reinterpret_cast<std::uint32_t*>(smem + kLutBytes);  // B images
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint32_t W = gridDim.x * kWarps;
  const std::uint32_t gw = blockIdx.x * kWarps + warp;
  const std::uint32_t u0 = std::uint32_t((std::uint64_t(a.units) * gw) / W);
  const std::uint32_t u1 = std::uint32_t((std::uint64_t(a.units) * (gw + 1)) / W);
  const std::uint32_t cu0 = std::uint32_t((std::uint64_t(a.units) * (blockIdx.x * kWarps)) / W);
  const std::uint32_t cu1 = std::uint32_t((std::uint64_t(a.units) * ((blockIdx.x + 1) * kWarps)) / W);

  // ---- prefetch the first code units (overlaps the prologue) -------------
  uint4 pf0[kPrefetch][2];
  uint4 pf1[STAGES > 1 ? kPrefetch : 1][2];
  uint2 pf1b[STAGES > 1 ? kPrefetch : 1][2];
  auto tile_index = [&](std::uint32_t u) -> std::size_t {
    std::uint32_t rt, ks, kc;
    unit_coords(a, u, rt, ks, kc);
    return (std::size_t(rt) * a.KS + ks) * 64 + lane;  // in 16-B lanes: 2 halves x 32 lanes
  };
#pragma unroll
  for (int i = 0; i < kPrefetch; ++i) {
    const std::uint32_t u = u0 + i;
    if (u < u1) {
      const std::size_t ti = tile_index(u);
      pf0[i][0] = ldg_stream(a.tiles0 + ti);
      pf0[i][1] = ldg_stream(a.tiles0 + ti + 32);
      if constexpr (STAGES > 1) {
        if constexpr (KIND1 == 0) {
          pf1[i][0] = ldg_stream(static_cast<const uint4*>(a.tiles1) + ti);
          pf1[i][1] = ldg_stream(static_cast<const uint4*>(a.tiles1) + ti + 32);
        } else {
          pf1b[i][0] = ldg_stream2(static_cast<const uint2*>(a.tiles1) + ti);
          pf1b[i][1] = ldg_stream2(static_cast<const uint2*>(a.tiles1) + ti + 32);
        }
      }
    }
  }

  // ---- LUTs: E8P nibbles replicated per lane (bytes [0,128) of each 256-B row),
  //      e8-1bit rows replicated per half-warp lane (bytes [128,256)) ---------
  for (std::uint32_t i = threadIdx.x; i < 256 * 32; i += kThreads) {
    const std::uint32_t row = i >> 5, l = i & 31;
    reinterpret_cast<std::uint32_t*>(lut + row * 256)[l] = a.lut_e8p[row];
  }
  if constexpr (STAGES > 1 && KIND1 == 1) {
    for (std::uint32_t i = threadIdx.x; i < 256 * 16; i += kThreads) {
      const std::uint32_t row = i >> 4, l = i & 15;
      reinterpret_cast<uint2*>(lut + row * 256 + 128)[l] =
          make_uint2(a.lut_e81[2 * row], a.lut_e81[2 * row + 1]);
    }
  }

  // ---- B images for the CTA's k-chunks ------------------------------------
  std::uint32_t rt_, ks_, kc_lo, kc_hi;
  unit_coords(a, cu0, rt_, ks_, kc_lo);
  unit_coords(a, cu1 > cu0 ? cu1 - 1 : cu0, rt_, ks_, kc_hi);
  const std::uint32_t nchunk = kc_hi - kc_lo + 1;  // <= kMaxChunks (host guarantees)
  for (std::uint32_t i = threadIdx.x; i < nchunk * kChunk * 32 * kBWords; i += kThreads) bsm[i] = 0;
  __syncthreads();
  {
    // task = (chunk, ksl, j, t, b): 8 activations of block 32 ks + 4 j + t of vector b
    const std::uint32_t tasks = nchunk * kChunk * 8 * 4 * a.batch;
    for (std::uint32_t task = threadIdx.x; task < tasks; task += kThreads) {
      std::uint32_t r = task;
      const std::uint32_t b = r % a.batch;
      r /= a.batch;
      const std::uint32_t tt = r & 3;
      r >>= 2;
      const std::uint32_t j = r & 7;
      r >>= 3;
      const std::uint32_t ksl = r % kChunk;
      const std::uint32_t ch = r / kChunk;
      const std::uint32_t ks = (kc_lo + ch) * kChunk + ksl;
      if (ks >= a.KS) continue;
      const std::uint32_t blk = ks * 32 + 4 * j + tt;
      float v[8];
      float am = a.amax[b];
      const float inv = am > 0.f ? kLimbMax / am : 0.f;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        v[c] = blk < a.nb ? a.t[std::size_t(b) * a.n + 8 * blk + c] : 0.f;
        sum += v[c];
      }
      std::uint32_t hi[2] = {0, 0}, lo[2] = {0, 0};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float s = v[c] * inv;
        const float h = rintf(s * (1.f / 128.f));
        const float l = rintf(s - 128.f * h);
        hi[c >> 2] |= (std::uint32_t(std::int32_t(h)) & 0xFFu) << (8 * (c & 3));
        lo[c >> 2] |= (std::uint32_t(std::int32_t(l)) & 0xFFu) << (8 * (c & 3));
      }
      // block sum / 8 in the same units
      const float s = sum * 0.125f * inv;
      const float h = rintf(s * (1.f / 128.f));
      const float l = rintf(s - 128.f * h);
      std::uint32_t* base = bsm + (std::size_t(ch) * kChunk + ksl) * 32 * kBWords;
      const std::uint32_t lane_hi = (2 * b) * 4 + tt, lane_lo = (2 * b + 1) * 4 + tt;
      base[lane_hi * kBWords + 2 * j] = hi[0];
      base[lane_hi * kBWords + 2 * j + 1] = hi[1];
      base[lane_lo * kBWords + 2 * j] = lo[0];
      base[lane_lo * kBWords + 2 * j + 1] = lo[1];
      reinterpret_cast<std::uint8_t*>(base + lane_hi * kBWords + 16 + (j >> 2))[j & 3] =
          std::uint8_t(std::int32_t(h));
      reinterpret_cast<std::uint8_t*>(base + lane_lo * kBWords + 16 + (j >> 2))[j & 3] =
          std::uint8_t(std::int32_t(l));
    }
  }
  __syncthreads();

  // ---- main loop ------------------------------------------------------------
  const std::uint32_t lanebase = std::uint32_t(lane) * 4u;
  const std::uint32_t lanebase8 = 128u + std::uint32_t(lane & 15) * 8u;
  int acc0[4] = {0, 0, 0, 0};
  int acc1[4] = {0, 0, 0, 0};
  std::uint32_t cur_rt = 0xFFFFFFFFu;
  const int g = lane >> 2, tq = lane & 3;

  auto flush = [&](std::uint32_t rt) {
    if (rt == 0xFFFFFFFFu || tq >= a.batch) return;
    const std::uint32_t r0 = rt * 16 + g;
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const int* acc = s == 0 ? acc0 : acc1;
      std::int32_t* z = a.zacc + (std::size_t(s) * 8 + 2 * tq) * a.rows_pad;
      atomicAdd(z + r0, acc[0]);
      atomicAdd(z + a.rows_pad + r0, acc[1]);
      atomicAdd(z + r0 + 8, acc[2]);
      atomicAdd(z + a.rows_pad + r0 + 8, acc[3]);
    }
  };

  for (std::uint32_t u = u0; u < u1; u += kPrefetch) {
#pragma unroll
    for (int i = 0; i < kPrefetch; ++i) {
      const std::uint32_t uu = u + i;
      if (uu >= u1) break;
      std::uint32_t rt, ks, kc;
      unit_coords(a, uu, rt, ks, kc);
      if (rt != cur_rt) {
        flush(cur_rt);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc0[q] = acc1[q] = 0;
        cur_rt = rt;
      }
      const uint4 c0 = pf0[i][0], c1 = pf0[i][1];
      uint4 d0, d1;
      uint2 e0, e1;
      if constexpr (STAGES > 1) {
        if constexpr (KIND1 == 0) {
          d0 = pf1[i][0];
          d1 = pf1[i][1];
        } else {
          e0 = pf1b[i][0];
          e1 = pf1b[i][1];
        }
      }
      // refill this slot with unit uu + kPrefetch
      const std::uint32_t un = uu + kPrefetch;
      if (un < u1) {
        const std::size_t ti = tile_index(un);
        pf0[i][0] = ldg_stream(a.tiles0 + ti);
        pf0[i][1] = ldg_stream(a.tiles0 + ti + 32);
        if constexpr (STAGES > 1) {
          if constexpr (KIND1 == 0) {
            pf1[i][0] = ldg_stream(static_cast<const uint4*>(a.tiles1) + ti);
            pf1[i][1] = ldg_stream(static_cast<const uint4*>(a.tiles1) + ti + 32);
          } else {
            pf1b[i][0] = ldg_stream2(static_cast<const uint2*>(a.tiles1) + ti);
            pf1b[i][1] = ldg_stream2(static_cast<const uint2*>(a.tiles1) + ti + 32);
          }
        }
      }
      // B fragments of this k-step
      const uint4* bp = reinterpret_cast<const uint4*>(
          bsm + (std::size_t(kc - kc_lo) * kChunk + (ks - kc * kChunk)) * 32 * kBWords + lane * kBWords);
      const uint4 b0 = bp[0], b1 = bp[1], b2 = bp[2], b3 = bp[3], b4 = bp[4];
      const std::uint32_t bw[18] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x,
                                    b2.y, b2.z, b2.w, b3.x, b3.y, b3.z, b3.w, b4.x, b4.y};
      // ---- stage 0 (E8P) ----
      {
        const std::uint32_t r00 = parity_fix(c0.z), r01 = parity_fix(c0.w);
        const std::uint32_t r10 = parity_fix(c1.z), r11 = parity_fix(c1.w);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          std::uint32_t a0, a1, a2, a3;
          e8p_operands(lut, j < 4 ? c0.x : c0.y, j < 4 ? r00 : r01, lanebase, j & 3, a0, a2);
          e8p_operands(lut, j < 4 ? c1.x : c1.y, j < 4 ? r10 : r11, lanebase, j & 3, a1, a3);
          mma_s8(acc0, a0, a1, a2, a3, bw[2 * j], bw[2 * j + 1]);
        }
        mma_s8(acc0, side_bytes(c0.z), side_bytes(c1.z), side_bytes(c0.w), side_bytes(c1.w), bw[16], bw[17]);
      }
      // ---- stage 1 ----
      if constexpr (STAGES > 1) {
        if constexpr (KIND1 == 0) {
          const std::uint32_t r00 = parity_fix(d0.z), r01 = parity_fix(d0.w);
          const std::uint32_t r10 = parity_fix(d1.z), r11 = parity_fix(d1.w);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            std::uint32_t a0, a1, a2, a3;
            e8p_operands(lut, j < 4 ? d0.x : d0.y, j < 4 ? r00 : r01, lanebase, j & 3, a0, a2);
            e8p_operands(lut, j < 4 ? d1.x : d1.y, j < 4 ? r10 : r11, lanebase, j & 3, a1, a3);
            mma_s8(acc1, a0, a1, a2, a3, bw[2 * j], bw[2 * j + 1]);
          }
          mma_s8(acc1, side_bytes(d0.z), side_bytes(d1.z), side_bytes(d0.w), side_bytes(d1.w), bw[16], bw[17]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            std::uint32_t a0, a1, a2, a3;
            e81_operands(lut, j < 4 ? e0.x : e0.y, lanebase8, j & 3, a0, a2);
            e81_operands(lut, j < 4 ? e1.x : e1.y, lanebase8, j & 3, a1, a3);
            mma_s8(acc1, a0, a1, a2, a3, bw[2 * j], bw[2 * j + 1]);
          }
        }
      }
    }
  }
  flush(cur_rt);
}

template <int S, int K>
void set_attr() {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemv_imma_kernel<S, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kLutBytes + kBBytes)),
               "imma smem attr");
  });
}

int sm_count() {
  static int v = [] {
    int d = 0, c = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, d);
    return c;
  }();
  return v;
}

}  // namespace

// ---- host: tables and tile transcoding --------------------------------------
void imma_tables(std::vector<std::uint32_t>& e8p, std::vector<std::uint32_t>& e81) {
  const E8PTable& t = e8p_table();
  e8p.assign(256, 0);
  for (int i = 0; i < 256; ++i) {
    std::uint32_t w = 0;
    for (int c = 0; c < 8; ++c) {
      std::uint32_t nib = std::uint32_t((t.doubled[i][c] - 1) / 2);  // 1,3,5 -> 0,1,2
      if (c == 0 && t.odd_parity[i]) nib |= 4u;
      w |= nib << (4 * c);
    }
    e8p[i] = w;
  }
  e81.assign(512, 0);
  const auto& d = e8_1bit_doubled();
  for (int i = 0; i < 256; ++i)
    for (int c = 0; c < 8; ++c)
      e81[2 * i + c / 4] |= (std::uint32_t(std::uint8_t(d[i][c])) << (8 * (c % 4)));
}

std::size_t imma_tile_bytes(std::uint32_t m_local, std::uint32_t n, int kind) {
  const std::size_t RT = (m_local + 15) / 16, KS = (n / 8 + 31) / 32;
  return RT * KS * 64 * (kind == 0 ? 16 : 8);
}

void imma_transcode(const std::uint16_t* codes, std::uint32_t m_local, std::uint32_t n, int kind,
                    std::uint8_t* out) {
  const std::uint32_t nb = n / 8;
  const std::uint32_t RT = (m_local + 15) / 16, KS = (nb + 31) / 32;
  const std::size_t lane_bytes = kind == 0 ? 16 : 8;
  for (std::uint32_t rt = 0; rt < RT; ++rt)
    for (std::uint32_t ks = 0; ks < KS; ++ks)
      for (int h = 0; h < 2; ++h)
        for (int lane = 0; lane < 32; ++lane) {
          const int g = lane >> 2, t = lane & 3;
          const std::uint32_t row = rt * 16 + g + 8 * h;
          std::uint16_t w[8];
          for (int j = 0; j < 8; ++j) {
            const std::uint32_t blk = ks * 32 + 4 * j + t;
            w[j] = (row < m_local && blk < nb) ? codes[std::size_t(row) * nb + blk] : 0;
          }
          std::uint8_t* o = out + ((std::size_t(rt) * KS + ks) * 64 + h * 32 + lane) * lane_bytes;
          if (kind == 0) {
            std::uint32_t r[2] = {0, 0};
            for (int j = 0; j < 8; ++j) {
              o[j] = std::uint8_t(w[j] >> 8);
              const int jj = j & 3;
              std::uint32_t& R = r[j >> 2];
              R |= std::uint32_t(w[j] & 1u) << jj;                      // slot (0, j'): shift bit
              for (int c = 1; c < 8; ++c) R |= std::uint32_t((w[j] >> (8 - c)) & 1u) << (4 * c + jj);
            }
            std::memcpy(o + 8, r, 8);
          } else {
            for (int j = 0; j < 8; ++j) o[j] = std::uint8_t(w[j]);
          }
        }
}

bool imma_supported(const q8p_layer& L, int batch) {
  return batch >= 1 && batch <= 4 && L.tiles[0].tiles != nullptr && L.cb[0] == Q8P_CB_E8P_2BIT &&
         (L.num_stages == 1 || L.tiles[1].tiles != nullptr);
}

void launch_gemv_imma(const q8p_layer& L, const float* t, const float* amax, std::int32_t* zacc,
                      std::uint32_t rows_pad, int batch, cudaStream_t s) {
  ImmaArgs a{};
  a.tiles0 = static_cast<const uint4*>(L.tiles[0].tiles);
  a.tiles1 = L.num_stages > 1 ? L.tiles[1].tiles : nullptr;
  a.stages = L.num_stages;
  a.kind1 = L.num_stages > 1 ? L.cb[1] : 0;
  a.n = L.n;
  a.nb = L.n / 8;
  a.RT = (L.m_local() + 15) / 16;
  a.KS = (a.nb + 31) / 32;
  a.NKC = (a.KS + kChunk - 1) / kChunk;
  a.KL = a.KS - (a.NKC - 1) * kChunk;
  a.units = a.RT * a.KS;
  a.t = t;
  a.amax = amax;
  a.batch = batch;
  a.zacc = zacc;
  a.rows_pad = rows_pad;
  a.lut_e8p = L.lut_e8p;
  a.lut_e81 = L.lut_e81;
  // Grid: one CTA per SM, but never so few that a CTA's unit range (<= ceil(units/grid) + 1)
  // exceeds one full chunk of units, so it touches at most kMaxChunks B chunks.
  std::uint32_t grid = std::uint32_t(sm_count());
  const std::uint32_t chunk_units = kChunk * a.RT;
  while ((a.units + grid - 1) / grid + 1 > chunk_units) ++grid;
  const std::size_t smem = kLutBytes + kBBytes;
  if (L.num_stages == 1) {
    set_attr<1, 0>();
    gemv_imma_kernel<1, 0><<<grid, kThreads, smem, s>>>(a);
  } else if (a.kind1 == 0) {
    set_attr<2, 0>();
    gemv_imma_kernel<2, 0><<<grid, kThreads, smem, s>>>(a);
  } else {
    set_attr<2, 1>();
    gemv_imma_kernel<2, 1><<<grid, kThreads, smem, s>>>(a);
  }
  cuda_check(cudaGetLastError(), "gemv_imma launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
