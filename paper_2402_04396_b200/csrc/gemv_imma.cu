// K2: E8P / RVQ decode fused into a batch-1..4 GEMV on the tensor cores.
//
// Semantics: z[r] = sum_s scale_s * sum_k <decode_s(codes[s][r][k]), t[8k:8k+8]>
// (core/src/pipeline.cpp:172-191) with decode = e8p_decode
// (core/src/e8p.cpp:81-100) or the e8-1bit table (core/src/codebook.cpp:65-72).
//
// Why tensor cores for a GEMV: at 2 bits/weight B200 HBM delivers ~11.6
// codewords per SM-clock, leaving ~11 issue slots per 8-weight codeword (and
// the ALU pipe half of that).  The decode is therefore reshaped so the tensor
// core does every multiply-add and the ALU only builds int8 operand bytes:
//
//   v_c = sigma_c d_c / 2 + s / 4       (d in {1,3,5}, s = 2b - 1 shift)
//   z   = 1/2 [ sum_c (sigma_c d_c) t_c + sum_k b_k T_k ] - 1/4 T
//         (T_k = block sum of t, T = sum of t, computed exactly in K1)
//
// A operand (s8) = sigma_c d_c: one byte-permute per 4 coordinates from the
// constant table {1,3,5,_,-1,-3,-5,_}; the selector nibbles are (magnitude
// index from a per-lane-replicated smem LUT) XOR (negate flags moved into
// place by one shift).  The b_k term is a "side" MMA with A = b (u8) against
// B = block sums.  Activations are L int8 limbs (L = 3 for batch <= 2, 2 for
// batch 3..4): t = alpha (sum_l 128^(L-1-l) limb_l), |err| <= alpha/2,
// alpha = max|t| / (127 * 128^(L-1)), carried as MMA columns, so the
// int32 accumulation is exact and split-K partials combine with integer
// atomics (deterministic).
//
// Device tile format (built once at upload; a lossless re-layout of the QSHP
// codes), 17 bits per codeword:
//   tile (row tile rt = 16 rows, k-step ks = 32 codewords = 256 columns):
//   codes  [rt][ks][half h][lane = 4 g + t][16 B]: the 8 codewords of row
//          16 rt + g + 8 h at blocks 32 ks + 4 j + t, j = 0..7:
//            bytes 0..7  idx_j = word_j >> 8
//            bytes 8..15 sign registers R0 (j = 0..3), R1 (j = 4..7):
//                        bit 4 c + j' = effective negate flag of coordinate c
//                        (c = 0: the parity-inferred sign, e8p.cpp:97-98,
//                        resolved at upload time)
//   shifts [rt][ks][lane][u16]: bit 8 h + 4 (j >> 2) + (j & 3) = shift bit of
//          codeword j of half h.
// The shift plane is 1/16 of the code bytes: it lets the hot loop skip the
// per-codeword parity fold (the 16-bit E8P word stores 7 explicit signs).
// e8-1bit tiles: [rt][ks][half][lane][8 B] = the 8 code bytes; A = LUT row.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "device.hpp"

// Experiment hooks (scratch/gemv_exp.cu); 0 in the product build.
#ifndef Q8P_EXP_MODE
#define Q8P_EXP_MODE 0
#endif

namespace q8p::detail {
namespace {

constexpr int kChunk = 8;        // k-steps per B chunk
constexpr int kMaxChunks = 2;    // B chunks resident per CTA
constexpr int kBWords = 20;      // u32 per (k-step, lane) in the B smem image (18 used)
constexpr std::size_t kBBytes = std::size_t(kMaxChunks) * kChunk * 32 * kBWords * 4;  // 40 KiB
constexpr int kMaxUnits = 40;    // per-warp unit list capacity (host sizes the grid to fit)
constexpr std::size_t kListBytes = 32 * kMaxUnits * 16;  // 20 KiB (32 warps)
constexpr std::size_t kSmemBytes = 128 * 1024 + 1024;  // 64-KiB-aligned LUT window + B images + lists
static_assert(kBBytes + kListBytes <= 63 * 1024, "B images + unit lists must fit below the LUT window");
__host__ __device__ constexpr float limb_max(int L) { return L == 3 ? 2080768.f : 16256.f; }  // 127*128^(L-1)

template <int STAGES>
struct Cfg {
  static constexpr int kWarps = STAGES == 1 ? 32 : 16;
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kPrefetch = 2;
};

struct ImmaArgs {
  const uint4* tiles0;             // stage 0 (always e8p-2bit)
  const std::uint16_t* shifts0;
  const void* tiles1;              // stage 1: e8p-2bit (uint4 lanes) or e8-1bit (uint2 lanes)
  const std::uint16_t* shifts1;
  int kind1;                       // stage 1 codebook: 0 = e8p, 1 = e8-1bit
  std::uint32_t RT, KS, NKC, KL;   // row tiles, k-steps, chunks, k-steps in last chunk
  std::uint32_t nb, n;
  std::uint32_t units;
  const float* t;                  // [batch][n]
  const float* amax;               // [batch]
  int batch;                       // 1..4
  int limbs;                       // 3 (batch <= 2) or 2
  std::int32_t* zacc;              // [stage][8][rows_pad]
  std::uint32_t rows_pad;
  const std::uint32_t* lut_e8p;    // [256]: nibble c = delta_c (0, 1, 2 for d = 1, 3, 5)
  const std::uint32_t* lut_e81;    // [256][2]: doubled coordinates as s8
};

__device__ __forceinline__ void mma_s8(int (&d)[4], std::uint32_t a0, std::uint32_t a1, std::uint32_t a2,
                                       std::uint32_t a3, std::uint32_t b0, std::uint32_t b1) {
  if (Q8P_EXP_MODE == 3 || Q8P_EXP_MODE == 5) {
    d[0] ^= a0 ^ b0; d[1] ^= a1 ^ b1; d[2] ^= a2; d[3] ^= a3;
    return;
  }
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_u8s8(int (&d)[4], std::uint32_t a0, std::uint32_t a1, std::uint32_t a2,
                                         std::uint32_t a3, std::uint32_t b0, std::uint32_t b1) {
  if (Q8P_EXP_MODE == 3 || Q8P_EXP_MODE == 5) {
    d[0] ^= a0 ^ b0; d[1] ^= a1 ^ b1; d[2] ^= a2; d[3] ^= a3;
    return;
  }
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
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
__device__ __forceinline__ std::uint32_t ldg_u16(const std::uint16_t* p) {
  std::uint16_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];\n" : "=h"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ std::uint32_t lds32(std::uint32_t addr) {
  std::uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint2 lds64(std::uint32_t addr) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(r.x), "=r"(r.y) : "r"(addr));
  return r;
}
// Raw PTX prmt (default mode): __byte_perm() masks the selector with 0x7777
// first, an extra LOP3 we do not need -- our selectors never set bit 3.
__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t sel) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
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

// Incremental walk over units in (chunk, row tile, k-step) order.
struct Cursor {
  std::uint32_t kc, rt, ksl, size;
  __device__ __forceinline__ void init(const ImmaArgs& a, std::uint32_t u) {
    std::uint32_t ks;
    unit_coords(a, u, rt, ks, kc);
    ksl = ks - kc * kChunk;
    size = (kc == a.NKC - 1) ? a.KL : kChunk;
  }
  __device__ __forceinline__ void next(const ImmaArgs& a) {
    if (++ksl == size) {
      ksl = 0;
      if (++rt == a.RT) {
        rt = 0;
        ++kc;
        size = (kc == a.NKC - 1) ? a.KL : kChunk;
      }
    }
  }
  __device__ __forceinline__ std::uint32_t tile(const ImmaArgs& a) const {
    return rt * a.KS + kc * kChunk + ksl;
  }
};

constexpr std::uint32_t kCtLo = 0x00050301u;  // {+1,+3,+5,0}
constexpr std::uint32_t kCtHi = 0x00FBFDFFu;  // {-1,-3,-5,0}

// A bytes of codeword jj (0..3) of an E8P register group.  `lb` = LUT window
// address bytes 2..3 | lane * 4 in byte 0; PRMT drops idx into byte 1, giving
// the shared-window address of this lane's LUT replica directly.
__device__ __forceinline__ void e8p_operands(std::uint32_t idxreg, std::uint32_t r, std::uint32_t lb, int jj,
                                             std::uint32_t& alo, std::uint32_t& ahi) {
  if (Q8P_EXP_MODE == 2 || Q8P_EXP_MODE == 5) {
    alo = idxreg + jj;
    ahi = r;
    return;
  }
  const std::uint32_t nib = lds32(prmt(idxreg, lb, 0x7604u | (std::uint32_t(jj) << 4)));
  std::uint32_t rs;
  if (jj == 0)
    rs = r * 4u;
  else if (jj == 1)
    rs = r * 2u;
  else if (jj == 2)
    rs = r;
  else
    rs = __umulhi(r, 0x80000000u);  // >> 1
  const std::uint32_t sel = nib ^ (rs & 0x44444444u);
  alo = prmt(kCtLo, kCtHi, sel);
  ahi = prmt(kCtLo, kCtHi, __umulhi(sel, 65536u));  // sel >> 16
}

__device__ __forceinline__ void e81_operands(std::uint32_t codereg, std::uint32_t lb8, int jj, std::uint32_t& alo,
                                             std::uint32_t& ahi) {
  const uint2 v = lds64(prmt(codereg, lb8, 0x7604u | (std::uint32_t(jj) << 4)));
  alo = v.x;
  ahi = v.y;
}

// Side-MMA A operands from the u16 shift word: byte j' = 8 b, matching the B
// side images (T_k / 8).
__device__ __forceinline__ void side_operands(std::uint32_t s, std::uint32_t& a0, std::uint32_t& a1,
                                              std::uint32_t& a2, std::uint32_t& a3) {
  // nibble q of s (bits 4q..4q+3) -> byte j' bit 3 (value 8 b) via one multiply
  a0 = ((s & 0xFu) * 0x01020408u) & 0x08080808u;                   // half 0, j 0..3
  a2 = ((__umulhi(s, 1u << 28) & 0xFu) * 0x01020408u) & 0x08080808u;  // half 0, j 4..7
  a1 = ((__umulhi(s, 1u << 24) & 0xFu) * 0x01020408u) & 0x08080808u;  // half 1, j 0..3
  a3 = ((__umulhi(s, 1u << 20) & 0xFu) * 0x01020408u) & 0x08080808u;  // half 1, j 4..7
}

template <int STAGES, int KIND1>
__global__ void __launch_bounds__(Cfg<STAGES>::kThreads, 1) gemv_imma_kernel(ImmaArgs a) {
  constexpr int kWarps = Cfg<STAGES>::kWarps, kThreads = Cfg<STAGES>::kThreads;
  constexpr int kPrefetch = Cfg<STAGES>::kPrefetch;
  extern __shared__ __align__(16) char smem[];
  // LUT at the first 64-KiB-aligned shared-window address inside the
  // allocation, so PRMT can compose complete LDS addresses.
  const std::uint32_t sbase = static_cast<std::uint32_t>(__cvta_generic_to_shared(smem));
  const std::uint32_t lutw = (sbase + 0xFFFFu) & ~0xFFFFu;
  char* lut = smem + (lutw - sbase);
  std::uint32_t* bsm =
      reinterpret_cast<std::uint32_t*>(lutw - sbase >= kBBytes + kListBytes ? smem : lut + 65536);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint32_t W = gridDim.x * kWarps;
  const std::uint32_t gw = blockIdx.x * kWarps + warp;
  const std::uint32_t u0 = std::uint32_t((std::uint64_t(a.units) * gw) / W);
  const std::uint32_t u1 = std::uint32_t((std::uint64_t(a.units) * (gw + 1)) / W);
  const std::uint32_t cu0 = std::uint32_t((std::uint64_t(a.units) * (blockIdx.x * kWarps)) / W);
  const std::uint32_t cu1 = std::uint32_t((std::uint64_t(a.units) * ((blockIdx.x + 1) * kWarps)) / W);

  // ---- per-warp unit lists (tile index, B-image offset, row tile) ---------
  // Built once by lane 0 of each warp; the main loop then reads one broadcast
  // 16-B entry per unit instead of walking a cursor (keeps the loop branch-light).
  std::uint32_t rt_, ks_, kc_lo, kc_hi;
  unit_coords(a, cu0, rt_, ks_, kc_lo);
  unit_coords(a, cu1 > cu0 ? cu1 - 1 : cu0, rt_, ks_, kc_hi);
  const std::uint32_t nchunk = kc_hi - kc_lo + 1;  // <= kMaxChunks (host guarantees)
  uint4* lists = reinterpret_cast<uint4*>(bsm + kBBytes / 4);
  uint4* list = lists + warp * kMaxUnits;
  const int nu = int(u1 - u0);  // <= kMaxUnits (host guarantees)
  if (lane == 0 && nu > 0) {
    Cursor c;
    c.init(a, u0);
    for (int i = 0; i < nu; ++i) {
      list[i] = make_uint4(c.tile(a), ((c.kc - kc_lo) * kChunk + c.ksl) * 32 * kBWords, c.rt, 0);
      c.next(a);
    }
  }
  __syncwarp();

  // ---- prefetch the first code units (overlaps the prologue) -------------
  uint4 pc0[kPrefetch][2];
  std::uint32_t ps0[kPrefetch];
  uint4 pc1[STAGES > 1 && KIND1 == 0 ? kPrefetch : 1][2];
  uint2 pe1[STAGES > 1 && KIND1 == 1 ? kPrefetch : 1][2];
  std::uint32_t ps1[STAGES > 1 && KIND1 == 0 ? kPrefetch : 1];
  auto load_unit = [&](int i, std::uint32_t tile) {
    const std::size_t ti = std::size_t(tile) * 64 + lane;
    pc0[i][0] = ldg_stream(a.tiles0 + ti);
    pc0[i][1] = ldg_stream(a.tiles0 + ti + 32);
    ps0[i] = ldg_u16(a.shifts0 + std::size_t(tile) * 32 + lane);
    if constexpr (STAGES > 1) {
      if constexpr (KIND1 == 0) {
        pc1[i][0] = ldg_stream(static_cast<const uint4*>(a.tiles1) + ti);
        pc1[i][1] = ldg_stream(static_cast<const uint4*>(a.tiles1) + ti + 32);
        ps1[i] = ldg_u16(a.shifts1 + std::size_t(tile) * 32 + lane);
      } else {
        pe1[i][0] = ldg_stream2(static_cast<const uint2*>(a.tiles1) + ti);
        pe1[i][1] = ldg_stream2(static_cast<const uint2*>(a.tiles1) + ti + 32);
      }
    }
  };
  if (nu > 0) {
#pragma unroll
    for (int i = 0; i < kPrefetch; ++i) load_unit(i, list[i < nu ? i : nu - 1].x);
  }

  // ---- LUTs: E8P nibbles replicated per lane (bytes [0,128) of each 256-B row),
  //      e8-1bit rows replicated per half-warp lane (bytes [128,256)) ---------
  if (Q8P_EXP_MODE != 1) {
    for (std::uint32_t row = threadIdx.x >> 1; row < 256; row += kThreads >> 1) {
      const std::uint32_t half = threadIdx.x & 1;
      const std::uint32_t v = a.lut_e8p[row];
      uint4* dst = reinterpret_cast<uint4*>(lut + row * 256 + half * 64);
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[k] = make_uint4(v, v, v, v);
      if constexpr (STAGES > 1 && KIND1 == 1) {
        const uint2 w = make_uint2(a.lut_e81[2 * row], a.lut_e81[2 * row + 1]);
        uint4* d2 = reinterpret_cast<uint4*>(lut + row * 256 + 128 + half * 64);
#pragma unroll
        for (int k = 0; k < 4; ++k) d2[k] = make_uint4(w.x, w.y, w.x, w.y);
      }
    }
  }

  // ---- B images for the CTA's k-chunks ------------------------------------
  for (std::uint32_t i = threadIdx.x; i < nchunk * kChunk * 32 * kBWords / 4; i += kThreads)
    reinterpret_cast<uint4*>(bsm)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // Everything above (LUT, weight prefetch) is independent of K1; t and amax are not.
  pdl_wait();
  pdl_trigger();
  if (Q8P_EXP_MODE != 1) {
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
      const float am = a.amax[b];
      const float inv = am > 0.f ? limb_max(a.limbs) / am : 0.f;
      if (blk < a.nb) {
        const float4* tp = reinterpret_cast<const float4*>(a.t + std::size_t(b) * a.n + 8 * blk);
        const float4 lo4 = tp[0], hi4 = tp[1];
        v[0] = lo4.x, v[1] = lo4.y, v[2] = lo4.z, v[3] = lo4.w, v[4] = hi4.x, v[5] = hi4.y, v[6] = hi4.z,
        v[7] = hi4.w;
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = 0.f;
      }
      const int L = a.limbs;
      float sum = 0.f;
      std::uint32_t lw[3][2] = {{0, 0}, {0, 0}, {0, 0}};
      auto split = [&](float v, std::int32_t (&out)[3]) {  // v in [-limb_max, limb_max]
        if (L == 3) {
          const float h = rintf(v * (1.f / 16384.f));
          const float r = v - 16384.f * h;
          const float m = rintf(r * (1.f / 128.f));
          out[0] = std::int32_t(h);
          out[1] = std::int32_t(m);
          out[2] = std::int32_t(rintf(r - 128.f * m));
        } else {
          const float h = rintf(v * (1.f / 128.f));
          out[0] = std::int32_t(h);
          out[1] = std::int32_t(rintf(v - 128.f * h));
          out[2] = 0;
        }
      };
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        sum += v[c];
        std::int32_t l3[3];
        split(v[c] * inv, l3);
#pragma unroll
        for (int l = 0; l < 3; ++l) lw[l][c >> 2] |= (std::uint32_t(l3[l]) & 0xFFu) << (8 * (c & 3));
      }
      // block sum in the side operand's units (A_side = 8 b)
      std::int32_t sl[3];
      split(sum * 0.125f * inv, sl);
      std::uint32_t* base = bsm + (std::size_t(ch) * kChunk + ksl) * 32 * kBWords;
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        if (l >= L) break;
        const std::uint32_t ln = (L * b + l) * 4 + tt;  // B column L*b + l  <->  lane group g
        base[ln * kBWords + 2 * j] = lw[l][0];
        base[ln * kBWords + 2 * j + 1] = lw[l][1];
        reinterpret_cast<std::uint8_t*>(base + ln * kBWords + 16 + (j >> 2))[j & 3] = std::uint8_t(sl[l]);
      }
    }
  }
  __syncthreads();

  // ---- main loop ------------------------------------------------------------
  const std::uint32_t lb = (lutw & 0xFFFF0000u) | (std::uint32_t(lane) * 4u);
  const std::uint32_t lb8 = (lutw & 0xFFFF0000u) | (128u + std::uint32_t(lane & 15) * 8u);
  int acc0[4] = {0, 0, 0, 0};
  int acc1[4] = {0, 0, 0, 0};
  const int g = lane >> 2, tq = lane & 3;
  const int ncols = a.limbs * a.batch;  // used B/C columns
  const bool w0 = 2 * tq < ncols, w1 = 2 * tq + 1 < ncols;
  std::int32_t* zrow = a.zacc + std::size_t(2 * tq) * a.rows_pad + g;

  auto flush = [&](std::uint32_t rt) {
    if (Q8P_EXP_MODE == 4 && acc0[0] != 12345) return;
    std::int32_t* z = zrow + rt * 16;  // column 2 tq, row 16 rt + g
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const int* acc = s == 0 ? acc0 : acc1;
      std::int32_t* zs = z + std::size_t(s) * 8 * a.rows_pad;
      if (w0) {
        atomicAdd(zs, acc[0]);
        atomicAdd(zs + 8, acc[2]);
      }
      if (w1) {
        atomicAdd(zs + a.rows_pad, acc[1]);
        atomicAdd(zs + a.rows_pad + 8, acc[3]);
      }
    }
  };

  auto e8p_unit = [&](int (&acc)[4], const uint4& c0, const uint4& c1, std::uint32_t s, const std::uint32_t* bw) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      std::uint32_t a0, a1, a2, a3;
      e8p_operands(j < 4 ? c0.x : c0.y, j < 4 ? c0.z : c0.w, lb, j & 3, a0, a2);
      e8p_operands(j < 4 ? c1.x : c1.y, j < 4 ? c1.z : c1.w, lb, j & 3, a1, a3);
      mma_s8(acc, a0, a1, a2, a3, bw[2 * j], bw[2 * j + 1]);
    }
    std::uint32_t s0, s1, s2, s3;
    side_operands(s, s0, s1, s2, s3);
    mma_u8s8(acc, s0, s1, s2, s3, bw[16], bw[17]);
  };

  auto compute = [&](int i, std::uint32_t boff) {
    const uint4* bp = reinterpret_cast<const uint4*>(bsm + boff + lane * kBWords);
    const uint4 b0 = bp[0], b1 = bp[1], b2 = bp[2], b3 = bp[3];
    const uint2 b4 = *reinterpret_cast<const uint2*>(bp + 4);
    const std::uint32_t bw[18] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x,
                                  b2.y, b2.z, b2.w, b3.x, b3.y, b3.z, b3.w, b4.x, b4.y};
    e8p_unit(acc0, pc0[i][0], pc0[i][1], ps0[i], bw);
    if constexpr (STAGES > 1) {
      if constexpr (KIND1 == 0) {
        e8p_unit(acc1, pc1[i][0], pc1[i][1], ps1[i], bw);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          std::uint32_t a0, a1, a2, a3;
          e81_operands(j < 4 ? pe1[i][0].x : pe1[i][0].y, lb8, j & 3, a0, a2);
          e81_operands(j < 4 ? pe1[i][1].x : pe1[i][1].y, lb8, j & 3, a1, a3);
          mma_s8(acc1, a0, a1, a2, a3, bw[2 * j], bw[2 * j + 1]);
        }
      }
    }
  };

  if (nu > 0) {
    std::uint32_t cur_rt = list[0].z;
    auto step = [&](int u, int i, bool refill) {
      const uint4 e = list[u];  // uniform smem broadcast
      if (e.z != cur_rt) {
        flush(cur_rt);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc0[q] = acc1[q] = 0;
        cur_rt = e.z;
      }
      compute(i, e.y);
      if (refill) load_unit(i, list[min(u + kPrefetch, nu - 1)].x);
    };
    int u = 0;
    // steady state; refills past the end re-load the last tile (harmless)
    for (; u + kPrefetch <= nu; u += kPrefetch) {
#pragma unroll
      for (int i = 0; i < kPrefetch; ++i) step(u + i, i, true);
    }
#pragma unroll
    for (int i = 0; i < kPrefetch; ++i)
      if (u + i < nu) step(u + i, i, false);
    flush(cur_rt);
  }
}

template <int S, int K>
void set_attr() {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(gemv_imma_kernel<S, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kSmemBytes)),
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
    for (int c = 0; c < 8; ++c) w |= std::uint32_t((t.doubled[i][c] - 1) / 2) << (4 * c);  // 1,3,5 -> 0,1,2
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
std::size_t imma_shift_bytes(std::uint32_t m_local, std::uint32_t n, int kind) {
  const std::size_t RT = (m_local + 15) / 16, KS = (n / 8 + 31) / 32;
  return kind == 0 ? RT * KS * 64 : 0;
}

void imma_transcode(const std::uint16_t* codes, std::uint32_t m_local, std::uint32_t n, int kind,
                    std::uint8_t* out, std::uint8_t* shifts) {
  const E8PTable& T = e8p_table();
  const std::uint32_t nb = n / 8;
  const std::uint32_t RT = (m_local + 15) / 16, KS = (nb + 31) / 32;
  const std::size_t lane_bytes = kind == 0 ? 16 : 8;
  for (std::uint32_t rt = 0; rt < RT; ++rt)
    for (std::uint32_t ks = 0; ks < KS; ++ks) {
      const std::size_t tile = std::size_t(rt) * KS + ks;
      for (int lane = 0; lane < 32; ++lane) {
        std::uint16_t sw = 0;
        for (int h = 0; h < 2; ++h) {
          const int g = lane >> 2, t = lane & 3;
          const std::uint32_t row = rt * 16 + g + 8 * h;
          std::uint16_t w[8];
          for (int j = 0; j < 8; ++j) {
            const std::uint32_t blk = ks * 32 + 4 * j + t;
            w[j] = (row < m_local && blk < nb) ? codes[std::size_t(row) * nb + blk] : 0;
          }
          std::uint8_t* o = out + (tile * 64 + h * 32 + lane) * lane_bytes;
          if (kind == 0) {
            std::uint32_t r[2] = {0, 0};
            for (int j = 0; j < 8; ++j) {
              o[j] = std::uint8_t(w[j] >> 8);
              const unsigned idx = w[j] >> 8, sb = (w[j] >> 1) & 0x7Fu;
              // effective negate flags (e8p.cpp:88-98): word bit k (1..7) -> coordinate 8 - k,
              // coordinate 0 restores the row's parity
              unsigned neg[8];
              neg[0] = unsigned(__builtin_popcount(sb) & 1) ^ T.odd_parity[idx];
              for (int c = 1; c < 8; ++c) neg[c] = (w[j] >> (8 - c)) & 1u;
              std::uint32_t& R = r[j >> 2];
              for (int c = 0; c < 8; ++c) R |= std::uint32_t(neg[c]) << (4 * c + (j & 3));
              sw |= std::uint16_t((w[j] & 1u) << (8 * h + 4 * (j >> 2) + (j & 3)));
            }
            std::memcpy(o + 8, r, 8);
          } else {
            for (int j = 0; j < 8; ++j) o[j] = std::uint8_t(w[j]);
          }
        }
        if (kind == 0) std::memcpy(shifts + (tile * 32 + lane) * 2, &sw, 2);
      }
    }
}

int imma_limbs(int batch) { return batch <= 2 ? 3 : 2; }
float imma_limb_max(int batch) { return limb_max(imma_limbs(batch)); }

bool imma_supported(const q8p_layer& L, int batch) {
  // the float4 RHT passes need m, n multiples of 4 (every plannable dim >= 4 is)
  return batch >= 1 && batch <= 4 && L.m % 4 == 0 && L.n % 4 == 0 && L.tiles[0].tiles != nullptr &&
         L.cb[0] == Q8P_CB_E8P_2BIT && (L.num_stages == 1 || L.tiles[1].tiles != nullptr);
}

void launch_gemv_imma(const q8p_layer& L, const float* t, const float* amax, std::int32_t* zacc,
                      std::uint32_t rows_pad, int batch, cudaStream_t s) {
  ImmaArgs a{};
  a.tiles0 = static_cast<const uint4*>(L.tiles[0].tiles);
  a.shifts0 = static_cast<const std::uint16_t*>(L.tiles[0].shifts);
  a.tiles1 = L.num_stages > 1 ? L.tiles[1].tiles : nullptr;
  a.shifts1 = L.num_stages > 1 ? static_cast<const std::uint16_t*>(L.tiles[1].shifts) : nullptr;
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
  a.limbs = imma_limbs(batch);
  a.zacc = zacc;
  a.rows_pad = rows_pad;
  a.lut_e8p = L.lut_e8p;
  a.lut_e81 = L.lut_e81;
  // One CTA per SM; never so few that a CTA's unit range (<= ceil(units/grid) + 1)
  // exceeds one full chunk of units, so it touches at most kMaxChunks B chunks.
  std::uint32_t grid = std::uint32_t(sm_count());
  const std::uint32_t chunk_units = kChunk * a.RT;
  const std::uint32_t warps = L.num_stages == 1 ? Cfg<1>::kWarps : Cfg<2>::kWarps;
  while ((a.units + grid - 1) / grid + 1 > chunk_units ||
         (a.units + grid * warps - 1) / (grid * warps) + 1 > std::uint32_t(kMaxUnits))
    ++grid;
  if (L.num_stages == 1) {
    set_attr<1, 0>();
    launch_pdl(gemv_imma_kernel<1, 0>, dim3(grid), dim3(Cfg<1>::kThreads), kSmemBytes, s, a);
  } else if (a.kind1 == 0) {
    set_attr<2, 0>();
    launch_pdl(gemv_imma_kernel<2, 0>, dim3(grid), dim3(Cfg<2>::kThreads), kSmemBytes, s, a);
  } else {
    set_attr<2, 1>();
    launch_pdl(gemv_imma_kernel<2, 1>, dim3(grid), dim3(Cfg<2>::kThreads), kSmemBytes, s, a);
  }
  cuda_check(cudaGetLastError(), "gemv_imma launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
