// K2 (decode batches 1..8): E8P / RVQ decode fused into the GEMV on warp-level
// tensor-core MMAs (mma.sync m16n8k32 s8 -> s32), every warp independent.
//
// Semantics: z[r] = sum_s scale_s * sum_k <decode_s(codes[s][r][k]), t[8k:8k+8]>
// (core/src/pipeline.cpp:172-191) with decode = e8p_decode (core/src/e8p.cpp:81-100)
// or the e8-1bit table (core/src/codebook.cpp:65-72).  The integer algebra is the
// one of gemv_tc.cu (K1's 25-bit activations Lt in 4 int8 limbs, alpha, TL):
//     Z = sum (sigma d) Lt + sum_k b_k S_k          (E8P stage)
//     Z = sum doubled Lt                            (e8-1bit stage)
// accumulated exactly in int32 and combined by K3 -- same accumulators, same
// K1 and K3, so this kernel and the tcgen05 kernel are interchangeable bit for bit.
//
// Why warp-level MMAs at batch <= 8: the decode (PRMT LUT address, LDS of the
// lane-replicated magnitude LUT, sign-flag LOP3, two PRMT from the byte table
// {1,3,5,_,-1,-3,-5,_}) is ~7 instructions per 8-weight codeword; the tensor core
// does every multiply-add from registers and no warp hands anything to another:
// a producer warp streams whole cells (8 row pairs' code records + the k step's
// activation B image, one contiguous byte range per stage) into a ring of shared
// memory slots with 1-D bulk copies; each consumer warp loads its half-record and
// B fragments into registers, hands the slot back, decodes and issues its MMAs.
//
// Data layout ("mma records", built once at upload from the plain codes; a
// lossless re-layout).  Cell = (row pair rp: 32 rows, k step ks:
// 32 codewords); record of one stage for one cell, per lane L = 4 g + t:
//   E8P, 2176 B:  [idx   words 0..3][32 lanes][16 B]   [idx   words 4..7][32][16 B]
//                 [flags words 0..3][32][16 B]          [flags words 4..7][32][16 B]
//                 [shift word][32][4 B]
//     word w = 4 (j >> 2) + 2 h + r8, byte / flag slot jj = j & 3: codeword
//     (row 32 rp + 16 h + 8 r8 + g, block 32 ks + 4 j + t); idx byte jj = word >> 8,
//     flag bit 4 c + jj = negate coordinate c (coordinate 0's sign resolved from the
//     parity at upload, e8p.cpp:97-98); shift bit q + 8 i (q = 4 h + 2 half + r8) =
//     shift bit of codeword (row 32 rp + 16 h + 8 r8 + g, block 32 ks + 16 half + 4 t + i)
//     -- the side MMA's A fragment order.
//   e8-1bit, 1024 B: [code words 0..3][32][16 B] [code words 4..7][32][16 B].
//   Records ordered [row block rb][ks][row pair in rb] (a cell's records are one
//   contiguous byte range); rp padded to whole row blocks of 8 row pairs.
// MMA j of a cell covers blocks 4j..4j+3: thread (g, t) holds codeword 4j + t, so
// a0/a2 = coordinates 0-3 / 4-7 of row g and a1/a3 of row g + 8; the B fragment of
// the same logical K order is 8 consecutive bytes of K1's B image (no permutation
// of the activations).
//
// CTA: TEAMS x 8 consumer warps (warp = row pair rp of the cell) + 1 producer warp;
// persistent over a contiguous range of cells (row-block-major), team t taking
// every TEAMS-th cell; per-row-block int32 accumulators flushed with integer atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "device.hpp"
#include "tc05.hpp"

namespace q8p::detail {
namespace {
using namespace tc05;

constexpr int kRowPairs = 8;                     // row pairs (32 rows) per cell
constexpr std::uint32_t kRecE8p = 2176, kRecE81 = 1024;
constexpr std::uint32_t kMaxSlots = 16;
constexpr std::uint32_t kCtl = 1024;             // barriers at the dynamic smem base
constexpr std::size_t kSmem = 227 * 1024;        // cell ring around a 64 KiB-aligned LUT window

struct MmaArgs {
  const std::uint8_t* codes[2];
  int kind1;                  // stage-1 codebook (0 e8p, 1 e8-1bit)
  std::uint32_t KSL;          // k steps
  std::uint32_t cells;        // row blocks x KSL
  const std::uint8_t* bimg;   // [KSL][b_bytes] (K1)
  std::uint32_t b_bytes;      // 9 * N * 32
  std::int32_t* zacc;         // [stage][N][rows_pad]
  std::uint32_t rows_pad, m_local;
  int ncols;                  // 4 * batch
  std::uint32_t smem_bytes;
  const std::uint32_t* nib;   // [256] E8P magnitude nibble words
  const uint2* e81;           // [256] e8-1bit doubled rows
  unsigned long long* trace;  // debug (Q8P_TRACE): per CTA globaltimer stamps, nullptr = off
};

__device__ __forceinline__ void gstamp(const MmaArgs& a, int ev) {
  if (a.trace != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[blockIdx.x * 4 + ev] = t;
  }
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ std::uint32_t ldg_stream32(const void* p) {
  std::uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];\n" : "=r"(r) : "l"(p));
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
// LUT reads: the window is constant after the fill, so these may be scheduled freely.
__device__ __forceinline__ std::uint32_t lut32(std::uint32_t addr) {
  std::uint32_t r;
  asm("ld.shared.u32 %0, [%1];\n" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint2 lut64(std::uint32_t addr) {
  uint2 r;
  asm("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(r.x), "=r"(r.y) : "r"(addr));
  return r;
}
__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t sel) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ void mma(int (&d)[4], std::uint32_t a0, std::uint32_t a1, std::uint32_t a2, std::uint32_t a3,
                                    std::uint32_t b0, std::uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

constexpr std::uint32_t kCtLo = 0x00050301u;  // {+1,+3,+5,0}
constexpr std::uint32_t kCtHi = 0x00FBFDFFu;  // {-1,-3,-5,0}

// A bytes (coordinates 0-3, 4-7) of E8P codeword slot jj of an idx / flag word pair.
template <int JJ>
__device__ __forceinline__ void e8p_a(std::uint32_t iw, std::uint32_t fw, std::uint32_t lb, std::uint32_t ct_lo,
                                      std::uint32_t ct_hi, std::uint32_t& lo, std::uint32_t& hi) {
  // Pipe balance (measured, tools/ubench_alu.cu): PRMT / LOP3 / SHF issue to the
  // ALU pipe at 16 lanes/clk, IMAD at 16, IMAD.HI (mul.hi) at only 8 lanes/clk.
  const std::uint32_t addr = prmt(iw, lb, 0x7604u | (std::uint32_t(JJ) << 4));
  const std::uint32_t nib = lut32(addr);
  std::uint32_t rs;
  if constexpr (JJ == 0)
    rs = fw << 2;
  else if constexpr (JJ == 1)
    rs = fw << 1;
  else if constexpr (JJ == 2)
    rs = fw;
  else
    rs = __umulhi(fw, 0x80000000u);  // fw >> 1 on the FMA pipe
  const std::uint32_t sel = nib ^ (rs & 0x44444444u);
  lo = prmt(ct_lo, ct_hi, sel);
  // sel >> 16: on the ALU (SHF) for even slots, on the FMA pipe (mul.hi) for odd ones
  hi = prmt(ct_lo, ct_hi, (JJ & 1) ? __umulhi(sel, 65536u) : sel >> 16);
}
template <int JJ>
__device__ __forceinline__ uint2 e81_a(std::uint32_t cw, std::uint32_t lb8) {
  return lut64(prmt(cw, lb8, 0x7604u | (std::uint32_t(JJ) << 4)));
}

__device__ __forceinline__ std::uint32_t w4(const uint4& v, int k) {
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}
__device__ __forceinline__ uint4 lds128(std::uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}

// One warp's half (H = 0: MMAs 0..3, H = 1: MMAs 4..7) of an E8P record, from smem.
struct HalfE8p {
  uint4 iw, fw;
  std::uint32_t sw;
};
// Main MMAs 4H..4H+3 of an E8P half-record into acc[h][nb] (B fragments bf[j][nb]).
template <int NB8>
__device__ __forceinline__ void e8p_half(const HalfE8p& r, const uint2 (&bf)[4][NB8], std::uint32_t lb,
                                         std::uint32_t ct_lo, std::uint32_t ct_hi, int (&acc)[2][NB8][4]) {
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      // word 2 h + r8 of the half: codeword (row 16 h + 8 r8 + g, block 4 (4H + jj) + t)
      const std::uint32_t iw0 = w4(r.iw, 2 * h), iw1 = w4(r.iw, 2 * h + 1);
      const std::uint32_t fw0 = w4(r.fw, 2 * h), fw1 = w4(r.fw, 2 * h + 1);
      std::uint32_t a0, a1, a2, a3;
      switch (jj) {
        case 0: e8p_a<0>(iw0, fw0, lb, ct_lo, ct_hi, a0, a2); e8p_a<0>(iw1, fw1, lb, ct_lo, ct_hi, a1, a3); break;
        case 1: e8p_a<1>(iw0, fw0, lb, ct_lo, ct_hi, a0, a2); e8p_a<1>(iw1, fw1, lb, ct_lo, ct_hi, a1, a3); break;
        case 2: e8p_a<2>(iw0, fw0, lb, ct_lo, ct_hi, a0, a2); e8p_a<2>(iw1, fw1, lb, ct_lo, ct_hi, a1, a3); break;
        default: e8p_a<3>(iw0, fw0, lb, ct_lo, ct_hi, a0, a2); e8p_a<3>(iw1, fw1, lb, ct_lo, ct_hi, a1, a3); break;
      }
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb) mma(acc[h][nb], a0, a1, a2, a3, bf[jj][nb].x, bf[jj][nb].y);
    }
  }
}
template <int NB8>
__device__ __forceinline__ void e81_half(const uint4& cw, const uint2 (&bf)[4][NB8], std::uint32_t lb8,
                                         int (&acc)[2][NB8][4]) {
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const std::uint32_t c0 = w4(cw, 2 * h), c1 = w4(cw, 2 * h + 1);
      uint2 v0, v1;
      switch (jj) {
        case 0: v0 = e81_a<0>(c0, lb8); v1 = e81_a<0>(c1, lb8); break;
        case 1: v0 = e81_a<1>(c0, lb8); v1 = e81_a<1>(c1, lb8); break;
        case 2: v0 = e81_a<2>(c0, lb8); v1 = e81_a<2>(c1, lb8); break;
        default: v0 = e81_a<3>(c0, lb8); v1 = e81_a<3>(c1, lb8); break;
      }
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb) mma(acc[h][nb], v0.x, v1.x, v0.y, v1.y, bf[jj][nb].x, bf[jj][nb].y);
    }
  }
}
// Side MMA of row tile h (A = shift bits b_k as 0/1 bytes, B = block sums S_k).
template <int h, int NB8>
__device__ __forceinline__ void side_mma(std::uint32_t sw, const uint2 (&bs)[NB8], int (&acc)[2][NB8][4]) {
  std::uint32_t s[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int sh = 4 * h + q;
    s[q] = (sh == 0 ? sw : __umulhi(sw, 1u << (32 - sh))) & 0x01010101u;
  }
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb) mma(acc[h][nb], s[0], s[1], s[2], s[3], bs[nb].x, bs[nb].y);
}

// TEAMS teams of 8 consumer warps (warp = row pair rp of the cell) + one producer
// warp.  Team t takes the CTA's local cells t, t + TEAMS, ...
template <int TEAMS>
struct Shape {
  static constexpr int kConsumers = kRowPairs * TEAMS;
  static constexpr int kThreads = (kConsumers + 1) * 32;
};

template <int NST, int K1, int NB8, int TEAMS>
__global__ void __launch_bounds__(Shape<TEAMS>::kThreads, 1) gemv_mma_kernel(MmaArgs a) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  constexpr int kCons = Shape<TEAMS>::kConsumers;
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const std::uint32_t sbase = smem_u32(smem);
  const std::uint32_t lutw = (sbase + kCtl + 0xFFFFu) & ~0xFFFFu;  // 64 KiB-aligned LUT window
  // cell slot: [stage-0 records of the 8 row pairs][stage-1 records][B image]
  const std::uint32_t rec0 = kRowPairs * kRecE8p;
  const std::uint32_t rec1 = NST == 2 ? kRowPairs * (K1 == 0 ? kRecE8p : kRecE81) : 0u;
  const std::uint32_t cell_bytes = rec0 + rec1 + a.b_bytes;
  const std::uint32_t slot_bytes = (cell_bytes + 127) & ~127u;
  // slots below the window, then above it
  const std::uint32_t lo0 = sbase + kCtl, n_lo = lutw > lo0 ? (lutw - lo0) / slot_bytes : 0u;
  const std::uint32_t hi0 = lutw + 65536, send = sbase + std::uint32_t(a.smem_bytes);
  std::uint32_t S = n_lo + (send > hi0 ? (send - hi0) / slot_bytes : 0u);
  if (S > kMaxSlots) S = kMaxSlots;
  auto slot_addr = [&](std::uint32_t st) { return st < n_lo ? lo0 + st * slot_bytes : hi0 + (st - n_lo) * slot_bytes; };
  const std::uint32_t bar_full = sbase, bar_empty = sbase + 8 * kMaxSlots, ct_slot = sbase + 16 * kMaxSlots;

  const std::uint32_t c0 = std::uint32_t((std::uint64_t(a.cells) * blockIdx.x) / gridDim.x);
  const std::uint32_t c1 = std::uint32_t((std::uint64_t(a.cells) * (blockIdx.x + 1)) / gridDim.x);
  const std::uint32_t count = c1 - c0;
  if (threadIdx.x == 0) gstamp(a, 0);
  if (S < 2) __trap();  // host sizing bug: fail loudly

  // producer: barriers, then the first S cells' code records right away (they do
  // not depend on K1); everyone else meets the barriers after __syncthreads
  const bool producer = warp == kCons;
  if (producer && lane == 0) {
    for (std::uint32_t i = 0; i < kMaxSlots; ++i) {
      mbar_init(bar_full + 8 * i, 1);
      mbar_init(bar_empty + 8 * i, kRowPairs);
    }
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(ct_slot), "r"(kCtLo), "r"(kCtHi) : "memory");
  }
  auto issue_codes = [&](std::uint32_t i) {
    const std::uint32_t st = i % S, dst = slot_addr(st), cell = c0 + i;
    mbar_arrive_expect_tx(bar_full + 8 * st, cell_bytes);
    bulk_g2s(dst, a.codes[0] + std::size_t(cell) * rec0, rec0, bar_full + 8 * st);
    if constexpr (NST == 2) bulk_g2s(dst + rec0, a.codes[1] + std::size_t(cell) * rec1, rec1, bar_full + 8 * st);
  };
  auto issue_b = [&](std::uint32_t i) {
    const std::uint32_t st = i % S, cell = c0 + i, ks = cell % a.KSL;
    bulk_g2s(slot_addr(st) + rec0 + rec1, a.bimg + std::size_t(ks) * a.b_bytes, a.b_bytes, bar_full + 8 * st);
  };
  // the first kEarly cells' codes before the CTA barrier (they overlap the previous
  // kernel under PDL); their B images follow as soon as K1 is done, ahead of the
  // remaining prefetch (bulk copies complete in issue order)
  constexpr std::uint32_t kEarly = 2;
  if (producer && lane == 0) {
    fence_mbar_init();
    for (std::uint32_t i = 0; i < count && i < kEarly; ++i) issue_codes(i);
  }
  // LUT window (E8P nibble words per lane; e8-1bit rows per half-warp lane)
  {
    std::uint8_t* win = smem + (lutw - sbase);
    for (int x = threadIdx.x; x < 512; x += Shape<TEAMS>::kThreads) {
      const int row = x >> 1, half = x & 1;
      const std::uint32_t w = __ldg(a.nib + row);
      uint4* d = reinterpret_cast<uint4*>(win + row * 256 + half * 64);
#pragma unroll
      for (int k = 0; k < 4; ++k) d[k] = make_uint4(w, w, w, w);
      if constexpr (NST == 2 && K1 == 1) {
        const uint2 e = __ldg(a.e81 + row);
#pragma unroll
        for (int k = 0; k < 4; ++k) d[8 + k] = make_uint4(e.x, e.y, e.x, e.y);
      }
    }
  }
  __syncthreads();
  pdl_trigger();
  if (threadIdx.x == 0) gstamp(a, 1);

  if (producer) {
    // ===== producer: B images once K1 is done, then the rest of the cells =====
    if (lane == 0 && count > 0) {
      pdl_wait();
      for (std::uint32_t i = 0; i < count && i < kEarly; ++i) issue_b(i);
      for (std::uint32_t i = kEarly; i < count && i < S; ++i) {
        issue_codes(i);
        issue_b(i);
      }
      for (std::uint32_t i = S; i < count; ++i) {
        mbar_wait(bar_empty + 8 * (i % S), ((i / S) - 1) & 1);
        issue_codes(i);
        issue_b(i);
      }
    }
    return;
  }

  // ===== consumers: warp = (team, row pair rp) =====
  const int team = warp / kRowPairs, rp = warp % kRowPairs;
  const int g = lane >> 2, t = lane & 3;
  const std::uint32_t lb0 = (lutw & 0xFFFF0000u) | (std::uint32_t(lane) * 4u);
  const std::uint32_t lb80 = (lutw & 0xFFFF0000u) | (128u + std::uint32_t(lane & 15) * 8u);
  // per-lane B fragment offset (MMA j at + j * NB8 * 256, column block nb at + nb * 256)
  const std::uint32_t bmain = std::uint32_t((t >> 1) * 128 + g * 16 + (t & 1) * 8);
  const std::uint32_t bside = 8u * NB8 * 256u + std::uint32_t(g * 16 + 4 * t);
  // the byte table read back from shared memory lives in ONE register each
  const uint2 ct = lds64(ct_slot);
  const std::uint32_t ct_lo = ct.x, ct_hi = ct.y;
  std::uint32_t lb = lb0, lb8 = lb80;
  asm volatile("" : "+r"(lb), "+r"(lb8));  // LUT reads (non-volatile asm) stay after the fill barrier
  int acc[NST][2][NB8][4];
#pragma unroll
  for (int s = 0; s < NST; ++s)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[s][h][nb][q] = 0;
  bool waited = false;
  // rows of this warp's row pair in row block rb (cell = rb * KSL + ks)
  auto flush = [&](std::uint32_t rb) {
    if (!waited) {
      pdl_wait();  // K1 zeroed the accumulators
      waited = true;
    }
    const std::uint32_t row0 = (rb * kRowPairs + std::uint32_t(rp)) * 32u + std::uint32_t(g);
#pragma unroll
    for (int s = 0; s < NST; ++s)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb) {
          const int col = nb * 8 + 2 * t;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const std::uint32_t row = row0 + 16u * h + 8u * (q >> 1);
            const int c = col + (q & 1);
            if (c < a.ncols && row < a.m_local)
              atomicAdd(a.zacc + (std::size_t(s) * (NB8 * 8) + c) * a.rows_pad + row, acc[s][h][nb][q]);
            acc[s][h][nb][q] = 0;
          }
        }
  };

  // incremental cursors: slot st / phase ph of local cell i, its row block rb and k step ks
  std::uint32_t st = std::uint32_t(team) % S, ph = (std::uint32_t(team) / S) & 1;
  std::uint32_t rb = (c0 + std::uint32_t(team)) / a.KSL, ks = (c0 + std::uint32_t(team)) % a.KSL;
  for (std::uint32_t i = std::uint32_t(team); i < count; i += TEAMS) {
    const std::uint32_t sl = slot_addr(st);
    mbar_wait(bar_full + 8 * st, ph);
    if (i == 0 && threadIdx.x == 0) gstamp(a, 2);
    const bool act = (rb * kRowPairs + std::uint32_t(rp)) * 32u < a.m_local;
    // this warp's operands into registers
    HalfE8p r0, r1, q0, q1;
    uint4 e0, e1;
    uint2 bf0[4][NB8], bf1[4][NB8], bs[NB8];
    if (act) {
      const std::uint32_t ra = sl + std::uint32_t(rp) * kRecE8p + lane * 16u;
      r0.iw = lds128(ra);
      r1.iw = lds128(ra + 512);
      r0.fw = lds128(ra + 1024);
      r1.fw = lds128(ra + 1536);
      r0.sw = lds32(sl + std::uint32_t(rp) * kRecE8p + 2048u + lane * 4u);
      if constexpr (NST == 2) {
        if constexpr (K1 == 0) {
          const std::uint32_t rq = sl + rec0 + std::uint32_t(rp) * kRecE8p + lane * 16u;
          q0.iw = lds128(rq);
          q1.iw = lds128(rq + 512);
          q0.fw = lds128(rq + 1024);
          q1.fw = lds128(rq + 1536);
          q0.sw = lds32(sl + rec0 + std::uint32_t(rp) * kRecE8p + 2048u + lane * 4u);
        } else {
          const std::uint32_t re = sl + rec0 + std::uint32_t(rp) * kRecE81 + lane * 16u;
          e0 = lds128(re);
          e1 = lds128(re + 512);
        }
      }
      const std::uint32_t bbase = sl + rec0 + rec1;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb) {
          bf0[jj][nb] = lds64(bbase + jj * NB8 * 256u + nb * 256u + bmain);
          bf1[jj][nb] = lds64(bbase + (4 + jj) * NB8 * 256u + nb * 256u + bmain);
        }
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
        bs[nb] = make_uint2(lds32(bbase + bside + nb * 256u), lds32(bbase + bside + nb * 256u + 128u));
    }
    const std::uint32_t rb_now = rb, st_now = st;
    st += TEAMS;
    if (st >= S) st -= S, ph ^= 1;
    ks += TEAMS;
    while (ks >= a.KSL) ks -= a.KSL, ++rb;
    if (act) {
      e8p_half<NB8>(r0, bf0, lb, ct_lo, ct_hi, acc[0]);
      e8p_half<NB8>(r1, bf1, lb, ct_lo, ct_hi, acc[0]);
      side_mma<0, NB8>(r0.sw, bs, acc[0]);
      side_mma<1, NB8>(r0.sw, bs, acc[0]);
      if constexpr (NST == 2) {
        if constexpr (K1 == 0) {
          e8p_half<NB8>(q0, bf0, lb, ct_lo, ct_hi, acc[1]);
          e8p_half<NB8>(q1, bf1, lb, ct_lo, ct_hi, acc[1]);
          side_mma<0, NB8>(q0.sw, bs, acc[1]);
          side_mma<1, NB8>(q0.sw, bs, acc[1]);
        } else {
          e81_half<NB8>(e0, bf0, lb8, acc[1]);
          e81_half<NB8>(e1, bf1, lb8, acc[1]);
        }
      }
    }
    // the slot goes back only after the MMAs consumed every register loaded from it
    // (an arrive right after the LDS could overtake them; WAR race with the refill)
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_empty + 8 * st_now);
    if (act && (i + TEAMS >= count || rb != rb_now)) flush(rb_now);
  }
  if (threadIdx.x == 0) gstamp(a, 3);
}

template <int NST, int K1, int NB8, int TEAMS>
void launch_k(MmaArgs a, cudaStream_t s) {
  kernel_attrs(reinterpret_cast<const void*>(gemv_mma_kernel<NST, K1, NB8, TEAMS>), int(kSmem));
  const int dev = current_device();
  static int sms[64] = {};
  if (!sms[dev & 63]) cuda_check(cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev), "sm count");
  const unsigned grid = unsigned(std::min<std::uint32_t>(a.cells, std::uint32_t(sms[dev & 63])));
  a.smem_bytes = std::uint32_t(kSmem);
  launch_pdl(gemv_mma_kernel<NST, K1, NB8, TEAMS>, dim3(grid ? grid : 1), dim3(Shape<TEAMS>::kThreads), kSmem, s, a);
}

// ---- transcode: plain codes [m_local][nb] (u16 E8P / u8 e8-1bit) -> records ----
// One thread per (cell record, lane).
__global__ void __launch_bounds__(256) mma_transcode_kernel(const void* __restrict__ codes, std::uint32_t m_local,
                                                            std::uint32_t nb, std::uint32_t KSL, std::uint32_t RP,
                                                            int kind, std::uint8_t* __restrict__ out,
                                                            const std::uint8_t* __restrict__ odd) {
  const std::size_t total = std::size_t(RP) * KSL * 32;
  const std::uint32_t rec_bytes = kind == 0 ? kRecE8p : kRecE81;
  for (std::size_t x = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; x < total;
       x += std::size_t(gridDim.x) * blockDim.x) {
    const std::uint32_t lane = std::uint32_t(x & 31);
    const std::size_t rec = x >> 5;  // records ordered [row block][k step][row pair in block]
    const std::uint32_t wr = std::uint32_t(rec % kRowPairs), ks = std::uint32_t((rec / kRowPairs) % KSL),
                        rp = std::uint32_t(rec / (std::size_t(kRowPairs) * KSL)) * kRowPairs + wr;
    const std::uint32_t g = lane >> 2, t = lane & 3;
    auto word_at = [&](std::uint32_t row, std::uint32_t k) -> std::uint32_t {
      if (row >= m_local || k >= nb) return 0u;
      return kind == 0 ? static_cast<const std::uint16_t*>(codes)[std::size_t(row) * nb + k]
                       : static_cast<const std::uint8_t*>(codes)[std::size_t(row) * nb + k];
    };
    std::uint32_t iw[8] = {0, 0, 0, 0, 0, 0, 0, 0}, fw[8] = {0, 0, 0, 0, 0, 0, 0, 0}, sw = 0;
    for (std::uint32_t w = 0; w < 8; ++w) {
      const std::uint32_t half = w >> 2, h = (w >> 1) & 1, r8 = w & 1;
      const std::uint32_t row = rp * 32 + h * 16 + r8 * 8 + g;
      for (std::uint32_t jj = 0; jj < 4; ++jj) {
        const std::uint32_t j = half * 4 + jj, k = ks * 32 + 4 * j + t;
        const std::uint32_t word = word_at(row, k);
        if (kind == 0) {
          const std::uint32_t idx = word >> 8, sb = (word >> 1) & 0x7Fu;
          iw[w] |= idx << (8 * jj);
          // effective negate flags (e8p.cpp:88-98): word bit k (1..7) -> coordinate 8 - k,
          // coordinate 0 restores the row's parity
          fw[w] |= ((std::uint32_t(__popc(sb)) & 1u) ^ odd[idx]) << jj;
          for (std::uint32_t c = 1; c < 8; ++c) fw[w] |= ((word >> (8 - c)) & 1u) << (4 * c + jj);
        } else {
          iw[w] |= word << (8 * jj);
        }
      }
    }
    if (kind == 0) {
      for (std::uint32_t q = 0; q < 8; ++q) {
        const std::uint32_t h = q >> 2, half = (q >> 1) & 1, r8 = q & 1;
        const std::uint32_t row = rp * 32 + h * 16 + r8 * 8 + g;
        for (std::uint32_t i = 0; i < 4; ++i) sw |= (word_at(row, ks * 32 + half * 16 + 4 * t + i) & 1u) << (q + 8 * i);
      }
    }
    std::uint8_t* r = out + rec * rec_bytes;
    *reinterpret_cast<uint4*>(r + lane * 16) = make_uint4(iw[0], iw[1], iw[2], iw[3]);
    *reinterpret_cast<uint4*>(r + 512 + lane * 16) = make_uint4(iw[4], iw[5], iw[6], iw[7]);
    if (kind == 0) {
      *reinterpret_cast<uint4*>(r + 1024 + lane * 16) = make_uint4(fw[0], fw[1], fw[2], fw[3]);
      *reinterpret_cast<uint4*>(r + 1536 + lane * 16) = make_uint4(fw[4], fw[5], fw[6], fw[7]);
      *reinterpret_cast<std::uint32_t*>(r + 2048 + lane * 4) = sw;
    }
  }
}

}  // namespace

std::uint32_t mma_row_blocks(std::uint32_t m_local) { return (m_local + 32 * kRowPairs - 1) / (32 * kRowPairs); }
std::size_t mma_code_bytes(std::uint32_t m_local, std::uint32_t n, int kind) {
  return std::size_t(mma_row_blocks(m_local)) * kRowPairs * tc_k_slabs(n) * (kind == 0 ? kRecE8p : kRecE81);
}

void mma_transcode_device(const void* codes, std::uint32_t m_local, std::uint32_t n, int kind, std::uint8_t* out,
                          const std::uint8_t* odd_parity_dev, cudaStream_t s) {
  const std::uint32_t nb = n / 8, KSL = tc_k_slabs(n), RP = mma_row_blocks(m_local) * kRowPairs;
  const std::size_t total = std::size_t(RP) * KSL * 32;
  const unsigned grid = unsigned(std::min<std::size_t>((total + 255) / 256, 148 * 16));
  mma_transcode_kernel<<<grid, 256, 0, s>>>(codes, m_local, nb, KSL, RP, kind, out, odd_parity_dev);
  cuda_check(cudaGetLastError(), "mma transcode launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// [256] E8P magnitude nibbles (d = 1,3,5 -> 0,1,2 at bits 4c), then [256][2] words of
// the e8-1bit doubled rows (8 x s8).
std::vector<std::uint32_t> mma_table_words() {
  const E8PTable& t = e8p_table();
  const auto& d = e8_1bit_doubled();
  std::vector<std::uint32_t> w(256 * 3, 0);
  for (int i = 0; i < 256; ++i) {
    for (int c = 0; c < 8; ++c) w[i] |= std::uint32_t((t.doubled[i][c] - 1) / 2) << (4 * c);
    for (int c = 0; c < 8; ++c) w[256 + 2 * i + c / 4] |= std::uint32_t(std::uint8_t(d[i][c])) << (8 * (c % 4));
  }
  return w;
}

bool mma_supported(const q8p_layer& L, int batch) {
  return batch >= 1 && batch <= kMmaMaxBatch && L.mma[0] != nullptr && L.cb[0] == Q8P_CB_E8P_2BIT &&
         (L.num_stages == 1 || L.mma[1] != nullptr) && L.mma_tables != nullptr;
}

void launch_gemv_mma(const q8p_layer& L, const std::uint8_t* bimg, std::int32_t* zacc, std::uint32_t rows_pad,
                     int batch, cudaStream_t s) {
  MmaArgs a{};
  a.codes[0] = static_cast<const std::uint8_t*>(L.mma[0]);
  a.codes[1] = static_cast<const std::uint8_t*>(L.mma[1]);
  a.kind1 = L.num_stages == 2 && L.cb[1] == Q8P_CB_E8_1BIT ? 1 : 0;
  const int N = tc_ncols_pad(4 * batch);
  a.KSL = tc_k_slabs(L.n);
  a.cells = mma_row_blocks(L.m_local()) * a.KSL;
  a.bimg = bimg;
  a.b_bytes = 9u * std::uint32_t(N) * 32u;
  a.zacc = zacc;
  a.rows_pad = rows_pad;
  a.m_local = L.m_local();
  a.ncols = 4 * batch;
  a.nib = L.mma_tables;
  a.e81 = reinterpret_cast<const uint2*>(L.mma_tables + 256);
  static const char* trace_env = std::getenv("Q8P_TRACE");  // debug: per-CTA timeline file
  unsigned long long* tr = nullptr;
  if (trace_env != nullptr) {
    cuda_check(cudaMalloc(&tr, 4096 * 8), "trace alloc");
    cuda_check(cudaMemset(tr, 0, 4096 * 8), "trace memset");
  }
  a.trace = tr;
  const int nst = L.num_stages;
#define Q8P_LAUNCH(NB8)                                     \
  if (nst == 1)                                             \
    launch_k<1, 0, NB8, NB8 == 1 ? 3 : 2>(a, s);            \
  else if (a.kind1 == 0)                                    \
    launch_k<2, 0, NB8, 2>(a, s);                           \
  else                                                      \
    launch_k<2, 1, NB8, 2>(a, s);
  switch (N) {
    case 8: Q8P_LAUNCH(1) break;
    case 16: Q8P_LAUNCH(2) break;
    default: Q8P_LAUNCH(4) break;
  }
#undef Q8P_LAUNCH
  cuda_check(cudaGetLastError(), "gemv_mma launch");
  if (tr != nullptr) {
    std::vector<unsigned long long> h(4096);
    cuda_check(cudaStreamSynchronize(s), "trace sync");
    cuda_check(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost), "trace copy");
    cudaFree(tr);
    static int seq = 0;
    const std::string path = std::string(trace_env) + ".mma." + std::to_string(seq++) + "." +
                             std::to_string(L.m_local()) + "x" + std::to_string(L.n) + ".bin";
    if (FILE* f = std::fopen(path.c_str(), "wb")) {
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
