// K2: E8P / RVQ decode fused into a small-batch GEMV on the 5th-gen tensor
// cores (tcgen05.mma kind::i8, A operand in tensor memory).
//
// Semantics: z[r] = sum_s scale_s * sum_k <decode_s(codes[s][r][k]), t[8k:8k+8]>
// (core/src/pipeline.cpp:172-191) with decode = e8p_decode
// (core/src/e8p.cpp:81-100) or the e8-1bit table (core/src/codebook.cpp:65-72).
//
// Algebra.  e8p_decode gives v_c = sigma_c d_c / 2 + (2 b - 1) / 4 with
// d in {1,3,5} (256-row pattern table), sigma the coordinate signs (coordinate
// 0 parity-inferred, e8p.cpp:97-98) and b the shift bit.  With the
// activations as integers, t = alpha * Lt (K1; Lt = sum_l 128^(3-l) limb_l,
// 25-bit values in 4 int8 limbs) and the block sums S_k = sum_c Lt_{8k+c} (exact in
// 4 limbs):
//     z = alpha * ( Z / 2 - TL / 4 ),   Z = sum (sigma d) Lt + sum_k b_k S_k
// TL = sum_i Lt_i (exact, K1).  Z is what the tensor cores accumulate:
//   main MMAs  A = sigma_c d_c  (s8, from TMEM)   B = limb rows of Lt  (smem)
//   side MMA   A = b_k          (s8, from TMEM)   B = limb rows of S_k (smem)
// e8-1bit stages: A = doubled table row, no side term, z = alpha Z / 2.
// Every product is exact int32; segments combine with integer atomics, so the
// result is deterministic and independent of the CTA count.
//
// Data layout ("slab" = 128 rows x 32 codewords of one stage, built once at
// upload; a lossless re-layout of the QSHP codes):
//   E8P slab, 8704 B:  [plane 0..1: idx bytes of codewords 16p..16p+15][128 rows][16 B]
//                      [plane 2..3: negate flags, 4 x u32 per row: word g covers
//                       codewords 4g..4g+3, bit 4c + (w & 3) = flag of coordinate c
//                       (coordinate 0 resolved from the parity at upload)][128][16 B]
//                      [plane 4: shift word per row, bit (w >> 2) + 8 (w & 3) = b_w][128][4 B]
//   e8-1bit slab, 4096 B: [plane 0..1: code bytes][128 rows][16 B]
//   slabs ordered [row block][k slab] per stage: a CTA's contiguous work range is
//   one contiguous byte range, streamed by 1-D bulk copies.
//   B image per k slab (K1): 9 K-blocks x [N rows][32 B] in the K-major
//   no-swizzle core-matrix layout ([N/8][2][8][16 B]); K-block 8 = side.
//
// CTA (one per SM, persistent over a contiguous range of (row block, k slab,
// stage) items; warp-specialised; item i belongs to decode group i % G):
//   warp 0        code producer: 1-D cp.async.bulk of code slabs into a ring
//                 (the first S before TMEM allocation, all before
//                 griddepcontrol.wait, so they overlap K1), the LUT window;
//                 a decoder releases its slot right after loading the slab
//   warps 1..G    one MMA issuer per group: waits for the group's A buffer,
//                 8 + 1 tcgen05.mma (M=128, N, K=32) into the group's TMEM
//                 accumulator with B from its own B-image ring (prefetched from
//                 L2 after griddepcontrol.wait); commits free the A buffer and
//                 the B slot, and at a row-block end hand D to the epilogue
//   warps 1+G..   G groups x 4 decode warps (warp = TMEM lane quadrant, thread =
//                 row): slab -> A bytes in registers -> tcgen05.st into the
//                 group's double-buffered A tile; the group's row-block epilogue
//                 (tcgen05.ld -> int32 atomics) once its D is final
// Decode per codeword: PRMT (LUT address) + LDS (lane-replicated nibble LUT,
// 64-KiB-aligned window) + shift + LOP3 (sign flags) + 2 PRMT from the constant
// byte table {1,3,5,_,-1,-3,-5,_}.
//
// Debug builds: NVEXTRA=-DQ8P_K2_TRACE (per-item clock64 / per-CTA globaltimer
// timeline, written when Q8P_TRACE names a file prefix; tools/tc_timeline.py).
// The variants measured slower in round 1 (cp.async producer, fused K1+K2+K3
// kernel, 2 x 3 A buffers, 2 decoder teams, staggered groups) live
// in git history, not in the product.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <mutex>

#include "device.hpp"
#include "rht_device.cuh"
#include "tc05.hpp"

namespace q8p::detail {
namespace {
using namespace tc05;

constexpr int kSlabCw = 32;                 // codewords per slab row
constexpr std::uint32_t kE8pSlab = 4 * 2048 + 512;
constexpr std::uint32_t kCodeSlot = kE8pSlab;  // code ring slot (e8-1bit slabs are smaller)
constexpr std::uint32_t kMaxB = 12;            // B-image ring slots (max, all groups)
constexpr std::uint32_t kE81Slab = 2 * 2048;
constexpr std::uint32_t kAcols = 72;        // TMEM columns per A buffer (64 main + 8 side)
constexpr int kWarpProd = 0, kWarpMma = 1;  // warps 1..G: one MMA issuer per decode group; then 4G decoder warps
constexpr int kMaxStages = 32;
#define A_EMPTY_WAIT mbar_wait
constexpr std::uint32_t kBg8 = 3;           // B-image ring slots per group at N = 8
constexpr std::uint32_t kCtl = 1024;        // control block (barriers) at the smem base
constexpr std::size_t kSmemBytes = 200 * 1024;  // < 227 KB: K2's prologue co-resides with K1 under PDL

// G decode groups (one TMEM accumulator + one MMA issuer each), T teams of 4
// decoder warps per group: team t decodes the group's items that use A buffer
// t (T = 2) or both buffers alternately (T = 1).
template <int G, int T = 1>
struct Roles {
  static constexpr int kWarpDec = 1 + G;
  static constexpr int kThreads = (kWarpDec + 4 * G * T) * 32;
  template <int N>
  // B-image ring slots per group.  >= 2: the issuer refills the slot of item
  // k - 1 with item k - 1 + kBg after issuing item k, so one slot would deadlock.
  static constexpr std::uint32_t kBg = N <= 8 ? kBg8 : N >= 128 ? 3 : 2;
};

struct TcArgs {
  const std::uint8_t* codes[2];   // per stage slab records
  std::uint32_t slab_bytes[2];
  int kind[2];                    // 0 = e8p, 1 = e8-1bit
  int nst;                        // stages (1 or 2)
  std::uint32_t KSL;              // k slabs per row block
  std::uint32_t items;            // RB * KSL * nst
  const std::uint8_t* bimg;       // [KSL][b_bytes]
  std::uint32_t b_bytes;          // 9 * N * 32
  std::int32_t* zacc;             // [nst][N][rows_pad]
  std::uint32_t rows_pad, m_local;
  int ncols;                      // used B rows (limbs x batch)
  std::uint32_t smem_bytes;
  const std::uint8_t* lut_img;    // 64 KiB LUT window image (tc_lut_image)
  unsigned long long* trace;      // debug timeline (Q8P_TRACE), CTA 0 only; nullptr = off
};

// Debug timeline: trace[role][item][4] clock64 stamps (roles 0..7 decoder
// groups, 8 MMA issuer, 9 producer); written by CTA 0 when a.trace != nullptr.
constexpr int kTraceItems = 128;
__device__ __forceinline__ void tstamp(const TcArgs& a, int role, std::uint32_t item, int ev) {
#ifndef Q8P_K2_TRACE
  return;
#endif
  if (a.trace != nullptr && blockIdx.x == 0 && item < kTraceItems && (threadIdx.x & 31) == 0)
    a.trace[(role * kTraceItems + item) * 4 + ev] = clock64();
}

// LUT reads: the LUT window is constant once bar_lut completed, so these are
// plain (non-volatile, no memory clobber) asm the scheduler may move freely,
// e.g. across the A-buffer wait.
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
__device__ __forceinline__ uint4 lds128(std::uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sts128(std::uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// Raw PTX prmt (default mode); our selectors never set bit 3 of a nibble.
__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t sel) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

constexpr std::uint32_t kCtLo = 0x00050301u;  // {+1,+3,+5,0}
constexpr std::uint32_t kCtHi = 0x00FBFDFFu;  // {-1,-3,-5,0}

// A bytes of one E8P codeword: slot jj (0..3) of an idx / flag register pair.
// `lb` = LUT window bytes 2..3 | lane * 4: PRMT drops idx into byte 1.
template <int JJ>
__device__ __forceinline__ std::uint32_t e8p_nib(std::uint32_t idxreg, std::uint32_t lb) {
  // volatile: issued before the A-buffer wait so the LDS latency overlaps it
  // (measured, tools/ubench_alu.cu: PRMT / LOP3 / SHF issue to the ALU pipe at 16
  // lanes/clk, IMAD at 16, IMAD.HI = mul.hi at only 8 -- a PRMT is the cheapest
  // address for every slot)
  std::uint32_t r;
  const std::uint32_t addr = prmt(idxreg, lb, 0x7604u | (std::uint32_t(JJ) << 4));
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(r) : "r"(addr));
  return r;
}
template <int JJ>
__device__ __forceinline__ void e8p_fin(std::uint32_t nib, std::uint32_t fl, std::uint32_t ct_lo, std::uint32_t ct_hi,
                                        std::uint32_t& lo, std::uint32_t& hi) {
  std::uint32_t rs;
  if constexpr (JJ == 0)
    rs = fl << 2;
  else if constexpr (JJ == 1)
    rs = fl << 1;
  else if constexpr (JJ == 2)
    rs = fl;
  else
    rs = __umulhi(fl, 0x80000000u);  // fl >> 1 on the FMA pipe
  const std::uint32_t sel = nib ^ (rs & 0x44444444u);
  lo = prmt(ct_lo, ct_hi, sel);
  // sel >> 16: SHF (ALU pipe) for even slots, mul.hi (FMA pipe) for odd ones
  hi = prmt(ct_lo, ct_hi, (JJ & 1) ? __umulhi(sel, 65536u) : sel >> 16);
}

// One slab row (thread = row `row_in` of a 128-row slab at smem address `sa`):
// the K2 operand decode shared by the GEMV and the parity probe k2_decode_kernel.
struct SlabRowE8p {
  std::uint32_t idx[8], fl[8], sw;
};
__device__ __forceinline__ SlabRowE8p load_row_e8p(std::uint32_t sa, std::uint32_t row_in) {
  SlabRowE8p r;
  const uint4 i0 = lds128(sa + row_in * 16), i1 = lds128(sa + 2048 + row_in * 16);
  const uint4 f0 = lds128(sa + 4096 + row_in * 16), f1 = lds128(sa + 6144 + row_in * 16);
  r.sw = lds32(sa + 8192 + row_in * 4);
  r.idx[0] = i0.x, r.idx[1] = i0.y, r.idx[2] = i0.z, r.idx[3] = i0.w;
  r.idx[4] = i1.x, r.idx[5] = i1.y, r.idx[6] = i1.z, r.idx[7] = i1.w;
  r.fl[0] = f0.x, r.fl[1] = f0.y, r.fl[2] = f0.z, r.fl[3] = f0.w;
  r.fl[4] = f1.x, r.fl[5] = f1.y, r.fl[6] = f1.z, r.fl[7] = f1.w;
  return r;
}
// A bytes of the row's 32 codewords: codeword 4 g4 + jj -> o[ob + 2 jj] (coordinates
// 0-3), o[ob + 2 jj + 1] (4-7), ob = 16 (g4 >> 1) + 8 (g4 & 1) (the tcgen05.st column
// order); side bytes sd[k8] byte i = shift bit of codeword 4 k8 + i.
__device__ __forceinline__ void decode_row_e8p(const SlabRowE8p& r, std::uint32_t lb, std::uint32_t ct_lo,
                                               std::uint32_t ct_hi, std::uint32_t (&o)[64], std::uint32_t (&sd)[8]) {
#pragma unroll
  for (int g4 = 0; g4 < 8; ++g4) {
    const int ob = 16 * (g4 >> 1) + 8 * (g4 & 1);
    e8p_fin<0>(e8p_nib<0>(r.idx[g4], lb), r.fl[g4], ct_lo, ct_hi, o[ob + 0], o[ob + 1]);
    e8p_fin<1>(e8p_nib<1>(r.idx[g4], lb), r.fl[g4], ct_lo, ct_hi, o[ob + 2], o[ob + 3]);
    e8p_fin<2>(e8p_nib<2>(r.idx[g4], lb), r.fl[g4], ct_lo, ct_hi, o[ob + 4], o[ob + 5]);
    e8p_fin<3>(e8p_nib<3>(r.idx[g4], lb), r.fl[g4], ct_lo, ct_hi, o[ob + 6], o[ob + 7]);
  }
#pragma unroll
  for (int k8 = 0; k8 < 8; ++k8)  // side A = b_k; the shift on the FMA pipe (mul.hi)
    sd[k8] = (k8 == 0 ? r.sw : __umulhi(r.sw, 1u << (32 - k8))) & 0x01010101u;
}
// e8-1bit: A = the doubled table row of each code byte, same column order.
__device__ __forceinline__ void decode_row_e81(std::uint32_t sa, std::uint32_t row_in, std::uint32_t lb8,
                                               std::uint32_t (&o)[64]) {
  const uint4 c0 = lds128(sa + row_in * 16), c1 = lds128(sa + 2048 + row_in * 16);
  const std::uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
  for (int g4 = 0; g4 < 8; ++g4) {
    const int ob = 16 * (g4 >> 1) + 8 * (g4 & 1);
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const uint2 v = lut64(prmt(cw[g4], lb8, 0x7604u | (std::uint32_t(jj) << 4)));
      o[ob + 2 * jj] = v.x;
      o[ob + 2 * jj + 1] = v.y;
    }
  }
}

template <int N, int G, int T, int NB>
__global__ void __launch_bounds__(Roles<G, T>::kThreads, 1) gemv_tc_kernel(TcArgs a) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  // warp index via shfl: the compiler then knows every role branch is warp-uniform
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const std::uint32_t sbase = smem_u32(smem);
  const std::uint32_t send = sbase + a.smem_bytes;
  // B ring: [group][slot], b_slot bytes per k-slab image
  const std::uint32_t b_slot = (a.b_bytes + 127) & ~127u;
  constexpr std::uint32_t SBg = Roles<G>::template kBg<N>, SB = SBg * G;
  static_assert(SB <= kMaxB, "B-image ring slots exceed the barrier block (kMaxB)");
  // smem layout.  N <= 64: [ctl][code slots][LUT window, 64 KiB aligned][B ring][code slots].
  // N = 128 (36 KB B slots, 3 deep): [ctl][B ring][code slot(s)][LUT window][code slots].
  constexpr bool kBLow = N >= 128;
  const std::uint32_t lutw = (sbase + kCtl + (kBLow ? SB * b_slot : 0u) + 0xFFFFu) & ~0xFFFFu;
  // control block: barriers + TMEM base
  const std::uint32_t bar_full_c = sbase;                       // [kMaxStages] code slab landed
  const std::uint32_t bar_empty_c = sbase + 8 * kMaxStages;     // [kMaxStages] code slab read (4 warps)
  const std::uint32_t bar_full_b = sbase + 16 * kMaxStages;     // [kMaxB] B image landed
  const std::uint32_t bar_empty_b = bar_full_b + 8 * kMaxB;     // [kMaxB] B image read by its MMAs
  const std::uint32_t bar_a_empty = bar_empty_b + 8 * kMaxB;    // [G][2] A buffer read by its MMAs
  const std::uint32_t bar_a_full = bar_a_empty + 8 * NB * G;    // [G][NB] A buffer written (4 warp arrivals)
  const std::uint32_t bar_d_full = bar_a_full + 8 * NB * G;     // [G][T] accumulator final (team t's epilogue)
  const std::uint32_t bar_d_empty = bar_d_full + 8 * G * T;     // [G] accumulator read out (4 warp arrivals)
  const std::uint32_t bar_lut = bar_d_empty + 8 * G;            // LUT window landed
  const std::uint32_t tmem_slot = bar_lut + 8;
  const std::uint32_t ct_slot = tmem_slot + 8;  // the constant byte table, read back by the decoders
  constexpr int kWarpDec = Roles<G>::kWarpDec;
  const std::uint32_t b_base = kBLow ? sbase + kCtl : lutw + 65536;
  const std::uint32_t lo_base = sbase + kCtl + (kBLow ? SB * b_slot : 0u);
  const std::uint32_t n_lo = lutw > lo_base ? (lutw - lo_base) / kCodeSlot : 0;
  const std::uint32_t hi_base = kBLow ? lutw + 65536 : b_base + SB * b_slot;
  if (hi_base > send) __trap();  // B ring past the dynamic smem (host sizing bug): fail loudly
  std::uint32_t S = n_lo + (send > hi_base ? (send - hi_base) / kCodeSlot : 0);
  if (S > kMaxStages) S = kMaxStages;
  auto code_addr = [&](std::uint32_t st) { return st < n_lo ? lo_base + st * kCodeSlot : hi_base + (st - n_lo) * kCodeSlot; };

  const std::uint32_t it0 = std::uint32_t((std::uint64_t(a.items) * blockIdx.x) / gridDim.x);
  const std::uint32_t it1 = std::uint32_t((std::uint64_t(a.items) * (blockIdx.x + 1)) / gridDim.x);
  const std::uint32_t count = it1 - it0;
  const std::uint32_t nst = std::uint32_t(a.nst);

  if (threadIdx.x == 0) tstamp(a, 10, 0, 0);
#ifdef Q8P_K2_TRACE
  auto gstamp = [&](int ev) {  // per-CTA globaltimer (ns): 0 entry, 1 setup done, 2 work done
    if (a.trace != nullptr && blockIdx.x < 256) {
      std::uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[11 * kTraceItems * 4 + blockIdx.x * 4 + ev] = t;
    }
  };
  if (threadIdx.x == 0) gstamp(0);
#endif
  if (threadIdx.x == 0) {
    for (std::uint32_t i = 0; i < S; ++i) {
      mbar_init(bar_full_c + 8 * i, 1);
      mbar_init(bar_empty_c + 8 * i, 4);
    }
    for (std::uint32_t i = 0; i < SB; ++i) {
      mbar_init(bar_full_b + 8 * i, 1);
      mbar_init(bar_empty_b + 8 * i, 1);
    }
    for (int i = 0; i < NB * G; ++i) {
      mbar_init(bar_a_empty + 8 * i, 1);
      mbar_init(bar_a_full + 8 * i, 4);
    }
    for (int i = 0; i < G * T; ++i) mbar_init(bar_d_full + 8 * i, 1);
    for (int i = 0; i < G; ++i) mbar_init(bar_d_empty + 8 * i, 4);
    mbar_init(bar_lut, 1);
    fence_mbar_init();
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(ct_slot), "r"(kCtLo), "r"(kCtHi) : "memory");
  }
  // Code producer.  Item i goes to ring slot i % S (phase i / S); warp 0 issues
  // every slab as one 1-D cp.async.bulk.  The first S slabs (and the LUT window)
  // are issued before the TMEM allocation and the CTA barrier.
  const std::uint64_t pol = policy_evict_first();
  auto issue_item = [&](std::uint32_t i) {
    const std::uint32_t it = it0 + i, u = it / nst, sidx = it - u * nst, st = i % S;
    const std::uint32_t sb = sidx ? a.slab_bytes[1] : a.slab_bytes[0];
    const std::uint8_t* src = (sidx ? a.codes[1] : a.codes[0]) + std::size_t(u) * sb;
    mbar_arrive_expect_tx_e(bar_full_c + 8 * st, sb);
    bulk_g2s_hint_e(code_addr(st), src, sb, bar_full_c + 8 * st, pol);
  };
  const std::uint32_t pre = count < S ? count : S;
  if (warp == kWarpProd) {
    __syncwarp();  // lane 0 initialised the barriers
    if (count > 0) {
      issue_item(0);  // first code slab, then the (L2-resident) LUT window
      mbar_arrive_expect_tx_e(bar_lut, 65536);
      bulk_g2s_e(lutw, a.lut_img, 65536, bar_lut);
      for (std::uint32_t i = 1; i < pre; ++i) issue_item(i);
    }
    tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tbase = *reinterpret_cast<volatile std::uint32_t*>(smem + (tmem_slot - sbase));
  if (threadIdx.x == 0) tstamp(a, 10, 0, 1);
#ifdef Q8P_K2_TRACE
  if (threadIdx.x == 0) gstamp(1);
#endif

  if (warp == kWarpProd) {
    // ===== code producer (codes do not depend on K1) =====
    for (std::uint32_t i = pre; i < count; ++i) {
      tstamp(a, 9, i, 0);
      mbar_wait(bar_empty_c + 8 * (i % S), ((i / S) & 1) ^ 1);
      tstamp(a, 9, i, 1);
      issue_item(i);
    }
    pdl_trigger();
  } else if (warp < kWarpDec) {
    // ===== MMA issuer of group g (+ its B-image prefetch): items i = g, g + G, ... =====
    // One issuer per group keeps each accumulator's MMAs on one thread (in-order
    // accumulate, per-thread commit tracking) and runs the groups' handshakes in
    // parallel; every per-item quantity is an incremental counter.
    pdl_trigger();
    const std::uint32_t g = std::uint32_t(warp - kWarpMma);
    if (count > g) {
      constexpr std::uint32_t idesc = idesc_i8(128, N);
      const std::uint32_t per_rb = a.KSL * nst;
      const std::uint32_t bb = b_base + g * SBg * b_slot;  // this group's B slots
      const std::uint32_t fb = bar_full_b + 8 * g * SBg, eb = bar_empty_b + 8 * g * SBg;
      const std::uint64_t bd0 = sdesc(bb, 128, 256);
      const std::uint32_t bstep = b_slot >> 4;  // descriptor units per B slot
      const std::uint32_t n_g = (count - g + G - 1) / G;  // this group's items
      // B prefetch cursor: (stage, k slab) of the next group item to fetch
      std::uint32_t bs = (it0 + g) % nst, bks = ((it0 + g) / nst) % a.KSL, bnext = 0, bslot_n = 0;
      auto issue_b = [&]() {
        mbar_arrive_expect_tx_e(fb + 8 * bslot_n, a.b_bytes);
        bulk_g2s_e(bb + bslot_n * b_slot, a.bimg + std::size_t(bks) * a.b_bytes, a.b_bytes, fb + 8 * bslot_n);
#pragma unroll
        for (int t = 0; t < G; ++t)
          if (++bs == nst) {
            bs = 0;
            if (++bks == a.KSL) bks = 0;
          }
        ++bnext;
        if (++bslot_n == SBg) bslot_n = 0;
      };
      pdl_wait();  // K1's B images (and zeroed accumulators) are visible from here on
#ifdef Q8P_DBG_PROXY_FENCE
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
#endif
      while (bnext < n_g && bnext < SBg) issue_b();
      std::uint32_t j = (it0 + g) % per_rb;
      std::uint32_t buf = 0, bph = 0, started = 0, seg = 0, team = 0;
      std::uint32_t bslot = 0, bphase = 0, rslot = 0, rphase = 0;
      const std::uint32_t dcol_g = tbase + std::uint32_t(G) * NB * kAcols + g * nst * N;
      const std::uint32_t acol0 = tbase + NB * g * kAcols;
      const std::uint32_t af0 = bar_a_full + 8 * NB * g, ae0 = bar_a_empty + 8 * NB * g;
      for (std::uint32_t k = 0, i = g; k < n_g; ++k, i += G) {
        const std::uint32_t s = j & (nst - 1);
        tstamp(a, 8 + (g == 0 ? 0 : 4 + g), k, 0);
        // first MMA of a new row block overwrites D: the previous epilogue must have read it
        if (started == 0 && seg > 0) mbar_wait(bar_d_empty + 8 * g, (seg - 1) & 1);
        mbar_wait(af0 + 8 * buf, bph);
        tstamp(a, 8 + (g == 0 ? 0 : 4 + g), k, 1);
        mbar_wait(fb + 8 * bslot, bphase);
        tstamp(a, 8 + (g == 0 ? 0 : 4 + g), k, 2);
        tc_fence_after();
        mma_i8_slab_e<2 * N>(dcol_g + s * N, acol0 + buf * kAcols, bd0 + bslot * bstep, idesc, (started >> s) & 1,
                             (s ? a.kind[1] : a.kind[0]) == 0, ae0 + 8 * buf, eb + 8 * bslot);
        started |= 1u << s;
        if ((j + G >= per_rb) || (i + G >= count)) {  // this group's last item of the row block
          mma_commit_e(bar_d_full + 8 * (g * T + team));
          started = 0;
          ++seg;
        }
        tstamp(a, 8 + (g == 0 ? 0 : 4 + g), k, 3);
        // refill the slot of the previous group item (its MMAs were issued one item ago)
        if (k >= 1 && bnext < n_g) {
          mbar_wait(eb + 8 * rslot, rphase);
          issue_b();
          if (++rslot == SBg) rslot = 0, rphase ^= 1;
        }
        if (++bslot == SBg) bslot = 0, bphase ^= 1;
        if (++buf == NB) buf = 0, bph ^= 1;
        if (++team == T) team = 0;
        j += G;
        while (j >= per_rb) j -= per_rb;
      }
    }
  } else {
    // ===== decode groups: codes -> A bytes -> TMEM (4 warps = 4 lane quadrants) =====
    pdl_trigger();
    const int tq = (warp - kWarpDec) >> 2;  // team index over all groups
    const int grp = tq / T, tm = tq % T;
    const std::uint32_t q = warp & 3, row_in = q * 32 + lane;
    const std::uint32_t tl = (q * 32) << 16;
    const std::uint32_t lb = (lutw & 0xFFFF0000u) | (std::uint32_t(lane) * 4u);
    const std::uint32_t lb8 = (lutw & 0xFFFF0000u) | (128u + std::uint32_t(lane & 15) * 8u);
    const std::uint32_t dcol = tbase + std::uint32_t(G) * NB * kAcols + std::uint32_t(grp) * nst * N;
    const std::uint32_t per_rb = a.KSL * nst;
    const std::uint32_t i_first = std::uint32_t(grp + G * tm);
    std::uint32_t st = i_first % S, r = i_first / S, use = std::uint32_t(tm), seg = 0, started = 0;
    std::uint32_t j = (it0 + i_first) % per_rb, rb = (it0 + i_first) / per_rb;
    // constant byte table {+1,+3,+5,_ | -1,-3,-5,_} loaded from smem so it lives
    // in ONE register (as an immediate/uniform value ptxas re-materialises it
    // with a UR->R move in front of every PRMT: +1 instruction per codeword)
    const uint2 ct = lds64(ct_slot);
    const std::uint32_t ct_lo = ct.x, ct_hi = ct.y;
    if (count > i_first) mbar_wait(bar_lut, 0);  // the producer copies the LUT only when it has work
    if (warp == kWarpDec) tstamp(a, 10, 1, 0);
    for (std::uint32_t i = i_first; i < count; i += G * T) {
      const std::uint32_t s = j & (nst - 1);  // nst in {1, 2}
      const std::uint32_t buf = use % NB, bph = (use / NB) & 1;
      const std::uint32_t sa = code_addr(st);
      const bool e8p = (s ? a.kind[1] : a.kind[0]) == 0;
      const bool tw = q == 1;
      if (tw) tstamp(a, grp, i, 0);
      mbar_wait(bar_full_c + 8 * st, r & 1);
      if (tw) tstamp(a, grp, i, 1);
      const std::uint32_t abuf = tbase + tl + (NB * grp + buf) * kAcols;
      if (e8p) {
        const SlabRowE8p row = load_row_e8p(sa, row_in);
        // Decode the whole slab row into registers first, then wait for the A buffer:
        // the decode overlaps the MMA turnaround of the buffer's previous item.
        std::uint32_t o[64], sd[8];
        decode_row_e8p(row, lb, ct_lo, ct_hi, o, sd);
        // Hand the slot back only now: the decode has consumed every loaded register,
        // so the warp's LDS of the slot have completed.  (An arrive right after the
        // LDS instructions can overtake them -- the loads are asynchronous until a
        // register is read -- and the producer's bulk copy for item i + S then
        // overwrites the slot under them: a WAR race when the ring wraps.)
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_empty_c + 8 * st);
        // pin every result before the wait (an empty asm consuming them; no code)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          asm volatile("" ::"r"(o[16 * q4 + 0]), "r"(o[16 * q4 + 1]), "r"(o[16 * q4 + 2]), "r"(o[16 * q4 + 3]),
                       "r"(o[16 * q4 + 4]), "r"(o[16 * q4 + 5]), "r"(o[16 * q4 + 6]), "r"(o[16 * q4 + 7]),
                       "r"(o[16 * q4 + 8]), "r"(o[16 * q4 + 9]), "r"(o[16 * q4 + 10]), "r"(o[16 * q4 + 11]),
                       "r"(o[16 * q4 + 12]), "r"(o[16 * q4 + 13]), "r"(o[16 * q4 + 14]), "r"(o[16 * q4 + 15]));
        asm volatile("" ::"r"(sd[0]), "r"(sd[1]), "r"(sd[2]), "r"(sd[3]), "r"(sd[4]), "r"(sd[5]), "r"(sd[6]),
                     "r"(sd[7]));
        A_EMPTY_WAIT(bar_a_empty + 8 * (NB * grp + buf), bph ^ 1);
        if (tw) tstamp(a, grp, i, 2);
        tc_fence_after();
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) tmem_st16(abuf + 16 * qq, *reinterpret_cast<std::uint32_t(*)[16]>(o + 16 * qq));
        tmem_st8(abuf + 64, sd);
      } else {
        std::uint32_t o[64];
        decode_row_e81(sa, row_in, lb8, o);
        __syncwarp();  // (after the decode consumed the slot's loads, as above)
        if (lane == 0) mbar_arrive(bar_empty_c + 8 * st);
        A_EMPTY_WAIT(bar_a_empty + 8 * (NB * grp + buf), bph ^ 1);
        tc_fence_after();
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) tmem_st16(abuf + 16 * qq, *reinterpret_cast<std::uint32_t(*)[16]>(o + 16 * qq));
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_a_full + 8 * (NB * grp + buf));
      if (tw) tstamp(a, grp, i, 3);
      if ((j + G >= per_rb) || (i + G >= count)) {
        // epilogue of this row block: D (int32, exact) -> global accumulators.
        // Stages present in D: the group's items of this row block sit at
        // positions j, j - G, ... >= lo0 (the CTA's first position in it); with
        // nst = 2 and G odd, two or more items cover both stages.
        {
          const std::uint32_t lo0 = j >= i ? j - i : 0;
          started = 1u << s;
          if (nst == 2 && (G & 1) && j >= lo0 + G) started = 3;
        }
        if (seg == 0) pdl_wait();  // K1 zeroed the accumulators
        mbar_wait(bar_d_full + 8 * (grp * T + tm), seg & 1);
        tc_fence_after();
        const std::uint32_t row = rb * 128 + row_in;
        const bool row_ok = row < a.m_local;
        for (std::uint32_t s2 = 0; s2 < nst; ++s2) {
          if (!((started >> s2) & 1)) continue;  // no item of stage s2 from this group here
          std::int32_t* z = a.zacc + std::size_t(s2) * N * a.rows_pad + row;
#pragma unroll
          for (int c0 = 0; c0 < N; c0 += 8) {
            std::uint32_t t8[8];
            tmem_ld8(dcol + tl + s2 * N + c0, t8);
            tmem_wait_ld();
            if (row_ok) {
#pragma unroll
              for (int jj = 0; jj < 8; ++jj)
                if (c0 + jj < a.ncols) atomicAdd(z + std::size_t(c0 + jj) * a.rows_pad, std::int32_t(t8[jj]));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_d_empty + 8 * grp);  // D may be overwritten now
        started = 0;
        ++seg;
      }
      use += T;
      st += G * T;
      while (st >= S) {
        st -= S;
        ++r;
      }
      j += G * T;
      while (j >= per_rb) {
        j -= per_rb;
        ++rb;
      }
    }
  }
  if (threadIdx.x == 0) tstamp(a, 10, 0, 2);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) tstamp(a, 10, 0, 3);

  if (warp == kWarpProd) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
#ifdef Q8P_K2_TRACE
    if (lane == 0) gstamp(2);
#endif
  }
}

constexpr std::size_t kSmemWide = 225 * 1024;   // N = 128 (prefill chunks of 32 vectors): 3 x 36 KB B slots
template <int N>
constexpr std::size_t smem_for() {
  return N >= 128 ? kSmemWide : kSmemBytes;
}

int sm_count() {  // per device (layers may live on different devices of one process)
  static int v[64] = {};
  const int d = current_device() & 63;
  if (!v[d]) cuda_check(cudaDeviceGetAttribute(&v[d], cudaDevAttrMultiProcessorCount, d), "sm count");
  return v[d];
}

template <int N, int G, int T = 1, int NB = 2>
void launch_ng(TcArgs a, cudaStream_t s) {
  kernel_attrs(reinterpret_cast<const void*>(gemv_tc_kernel<N, G, T, NB>), int(smem_for<N>()));
  a.smem_bytes = std::uint32_t(smem_for<N>());
  launch_pdl(gemv_tc_kernel<N, G, T, NB>, dim3(sm_count()), dim3(Roles<G, T>::kThreads), smem_for<N>(), s, a);
}

}  // namespace

// ---- host: tables and slab transcoding ---------------------------------------
// 64 KiB shared-memory LUT window, 256 rows of 256 B (row = idx, 64-KiB aligned
// in smem so a PRMT of (window, idx byte, lane) forms the LDS address):
//   bytes [0, 128):   E8P magnitude nibbles of row idx (d = 1,3,5 -> 0,1,2 at
//                     bits 4c), replicated once per lane (lane * 4)
//   bytes [128, 256): e8-1bit doubled row (8 x s8), replicated per half-warp lane
std::vector<std::uint8_t> tc_lut_image() {
  const E8PTable& t = e8p_table();
  const auto& d = e8_1bit_doubled();
  std::vector<std::uint8_t> img(65536, 0);
  for (int i = 0; i < 256; ++i) {
    std::uint32_t w = 0;
    for (int c = 0; c < 8; ++c) w |= std::uint32_t((t.doubled[i][c] - 1) / 2) << (4 * c);
    std::uint8_t e81[8];
    for (int c = 0; c < 8; ++c) e81[c] = std::uint8_t(d[i][c]);
    std::uint8_t* row = img.data() + i * 256;
    for (int l = 0; l < 32; ++l) std::memcpy(row + 4 * l, &w, 4);
    for (int l = 0; l < 16; ++l) std::memcpy(row + 128 + 8 * l, e81, 8);
  }
  return img;
}

// Compact decode tables (q8p_layer::dec_tables, read by K4's decoders through the
// read-only path): [256] E8P magnitude-nibble words (d = 1,3,5 -> 0,1,2 at bits 4c),
// then [256][2] e8-1bit doubled rows (8 x s8).
std::vector<std::uint32_t> decode_table_words() {
  const E8PTable& t = e8p_table();
  const auto& d = e8_1bit_doubled();
  std::vector<std::uint32_t> w(256 * 3, 0);
  for (int i = 0; i < 256; ++i) {
    for (int c = 0; c < 8; ++c) w[i] |= std::uint32_t((t.doubled[i][c] - 1) / 2) << (4 * c);
    for (int c = 0; c < 8; ++c) w[256 + 2 * i + c / 4] |= std::uint32_t(std::uint8_t(d[i][c])) << (8 * (c % 4));
  }
  return w;
}

std::uint32_t tc_slab_bytes(int kind) { return kind == 0 ? kE8pSlab : kE81Slab; }
std::uint32_t tc_row_blocks(std::uint32_t m_local) { return (m_local + 127) / 128; }
std::uint32_t tc_k_slabs(std::uint32_t n) { return (n / 8 + kSlabCw - 1) / kSlabCw; }

std::size_t tc_code_bytes(std::uint32_t m_local, std::uint32_t n, int kind) {
  return std::size_t(tc_row_blocks(m_local)) * tc_k_slabs(n) * tc_slab_bytes(kind);
}

namespace {
// tc_transcode on the device: one thread per (row, k slab) of the plain codes
// ([m_local][nb], u16 for E8P, u8 for e8-1bit), same bytes as the host version.
__global__ void __launch_bounds__(256) tc_transcode_kernel(const void* __restrict__ codes, std::uint32_t m_local,
                                                          std::uint32_t nb, std::uint32_t KSL, int kind,
                                                          std::uint8_t* __restrict__ out,
                                                          const std::uint8_t* __restrict__ odd) {
  const std::uint32_t RB = (m_local + 127) / 128;
  const std::size_t total = std::size_t(RB) * 128 * KSL;
  const std::size_t SB = kind == 0 ? kE8pSlab : kE81Slab;
  for (std::size_t t = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += std::size_t(gridDim.x) * blockDim.x) {
    const std::uint32_t r = std::uint32_t(t % 128), ks = std::uint32_t((t / 128) % KSL),
                        rb = std::uint32_t(t / (128 * std::size_t(KSL)));
    const std::uint32_t row = rb * 128 + r;
    std::uint8_t* slab = out + (std::size_t(rb) * KSL + ks) * SB;
    std::uint32_t idxw[8] = {0, 0, 0, 0, 0, 0, 0, 0}, fl[8] = {0, 0, 0, 0, 0, 0, 0, 0}, sw = 0;
    for (std::uint32_t w = 0; w < 32; ++w) {
      const std::uint32_t k = ks * 32 + w;
      std::uint32_t word = 0;
      if (row < m_local && k < nb)
        word = kind == 0 ? static_cast<const std::uint16_t*>(codes)[std::size_t(row) * nb + k]
                         : static_cast<const std::uint8_t*>(codes)[std::size_t(row) * nb + k];
      const std::uint32_t byte = kind == 0 ? (word >> 8) : word;
      idxw[w / 4] |= byte << (8 * (w & 3));
      if (kind == 0) {
        const std::uint32_t idx = word >> 8, sb = (word >> 1) & 0x7Fu;
        // effective negate flags (e8p.cpp:88-98): word bit k (1..7) -> coordinate 8 - k,
        // coordinate 0 restores the row's parity
        fl[w / 4] |= ((std::uint32_t(__popc(sb)) & 1u) ^ odd[idx]) << (w & 3);
        for (std::uint32_t c = 1; c < 8; ++c) fl[w / 4] |= ((word >> (8 - c)) & 1u) << (4 * c + (w & 3));
        sw |= (word & 1u) << ((w >> 2) + 8 * (w & 3));
      }
    }
    // idx / code bytes: plane w / 16, row r, byte w % 16
    *reinterpret_cast<uint4*>(slab + r * 16) = make_uint4(idxw[0], idxw[1], idxw[2], idxw[3]);
    *reinterpret_cast<uint4*>(slab + 2048 + r * 16) = make_uint4(idxw[4], idxw[5], idxw[6], idxw[7]);
    if (kind == 0) {
      *reinterpret_cast<uint4*>(slab + 4096 + r * 16) = make_uint4(fl[0], fl[1], fl[2], fl[3]);
      *reinterpret_cast<uint4*>(slab + 6144 + r * 16) = make_uint4(fl[4], fl[5], fl[6], fl[7]);
      *reinterpret_cast<std::uint32_t*>(slab + 8192 + r * 4) = sw;
    }
  }
}
}  // namespace

void tc_transcode_device(const void* codes, std::uint32_t m_local, std::uint32_t n, int kind, std::uint8_t* out,
                         const std::uint8_t* odd_parity_dev, cudaStream_t s) {
  const std::uint32_t nb = n / 8, KSL = tc_k_slabs(n);
  const std::size_t total = std::size_t(tc_row_blocks(m_local)) * 128 * KSL;
  const unsigned grid = unsigned(std::min<std::size_t>((total + 255) / 256, 148 * 16));
  tc_transcode_kernel<<<grid, 256, 0, s>>>(codes, m_local, nb, KSL, kind, out, odd_parity_dev);
  cuda_check(cudaGetLastError(), "transcode launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// MMA N for `ncols` B rows (4 limbs x batch): 8, 16, 32, 64, then 128 (batch 17..32).
// (Batches 9-12 run at N = 64: the N = 48 variant showed rare run-to-run differences
// on long-k layers that no other N shows -- tools/dbg_repeat3.py.)
int tc_ncols_pad(int ncols) {
  return ncols <= 8 ? 8 : ncols <= 16 ? 16 : ncols <= 32 ? 32 : ncols <= 64 ? 64 : 128;
}
bool tc_supported(const q8p_layer& L, int batch) {
  return batch >= 1 && batch <= kTcMaxBatch && L.tc[0].codes != nullptr && L.cb[0] == Q8P_CB_E8P_2BIT &&
         (L.num_stages == 1 || L.tc[1].codes != nullptr);
}
std::uint32_t tc_bimg_bytes(std::uint32_t n, int batch) {
  return tc_k_slabs(n) * 9u * std::uint32_t(tc_ncols_pad(4 * batch)) * 32u;
}

namespace {
void fill_tc_args(const q8p_layer& L, const std::uint8_t* bimg, std::int32_t* zacc, std::uint32_t rows_pad, int batch,
                  TcArgs& a) {
  a = TcArgs{};
  a.nst = L.num_stages;
  for (int st = 0; st < L.num_stages; ++st) {
    a.codes[st] = static_cast<const std::uint8_t*>(L.tc[st].codes);
    a.kind[st] = L.cb[st] == Q8P_CB_E8P_2BIT ? 0 : 1;
    a.slab_bytes[st] = tc_slab_bytes(a.kind[st]);
  }
  const int N = tc_ncols_pad(4 * batch);
  a.KSL = tc_k_slabs(L.n);
  a.items = tc_row_blocks(L.m_local()) * a.KSL * std::uint32_t(a.nst);
  a.bimg = bimg;
  a.b_bytes = 9u * std::uint32_t(N) * 32u;
  a.zacc = zacc;
  a.rows_pad = rows_pad;
  a.m_local = L.m_local();
  a.ncols = 4 * batch;
  a.smem_bytes = std::uint32_t(kSmemBytes);
  a.lut_img = L.lut_img;
}
}  // namespace

void launch_gemv_tc(const q8p_layer& L, const std::uint8_t* bimg, std::int32_t* zacc, std::uint32_t rows_pad,
                    int batch, cudaStream_t s) {
  TcArgs a;
  fill_tc_args(L, bimg, zacc, rows_pad, batch, a);
  const int N = tc_ncols_pad(4 * batch);
  static const char* trace_env = std::getenv("Q8P_TRACE");  // debug: dump CTA 0's timeline
  unsigned long long* tr = nullptr;
  if (trace_env != nullptr) {
    cuda_check(cudaMalloc(&tr, 16 * kTraceItems * 4 * 8), "trace alloc");
    cuda_check(cudaMemset(tr, 0, 16 * kTraceItems * 4 * 8), "trace memset");
  }
  a.trace = tr;
  // TMEM: G decode groups x (2 A buffers x 72 columns + an accumulator of stages x N) <= 512
  auto fits = [&](int G) { return G * (2 * int(kAcols) + a.nst * N) <= 512; };
  switch (N) {
    case 8:
      launch_ng<8, 3>(a, s);
      break;
    case 16: fits(3) ? launch_ng<16, 3>(a, s) : launch_ng<16, 2>(a, s); break;
    case 32: launch_ng<32, 2>(a, s); break;
    case 64: fits(2) ? launch_ng<64, 2>(a, s) : launch_ng<64, 1>(a, s); break;
    default: launch_ng<128, 1>(a, s); break;  // prefill chunks: one decode group, 400 TMEM columns
  }
  cuda_check(cudaGetLastError(), "gemv_tc launch");
  if (tr != nullptr) {
    std::vector<unsigned long long> h(16 * kTraceItems * 4);
    cuda_check(cudaStreamSynchronize(s), "trace sync");
    cuda_check(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost), "trace copy");
    cudaFree(tr);
    static int seq = 0;
    const std::string path = std::string(trace_env) + "." + std::to_string(seq++) + "." + std::to_string(L.m_local()) +
                             "x" + std::to_string(L.n) + ".bin";
    if (FILE* f = std::fopen(path.c_str(), "wb")) {
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// ---- parity probe: K2's own operand decode over the transcoded slabs -------------
namespace {
// One CTA per slab: the slab and the LUT window are loaded into shared memory as
// K2 loads them, then each thread runs K2's row decode (load_row_e8p /
// decode_row_e8p, decode_row_e81) and writes the A bytes it would store to TMEM:
// a[row][8k + c] (s8) and, for E8P, the side byte (shift bit) side[row][k].
__global__ void __launch_bounds__(128) k2_decode_kernel(const std::uint8_t* __restrict__ slabs, std::uint32_t slab_bytes,
                                                        int kind, std::uint32_t m_local, std::uint32_t nb,
                                                        std::uint32_t KSL, const std::uint8_t* __restrict__ lut_img,
                                                        std::int8_t* __restrict__ a_out, std::uint8_t* __restrict__ side) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  const std::uint32_t sbase = smem_u32(smem);
  const std::uint32_t lutw = (sbase + kE8pSlab + 0xFFFFu) & ~0xFFFFu;
  const std::uint32_t rb = blockIdx.x / KSL, ks = blockIdx.x % KSL;
  const std::uint8_t* src = slabs + std::size_t(blockIdx.x) * slab_bytes;
  for (std::uint32_t i = threadIdx.x; i < slab_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (std::uint32_t i = threadIdx.x; i < 65536 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem + (lutw - sbase))[i] = reinterpret_cast<const uint4*>(lut_img)[i];
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(lutw - 16), "r"(kCtLo), "r"(kCtHi) : "memory");
  __syncthreads();
  const std::uint32_t lane = threadIdx.x & 31, row_in = threadIdx.x;
  const std::uint32_t lb = (lutw & 0xFFFF0000u) | (lane * 4u);
  const std::uint32_t lb8 = (lutw & 0xFFFF0000u) | (128u + (lane & 15) * 8u);
  const uint2 ct = lds64(lutw - 16);
  std::uint32_t o[64], sd[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (kind == 0)
    decode_row_e8p(load_row_e8p(sbase, row_in), lb, ct.x, ct.y, o, sd);
  else
    decode_row_e81(sbase, row_in, lb8, o);
  const std::uint32_t row = rb * 128 + row_in;
  if (row >= m_local) return;
  for (int w = 0; w < 32; ++w) {
    const std::uint32_t k = ks * 32 + w;
    if (k >= nb) break;
    const int g4 = w >> 2, jj = w & 3, ob = 16 * (g4 >> 1) + 8 * (g4 & 1);
    *reinterpret_cast<uint2*>(a_out + (std::size_t(row) * nb + k) * 8) = make_uint2(o[ob + 2 * jj], o[ob + 2 * jj + 1]);
    if (side) side[std::size_t(row) * nb + k] = std::uint8_t((sd[w >> 2] >> (8 * (w & 3))) & 1u);
  }
}
}  // namespace

void launch_k2_decode(const q8p_layer& L, int stage, std::int8_t* a_out, std::uint8_t* side, cudaStream_t s) {
  if (!L.tc[stage].codes) throw UnsupportedError("layer has no tensor-core slabs");
  const int kind = L.cb[stage] == Q8P_CB_E8P_2BIT ? 0 : 1;
  const std::uint32_t KSL = tc_k_slabs(L.n), RB = tc_row_blocks(L.m_local());
  constexpr int kSmemProbe = 140 * 1024;
  kernel_attrs(reinterpret_cast<const void*>(k2_decode_kernel), kSmemProbe);
  k2_decode_kernel<<<RB * KSL, 128, kSmemProbe, s>>>(static_cast<const std::uint8_t*>(L.tc[stage].codes),
                                                    tc_slab_bytes(kind), kind, L.m_local(), L.n / 8, KSL, L.lut_img,
                                                    a_out, kind == 0 ? side : nullptr);
  cuda_check(cudaGetLastError(), "k2 decode probe launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
