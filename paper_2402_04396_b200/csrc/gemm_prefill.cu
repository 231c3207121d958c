// K4: prefill (large batch) decode-GEMM on the 5th-gen tensor cores,
// weight-stationary per tile: every weight tile is decoded ONCE into shared
// memory and multiplied against 256 vectors (tcgen05.mma kind::i8, s8 x s8 ->
// exact s32 accumulators in tensor memory).
//
// Semantics: z[b][r] = sum_s scale_s * sum_k <decode_s(codes[s][r][k]), t_b[8k:8k+8]>
// (core/src/pipeline.cpp:172-191; the reference CLI loops infer per vector,
// latq_cli.cpp:211-212), t = T_v x from K1's fp32 flavour, y = T_u^T z by K3.
//
// Operands.  A = 4 v exactly: E8P 4 v = 2 sigma d + 2 b - 1 (odd integers in
// [-11, 11], e8p.cpp:81-100), e8-1bit 4 v = 2 * doubled (codebook.cpp:65-72) --
// exact in s8.  B: per vector b one fixed-point scale alpha_b = max_s scale_s *
// max|t_b| / 32000 (pack kernel), L = rint(scale_s t / alpha_b) (|L| <= 32000,
// 16-bit activations, the precision of the former bf16 hi/lo split) as two balanced
// s8 limbs L = 256 h + l; D_h, D_l = A . h, A . l in two s32 accumulators (exact:
// |D| < 2^27), z = alpha_b (256 D_h + D_l) / 4 in the epilogue; RVQ stages are
// further K items against their own L (same alpha_b).  kind::i8 runs K = 32 per
// MMA at the f16 rate of K = 16, so the two limbs cost what ONE bf16 term did.
//
// Layout.  Codes: the tensor-core slabs of gemv_tc.cu (128 rows x 32 codewords
// per stage, [row block][k slab]).  B tiles (written by the pack kernel): per
// (N tile of 256 vectors, K chunk of 32, stage) one contiguous 16 KiB region
// [limb h/l][32 vector groups][2 K halves][8 vectors][16 B] = the canonical
// K-major no-swizzle UMMA layout (LBO 128 B, SBO 256 B), then alpha per vector;
// the A tile of a K chunk is the same layout over 128 rows (4 KiB).
//
// CTA (persistent, stream-K: equal shares of the tiles' k-slab steps; a tile = (N
// tile, M tile) of 128 rows x 256 vectors, split at CTA boundaries into pieces
// that K3 sums):
//   warp 0   producer: code slabs (1-D bulk copies, one per k slab and stage) and
//            B regions (one 16 KiB bulk copy per item) into rings
//   warp 1   MMA issuer: per item (K chunk, stage) 2 limbs x tcgen05.mma M=128
//            N=256 K=32 into the limbs' accumulators (2 x 256 TMEM columns)
//   warps 2-17 decoders, four teams of 4 (warp = team x lane quadrant, thread =
//            row; team = K chunk mod 4): slab -> s8 A tile per item; then the
//            unit's epilogue (tcgen05.ld -> z rows, a team per 64 columns)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "device.hpp"
#include "tc05.hpp"

namespace q8p::detail {
namespace {
using namespace tc05;

constexpr int kNT = 256;                              // vectors per N tile (MMA N)
constexpr int kKC = 32;                               // K per pipeline item (one s8 MMA K)
constexpr int kMT = 1;                                // M tiles (128 rows) per CTA (TMEM: 2 limbs x 256 columns)
constexpr std::uint32_t kATile = 128u * kKC;          // 4 KiB per M tile (s8)
constexpr std::uint32_t kABytes = kMT * kATile;
constexpr std::uint32_t kBLimb = kNT * kKC;           // 8 KiB per s8 limb
constexpr std::uint32_t kBBytes = 2u * kBLimb;        // h + l
// A / B pipeline depth.  A team's consecutive items are up to (kTeams - 1) * nst + 1
// apart (nst <= 2: 7); its parity wait on an A slot is only unambiguous when that
// gap is <= kSlots (the slot's previous phase is then known complete).
constexpr std::uint32_t kSlots = 9;
// Code slab ring: a decoder's A-slot wait keeps it within kSlots items of the MMA;
// with kSlots <= 8 nst + 1 (a k slab holds 8 nst items) a decoder entering k slab
// k + 2 implies all of k slab k is done, so at most 2 k slabs x nst stages are in flight.
constexpr std::uint32_t kCodeSlots = 4;
constexpr std::uint32_t kCodeSlot = 4 * 2048 + 512;   // E8P slab bytes (e8-1bit slabs are smaller)
constexpr int kTeams = 4;                             // decoder teams: K chunk kc goes to team kc % 4
constexpr int kDecTeam = 4 * kMT;                     // decoder warps per team: M tiles x 4 lane quadrants
constexpr float kLMax = 32000.f;                      // |L| bound: balanced limbs h, l in [-128, 127]
static_assert((kTeams - 1) * 2 + 1 <= int(kSlots), "A/B ring too shallow for the decoder teams");
static_assert(kSlots <= 8 * 1 + 1 && kCodeSlots >= 2 * 2, "code ring sized for decoders within one k slab of the MMA");
constexpr int kDec = kTeams * kDecTeam;
constexpr int kThreads = (2 + kDec) * 32;
constexpr std::uint32_t kCtl = 1024, kTab = 4096;     // barriers; decode tables
constexpr std::uint32_t kOffA = kCtl + kTab, kOffB = kOffA + kSlots * kABytes, kOffC = kOffB + kSlots * kBBytes;
constexpr std::size_t kSmem = kOffC + kCodeSlots * kCodeSlot;
static_assert(kSmem <= 227 * 1024, "prefill smem");


struct PrefillArgs {
  const std::uint8_t* codes[2];  // tensor-core slabs per stage
  std::uint32_t slab_bytes[2];
  int kind[2];                   // 0 e8p, 1 e8-1bit
  int nst;
  std::uint32_t KSL, KC;         // k slabs (32 codewords), K chunks (32 columns)
  std::uint32_t MT, NTL;         // M tiles (128 rows), N tiles (256 vectors)
  const std::uint8_t* btiles;    // [NTL][KC][nst][kBBytes]
  float* z;                      // [slices][batch][m]: piece k of a tile writes slice k
  K4Sched sched;                 // stream-K schedule (device.hpp)
  std::uint32_t m, batch;
  const std::uint32_t* nib;      // [256] E8P magnitude nibbles
  const uint2* e81;              // [256] e8-1bit doubled rows
  const float* alpha;            // [NTL * 256] per-vector fixed-point scale (pack kernel)
  unsigned long long* trace;     // debug timeline (Q8P_K4_TRACE builds + Q8P_TRACE): CTA 0, nullptr = off
};

// Debug timeline: trace[role][item][8] clock64 stamps of CTA 0 (role 0 MMA issuer,
// 1 producer, 2 + w decoder warp w); compiled in only with -DQ8P_K4_TRACE.
constexpr int kK4TraceItems = 512;
__device__ __forceinline__ void k4_stamp(const PrefillArgs& a, int role, std::uint32_t item, int ev) {
#ifdef Q8P_K4_TRACE
  if (a.trace != nullptr && blockIdx.x == 0 && item < kK4TraceItems && (threadIdx.x & 31) == 0)
    a.trace[(role * kK4TraceItems + item) * 8 + ev] = clock64();
#endif
}

__device__ __forceinline__ std::uint32_t lds32(std::uint32_t addr) {
  std::uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sts128(std::uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t sel) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// 32 lanes x 32 columns of fp32 from tensor memory.
__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, float (&v)[32]) {
  std::uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// s8 bytes of 4 v = 2 sigma d + 2 b - 1 (odd integers in [-11, 11]), looked up by
// PRMT with the nibble sel = m | sigma << 2 (m = 0, 1, 2 for d = 1, 3, 5; the LUT
// nibble XOR the negate flag, as in K2):
//   b = 0:  [01 05 09 _ | FD F9 F5 _]  (1, 5, 9 | -3, -7, -11)
//   b = 1:  [03 07 0B _ | FF FB F7 _]  (3, 7, 11 | -1, -5, -9) = the b = 0 table + 2
//   per byte (no carries).
constexpr std::uint32_t kI8Pos = 0x00090501u, kI8Neg = 0x00F5F9FDu;

// 4 v of one E8P codeword (slot jj of the 4-codeword idx / flag words, shift bit b)
// as 8 s8 (coordinates 0..7).
__device__ __forceinline__ uint2 e8p_s8(std::uint32_t idx, std::uint32_t fw, int jj, std::uint32_t b,
                                        std::uint32_t tab) {
  const std::uint32_t nib = lds32(tab + idx * 4u);
  const std::uint32_t rs = jj == 0 ? fw << 2 : jj == 1 ? fw << 1 : jj == 2 ? fw : fw >> 1;
  const std::uint32_t sel = nib ^ (rs & 0x44444444u);
  const std::uint32_t bb = b * 0x00020202u;
  return make_uint2(prmt(kI8Pos + bb, kI8Neg + bb, sel), prmt(kI8Pos + bb, kI8Neg + bb, sel >> 16));
}
// 4 v = 2 * doubled of an e8-1bit code (bytewise doubling; |doubled| <= 63).
__device__ __forceinline__ uint2 e81_s8(std::uint32_t code, std::uint32_t tab) {
  const std::uint32_t lo = lds32(tab + 1024u + code * 8u), hi = lds32(tab + 1024u + code * 8u + 4u);
  return make_uint2((lo << 1) & 0xFEFEFEFEu, (hi << 1) & 0xFEFEFEFEu);
}

// One item's MMAs: limb h into D (columns d ..), limb l into D + kNT, both with the
// item's A tile; commits free the A and B slots.  Issued by one elected lane of a
// converged warp (one asm block: no per-MMA R2UR waterfall).
__device__ __forceinline__ void mma_s8_item_e(std::uint32_t d, std::uint64_t a_desc, std::uint64_t b_desc,
                                              std::uint32_t idesc, std::uint32_t acc, std::uint32_t bar0,
                                              std::uint32_t bar1) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 b;\n\t.reg .b32 x;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "add.s64 b, %2, %7;\n\tadd.s32 x, %0, %8;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [x], %1, b, %3, p;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t"
      "}\n" ::"r"(d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc), "r"(bar0), "r"(bar1), "n"(kBLimb / 16), "n"(kNT)
      : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) prefill_kernel(PrefillArgs a) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const std::uint32_t sb = smem_u32(smem);
  const std::uint32_t bar_af = sb, bar_ae = sb + 8 * kSlots, bar_bf = sb + 16 * kSlots, bar_be = sb + 24 * kSlots;
  const std::uint32_t bar_cf = sb + 32 * kSlots, bar_ce = bar_cf + 8 * kCodeSlots;
  const std::uint32_t bar_df = bar_ce + 8 * kCodeSlots, bar_de = bar_df + 8, tmem_slot = bar_de + 8;
  const std::uint32_t tab = sb + kCtl;
  const std::uint32_t nst = std::uint32_t(a.nst);
  const std::uint32_t MP = a.sched.MP, KS8 = a.sched.KS8;  // M pairs; k slabs (8 K chunks) per tile
  // Stream-K: this CTA's steps [s_begin, s_end) of the tiles x KS8 k-slab steps; a
  // "unit" = the part of one tile inside that range (tile = nt * MP + mp), its K
  // chunks [kc0, kc1) and its piece index p (z slice).
  const std::uint32_t s_begin = k4_bound(a.sched, blockIdx.x), s_end = k4_bound(a.sched, blockIdx.x + 1);
  struct Unit {
    std::uint32_t nt, mp, p, kc0, kc1;
  };
  auto unit_at = [&](std::uint32_t step) {  // the unit starting at `step` (inside this CTA's range)
    Unit un;
    const std::uint32_t tile = step / KS8;
    const std::uint32_t t0 = tile * KS8;
    un.nt = tile / MP;
    un.mp = tile % MP;
    un.p = blockIdx.x - k4_cta_of(a.sched, t0);
    un.kc0 = (step - t0) * 8;
    un.kc1 = ((s_end < t0 + KS8 ? s_end : t0 + KS8) - t0) * 8;
    return un;
  };
  auto next_step = [&](std::uint32_t step) {  // first step after the unit starting at `step`
    const std::uint32_t t1 = (step / KS8 + 1) * KS8;
    return t1 < s_end ? t1 : s_end;
  };

  if (threadIdx.x == 0) {
    for (std::uint32_t i = 0; i < kSlots; ++i) {
      mbar_init(bar_af + 8 * i, kDecTeam);  // an item is decoded by one team
      mbar_init(bar_ae + 8 * i, 1);
      mbar_init(bar_bf + 8 * i, 1);
      mbar_init(bar_be + 8 * i, 1);
    }
    for (std::uint32_t i = 0; i < kCodeSlots; ++i) {
      mbar_init(bar_cf + 8 * i, 1);
      mbar_init(bar_ce + 8 * i, 4 * kTeams);  // the 4 decoder warps of the slab's M tile, per team
    }
    mbar_init(bar_df, 1);
    mbar_init(bar_de, kDec);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 256; i += kThreads) {  // decode tables (static data)
    reinterpret_cast<std::uint32_t*>(smem + kCtl)[i] = __ldg(a.nib + i);
    reinterpret_cast<uint2*>(smem + kCtl + 1024)[i] = __ldg(a.e81 + i);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tbase = *reinterpret_cast<volatile std::uint32_t*>(smem + (tmem_slot - sb));
  pdl_wait();  // t tiles / z of the previous kernels
  pdl_trigger();

  // code slab c of a unit: k slab ks, stage s, M tile t -> ring index (ks * nst + s) * kMT + t
  if (warp == 0) {
    // ===== producer (the whole warp, converged; elected lanes issue the copies) =====
    {
      std::uint32_t g = 0, cg = 0;  // item / code-slab counters over the CTA's units
      for (std::uint32_t st = s_begin; st < s_end; st = next_step(st)) {
        const Unit un = unit_at(st);
        const std::uint32_t nt = un.nt, mp = un.mp, kc0 = un.kc0, kc1 = un.kc1;
        for (std::uint32_t kc = kc0; kc < kc1; ++kc) {
          if (kc % 8 == 0) {
            for (std::uint32_t s = 0; s < nst; ++s)
              for (std::uint32_t t = 0; t < kMT; ++t, ++cg) {
                const std::uint32_t cs = cg % kCodeSlots, mt = mp * kMT + t;
                if (cg >= kCodeSlots) mbar_wait(bar_ce + 8 * cs, ((cg / kCodeSlots) - 1) & 1);
                const std::uint32_t bytes = s ? a.slab_bytes[1] : a.slab_bytes[0];
                if (mt < a.MT) {
                  mbar_arrive_expect_tx_e(bar_cf + 8 * cs, bytes);
                  bulk_g2s_e(sb + kOffC + cs * kCodeSlot,
                           (s ? a.codes[1] : a.codes[0]) + (std::size_t(mt) * a.KSL + kc / 8) * bytes,
                           bytes, bar_cf + 8 * cs);
                } else {
                  mbar_arrive_e(bar_cf + 8 * cs);  // past the last row block: nothing to load
                }
              }
          }
          for (std::uint32_t s = 0; s < nst; ++s, ++g) {
            const std::uint32_t bs = g % kSlots;
            if (g >= kSlots) mbar_wait(bar_be + 8 * bs, ((g / kSlots) - 1) & 1);
            mbar_arrive_expect_tx_e(bar_bf + 8 * bs, kBBytes);
            bulk_g2s_e(sb + kOffB + bs * kBBytes, a.btiles + ((std::size_t(nt) * a.KC + kc) * nst + s) * kBBytes,
                     kBBytes, bar_bf + 8 * bs);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: per item 2 limbs =====
    // The whole warp runs the loop (converged, uniform operands); one elected lane
    // issues each item's 8 MMAs + 2 commits in a single asm block.  (Issued from a
    // divergent `lane == 0` branch they cost ~100 cycles each: R2UR waterfalls.)
    constexpr std::uint32_t idesc = idesc_i8(128, kNT);
    std::uint32_t g = 0, ul = 0;
    for (std::uint32_t st = s_begin; st < s_end; st = next_step(st), ++ul) {
      if (ul >= 1) mbar_wait(bar_de, (ul - 1) & 1);  // the previous unit's epilogue read the accumulators
      tc_fence_after();
      const Unit un = unit_at(st);
      const std::uint32_t uitems = (un.kc1 - un.kc0) * nst;
      for (std::uint32_t it = 0; it < uitems; ++it, ++g) {
        const std::uint32_t sl = g % kSlots, ph = (g / kSlots) & 1;
        k4_stamp(a, 0, g, 0);
        mbar_wait(bar_af + 8 * sl, ph);
        k4_stamp(a, 0, g, 1);
        mbar_wait(bar_bf + 8 * sl, ph);
        k4_stamp(a, 0, g, 2);
        tc_fence_after();
        const std::uint32_t sa = sb + kOffA + sl * kABytes, sbb = sb + kOffB + sl * kBBytes;
        mma_s8_item_e(tbase, sdesc(sa, 128, 256), sdesc(sbb, 128, 256), idesc, it != 0, bar_ae + 8 * sl,
                      bar_be + 8 * sl);
        k4_stamp(a, 0, g, 3);
      }
      mma_commit_e(bar_df);
    }
  } else {
    // ===== decoders: warp = (M tile t, lane quadrant q), thread = row; then the epilogue =====
    const std::uint32_t q = std::uint32_t(warp & 3), row_in = q * 32 + std::uint32_t(lane);
    const std::uint32_t t = (std::uint32_t(warp - 2) >> 2) % kMT;  // M tile
    const std::uint32_t team = std::uint32_t(warp - 2) / kDecTeam;  // K chunks kc with kc % kTeams == team
    std::uint32_t g = 0, cg = 0, ul = 0;
    const int kind0 = a.kind[0], kind1 = a.kind[1];  // (no runtime indexing of the parameter block)
    // One item = (K chunk kc, stage s): 4 codewords per thread into the item's A slot.
    struct Item {
      std::uint32_t kc, s, cs, cph, sl, g;
    };
    for (std::uint32_t su = s_begin; su < s_end; su = next_step(su), ++ul) {
      const Unit un = unit_at(su);
      const std::uint32_t p = un.p, nt = un.nt, mt = un.mp * kMT + t, kc0 = un.kc0, kc1 = un.kc1;
      const bool live = mt < a.MT;
      const std::uint32_t uitems = (kc1 - kc0) * nst;
      auto item = [&](std::uint32_t i) {
        Item it;
        it.kc = kc0 + (nst == 1 ? i : i >> 1);  // nst in {1, 2}
        it.s = nst == 1 ? 0u : i & 1u;
        const std::uint32_t cidx = cg + ((it.kc - kc0) / 8) * nst * kMT + it.s * kMT + t;
        it.cs = cidx % kCodeSlots;
        it.cph = (cidx / kCodeSlots) & 1;
        it.g = g + i;
        it.sl = it.g % kSlots;
        return it;
      };
      auto wait_item = [&](const Item& it) {
        mbar_wait(bar_cf + 8 * it.cs, it.cph);
        if (it.g >= kSlots) mbar_wait(bar_ae + 8 * it.sl, ((it.g / kSlots) - 1) & 1);
      };
      // decode one item's 4 codewords of this row into s8 A bytes
      auto decode = [&](const Item& it, uint2 (&v)[4]) {
        const std::uint32_t sc = sb + kOffC + it.cs * kCodeSlot, cq = it.kc % 8;
        const std::uint32_t wofs = (cq / 4) * 2048u + row_in * 16u + (cq % 4) * 4u;
        const std::uint32_t iw = lds32(sc + wofs);
        if ((it.s ? kind1 : kind0) == 0) {
          const std::uint32_t fw = lds32(sc + 4096u + wofs), sw = lds32(sc + 8192u + row_in * 4u);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            v[jj] = e8p_s8((iw >> (8 * jj)) & 0xFFu, fw, jj, (sw >> (cq + 8 * jj)) & 1u, tab);
        } else {
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) v[jj] = e81_s8((iw >> (8 * jj)) & 0xFFu, tab);
        }
      };
      // codeword jj = K bytes 8 jj .. 8 jj + 7 of the chunk: K half jj / 2 (16-byte core-matrix rows)
      auto store = [&](const Item& it, const uint2 (&v)[4]) {
        const std::uint32_t sa = sb + kOffA + it.sl * kABytes + t * kATile + (row_in >> 3) * 256u + (row_in & 7) * 16u;
        sts128(sa, make_uint4(v[0].x, v[0].y, v[1].x, v[1].y));
        sts128(sa + 128u, make_uint4(v[2].x, v[2].y, v[3].x, v[3].y));
      };
      auto release = [&](const Item& it) {  // lane 0, after the warp's stores are fenced
        mbar_arrive(bar_af + 8 * it.sl);
        if (it.kc % 8 >= 8 - kTeams) mbar_arrive(bar_ce + 8 * it.cs);  // this team's last chunk of the slab
      };
      // One item at a time per warp, the teams on K chunks kc % kTeams: a single
      // item's chain (slab load -> LUT load -> PRMTs -> stores -> proxy fence) is
      // latency-bound, so the teams keep kTeams items in flight per lane quadrant.
      for (std::uint32_t i = team * nst; i < uitems; i += (i % nst == nst - 1) ? 1 + (kTeams - 1) * nst : 1) {
        const Item it = item(i);
        k4_stamp(a, 2 + warp - 2, it.g, 0);
        wait_item(it);
        k4_stamp(a, 2 + warp - 2, it.g, 2);
        if (live) {
          uint2 v[4];
          decode(it, v);
          store(it, v);
          k4_stamp(a, 2 + warp - 2, it.g, 4);
          fence_proxy_async_smem();  // generic smem writes -> the tensor core's operand reads
        }
        __syncwarp();
        k4_stamp(a, 2 + warp - 2, it.g, 3);
        if (lane == 0) release(it);
      }
      g += uitems;
      cg += ((kc1 - kc0 + 7) / 8) * nst * kMT;
      // epilogue: z[b][r] = alpha_b (256 D_h[r][b] + D_l[r][b]) / 4 for the M tile's
      // 128 rows x 256 vectors
      mbar_wait(bar_df, ul & 1);
      tc_fence_after();
      const std::uint32_t row = mt * 128 + row_in;
      for (std::uint32_t c0 = team * (kNT / kTeams); c0 < (team + 1) * (kNT / kTeams); c0 += 32) {  // team's columns
        float dh[32], dl[32];
        tmem_ld32(tbase + ((q * 32) << 16) + c0, dh);
        tmem_ld32(tbase + ((q * 32) << 16) + kNT + c0, dl);
        if (live && row < a.m) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const std::uint32_t b = nt * kNT + c0 + j;
            if (b < a.batch)
              a.z[(std::size_t(p) * a.batch + b) * a.m + row] =
                  0.25f * __ldg(a.alpha + b) *
                  fmaf(256.f, float(__float_as_int(dh[j])), float(__float_as_int(dl[j])));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_de);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// B tiles from t [batch][n] fp32.  CTA = one vector v of the N tiles (vectors
// beyond batch: zeros, alpha 0): alpha_v = max_s scale_s * max|t_v| / kLMax (max|t_v|
// from K1's pass 2, in amax_alpha[v]), then per (K chunk, stage) the balanced s8
// limbs h, l of L = rint(scale_s t / alpha_v) (L = 256 h + l) in the K-major
// core-matrix layout, 8 bytes per (limb, 8-column group).  alpha replaces the max
// in amax_alpha[v] for the epilogue.
__global__ void __launch_bounds__(256) pack_b_kernel(const float* __restrict__ t, std::uint32_t n,
                                                     std::uint32_t batch, int nst, float s0, float s1,
                                                     std::uint8_t* __restrict__ out, float* __restrict__ amax_alpha) {
  const std::uint32_t v = blockIdx.x, nt = v / kNT, vi = v % kNT, KC = n / kKC, groups = n / 8;
  const bool live = v < batch;
  const float* tv = t + std::size_t(v) * n;
  const float mx = live ? amax_alpha[v] : 0.f;
  const float smax = nst > 1 ? fmaxf(s0, s1) : s0;
  const float al = smax * mx / kLMax, inv = al > 0.f ? 1.f / al : 0.f;
  __syncthreads();  // every thread has read the max before thread 0 overwrites it
  if (threadIdx.x == 0) amax_alpha[v] = al;
  for (std::uint32_t kg = threadIdx.x; kg < groups; kg += blockDim.x) {
    const std::uint32_t kc = kg / 4, j = kg % 4;
    float xv[8];
    if (live) {
      const float4 lo4 = __ldg(reinterpret_cast<const float4*>(tv + 8 * kg));
      const float4 hi4 = __ldg(reinterpret_cast<const float4*>(tv + 8 * kg + 4));
      xv[0] = lo4.x, xv[1] = lo4.y, xv[2] = lo4.z, xv[3] = lo4.w, xv[4] = hi4.x, xv[5] = hi4.y, xv[6] = hi4.z,
      xv[7] = hi4.w;
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) xv[c] = 0.f;
    }
    const std::size_t o = (vi >> 3) * 256 + (j >> 1) * 128 + (vi & 7) * 16 + (j & 1) * 8;
    for (int s = 0; s < nst; ++s) {
      const float sc = s ? s1 : s0;
      std::uint32_t h[2] = {0, 0}, l[2] = {0, 0};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int L = __float2int_rn(sc * xv[c] * inv);  // |L| <= kLMax
        const int lo = ((L + 128) & 255) - 128, hi = (L - lo) >> 8;
        h[c >> 2] |= std::uint32_t(hi & 255) << (8 * (c & 3));
        l[c >> 2] |= std::uint32_t(lo & 255) << (8 * (c & 3));
      }
      std::uint8_t* reg = out + ((std::size_t(nt) * KC + kc) * nst + s) * kBBytes;
      *reinterpret_cast<uint2*>(reg + o) = make_uint2(h[0], h[1]);
      *reinterpret_cast<uint2*>(reg + kBLimb + o) = make_uint2(l[0], l[1]);
    }
  }
}

}  // namespace

bool prefill_supported(const q8p_layer& L, int batch) {
  // whole k slabs of 8 K chunks (both decoder teams have chunks in every slab); rht
  // output side (K3 sums the stream-K pieces; the rfft K3 reads one z array)
  return batch >= kPrefillMinBatch && L.side_u.kind == 0 && L.tc[0].codes != nullptr &&
         (L.num_stages == 1 || L.tc[1].codes != nullptr) &&
         L.n % (8 * kKC) == 0 && L.dec_tables != nullptr;
}

K4Sched prefill_sched(const q8p_layer& L, int batch) {
  K4Sched s;
  s.MP = (tc_row_blocks(L.m_local()) + kMT - 1) / kMT;
  s.NTL = std::uint32_t((batch + kNT - 1) / kNT);
  s.KS8 = (L.n / kKC) / 8;
  s.nt = kNT;
  s.mrows = kMT * 128;
  int sms = 0;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device()), "sm count");
  if (std::uint64_t(s.MP) * s.NTL * s.KS8 * std::uint64_t(sms) >= (1ull << 32))
    throw SizeError("prefill: layer x batch too large for the stream-K schedule");
  s.grid = std::min(std::uint32_t(sms), k4_total(s));
  s.slices = 1;
  for (std::uint32_t tile = 0; tile < s.MP * s.NTL; ++tile) s.slices = std::max(s.slices, k4_pieces(s, tile));
  return s;
}

std::uint32_t prefill_parts(const q8p_layer& L, int batch) { return prefill_sched(L, batch).slices; }

float* prefill_amax(const q8p_layer& L, int batch, std::uint8_t* btiles) {  // after the B tiles
  const std::size_t ntl = (std::size_t(batch) + kNT - 1) / kNT;
  return reinterpret_cast<float*>(btiles + ntl * (L.n / kKC) * std::size_t(L.num_stages) * kBBytes);
}

std::size_t prefill_btile_bytes(const q8p_layer& L, int batch) {  // B tiles, then alpha per vector
  const std::size_t ntl = (std::size_t(batch) + kNT - 1) / kNT;
  return ntl * (L.n / kKC) * std::size_t(L.num_stages) * kBBytes + ntl * kNT * 4;
}

void launch_prefill(const q8p_layer& L, const float* t, std::uint8_t* btiles, float* z, int batch, cudaStream_t s) {
  const std::uint32_t NTL = std::uint32_t((batch + kNT - 1) / kNT);
  float* const alpha = prefill_amax(L, batch, btiles);  // holds K1's max |t| per vector; pack_b makes it alpha
  pack_b_kernel<<<NTL * kNT, 256, 0, s>>>(t, L.n, std::uint32_t(batch), L.num_stages, L.scale[0], L.scale[1], btiles,
                                          alpha);
  cuda_check(cudaGetLastError(), "prefill pack launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  PrefillArgs a{};
  a.nst = L.num_stages;
  for (int st = 0; st < L.num_stages; ++st) {
    a.codes[st] = static_cast<const std::uint8_t*>(L.tc[st].codes);
    a.kind[st] = L.cb[st] == Q8P_CB_E8P_2BIT ? 0 : 1;
    a.slab_bytes[st] = tc_slab_bytes(a.kind[st]);
  }
  a.KSL = tc_k_slabs(L.n);
  a.KC = L.n / kKC;
  if (a.KC % 8 != 0 && a.KC > 8) throw UnsupportedError("prefill: K chunks must fill whole k slabs");
  a.MT = tc_row_blocks(L.m_local());
  a.NTL = NTL;
  a.btiles = btiles;
  a.z = z;
  a.sched = prefill_sched(L, batch);
  a.m = L.m_local();
  a.batch = std::uint32_t(batch);
  a.nib = L.dec_tables;
  a.e81 = reinterpret_cast<const uint2*>(L.dec_tables + 256);
  a.alpha = alpha;
#ifdef Q8P_K4_TRACE
  static const char* trace_env = std::getenv("Q8P_TRACE");
  if (trace_env) {
    constexpr std::size_t words = (2 + kDec) * kK4TraceItems * 8;
    cuda_check(cudaMalloc(&a.trace, words * 8), "trace alloc");
    cuda_check(cudaMemset(a.trace, 0, words * 8), "trace memset");
  }
#endif
  kernel_attrs(reinterpret_cast<const void*>(prefill_kernel), int(kSmem));
  launch_pdl(prefill_kernel, dim3(a.sched.grid), dim3(kThreads), kSmem, s, a);
  cuda_check(cudaGetLastError(), "prefill launch");
#ifdef Q8P_K4_TRACE
  if (a.trace) {
    std::vector<unsigned long long> h((2 + kDec) * kK4TraceItems * 8);
    cuda_check(cudaStreamSynchronize(s), "trace sync");
    cuda_check(cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost), "trace copy");
    cudaFree(a.trace);
    if (FILE* f = std::fopen((std::string(trace_env) + ".k4.bin").c_str(), "wb")) {
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
#endif
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
