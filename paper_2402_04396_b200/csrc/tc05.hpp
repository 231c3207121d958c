// Thin PTX wrappers for the sm_100a features the q8p kernels use:
// mbarriers, 1-D bulk async copies (TMA engine), tcgen05 tensor memory
// (alloc / st / ld) and tcgen05.mma kind::i8 / kind::f16.
//
// Descriptor encodings (PTX ISA "tcgen05 instruction descriptor" and
// "shared memory descriptor"), K-major, no swizzle ("interleave"):
//   core matrix = 8 rows x 16 B stored contiguously (128 B);
//   LBO = byte distance between the two 16-B K-chunks of a 32-B K slice,
//   SBO = byte distance between consecutive 8-row groups.
#pragma once

#include <cstdint>

namespace q8p::detail::tc05 {

#ifdef __CUDACC__

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(std::uint32_t bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint32_t bar, std::uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(std::uint32_t bar, std::uint32_t parity) {
  std::uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Spin inside the asm: a C++ retry loop makes the compiler treat everything
// after the wait as potentially divergent (per-lane predicate), which demotes
// uniform values to per-lane registers (R2UR + VOTEU in front of every
// tcgen05 / bulk-copy issue).
__device__ __forceinline__ void mbar_wait(std::uint32_t bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Busy-poll variant (mbarrier.test_wait never suspends the thread).
__device__ __forceinline__ void mbar_wait_poll(std::uint32_t bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "P_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra P_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// ---- bulk async copy global -> shared (completes on an mbarrier) --------------
__device__ __forceinline__ void bulk_g2s(std::uint32_t dst, const void* src, std::uint32_t bytes, std::uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(std::uint32_t dst, const void* src, std::uint32_t bytes, std::uint32_t bar,
                                              std::uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ std::uint64_t policy_evict_first() {
  std::uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ std::uint64_t policy_evict_last() {
  std::uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma operand reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ---- tensor memory ----------------------------------------------------------
template <int kCols>
__device__ __forceinline__ void tmem_alloc(std::uint32_t dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(dst_smem), "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(std::uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// 32 lanes x 32-bit x N columns: thread i of the warp owns lane (base + i).
__device__ __forceinline__ void tmem_st8(std::uint32_t taddr, const std::uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
      "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(std::uint32_t taddr, const std::uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(std::uint32_t taddr, std::uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}

// ---- descriptors ------------------------------------------------------------
// K-major, SWIZZLE_NONE shared-memory matrix descriptor (version 1 = sm_100).
__device__ __forceinline__ std::uint64_t sdesc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  return std::uint64_t((saddr >> 4) & 0x3FFFu) | (std::uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (std::uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (std::uint64_t(1) << 46);
}
#endif  // __CUDACC__

// Instruction descriptor, kind::i8: s8 x s8 -> s32, both K-major.
constexpr std::uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (std::uint32_t(N >> 3) << 17) | (std::uint32_t(M >> 4) << 24);
}
// Instruction descriptor, kind::f16: f16 x f16 -> f32, both K-major.
constexpr std::uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (std::uint32_t(N >> 3) << 17) | (std::uint32_t(M >> 4) << 24);
}

#ifdef __CUDACC__
// D[tmem] (+)= A[tmem] . B[smem]^T ; issued by ONE thread.
__device__ __forceinline__ void mma_i8_ts(std::uint32_t d_tmem, std::uint32_t a_tmem, std::uint64_t b_desc,
                                          std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T ; issued by ONE thread.
__device__ __forceinline__ void mma_f16_ss(std::uint32_t d_tmem, std::uint64_t a_desc, std::uint64_t b_desc,
                                           std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on `bar` once all previously issued tcgen05 async ops of this thread complete.
__device__ __forceinline__ void mma_commit(std::uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
// ---- warp-converged, lane-elected issue -------------------------------------
// Executed by ALL 32 lanes of a converged warp; `elect.sync` picks one lane
// inside the asm.  Issuing tcgen05/bulk-copy instructions from a divergent
// `if (lane == 0)` region makes the compiler wrap each one in a BRA.U.ANY
// waterfall loop (R2UR per operand): measured 44-80 cycles per tcgen05.mma
// vs 14 cycles converged (tools/ubench_tc.cu, B200).
__device__ __forceinline__ void mma_i8_ts_e(std::uint32_t d_tmem, std::uint32_t a_tmem, std::uint64_t b_desc,
                                            std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// One slab of a K-major kind::i8 product, lane-elected once: 8 MMAs walking K
// (A: +8 TMEM columns = 32 B of K, B: +b_step descriptor units of 16 B),
// accumulate predicate on the first, then (when `side`) a 9th MMA with A at
// column 64 and B at 8 * b_step, then two commits.  All in one asm block so
// the issue costs one elect and no per-MMA predicate plumbing.
template <int BStep>
__device__ __forceinline__ void mma_i8_slab_e(std::uint32_t d, std::uint32_t a, std::uint64_t bdesc,
                                              std::uint32_t idesc, std::uint32_t acc, std::uint32_t side,
                                              std::uint32_t bar0, std::uint32_t bar1) {
  asm volatile(
      "{\n\t.reg .pred e, p, q;\n\t.reg .b64 b;\n\t.reg .b32 x;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t"
      "add.s32 x, %1, 8;\n\tadd.s64 b, %2, %8;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [x], b, %3, 1;\n\t"
      "add.s32 x, %1, 16;\n\tadd.s64 b, %2, %9;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [x], b, %3, 1;\n\t"
      "add.s32 x, %1, 24;\n\tadd.s64 b, %2, %10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [x], b, %3, 1;\n\t"
      "add.s32 x, %1, 32;\n\tadd.s64 b, %2, %11;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [x], b, %3, 1;\n\t"
      "add.s32 x, %1, 40;\n\tadd.s64 b, %2, %12;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [x], b, %3, 1;\n\t"
      "add.s32 x, %1, 48;\n\tadd.s64 b, %2, %13;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [x], b, %3, 1;\n\t"
      "add.s32 x, %1, 56;\n\tadd.s64 b, %2, %14;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [x], b, %3, 1;\n\t"
      "add.s32 x, %1, 64;\n\tadd.s64 b, %2, %15;\n\t"
      "and.pred q, q, e;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::i8 [%0], [x], b, %3, 1;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t"
      "}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc), "r"(side), "r"(bar0), "r"(bar1), "n"(1 * BStep), "n"(2 * BStep),
      "n"(3 * BStep), "n"(4 * BStep), "n"(5 * BStep), "n"(6 * BStep), "n"(7 * BStep), "n"(8 * BStep)
      : "memory");
}
__device__ __forceinline__ void mma_commit_e(std::uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_e(std::uint32_t bar, std::uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b64 st;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_e(std::uint32_t dst, const void* src, std::uint32_t bytes, std::uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint_e(std::uint32_t dst, const void* src, std::uint32_t bytes,
                                                std::uint32_t bar, std::uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;\n\t}\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_e(std::uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b64 st;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar)
      : "memory");
}
// One K4 item (gemm_prefill.cu), lane-elected once: for M tiles t = 0, 1, K-blocks
// j = 0, 1 and bf16 terms h = hi, lo, tcgen05.mma kind::f16 into D_t = d + t * DStep
// with A at a_desc + t * AStep + j * AKStep and B at b_desc + j * BKStep + h * BTerm
// (descriptor units of 16 B); the first MMA of each tile accumulates iff `acc`.
// Then two commits.
template <int DStep, int AStep, int AKStep, int BKStep, int BTerm>
__device__ __forceinline__ void mma_f16_item_e(std::uint32_t d, std::uint64_t a_desc, std::uint64_t b_desc,
                                               std::uint32_t idesc, std::uint32_t acc, std::uint32_t bar0,
                                               std::uint32_t bar1) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 a, b;\n\t.reg .b32 x;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      // tile 0
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "add.s64 b, %2, %10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, b, %3, 1;\n\t"
      "add.s64 a, %1, %8;\n\tadd.s64 b, %2, %9;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s64 b, b, %10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"
      // tile 1
      "add.s32 x, %0, %11;\n\tadd.s64 a, %1, %7;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [x], a, %2, %3, p;\n\t"
      "add.s64 b, %2, %10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [x], a, b, %3, 1;\n\t"
      "add.s64 a, a, %8;\n\tadd.s64 b, %2, %9;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [x], a, b, %3, 1;\n\t"
      "add.s64 b, b, %10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [x], a, b, %3, 1;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t"
      "}\n" ::"r"(d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc), "r"(bar0), "r"(bar1), "n"(AStep), "n"(AKStep), "n"(BKStep),
      "n"(BTerm), "n"(DStep)
      : "memory");
}
#endif  // __CUDACC__

}  // namespace q8p::detail::tc05
