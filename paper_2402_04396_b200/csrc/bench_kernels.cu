// Benchmark support (the reference's bm_infer counterpart, bench.cpp:103-120):
// the HBM stream ceiling for a byte range, read the way K2 reads its code slabs
// (one persistent CTA per SM, a contiguous range per CTA, 1-D bulk copies into a
// shared-memory ring completing on mbarriers), so bench.py can report K2's
// time next to the time a pure read of the same bytes takes in the same harness.
#include <cuda_runtime.h>

#include <algorithm>

#include "device.hpp"
#include "tc05.hpp"

namespace q8p::detail {
namespace {
using namespace tc05;

constexpr std::uint32_t kChunk = 16384;  // bytes per bulk copy
constexpr std::uint32_t kSlots = 12;     // ring depth (192 KiB in flight per SM)

__global__ void __launch_bounds__(32, 1) stream_kernel(const std::uint8_t* __restrict__ src, std::size_t bytes,
                                                       unsigned* sink) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  const std::uint32_t sbase = smem_u32(smem), bars = sbase, ring = sbase + 1024;
  const std::size_t chunks = (bytes + kChunk - 1) / kChunk;
  const std::size_t c0 = chunks * blockIdx.x / gridDim.x, c1 = chunks * (blockIdx.x + 1) / gridDim.x;
  pdl_trigger();
  if (threadIdx.x != 0) return;
  for (std::uint32_t i = 0; i < kSlots; ++i) mbar_init(bars + 8 * i, 1);
  fence_mbar_init();
  const std::uint64_t pol = policy_evict_first();
  auto issue = [&](std::size_t c) {
    const std::uint32_t st = std::uint32_t((c - c0) % kSlots);
    const std::size_t off = c * kChunk;
    const std::uint32_t n = std::uint32_t(std::min<std::size_t>(kChunk, bytes - off));
    mbar_arrive_expect_tx(bars + 8 * st, n);
    bulk_g2s_hint(ring + st * kChunk, src + off, n, bars + 8 * st, pol);
  };
  for (std::size_t c = c0; c < c1 && c < c0 + kSlots; ++c) issue(c);
  for (std::size_t c = c0; c < c1; ++c) {
    const std::size_t k = c - c0;
    mbar_wait(bars + 8 * (k % kSlots), std::uint32_t((k / kSlots) & 1));
    if (c + kSlots < c1) issue(c + kSlots);
  }
  if (c1 > c0 && sink != nullptr) *sink = 1u;  // keep the reads observable
}
}  // namespace

void launch_stream(const void* src, std::size_t bytes, unsigned* sink, cudaStream_t s) {
  const std::size_t smem = 1024 + std::size_t(kChunk) * kSlots;
  kernel_attrs(reinterpret_cast<const void*>(stream_kernel), int(smem));
  int sms = 0;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device()), "sm count");
  launch_pdl(stream_kernel, dim3(sms), dim3(32), smem, s, static_cast<const std::uint8_t*>(src), bytes, sink);
  cuda_check(cudaGetLastError(), "stream launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
