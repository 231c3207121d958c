// Microbenchmark: HBM streaming through a per-CTA bulk-copy ring (the K2
// skeleton without decode/MMA): 1 producer warp, C consumer warps that just
// wait + release each slot.  Reports GB/s for a 62.6 MB stream (70B MLP layer
// in the 17-bit tile format), cold L2 (a 512 MB scrub between runs).
//   nvcc -std=c++20 -O3 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2402_04396_b200/csrc tools/ubench_stream.cu -o tools/ubench_stream
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc05.hpp"
using namespace q8p::detail::tc05;

template <int SLOT, int S, int CONS, int NP = 1>
__global__ void __launch_bounds__(32 * (NP + CONS), 1) k_stream(const std::uint8_t* src, std::uint32_t items,
                                                             unsigned long long* sink) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  const std::uint32_t sb = smem_u32(smem);
  const std::uint32_t full = sb, empty = sb + 8 * S, ring = sb + 1024;
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  const std::uint32_t it0 = std::uint32_t((std::uint64_t(items) * blockIdx.x) / gridDim.x);
  const std::uint32_t it1 = std::uint32_t((std::uint64_t(items) * (blockIdx.x + 1)) / gridDim.x);
  const std::uint32_t count = it1 - it0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + 8 * i, 1);
      mbar_init(empty + 8 * i, 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp < NP) {  // NP producer warps, item i issued by warp i % NP
    std::uint32_t st = 0, r = 0;
    for (std::uint32_t i = 0; i < count; ++i) {
      if (int(i % NP) == warp) {
        if (i >= S) mbar_wait(empty + 8 * st, (r & 1) ^ 1);
        mbar_arrive_expect_tx_e(full + 8 * st, SLOT);
        bulk_g2s_e(ring + st * SLOT, src + std::size_t(it0 + i) * SLOT, SLOT, full + 8 * st);
      }
      if (++st == S) st = 0, ++r;
    }
  } else {
    const int cw = warp - NP;
    std::uint32_t acc = 0;
    std::uint32_t st = 0, r = 0;
    for (std::uint32_t i = 0; i < count; ++i) {
      if (int(i % CONS) == cw) {
        mbar_wait(full + 8 * st, r & 1);
        std::uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(ring + st * SLOT + (threadIdx.x & 31) * 4));
        acc += v;
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(empty + 8 * st);
      }
      if (++st == S) st = 0, ++r;
    }
    if (acc == 0x12345679u) sink[0] = acc;
  }
}

__global__ void scrub(uint4* p, std::size_t n) {  // read-only L2 scrub (no dirty lines left behind)
  unsigned x = 0;
  for (std::size_t i = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x; i < n; i += std::size_t(gridDim.x) * blockDim.x)
    x ^= p[i].x;
  if (x == 0x12345679u) p[0].y = x;
}

// cp.async (LDGSTS, 16 B per lane) ring: NP producer warps, item i loaded by warp i % NP,
// completion tracked with cp.async.mbarrier.arrive.noinc (full barrier count 32).
template <int SLOT, int S, int CONS, int NP>
__global__ void __launch_bounds__(32 * (NP + CONS), 1) k_stream_ca(const std::uint8_t* src, std::uint32_t items,
                                                                 unsigned long long* sink) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  const std::uint32_t sb = smem_u32(smem);
  const std::uint32_t full = sb, empty = sb + 8 * S, ring = sb + 1024;
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const std::uint32_t it0 = std::uint32_t((std::uint64_t(items) * blockIdx.x) / gridDim.x);
  const std::uint32_t it1 = std::uint32_t((std::uint64_t(items) * (blockIdx.x + 1)) / gridDim.x);
  const std::uint32_t count = it1 - it0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + 8 * i, 32);
      mbar_init(empty + 8 * i, 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp < NP) {
    std::uint32_t st = 0, r = 0;
    for (std::uint32_t i = 0; i < count; ++i) {
      if (int(i % NP) == warp) {
        if (i >= S) mbar_wait(empty + 8 * st, (r & 1) ^ 1);
        const std::uint8_t* g = src + std::size_t(it0 + i) * SLOT;
        const std::uint32_t d = ring + st * SLOT;
        for (int o = lane * 16; o < SLOT; o += 512)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + o), "l"(g + o) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full + 8 * st) : "memory");
      }
      if (++st == S) st = 0, ++r;
    }
  } else {
    const int cw = warp - NP;
    std::uint32_t acc = 0;
    std::uint32_t st = 0, r = 0;
    for (std::uint32_t i = 0; i < count; ++i) {
      if (int(i % CONS) == cw) {
        mbar_wait(full + 8 * st, r & 1);
        std::uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(ring + st * SLOT + lane * 4));
        acc += v;
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + 8 * st);
      }
      if (++st == S) st = 0, ++r;
    }
    if (acc == 0x12345679u) sink[0] = acc;
  }
}

template <int SLOT, int S, int CONS, int NP>
void run_ca(const std::uint8_t* src, std::size_t bytes, uint4* junk, std::size_t jn, unsigned long long* sink) {
  const std::uint32_t items = std::uint32_t(bytes / SLOT);
  auto k = k_stream_ca<SLOT, S, CONS, NP>;
  const int smem = 1024 + SLOT * S;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int rep = 0; rep < 6; ++rep) {
    scrub<<<592, 512>>>(junk, jn);
    cudaEventRecord(a);
    k<<<148, 32 * (NP + CONS), smem>>>(src, items, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0) best = ms < best ? ms : best;
  }
  printf("cp.async np %d slot %5d x %2d, bytes %zu: best %.2f us (%.0f GB/s) err=%s\n", NP, SLOT, S, bytes, best * 1e3,
         bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

// LDG streaming: each thread reads 16 B vectors, U independent loads in flight.
template <int U>
__global__ void __launch_bounds__(512) k_ldg(const uint4* src, std::size_t n, unsigned long long* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
  std::size_t i = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc.x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) acc.x ^= src[i].x;
  if (acc.x == 0x12345679u) sink[0] = acc.x;
}

template <int U>
void run_ldg(const std::uint8_t* src, std::size_t bytes, uint4* junk, std::size_t jn, unsigned long long* sink, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int rep = 0; rep < 6; ++rep) {
    scrub<<<592, 512>>>(junk, jn);
    cudaEventRecord(a);
    k_ldg<U><<<blocks, 512>>>(reinterpret_cast<const uint4*>(src), bytes / 16, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0) best = ms < best ? ms : best;
  }
  printf("ldg U=%d blocks=%d bytes=%zu: best %.2f us (%.0f GB/s)\n", U, blocks, bytes, best * 1e3, bytes / (best * 1e-3) / 1e9);
}

__global__ void empty_k() {}


template <int SLOT, int S, int CONS, int NP = 1>
void run(const std::uint8_t* src, std::size_t bytes, uint4* junk, std::size_t jn, unsigned long long* sink) {
  const std::uint32_t items = std::uint32_t(bytes / SLOT);
  auto k = k_stream<SLOT, S, CONS, NP>;
  const int smem = 1024 + SLOT * S;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f, sum = 0.f;
  for (int rep = 0; rep < 6; ++rep) {
    scrub<<<592, 512>>>(junk, jn);
    cudaEventRecord(a);
    k<<<148, 32 * (NP + CONS), smem>>>(src, items, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0) {
      best = ms < best ? ms : best;
      sum += ms;
    }
  }
  printf("np %d slot %5d B x %2d stages, %d consumers: best %.2f us (%.0f GB/s), mean %.2f us  err=%s\n", NP, SLOT, S, CONS,
         best * 1e3, items * double(SLOT) / (best * 1e-3) / 1e9, sum / 5 * 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const std::size_t bytes = 62652416;  // 224 row blocks x 32 k slabs x 8704 B  (28672 x 8192, 17-bit tiles)
  std::uint8_t* src;
  cudaMalloc(&src, 2 * bytes + (1 << 20));
  cudaMemset(src, 1, 2 * bytes);
  const std::size_t jn = (512ull << 20) / 16;
  uint4* junk;
  cudaMalloc(&junk, jn * 16);
  unsigned long long* sink;
  cudaMalloc(&sink, 64);
  run<8704, 16, 4>(src, bytes, junk, jn, sink);
  run<8704, 16, 4>(src, bytes * 2, junk, jn, sink);
  run_ldg<4>(src, bytes, junk, jn, sink, 148 * 4);
  run_ldg<4>(src, bytes * 2, junk, jn, sink, 148 * 4);
  run_ca<8704, 16, 4, 1>(src, bytes, junk, jn, sink);
  run_ca<8704, 16, 4, 1>(src, bytes * 2, junk, jn, sink);
  run_ca<8704, 16, 4, 2>(src, bytes, junk, jn, sink);
  run_ca<8704, 16, 4, 2>(src, bytes * 2, junk, jn, sink);
  run_ca<8704, 16, 4, 4>(src, bytes, junk, jn, sink);
  run_ca<8704, 16, 4, 4>(src, bytes * 2, junk, jn, sink);
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    scrub<<<592, 512>>>(junk, jn);
    cudaEventRecord(a);
    empty_k<<<148, 128>>>();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("empty kernel after scrub: %.2f us\n", ms * 1e3);
  }

  return 0;
}
