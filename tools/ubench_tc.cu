// Microbenchmark: tcgen05.mma kind::i8 issue/drain rate at small N, A in TMEM
// vs A in smem, and tcgen05.st throughput.  Not part of the product; run with
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2402_04396_b200/csrc tools/ubench_tc.cu -o /tmp/ub && /tmp/ub
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc05.hpp"
using namespace q8p::detail::tc05;

__device__ __forceinline__ std::uint64_t sdesc_ss(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  return sdesc(saddr, lbo, sbo);
}
__device__ __forceinline__ void mma_i8_ts_elect(std::uint32_t d, std::uint32_t a, std::uint64_t b, std::uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void mma_i8_ss(std::uint32_t d, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                          std::uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int N, bool TS, int R = 1, bool WARP = false, int STW = 0, int CPG = 0>
__global__ void __launch_bounds__(128 + 32 * STW, 1) k_mma(int groups, int per_group, unsigned long long* out) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  const std::uint32_t sb = smem_u32(smem);
  const std::uint32_t bar = sb, slot = sb + 8;  // extra barriers at sb + 16 ..
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<std::uint32_t*>(smem + 1024)[i] = 0x01010101u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    for (int c = 0; c < 4; ++c) mbar_init(bar + 16 + 8 * c, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  fence_proxy_async_smem();
  const std::uint32_t tb = *reinterpret_cast<volatile std::uint32_t*>(smem + 8);
  __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp >= 4) {
    // concurrent TMEM writers: x16 stores into columns 128..255 of their lane quadrant
    std::uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * i;
    const std::uint32_t ta = tb + (std::uint32_t((warp & 3) * 32) << 16) + 128;
    int it = 0;
    while (*reinterpret_cast<volatile int*>(&stop) == 0) {
#pragma unroll
      for (int c = 0; c < 8; ++c) tmem_st16(ta + 16 * c, v);
      v[0] += ++it;
    }
    tmem_wait_st();
  }
  if (WARP ? warp == 0 : threadIdx.x == 0) {
    constexpr std::uint32_t idesc = idesc_i8(128, N);
    const std::uint32_t bsm = sb + 1024, asm_ = sb + 1024 + 16384;
    std::uint64_t bd[8], ad[8];
    std::uint32_t dd[8], at[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      bd[k] = sdesc(bsm + k * N * 32, 128, 256);
      ad[k] = sdesc(asm_ + k * 4096, 128, 256);
      dd[k] = tb + 256 + (k % R) * N;
      at[k] = tb + 8 * k;
    }
    std::uint64_t t0 = clock64();
    for (int g = 0; g < groups; ++g) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if constexpr (WARP)
          mma_i8_ts_elect(dd[k], at[k], bd[k], idesc);
        else if constexpr (TS)
          mma_i8_ts(dd[k], at[k], bd[k], idesc, 1);
        else
          mma_i8_ss(dd[k], ad[k], bd[k], idesc, 1);
      }
      for (int c = 0; c < CPG; ++c) mma_commit_e(bar + 16 + 8 * c);
    }
    if (!WARP || (threadIdx.x & 31) == 0) mma_commit(bar);
    mbar_wait(bar, 0);
    std::uint64_t t1 = clock64();
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[0] = t1 - t0;
    if ((threadIdx.x & 31) == 0) atomicExch(&stop, 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

// NI issuer warps, each issuing groups of 9 MMAs (N=8) into its own D with its own A columns.
template <int NI, int FENCE, int STW = 0, int SLEEP = 0, int LDSW = 0, int ALUW = 0>
__global__ void __launch_bounds__(512, 1) k_multi(int groups, unsigned long long* out) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  const std::uint32_t sb = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16 * 1024 / 4; i += blockDim.x) reinterpret_cast<std::uint32_t*>(smem + 1024)[i] = 0x01010101u;
  if (threadIdx.x == 0) {
    for (int c = 0; c < 8; ++c) mbar_init(sb + 16 + 8 * c, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(sb + 8);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  fence_proxy_async_smem();
  const std::uint32_t tb = *reinterpret_cast<volatile std::uint32_t*>(smem + 8);
  __shared__ int stop2;
  if (threadIdx.x == 0) stop2 = 0;
  __syncthreads();
  if (ALUW && warp >= 4 && warp < 4 + ALUW) {  // ALU-heavy decode-like work (PRMT / LOP3 chains)
    std::uint32_t a0 = threadIdx.x, a1 = threadIdx.x * 7u, a2 = 0x00050301u, a3 = 0x00FBFDFFu, acc = 0;
    while (*reinterpret_cast<volatile int*>(&stop2) == 0) {
#pragma unroll 16
      for (int k = 0; k < 64; ++k) {
        std::uint32_t r;
        asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a2), "r"(a3), "r"(a0));
        a0 = (a0 ^ (a1 & 0x44444444u)) + r;
        asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a2), "r"(a3), "r"(a1));
        a1 ^= r;
        acc += r;
      }
    }
    if (acc == 0x12345679u) out[10] = acc;
  }
  if (LDSW && warp >= 4 && warp < 4 + LDSW) {  // LUT-style LDS traffic (lane-replicated rows)
    std::uint32_t acc = threadIdx.x, x = threadIdx.x * 2654435761u;
    const std::uint32_t lut = sb + 1024 + 8192;
    while (*reinterpret_cast<volatile int*>(&stop2) == 0) {
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        x = x * 1664525u + 1013904223u;
        std::uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(lut + ((x >> 24) & 63) * 256 + (threadIdx.x & 31) * 4));
        acc += v;
      }
    }
    if (acc == 0x12345679u) out[9] = acc;
  }
  if (warp >= 4 && warp < 4 + STW) {
    std::uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * i;
    const std::uint32_t ta = tb + (std::uint32_t((warp & 3) * 32) << 16) + 296 + 8 * ((warp >> 2) & 1);
    unsigned long long bytes = 0;
    const std::uint64_t t0 = clock64();
    while (*reinterpret_cast<volatile int*>(&stop2) == 0) {
      for (int c = 0; c < 4; ++c) tmem_st16(ta, v);
      tmem_st8(ta, *reinterpret_cast<std::uint32_t(*)[8]>(v));
      tmem_wait_st();
      bytes += 32 * 72 * 4;
      v[0] += 1;
      if (SLEEP) __nanosleep(SLEEP);
    }
    const std::uint64_t t1 = clock64();
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && warp == 4) out[8] = bytes * 1000 / (t1 - t0);  // per warp B/kcyc
  }
  if (warp < NI) {
    constexpr std::uint32_t idesc = idesc_i8(128, 8);
    const std::uint64_t bd = sdesc(sb + 1024 + warp * 2304, 128, 256);
    const std::uint32_t a = tb + warp * 144, d = tb + 448 + warp * 16;
    std::uint64_t t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (FENCE & 1) tc_fence_after();
      if (FENCE & 2) mbar_wait(sb + 48 + 8 * warp, 1);  // fresh barrier: completes at once
      mma_i8_slab_e<16>(d, a + (g & 1) * 72, bd, idesc, 1, 1, sb + 16 + 8 * warp, sb + 16 + 8 * warp);
    }
    mma_commit_e(sb + 16 + 8 * warp);
    // drain: wait for the final phase parity of this warp's barrier (2 commits/group + 1)
    const std::uint32_t total = 2u * groups + 1u;
    mbar_wait(sb + 16 + 8 * warp, (total - 1) & 1);
    std::uint64_t t1 = clock64();
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[warp] = t1 - t0;
    if ((threadIdx.x & 31) == 0) atomicAdd(&stop2, 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int NI, int FENCE = 0, int STW = 0, int SLEEP = 0, int LDSW = 0, int ALUW = 0>
void run_multi(unsigned long long* d) {
  const int groups = 2000;
  cudaFuncSetAttribute(k_multi<NI, FENCE, STW, SLEEP, LDSW, ALUW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  k_multi<NI, FENCE, STW, SLEEP, LDSW, ALUW><<<148, 128 + 32 * (STW > LDSW ? (STW > ALUW ? STW : ALUW) : (LDSW > ALUW ? LDSW : ALUW)), 32 * 1024>>>(groups, d);
  cudaDeviceSynchronize();
  unsigned long long c[4] = {0, 0, 0, 0};
  cudaMemcpy(c, d, 8 * NI, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < NI; ++i) mx = c[i] > mx ? c[i] : mx;
  unsigned long long sb8 = 0; cudaMemcpy(&sb8, d + 8, 8, cudaMemcpyDeviceToHost);
  printf("multi-issuer aluw=%d ldsw=%d fence=%d NI=%d stw=%d sleep=%d (sttm %.0f B/kcyc/warp): %.1f cyc per 9-MMA group per issuer, %.1f cyc per MMA aggregate (err=%s)\n", ALUW, LDSW, FENCE, NI, STW, SLEEP, double(sb8),
         double(mx) / groups, double(mx) / (groups * 9.0 * NI), cudaGetErrorString(cudaGetLastError()));
}

// 4 warps store x16 columns repeatedly into TMEM.
__global__ void __launch_bounds__(128, 1) k_sttm(int iters, unsigned long long* out) {
  __shared__ std::uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(smem_u32(&slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tb = slot + (std::uint32_t(warp * 32) << 16);
  std::uint32_t v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * i;
  std::uint64_t t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_st16(tb + (it & 3) * 64 + 16 * c, v);
    v[0] += it;
  }
  tmem_wait_st();
  std::uint64_t t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(slot);
  }
}

template <int N, bool TS, int R = 1, bool WARP = false, int STW = 0, int CPG = 0>
void run(unsigned long long* d) {
  const int groups = 2000, per = 8;
  auto k = k_mma<N, TS, R, WARP, STW, CPG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<148, 128 + 32 * STW, 100 * 1024>>>(groups, per, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<148, 128 + 32 * STW, 100 * 1024>>>(groups, per, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("mma i8 M=128 N=%d K=32 R=%d warp=%d stw=%d commits/8=%d %s: %.1f cyc/mma  (%.1f us total, err=%s)\n", N, R, int(WARP), STW, CPG, TS ? "A=TMEM" : "A=SMEM",
         double(c) / (groups * per), ms * 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  run<8, true, 1, true>(d);
  cudaMemset(d, 0, 64 * 8);
  run_multi<3>(d);
  run_multi<3, 0, 0, 0, 0, 4>(d);
  run_multi<3, 0, 0, 0, 0, 12>(d);
  k_sttm<<<148, 128>>>(4000, d);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("sttm x16 (4 warps): %.1f cyc per 4x x16 round => %.1f B/cyc\n", double(c) / 4000,
         4.0 * 4 * 32 * 16 * 4 / (double(c) / 4000));
  return 0;
}
