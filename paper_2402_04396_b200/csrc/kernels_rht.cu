// K1 / K3: randomized Hadamard transforms around the tensor-core GEMV.
//
// SideTransform (core/src/transforms.cpp:28-47) with had_apply
// (core/src/hadamard.cpp:170-210):  H = (H_p (x) B_q) / sqrt(n), flat index
// i = a * q + b.  Split a = a_hi * P2 + a_lo.  The Kronecker factors act on
// different index digits and commute, so each side is two passes, each one
// kernel over many small CTAs (a 1-CTA transform of a 32-112 KB vector is
// latency-bound at several microseconds on B200):
//   pass 1  CTA = one contiguous chunk [a_hi][0..P2)[0..q):
//           signs (fwd) | int32-limb -> fp32 (K3), base B_q (or B_q^T) on each
//           q-row, FWHT over a_lo (stride q)
//   pass 2  CTA = 4 adjacent columns (a_lo, b) x all P1 = p / P2 values of a_hi:
//           FWHT over a_hi, 1/sqrt(n), signs (K3) / amax of t (K1)
// K1 also zeroes the GEMV's int32 accumulators; K3 consumes them.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "device.hpp"
#include "rht_device.cuh"

namespace q8p::detail {
namespace {

// Row-sharded forward: this rank's z rows [0, m_local) as fp32 [batch][m_local]
// (all-gathered by the caller), same arithmetic as K3 pass 1.
__global__ void __launch_bounds__(256) combine_kernel(RhtArgs a, float* z, std::uint32_t m_local) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  for (std::uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; 4 * v < m_local; v += gridDim.x * blockDim.x) {
    const float4 r = combine4(a, b, 4 * v);
    float* o = z + std::size_t(b) * m_local + 4 * v;
    if (4 * v + 4 <= m_local && (m_local & 3) == 0) {
      *reinterpret_cast<float4*>(o) = r;
    } else {
      const float rv[4] = {r.x, r.y, r.z, r.w};
      for (int k = 0; k < 4 && 4 * v + k < m_local; ++k) o[k] = rv[k];
    }
  }
}

constexpr int kP1Threads = 256;

// Pass 1.  grid = (P1 chunks [+ zeroing CTAs], batch).
template <int Q>
__global__ void __launch_bounds__(kP1Threads) rht_pass1(RhtArgs a) {
  extern __shared__ __align__(16) float sm1[];
  const int b = blockIdx.y;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x >= a.P1) {
    if (b == 0) {
      const std::size_t nz = gridDim.x - a.P1;
      const std::size_t t0 = (blockIdx.x - a.P1) * std::size_t(blockDim.x) + threadIdx.x;
      if (a.zero_ptr) {
        int4* zp = reinterpret_cast<int4*>(a.zero_ptr);
        for (std::size_t i = t0; i < a.zero_words / 4; i += nz * blockDim.x) zp[i] = make_int4(0, 0, 0, 0);
      }
      if (a.zero2_ptr) {
        int4* zp = reinterpret_cast<int4*>(a.zero2_ptr);
        for (std::size_t i = t0; i < a.zero2_bytes / 16; i += nz * blockDim.x) zp[i] = make_int4(0, 0, 0, 0);
      }
    }
    return;
  }
  if (a.fwd && blockIdx.x == 0) {
    if (a.amax_out && threadIdx.x == 0) a.amax_out[b] = 0.f;
    if (a.tl_out && threadIdx.x == 0) a.tl_out[b] = 0;
    // sum_i t_i = (p / sqrt(n)) sum_{b' < q} colsum[b'] s_b' x_b'  (Sylvester columns sum to p * delta)
    if (a.tsum_out && threadIdx.x == 32) {
      float acc = 0.f;
      for (std::uint32_t j = 0; j < Q; ++j) {
        float v = a.in[std::size_t(b) * a.n + j];
        if ((a.signs[j >> 3] >> (j & 7)) & 1) v = -v;
        acc += a.colsum[j] * v;
      }
      a.tsum_out[b] = acc * float(a.p) * rsqrtf(float(a.n));
    }
  }
  __shared__ float red1[32];
  rht_p1_body<Q>(a, blockIdx.x, b, sm1, red1, block_team());
}

// Pass 2.  grid = (P2 * q / 4 column groups, batch); block = 128 threads.
__global__ void __launch_bounds__(128) rht_pass2(RhtArgs a) {
  extern __shared__ __align__(16) float sm2[];
  __shared__ float red[32];
  pdl_wait();
  pdl_trigger();
  rht_p2_body(a, blockIdx.x, blockIdx.y, sm2, red, block_team());
}

// Pass 2 of K1, limb flavour: grid = (P2 * q / 8 codeword columns, batch).
// Each CTA owns 8 adjacent flat columns = one codeword per a_hi row: FWHT over
// a_hi, 1/sqrt(n), then the integer activations of the tensor-core GEMV
// (gemv_tc.cu): Lt = rint(t / alpha) with alpha = the power of two >=
// |x|_2 / kActMax (|t_i| <= |t|_2 = |x|_2, so no clamping is ever active),
// four balanced base-128 int8 limbs per value (25-bit activations), the exact
// block sums S_k = sum_c Lt for the side MMA, and TL = sum_i Lt_i.
__global__ void __launch_bounds__(128) rht_pass2_limbs(RhtArgs a) {
  extern __shared__ __align__(16) float sm2[];
  __shared__ long long redl[32];
  __shared__ float s_alpha[2];
  pdl_wait();
  pdl_trigger();
  rht_p2_limbs_body(a, blockIdx.x, blockIdx.y, sm2, redl, s_alpha, block_team());
}


// ---------------------------------------------------------------------------
// Single-kernel cluster RHT (replaces pass1 + pass2 on the tensor-core path).
// One thread-block cluster of C CTAs per vector (grid = (C, batch [+ zeroing])):
//   CTA c loads the contiguous chunk of rows a in [c p/C, (c+1) p/C)
//   (n/C floats: signs | limb-accumulator combine), applies the base B_q
//   (B_q^T for K3) along each q-row, FWHT over the local a bits, then the
//   chunks are transposed through distributed shared memory: CTA c takes
//   columns [c W, (c+1) W) (W = n/C^2) of every source CTA, FWHT over the
//   log2(C) cluster bits, and writes its part of the result.
// Same H = (H_p (x) B_q) / sqrt(n) as had_apply (hadamard.cpp:170-210); the
// butterflies are split differently from pass1/pass2, so fp32 rounding (not
// the math) differs.  Smem per CTA is 2 n/C floats, small enough to co-reside
// with the GEMV's CTAs under programmatic dependent launch.
enum RhtMode { kK1Limbs = 0, kK3Acc = 1, kK3F32 = 2 };
constexpr int kClThreads = 256;
constexpr int kClMaxJ = 16;  // base-product outputs per thread (n/C <= 4096)

__device__ __forceinline__ std::uint32_t cluster_ctarank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(const float* local_ptr, std::uint32_t cta) {
  std::uint32_t a = static_cast<std::uint32_t>(__cvta_generic_to_shared(local_ptr)), r;
  float v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(r));
  return v;
}
__device__ __forceinline__ float4 ld_dsmem_f32x4(const float* local_ptr, std::uint32_t cta) {
  std::uint32_t a = static_cast<std::uint32_t>(__cvta_generic_to_shared(local_ptr)), r;
  float4 v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(r));
  return v;
}

template <int Q, int MODE>
__global__ void __launch_bounds__(kClThreads) rht_cluster(RhtArgs a, std::uint32_t C) {
  extern __shared__ __align__(16) float smc[];
  __shared__ float s_ss;
  __shared__ long long s_tl;
  __shared__ float red_f[kClThreads / 32];
  __shared__ long long red_l[kClThreads / 32];
  const int b = blockIdx.y;
  const std::uint32_t c = cluster_ctarank();
  pdl_wait();
  pdl_trigger();
  if (b >= a.batch) {  // K1: zero the GEMV accumulators / B-image tail (one cluster row)
    if constexpr (MODE == kK1Limbs) {
      const std::size_t nz = std::size_t(gridDim.x) * (gridDim.y - a.batch) * blockDim.x;
      const std::size_t t0 = (std::size_t(b - a.batch) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
      if (a.zero_ptr)
        for (std::size_t i = t0; i < a.zero_words / 4; i += nz)
          reinterpret_cast<int4*>(a.zero_ptr)[i] = make_int4(0, 0, 0, 0);
      if (a.zero2_ptr)
        for (std::size_t i = t0; i < a.zero2_bytes / 16; i += nz)
          reinterpret_cast<int4*>(a.zero2_ptr)[i] = make_int4(0, 0, 0, 0);
    }
    return;
  }
  const std::uint32_t n = a.n, chunk = n / C, P = a.p / C, W = chunk / C;
  const std::uint32_t e0 = c * chunk;
  float* x = smc;              // [P][Q] local chunk
  float* T = smc + chunk;      // [C][W] gathered columns
  float* Bs = smc + 2 * chunk; // base (float for Q <= 28, int8 for 172)
  if constexpr (Q > 1) {
    if constexpr (Q <= 28) {
      for (std::uint32_t i = threadIdx.x; i < Q * Q; i += blockDim.x) Bs[i] = float(a.base[i]);
    } else {
      for (std::uint32_t i = threadIdx.x; i < Q * Q / 4; i += blockDim.x)
        reinterpret_cast<std::uint32_t*>(Bs)[i] = reinterpret_cast<const std::uint32_t*>(a.base)[i];
    }
  }
  float ss = 0.f;
  for (std::uint32_t v = threadIdx.x; v < chunk / 4; v += blockDim.x) {
    const std::uint32_t i = e0 + 4 * v;
    float4 val;
    if constexpr (MODE == kK3Acc) {
      val = combine4(a, b, i);
    } else {
      val = *reinterpret_cast<const float4*>(a.in + std::size_t(b) * n + i);
      if constexpr (MODE == kK1Limbs) {
        ss += val.x * val.x + val.y * val.y + val.z * val.z + val.w * val.w;
        val = sign4(val, (a.signs[i >> 3] >> (i & 4)) & 0xFu);
      }
    }
    reinterpret_cast<float4*>(x)[v] = val;
  }
  if constexpr (MODE == kK1Limbs) {  // deterministic CTA partial of |x|^2 (fixed tree)
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red_f[threadIdx.x >> 5] = ss;
  }
  __syncthreads();
  if constexpr (MODE == kK1Limbs) {
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < kClThreads / 32; ++w) t += red_f[w];
      s_ss = t;
    }
  }
  if constexpr (Q > 1) {
    // base along each q-row, two-phase through registers (in place)
    float outv[kClMaxJ];
#pragma unroll
    for (int j = 0; j < kClMaxJ; ++j) {
      const std::uint32_t e = threadIdx.x + j * kClThreads;
      if (e < chunk) {
        const std::uint32_t r = e / Q, cc = e - r * Q;
        const float* xr = x + r * Q;
        float acc = 0.f;
        if constexpr (Q <= 28) {
          if constexpr (MODE == kK1Limbs) {
#pragma unroll 4
            for (int k = 0; k < Q; ++k) acc += Bs[cc * Q + k] * xr[k];
          } else {
#pragma unroll 4
            for (int k = 0; k < Q; ++k) acc += Bs[k * Q + cc] * xr[k];
          }
        } else {
          const std::int8_t* B8 = reinterpret_cast<const std::int8_t*>(Bs);
          if constexpr (MODE == kK1Limbs) {
#pragma unroll 4
            for (int k = 0; k < Q; ++k) acc += float(B8[cc * Q + k]) * xr[k];
          } else {
#pragma unroll 4
            for (int k = 0; k < Q; ++k) acc += float(B8[k * Q + cc]) * xr[k];
          }
        }
        outv[j] = acc;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kClMaxJ; ++j) {
      const std::uint32_t e = threadIdx.x + j * kClThreads;
      if (e < chunk) x[e] = outv[j];
    }
    __syncthreads();
  }
  fwht_rows<Q>(x, P, block_team());  // local a bits (ends with __syncthreads)
  // -------- cluster transpose + FWHT over the C cluster bits --------
  const float* res;    // this CTA's results: [C][W] with flat index s * chunk + c * W + w
  std::uint32_t rstride;
  if (C > 1) {
    cluster_sync_all();  // every chunk is final and visible cluster-wide
    for (std::uint32_t v = threadIdx.x; v < C * W / 4; v += blockDim.x) {
      const std::uint32_t src = (4 * v) / W, w = (4 * v) - src * W;
      reinterpret_cast<float4*>(T)[v] = ld_dsmem_f32x4(x + c * W + w, src);
    }
    __syncthreads();
    for (std::uint32_t len = 1; len < C; len <<= 1) {  // radix-2 over the source-CTA index
      for (std::uint32_t t = threadIdx.x; t < (C / 2) * W; t += blockDim.x) {
        const std::uint32_t w = t % W, pr = t / W;
        const std::uint32_t lo = ((pr / len) * 2 * len) + (pr % len), hi = lo + len;
        const float u = T[lo * W + w], v2 = T[hi * W + w];
        T[lo * W + w] = u + v2;
        T[hi * W + w] = u - v2;
      }
      __syncthreads();
    }
    res = T;
    rstride = W;
  } else {
    res = x;
    rstride = chunk;
  }
  const float sc = rsqrtf(float(n));
  if constexpr (MODE == kK1Limbs) {
    // alpha: power of two >= |x|_2 / kLtMax from the cluster's |x|^2 partials (fixed order)
    float ssum = 0.f;
    if (C > 1) {
      for (std::uint32_t r = 0; r < C; ++r) ssum += ld_dsmem_f32(&s_ss, r);
    } else {
      ssum = s_ss;
    }
    const float vv = sqrtf(ssum) * (1.0f + 1.0f / 1024.f) / float(kActMax);
    int ex = 0;
    if (vv > 0.f) frexpf(vv, &ex);
    const float alpha = vv > 0.f ? ldexpf(1.f, ex) : 1.f, inv = vv > 0.f ? ldexpf(1.f, -ex) : 1.f;
    if (c == 0 && threadIdx.x == 0) a.alpha_out[b] = alpha;
    long long tl = 0;
    const std::uint32_t N = a.bcols, cw_per_row = rstride / 8, ncw = (C > 1 ? C : 1) * cw_per_row;
    for (std::uint32_t t = threadIdx.x; t < ncw; t += blockDim.x) {
      const std::uint32_t srow = t / cw_per_row, wc = (t - srow * cw_per_row) * 8;
      const float* v = res + srow * rstride + wc;
      const std::uint32_t flat = C > 1 ? srow * chunk + c * W + wc : e0 + wc;
      const std::uint32_t k = flat >> 3;  // codeword index
      int lt[8];
      long long S = 0;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        float tt = rintf(v[cc] * sc * inv);
        tt = fminf(fmaxf(tt, -float(kActMax)), float(kActMax));
        lt[cc] = int(tt);
        S += lt[cc];
      }
      tl += S;
      const int qk = int(S);  // exact block sum
      std::uint32_t wv[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        int l[4];
        limbs4(lt[cc], l);
#pragma unroll
        for (int i = 0; i < 4; ++i) wv[i][cc >> 2] |= (std::uint32_t(l[i]) & 0xFFu) << (8 * (cc & 3));
      }
      int ql[4];
      limbs4(qk, ql);
      const std::uint32_t ks = k >> 5, j = k & 31, kb = j >> 2;
      std::uint8_t* slab = a.bimg + std::size_t(ks) * a.b_bytes;
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const std::uint32_t row = 4 * b + l;
        const std::uint32_t rowoff = (row >> 3) * 256 + (row & 7) * 16;
        *reinterpret_cast<uint2*>(slab + kb * N * 32 + rowoff + ((j & 3) >> 1) * 128 + (j & 1) * 8) =
            make_uint2(wv[l][0], wv[l][1]);
        slab[8 * N * 32 + rowoff + (j >> 4) * 128 + (j & 15)] = std::uint8_t(ql[l]);
      }
    }
    for (int o = 16; o > 0; o >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, o);
    if ((threadIdx.x & 31) == 0) red_l[threadIdx.x >> 5] = tl;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int w = 0; w < kClThreads / 32; ++w) t += red_l[w];
      s_tl = t;
    }
    if (C > 1) {
      cluster_sync_all();  // partial TLs visible; no CTA leaves while its smem is read
      if (c == 0 && threadIdx.x == 0) {
        long long t = 0;
        for (std::uint32_t r = 0; r < C; ++r) {
          std::uint32_t aa = static_cast<std::uint32_t>(__cvta_generic_to_shared(&s_tl)), rr;
          long long v;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rr) : "r"(aa), "r"(r));
          asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(rr));
          t += v;
        }
        a.tl_out[b] = t;
      }
      cluster_sync_all();
    } else {
      __syncthreads();
      if (threadIdx.x == 0) a.tl_out[b] = s_tl;
    }
  } else {
    // K3: y_i = s_i (H^T z)_i / sqrt(n)
    for (std::uint32_t t = threadIdx.x; t < (C > 1 ? C : 1) * rstride; t += blockDim.x) {
      const std::uint32_t srow = t / rstride, w = t - srow * rstride;
      const std::uint32_t flat = C > 1 ? srow * chunk + c * W + w : e0 + w;
      float v = res[srow * rstride + w] * sc;
      if ((a.signs[flat >> 3] >> (flat & 7)) & 1) v = -v;
      a.out[std::size_t(b) * n + flat] = v;
    }
    if (C > 1) cluster_sync_all();  // no CTA leaves while its smem may still be read
  }
}

// Cluster size for the single-kernel RHT: the largest C in {8, 4, 2, 1} with
// C | p, (n / C^2) % 8 == 0 (codewords stay within one CTA's column block) and
// n / C <= 4096 (register budget of the base product); 0 = unsupported.
std::uint32_t cluster_size_for(const DevSide& side) {
  // experiment knob: Q8P_RHT_MAXC=0 -> two-pass RHT, else the largest cluster size tried
  static const int maxc = [] {
    const char* e = std::getenv("Q8P_RHT_MAXC");
    return e ? std::atoi(e) : 0;  // default: two-pass (measured faster in the pipeline)
  }();
  if (maxc <= 0) return 0;
  for (std::uint32_t C = std::uint32_t(maxc); C >= 1; C >>= 1) {
    if (side.p % C) continue;
    const std::uint32_t chunk = side.n / C;
    if (chunk > 4096 || chunk % 4) continue;
    if (C > 1 && (chunk % C || (chunk / C) % 8)) continue;
    if (C == 1 && chunk % 8) continue;
    if ((side.q > 1) && chunk > kClThreads * kClMaxJ) continue;
    return C;
  }
  return 0;
}

template <int Q, int MODE>
void launch_cluster_q(const RhtArgs& a, std::uint32_t C, std::uint32_t zero_rows, cudaStream_t s) {
  const std::size_t chunk = a.n / C;
  const std::size_t bsz = Q == 1 ? 0 : (Q <= 28 ? Q * Q * 4 : (Q * Q + 15) / 16 * 16);
  const std::size_t smem = 2 * chunk * 4 + bsz;
  kernel_attrs(reinterpret_cast<const void*>(rht_cluster<Q, MODE>), 96 * 1024, true);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C, a.batch + zero_rows);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool no_pdl = std::getenv("Q8P_RHT_CLUSTER_NOPDL") != nullptr;  // experiment knob
  cfg.numAttrs = no_pdl ? 1 : 2;
  cuda_check(cudaLaunchKernelEx(&cfg, rht_cluster<Q, MODE>, a, C), "rht cluster launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

template <int MODE>
void launch_cluster(const RhtArgs& a, std::uint32_t C, std::uint32_t zero_rows, cudaStream_t s) {
  switch (a.q) {
    case 1: launch_cluster_q<1, MODE>(a, C, zero_rows, s); break;
    case 4: launch_cluster_q<4, MODE>(a, C, zero_rows, s); break;
    case 12: launch_cluster_q<12, MODE>(a, C, zero_rows, s); break;
    case 20: launch_cluster_q<20, MODE>(a, C, zero_rows, s); break;
    case 28: launch_cluster_q<28, MODE>(a, C, zero_rows, s); break;
    case 172: launch_cluster_q<172, MODE>(a, C, zero_rows, s); break;
    default: throw SizeError("rht: unsupported base order");
  }
}


// ---------------------------------------------------------------------------
// Single-CTA RHT for power-of-two n <= kSingleMaxN (q = 1): one 1024-thread CTA
// per vector holds the whole vector in smem: load (signs | limb combine), all
// log2(n) FWHT stages, then the limb B images (K1) or y (K3) straight from
// smem -- one launch and one global round trip instead of two passes.
constexpr std::uint32_t kSingleMaxN = 8192;
enum SingleMode { kSingleK1 = 0, kSingleK3Acc = 1, kSingleK3F32 = 2 };

template <int MODE>
__global__ void __launch_bounds__(1024) rht_single(RhtArgs a) {
  extern __shared__ __align__(16) float sx[];
  __shared__ float red[32];
  __shared__ long long redl[32];
  __shared__ float s_ss;
  const int b = blockIdx.x;
  pdl_wait();
  pdl_trigger();
  if (b >= a.batch) {  // K1: zero the GEMV accumulators / ragged B-image tail
    if constexpr (MODE == kSingleK1) {
      const std::size_t nz = std::size_t(gridDim.x - a.batch) * blockDim.x;
      const std::size_t t0 = std::size_t(b - a.batch) * blockDim.x + threadIdx.x;
      if (a.zero_ptr)
        for (std::size_t i = t0; i < a.zero_words / 4; i += nz)
          reinterpret_cast<int4*>(a.zero_ptr)[i] = make_int4(0, 0, 0, 0);
      if (a.zero2_ptr)
        for (std::size_t i = t0; i < a.zero2_bytes / 16; i += nz)
          reinterpret_cast<int4*>(a.zero2_ptr)[i] = make_int4(0, 0, 0, 0);
    }
    return;
  }
  const Team tm = block_team();
  const std::uint32_t n = a.n;
  float ss = 0.f;
  for (std::uint32_t v = threadIdx.x; v < n / 4; v += blockDim.x) {
    const std::uint32_t i = 4 * v;
    float4 val;
    if constexpr (MODE == kSingleK3Acc) {
      val = combine4(a, b, i);
    } else {
      val = *reinterpret_cast<const float4*>(a.in + std::size_t(b) * n + i);
      if constexpr (MODE == kSingleK1) {
        ss += val.x * val.x + val.y * val.y + val.z * val.z + val.w * val.w;
        val = sign4(val, (a.signs[i >> 3] >> (i & 4)) & 0xFu);
      }
    }
    reinterpret_cast<float4*>(sx)[v] = val;
  }
  if constexpr (MODE == kSingleK1) {
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  }
  __syncthreads();
  if constexpr (MODE == kSingleK1) {
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (std::uint32_t w = 0; w < blockDim.x / 32; ++w) t += red[w];
      s_ss = t;
    }
  }
  fwht_rows<1>(sx, n, tm);  // all log2(n) stages (ends with __syncthreads)
  const float sc = rsqrtf(float(n));
  if constexpr (MODE == kSingleK1) {
    const float2 al = alpha_of(s_ss);
    if (threadIdx.x == 0) a.alpha_out[b] = al.x;
    long long tl = 0;
    for (std::uint32_t k = threadIdx.x; k < n / 8; k += blockDim.x) tl += emit_limbs(a, b, k, sx + 8 * k, sc, al.y);
    for (int o = 16; o > 0; o >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, o);
    if ((threadIdx.x & 31) == 0) redl[threadIdx.x >> 5] = tl;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (std::uint32_t w = 0; w < blockDim.x / 32; ++w) t += redl[w];
      a.tl_out[b] = t;
    }
  } else {
    for (std::uint32_t v = threadIdx.x; v < n / 4; v += blockDim.x) {
      const std::uint32_t i = 4 * v;
      float4 val = reinterpret_cast<const float4*>(sx)[v];
      val = make_float4(val.x * sc, val.y * sc, val.z * sc, val.w * sc);
      val = sign4(val, (a.signs[i >> 3] >> (i & 4)) & 0xFu);
      *reinterpret_cast<float4*>(a.out + std::size_t(b) * n + i) = val;
    }
  }
}

bool single_ok(const DevSide& side) {
  // experiment knob (Q8P_RHT_SINGLE=1): correct, but one SM doing all log2(n)
  // stages is issue-bound (~750 instructions per warp, ~3 us even at full issue)
  // and slower in the pipeline than the two passes
  static const bool on = std::getenv("Q8P_RHT_SINGLE") != nullptr;
  return on && side.q == 1 && side.n <= kSingleMaxN && side.n % 8 == 0;
}

template <int MODE>
void launch_single(const RhtArgs& a, std::uint32_t zero_ctas, cudaStream_t s) {
  kernel_attrs(reinterpret_cast<const void*>(rht_single<MODE>), int(kSingleMaxN * 4));
  launch_pdl(rht_single<MODE>, dim3(a.batch + zero_ctas), dim3(1024), std::size_t(a.n) * 4, s, a);
  cuda_check(cudaGetLastError(), "rht single launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void plan_split_impl(const DevSide& side, RhtArgs& a) {
  a.n = side.n;
  a.p = side.p;
  a.q = side.q;
  // pass-1 chunk P2 * q: ~1K floats (<= 512 for the order-172 base, whose
  // dense product dominates pass 1)
  static const std::uint32_t tune = [] {  // experiment knob: pass-1 chunk target (floats)
    const char* e = std::getenv("Q8P_RHT_CHUNK");
    return e ? std::uint32_t(std::atoi(e)) : 0u;
  }();
  const std::uint32_t target = tune ? tune : 512;  // 512 measured best for the step (1024: +3 %)
  std::uint32_t P2 = 1;
  while (P2 * 2 <= side.p && P2 * 2 * side.q <= target) P2 *= 2;
  if ((P2 * side.q) % 4 != 0) throw SizeError("rht: dimension too small for the float4 passes");
  a.P2 = P2;
  a.P1 = side.p / P2;
  if (std::size_t(a.P1) * 16 > 96 * 1024) throw SizeError("rht: dimension too large");
}

template <int Q>
void launch_pass1_q(const RhtArgs& a, std::uint32_t extra_ctas, cudaStream_t s) {
  const std::size_t chunk = std::size_t(a.P2) * Q;
  const std::size_t bsz = Q == 1 ? 0 : (Q <= 28 ? Q * Q * 4 : (Q * Q + 15) / 16 * 16);
  const std::size_t smem = chunk * 4 * (Q > 1 ? 2 : 1) + bsz;
  kernel_attrs(reinterpret_cast<const void*>(rht_pass1<Q>), 96 * 1024);
  launch_pdl(rht_pass1<Q>, dim3(a.P1 + extra_ctas, a.batch), dim3(kP1Threads), smem, s, a);
}

void launch_pass1(const RhtArgs& a, std::uint32_t extra, cudaStream_t s) {
  switch (a.q) {
    case 1: launch_pass1_q<1>(a, extra, s); break;
    case 4: launch_pass1_q<4>(a, extra, s); break;
    case 12: launch_pass1_q<12>(a, extra, s); break;
    case 20: launch_pass1_q<20>(a, extra, s); break;
    case 28: launch_pass1_q<28>(a, extra, s); break;
    case 172: launch_pass1_q<172>(a, extra, s); break;
    default: throw SizeError("rht: unsupported base order");
  }
  cuda_check(cudaGetLastError(), "rht pass1 launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_pass2(const RhtArgs& a, cudaStream_t s) {
  const std::uint32_t groups = a.P2 * a.q / 4;
  kernel_attrs(reinterpret_cast<const void*>(rht_pass2), 96 * 1024);
  launch_pdl(rht_pass2, dim3(groups, a.batch), dim3(128), std::size_t(a.P1) * 16, s, a);
  cuda_check(cudaGetLastError(), "rht pass2 launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_pass2_limbs(const RhtArgs& a, cudaStream_t s) {
  const std::uint32_t chunk = a.P2 * a.q;
  if (chunk % 8 != 0) throw SizeError("rht: chunk not a multiple of the codeword dimension");
  kernel_attrs(reinterpret_cast<const void*>(rht_pass2_limbs), 96 * 1024);
  launch_pdl(rht_pass2_limbs, dim3(chunk / 8, a.batch), dim3(128), std::size_t(a.P1) * 32, s, a);
  cuda_check(cudaGetLastError(), "rht pass2 limbs launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace

void rht_plan_split(const DevSide& side, RhtArgs& a) { plan_split_impl(side, a); }
std::size_t rht_p1_smem_bytes(const DevSide& side) {
  RhtArgs a{};
  plan_split_impl(side, a);
  switch (side.q) {
    case 1: return p1_smem_bytes<1>(a.P2);
    case 4: return p1_smem_bytes<4>(a.P2);
    case 12: return p1_smem_bytes<12>(a.P2);
    case 20: return p1_smem_bytes<20>(a.P2);
    case 28: return p1_smem_bytes<28>(a.P2);
    case 172: return p1_smem_bytes<172>(a.P2);
    default: throw SizeError("rht: unsupported base order");
  }
}
std::size_t rht_p2_smem_bytes(const DevSide& side) {
  RhtArgs a{};
  plan_split_impl(side, a);
  return std::size_t(a.P1) * 32;
}

void launch_rht_in(const DevSide& side, const float* x, float* t, float* u_scratch, float* amax, float* tsum,
                   std::int32_t* zero_ptr, std::size_t zero_words, int batch, cudaStream_t s) {
  if (batch <= 0) return;
  if (side.kind == 1) {
    if (amax || tsum) throw UnsupportedError("rfft: amax / tsum outputs are rht-only");
    launch_rfft_f32(side, x, u_scratch, t, batch, false, s);
    return;
  }
  RhtArgs a{};
  plan_split_impl(side, a);
  a.signs = side.signs;
  a.base = side.base;
  a.in = x;
  a.mid = u_scratch;
  a.out = t;
  a.amax_out = amax;
  a.tsum_out = tsum;
  a.colsum = side.colsum;
  a.zero_ptr = zero_ptr;
  a.zero_words = zero_words;
  a.batch = batch;
  a.fwd = 1;
  launch_pass1(a, zero_ptr && zero_words ? 32 : 0, s);
  launch_pass2(a, s);
}

void launch_rht_out(const DevSide& side, const float* zin, float* u_scratch, float* y, int batch, cudaStream_t s) {
  if (batch <= 0) return;
  if (side.kind == 1) {
    launch_rfft_f32(side, zin, u_scratch, y, batch, true, s);
    return;
  }
  RhtArgs a{};
  plan_split_impl(side, a);
  a.signs = side.signs;
  a.base = side.base;
  a.in = zin;
  a.mid = u_scratch;
  a.out = y;
  a.batch = batch;
  a.fwd = 0;
  if (single_ok(side)) {
    launch_single<kSingleK3F32>(a, 0, s);
    return;
  }
  if (const std::uint32_t C = cluster_size_for(side)) {
    launch_cluster<kK3F32>(a, C, 0, s);
    return;
  }
  launch_pass1(a, 0, s);
  launch_pass2(a, s);
}

void launch_rht_in_limbs(const DevSide& side, const float* x, float* u_scratch, float* ssq, float* alpha,
                         long long* tl, std::uint8_t* bimg, std::uint32_t b_bytes, std::uint32_t bcols,
                         std::uint8_t* bimg_tail, std::size_t tail_bytes, std::int32_t* zero_ptr,
                         std::size_t zero_words, int batch, cudaStream_t s, std::uint32_t chunk_vec,
                         std::size_t chunk_bytes) {
  if (batch <= 0) return;
  if (side.kind == 1) {
    if (chunk_vec) throw UnsupportedError("rfft: multi-chunk K1");
    launch_rfft_in_limbs(side, x, u_scratch, ssq, alpha, tl, bimg, b_bytes, bcols, bimg_tail, tail_bytes, zero_ptr,
                         zero_words, batch, s);
    return;
  }
  RhtArgs a{};
  plan_split_impl(side, a);
  a.signs = side.signs;
  a.base = side.base;
  a.in = x;
  a.mid = u_scratch;
  a.ssq = ssq;
  a.alpha_out = alpha;
  a.tl_out = tl;
  a.bimg = bimg;
  a.b_bytes = b_bytes;
  a.bcols = bcols;
  a.zero_ptr = zero_ptr;
  a.zero_words = zero_words;
  a.zero2_ptr = bimg_tail;
  a.zero2_bytes = tail_bytes;
  a.batch = batch;
  a.fwd = 1;
  a.chunk_vec = chunk_vec;
  a.chunk_bytes = chunk_bytes;
  if (single_ok(side)) {
    launch_single<kSingleK1>(a, (zero_ptr && zero_words) || (bimg_tail && tail_bytes) ? 16 : 0, s);
    return;
  }
  if (const std::uint32_t C = cluster_size_for(side)) {
    launch_cluster<kK1Limbs>(a, C, (zero_ptr && zero_words) || (bimg_tail && tail_bytes) ? 4 : 0, s);
    return;
  }
  launch_pass1(a, 32, s);
  launch_pass2_limbs(a, s);
}

void launch_rht_out_acc(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                        std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                        const long long* tl, float* u_scratch, float* y, int batch, cudaStream_t s,
                        bool zero_after) {
  if (batch <= 0) return;
  if (side.kind == 1) {  // rfft: pass 1 combines z from the accumulators itself
    launch_rfft_out_acc(side, zacc, zacc_stages, zacc_rows, zacc_cols, zscale, ze8p, alpha, tl, u_scratch, y, batch,
                        s);
    return;
  }
  RhtArgs a{};
  plan_split_impl(side, a);
  a.signs = side.signs;
  a.base = side.base;
  a.zacc = zacc;
  a.zrows = zacc_rows;
  a.zcols = zacc_cols;
  a.zstages = zacc_stages;
  a.zscale0 = zscale[0];
  a.zscale1 = zscale[1];
  a.ze8p0 = ze8p[0];
  a.ze8p1 = ze8p[1];
  a.alpha_in = alpha;
  a.tl_in = tl;
  a.mid = u_scratch;
  a.out = y;
  a.batch = batch;
  a.fwd = 0;
  a.zacc_zero = zero_after ? 1 : 0;
  if (zero_after) {  // the two-pass kernels clear what they read
    if (side.kind == 1) throw UnsupportedError("rfft: zero-after K3");
    launch_pass1(a, 0, s);
    launch_pass2(a, s);
    return;
  }
  if (single_ok(side)) {
    launch_single<kSingleK3Acc>(a, 0, s);
    return;
  }
  if (const std::uint32_t C = cluster_size_for(side)) {
    launch_cluster<kK3Acc>(a, C, 0, s);
    return;
  }
  launch_pass1(a, 0, s);
  launch_pass2(a, s);
}

void launch_combine_acc(const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows, std::uint32_t zacc_cols,
                        const float zscale[2], const int ze8p[2], const float* alpha, const long long* tl, float* z,
                        std::uint32_t m_local, int batch, cudaStream_t s) {
  if (batch <= 0 || m_local == 0) return;
  RhtArgs a{};
  a.zacc = zacc;
  a.zrows = zacc_rows;
  a.zcols = zacc_cols;
  a.zstages = zacc_stages;
  a.zscale0 = zscale[0];
  a.zscale1 = zscale[1];
  a.ze8p0 = ze8p[0];
  a.ze8p1 = ze8p[1];
  a.alpha_in = alpha;
  a.tl_in = tl;
  const std::uint32_t quads = (m_local + 3) / 4;
  kernel_attrs(reinterpret_cast<const void*>(combine_kernel), 0);
  launch_pdl(combine_kernel, dim3(std::min<std::uint32_t>((quads + 255) / 256, 148), batch), dim3(256), 0, s, a, z,
             m_local);
  cuda_check(cudaGetLastError(), "combine launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
