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

#include "device.hpp"

namespace q8p::detail {
namespace {

__device__ __forceinline__ void atomic_max_pos(float* addr, float v) {
  // |t| >= 0: IEEE ordering of non-negative floats equals their int ordering.
  atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
}

__device__ __forceinline__ float4 sign4(float4 v, std::uint32_t nib) {
  if (nib & 1) v.x = -v.x;
  if (nib & 2) v.y = -v.y;
  if (nib & 4) v.z = -v.z;
  if (nib & 8) v.w = -v.w;
  return v;
}

// Radix-2^R FWHT pass over index bits [sbit, sbit + R) of the row index of an
// smem matrix with `rows` rows of Q floats (row stride Q): each task loads 2^R
// elements, does R butterfly stages in registers, stores them back.
template <int R, int Q>
__device__ __forceinline__ void fwht_pass(float* s, std::uint32_t rows, std::uint32_t sbit) {
  constexpr int K = 1 << R;
  const std::uint32_t tasks = (rows >> R) * Q;
  const std::uint32_t lowmask = (1u << sbit) - 1;
  for (std::uint32_t t = threadIdx.x; t < tasks; t += blockDim.x) {
    const std::uint32_t b = t % Q, tr = t / Q;
    const std::uint32_t base = ((((tr >> sbit) << (sbit + R)) | (tr & lowmask)) * Q) + b;
    float v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = s[base + ((std::uint32_t(k) << sbit) * Q)];
#pragma unroll
    for (int len = 1; len < K; len <<= 1)
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (!(k & len)) {
          const float x = v[k], y = v[k + len];
          v[k] = x + y;
          v[k + len] = x - y;
        }
#pragma unroll
    for (int k = 0; k < K; ++k) s[base + ((std::uint32_t(k) << sbit) * Q)] = v[k];
  }
  __syncthreads();
}

template <int Q>
__device__ void fwht_rows(float* s, std::uint32_t rows) {
  const std::uint32_t lb = 31 - __clz(rows);
  std::uint32_t b = 0;
  for (; b + 3 <= lb; b += 3) fwht_pass<3, Q>(s, rows, b);
  if (b + 2 <= lb) {
    fwht_pass<2, Q>(s, rows, b);
    b += 2;
  }
  if (b + 1 <= lb) fwht_pass<1, Q>(s, rows, b);
}

struct RhtArgs {
  std::uint32_t n, p, q, P2, P1;
  const std::uint8_t* signs;   // ceil(n/8) bytes, LSB-first, bit set = -1
  const std::int8_t* base;     // q x q (+-1) when q > 1
  const float* in;             // pass 1 fp32 input [batch][n] (or nullptr with zacc)
  const std::int32_t* zacc;    // K3 pass 1: int32 limb accumulators [stage][zcols][zrows]
  std::uint32_t zrows, zcols;
  int zstages;
  int ze8p0, ze8p1;            // K3: stage s is E8P (subtract TL / 4)
  float zscale0, zscale1;      // K3: stage scales
  const float* alpha_in;       // K3: per-vector activation scale
  const long long* tl_in;      // K3: per-vector sum of integer activations
  const float* colsum;         // K1 (fp32 path): base column sums (q floats)
  float* tsum_out;             // K1 (fp32 path): per-vector sum of t
  float* mid;                  // [batch][n] intermediate
  float* out;                  // [batch][n] (fp32 path)
  float* amax_out;             // K1 (fp32 path): per-vector amax
  float* ssq;                  // K1 (limb path): [batch][P1] per-chunk sums of squares of x
  float* alpha_out;            // K1 (limb path): [batch]
  long long* tl_out;           // K1 (limb path): [batch]
  std::uint8_t* bimg;          // K1 (limb path): B images [KSL][9][bcols/8][2][8][16]
  std::uint32_t b_bytes, bcols;
  std::int32_t* zero_ptr;      // K1: accumulators to zero (pass-1 spare CTAs)
  std::size_t zero_words;
  std::uint8_t* zero2_ptr;     // K1: B-image tail to zero
  std::size_t zero2_bytes;
  int batch;
  int fwd;
};

// z rows i..i+3 of vector b from the int32 limb accumulators:
// z = sum_s scale_s alpha (2 Z_s - [E8P] TL) / 4, Z_s = sum_l 128^(3-l) zacc[s][4b + l]
// (exact int64 combine, one double rounding per stage sum, then fp32).  Shared by
// K3 pass 1 and the row-sharded combine kernel so both round identically.
__device__ __forceinline__ float4 combine4(const RhtArgs& a, int b, std::uint32_t i) {
  const double al = double(a.alpha_in[b]) * 0.25;
  const long long tl = a.tl_in[b];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int st = 0; st < a.zstages; ++st) {
    const std::int32_t* z = a.zacc + (std::size_t(st) * a.zcols + 4 * b) * a.zrows + i;
    const int4 v0 = *reinterpret_cast<const int4*>(z);
    const int4 v1 = *reinterpret_cast<const int4*>(z + a.zrows);
    const int4 v2 = *reinterpret_cast<const int4*>(z + 2 * std::size_t(a.zrows));
    const int4 v3 = *reinterpret_cast<const int4*>(z + 3 * std::size_t(a.zrows));
    const long long sub = (st == 0 ? a.ze8p0 : a.ze8p1) ? tl : 0;
    const double c = al * double(st == 0 ? a.zscale0 : a.zscale1);
    auto zt = [&](int x0, int x1, int x2, int x3) {
      const long long Z = ((static_cast<long long>(x0) * 128 + x1) * 128 + x2) * 128 + x3;
      return double(2 * Z - sub) * c;
    };
    acc[0] += zt(v0.x, v1.x, v2.x, v3.x);
    acc[1] += zt(v0.y, v1.y, v2.y, v3.y);
    acc[2] += zt(v0.z, v1.z, v2.z, v3.z);
    acc[3] += zt(v0.w, v1.w, v2.w, v3.w);
  }
  return make_float4(float(acc[0]), float(acc[1]), float(acc[2]), float(acc[3]));
}

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
  const std::uint32_t chunk = a.P2 * Q;  // floats, multiple of 4
  const std::uint32_t e0 = blockIdx.x * chunk;
  float* x = sm1;                         // [P2][Q]
  float* y = sm1 + chunk;                 // base output (Q > 1)
  float* Bs = sm1 + 2 * chunk;            // Q x Q base as float (Q <= 28) / int8 (Q = 172)
  if constexpr (Q > 1) {
    if constexpr (Q <= 28) {
      for (std::uint32_t i = threadIdx.x; i < Q * Q; i += blockDim.x) Bs[i] = float(a.base[i]);
    } else {
      std::int8_t* B8 = reinterpret_cast<std::int8_t*>(Bs);
      for (std::uint32_t i = threadIdx.x; i < Q * Q / 4; i += blockDim.x)
        reinterpret_cast<std::uint32_t*>(B8)[i] = reinterpret_cast<const std::uint32_t*>(a.base)[i];
    }
  }
  // load (float4, contiguous chunk)
  float ss = 0.f;
  for (std::uint32_t v = threadIdx.x; v < chunk / 4; v += blockDim.x) {
    const std::uint32_t i = e0 + 4 * v;
    float4 val;
    if (a.zacc) {
      val = combine4(a, b, i);
    } else {
      val = *reinterpret_cast<const float4*>(a.in + std::size_t(b) * a.n + i);
      ss += val.x * val.x + val.y * val.y + val.z * val.z + val.w * val.w;
      if (a.fwd) val = sign4(val, (a.signs[i >> 3] >> (i & 4)) & 0xFu);
    }
    reinterpret_cast<float4*>(x)[v] = val;
  }
  if (a.ssq) {  // deterministic per-chunk sum of squares (fixed reduction tree)
    __shared__ float red1[kP1Threads / 32];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red1[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < kP1Threads / 32; ++w) t += red1[w];
      a.ssq[std::size_t(b) * a.P1 + blockIdx.x] = t;
    }
  }
  __syncthreads();
  float* cur = x;
  if constexpr (Q > 1) {
    // base along each contiguous q-row: y[r][c] = sum_k B[c][k] x[r][k] (fwd) or B[k][c] (K3)
    for (std::uint32_t e = threadIdx.x; e < chunk; e += blockDim.x) {
      const std::uint32_t r = e / Q, c = e - r * Q;
      const float* xr = x + r * Q;
      float acc = 0.f;
      if constexpr (Q <= 28) {
        if (a.fwd) {
#pragma unroll 4
          for (int k = 0; k < Q; ++k) acc += Bs[c * Q + k] * xr[k];
        } else {
#pragma unroll 4
          for (int k = 0; k < Q; ++k) acc += Bs[k * Q + c] * xr[k];
        }
      } else {
        const std::int8_t* B8 = reinterpret_cast<const std::int8_t*>(Bs);
        if (a.fwd) {
#pragma unroll 4
          for (int k = 0; k < Q; ++k) acc += float(B8[c * Q + k]) * xr[k];
        } else {
#pragma unroll 4
          for (int k = 0; k < Q; ++k) acc += float(B8[k * Q + c]) * xr[k];
        }
      }
      y[e] = acc;
    }
    __syncthreads();
    cur = y;
  }
  fwht_rows<Q>(cur, a.P2);
  for (std::uint32_t v = threadIdx.x; v < chunk / 4; v += blockDim.x)
    *reinterpret_cast<float4*>(a.mid + std::size_t(b) * a.n + e0 + 4 * v) = reinterpret_cast<float4*>(cur)[v];
}

// Pass 2.  grid = (P2 * q / 4 column groups, batch); block = 128 threads.
__global__ void __launch_bounds__(128) rht_pass2(RhtArgs a) {
  extern __shared__ __align__(16) float sm2[];
  __shared__ float red[4];
  const int b = blockIdx.y;
  pdl_wait();
  pdl_trigger();
  const std::uint32_t stride = a.P2 * a.q;          // elements between consecutive a_hi
  const std::uint32_t col = blockIdx.x * 4;         // 4 adjacent columns
  for (std::uint32_t r = threadIdx.x; r < a.P1; r += blockDim.x)
    reinterpret_cast<float4*>(sm2)[r] =
        *reinterpret_cast<const float4*>(a.mid + std::size_t(b) * a.n + std::size_t(r) * stride + col);
  __syncthreads();
  fwht_rows<4>(sm2, a.P1);
  const float sc = rsqrtf(float(a.n));
  float mx = 0.f;
  for (std::uint32_t r = threadIdx.x; r < a.P1; r += blockDim.x) {
    const std::uint32_t i = r * stride + col;
    float4 v = reinterpret_cast<float4*>(sm2)[r];
    v = make_float4(v.x * sc, v.y * sc, v.z * sc, v.w * sc);
    if (!a.fwd) v = sign4(v, (a.signs[i >> 3] >> (i & 4)) & 0xFu);
    *reinterpret_cast<float4*>(a.out + std::size_t(b) * a.n + i) = v;
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  if (a.fwd && a.amax_out) {
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      const float m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
      atomic_max_pos(a.amax_out + b, m);
    }
  }
}

// Pass 2 of K1, limb flavour: grid = (P2 * q / 8 codeword columns, batch).
// Each CTA owns 8 adjacent flat columns = one codeword per a_hi row: FWHT over
// a_hi, 1/sqrt(n), then the integer activations of the tensor-core GEMV
// (gemv_tc.cu): Lt = rint(t / alpha) with alpha = the power of two >=
// |x|_2 / kLtMax (|t_i| <= |t|_2 = |x|_2, so no clamping is ever active),
// four balanced base-128 int8 limbs per value (28-bit activations), the block term
// q_k = floor(sum_c Lt / 8) for the side MMA, and TL = sum_i Lt_i.
constexpr int kLtMax = 266338304;  // 127 * 128^3

// Balanced base-128 digits: v in [-kLtMax, kLtMax] -> l0 in [-127, 127], l1..l3 in [-64, 64].
__device__ __forceinline__ void limbs4(int v, int (&l)[4]) {
  l[0] = (v + (1 << 20)) >> 21;
  int rem = v - (l[0] << 21);
  l[1] = (rem + (1 << 13)) >> 14;
  rem -= l[1] << 14;
  l[2] = (rem + 64) >> 7;
  l[3] = rem - (l[2] << 7);
}

__global__ void __launch_bounds__(128) rht_pass2_limbs(RhtArgs a) {
  extern __shared__ __align__(16) float sm2[];
  __shared__ long long red[4];
  __shared__ float s_alpha[2];
  const int b = blockIdx.y;
  pdl_wait();
  pdl_trigger();
  const std::uint32_t stride = a.P2 * a.q;  // elements between consecutive a_hi
  const std::uint32_t col = blockIdx.x * 8;
  for (std::uint32_t r = threadIdx.x; r < 2 * a.P1; r += blockDim.x)
    reinterpret_cast<float4*>(sm2)[r] = *reinterpret_cast<const float4*>(
        a.mid + std::size_t(b) * a.n + std::size_t(r >> 1) * stride + col + 4 * (r & 1));
  if (threadIdx.x == 0) {
    float ss = 0.f;
    for (std::uint32_t j = 0; j < a.P1; ++j) ss += a.ssq[std::size_t(b) * a.P1 + j];
    const float v = sqrtf(ss) * (1.0f + 1.0f / 1024.f) / float(kLtMax);
    int e = 0;
    if (v > 0.f) frexpf(v, &e);
    s_alpha[0] = v > 0.f ? ldexpf(1.f, e) : 1.f;
    s_alpha[1] = v > 0.f ? ldexpf(1.f, -e) : 1.f;
    if (blockIdx.x == 0) a.alpha_out[b] = s_alpha[0];
  }
  __syncthreads();
  fwht_rows<8>(sm2, a.P1);
  const float sc = rsqrtf(float(a.n)), inv = s_alpha[1];
  long long tl = 0;
  const std::uint32_t N = a.bcols;
  for (std::uint32_t r = threadIdx.x; r < a.P1; r += blockDim.x) {
    const std::uint32_t k = (r * stride + col) >> 3;  // codeword index
    const float* v = sm2 + r * 8;
    int lt[8];
    long long S = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float t = rintf(v[c] * sc * inv);
      t = fminf(fmaxf(t, -float(kLtMax)), float(kLtMax));
      lt[c] = int(t);
      S += lt[c];
    }
    tl += S;
    const int qk = int(S >> 3);  // floor(S / 8)
    std::uint32_t w[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      int l[4];
      limbs4(lt[c], l);
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i][c >> 2] |= (std::uint32_t(l[i]) & 0xFFu) << (8 * (c & 3));
    }
    int ql[4];
    limbs4(qk, ql);
    const std::uint32_t ks = k >> 5, j = k & 31, kb = j >> 2;
    std::uint8_t* slab = a.bimg + std::size_t(ks) * a.b_bytes;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const std::uint32_t row = 4 * b + l;
      const std::uint32_t rowoff = (row >> 3) * 256 + (row & 7) * 16;
      // main: K-block kb, K bytes 8 (j % 4) .. +7 -> chunk (j % 4) / 2, offset 8 (j % 2)
      *reinterpret_cast<uint2*>(slab + kb * N * 32 + rowoff + ((j & 3) >> 1) * 128 + (j & 1) * 8) =
          make_uint2(w[l][0], w[l][1]);
      // side: K-block 8, K byte j
      slab[8 * N * 32 + rowoff + (j >> 4) * 128 + (j & 15)] = std::uint8_t(ql[l]);
    }
  }
  for (int o = 16; o > 0; o >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = tl;
  __syncthreads();
  if (threadIdx.x == 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(a.tl_out + b),
              static_cast<unsigned long long>(red[0] + red[1] + red[2] + red[3]));
}

void plan_split(const DevSide& side, RhtArgs& a) {
  a.n = side.n;
  a.p = side.p;
  a.q = side.q;
  // pass-1 chunk P2 * q: ~1K floats (<= 512 for the order-172 base, whose
  // dense product dominates pass 1)
  const std::uint32_t target = side.q > 28 ? 512 : 1024;
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
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(rht_pass1<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024),
               "rht smem attr");
    cuda_check(cudaFuncSetAttribute(rht_pass1<Q>, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
  });
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
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(rht_pass2, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024),
               "rht smem attr");
    cuda_check(cudaFuncSetAttribute(rht_pass2, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
  });
  launch_pdl(rht_pass2, dim3(groups, a.batch), dim3(128), std::size_t(a.P1) * 16, s, a);
  cuda_check(cudaGetLastError(), "rht pass2 launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_pass2_limbs(const RhtArgs& a, cudaStream_t s) {
  const std::uint32_t chunk = a.P2 * a.q;
  if (chunk % 8 != 0) throw SizeError("rht: chunk not a multiple of the codeword dimension");
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(rht_pass2_limbs, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024),
               "rht smem attr");
    cuda_check(cudaFuncSetAttribute(rht_pass2_limbs, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
  });
  launch_pdl(rht_pass2_limbs, dim3(chunk / 8, a.batch), dim3(128), std::size_t(a.P1) * 32, s, a);
  cuda_check(cudaGetLastError(), "rht pass2 limbs launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace

void launch_rht_in(const DevSide& side, const float* x, float* t, float* u_scratch, float* amax, float* tsum,
                   std::int32_t* zero_ptr, std::size_t zero_words, int batch, cudaStream_t s) {
  if (batch <= 0) return;
  RhtArgs a{};
  plan_split(side, a);
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
  RhtArgs a{};
  plan_split(side, a);
  a.signs = side.signs;
  a.base = side.base;
  a.in = zin;
  a.mid = u_scratch;
  a.out = y;
  a.batch = batch;
  a.fwd = 0;
  launch_pass1(a, 0, s);
  launch_pass2(a, s);
}

void launch_rht_in_limbs(const DevSide& side, const float* x, float* u_scratch, float* ssq, float* alpha,
                         long long* tl, std::uint8_t* bimg, std::uint32_t b_bytes, std::uint32_t bcols,
                         std::uint8_t* bimg_tail, std::size_t tail_bytes, std::int32_t* zero_ptr,
                         std::size_t zero_words, int batch, cudaStream_t s) {
  if (batch <= 0) return;
  RhtArgs a{};
  plan_split(side, a);
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
  launch_pass1(a, 32, s);
  launch_pass2_limbs(a, s);
}

void launch_rht_out_acc(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                        std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                        const long long* tl, float* u_scratch, float* y, int batch, cudaStream_t s) {
  if (batch <= 0) return;
  RhtArgs a{};
  plan_split(side, a);
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
  launch_pdl(combine_kernel, dim3(std::min<std::uint32_t>((quads + 255) / 256, 148), batch), dim3(256), 0, s, a, z,
             m_local);
  cuda_check(cudaGetLastError(), "combine launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace q8p::detail
