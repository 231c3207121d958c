// K1 / K3 for the rfft transform (core/src/rfft.cpp:39-71, SideTransform
// kind rfft, transforms.cpp:28-47):
//   apply            c_k = (x[2k] + i x[2k+1]) e^{i theta_k};  X = DFT_M(c) / sqrt(M)
//   apply_transpose  X = IDFT_M(c) (unnormalized);  X_k *= e^{-i theta_k} / sqrt(M)
// with M = n / 2, DFT_M the FFTW_FORWARD transform (exponent -2 pi i jk / M).
//
// Two-pass ("four-step") DFT over M = M1 * M2, input index j = j1 + M1 j2,
// output index k = k2 + M2 k1:
//   X[k2 + M2 k1] = sum_j1 W_M1^{j1 k1} [ W_M^{j1 k2} sum_j2 W_M2^{j2 k2} c[j1 + M1 j2] ]
//   pass 1  CTA = a tile of TJ consecutive j1 (x all j2): phase rotation (apply),
//           length-M2 DFTs, twiddle W_M^{j1 k2} -> mid[k2][j1] (k2-major)
//   pass 2  CTA = R consecutive k2 rows (contiguous in mid) x a range of k1:
//           length-M1 DFTs, 1/sqrt(M), then either the fp32 output (conjugate
//           phases for the transpose) or -- K1 with R = 4, so each k1 gives 4
//           consecutive complex = 8 reals = one codeword -- the integer
//           activations of the tensor-core GEMV (emit_limbs, rht_device.cuh).
// Sub-DFTs are direct sums over an smem tile with twiddles from one M-entry
// table computed on the host in double (W_M^e, e = j k mod M exact in
// integers), so any even n works (n = 11008: M = 5504 = 64 x 86, no
// power-of-two restriction) at O(M (M1 + M2)) fp32 work.  Accuracy ~1e-6
// relative (fp32), the tolerance the parity tests state.
//
// The transform is orthogonal, so K1's activation scale alpha comes from
// |x|_2 exactly as on the rht path (per-tile sums of squares, combined in a
// fixed order by every pass-2 CTA).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "device.hpp"
#include "rht_device.cuh"

namespace q8p::detail {
namespace {

constexpr std::size_t kMaxSmem = 216 * 1024;  // dynamic smem cap (227 KB less static smem)
constexpr int kP1Threads = 256, kP2Threads = 128;

struct RfftArgs {
  std::uint32_t n, M, M1, M2;
  std::uint32_t TJ, tiles1, ks1;  // pass 1: TJ columns j1 per tile, tiles, k2 splits per tile
  std::uint32_t R, groups2, ks2;  // pass 2: R rows k2 per group, groups, k1 splits per group
  const float2* rot;              // [M] e^{i theta_k}
  const float2* tw;               // [M] e^{-2 pi i e / M}
  const float* in;                // [batch][n]
  float2* mid;                    // [batch][M], mid[k2 * M1 + j1]
  float* out;                     // [batch][n] (fp32 output)
  int fwd;                        // 1: apply, 0: apply_transpose
  int limbs;                      // pass 2 emits the GEMV's integer activations (K1)
  RhtArgs k;                      // limb / ssq / zeroing fields (emit_limbs)
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x));
  acc.y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y));
  return acc;
}
__device__ __forceinline__ float2 tw_dir(const RfftArgs& a, std::uint32_t e) {
  float2 w = __ldg(a.tw + e);
  if (!a.fwd) w.y = -w.y;  // backward DFT: exp(+2 pi i e / M)
  return w;
}

// sum_j x[j * stride] W^{j k} (length L, twiddles w[e] = W^e): two interleaved
// accumulators so the dependent complex-FMA chains overlap.
__device__ __forceinline__ float2 dft_sum(const float2* x, std::uint32_t stride, const float2* w, std::uint32_t L,
                                          std::uint32_t k) {
  float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0;
  const std::uint32_t k2 = (2 * k) % L;
  std::uint32_t e0 = 0, e1 = k % L, j = 0;
  for (; j + 1 < L; j += 2) {
    acc0 = cfma(x[j * stride], w[e0], acc0);
    acc1 = cfma(x[(j + 1) * stride], w[e1], acc1);
    e0 += k2;
    if (e0 >= L) e0 -= L;
    e1 += k2;
    if (e1 >= L) e1 -= L;
  }
  if (j < L) acc0 = cfma(x[j * stride], w[e0], acc0);
  return make_float2(acc0.x + acc1.x, acc0.y + acc1.y);
}

// Pass 1.  grid = (tiles1 * ks1 [+ zeroing CTAs], batch).
__global__ void __launch_bounds__(kP1Threads) rfft_pass1(RfftArgs a) {
  extern __shared__ __align__(16) float2 sm[];
  __shared__ float red[32];
  const int b = blockIdx.y;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x >= a.tiles1 * a.ks1) {  // K1 duties: zero the GEMV accumulators / B-image tail
    if (b == 0) {
      const std::size_t nz = gridDim.x - a.tiles1 * a.ks1;
      const std::size_t t0 = (blockIdx.x - a.tiles1 * a.ks1) * std::size_t(blockDim.x) + threadIdx.x;
      if (a.k.zero_ptr)
        for (std::size_t i = t0; i < a.k.zero_words / 4; i += nz * blockDim.x)
          reinterpret_cast<int4*>(a.k.zero_ptr)[i] = make_int4(0, 0, 0, 0);
      if (a.k.zero2_ptr)
        for (std::size_t i = t0; i < a.k.zero2_bytes / 16; i += nz * blockDim.x)
          reinterpret_cast<int4*>(a.k.zero2_ptr)[i] = make_int4(0, 0, 0, 0);
    }
    return;
  }
  if (a.limbs && blockIdx.x == 0 && threadIdx.x == 0) a.k.tl_out[b] = 0;
  const std::uint32_t tile = blockIdx.x / a.ks1, ksp = blockIdx.x - tile * a.ks1;
  const std::uint32_t j10 = tile * a.TJ, cols = min(a.TJ, a.M1 - j10);
  float2* v = sm;                   // [M2][TJ]
  float2* w2 = sm + a.M2 * a.TJ;    // [M2] W_M2^e = W_M^{e M1}
  const float2* x = reinterpret_cast<const float2*>(a.in + (a.in ? std::size_t(b) * a.n : 0));
  float ss = 0.f;
  for (std::uint32_t t = threadIdx.x; t < a.M2 * cols; t += blockDim.x) {
    const std::uint32_t j2 = t / cols, jj = t - j2 * cols, idx = j10 + jj + a.M1 * j2;
    float2 c = a.k.zacc ? combine2(a.k, b, 2 * idx) : __ldcg(x + idx);  // K3: z from the limb accumulators
    ss += c.x * c.x + c.y * c.y;
    if (a.fwd) c = cmul(c, __ldg(a.rot + idx));
    v[j2 * a.TJ + jj] = c;
  }
  for (std::uint32_t e = threadIdx.x; e < a.M2; e += blockDim.x) w2[e] = tw_dir(a, e * a.M1);
  if (a.limbs && ksp == 0) {  // deterministic per-tile sum of squares of x (fixed reduction tree)
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (std::uint32_t w = 0; w < blockDim.x / 32; ++w) t += red[w];
      a.k.ssq[std::size_t(b) * a.tiles1 + tile] = t;
    }
  }
  __syncthreads();
  const std::uint32_t k2a = a.M2 * ksp / a.ks1, k2b = a.M2 * (ksp + 1) / a.ks1;
  const std::uint32_t nout = (k2b - k2a) * cols;
  float2* dst = a.mid + std::size_t(b) * a.M;
  for (std::uint32_t o = threadIdx.x; o < nout; o += blockDim.x) {
    const std::uint32_t k2 = k2a + o / cols, jj = o % cols;
    const float2 acc = dft_sum(v + jj, a.TJ, w2, a.M2, k2);
    dst[std::size_t(k2) * a.M1 + j10 + jj] = cmul(acc, tw_dir(a, (j10 + jj) * k2));  // j1 k2 < M
  }
}

// Pass 2.  grid = (groups2 * ks2, batch).
__global__ void __launch_bounds__(kP2Threads) rfft_pass2(RfftArgs a) {
  extern __shared__ __align__(16) float2 sm[];
  __shared__ long long redl[32];
  __shared__ float s_alpha[2];
  const int b = blockIdx.y;
  pdl_wait();
  pdl_trigger();
  const std::uint32_t grp = blockIdx.x / a.ks2, ksp = blockIdx.x - grp * a.ks2;
  const std::uint32_t k20 = grp * a.R, rows = min(a.R, a.M2 - k20);
  float2* u = sm;                  // [R][M1]
  float2* w1 = sm + a.R * a.M1;    // [M1] W_M1^e = W_M^{e M2}
  const float2* src = a.mid + std::size_t(b) * a.M + std::size_t(k20) * a.M1;
  for (std::uint32_t t = threadIdx.x; t < rows * a.M1; t += blockDim.x) u[t] = __ldcg(src + t);
  for (std::uint32_t e = threadIdx.x; e < a.M1; e += blockDim.x) w1[e] = tw_dir(a, e * a.M2);
  if (a.limbs && threadIdx.x == 0) {
    float ss = 0.f;
    for (std::uint32_t j = 0; j < a.tiles1; ++j) ss += __ldcg(a.k.ssq + std::size_t(b) * a.tiles1 + j);
    const float2 al = alpha_of(ss);
    s_alpha[0] = al.x;
    s_alpha[1] = al.y;
    if (blockIdx.x == 0) a.k.alpha_out[b] = al.x;
  }
  __syncthreads();
  const float sc = rsqrtf(float(a.M));
  const std::uint32_t k1a = a.M1 * ksp / a.ks2, k1b = a.M1 * (ksp + 1) / a.ks2;
  if (a.limbs) {  // R = 4 (M2 % 4 == 0): one codeword per k1
    const float inv = s_alpha[1];
    long long tl = 0;
    for (std::uint32_t k1 = k1a + threadIdx.x; k1 < k1b; k1 += blockDim.x) {
      float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
      std::uint32_t e = 0;  // j1 k1 mod M1
      for (std::uint32_t j1 = 0; j1 < a.M1; ++j1) {
        const float2 w = w1[e];
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r] = cfma(u[r * a.M1 + j1], w, acc[r]);
        e += k1;
        if (e >= a.M1) e -= a.M1;
      }
      const float v[8] = {acc[0].x, acc[0].y, acc[1].x, acc[1].y, acc[2].x, acc[2].y, acc[3].x, acc[3].y};
      const std::uint32_t k = k20 + a.M2 * k1;  // complex index of v[0..1]: codeword 2k / 8
      tl += emit_limbs(a.k, b, k >> 2, v, sc, inv);
    }
    for (int o = 16; o > 0; o >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, o);
    if ((threadIdx.x & 31) == 0) redl[threadIdx.x >> 5] = tl;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (std::uint32_t w = 0; w < blockDim.x / 32; ++w) t += redl[w];
      atomicAdd(reinterpret_cast<unsigned long long*>(a.k.tl_out + b), static_cast<unsigned long long>(t));
    }
    return;
  }
  float2* y = reinterpret_cast<float2*>(a.out + std::size_t(b) * a.n);
  const std::uint32_t nout = (k1b - k1a) * rows;
  for (std::uint32_t o = threadIdx.x; o < nout; o += blockDim.x) {
    const std::uint32_t r = o % rows, k1 = k1a + o / rows;
    float2 acc = dft_sum(u + r * a.M1, 1, w1, a.M1, k1);
    const std::uint32_t k = k20 + r + a.M2 * k1;
    acc = make_float2(acc.x * sc, acc.y * sc);
    if (!a.fwd) {
      float2 c = __ldg(a.rot + k);
      c.y = -c.y;
      acc = cmul(acc, c);
    }
    y[k] = acc;
  }
}

std::size_t smem1_of(std::uint32_t M2, std::uint32_t TJ) { return (std::size_t(M2) * TJ + M2) * 8; }
std::size_t smem2_of(std::uint32_t M1, std::uint32_t R) { return (std::size_t(R) * M1 + M1) * 8; }

void plan(const DevSide& side, RfftArgs& a) {
  a.n = side.n;
  a.M = side.n / 2;
  a.M1 = side.M1;
  a.M2 = side.M2;
  a.rot = side.rot;
  a.tw = side.tw;
  a.TJ = std::min<std::uint32_t>(8, a.M1);
  while (a.TJ > 1 && smem1_of(a.M2, a.TJ) > kMaxSmem) a.TJ /= 2;
  a.tiles1 = (a.M1 + a.TJ - 1) / a.TJ;
  // split the outputs so each pass has >= ~128 CTAs per vector and no CTA does
  // more than ~2^13 complex MACs (latency: the transform is a few us of the step)
  auto split = [](std::uint64_t work, std::uint32_t units, std::uint32_t cap) {
    const std::uint64_t k = std::max<std::uint64_t>((work + 8191) >> 13, (128 + units - 1) / units);
    return std::uint32_t(std::min<std::uint64_t>(cap, std::max<std::uint64_t>(1, k)));
  };
  a.ks1 = split(std::uint64_t(a.M2) * a.M2 * a.TJ, a.tiles1, a.M2);
  a.R = a.M2 % 4 == 0 ? 4 : 1;
  a.groups2 = (a.M2 + a.R - 1) / a.R;
  a.ks2 = split(std::uint64_t(a.R) * a.M1 * a.M1, a.groups2, a.M1);
}

void set_smem_attrs() {
  kernel_attrs(reinterpret_cast<const void*>(rfft_pass1), int(kMaxSmem));
  kernel_attrs(reinterpret_cast<const void*>(rfft_pass2), int(kMaxSmem));
}

void launch_passes(const RfftArgs& a, int batch, std::uint32_t zero_ctas, cudaStream_t s) {
  set_smem_attrs();
  launch_pdl(rfft_pass1, dim3(a.tiles1 * a.ks1 + zero_ctas, batch), dim3(kP1Threads), smem1_of(a.M2, a.TJ), s, a);
  cuda_check(cudaGetLastError(), "rfft pass1 launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(rfft_pass2, dim3(a.groups2 * a.ks2, batch), dim3(kP2Threads), smem2_of(a.M1, a.R), s, a);
  cuda_check(cudaGetLastError(), "rfft pass2 launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace

bool rfft_factor(std::uint32_t n, bool codewords, std::uint32_t& M1, std::uint32_t& M2) {
  if (n == 0 || n % 2 != 0) return false;
  const std::uint32_t M = n / 2;
  const bool need4 = codewords && M % 4 == 0;
  std::uint64_t best = ~0ull;
  for (std::uint32_t d = 1; d <= M; ++d) {  // d = M2
    if (M % d != 0 || (need4 && d % 4 != 0)) continue;
    const std::uint32_t m1 = M / d, r = d % 4 == 0 ? 4 : 1;
    if (smem1_of(d, 1) > kMaxSmem || smem2_of(m1, r) > kMaxSmem) continue;
    const std::uint64_t cost = std::uint64_t(m1) + d;
    if (cost < best) {
      best = cost;
      M1 = m1;
      M2 = d;
    }
  }
  return best != ~0ull;
}

void rfft_tables(std::uint32_t n, const float* phases, std::vector<float>& rot, std::vector<float>& tw) {
  const std::uint32_t M = n / 2;
  rot.resize(2 * std::size_t(M));
  tw.resize(2 * std::size_t(M));
  const double two_pi = 6.283185307179586476925286766559;
  for (std::uint32_t k = 0; k < M; ++k) {
    const double th = double(phases[k]);  // PhaseVector angles are f32-exact (bitpack.cpp:42-53)
    rot[2 * k] = float(std::cos(th));
    rot[2 * k + 1] = float(std::sin(th));
    const double ang = two_pi * double(k) / double(M);
    tw[2 * k] = float(std::cos(ang));
    tw[2 * k + 1] = float(-std::sin(ang));
  }
}

void launch_rfft_f32(const DevSide& side, const float* x, float* u_scratch, float* y, int batch, bool transpose,
                     cudaStream_t s) {
  if (batch <= 0) return;
  RfftArgs a{};
  plan(side, a);
  a.in = x;
  a.mid = reinterpret_cast<float2*>(u_scratch);
  a.out = y;
  a.fwd = transpose ? 0 : 1;
  launch_passes(a, batch, 0, s);
}

void launch_rfft_out_acc(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                         std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                         const long long* tl, float* u_scratch, float* y, int batch, cudaStream_t s) {
  if (batch <= 0) return;
  RfftArgs a{};
  plan(side, a);
  a.in = nullptr;
  a.mid = reinterpret_cast<float2*>(u_scratch);
  a.out = y;
  a.fwd = 0;
  a.k.zacc = zacc;
  a.k.zrows = zacc_rows;
  a.k.zcols = zacc_cols;
  a.k.zstages = zacc_stages;
  a.k.zscale0 = zscale[0];
  a.k.zscale1 = zscale[1];
  a.k.ze8p0 = ze8p[0];
  a.k.ze8p1 = ze8p[1];
  a.k.alpha_in = alpha;
  a.k.tl_in = tl;
  // every k2 split of a tile re-combines the tile from the accumulators (int64 /
  // double arithmetic): keep the splits few
  a.ks1 = std::min<std::uint32_t>(a.ks1, 2);
  launch_passes(a, batch, 0, s);
}

void launch_rfft_in_limbs(const DevSide& side, const float* x, float* u_scratch, float* ssq, float* alpha,
                          long long* tl, std::uint8_t* bimg, std::uint32_t b_bytes, std::uint32_t bcols,
                          std::uint8_t* bimg_tail, std::size_t tail_bytes, std::int32_t* zero_ptr,
                          std::size_t zero_words, int batch, cudaStream_t s) {
  if (batch <= 0) return;
  RfftArgs a{};
  plan(side, a);
  if (a.R != 4) throw SizeError("rfft: K1 needs a factorization with M2 % 4 == 0");
  a.in = x;
  a.mid = reinterpret_cast<float2*>(u_scratch);
  a.fwd = 1;
  a.limbs = 1;
  a.k.ssq = ssq;
  a.k.alpha_out = alpha;
  a.k.tl_out = tl;
  a.k.bimg = bimg;
  a.k.b_bytes = b_bytes;
  a.k.bcols = bcols;
  a.k.zero_ptr = zero_ptr;
  a.k.zero_words = zero_words;
  a.k.zero2_ptr = bimg_tail;
  a.k.zero2_bytes = tail_bytes;
  a.k.batch = batch;
  launch_passes(a, batch, (zero_ptr && zero_words) || (bimg_tail && tail_bytes) ? 32 : 0, s);
}

}  // namespace q8p::detail
