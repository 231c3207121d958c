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

// Pass 1.  grid = (P1 chunks [+ zeroing CTAs], batch / vpb).  kWarp: one vector
// per warp (prefill batches, a.warp_teams), else the whole CTA on one vector
// (compile-time, so each flavour's barriers and loops specialise).
template <int Q, bool kWarp>
__global__ void __launch_bounds__(kP1Threads) rht_pass1(RhtArgs a) {
  extern __shared__ __align__(16) float sm1[];
  pdl_wait();
  pdl_trigger();
  // push all-gather: this call's tag (the previous call's pass 2 finished before our predecessors)
  const std::uint32_t ll_tag = a.push.ctl ? std::uint32_t(ld_epoch(a.push.ctl) + 1) : 0u;
  const std::uint32_t nch = a.p1_count ? a.p1_count : a.P1;  // chunk CTAs (this rank's, when sharded)
  if (blockIdx.x >= nch) {
    if (blockIdx.y == 0) {
      const std::size_t nz = gridDim.x - nch;
      const std::size_t t0 = (blockIdx.x - nch) * std::size_t(blockDim.x) + threadIdx.x;
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
  __shared__ float red1[32];
  __shared__ int s_pieces[kP1Tiles];
  float* const Bs = sm1;
  if (a.in_sched) p1_tile_pieces(a, a.ch0 + blockIdx.x, a.P2 * Q, int(blockIdx.y) * (a.vpb > 1 ? a.vpb : 1), s_pieces);
  if constexpr (kWarp) {  // shared by the CTA's warp teams: once, up front (else the body loads it)
    p1_load_base<Q>(a, Bs);
    __syncthreads();
  } else {
    if (a.in_sched) __syncthreads();
  }
  // vectors blockIdx.y * vpb .. : large batches amortise the CTA over several vectors,
  // one per warp so a pass's barriers are warp-local
  const Team tm = kWarp ? warp_team() : block_team();
  const int team = kWarp ? int(threadIdx.x >> 5) : 0, teams = kWarp ? int(blockDim.x >> 5) : 1;
  float* const xs = sm1 + p1_base_bytes<Q>() / 4 + std::size_t(team) * (p1_team_bytes<Q>(a.P2) / 4);
  const int vpb = a.vpb > 1 ? a.vpb : 1, b_end = min(a.batch, int(blockIdx.y + 1) * vpb);
  for (int b = int(blockIdx.y) * vpb + team; b < b_end; b += teams) {
    if (a.fwd && blockIdx.x == 0) {
      if (a.amax_out && tm.tid == 0) a.amax_out[b] = 0.f;
      if (a.tl_out && tm.tid == 0) a.tl_out[b] = 0;
      // sum_i t_i = (p / sqrt(n)) sum_{b' < q} colsum[b'] s_b' x_b'  (Sylvester columns sum to p * delta)
      if (a.tsum_out && tm.tid == (tm.warp ? 1u : 32u)) {
        float acc = 0.f;
        for (std::uint32_t j = 0; j < Q; ++j) {
          float v = a.in[std::size_t(b) * a.n + j];
          if ((a.signs[j >> 3] >> (j & 7)) & 1) v = -v;
          acc += a.colsum[j] * v;
        }
        a.tsum_out[b] = acc * float(a.p) * rsqrtf(float(a.n));
      }
    }
    rht_p1_body<Q>(a, a.ch0 + blockIdx.x, b, xs, Bs, red1, tm, ll_tag, s_pieces);
  }
}

// Pass 2.  grid = (P2 * q / 4 column groups, batch / vpb); block = 128 threads,
// or one warp per vector (warp_teams).  kPush: the push all-gather's flavour
// (its own instantiation, so the polling path costs the plain one nothing).
template <bool kPush>
__global__ void __launch_bounds__(256) rht_pass2(RhtArgs a) {
  extern __shared__ __align__(16) float sm2[];
  __shared__ float red[32];
  pdl_wait();
  pdl_trigger();
  const Team tm = a.warp_teams ? warp_team() : block_team();
  const int team = a.warp_teams ? int(threadIdx.x >> 5) : 0, teams = a.warp_teams ? int(blockDim.x >> 5) : 1;
  float* const s = sm2 + std::size_t(team) * a.P1 * 4;
  const int vpb = a.vpb > 1 ? a.vpb : 1, b_end = min(a.batch, int(blockIdx.y + 1) * vpb);
  if constexpr (kPush) {  // push all-gather: read this call's window as its tagged words arrive
    // (the epoch was advanced by the previous call's pass 2, complete before our predecessors ran)
    const unsigned long long e = ld_epoch(a.push.ctl);
    const unsigned long long* const win = a.push.self_win + (e & 1) * a.push.win_words;
    for (int b = int(blockIdx.y) * vpb + team; b < b_end; b += teams)
      rht_p2_body(a, blockIdx.x, b, s, red, tm, win, std::uint32_t(e + 1));
    push_done(a, e);
  } else {
    for (int b = int(blockIdx.y) * vpb + team; b < b_end; b += teams) rht_p2_body(a, blockIdx.x, b, s, red, tm);
  }
}

// Pass 2 for prefill batches (P1 <= 64): one warp per (vector, 32 adjacent flat
// columns), lane = column, the FWHT over a_hi entirely in registers -- every row
// is one coalesced 128 B segment and there is no shared memory or barrier.  Same
// butterfly order as fwht_rows (stages by increasing index bit), so the output
// is bitwise that of rht_pass2.  grid = ceil(batch * ceil(P2 q / 32) / 8); 256 threads.
// kPush: the push all-gather's flavour -- the column is read from this rank's window
// of the call's parity as tagged words (polled until every word carries the tag).
template <int P1, bool kPush>
__global__ void __launch_bounds__(256) rht_pass2_reg(RhtArgs a) {
  pdl_wait();
  pdl_trigger();
  const std::uint32_t stride = a.P2 * a.q, ncg = (stride + 31) / 32;
  const std::uint32_t w = blockIdx.x * 8 + (threadIdx.x >> 5);
  const bool warp_live = w < ncg * std::uint32_t(a.batch);  // (no early return: push_done syncs the CTA)
  const int b = warp_live ? int(w / ncg) : 0;
  const std::uint32_t col = (w % ncg) * 32 + (threadIdx.x & 31u);
  const bool live = warp_live && col < stride;
  unsigned long long e = 0;
  const unsigned long long* win = nullptr;
  if constexpr (kPush) {
    e = ld_epoch(a.push.ctl);
    win = a.push.self_win + (e & 1) * a.push.win_words;
  }
  float v[P1];
  if constexpr (kPush) {
    const std::uint32_t tag = std::uint32_t(e + 1);
    bool ok = true;
#pragma unroll
    for (int r = 0; r < P1; ++r) {
      unsigned long long wd = 0;
      if (live)
        asm volatile("ld.volatile.u64 %0, [%1];\n"
                     : "=l"(wd)
                     : "l"(win + rank_major(b, r * stride + col, a.mid_rows, a.batch, a.n)));
      ok &= !live || std::uint32_t(wd >> 32) == tag;
      v[r] = __uint_as_float(std::uint32_t(wd));
    }
    if (!ok) {  // a peer's words not all here yet: poll them one by one
#pragma unroll
      for (int r = 0; r < P1; ++r)
        v[r] = ll_load1(win + rank_major(b, r * stride + col, a.mid_rows, a.batch, a.n), tag, a.push.rank);
    }
  } else if (a.mid_rows) {  // gathered rank-major rows (sharded)
#pragma unroll
    for (int r = 0; r < P1; ++r)
      v[r] = live ? __ldcg(a.mid + rank_major(b, r * stride + col, a.mid_rows, a.batch, a.n)) : 0.f;
  } else {
    const float* const src = a.mid + std::size_t(b) * a.n + col;
#pragma unroll
    for (int r = 0; r < P1; ++r) v[r] = live ? __ldcg(src + r * stride) : 0.f;
  }
  // K3's output signs (bit r = row r's sign of this lane's column)
  unsigned long long neg = 0;
  if (!a.fwd) {
    if (stride % 32 == 0 && (reinterpret_cast<std::uintptr_t>(a.signs) & 3) == 0 && warp_live) {
      // lane l loads the 32 sign bits of the warp's columns in rows l and l + 32, and a
      // 32 x 32 bit transpose across the lanes hands lane c its column's bits
      const std::uint32_t c0 = col - (threadIdx.x & 31u), lane = threadIdx.x & 31u;
      auto row_word = [&](std::uint32_t r) {
        return r < std::uint32_t(P1)
                   ? *reinterpret_cast<const std::uint32_t*>(a.signs + (std::size_t(r) * stride + c0) / 8)
                   : 0u;
      };
      auto transpose32 = [&](std::uint32_t x) {
#pragma unroll
        for (int sft = 16; sft > 0; sft >>= 1) {
          const std::uint32_t m = sft == 16 ? 0x0000FFFFu : sft == 8 ? 0x00FF00FFu : sft == 4 ? 0x0F0F0F0Fu
                                : sft == 2 ? 0x33333333u : 0x55555555u;
          const std::uint32_t y = __shfl_xor_sync(0xffffffffu, x, sft);
          x = (lane & sft) ? (x & ~m) | ((y >> sft) & m) : (x & m) | ((y << sft) & ~m);
        }
        return x;
      };
      const std::uint32_t lo = transpose32(row_word(lane));
      const std::uint32_t hi = P1 > 32 ? transpose32(row_word(lane + 32)) : 0u;
      neg = (static_cast<unsigned long long>(hi) << 32) | lo;
    } else if (live) {
#pragma unroll
      for (int r = 0; r < P1; ++r) {
        const std::uint32_t i = r * stride + col;
        neg |= static_cast<unsigned long long>((a.signs[i >> 3] >> (i & 7)) & 1) << r;
      }
    }
  }
#pragma unroll
  for (int len = 1; len < P1; len <<= 1)
#pragma unroll
    for (int k = 0; k < P1; ++k)
      if (!(k & len)) {
        const float x = v[k], y = v[k + len];
        v[k] = x + y;
        v[k + len] = x - y;
      }
  const float sc = rsqrtf(float(a.n));
  float mx = 0.f;
  if (live) {
#pragma unroll
    for (int r = 0; r < P1; ++r) {
      const std::uint32_t i = r * stride + col;
      float o = v[r] * sc;
      if ((neg >> r) & 1) o = -o;
      a.out[std::size_t(b) * a.n + i] = o;
      mx = fmaxf(mx, fabsf(o));
    }
  }
  if (a.fwd && a.amax_out && warp_live) {
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomic_max_pos(a.amax_out + b, mx);
  }
  if constexpr (kPush) push_done(a, e);
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


void plan_split_impl(const DevSide& side, RhtArgs& a) {
  a.n = side.n;
  a.p = side.p;
  a.q = side.q;
  // pass-1 chunk P2 * q: ~1K floats (<= 512 for the order-172 base, whose
  // dense product dominates pass 1)
  const std::uint32_t target = 512;  // measured best for the step (1024: +3 %)
  std::uint32_t P2 = 1;
  while (P2 * 2 <= side.p && P2 * 2 * side.q <= target) P2 *= 2;
  if ((P2 * side.q) % 4 != 0) throw SizeError("rht: dimension too small for the float4 passes");
  a.P2 = P2;
  a.P1 = side.p / P2;
  if (std::size_t(a.P1) * 16 > 96 * 1024) throw SizeError("rht: dimension too large");
}

template <int Q>
void launch_pass1_q(const RhtArgs& a, std::uint32_t extra_ctas, cudaStream_t s) {
  RhtArgs b = a;
  const int vpb = a.vpb > 1 ? a.vpb : 1;
  b.warp_teams = vpb == kP1Threads / 32;  // prefill batches: one vector per warp
  const std::size_t smem = p1_base_bytes<Q>() + (b.warp_teams ? vpb : 1) * p1_team_bytes<Q>(a.P2);
  auto* k = b.warp_teams ? rht_pass1<Q, true> : rht_pass1<Q, false>;
  kernel_attrs(reinterpret_cast<const void*>(k), 96 * 1024);
  launch_pdl(k, dim3((a.p1_count ? a.p1_count : a.P1) + extra_ctas, (a.batch + vpb - 1) / vpb), dim3(kP1Threads),
             smem, s, b);
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

template <int P1>
void launch_pass2_reg(const RhtArgs& a, cudaStream_t s) {
  const std::uint32_t warps = (a.P2 * a.q + 31) / 32 * std::uint32_t(a.batch);
  launch_pdl(a.push.ctl ? rht_pass2_reg<P1, true> : rht_pass2_reg<P1, false>, dim3((warps + 7) / 8), dim3(256), 0, s,
             a);
}

void launch_pass2(const RhtArgs& a, cudaStream_t s) {
  if (a.vpb > 1 && a.P1 <= 64) {  // prefill batches: register FWHT, one warp per 32 columns
    switch (a.P1) {
      case 1: launch_pass2_reg<1>(a, s); break;
      case 2: launch_pass2_reg<2>(a, s); break;
      case 4: launch_pass2_reg<4>(a, s); break;
      case 8: launch_pass2_reg<8>(a, s); break;
      case 16: launch_pass2_reg<16>(a, s); break;
      case 32: launch_pass2_reg<32>(a, s); break;
      default: launch_pass2_reg<64>(a, s); break;
    }
  } else {
    const std::uint32_t groups = a.P2 * a.q / 4;
    auto* k = a.push.ctl ? rht_pass2<true> : rht_pass2<false>;
    kernel_attrs(reinterpret_cast<const void*>(k), 96 * 1024);
    RhtArgs b = a;
    const int vpb = a.vpb > 1 ? a.vpb : 1;
    b.warp_teams = vpb > 1 && a.P1 <= 512;  // one vector per warp while a warp's share stays small
    const int threads = b.warp_teams ? 32 * vpb : 128;
    launch_pdl(k, dim3(groups, (a.batch + vpb - 1) / vpb), dim3(threads),
               std::size_t(a.P1) * 16 * (b.warp_teams ? vpb : 1), s, b);
  }
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


// Large (prefill) batches: 8 vectors per transform CTA (the per-vector work of a
// pass is a few hundred floats; thousands of tiny CTAs are launch-bound).
int vectors_per_block(int batch) { return batch >= 64 ? 8 : 1; }

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
  a.vpb = vectors_per_block(batch);
  launch_pass1(a, zero_ptr && zero_words ? 32 : 0, s);
  launch_pass2(a, s);
}

void launch_rht_out(const DevSide& side, const float* zin, float* u_scratch, float* y, int batch, cudaStream_t s,
                    int in_parts, const K4Sched* sched) {
  if (batch <= 0) return;
  if (side.kind == 1) {
    if (in_parts > 1) throw UnsupportedError("rfft: K-split partial inputs");
    launch_rfft_f32(side, zin, u_scratch, y, batch, true, s);
    return;
  }
  RhtArgs a{};
  plan_split_impl(side, a);
  a.signs = side.signs;
  a.base = side.base;
  a.in = zin;
  a.in_parts = in_parts;
  if (sched) {
    if (a.P2 * a.q > 512 || sched->mrows < 128 || (sched->mrows & (sched->mrows - 1)) || sched->nt % 8 != 0)
      throw UnsupportedError("rht: K4 pieces need chunks <= 512 rows, M tiles >= 128 rows and 8 | the N tile");
    a.sched = *sched, a.in_sched = 1;
  }
  a.mid = u_scratch;
  a.out = y;
  a.batch = batch;
  a.fwd = 0;
  a.vpb = vectors_per_block(batch);
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
  launch_pass1(a, 32, s);
  launch_pass2_limbs(a, s);
}

bool rht_sharded_k3_ok(const DevSide& side, std::uint32_t row0, std::uint32_t m_local) {
  if (side.kind != 0) return false;
  RhtArgs a{};
  plan_split_impl(side, a);
  const std::uint32_t chunk = a.P2 * a.q;
  return m_local % chunk == 0 && row0 % chunk == 0;
}

void launch_rht_out_acc_local(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                              std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                              const long long* tl, std::uint32_t row0, std::uint32_t m_local, float* z_send, int batch,
                              cudaStream_t s) {
  RhtArgs a{};
  plan_split_impl(side, a);
  const std::uint32_t chunk = a.P2 * a.q;
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
  a.mid = z_send;
  a.batch = batch;
  a.fwd = 0;
  a.ch0 = row0 / chunk;
  a.p1_count = m_local / chunk;
  a.row0 = row0;
  a.p1_out_rows = m_local;
  launch_pass1(a, 0, s);
}

void launch_rht_out_acc_push(const DevSide& side, const std::int32_t* zacc, int zacc_stages, std::uint32_t zacc_rows,
                             std::uint32_t zacc_cols, const float zscale[2], const int ze8p[2], const float* alpha,
                             const long long* tl, std::uint32_t row0, std::uint32_t m_local, const PushArgs& push,
                             int batch, cudaStream_t s) {
  RhtArgs a{};
  plan_split_impl(side, a);
  const std::uint32_t chunk = a.P2 * a.q;
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
  a.batch = batch;
  a.fwd = 0;
  a.ch0 = row0 / chunk;
  a.p1_count = m_local / chunk;
  a.row0 = row0;
  a.p1_out_rows = m_local;
  a.push = push;
  launch_pass1(a, 0, s);
}

void launch_rht_out_local_f32(const DevSide& side, const float* zparts, int parts, std::uint32_t row0,
                              std::uint32_t m_local, float* z_send, const PushArgs* push, int batch,
                              cudaStream_t s, const K4Sched* sched) {
  RhtArgs a{};
  plan_split_impl(side, a);
  const std::uint32_t chunk = a.P2 * a.q;
  a.signs = side.signs;
  a.base = side.base;
  a.in = zparts;
  a.in_parts = parts;
  a.in_local = 1;
  if (sched) {
    if (a.P2 * a.q > 512 || sched->mrows < 128 || (sched->mrows & (sched->mrows - 1)) || sched->nt % 8 != 0)
      throw UnsupportedError("rht: K4 pieces need chunks <= 512 rows, M tiles >= 128 rows and 8 | the N tile");
    a.sched = *sched, a.in_sched = 1;
  }
  a.mid = z_send;
  a.batch = batch;
  a.fwd = 0;
  a.ch0 = row0 / chunk;
  a.p1_count = m_local / chunk;
  a.row0 = row0;
  a.p1_out_rows = m_local;
  a.vpb = vectors_per_block(batch);
  if (push) a.push = *push;
  launch_pass1(a, 0, s);
}

void launch_rht_out_pass2_push(const DevSide& side, std::uint32_t m_local, const PushArgs& push, float* y, int batch,
                               cudaStream_t s) {
  RhtArgs a{};
  plan_split_impl(side, a);
  const std::uint32_t chunk = a.P2 * a.q;
  a.signs = side.signs;
  a.base = side.base;
  a.mid_rows = m_local;
  a.out = y;
  a.batch = batch;
  a.fwd = 0;
  a.push = push;
  a.vpb = vectors_per_block(batch);
  launch_pass2(a, s);
}

void launch_rht_out_pass2_gathered(const DevSide& side, const float* mid_gathered, std::uint32_t m_local, float* y,
                                   int batch, cudaStream_t s) {
  RhtArgs a{};
  plan_split_impl(side, a);
  a.signs = side.signs;
  a.base = side.base;
  a.mid = const_cast<float*>(mid_gathered);
  a.mid_rows = m_local;
  a.out = y;
  a.batch = batch;
  a.fwd = 0;
  a.vpb = vectors_per_block(batch);
  launch_pass2(a, s);
}

void launch_rht_out_gathered(const DevSide& side, const float* z_gathered, std::uint32_t m_local, float* u_scratch,
                             float* y, int batch, cudaStream_t s) {
  RhtArgs a{};
  plan_split_impl(side, a);
  a.signs = side.signs;
  a.base = side.base;
  a.in = z_gathered;
  a.in_rows = m_local;
  a.mid = u_scratch;
  a.out = y;
  a.batch = batch;
  a.fwd = 0;
  launch_pass1(a, 0, s);
  launch_pass2(a, s);
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
