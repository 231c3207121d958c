// Device-side pieces of the randomized Hadamard transforms (K1 / K3) of the
// RHT kernels (kernels_rht.cu).  The pass bodies run on a "team" of threads: a
// whole CTA (__syncthreads) for small batches, where one vector's pass is
// spread over the CTA, or a single warp (__syncwarp) for prefill batches, where
// each warp of a CTA carries its own vector and the CTA has 8 in flight.
//
// SideTransform (core/src/transforms.cpp:28-47) with had_apply
// (core/src/hadamard.cpp:170-210):  H = (H_p (x) B_q) / sqrt(n), flat index
// i = a * q + b, a = a_hi * P2 + a_lo.  Pass 1 = a contiguous chunk
// [a_hi][0..P2)[0..q) (signs | limb combine, base B_q or B_q^T on each q-row,
// FWHT over a_lo); pass 2 = a group of adjacent columns (a_lo, b) over all P1
// values of a_hi (FWHT over a_hi, 1/sqrt(n), signs / integer limbs).
#pragma once

#include <cstdint>
#include <cstdio>

namespace q8p::detail {

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
  // multi-chunk K1 (batches above the GEMV's 32 vectors): vector b's B images go to
  // chunk b / chunk_vec (chunk_bytes apart) as local column b % chunk_vec; 0 = off
  std::uint32_t chunk_vec;
  std::size_t chunk_bytes;
  int zacc_zero;                // K3 pass 1: zero the accumulators after reading them (next chunk's K2)
  // Row-sharded K3 (q8p_forward_sharded): pass 1 over this rank's chunks only --
  // chunks ch0 .. ch0 + p1_count, accumulator rows and pass-1 outputs indexed from
  // row0, outputs written as [batch][p1_out_rows] (the all-gather send buffer);
  // pass 2 reads the gathered [world][batch][mid_rows] ("rank-major") layout.
  // in_rows: pass 1's fp32 input in the same rank-major layout.  0 = off.
  std::uint32_t ch0, p1_count, row0, p1_out_rows, mid_rows, in_rows;
  int vpb;                      // vectors per CTA (fp32 passes; 0/1 = one)
  int in_parts;                 // pass 1 fp32 input = sum of in_parts partial arrays [batch][n] (0/1 = one)
  K4Sched sched;                // in_sched: the input is K4's z slices; a row/vector tile's piece
  int in_sched;                 //   count (k4_pieces) says how many of the in_parts slices it sums
  int in_local;                 // row-sharded prefill: the fp32 input holds this rank's rows only,
                                // [in_parts][batch][p1_out_rows] (row i at i - row0)
  // Push all-gather (device.hpp PushArgs; push.ctl == nullptr = off): pass 1 stores
  // its rows as tagged words into every rank's window (rank-major
  // [world][batch][p1_out_rows]); pass 2 reads its own window of the call's parity
  // once the words carry the call's tag (the kernels pass window and tag to the
  // bodies: the kernel parameters are never written, so they stay in the constant bank).
  PushArgs push;
  int warp_teams;               // fp32 passes: one vector per warp (vpb > 1; set by the launchers)
};

// Element (b, i) of a [batch][n] vector set stored rank-major with `rows` rows per
// rank ([n / rows][batch][rows]) -- the all-gather output layout; rows % 4 == 0.
__device__ __forceinline__ std::size_t rank_major(std::size_t b, std::uint32_t i, std::uint32_t rows, int batch,
                                                  std::uint32_t n) {
  return rows ? (std::size_t(i / rows) * batch + b) * rows + i % rows : b * n + i;
}

struct Team {
  std::uint32_t tid, n, warp;  // thread index in the team, team size, 1 = the team is one warp
};

namespace {


// Push all-gather, LL protocol (device.hpp).  A tagged word = float bits | tag << 32.
__device__ __forceinline__ unsigned long long ll_word(float v, std::uint32_t tag) {
  return (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(v);
}
__device__ __forceinline__ unsigned long long ld_epoch(const PeerCtl* c) {
  return *reinterpret_cast<const volatile unsigned long long*>(&c->epoch);
}
// Pass 1's output float4s [0, nv) from smem `cur` into every rank's window at word
// offset `off`, as tagged words (NVLink stores).
__device__ __forceinline__ void push_store(unsigned long long* const* wins, int world, const float* cur,
                                           std::size_t off, std::uint32_t nv, std::uint32_t tag, std::uint32_t tid,
                                           std::uint32_t nthreads) {
#pragma unroll 1
  for (int r = 0; r < world; ++r) {
    unsigned long long* const mo = wins[r] + off;
    for (std::uint32_t v = tid; v < nv; v += nthreads) {
      const float4 c = reinterpret_cast<const float4*>(cur)[v];
      reinterpret_cast<ulonglong2*>(mo + 4 * v)[0] = make_ulonglong2(ll_word(c.x, tag), ll_word(c.y, tag));
      reinterpret_cast<ulonglong2*>(mo + 4 * v)[1] = make_ulonglong2(ll_word(c.z, tag), ll_word(c.w, tag));
    }
  }
}
// Cold path of ll_load4: a peer never wrote this call's words.
__device__ __noinline__ void ll_timeout(int rank, std::uint32_t tag, std::uint32_t have) {
  printf("q8p push all-gather: rank %d waited 20 s for call tag %u (word has tag %u)\n", rank, tag, have);
  __trap();
}
// Four consecutive tagged words (16 B aligned) once all carry `tag`; a peer that
// never writes them makes the reader trap after ~20 s.
__device__ __forceinline__ float4 ll_load4(const unsigned long long* p, std::uint32_t tag, int rank) {
  unsigned long long w0, w1, w2, w3;
  std::uint64_t t0 = 0;
  for (int spin = 0;; ++spin) {
    asm volatile("ld.volatile.v2.u64 {%0, %1}, [%2];\n" : "=l"(w0), "=l"(w1) : "l"(p));
    asm volatile("ld.volatile.v2.u64 {%0, %1}, [%2];\n" : "=l"(w2), "=l"(w3) : "l"(p + 2));
    if (std::uint32_t(w0 >> 32) == tag && std::uint32_t(w1 >> 32) == tag && std::uint32_t(w2 >> 32) == tag &&
        std::uint32_t(w3 >> 32) == tag)
      break;
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (spin == 0) t0 = t;
    if (t - t0 > 20000000000ull) ll_timeout(rank, tag, std::uint32_t(w0 >> 32));
    __nanosleep(32);
  }
  return make_float4(__uint_as_float(std::uint32_t(w0)), __uint_as_float(std::uint32_t(w1)),
                     __uint_as_float(std::uint32_t(w2)), __uint_as_float(std::uint32_t(w3)));
}
// One tagged word once it carries `tag` (as ll_load4).
__device__ __forceinline__ float ll_load1(const unsigned long long* p, std::uint32_t tag, int rank) {
  unsigned long long w;
  std::uint64_t t0 = 0;
  for (int spin = 0;; ++spin) {
    asm volatile("ld.volatile.u64 %0, [%1];\n" : "=l"(w) : "l"(p));
    if (std::uint32_t(w >> 32) == tag) break;
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (spin == 0) t0 = t;
    if (t - t0 > 20000000000ull) ll_timeout(rank, tag, std::uint32_t(w >> 32));
    __nanosleep(32);
  }
  return __uint_as_float(std::uint32_t(w));
}
// End of a pass-2 CTA: the last one of the call advances the rank's epoch.
__device__ __forceinline__ void push_done(const RhtArgs& a, unsigned long long e) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long total = std::uint64_t(gridDim.x) * gridDim.y;
    if (atomicAdd(&a.push.ctl->done, 1ull) == total - 1) {
      a.push.ctl->done = 0;
      __threadfence();
      *reinterpret_cast<volatile unsigned long long*>(&a.push.ctl->epoch) = e + 1;
    }
  }
}

__device__ __forceinline__ Team block_team() { return Team{threadIdx.x, blockDim.x, 0u}; }
__device__ __forceinline__ Team warp_team() { return Team{threadIdx.x & 31u, 32u, 1u}; }
__device__ __forceinline__ void team_sync(const Team& t) {
  if (t.warp)
    __syncwarp();
  else
    __syncthreads();
}
// Team-wide sum / max; red: >= 32 floats of team-shared smem (unused by warp teams).
// The reduction tree is fixed, so the result is deterministic.
template <bool kMax>
__device__ __forceinline__ float team_reduce(float v, float* red, const Team& tm) {
  for (int o = 16; o > 0; o >>= 1) {
    const float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = kMax ? fmaxf(v, w) : v + w;
  }
  if (tm.warp) return v;
  if ((tm.tid & 31) == 0) red[tm.tid >> 5] = v;
  team_sync(tm);
  float t = 0.f;
  for (std::uint32_t w = 0; w < (tm.n + 31) / 32; ++w) t = kMax ? fmaxf(t, red[w]) : t + red[w];
  return t;
}

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
__device__ __forceinline__ void fwht_pass(float* s, std::uint32_t rows, std::uint32_t sbit, const Team& tm) {
  constexpr int K = 1 << R;
  const std::uint32_t tasks = (rows >> R) * Q;
  const std::uint32_t lowmask = (1u << sbit) - 1;
  for (std::uint32_t t = tm.tid; t < tasks; t += tm.n) {
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
  team_sync(tm);
}

template <int Q>
__device__ void fwht_rows(float* s, std::uint32_t rows, const Team& tm) {
  const std::uint32_t lb = 31 - __clz(rows);
  std::uint32_t b = 0;
  for (; b + 3 <= lb; b += 3) fwht_pass<3, Q>(s, rows, b, tm);
  if (b + 2 <= lb) {
    fwht_pass<2, Q>(s, rows, b, tm);
    b += 2;
  }
  if (b + 1 <= lb) fwht_pass<1, Q>(s, rows, b, tm);
}

// z rows i..i+3 of vector b from the int32 limb accumulators:
// z = sum_s scale_s alpha (2 Z_s - [E8P] TL) / 4, Z_s = sum_l 128^(3-l) zacc[s][4b + l]
// (exact int64 combine, one double rounding per stage sum, then fp32).  Shared by
// K3 pass 1 and the row-sharded combine kernel so both round identically.
__device__ __forceinline__ float4 combine4(const RhtArgs& a, int b, std::uint32_t i) {
  // __ldcg: written earlier in the same fused kernel by other CTAs (L1 is not coherent)
  const double al = double(__ldcg(a.alpha_in + b)) * 0.25;
  const long long tl = __ldcg(a.tl_in + b);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int st = 0; st < a.zstages; ++st) {
    const std::int32_t* z = a.zacc + (std::size_t(st) * a.zcols + 4 * b) * a.zrows + (i - a.row0);
    const int4 v0 = __ldcg(reinterpret_cast<const int4*>(z));
    const int4 v1 = __ldcg(reinterpret_cast<const int4*>(z + a.zrows));
    const int4 v2 = __ldcg(reinterpret_cast<const int4*>(z + 2 * std::size_t(a.zrows)));
    const int4 v3 = __ldcg(reinterpret_cast<const int4*>(z + 3 * std::size_t(a.zrows)));
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

// z rows i, i + 1 (i even) of vector b: combine4's arithmetic on an aligned pair
// (the rfft K3 reads complex pairs).
__device__ __forceinline__ float2 combine2(const RhtArgs& a, int b, std::uint32_t i) {
  const double al = double(__ldcg(a.alpha_in + b)) * 0.25;
  const long long tl = __ldcg(a.tl_in + b);
  double acc[2] = {0.0, 0.0};
  for (int st = 0; st < a.zstages; ++st) {
    const std::int32_t* z = a.zacc + (std::size_t(st) * a.zcols + 4 * b) * a.zrows + i;
    const int2 v0 = __ldcg(reinterpret_cast<const int2*>(z));
    const int2 v1 = __ldcg(reinterpret_cast<const int2*>(z + a.zrows));
    const int2 v2 = __ldcg(reinterpret_cast<const int2*>(z + 2 * std::size_t(a.zrows)));
    const int2 v3 = __ldcg(reinterpret_cast<const int2*>(z + 3 * std::size_t(a.zrows)));
    const long long sub = (st == 0 ? a.ze8p0 : a.ze8p1) ? tl : 0;
    const double c = al * double(st == 0 ? a.zscale0 : a.zscale1);
    auto zt = [&](int x0, int x1, int x2, int x3) {
      const long long Z = ((static_cast<long long>(x0) * 128 + x1) * 128 + x2) * 128 + x3;
      return double(2 * Z - sub) * c;
    };
    acc[0] += zt(v0.x, v1.x, v2.x, v3.x);
    acc[1] += zt(v0.y, v1.y, v2.y, v3.y);
  }
  return make_float2(float(acc[0]), float(acc[1]));
}


// K4 stream-K piece counts for pass 1's CTA (in_sched): the (<= kP1Tiles) M tiles of
// chunk `ch` for the N tile of vector b0 (a CTA's vectors share it: vpb divides the
// N tile).  Threads 0..kP1Tiles-1 write s_pieces[]; the caller syncs.
constexpr int kP1Tiles = 8;  // a <= 512-row chunk touches <= 5 tiles of >= 128 rows
__device__ __forceinline__ void p1_tile_pieces(const RhtArgs& a, std::uint32_t ch, std::uint32_t chunk, int b0,
                                               int* s_pieces) {
  if (threadIdx.x < kP1Tiles) {
    const std::uint32_t e0 = ch * chunk, r0 = a.in_local ? e0 - a.row0 : e0;
    const std::uint32_t mp = r0 / a.sched.mrows + threadIdx.x, mp_last = (r0 + chunk - 1) / a.sched.mrows;
    s_pieces[threadIdx.x] =
        mp <= mp_last ? int(k4_pieces(a.sched, (std::uint32_t(b0) / a.sched.nt) * a.sched.MP + mp)) : 1;
  }
}

// Pass-1 smem: the Q x Q base (float for Q <= 28, int8 for the order-172 one;
// shared by the CTA's teams), then per team the chunk x and the base output y.
template <int Q>
__host__ __device__ constexpr std::size_t p1_base_bytes() {
  return Q == 1 ? 0 : (Q <= 28 ? Q * Q * 4 : (Q * Q + 15) / 16 * 16);
}
template <int Q>
__host__ __device__ constexpr std::size_t p1_team_bytes(std::uint32_t P2) {
  return std::size_t(P2) * Q * 4 * (Q > 1 ? 2 : 1);
}
// Base into smem (whole CTA; synced by the caller or by the body's first team sync).
template <int Q>
__device__ void p1_load_base(const RhtArgs& a, float* Bs) {
  if constexpr (Q > 1) {
    if constexpr (Q <= 28) {
      for (std::uint32_t i = threadIdx.x; i < Q * Q; i += blockDim.x) Bs[i] = float(a.base[i]);
    } else {
      for (std::uint32_t i = threadIdx.x; i < Q * Q / 4; i += blockDim.x)
        reinterpret_cast<std::uint32_t*>(Bs)[i] = reinterpret_cast<const std::uint32_t*>(a.base)[i];
    }
  }
}

// Pass 1 on chunk `ch` of vector b.  xs: the team's [2][chunk] floats; Bs: the
// base (p1_load_base); red: >= 32 floats of team-shared smem.
// ll_tag: the push all-gather's call tag (a.push.ctl set), else unused.
// pieces (in_sched): K4 stream-K piece counts of the (<= kP1Tiles) M tiles the chunk's rows
// touch, for this vector's N tile, from M pair p1_mp_first on (p1_tile_pieces).
template <int Q>
__device__ void rht_p1_body(const RhtArgs& a, std::uint32_t ch, int b, float* xs, const float* Bs, float* red,
                            const Team& tm, std::uint32_t ll_tag = 0, const int* pieces = nullptr) {
  const std::uint32_t chunk = a.P2 * Q;  // floats, multiple of 4
  const std::uint32_t e0 = ch * chunk;
  float* x = xs;                          // [P2][Q]
  float* y = xs + chunk;                  // base output (Q > 1)
  // whole-CTA team: the base load overlaps the chunk loads (the sync below covers both)
  if (!tm.warp) p1_load_base<Q>(a, const_cast<float*>(Bs));
  float ss = 0.f;
  if (a.zacc) {
    for (std::uint32_t v = tm.tid; v < chunk / 4; v += tm.n) {
      const std::uint32_t i = e0 + 4 * v;
      reinterpret_cast<float4*>(x)[v] = combine4(a, b, i);
      if (a.zacc_zero) {  // each (vector, row quad) is read by exactly one thread: clear it for the next chunk
        for (int st = 0; st < a.zstages; ++st)
          for (int l = 0; l < 4; ++l)
            *reinterpret_cast<int4*>(const_cast<std::int32_t*>(a.zacc) +
                                     (std::size_t(st) * a.zcols + 4 * b + l) * a.zrows + (i - a.row0)) =
                make_int4(0, 0, 0, 0);
      }
    }
  } else {
    const std::uint32_t mp_first = a.in_sched ? (a.in_local ? e0 - a.row0 : e0) / a.sched.mrows : 0;
    const int msh = a.in_sched ? __ffs(int(a.sched.mrows)) - 1 : 0;  // K4 M tiles are 128 or 256 rows
    for (std::uint32_t v = tm.tid; v < chunk / 4; v += tm.n) {
      const std::uint32_t i = e0 + 4 * v;
      // element (part pp, vector b, row i) of the input
      const std::uint32_t rows = a.in_local ? a.p1_out_rows : a.n, ri = a.in_local ? i - a.row0 : i;
      float4 val = __ldcg(reinterpret_cast<const float4*>(
          a.in + (a.in_local ? std::size_t(b) * rows + ri : rank_major(b, i, a.in_rows, a.batch, a.n))));
      // K-split partials (prefill), summed in piece order: all in_parts slices, or the
      // pieces of this (vector, row) tile under K4's stream-K schedule
      const int parts = a.in_sched ? pieces[(ri >> msh) - mp_first] : a.in_parts;
      for (int pp = 1; pp < parts; ++pp) {
        const float4 w4 =
            __ldcg(reinterpret_cast<const float4*>(a.in + (std::size_t(pp) * a.batch + b) * rows + ri));
        val = make_float4(val.x + w4.x, val.y + w4.y, val.z + w4.z, val.w + w4.w);
      }
      ss += val.x * val.x + val.y * val.y + val.z * val.z + val.w * val.w;
      if (a.fwd) val = sign4(val, (a.signs[i >> 3] >> (i & 4)) & 0xFu);
      reinterpret_cast<float4*>(x)[v] = val;
    }
  }
  if (a.ssq) {  // deterministic per-chunk sum of squares
    const float t = team_reduce<false>(ss, red, tm);
    if (tm.tid == 0) a.ssq[std::size_t(b) * a.P1 + ch] = t;
  }
  team_sync(tm);
  float* cur = x;
  if constexpr (Q > 1) {
    // base along each contiguous q-row: y[r][c] = sum_k B[c][k] x[r][k] (fwd) or B[k][c] (K3)
    if constexpr (Q <= 28) {
      if (tm.warp) {
        // warp teams (prefill): lane = output column c with its base row (fwd) / column
        // in registers; each x row is Q / 4 broadcast float4 reads.  Same FMA order as
        // the per-element loop below, so both give the same bits.
        const std::uint32_t c = tm.tid & 31u;
        if (c < std::uint32_t(Q)) {
          float bc[Q];
#pragma unroll
          for (int k = 0; k < Q; ++k) bc[k] = a.fwd ? Bs[c * Q + k] : Bs[k * Q + c];
          for (std::uint32_t r = 0; r < a.P2; ++r) {
            const float4* xr = reinterpret_cast<const float4*>(x + r * Q);
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < Q / 4; ++j) {
              const float4 x4 = xr[j];
              acc += bc[4 * j] * x4.x;
              acc += bc[4 * j + 1] * x4.y;
              acc += bc[4 * j + 2] * x4.z;
              acc += bc[4 * j + 3] * x4.w;
            }
            y[r * Q + c] = acc;
          }
        }
      } else {
        // whole-CTA teams (decode batches): one output per thread and step (more
        // parallel chains than the broadcast form for a single vector)
        for (std::uint32_t e = tm.tid; e < chunk; e += tm.n) {
          const std::uint32_t r = e / Q, c = e - r * Q;
          const float* xr = x + r * Q;
          float acc = 0.f;
          if (a.fwd) {
#pragma unroll 4
            for (int k = 0; k < Q; ++k) acc += Bs[c * Q + k] * xr[k];
          } else {
#pragma unroll 4
            for (int k = 0; k < Q; ++k) acc += Bs[k * Q + c] * xr[k];
          }
          y[e] = acc;
        }
      }
    } else {
      const std::int8_t* B8 = reinterpret_cast<const std::int8_t*>(Bs);
      for (std::uint32_t e = tm.tid; e < chunk; e += tm.n) {
        const std::uint32_t r = e / Q, c = e - r * Q;
        const float* xr = x + r * Q;
        float acc = 0.f;
        if (a.fwd) {
#pragma unroll 4
          for (int k = 0; k < Q; ++k) acc += float(B8[c * Q + k]) * xr[k];
        } else {
#pragma unroll 4
          for (int k = 0; k < Q; ++k) acc += float(B8[k * Q + c]) * xr[k];
        }
        y[e] = acc;
      }
    }
    team_sync(tm);
    cur = y;
  }
  fwht_rows<Q>(cur, a.P2, tm);
  if (a.push.ctl) {
    push_store(a.push.wins, a.push.world, cur,
               (ll_tag & 1 ? 0 : a.push.win_words) +  // parity = epoch & 1 = (tag - 1) & 1
                   (std::size_t(a.push.rank) * a.batch + b) * a.p1_out_rows + (e0 - a.row0),
               chunk / 4, ll_tag, tm.tid, tm.n);
  } else {
    float* const mo = a.p1_out_rows ? a.mid + std::size_t(b) * a.p1_out_rows + (e0 - a.row0)
                                    : a.mid + std::size_t(b) * a.n + e0;
    for (std::uint32_t v = tm.tid; v < chunk / 4; v += tm.n)
      *reinterpret_cast<float4*>(mo + 4 * v) = reinterpret_cast<float4*>(cur)[v];
  }
  team_sync(tm);  // smem reusable by the caller
}

// Pass 2 (fp32 output) on the 4-column group `cg` of vector b.  red: >= 32 floats.
// ll_mid: the push all-gather's window of this call (tagged words, tag ll_tag), else nullptr.
__device__ void rht_p2_body(const RhtArgs& a, std::uint32_t cg, int b, float* sm2, float* red, const Team& tm,
                            const unsigned long long* ll_mid = nullptr, std::uint32_t ll_tag = 0) {
  const std::uint32_t stride = a.P2 * a.q;  // elements between consecutive a_hi
  const std::uint32_t col = cg * 4;         // 4 adjacent columns
  for (std::uint32_t r = tm.tid; r < a.P1; r += tm.n) {
    const std::size_t idx = rank_major(b, r * stride + col, a.mid_rows, a.batch, a.n);
    reinterpret_cast<float4*>(sm2)[r] = ll_mid ? ll_load4(ll_mid + idx, ll_tag, a.push.rank)
                                               : __ldcg(reinterpret_cast<const float4*>(a.mid + idx));
  }
  team_sync(tm);
  fwht_rows<4>(sm2, a.P1, tm);
  const float sc = rsqrtf(float(a.n));
  float mx = 0.f;
  for (std::uint32_t r = tm.tid; r < a.P1; r += tm.n) {
    const std::uint32_t i = r * stride + col;
    float4 v = reinterpret_cast<float4*>(sm2)[r];
    v = make_float4(v.x * sc, v.y * sc, v.z * sc, v.w * sc);
    if (!a.fwd) v = sign4(v, (a.signs[i >> 3] >> (i & 4)) & 0xFu);
    *reinterpret_cast<float4*>(a.out + std::size_t(b) * a.n + i) = v;
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  if (a.fwd && a.amax_out) {
    const float m = team_reduce<true>(mx, red, tm);
    if (tm.tid == 0) atomic_max_pos(a.amax_out + b, m);
  }
  team_sync(tm);
}

// Integer activations of the tensor-core GEMV (gemv_tc.cu): Lt = rint(t / alpha)
// with alpha = the power of two >= |x|_2 / kActMax (|t_i| <= |t|_2 = |x|_2, so no
// clamping is ever active), four balanced base-128 int8 limbs per value, the
// block sums S_k = sum_c Lt_{8k+c} for the side MMA, and TL = sum_i Lt_i.
constexpr int kLtMax = 266338304;  // 127 * 128^3: range of 4 balanced base-128 int8 limbs
// Activations are 25-bit (|Lt| <= kActMax) so the block sums S_k = sum_c Lt_{8k+c}
// of the side MMA also fit 4 limbs exactly (|S_k| <= 8 kActMax <= kLtMax): the
// shift term sum_k b_k S_k is then exact.  (A q_k = floor(S_k / 8) side operand
// drops sum_k b_k (S_k mod 8) -- a per-row bias that accumulates in y_0 = sum z / sqrt(m).)
constexpr int kActMax = kLtMax / 8;

// Balanced base-128 digits: v in [-kLtMax, kLtMax] -> l0 in [-127, 127], l1..l3 in [-64, 64].
__device__ __forceinline__ void limbs4(int v, int (&l)[4]) {
  l[0] = (v + (1 << 20)) >> 21;
  int rem = v - (l[0] << 21);
  l[1] = (rem + (1 << 13)) >> 14;
  rem -= l[1] << 14;
  l[2] = (rem + 64) >> 7;
  l[3] = rem - (l[2] << 7);
}

// One codeword k of vector b (8 transformed values v): integer activations,
// limbs into the B image, returns sum_c Lt_c (for TL).
__device__ __forceinline__ long long emit_limbs(const RhtArgs& a, int b, std::uint32_t k, const float* v, float sc,
                                                float inv) {
  const std::uint32_t N = a.bcols;
  int lt[8];
  long long S = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    float t = rintf(v[c] * sc * inv);
    t = fminf(fmaxf(t, -float(kActMax)), float(kActMax));
    lt[c] = int(t);
    S += lt[c];
  }
  const int qk = int(S);  // exact block sum (|S| <= kLtMax)
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
  std::uint32_t bl = std::uint32_t(b);
  if (a.chunk_vec) {
    slab += std::size_t(bl / a.chunk_vec) * a.chunk_bytes;
    bl %= a.chunk_vec;
  }
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const std::uint32_t row = 4 * bl + l;
    const std::uint32_t rowoff = (row >> 3) * 256 + (row & 7) * 16;
    // main: K-block kb, K bytes 8 (j % 4) .. +7 -> chunk (j % 4) / 2, offset 8 (j % 2)
    *reinterpret_cast<uint2*>(slab + kb * N * 32 + rowoff + ((j & 3) >> 1) * 128 + (j & 1) * 8) =
        make_uint2(w[l][0], w[l][1]);
    // side: K-block 8, K byte j
    slab[8 * N * 32 + rowoff + (j >> 4) * 128 + (j & 15)] = std::uint8_t(ql[l]);
  }
  return S;
}

// alpha = the power of two >= |x|_2 (1 + 2^-10) / kActMax; returns {alpha, 1/alpha}.
__device__ __forceinline__ float2 alpha_of(float ss) {
  const float v = sqrtf(ss) * (1.0f + 1.0f / 1024.f) / float(kActMax);
  int e = 0;
  if (v > 0.f) frexpf(v, &e);
  return v > 0.f ? make_float2(ldexpf(1.f, e), ldexpf(1.f, -e)) : make_float2(1.f, 1.f);
}

// Pass 2 of K1, limb flavour, on the 8-column group `cg` (one codeword per a_hi
// row) of vector b.  redl: >= 32 long longs; s_alpha: 2 floats (team-shared).
__device__ void rht_p2_limbs_body(const RhtArgs& a, std::uint32_t cg, int b, float* sm2, long long* redl,
                                  float* s_alpha, const Team& tm) {
  const std::uint32_t stride = a.P2 * a.q;  // elements between consecutive a_hi
  const std::uint32_t col = cg * 8;
  for (std::uint32_t r = tm.tid; r < 2 * a.P1; r += tm.n)
    reinterpret_cast<float4*>(sm2)[r] = __ldcg(reinterpret_cast<const float4*>(
        a.mid + std::size_t(b) * a.n + std::size_t(r >> 1) * stride + col + 4 * (r & 1)));
  if (tm.tid == 0) {
    float ss = 0.f;
    for (std::uint32_t j = 0; j < a.P1; ++j) ss += __ldcg(a.ssq + std::size_t(b) * a.P1 + j);
    const float2 al = alpha_of(ss);
    s_alpha[0] = al.x;
    s_alpha[1] = al.y;
    if (cg == 0) a.alpha_out[b] = s_alpha[0];
  }
  team_sync(tm);
  fwht_rows<8>(sm2, a.P1, tm);
  const float sc = rsqrtf(float(a.n)), inv = s_alpha[1];
  long long tl = 0;
  for (std::uint32_t r = tm.tid; r < a.P1; r += tm.n) tl += emit_limbs(a, b, (r * stride + col) >> 3, sm2 + r * 8, sc, inv);
  for (int o = 16; o > 0; o >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, o);
  if ((tm.tid & 31) == 0) redl[tm.tid >> 5] = tl;
  team_sync(tm);
  if (tm.tid == 0) {
    long long t = 0;
    for (std::uint32_t w = 0; w < (tm.n + 31) / 32; ++w) t += redl[w];
    atomicAdd(reinterpret_cast<unsigned long long*>(a.tl_out + b), static_cast<unsigned long long>(t));
  }
  team_sync(tm);
}

}  // namespace
}  // namespace q8p::detail
