/* CPU restatement of the reference `latq` quantized-linear inference path.
 *
 * TEST INFRASTRUCTURE ONLY.  Used by tests/ and __graft_entry__.smoke() as
 * the parity checker and by bench.py's cpu_baseline leg; never linked or
 * called by the product (paper_2402_04396_b200/).
 *
 * Each function restates the reference algorithm it cites (paths relative to
 * /root/reference/proj).  Arithmetic order follows the reference exactly and
 * the file is compiled with -ffp-contract=off, so for every shape the
 * reference can plan, oracle_infer() is bit-identical to latq::infer (pinned
 * by tests/test_oracle.py against oracle/_ref, the reference compiled in
 * place, and against the golden fixtures in tests/golden/).
 *
 * The rfft transform (rfft.cpp) is restated with a direct DFT in place of
 * FFTW3 (absent): equal to the reference to rounding (~1e-15), pinned
 * against the reference compiled with oracle/shim/fftw3.h and against the
 * properties test_rfft.cpp checks (tests/test_oracle.py).
 *
 * One deliberate extension: the Hadamard registry gains order 172
 * (oracle/had172.h) so n = 11008 = 64 * 172 can be planned; the reference
 * throws SizeError there (core/src/hadamard.cpp:156-168).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "had172.h"

enum { OK = 0, E_SIZE = 1, E_VALIDATION = 2, E_FORMAT = 3, E_BADMAGIC = 4, E_VERSION = 5, E_TRUNC = 6 };

/* ------------------------------------------------------------------------ */
/* E8P tables: core/src/e8p.cpp:17-79                                        */
/* ------------------------------------------------------------------------ */

/* The 29 padding rows (doubled coordinates, sum of squares 48) in the
 * codebook's canonical order; part of the serialized format
 * (core/src/e8p.cpp:17-33, pinned by tests/acceptance.cpp:137-151). */
static const int8_t kPad[29][8] = {
    {3, 1, 1, 1, 3, 3, 3, 3}, {1, 3, 1, 1, 3, 3, 3, 3}, {1, 1, 3, 1, 3, 3, 3, 3},
    {1, 1, 1, 3, 3, 3, 3, 3}, {3, 3, 3, 1, 3, 3, 1, 1}, {3, 3, 3, 1, 3, 1, 3, 1},
    {3, 3, 3, 1, 1, 3, 3, 1}, {3, 3, 3, 1, 3, 1, 1, 3}, {3, 3, 3, 1, 1, 3, 1, 3},
    {3, 3, 3, 1, 1, 1, 3, 3}, {3, 3, 1, 3, 3, 3, 1, 1}, {3, 3, 1, 3, 3, 1, 3, 1},
    {3, 3, 1, 3, 1, 3, 3, 1}, {3, 3, 1, 3, 3, 1, 1, 3}, {3, 3, 1, 3, 1, 3, 1, 3},
    {3, 3, 1, 3, 1, 1, 3, 3}, {3, 1, 3, 3, 3, 3, 1, 1}, {3, 1, 3, 3, 3, 1, 3, 1},
    {3, 1, 3, 3, 1, 3, 3, 1}, {3, 1, 3, 3, 3, 1, 1, 3}, {3, 1, 3, 3, 1, 3, 1, 3},
    {1, 3, 3, 3, 1, 1, 3, 3}, {1, 3, 3, 3, 3, 3, 1, 1}, {1, 3, 3, 3, 3, 1, 3, 1},
    {1, 3, 3, 3, 1, 3, 3, 1}, {1, 3, 3, 3, 3, 1, 1, 3}, {1, 3, 3, 3, 1, 3, 1, 3},
    {1, 1, 3, 3, 1, 3, 3, 3}, {3, 3, 1, 1, 3, 3, 3, 1},
};

static int8_t g_doubled[256][8];
static uint8_t g_odd[256];
static double g_e81[256][8]; /* e8-1bit table */
static pthread_once_t g_once = PTHREAD_ONCE_INIT;

/* build_e8p (e8p.cpp:37-74): all {1,3,5}^8 with sum of squares <= 40 in
 * ascending lexicographic order (odometer enumeration with the last
 * coordinate fastest is already lexicographic), then the 29 pad rows;
 * odd_parity[i] = (row sum % 4 == 2). */
static void build_e8p_tables(void) {
  int n = 0;
  for (int code = 0; code < 6561; ++code) {
    int8_t row[8];
    int rem = code, ss = 0;
    for (int c = 7; c >= 0; --c) {
      row[c] = (int8_t)(1 + 2 * (rem % 3));
      rem /= 3;
      ss += row[c] * row[c];
    }
    if (ss <= 40) memcpy(g_doubled[n++], row, 8);
  }
  /* n == 227 by construction (checked in tests against the reference). */
  for (int i = 0; i < 29; ++i) memcpy(g_doubled[227 + i], kPad[i], 8);
  for (int i = 0; i < 256; ++i) {
    int s = 0;
    for (int c = 0; c < 8; ++c) s += g_doubled[i][c];
    g_odd[i] = (uint8_t)(s % 4 == 2);
  }
}

/* build_lattice_ball(e8, dim 8, bits 1) (codebook.cpp:162-243): doubled
 * integer vectors (all even, or all odd) with coordinate sum = 0 mod 4 and
 * squared norm <= r2, r2 = 32 doubled (i.e. norm^2 <= 8 undoubled) -- already
 * >= 256 points -- sorted by squared norm then lexicographically, first 256. */
typedef struct {
  int64_t v[8];
  int64_t n2;
} pt_t;
static pt_t* g_pts;
static int g_npts, g_cap;
static void push_pt(const int64_t* v) {
  if (g_npts == g_cap) {
    g_cap = g_cap ? 2 * g_cap : 4096;
    g_pts = (pt_t*)realloc(g_pts, sizeof(pt_t) * (size_t)g_cap);
  }
  pt_t* p = &g_pts[g_npts++];
  p->n2 = 0;
  for (int c = 0; c < 8; ++c) {
    p->v[c] = v[c];
    p->n2 += v[c] * v[c];
  }
}
static int64_t isqrt_floor(int64_t r) {
  if (r < 0) return -1;
  int64_t s = (int64_t)sqrt((double)r);
  while (s * s > r) --s;
  while ((s + 1) * (s + 1) <= r) ++s;
  return s;
}
/* enumerate_shell (codebook.cpp:162-184), mod4 = true. */
static void shell_rec(int64_t* cur, int pos, int odd, int64_t rem, int64_t sum) {
  if (pos == 8) {
    if (((sum % 4) + 4) % 4 == 0) push_pt(cur);
    return;
  }
  int64_t tmax = isqrt_floor(rem);
  if (odd) {
    if (tmax % 2 == 0) --tmax;
  } else {
    if (tmax % 2 != 0) --tmax;
  }
  for (int64_t t = -tmax; t <= tmax; t += 2) {
    cur[pos] = t;
    shell_rec(cur, pos + 1, odd, rem - t * t, sum + t);
  }
}
static int cmp_pt(const void* a, const void* b) {
  const pt_t* x = (const pt_t*)a;
  const pt_t* y = (const pt_t*)b;
  if (x->n2 != y->n2) return x->n2 < y->n2 ? -1 : 1;
  for (int c = 0; c < 8; ++c)
    if (x->v[c] != y->v[c]) return x->v[c] < y->v[c] ? -1 : 1;
  return 0;
}
static void build_e8_1bit(void) {
  int64_t r2 = 32, cur[8];
  for (;;) {
    g_npts = 0;
    shell_rec(cur, 0, 0, r2, 0);
    shell_rec(cur, 0, 1, r2, 0);
    if (g_npts >= 256) break;
    r2 *= 2;
  }
  qsort(g_pts, (size_t)g_npts, sizeof(pt_t), cmp_pt);
  for (int i = 0; i < 256; ++i)
    for (int c = 0; c < 8; ++c) g_e81[i][c] = 0.5 * (double)g_pts[i].v[c];
  free(g_pts);
  g_pts = NULL;
  g_cap = 0;
}

static void init_tables(void) {
  build_e8p_tables();
  build_e8_1bit();
}
static void ensure(void) { pthread_once(&g_once, init_tables); }

int oracle_e8p_tables(int8_t* doubled, uint8_t* odd_parity) {
  ensure();
  memcpy(doubled, g_doubled, sizeof g_doubled);
  memcpy(odd_parity, g_odd, sizeof g_odd);
  return OK;
}

/* e8p_decode (e8p.cpp:81-100). */
void oracle_e8p_decode(uint16_t word, double* out) {
  ensure();
  const unsigned idx = word >> 8;
  const unsigned sb = (word >> 1) & 0x7Fu;
  const double shift = (word & 1u) ? 0.25 : -0.25;
  double v[8];
  unsigned flips = 0;
  for (int c = 0; c < 8; ++c) v[c] = 0.5 * g_doubled[idx][c];
  for (unsigned j = 1; j <= 7; ++j)
    if ((sb >> (j - 1)) & 1u) {
      v[8 - j] = -v[8 - j];
      ++flips;
    }
  if ((flips & 1u) != g_odd[idx]) v[0] = -v[0];
  for (int c = 0; c < 8; ++c) out[c] = v[c] + shift;
}

int oracle_e8_1bit_table(double* out) {
  ensure();
  memcpy(out, g_e81, sizeof g_e81);
  return OK;
}

/* ------------------------------------------------------------------------ */
/* Hadamard: core/src/hadamard.cpp                                            */
/* ------------------------------------------------------------------------ */

static int64_t pow_mod(int64_t a, int64_t e, int64_t q) {
  int64_t r = 1;
  a %= q;
  while (e > 0) {
    if (e & 1) r = r * a % q;
    a = a * a % q;
    e >>= 1;
  }
  return r;
}
/* legendre (hadamard.cpp:24-30) */
static int legendre(int64_t a, int64_t q) {
  a %= q;
  if (a < 0) a += q;
  if (a == 0) return 0;
  return pow_mod(a, (q - 1) / 2, q) == 1 ? 1 : -1;
}

/* Fills out[q*q] (row-major +-1); returns 0 or E_SIZE.
 * Sylvester (hadamard.cpp:32-39), Paley I (:44-61), Paley II (:66-97),
 * registry {1,4,12,20,28} (:114-145), + 172 (extension). */
int oracle_hadamard_base(size_t q, int8_t* out) {
  if (q == 1) {
    out[0] = 1;
    return OK;
  }
  if (q == 4) {
    for (size_t i = 0; i < 4; ++i)
      for (size_t j = 0; j < 4; ++j) out[i * 4 + j] = (__builtin_popcountll(i & j) % 2 == 0) ? 1 : -1;
    return OK;
  }
  if (q == 12 || q == 20) {
    const int64_t p = (int64_t)q - 1;
    const size_t n = q;
    out[0] = 1;
    for (size_t j = 1; j < n; ++j) out[j] = 1;
    for (size_t i = 1; i < n; ++i) out[i * n] = -1;
    for (size_t i = 1; i < n; ++i)
      for (size_t j = 1; j < n; ++j)
        out[i * n + j] = (int8_t)(i == j ? 1 : legendre((int64_t)i - (int64_t)j, p));
    return OK;
  }
  if (q == 28) {
    const int64_t prime = 13;
    const size_t m = 14, n = 28;
    int8_t s[14 * 14];
    memset(s, 0, sizeof s);
    for (size_t j = 1; j < m; ++j) {
      s[j] = 1;
      s[j * m] = 1;
    }
    for (size_t i = 1; i < m; ++i)
      for (size_t j = 1; j < m; ++j)
        s[i * m + j] = (int8_t)(i == j ? 0 : legendre((int64_t)j - (int64_t)i, prime));
    for (size_t i = 0; i < m; ++i)
      for (size_t j = 0; j < m; ++j) {
        int8_t b[2][2];
        if (s[i * m + j] == 0) {
          b[0][0] = 1, b[0][1] = -1, b[1][0] = -1, b[1][1] = -1;
        } else {
          const int8_t v = s[i * m + j];
          b[0][0] = v, b[0][1] = v, b[1][0] = v, b[1][1] = (int8_t)-v;
        }
        for (int a = 0; a < 2; ++a)
          for (int c = 0; c < 2; ++c) out[(2 * i + a) * n + (2 * j + c)] = b[a][c];
      }
    return OK;
  }
  if (q == 172) {
    for (size_t r = 0; r < 172; ++r)
      for (size_t c = 0; c < 172; ++c)
        out[r * 172 + c] = ((oracle_had172_bits[r][c / 64] >> (c % 64)) & 1) ? -1 : 1;
    return OK;
  }
  return E_SIZE;
}

static const size_t kRegistry[] = {1, 4, 12, 20, 28, 172};

/* plan_hadamard (hadamard.cpp:156-168): largest power of two p dividing n,
 * reduced until q = n / p is in the registry. */
int oracle_plan_hadamard(size_t n, size_t* p_out, size_t* q_out) {
  if (n == 0) return E_SIZE;
  for (size_t p = (size_t)1 << __builtin_ctzll(n); p >= 1; p >>= 1) {
    const size_t q = n / p;
    for (size_t i = 0; i < sizeof kRegistry / sizeof kRegistry[0]; ++i)
      if (kRegistry[i] == q) {
        *p_out = p;
        *q_out = q;
        return OK;
      }
    if (p == 1) break;
  }
  return E_SIZE;
}

/* had_apply (hadamard.cpp:170-210). */
int oracle_had_apply(size_t n, double* x, int transpose) {
  size_t p, q;
  if (oracle_plan_hadamard(n, &p, &q) != OK) return E_SIZE;
  for (size_t len = 1; len < p; len <<= 1)
    for (size_t i = 0; i < p; i += len << 1)
      for (size_t k = i; k < i + len; ++k) {
        double* a = x + k * q;
        double* b = x + (k + len) * q;
        for (size_t j = 0; j < q; ++j) {
          const double u = a[j], v = b[j];
          a[j] = u + v;
          b[j] = u - v;
        }
      }
  const double scale = 1.0 / sqrt((double)n);
  if (q == 1) {
    for (size_t i = 0; i < n; ++i) x[i] *= scale;
    return OK;
  }
  int8_t* base = (int8_t*)malloc(q * q);
  double* tmp = (double*)malloc(q * sizeof(double));
  oracle_hadamard_base(q, base);
  for (size_t r = 0; r < p; ++r) {
    double* seg = x + r * q;
    for (size_t a = 0; a < q; ++a) {
      double acc = 0.0;
      const int8_t* row = base + (transpose ? a : a * q);
      if (transpose)
        for (size_t b = 0; b < q; ++b) acc += row[b * q] * seg[b];
      else
        for (size_t b = 0; b < q; ++b) acc += row[b] * seg[b];
      tmp[a] = acc * scale;
    }
    memcpy(seg, tmp, q * sizeof(double));
  }
  free(base);
  free(tmp);
  return OK;
}

/* SignVector::apply (bitpack.cpp:36-40): x[i] = -x[i] where bit i (LSB-first) set. */
static void sign_apply(const uint8_t* bytes, size_t n, double* x) {
  for (size_t i = 0; i < n; ++i)
    if ((bytes[i >> 3] >> (i & 7)) & 1) x[i] = -x[i];
}

/* SideTransform::apply (transforms.cpp:28-36) / apply_transpose (:38-47), rht. */
int oracle_side_apply(size_t n, const uint8_t* sign_bytes, double* x, int transpose) {
  int st;
  if (!transpose) {
    sign_apply(sign_bytes, n, x);
    return oracle_had_apply(n, x, 0);
  }
  if ((st = oracle_had_apply(n, x, 1)) != OK) return st;
  sign_apply(sign_bytes, n, x);
  return OK;
}

/* rfft_apply (core/src/rfft.cpp:39-71): pairs (x[2k], x[2k+1]) as complex
 * c_k; forward: c_k *= e^{i theta_k}, unnormalized forward DFT of length
 * M = n/2 (FFTW_FORWARD, exponent -2 pi i jk/M), then * 1/sqrt(M); transpose:
 * unnormalized backward DFT, then * (1/sqrt(M)) e^{-i theta_k}.  FFTW3 (the
 * reference's dependency, version unpinned, absent here) is restated by the
 * DFT definition, computed directly in double (O(M^2)); the reference
 * compiled against oracle/shim/fftw3.h runs the same formula. */
static void dft_direct(size_t M, double* re, double* im, int sign) {
  const double two_pi = 6.283185307179586476925286766559;
  double* c = (double*)malloc(M * sizeof(double));
  double* s = (double*)malloc(M * sizeof(double));
  double* r0 = (double*)malloc(M * sizeof(double));
  double* i0 = (double*)malloc(M * sizeof(double));
  for (size_t e = 0; e < M; ++e) {
    const double a = two_pi * (double)e / (double)M;
    c[e] = cos(a);
    s[e] = (double)sign * sin(a);
  }
  memcpy(r0, re, M * sizeof(double));
  memcpy(i0, im, M * sizeof(double));
  for (size_t k = 0; k < M; ++k) {
    double ar = 0.0, ai = 0.0;
    size_t e = 0; /* j k mod M */
    for (size_t j = 0; j < M; ++j) {
      ar += r0[j] * c[e] - i0[j] * s[e];
      ai += r0[j] * s[e] + i0[j] * c[e];
      e += k;
      if (e >= M) e -= M;
    }
    re[k] = ar;
    im[k] = ai;
  }
  free(c);
  free(s);
  free(r0);
  free(i0);
}

int oracle_rfft_apply(size_t n, const double* phases, double* x, int transpose) {
  if (n == 0 || n % 2 != 0) return E_SIZE;
  const size_t M = n / 2;
  double* re = (double*)malloc(M * sizeof(double));
  double* im = (double*)malloc(M * sizeof(double));
  for (size_t k = 0; k < M; ++k) {
    re[k] = x[2 * k];
    im[k] = x[2 * k + 1];
  }
  const double scale = 1.0 / sqrt((double)M);
  if (!transpose) {
    for (size_t k = 0; k < M; ++k) { /* buf[k] *= polar(1, theta) */
      const double pc = cos(phases[k]), ps = sin(phases[k]);
      const double r = re[k] * pc - im[k] * ps, i = re[k] * ps + im[k] * pc;
      re[k] = r;
      im[k] = i;
    }
    dft_direct(M, re, im, -1);
    for (size_t k = 0; k < M; ++k) {
      re[k] *= scale;
      im[k] *= scale;
    }
  } else {
    dft_direct(M, re, im, +1);
    for (size_t k = 0; k < M; ++k) { /* buf[k] *= scale * polar(1, -theta) */
      const double pc = scale * cos(-phases[k]), ps = scale * sin(-phases[k]);
      const double r = re[k] * pc - im[k] * ps, i = re[k] * ps + im[k] * pc;
      re[k] = r;
      im[k] = i;
    }
  }
  for (size_t k = 0; k < M; ++k) {
    x[2 * k] = re[k];
    x[2 * k + 1] = im[k];
  }
  free(re);
  free(im);
  return OK;
}

/* ------------------------------------------------------------------------ */
/* QSHP v1 parse: core/src/pipeline.cpp:323-383                              */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint32_t m, n;
  int stages;
  int kind[8]; /* 0 = e8p-2bit, 1 = e8-1bit */
  double scale[8];
  int transform; /* 0 = rht, 1 = rfft */
  const uint8_t* sign_u;
  const uint8_t* sign_v;
  const uint8_t* phase_u; /* rfft: m/2 f32 angles (LE) */
  const uint8_t* phase_v; /* rfft: n/2 f32 angles */
  const uint8_t* codes[8];
} art_t;

static int parse(const uint8_t* b, size_t len, art_t* a) {
  size_t pos = 0;
#define TAKE(k)                           \
  do {                                    \
    if (pos + (k) > len) return E_TRUNC;  \
  } while (0)
  TAKE(4);
  if (memcmp(b, "QSHP", 4) != 0) return E_BADMAGIC;
  pos = 4;
  TAKE(2);
  if ((b[4] | (b[5] << 8)) != 1) return E_VERSION;
  pos = 6;
  TAKE(10);
  memcpy(&a->m, b + 6, 4);
  memcpy(&a->n, b + 10, 4);
  const uint8_t kind = b[14];
  if (kind > 1) return E_FORMAT;
  a->stages = b[15];
  pos = 16;
  if (a->stages == 0) return E_FORMAT;
  if (a->stages > 8) return E_VALIDATION;
  for (int s = 0; s < a->stages; ++s) {
    TAKE(1);
    const size_t idl = b[pos++];
    TAKE(idl);
    if (idl == 8 && memcmp(b + pos, "e8p-2bit", 8) == 0)
      a->kind[s] = 0;
    else if (idl == 7 && memcmp(b + pos, "e8-1bit", 7) == 0)
      a->kind[s] = 1;
    else
      return E_VALIDATION; /* other codebooks are not on this path */
    pos += idl;
    TAKE(4);
    float f;
    memcpy(&f, b + pos, 4);
    a->scale[s] = (double)f;
    pos += 4;
  }
  a->transform = kind;
  if (kind == 0) {
    TAKE((a->m + 7) / 8);
    a->sign_u = b + pos;
    pos += (a->m + 7) / 8;
    TAKE((a->n + 7) / 8);
    a->sign_v = b + pos;
    pos += (a->n + 7) / 8;
  } else { /* read_phases (pipeline.cpp:259-265, 353-357) */
    if (a->m % 2 != 0 || a->n % 2 != 0) return E_FORMAT;
    TAKE((size_t)a->m / 2 * 4);
    a->phase_u = b + pos;
    pos += (size_t)a->m / 2 * 4;
    TAKE((size_t)a->n / 2 * 4);
    a->phase_v = b + pos;
    pos += (size_t)a->n / 2 * 4;
  }
  if (a->n % 8 != 0) return E_FORMAT;
  const size_t words = (size_t)a->m * (a->n / 8);
  for (int s = 0; s < a->stages; ++s) {
    const size_t bytes = a->kind[s] == 0 ? 2 : 1;
    TAKE(words * bytes);
    a->codes[s] = b + pos;
    pos += words * bytes;
  }
  if (pos != len) return E_FORMAT;
  return OK;
#undef TAKE
}

/* f32 phases widened to double (PhaseVector keeps f32-exact angles). */
static double* phases_of(const uint8_t* p, size_t count) {
  double* out = (double*)malloc((count ? count : 1) * sizeof(double));
  for (size_t k = 0; k < count; ++k) {
    float f;
    memcpy(&f, p + 4 * k, 4);
    out[k] = (double)f;
  }
  return out;
}

int oracle_artifact_info(const uint8_t* b, size_t len, uint32_t* m, uint32_t* n, int* stages) {
  art_t a;
  const int st = parse(b, len, &a);
  if (st) return st;
  *m = a.m;
  *n = a.n;
  *stages = a.stages;
  return OK;
}

/* ------------------------------------------------------------------------ */
/* infer: core/src/pipeline.cpp:151-197                                      */
/* ------------------------------------------------------------------------ */

static inline uint16_t code_at(const art_t* a, int s, size_t i) {
  return a->kind[s] == 0 ? (uint16_t)(a->codes[s][2 * i] | (a->codes[s][2 * i + 1] << 8))
                         : (uint16_t)a->codes[s][i];
}
static inline void decode_at(const art_t* a, int s, uint16_t w, double* pt) {
  if (a->kind[s] == 0)
    oracle_e8p_decode(w, pt);
  else
    for (int c = 0; c < 8; ++c) pt[c] = g_e81[w][c];
}

/* z[r] for rows [r0, r1): the decode-accumulate-dot loop (pipeline.cpp:172-191). */
static void rows_dot(const art_t* a, const double* t, double* z, size_t r0, size_t r1) {
  const size_t nb = a->n / 8;
  double point[8], block[8];
  for (size_t r = r0; r < r1; ++r) {
    double acc = 0.0;
    for (size_t k = 0; k < nb; ++k) {
      for (int c = 0; c < 8; ++c) block[c] = 0.0;
      for (int s = 0; s < a->stages; ++s) {
        decode_at(a, s, code_at(a, s, r * nb + k), point);
        for (int c = 0; c < 8; ++c) block[c] += a->scale[s] * point[c];
      }
      const double* tv = t + k * 8;
      for (int c = 0; c < 8; ++c) acc += block[c] * tv[c];
    }
    z[r] = acc;
  }
}

typedef struct {
  const art_t* a;
  const double* t;
  double* z;
  size_t r0, r1;
} job_t;
static void* job_run(void* p) {
  job_t* j = (job_t*)p;
  rows_dot(j->a, j->t, j->z, j->r0, j->r1);
  return NULL;
}

/* y[i] = infer(a, x[i]) for count vectors (row-major count x n -> count x m).
 * threads > 1 splits the row loop of each vector (per-row arithmetic and
 * hence results are unchanged). */
int oracle_infer(const uint8_t* qshp, size_t len, const double* x, int count, double* y, int threads) {
  ensure();
  art_t a;
  int st = parse(qshp, len, &a);
  if (st) return st;
  size_t p, q;
  double *ph_u = NULL, *ph_v = NULL;
  if (a.transform == 0) {
    if (oracle_plan_hadamard(a.n, &p, &q) || oracle_plan_hadamard(a.m, &p, &q)) return E_SIZE;
  } else {
    ph_u = phases_of(a.phase_u, a.m / 2);
    ph_v = phases_of(a.phase_v, a.n / 2);
  }
  double* t = (double*)malloc(sizeof(double) * a.n);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  for (int i = 0; i < count; ++i) {
    memcpy(t, x + (size_t)i * a.n, sizeof(double) * a.n);
    if (a.transform == 0)
      oracle_side_apply(a.n, a.sign_v, t, 0); /* t = T_v x */
    else
      oracle_rfft_apply(a.n, ph_v, t, 0);
    double* z = y + (size_t)i * a.m;
    if (threads == 1) {
      rows_dot(&a, t, z, 0, a.m);
    } else {
      pthread_t th[256];
      job_t jobs[256];
      for (int k = 0; k < threads; ++k) {
        jobs[k] = (job_t){&a, t, z, (size_t)a.m * k / threads, (size_t)a.m * (k + 1) / threads};
        pthread_create(&th[k], NULL, job_run, &jobs[k]);
      }
      for (int k = 0; k < threads; ++k) pthread_join(th[k], NULL);
    }
    if (a.transform == 0)
      oracle_side_apply(a.m, a.sign_u, z, 1); /* y = T_u^T z */
    else
      oracle_rfft_apply(a.m, ph_u, z, 1);
  }
  free(t);
  free(ph_u);
  free(ph_v);
  return OK;
}

/* Unscaled incoherent-domain decode of one stage -> row-major m x n (f64). */
int oracle_decode_stage(const uint8_t* qshp, size_t len, int stage, double* w) {
  ensure();
  art_t a;
  int st = parse(qshp, len, &a);
  if (st) return st;
  if (stage < 0 || stage >= a.stages) return E_VALIDATION;
  const size_t nb = a.n / 8;
  for (size_t r = 0; r < a.m; ++r)
    for (size_t k = 0; k < nb; ++k) decode_at(&a, stage, code_at(&a, stage, r * nb + k), w + r * a.n + k * 8);
  return OK;
}
