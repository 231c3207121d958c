// Minimal FFTW3 API shim for compiling the UNMODIFIED reference rfft.cpp
// (proj/core/src/rfft.cpp) in the oracle build.  TEST INFRASTRUCTURE ONLY.
//
// FFTW3 (the reference's dependency, unpinned version; absent from this
// image) computes the unnormalized DFT
//     out[k] = sum_j in[j] * exp(sign * 2 pi i j k / n),  sign = FFTW_FORWARD (-1) or FFTW_BACKWARD (+1).
// This shim computes exactly that definition directly (O(n^2), double,
// twiddles exp(sign 2 pi i e / n) with e = j k mod n from a per-plan table),
// so results agree with FFTW to rounding (~1e-15 relative), not bit for bit.
// Only the entry points rfft.cpp uses are provided.
#pragma once

#include <cmath>
#include <cstring>
#include <vector>

typedef double fftw_complex[2];

struct q8p_fftw_plan_s {
  int n;
  std::vector<double> c, s;  // cos / (sign * sin) of 2 pi e / n
};
typedef q8p_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

inline fftw_plan fftw_plan_dft_1d(int n, fftw_complex*, fftw_complex*, int sign, unsigned) {
  if (n <= 0) return nullptr;
  auto* p = new q8p_fftw_plan_s{n, std::vector<double>(n), std::vector<double>(n)};
  const double two_pi = 6.283185307179586476925286766559;
  for (int e = 0; e < n; ++e) {
    const double a = two_pi * double(e) / double(n);
    p->c[e] = std::cos(a);
    p->s[e] = double(sign) * std::sin(a);
  }
  return p;
}

inline void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  const std::size_t n = std::size_t(p->n);
  std::vector<double> re(n), im(n);
  for (std::size_t j = 0; j < n; ++j) {
    re[j] = in[j][0];
    im[j] = in[j][1];
  }
  for (std::size_t k = 0; k < n; ++k) {
    double ar = 0.0, ai = 0.0;
    std::size_t e = 0;  // j k mod n
    for (std::size_t j = 0; j < n; ++j) {
      ar += re[j] * p->c[e] - im[j] * p->s[e];
      ai += re[j] * p->s[e] + im[j] * p->c[e];
      e += k;
      if (e >= n) e -= n;
    }
    out[k][0] = ar;
    out[k][1] = ai;
  }
}
