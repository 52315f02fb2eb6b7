// Real-basis Clebsch–Gordan table (host), the CG operand of the cfg4 tensor
// product (BASELINE.json configs[3]; no reference counterpart — the
// reference corpus uses random CG tensors, acceptance.cpp:147). Paths
// (l1, l2, l3) with |l1-l2| <= l3 <= l1+l2 and l1+l2+l3 even (the parity
// rule for 0e+1o+2e+3o x spherical harmonics), ordered by (l1, l2, l3);
// entries (i = l3^2+m3, j = l1^2+m1, k = l2^2+m2, path, value) with
// |value| > 1e-12. Complex CG by the Racah formula, then the standard
// complex -> real spherical-harmonic basis change.
#include <cmath>
#include <complex>
#include <vector>

#include "ixb_internal.h"

namespace {

double lfact(int n) { return std::lgamma(static_cast<double>(n) + 1.0); }

double cg_complex(int l1, int m1, int l2, int m2, int l3, int m3) {
  if (m1 + m2 != m3 || std::abs(m1) > l1 || std::abs(m2) > l2 || std::abs(m3) > l3) return 0.0;
  if (l3 < std::abs(l1 - l2) || l3 > l1 + l2) return 0.0;
  const double pre = 0.5 * (std::log(2.0 * l3 + 1.0) + lfact(l3 + l1 - l2) + lfact(l3 - l1 + l2) +
                            lfact(l1 + l2 - l3) - lfact(l1 + l2 + l3 + 1) + lfact(l3 + m3) +
                            lfact(l3 - m3) + lfact(l1 - m1) + lfact(l1 + m1) + lfact(l2 - m2) +
                            lfact(l2 + m2));
  double sum = 0.0;
  for (int k = 0; k <= l1 + l2 + l3; ++k) {
    const int a = l1 + l2 - l3 - k, b = l1 - m1 - k, c = l2 + m2 - k, d = l3 - l2 + m1 + k,
              e = l3 - l1 - m2 + k;
    if (a < 0 || b < 0 || c < 0 || d < 0 || e < 0) continue;
    const double t = -(lfact(k) + lfact(a) + lfact(b) + lfact(c) + lfact(d) + lfact(e));
    sum += ((k & 1) ? -1.0 : 1.0) * std::exp(pre + t);
  }
  return sum;
}

// U[r][mu]: real_r = sum_mu U[r][mu] complex_mu, r = m + l, mu = m' + l.
std::vector<std::complex<double>> real_basis(int l) {
  const int n = 2 * l + 1;
  std::vector<std::complex<double>> U(static_cast<size_t>(n * n));
  const double s = 1.0 / std::sqrt(2.0);
  for (int m = -l; m <= l; ++m) {
    const int r = m + l;
    if (m == 0) {
      U[r * n + l] = 1.0;
    } else if (m > 0) {
      U[r * n + (-m + l)] = s;
      U[r * n + (m + l)] = (m & 1) ? -s : s;
    } else {
      const int am = -m;
      U[r * n + (m + l)] = std::complex<double>(0.0, s);
      U[r * n + (am + l)] = std::complex<double>(0.0, (am & 1) ? s : -s);
    }
  }
  return U;
}

}  // namespace

extern "C" int ixb_cg_table(int l_max, int32_t* ci, int32_t* cj, int32_t* ck, int32_t* cl,
                            float* cv, int64_t* count, int32_t* npaths) {
  return ixb_guard([&] {
    if (l_max < 0 || l_max > 8) ixb::fail(IXB_SHAPE, "ixb_cg_table: l_max must be in [0, 8]");
    int64_t cnt = 0;
    int path = 0;
    for (int l1 = 0; l1 <= l_max; ++l1) {
      for (int l2 = 0; l2 <= l_max; ++l2) {
        for (int l3 = 0; l3 <= l_max; ++l3) {
          if (l3 < std::abs(l1 - l2) || l3 > l1 + l2 || ((l1 + l2 + l3) & 1)) continue;
          const int n1 = 2 * l1 + 1, n2 = 2 * l2 + 1, n3 = 2 * l3 + 1;
          const auto U1 = real_basis(l1), U2 = real_basis(l2), U3 = real_basis(l3);
          for (int c = 0; c < n3; ++c) {
            for (int a = 0; a < n1; ++a) {
              for (int b = 0; b < n2; ++b) {
                std::complex<double> acc = 0.0;
                for (int m1 = -l1; m1 <= l1; ++m1) {
                  for (int m2 = -l2; m2 <= l2; ++m2) {
                    const int m3 = m1 + m2;
                    if (std::abs(m3) > l3) continue;
                    const double g = cg_complex(l1, m1, l2, m2, l3, m3);
                    if (g == 0.0) continue;
                    acc += g * U3[c * n3 + m3 + l3] * std::conj(U1[a * n1 + m1 + l1]) *
                           std::conj(U2[b * n2 + m2 + l2]);
                  }
                }
                if (std::fabs(acc.real()) > 1e-12) {
                  if (ci) {
                    ci[cnt] = l3 * l3 + c;
                    cj[cnt] = l1 * l1 + a;
                    ck[cnt] = l2 * l2 + b;
                    cl[cnt] = path;
                    cv[cnt] = static_cast<float>(acc.real());
                  }
                  ++cnt;
                }
              }
            }
          }
          ++path;
        }
      }
    }
    *count = cnt;
    if (npaths) *npaths = path;
  });
}
