// tables.cpp — see tables.hpp
#include "tables.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>

#include "common.hpp"

namespace hfmm_b200 {

namespace {
constexpr long double kPiL = 3.14159265358979323846264338327950288L;

long double factorial_ld(int n) {
  static long double tab[128];
  static bool ready = [] {
    tab[0] = 1;
    for (int i = 1; i < 128; ++i) tab[i] = tab[i - 1] * i;
    return true;
  }();
  (void)ready;
  return tab[n];
}
}  // namespace

long double double_factorial(int n) {  // n odd, n >= -1
  long double r = 1;
  for (int j = n; j > 1; j -= 2) r *= j;
  return r;
}

// ascending series below 1 (alternating terms shrink from the first), Miller's downward
// recurrence normalised by j_0 above — the two regimes of reference src/special.cpp:16-54
void sph_jn_ld(int nmax, long double z, long double* out) {
  if (fabsl(z) < 1.0L) {
    const long double h = 0.5L * z * z;
    long double zn = 1, df = 1;
    for (int n = 0; n <= nmax; ++n) {
      long double term = 1, sum = 1;
      for (int j = 1; j < 60; ++j) {
        term *= -h / ((long double)j * (2 * n + 2 * j + 1));
        sum += term;
        if (fabsl(term) < 1e-22L * fabsl(sum)) break;
      }
      out[n] = zn / df * sum;
      zn *= z;
      df *= (2 * n + 3);
    }
    return;
  }
  const int start = nmax + 24 + int(fabsl(z));
  long double above = 0, cur = 1e-40L;
  std::vector<long double> keep(nmax + 1);
  for (int n = start; n >= 0; --n) {
    const long double below = (2.0L * n + 3.0L) / z * cur - above;
    above = cur;
    cur = below;
    if (n <= nmax) keep[n] = cur;
    if (fabsl(cur) > 1e2000L) {
      cur *= 1e-2000L;
      above *= 1e-2000L;
      for (int i = std::min(n, nmax); i <= nmax; ++i) keep[i] *= 1e-2000L;
    }
  }
  const long double scale = (sinl(z) / z) / cur;
  for (int n = 0; n <= nmax; ++n) out[n] = keep[n] * scale;
}

// hhat_n = h_n(z) z^{n+1} / (2n-1)!!  obeys  hhat_{n+1} = hhat_n - z^2/((2n+1)(2n-1)) hhat_{n-1}
// (the upward recurrence of reference src/special.cpp:56-65 in overflow-free form)
void sph_hn_scaled(int nmax, double z, double* re, double* im) {
  const std::complex<long double> e = std::polar(1.0L, (long double)z);
  std::complex<long double> h0 = std::complex<long double>(0, -1) * e;          // h_0 z
  std::complex<long double> h1 = -e * std::complex<long double>(z, 1);           // h_1 z^2
  re[0] = double(h0.real());
  im[0] = double(h0.imag());
  if (nmax == 0) return;
  re[1] = double(h1.real());
  im[1] = double(h1.imag());
  const long double z2 = (long double)z * z;
  for (int n = 1; n < nmax; ++n) {
    const std::complex<long double> hn = h1 - z2 / ((2.0L * n + 1) * (2.0L * n - 1)) * h0;
    h0 = h1;
    h1 = hn;
    re[n + 1] = double(hn.real());
    im[n + 1] = double(hn.imag());
  }
}

// the same two functions for a complex argument (complex wavenumber k = k_r + i k_i,
// reference src/special.cpp:16-65 takes cplx z throughout)
using cld = std::complex<long double>;
void sph_jn_cld(int nmax, cld z, cld* out) {
  if (std::abs(z) < 1.0L) {
    const cld h = 0.5L * z * z;
    cld zn = 1;
    long double df = 1;
    for (int n = 0; n <= nmax; ++n) {
      cld term = 1, sum = 1;
      for (int j = 1; j < 60; ++j) {
        term *= -h / ((long double)j * (2 * n + 2 * j + 1));
        sum += term;
        if (std::abs(term) < 1e-22L * std::abs(sum)) break;
      }
      out[n] = zn / df * sum;
      zn *= z;
      df *= (2 * n + 3);
    }
    return;
  }
  const int start = nmax + 24 + int(std::abs(z));
  cld above = 0, cur = 1e-40L;
  std::vector<cld> keep(nmax + 1);
  for (int n = start; n >= 0; --n) {
    const cld below = (2.0L * n + 3.0L) / z * cur - above;
    above = cur;
    cur = below;
    if (n <= nmax) keep[n] = cur;
    if (std::abs(cur) > 1e2000L) {
      cur *= 1e-2000L;
      above *= 1e-2000L;
      for (int i = std::min(n, nmax); i <= nmax; ++i) keep[i] *= 1e-2000L;
    }
  }
  const cld scale = (std::sin(z) / z) / cur;
  for (int n = 0; n <= nmax; ++n) out[n] = keep[n] * scale;
}
// hhat_n = h_n(z) z^{n+1} / (2n-1)!!, complex z
void sph_hn_scaled_cld(int nmax, cld z, cld* out) {
  const cld e = std::exp(cld(0, 1) * z);
  cld h0 = cld(0, -1) * e;          // h_0 z
  cld h1 = -e * (z + cld(0, 1));    // h_1 z^2
  out[0] = h0;
  if (nmax == 0) return;
  out[1] = h1;
  const cld z2 = z * z;
  for (int n = 1; n < nmax; ++n) {
    const cld hn = h1 - z2 / ((2.0L * n + 1) * (2.0L * n - 1)) * h0;
    h0 = h1;
    h1 = hn;
    out[n + 1] = hn;
  }
}

// Racah's single-sum formula with log-factorials (as reference src/special.cpp:126-155)
double wigner3j(int j1, int j2, int j3, int m1, int m2, int m3) {
  if (m1 + m2 + m3 != 0) return 0;
  if (j3 < std::abs(j1 - j2) || j3 > j1 + j2) return 0;
  if (std::abs(m1) > j1 || std::abs(m2) > j2 || std::abs(m3) > j3) return 0;
  auto lf = [](int n) { return lgammal((long double)n + 1); };
  const long double pre = 0.5L * (lf(j1 + j2 - j3) + lf(j1 - j2 + j3) + lf(-j1 + j2 + j3) -
                                  lf(j1 + j2 + j3 + 1) + lf(j1 + m1) + lf(j1 - m1) + lf(j2 + m2) +
                                  lf(j2 - m2) + lf(j3 + m3) + lf(j3 - m3));
  const int lo = std::max({0, j2 - j3 - m1, j1 - j3 + m2});
  const int hi = std::min({j1 + j2 - j3, j1 - m1, j2 + m2});
  long double sum = 0;
  for (int t = lo; t <= hi; ++t) {
    const long double den = lf(t) + lf(j1 + j2 - j3 - t) + lf(j1 - m1 - t) + lf(j2 + m2 - t) +
                            lf(j3 - j2 + m1 + t) + lf(j3 - j1 - m2 + t);
    const long double term = expl(pre - den);
    sum += (t & 1) ? -term : term;
  }
  const int ph = j1 - j2 - m3;
  return double((((ph % 2) + 2) % 2) ? -sum : sum);
}

// explicit (Wigner) sum; long double keeps the alternating sum clean up to n ~ 20
double wigner_d(int n, int mp, int m, double cos_beta) {
  const long double cb = std::clamp((long double)cos_beta, -1.0L, 1.0L);
  const long double c = sqrtl((1 + cb) / 2), s = sqrtl((1 - cb) / 2);
  const long double pre = sqrtl(factorial_ld(n + mp) * factorial_ld(n - mp) * factorial_ld(n + m) *
                                factorial_ld(n - m));
  long double sum = 0;
  for (int k = std::max(0, m - mp); k <= std::min(n + m, n - mp); ++k) {
    const int pc = 2 * n - 2 * k + m - mp, ps = 2 * k - m + mp;
    const long double term = powl(c, pc) * powl(s, ps) /
                             (factorial_ld(n + m - k) * factorial_ld(k) * factorial_ld(n - k - mp) *
                              factorial_ld(k - m + mp));
    sum += ((k - m + mp) & 1) ? -term : term;
  }
  return double(pre * sum);
}

void build_rotation_table(int order, double cos_theta, float* out) {
  // explicit Wigner sum with the powers of cos(beta/2), sin(beta/2) tabulated once
  const long double cb = std::clamp((long double)cos_theta, -1.0L, 1.0L);
  const long double c = sqrtl((1 + cb) / 2), s = sqrtl((1 - cb) / 2);
  std::vector<long double> cp(2 * order + 2), sp(2 * order + 2);
  cp[0] = sp[0] = 1;
  for (int i = 1; i <= 2 * order + 1; ++i) {
    cp[i] = cp[i - 1] * c;
    sp[i] = sp[i - 1] * s;
  }
  std::fill(out, out + rot_table_size(order), 0.0f);
  // 1 / i! and sqrt(i!) once per process (the sums below are multiplications only)
  static long double inv_fact[128], root_fact[128];
  static const bool ready = [] {
    for (int i = 0; i < 128; ++i) {
      inv_fact[i] = 1.0L / factorial_ld(i);
      root_fact[i] = sqrtl(factorial_ld(i));
    }
    return true;
  }();
  (void)ready;
  std::vector<long double> d;
  for (int n = 0; n <= order; ++n) {
    const int w = 2 * n + 1;
    d.assign(size_t(w) * w, 0.0L);  // d[(a+n)*w + (b+n)] = d^n_{a,b}; only b >= 0 is read below
    for (int a = -n; a <= n; ++a)
      for (int b = 0; b <= n; ++b) {
        const long double pre = root_fact[n + a] * root_fact[n - a] * root_fact[n + b] * root_fact[n - b];
        long double sum = 0;
        for (int k = std::max(0, b - a); k <= std::min(n + b, n - a); ++k) {
          const long double term = cp[2 * n - 2 * k + b - a] * sp[2 * k - b + a] * inv_fact[n + b - k] *
                                   inv_fact[k] * inv_fact[n - k - a] * inv_fact[k - b + a];
          sum += ((k - b + a) & 1) ? -term : term;
        }
        d[size_t(a + n) * w + (b + n)] = pre * sum;
      }
    auto D = [&](int a, int b) { return d[size_t(a + n) * w + (b + n)]; };
    // forward operator M_{r,k} = d_{k,r} (input k -> output r); a_{rk} = M_{r,k},
    // b'_{rk} = (-1)^k M_{r,-k} = (-1)^k d_{-k,r}
    float* plus = out + rot_block_offset(n);
    float* minus = out + rot_minus_offset(n);
    const int ps = rot_plus_stride(n), ms = rot_minus_stride(n);
    for (int k = 0; k <= n; ++k)
      for (int r = 0; r <= n; ++r) {
        const long double a = D(k, r), bp = ((k & 1) ? -1.0L : 1.0L) * D(-k, r);
        long double v;
        if (k == 0) v = r == 0 ? a : 2 * a;   // x_0 feeds y_0 once and u_r = y_r + yt_{-r} twice
        else if (r == 0) v = a;               // y_0 = a_00 x_0 + sum a_0k s_k
        else v = a + bp;
        plus[k * ps + r] = float(v);
        if (k >= 1 && r >= 1) minus[(k - 1) * ms + (r - 1)] = float(a - bp);
      }
  }
}

void unfold_rotation_block(int n, const float* table, double* out) {
  const int w = 2 * n + 1;
  const float* plus = table + rot_block_offset(n);
  const float* minus = table + rot_minus_offset(n);
  const int ps = rot_plus_stride(n), ms = rot_minus_stride(n);
  auto M = [&](int r, int k) -> double& { return out[size_t(k + n) * w + (r + n)]; };  // E[k][r]
  for (int k = 0; k <= n; ++k)
    for (int r = 0; r <= n; ++r) {
      const double sp_ = plus[k * ps + r];
      const double sm_ = (k >= 1 && r >= 1) ? minus[(k - 1) * ms + (r - 1)] : 0.0;
      double a, bp;
      if (k == 0) {
        a = r == 0 ? sp_ : sp_ / 2;
        bp = a;
      } else if (r == 0) {
        a = sp_;
        bp = a;
      } else {
        a = (sp_ + sm_) / 2;
        bp = (sp_ - sm_) / 2;
      }
      const double sk = (k & 1) ? -1.0 : 1.0, sr = (r & 1) ? -1.0 : 1.0;
      M(r, k) = a;
      if (k > 0) M(r, -k) = sk * bp;
      if (r > 0) M(-r, k) = sr * bp;
      if (r > 0 && k > 0) M(-r, -k) = sr * sk * a;
      if (r > 0 && k == 0) M(-r, 0) = sr * a;
    }
}

CoaxBuilder::CoaxBuilder(int order) : order_(order) {
  const int P = order;
  offset_.assign(size_t(P + 1) * (P + 1) * (P + 1) + 1, 0);
  for (int m = 0; m <= P; ++m)
    for (int nu = 0; nu <= P; ++nu)
      for (int n = 0; n <= P; ++n) {
        offset_[slot(m, nu, n)] = uint32_t(coef_.size());
        if (nu < m || n < m) continue;
        for (int lam = std::abs(n - nu); lam <= n + nu; lam += 2) {
          const double w0 = wigner3j(nu, lam, n, 0, 0, 0);
          const double wm = wigner3j(nu, lam, n, -m, 0, m);
          const int half = (nu + lam - n) / 2;
          const double sign = ((half + m) & 1) ? -1.0 : 1.0;
          coef_.push_back(sign * (2 * lam + 1) * std::sqrt(double(2 * nu + 1) * (2 * n + 1)) * w0 * wm);
        }
      }
  offset_.back() = uint32_t(coef_.size());
}

const CoaxBuilder& CoaxBuilder::shared(int order) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<CoaxBuilder>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = cache[order];
  if (!slot) slot = std::make_unique<CoaxBuilder>(order);
  return *slot;
}

size_t CoaxBuilder::slot(int m, int nu, int n) const {
  return (size_t(m) * (order_ + 1) + nu) * (order_ + 1) + n;
}

void CoaxBuilder::build(CoaxKind kind, double k, double dist, double s_src, double s_dst,
                        float* out, double k_imag) const {
  const int P = order_, lmax = 2 * P;
  // z = (k + i k_imag) dist.  The radial factors are kept in a form that cannot overflow:
  // rad[lam] * radscale(lam) = z_lam(z), radscale positive (|z| powers), phases inside rad
  const cld zc = cld((long double)k, (long double)k_imag) * (long double)dist;
  const long double z = std::abs(zc);
  std::vector<long double> rr(lmax + 1), ri(lmax + 1, 0.0L);
  if (k_imag == 0.0) {
    if (kind == CoaxKind::m2l) {
      std::vector<double> hr(lmax + 1), hi(lmax + 1);
      sph_hn_scaled(lmax, double(z), hr.data(), hi.data());
      for (int l = 0; l <= lmax; ++l) {
        rr[l] = hr[l];
        ri[l] = hi[l];
      }
    } else {
      sph_jn_ld(lmax, z, rr.data());
    }
  } else {
    std::vector<cld> rad(lmax + 1);
    if (kind == CoaxKind::m2l) {
      // h_lam = hhat_lam (2 lam - 1)!! / z^{lam+1}: the modulus of z^{lam+1} goes into the log scale
      // below, its phase stays here
      sph_hn_scaled_cld(lmax, zc, rad.data());
      const long double arg = std::arg(zc);
      for (int l = 0; l <= lmax; ++l) rad[l] *= std::polar(1.0L, -(l + 1) * arg);
    } else {
      sph_jn_cld(lmax, zc, rad.data());
    }
    for (int l = 0; l <= lmax; ++l) {
      rr[l] = rad[l].real();
      ri[l] = rad[l].imag();
    }
  }
  // positive scale multiplying A * rad, as a product of three factors (per lam, per nu, per n):
  //   M2L: (2 lam - 1)!! / z^{lam+1}  *  s_dst^nu / (2 nu - 1)!!  *  s_src^n / (2n + 1)!!
  //   M2M: 1                          *  (2 nu + 1)!! / s_dst^nu   *  s_src^n / (2n + 1)!!
  //   L2L: 1                          *  s_dst^nu / (2 nu - 1)!!  *  (2n - 1)!! / s_src^n
  // long double carries 15 bits of exponent: none of the factors can overflow or vanish for
  // orders <= kMaxOrder and the box sizes the gates admit (|log10| of a factor stays below ~200)
  std::vector<long double> f_lam(lmax + 1, 1.0L), f_nu(P + 1), f_n(P + 1);
  {
    long double zp = z, sd = 1.0L, ss = 1.0L;  // z^{lam+1}, s_dst^nu, s_src^n
    for (int lam = 0; lam <= lmax; ++lam) {
      if (kind == CoaxKind::m2l) f_lam[lam] = double_factorial(2 * lam - 1) / zp;
      zp *= z;
    }
    for (int j = 0; j <= P; ++j) {
      if (kind == CoaxKind::m2l) {
        f_nu[j] = sd / double_factorial(2 * j - 1);
        f_n[j] = ss / double_factorial(2 * j + 1);
      } else if (kind == CoaxKind::m2m) {
        f_nu[j] = double_factorial(2 * j + 1) / sd;
        f_n[j] = ss / double_factorial(2 * j + 1);
      } else {
        f_nu[j] = sd / double_factorial(2 * j - 1);
        f_n[j] = double_factorial(2 * j - 1) / ss;
      }
      sd *= (long double)s_dst;
      ss *= (long double)s_src;
    }
  }
  std::fill(out, out + 2 * size_t(coax_table_size(P)), 0.0f);
  for (int m = 0; m <= P; ++m)
    for (int n = m; n <= P; ++n)
      for (int nu = m; nu <= P; ++nu) {
        const int idx = coax_block_offset(P, m) + (n - m) * coax_row_stride(P, m) + (nu - m);
        const double* a = coef_.data() + offset_[slot(m, nu, n)];
        const long double fnn = f_nu[nu] * f_n[n];
        long double sr = 0, si = 0;
        int t = 0;
        for (int lam = std::abs(n - nu); lam <= n + nu; lam += 2, ++t) {
          const long double f = fnn * f_lam[lam] * a[t];
          sr += f * rr[lam];
          si += f * ri[lam];
        }
        out[2 * idx] = float(sr);
        out[2 * idx + 1] = float(si);
      }
}

void build_legendre_coefficients(int order, float* diag, float* sub, float* a, float* b) {
  for (int m = 0; m <= order; ++m) {
    diag[m] = m == 0 ? 0.0f : float(-std::sqrt((2.0 * m + 1.0) / (2.0 * m)));
    sub[m] = float(std::sqrt(2.0 * m + 3.0));
  }
  for (int n = 0; n <= order; ++n)
    for (int m = 0; m <= n; ++m) {
      const int i = n * (n + 1) / 2 + m;
      if (n < m + 2) {
        a[i] = b[i] = 0;
        continue;
      }
      const double den = double(n) * n - double(m) * m;
      a[i] = float(std::sqrt((4.0 * n * n - 1.0) / den));
      b[i] = float(std::sqrt(((2.0 * n + 1.0) * (n - 1.0 + m) * (n - 1.0 - m)) / ((2.0 * n - 3.0) * den)));
    }
  (void)kPiL;
}

}  // namespace hfmm_b200
